// Friction cube root, kernels.py:240-241 (np.cbrt(du)).
//
// np.cbrt is SVML on AVX-512 hosts and libm elsewhere, so the reference's
// value is host dependent.  The product defines cbrt once, as a correctly
// rounded (up to ~1e-10 ulp of a midpoint) fma-exact sequence that compiles
// identically for the host (ts_cbrt_host, the "host twin") and the device;
// the oracle's oracle_cbrt is an independent transcription of the same
// algorithm, and tests check all three bitwise plus against exact rationals.
//
// x = m 2^e, m in [1,2), e = 3q + r; t = m 2^r in [1,8)
// R ~ t^(-1/3): degree-7 polynomial in m times 2^(-r/3), one Newton step;
// y = (t R) R, then y -= (y^3 - t) R^2 / 3 with the residual from exact fma
// products; result y 2^q.  ~25 DP instructions, no divisions.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define TS_HD __host__ __device__ __forceinline__
#else
#define TS_HD inline
#endif

#if defined(__CUDA_ARCH__)
#define TS_FMA(a, b, c) __fma_rn((a), (b), (c))
#define TS_MUL(a, b) __dmul_rn((a), (b))
#define TS_ADD(a, b) __dadd_rn((a), (b))
TS_HD uint64_t ts_bits(double x) { return (uint64_t)__double_as_longlong(x); }
TS_HD double ts_from_bits(uint64_t b) { return __longlong_as_double((long long)b); }
#else
#include <cmath>
#include <cstring>
#define TS_FMA(a, b, c) std::fma((a), (b), (c))
#define TS_MUL(a, b) ((a) * (b))
#define TS_ADD(a, b) ((a) + (b))
TS_HD uint64_t ts_bits(double x) { uint64_t b; std::memcpy(&b, &x, 8); return b; }
TS_HD double ts_from_bits(uint64_t b) { double x; std::memcpy(&x, &b, 8); return x; }
#endif

// polynomial coefficients c7..c0, 2^(-r/3) for r = 0, 1, 2, and 1/3.  The
// device reads them from the constant bank (a DFMA operand) instead of
// rematerialising each 64-bit literal with two uniform moves per use.
#define TS_CBRT_TABLE                                                                 \
    -0x1.9975209200000p-8, 0x1.36f21412b8c00p-4, -0x1.9bda02c244c00p-2,                \
    0x1.378ae90591ba8p+0, -0x1.283918219a43ep+1, 0x1.704716488edf7p+1,                 \
    -0x1.34eeb196c1ab5p+1, 0x1.f7574f9197f7cp+0, 0x1.0p+0, 0x1.965fea53d6e3dp-1,       \
    0x1.428a2f98d728bp-1, 0x1.5555555555555p-2
#if defined(__CUDACC__)
static __constant__ double ts_cbrt_k_dev[12] = {TS_CBRT_TABLE};
#endif
static const double ts_cbrt_k_host[12] = {TS_CBRT_TABLE};
#if defined(__CUDA_ARCH__)
#define TS_CBRT_K(i) ts_cbrt_k_dev[i]
#else
#define TS_CBRT_K(i) ts_cbrt_k_host[i]
#endif

TS_HD double ts_cbrt_pos_normal(double x, int extra_exp)
{
    const uint64_t b = ts_bits(x);
    // e = 3q + r with q = floor(e / 3): k = e + 1200 >= 0 and floor(k / 3)
    // = (k * 21846) >> 16 for k < 32768 (integer ops only, no branch)
    const int k = (int)(b >> 52) - 1023 + 1200;
    const int qk = (k * 21846) >> 16;
    const int q = qk - 400, r = k - 3 * qk;
    const uint64_t mant = b & 0x000fffffffffffffULL;
    const double m = ts_from_bits(mant | 0x3ff0000000000000ULL);
    const double t = ts_from_bits(mant | ((uint64_t)(1023 + r) << 52));     // m * 2^r, exact
    double p = TS_CBRT_K(0);
    p = TS_FMA(p, m, TS_CBRT_K(1));
    p = TS_FMA(p, m, TS_CBRT_K(2));
    p = TS_FMA(p, m, TS_CBRT_K(3));
    p = TS_FMA(p, m, TS_CBRT_K(4));
    p = TS_FMA(p, m, TS_CBRT_K(5));
    p = TS_FMA(p, m, TS_CBRT_K(6));
    p = TS_FMA(p, m, TS_CBRT_K(7));
    const double c3 = TS_CBRT_K(8 + r);
    const double third = TS_CBRT_K(11);
    double R = TS_MUL(p, c3);
    const double R3 = TS_MUL(TS_MUL(R, R), R);
    const double en = TS_FMA(-t, R3, 1.0);
    R = TS_FMA(TS_MUL(R, en), third, R);
    double y = TS_MUL(TS_MUL(t, R), R);
    const double y2 = TS_MUL(y, y);
    const double y2l = TS_FMA(y, y, -y2);
    double res = TS_FMA(y2, y, -t);
    res = TS_FMA(y2l, y, res);
    y = TS_ADD(y, -TS_MUL(TS_MUL(res, TS_MUL(R, R)), third));
    return TS_MUL(y, ts_from_bits((uint64_t)(q + extra_exp + 1023) << 52));
}

TS_HD double ts_cbrt(double x)
{
    if (!(x > 0.0) || !(x < 0x1.fffffffffffffp+1023)) {
        // NaN, +-0, negatives, +-inf: cold path
        if (x != x) return x + x;
        if (x == 0.0 || x == 2.0 * x) return x;            // +-0, +-inf
        if (x < 0.0) {
            const double ax = -x;
            if (ax < 0x1p-1022) return -ts_cbrt_pos_normal(TS_MUL(ax, 0x1p54), -18);
            return -ts_cbrt_pos_normal(ax, 0);
        }
    }
    if (x < 0x1p-1022) return ts_cbrt_pos_normal(TS_MUL(x, 0x1p54), -18);
    return ts_cbrt_pos_normal(x, 0);
}
