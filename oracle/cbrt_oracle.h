/*
 * TEST INFRASTRUCTURE — part of the CPU oracle (see oracle/README.md).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * use anything under oracle/.  Never linked into the product.
 *
 * The cube root used by the friction term (reference: np.cbrt at
 * /root/reference/pkg/src/blockswe/kernels.py:240-241).  numpy dispatches
 * np.cbrt to SVML on AVX-512 hosts and to libm elsewhere, so the reference's
 * own cbrt is host dependent and ~0.6 % of its results are 1 ulp off correct
 * rounding.  Parity is therefore pinned against a
 * "cbrt-aligned" reference: the reference run with np.cbrt replaced by this
 * function (tests/golden/make_golden.py).  The product's device cbrt
 * (paper_2408_07609_b200/csrc/cbrt.cuh) is an independent transcription of
 * the same algorithm; tests check host/device bitwise agreement and check
 * this function against exact rational arithmetic (it is correctly rounded
 * except within ~1e-10 ulp of a rounding midpoint).
 *
 * Algorithm (fma-exact, no libm):
 *   x = m 2^e, m in [1,2); e = 3q + r, r in {0,1,2}; t = m 2^r in [1,8)
 *   R0 = P7(m) * 2^(-r/3)          ~ t^(-1/3), |rel err| < 1.7e-7
 *   R  = R0 + R0 (1 - t R0^3) / 3   one Newton step, ~1e-13
 *   y  = (t R) R                    ~ t^(1/3)
 *   y  = y - (y^3 - t) R^2 / 3      residual with exact fma products
 *   cbrt(x) = y 2^q
 */
#ifndef CBRT_ORACLE_H
#define CBRT_ORACLE_H
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline double oracle_cbrt(double x)
{
    if (x != x) return x + x;
    if (x == 0.0 || isinf(x)) return x;
    if (x < 0.0) return -oracle_cbrt(-x);
    uint64_t b;
    memcpy(&b, &x, 8);
    int scale = 0;
    if ((b >> 52) == 0) {              /* subnormal: lift by 2^54 */
        x = x * 0x1p54;
        memcpy(&b, &x, 8);
        scale = -18;
    }
    int e = (int)(b >> 52) - 1023;
    uint64_t mb = (b & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
    double m;
    memcpy(&m, &mb, 8);
    int q = (e >= 0) ? e / 3 : -((-e + 2) / 3);
    int r = e - 3 * q;
    double t = m * (double)(1 << r);
    double p = -0x1.9975209200000p-8;
    p = fma(p, m, 0x1.36f21412b8c00p-4);
    p = fma(p, m, -0x1.9bda02c244c00p-2);
    p = fma(p, m, 0x1.378ae90591ba8p+0);
    p = fma(p, m, -0x1.283918219a43ep+1);
    p = fma(p, m, 0x1.704716488edf7p+1);
    p = fma(p, m, -0x1.34eeb196c1ab5p+1);
    p = fma(p, m, 0x1.f7574f9197f7cp+0);
    static const double c3[3] = {0x1.0p+0, 0x1.965fea53d6e3dp-1,
                                 0x1.428a2f98d728bp-1};
    const double third = 0x1.5555555555555p-2;
    double R = p * c3[r];
    double R3 = (R * R) * R;
    double en = fma(-t, R3, 1.0);
    R = fma(R * en, third, R);
    double y = (t * R) * R;
    double y2 = y * y;
    double y2l = fma(y, y, -y2);
    double res = fma(y2, y, -t);
    res = fma(y2l, y, res);
    y = y - (res * (R * R)) * third;
    uint64_t pb = (uint64_t)(q + scale + 1023) << 52;
    double p2;
    memcpy(&p2, &pb, 8);
    return y * p2;
}
#endif
