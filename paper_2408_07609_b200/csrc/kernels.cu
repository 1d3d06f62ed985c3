// sm_100a kernels of the nested-grid shallow-water step.
//
// Numerics follow the reference's evaluation order exactly:
// the file is compiled with -fmad=false (no FMA contraction), IEEE / and
// sqrt (fastmath.cuh replays nvcc's own expansions), numpy maximum/sign
// semantics (np_max / np_sign), and the product's cbrt (cbrt.cuh).  The
// reference's stored "wet" flags are derived on the fly as h + eta >= thr,
// which equals the stored flag at every read site (checked by
// the parity tests against the oracle, which keeps the explicit array).
//
// Kernels:
//   k_mass      K_mass: continuity (kernels.py:123-155), fused with the
//               running-maxima fold of the previous step (kernels.py:322-343);
//               one CTA per tile, one thread per cell (memory-bound)
//   k_accum     standalone fold (end-of-run flush, kernel-level API)
//   k_momentum  K_mom: both flux components (kernels.py:158-271) in one
//               march down each tile's rows; face prelims computed once and
//               shared through registers (x) and a 3-row shared ring (y)
//   k_restrict  3x3 ring averages child -> parent (coupling.py:278-315)
//   k_prolong   parent face -> 3 child faces (coupling.py:318-340)
//   k_copy      halo strips (exchange.py:218-275) and edge BCs
//               (kernels.py:274-306) as deduplicated element copies
#include <cuda_runtime.h>
#include <stdint.h>

#include "cbrt.cuh"
#include "common.cuh"
#include "fastmath.cuh"

namespace {

constexpr int kFlatThreads = 256;

__device__ __forceinline__ bool stop_requested(const unsigned long long *err)
{
    __shared__ int s_stop;
    if (threadIdx.x == 0) s_stop = (*(volatile const unsigned long long *)err != TS_NO_ERROR);
    __syncthreads();
    return s_stop != 0;
}

__device__ __forceinline__ void report(unsigned long long *err, int order, int what, int i, int j)
{
    atomicMin(err, ts_err_key(order, what, i, j));
}

// ------------------------------------------------------------------ mass
// accumulate_outputs for one cell (kernels.py:327-343)
__device__ __forceinline__ void fold_cell(const DevBlock *B, size_t ac, double e, double h, double d,
                                          double Ml, double Mr, double Nl, double Nr, double thr)
{
    const bool w = d >= thr;
    const double mc = 0.5 * (Ml + Mr);
    const double nc = 0.5 * (Nl + Nr);
    const double ds = np_max(d, thr);
    bool ok = true;
    const TsRcp R = ts_rcp(ds);
    const double u = ts_div(mc, R, ok), v = ts_div(nc, R, ok);
    double sp = ts_sqrt(u * u + v * v, ok);
    if (!ok) {
        const double uu = mc / ds, vv = nc / ds;
        sp = sqrt(uu * uu + vv * vv);
    }
    if (w) {
        const double me = B->acc_eta[ac], nme = np_max(me, e);
        if (!(nme == me || (nme != nme && me != me))) B->acc_eta[ac] = nme;
        const double ms = B->acc_speed[ac], nms = np_max(ms, sp);
        if (!(nms == ms || (nms != nms && ms != ms))) B->acc_speed[ac] = nms;
        if (h < 0.0) {
            const double mi = B->acc_inund[ac], nmi = np_max(mi, d);
            if (!(nmi == mi || (nmi != nmi && mi != mi))) B->acc_inund[ac] = nmi;
        }
    }
}

// Cells of a tile: rows [i0, min(i1, ni)) x columns [j0, min(j1, nj)),
// visited as a flat index so each thread has several independent cells and
// all their loads in flight (the kernel is HBM-bound).
struct CellRange {
    int i0, j0, ncol, n;
    float inv;
};

__device__ __forceinline__ CellRange cell_range(const Tile &tl, int ni, int nj)
{
    CellRange c;
    c.i0 = tl.i0;
    c.j0 = tl.j0;
    c.ncol = min(tl.j1, nj) - tl.j0;
    const int nrow = min(tl.i1, ni) - tl.i0;
    c.n = (c.ncol > 0 && nrow > 0) ? c.ncol * nrow : 0;
    c.inv = c.ncol > 0 ? 1.0f / (float)c.ncol : 0.0f;
    return c;
}

// k -> (row, col) of the range; exact while k < 2^20 (tiles are far smaller)
__device__ __forceinline__ void cell_of(const CellRange &c, int k, int &i, int &j)
{
    const int di = __float2int_rz(((float)k + 0.5f) * c.inv);
    i = c.i0 + di;
    j = c.j0 + (k - di * c.ncol);
}

template <bool FOLD>
__global__ void __launch_bounds__(kFlatThreads)
k_mass(StepArgs a, const Tile *__restrict__ tiles)
{
    if (stop_requested(a.err)) return;
    const Tile tl = tiles[blockIdx.x];
    const DevBlock *B = a.blocks + tl.blk;
    const CellRange cr = cell_range(tl, B->ni, B->nj);
    const int P = B->P, cur = a.cur;
    const double *__restrict__ eo = B->eta[cur];
    double *__restrict__ en = B->eta[cur ^ 1];
    const double *__restrict__ mo = B->m[cur];
    const double *__restrict__ no = B->n[cur];
    const double *__restrict__ hh = B->h;
    const double r = B->r, thr = a.thr;
    const bool fold = FOLD && (*a.acc_flag != 0);
    const int order = B->order;
#pragma unroll 4
    for (int k = threadIdx.x; k < cr.n; k += kFlatThreads) {
        int i, j;
        cell_of(cr, k, i, j);
        const size_t row = (size_t)(i + TS_G) * P + j + TS_G;
        const double Mi = __ldg(mo + row), Mi1 = __ldg(mo + row + P);
        const double Nj = __ldg(no + row), Nj1 = __ldg(no + row + 1);
        const double e0 = __ldg(eo + row), h = __ldg(hh + row);
        const double d = h + e0;
        // accumulate_outputs of the previous step (kernels.py:322-343): its
        // eta_new/m_new/n_new are this step's old buffers
        if (fold) fold_cell(B, (size_t)i * P + j, e0, h, d, Mi, Mi1, Nj, Nj1, thr);
        // update_mass (kernels.py:134-155); wet_old derived as h + eta_old >= thr
        const double div = r * (Mi1 - Mi) + r * (Nj1 - Nj);
        double e = e0 - div;
        if (!(d >= thr) && div != 0.0) e = np_max(e0, -h) - div;
        if (div != 0.0 && h + e < 0.0) e = -h;
        if (!isfinite(e)) report(a.err, order, 0, i, j);
        en[row] = e;
    }
}

// ------------------------------------------------------ standalone fold
__global__ void __launch_bounds__(kFlatThreads)
k_accum(StepArgs a, const Tile *__restrict__ tiles)
{
    // a.cur names the buffer to read (the "new" role of kernels.py:327-335)
    const Tile tl = tiles[blockIdx.x];
    const DevBlock *B = a.blocks + tl.blk;
    const CellRange cr = cell_range(tl, B->ni, B->nj);
    const int P = B->P;
    const double *eta = B->eta[a.cur], *m = B->m[a.cur], *n = B->n[a.cur];
#pragma unroll 4
    for (int k = threadIdx.x; k < cr.n; k += kFlatThreads) {
        int i, j;
        cell_of(cr, k, i, j);
        const size_t row = (size_t)(i + TS_G) * P + j + TS_G;
        const double e = eta[row], h = B->h[row];
        fold_cell(B, (size_t)i * P + j, e, h, h + e, m[row], m[row + P], n[row], n[row + 1], a.thr);
    }
}

// -------------------------------------------------------------- momentum
// Face quantities of _momentum_axis (kernels.py:173-215) for one face with
// left/right cells (el, hl, Dl = hl + el) | (er, hr, Dr).
struct Face {
    double f0, qbar, dface, grad, dsafe, fa, fc;
    bool both, active;
};

__device__ __forceinline__ void face_geom(Face &F, double el, double er, double hl, double hr, double Dl,
                                          double Dr, double f0, double qbar, double thr)
{
    F.f0 = f0;
    F.qbar = qbar;
    const bool wl = Dl >= thr, wr = Dr >= thr;
    double df = 0.5 * (Dl + Dr);
    double gr = er - el;
    bool active = wl && wr;
    F.both = active;
    if (wl != wr) {
        if (wl) {                           // front_r (kernels.py:191-196)
            const double d_r = el + hr;
            active = d_r >= thr;
            df = d_r;
            gr = np_max(er, -hr) - el;
        } else {                            // front_l (kernels.py:197-202)
            const double d_l = er + hl;
            active = d_l >= thr;
            df = d_l;
            gr = er - np_max(el, -hl);
        }
    }
    F.dface = df;
    F.grad = gr;
    F.active = active;
    F.dsafe = np_max(df, thr);
}

// fadv = f0*f0/dsafe, fcross = f0*(qbar/dsafe): one shared reciprocal
__device__ __forceinline__ void face_flux(Face &F, bool &ok)
{
    const TsRcp R = ts_rcp(F.dsafe);
    F.fa = ts_div(F.f0 * F.f0, R, ok);
    F.fc = F.f0 * ts_div(F.qbar, R, ok);
}

__device__ __forceinline__ double face_adv(const Face &F, double fa_lo, double fa_hi, double fc_lo,
                                           double fc_hi)
{
    const double m0 = F.f0, q0 = F.qbar;
    double adv = 0.5 * ((fa_hi - fa_lo) - np_sign(m0) * ((fa_hi + fa_lo) - 2.0 * F.fa));
    adv = adv + 0.5 * ((fc_hi - fc_lo) - np_sign(q0) * ((fc_hi + fc_lo) - 2.0 * F.fc));
    return adv * (F.both ? 1.0 : 0.0);
}

// kernels.py:235-247: friction, numerator, semi-implicit divide
__device__ __forceinline__ double face_finish(const Face &F, double adv, double kfric, double r, double grr,
                                              bool &ok)
{
    const double m0 = F.f0, q0 = F.qbar, du = F.dsafe;
    const double s = ts_sqrt(m0 * m0 + q0 * q0, ok);
    const double den = du * du * ts_cbrt(du);
    const double fr = ts_div(kfric * s, ts_rcp(den), ok);
    const double numer = m0 - r * adv - grr * F.dface * F.grad;
    return ts_div(numer, ts_rcp(1.0 + fr), ok);
}

__device__ __noinline__ double face_finish_ieee(double m0, double q0, double du, double dface, double grad,
                                                double adv, double kfric, double r, double grr)
{
    const double fr = kfric * sqrt(m0 * m0 + q0 * q0) / (du * du * ts_cbrt(du));
    const double numer = m0 - r * adv - grr * dface * grad;
    return numer / (1.0 + fr);
}

// row r of column c as loaded (Mn/Mnl: M faces r+1 at columns c, c-1), plus
// D = h + eta computed once per cell
struct RowLd {
    double e, h, el, hl, Nc, Nc1, Mn, Mnl, D;
};

struct MomCtx {
    const double *eta, *hh, *mo, *no, *nman;
    double *mn, *nn;
    double *sFC, *sFA;                 // [3][NT] shared rings
    unsigned long long *err;
    double thr, r, grr, kf, dtg;
    int P, ni, nj, c, tid, i0, i1, order, NT;
    bool colM, colN, updM, updN, has_nman;
};

__device__ __forceinline__ void load_row(const MomCtx &X, int row, RowLd &L)
{
    const size_t rc = (size_t)(row + TS_G) * X.P + X.c + TS_G;
    L.e = __ldg(X.eta + rc);
    L.h = __ldg(X.hh + rc);
    L.el = __ldg(X.eta + rc - 1);
    L.hl = __ldg(X.hh + rc - 1);
    L.Nc = __ldg(X.no + rc);
    L.Nc1 = __ldg(X.no + rc + 1);
    L.Mn = __ldg(X.mo + rc + X.P);
    L.Mnl = __ldg(X.mo + rc + X.P - 1);
}

// One march step at row rr (iteration it): prelims of M face rr and N row
// rr from rows rr-1 (Lp) and rr (Lc), then the updates of M face rr-1 and
// N row rr-1 (their centre faces in FpM/FpN, FA_M/FC_N of row rr-2 in
// Fpp_M/Fpp_N).  Lf receives the prefetch of row rr+1; SLOT is the
// compile-time shared-ring slot of row rr.
template <int SLOT>
__device__ __forceinline__ void mom_step(const MomCtx &X, int it, const RowLd &Lp, RowLd &Lc, RowLd &Lf,
                                         const Face &Fpp_M, const Face &Fpp_N, const Face &FpM,
                                         const Face &FpN, Face &FcM, Face &FcN)
{
    constexpr int PSLOT = (SLOT + 2) % 3;
    const int rr = X.i0 - 1 + it;
    const bool rowOK = rr <= X.i1;
    if (X.colN && rr + 1 <= X.i1) load_row(X, rr + 1, Lf);
    Lc.D = Lc.h + Lc.e;
    // M face rr, column c: cells (rr-1, c) | (rr, c); Mc = M(rr, c) = Lp.Mn
    face_geom(FcM, Lp.e, Lc.e, Lp.h, Lc.h, Lp.D, Lc.D, Lp.Mn,
              0.25 * ((Lp.Nc + Lc.Nc) + (Lp.Nc1 + Lc.Nc1)), X.thr);
    // N face c of row rr: cells (rr, c-1) | (rr, c)
    face_geom(FcN, Lc.el, Lc.e, Lc.hl, Lc.h, Lc.hl + Lc.el, Lc.D, Lc.Nc,
              0.25 * ((Lp.Mnl + Lp.Mn) + (Lc.Mnl + Lc.Mn)), X.thr);
    bool ok = true;
    face_flux(FcM, ok);
    face_flux(FcN, ok);
    if (!ok) {
        FcM.fa = FcM.f0 * FcM.f0 / FcM.dsafe;
        FcM.fc = FcM.f0 * (FcM.qbar / FcM.dsafe);
        FcN.fa = FcN.f0 * FcN.f0 / FcN.dsafe;
        FcN.fc = FcN.f0 * (FcN.qbar / FcN.dsafe);
    }
    X.sFC[SLOT * X.NT + X.tid] = FcM.fc;
    X.sFA[SLOT * X.NT + X.tid] = FcN.fa;
    __syncthreads();
    if (it < 2) return;
    const int f = rr - 1;
    const bool dM = X.updM && f < X.i1 && rowOK;
    const bool dN = X.updN && f < X.i1 && f < X.ni && rowOK;
    const double advM = face_adv(FpM, Fpp_M.fa, FcM.fa, X.sFC[PSLOT * X.NT + X.tid - 1],
                                 X.sFC[PSLOT * X.NT + X.tid + 1]);
    const double advN = face_adv(FpN, X.sFA[PSLOT * X.NT + X.tid - 1], X.sFA[PSLOT * X.NT + X.tid + 1],
                                 Fpp_N.fc, FcN.fc);
    double kM = X.kf, kN = X.kf;
    const size_t fc = (size_t)(f + TS_G) * X.P + X.c + TS_G;
    if (X.has_nman && (dM || dN)) {
        const double nfM = 0.5 * (X.nman[fc - X.P] + X.nman[fc]);
        const double nfN = 0.5 * (X.nman[fc - 1] + X.nman[fc]);
        kM = X.dtg * nfM * nfM;
        kN = X.dtg * nfN * nfN;
    }
    bool okM = true, okN = true;
    double vM = face_finish(FpM, advM, kM, X.r, X.grr, okM);
    double vN = face_finish(FpN, advN, kN, X.r, X.grr, okN);
    if (!((okM || !FpM.active) && (okN || !FpN.active))) {
        vM = face_finish_ieee(FpM.f0, FpM.qbar, FpM.dsafe, FpM.dface, FpM.grad, advM, kM, X.r, X.grr);
        vN = face_finish_ieee(FpN.f0, FpN.qbar, FpN.dsafe, FpN.dface, FpN.grad, advN, kN, X.r, X.grr);
    }
    if (dM) {
        const double v = FpM.active ? vM : 0.0;
        if (!isfinite(v)) report(X.err, X.order, 1, f, X.c);
        X.mn[fc] = v;
    }
    if (dN) {
        const double v = FpN.active ? vN : 0.0;
        if (!isfinite(v)) report(X.err, X.order, 2, f, X.c);
        X.nn[fc] = v;
    }
}

// One thread per column c in [j0-1, j1] of a tile (W warps per tile, TPC
// tiles per CTA); the march visits rows r = i0-1 .. i0+T (T+2 a multiple of
// 3).  Unrolled by 3 so load buffers, face sets and shared-ring slots rotate
// by renaming only.
#ifndef TS_MOM_MINB
#define TS_MOM_MINB 1
#endif
template <int W, int TPC>
__global__ void __launch_bounds__(32 * W * TPC, TS_MOM_MINB)
k_momentum(StepArgs a, const Tile *__restrict__ tiles, int ntiles, int T)
{
    constexpr int NT = 32 * W * TPC;
    __shared__ double sFC[3 * NT];
    __shared__ double sFA[3 * NT];
    if (stop_requested(a.err)) return;
    const int tid = threadIdx.x;
    const int lt = tid / (32 * W), ci = tid % (32 * W);
    const int t = blockIdx.x * TPC + lt;
    const bool tv = t < ntiles;
    Tile tl;
    if (tv) tl = tiles[t];
    else tl = Tile{0, 0, 0, 0, 0, 0};
    const DevBlock *B = a.blocks + tl.blk;
    MomCtx X;
    X.ni = B->ni;
    X.nj = B->nj;
    X.P = B->P;
    X.c = tl.j0 - 1 + ci;
    const bool inTile = tv && X.c <= tl.j1;
    X.colM = inTile && X.c <= X.nj;               // M window columns -1..nj
    X.colN = inTile && X.c <= X.nj + 1;           // N window faces -1..nj+1
    X.updM = tv && X.c >= tl.j0 && X.c < tl.j1 && X.c < X.nj;
    X.updN = tv && X.c >= tl.j0 && X.c < tl.j1 && X.c <= X.nj;
    const int cur = a.cur;
    X.eta = B->eta[cur ^ 1];
    X.hh = B->h;
    X.mo = B->m[cur];
    X.no = B->n[cur];
    X.mn = B->m[cur ^ 1];
    X.nn = B->n[cur ^ 1];
    X.nman = B->nman;
    X.has_nman = B->has_nman != 0;
    X.thr = a.thr;
    X.r = B->r;
    X.grr = B->grr;
    X.kf = B->kf;
    X.dtg = B->dtg;
    X.order = B->order;
    X.err = a.err;
    X.sFC = sFC;
    X.sFA = sFA;
    X.tid = tid;
    X.NT = NT;
    X.i0 = tl.i0;
    X.i1 = tl.i1;

    RowLd L0{}, L1{}, L2{};
    Face A0{}, A1{}, A2{}, B0{}, B1{}, B2{};      // M / N face sets
    if (X.colN) {
        load_row(X, X.i0 - 2, L2);                // row i0-2 (prev of the first step)
        load_row(X, X.i0 - 1, L0);                // row i0-1 (first step)
    }
    L2.D = L2.h + L2.e;
    // step k: current row in L[k%3], prev in L[(k+2)%3], prefetch into L[(k+1)%3]
    for (int it = 0; it < T + 2; it += 3) {
        mom_step<0>(X, it, L2, L0, L1, A1, B1, A2, B2, A0, B0);
        mom_step<1>(X, it + 1, L0, L1, L2, A2, B2, A0, B0, A1, B1);
        mom_step<2>(X, it + 2, L1, L2, L0, A0, B0, A1, B1, A2, B2);
    }
}

// ---------------------------------------------------- restriction / prolong
template <typename S>
__device__ __forceinline__ int find_seg(const S *segs, int nseg, int64_t e)
{
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (segs[mid].first <= e) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// mode 0: direct, 1: gather into stage, 2: scatter from stage
__global__ void k_restrict(StepArgs a, const RSeg *__restrict__ segs, int nseg, int64_t nelem,
                           double *__restrict__ stage, int mode)
{
    if (stop_requested(a.err)) return;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nelem) return;
    const RSeg S = segs[find_seg(segs, nseg, e)];
    const int p = (int)(e - S.first);
    double v;
    if (mode != 2) {
        // _ring_patch_means (coupling.py:278-294): y outer, x inner
        const DevBlock *C = a.blocks + S.child;
        const double *E = C->eta[a.cur ^ 1];
        const int x0 = S.ns ? S.a + 3 * p : S.ring;
        const int y0 = S.ns ? S.ring : S.a + 3 * p;
        const int Pc = C->P;
        double acc = 0.0;
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx)
                acc = acc + E[(size_t)(x0 + dx + TS_G) * Pc + y0 + dy + TS_G];
        v = acc * (1.0 / 9.0);
    } else {
        v = stage[e];
    }
    if (mode == 1) {
        stage[e] = v;
        return;
    }
    // apply_restricted_eta (coupling.py:303-315); the parent's wet flag is
    // derived from the value written here
    const DevBlock *Pb = a.blocks + S.parent;
    const int x = S.ns ? S.pa + p : S.pline;
    const int y = S.ns ? S.pline : S.pa + p;
    Pb->eta[a.cur ^ 1][(size_t)(x + TS_G) * Pb->P + y + TS_G] = v;
}

// elements are child faces (3 per parent face)
__global__ void k_prolong(StepArgs a, const PSeg *__restrict__ segs, int nseg, int64_t nelem,
                          double *__restrict__ stage, int mode)
{
    if (stop_requested(a.err)) return;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nelem) return;
    const PSeg S = segs[find_seg(segs, nseg, e)];
    const int k = (int)(e - S.first);
    const int p = k / 3;
    double v;
    if (mode != 2) {
        const DevBlock *Pb = a.blocks + S.parent;
        // prolong_flux (coupling.py:318-327)
        if (S.ns) v = Pb->n[a.cur ^ 1][(size_t)(S.pa + p + TS_G) * Pb->P + S.pline + TS_G];
        else      v = Pb->m[a.cur ^ 1][(size_t)(S.pline + TS_G) * Pb->P + S.pa + p + TS_G];
    } else {
        v = stage[e];
    }
    if (mode == 1) {
        stage[e] = v;
        return;
    }
    // apply_prolonged_flux (coupling.py:330-340)
    const DevBlock *C = a.blocks + S.child;
    const int along = S.a + k;
    if (S.ns) C->n[a.cur ^ 1][(size_t)(along + TS_G) * C->P + S.cline + TS_G] = v;
    else      C->m[a.cur ^ 1][(size_t)(S.cline + TS_G) * C->P + along + TS_G] = v;
}

__device__ __forceinline__ double *arr_of(const DevBlock *B, int arr, int nb)
{
    return arr == 0 ? B->eta[nb] : (arr == 1 ? B->m[nb] : B->n[nb]);
}

__global__ void k_copy(StepArgs a, const Copy *__restrict__ cp, int64_t n, int serial)
{
    if (stop_requested(a.err)) return;
    const int nb = a.cur ^ 1;
    if (serial) {
        if (blockIdx.x != 0 || threadIdx.x != 0) return;
        for (int64_t e = 0; e < n; ++e) {
            const Copy k = cp[e];
            const int arr = (k.src_blk >> 28) & 3, sb = k.src_blk & 0x0fffffff;
            const double v = k.src_idx < 0 ? 0.0 : arr_of(a.blocks + sb, arr, nb)[k.src_idx];
            arr_of(a.blocks + k.dst_blk, arr, nb)[k.dst_idx] = v;
        }
        return;
    }
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const Copy k = cp[e];
    const int arr = (k.src_blk >> 28) & 3, sb = k.src_blk & 0x0fffffff;
    const double v = k.src_idx < 0 ? 0.0 : arr_of(a.blocks + sb, arr, nb)[k.src_idx];
    arr_of(a.blocks + k.dst_blk, arr, nb)[k.dst_idx] = v;
}

__global__ void k_cbrt(const double *in, double *out, int64_t n)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) out[e] = ts_cbrt(in[e]);
}

template <int W>
constexpr int tiles_per_cta() { return W == 1 ? 4 : (W == 2 ? 2 : 1); }

}  // namespace

// ------------------------------------------------------------- launchers
void launch_mass(const StepArgs &a, const Tile *tiles, int ntiles, bool fold, cudaStream_t s)
{
    if (ntiles <= 0) return;
    if (fold) k_mass<true><<<ntiles, kFlatThreads, 0, s>>>(a, tiles);
    else k_mass<false><<<ntiles, kFlatThreads, 0, s>>>(a, tiles);
}

void launch_accumulate(const StepArgs &a, const Tile *tiles, int ntiles, cudaStream_t s)
{
    if (ntiles <= 0) return;
    k_accum<<<ntiles, kFlatThreads, 0, s>>>(a, tiles);
}

void launch_momentum(const StepArgs &a, const Tile *tiles, int ntiles, int W, int T, cudaStream_t s)
{
    if (ntiles <= 0) return;
#define TS_MOM(WW)                                                                          \
    {                                                                                       \
        constexpr int TPC = tiles_per_cta<WW>();                                            \
        k_momentum<WW, TPC><<<(ntiles + TPC - 1) / TPC, 32 * WW * TPC, 0, s>>>(a, tiles, ntiles, T); \
    }
    switch (W) {
    case 1: TS_MOM(1); break;
    case 2: TS_MOM(2); break;
    case 3: TS_MOM(3); break;
    default: TS_MOM(4); break;
    }
#undef TS_MOM
}

void launch_restrict(const StepArgs &a, const RSeg *segs, int nseg, int64_t nelem, double *stage,
                     int mode, cudaStream_t s)
{
    if (nelem <= 0) return;
    k_restrict<<<(unsigned)((nelem + 255) / 256), 256, 0, s>>>(a, segs, nseg, nelem, stage, mode);
}

void launch_prolong(const StepArgs &a, const PSeg *segs, int nseg, int64_t nelem, double *stage,
                    int mode, cudaStream_t s)
{
    if (nelem <= 0) return;
    k_prolong<<<(unsigned)((nelem + 255) / 256), 256, 0, s>>>(a, segs, nseg, nelem, stage, mode);
}

void launch_copies(const StepArgs &a, const Copy *c, int64_t n, bool serial, cudaStream_t s)
{
    if (n <= 0) return;
    if (serial) k_copy<<<1, 32, 0, s>>>(a, c, n, 1);
    else k_copy<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, c, n, 0);
}

void launch_cbrt(const double *in, double *out, int64_t n, cudaStream_t s)
{
    if (n <= 0) return;
    k_cbrt<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, out, n);
}
