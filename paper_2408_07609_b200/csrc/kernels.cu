// sm_100a kernels of the nested-grid shallow-water step.
//
// Numerics follow the reference's evaluation order exactly:
// the file is compiled with -fmad=false (no FMA contraction), IEEE / and
// sqrt, numpy maximum/sign semantics (np_max / np_sign), and the product's
// cbrt (cbrt.cuh).  The stored "wet" flags of the reference are derived on
// the fly as h + eta >= thr, which equals the stored flag at every read site
// (checked by the parity tests against the oracle, which keeps
// the explicit array).
//
// Kernels:
//   k_mass      K_mass: continuity (kernels.py:123-155), fused with the
//               running-maxima fold of the previous step (kernels.py:322-343)
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
// accumulate_outputs for one cell (kernels.py:327-343); returns false if a
// batched fast op was out of range (caller redoes it with fold_cell_ieee)
__device__ __forceinline__ bool fold_cell(const DevBlock *B, size_t ac, double e, double h, double d,
                                          double Ml, double Mr, double Nl, double Nr, double thr)
{
    const bool w = d >= thr;
    const double mc = 0.5 * (Ml + Mr);
    const double nc = 0.5 * (Nl + Nr);
    const double ds = np_max(d, thr);
    bool ok = true;
    const double y = ts_rcp(ds);
    const double u = ts_div(mc, ds, y, ok), v = ts_div(nc, ds, y, ok);
    const double sp = ts_sqrt(u * u + v * v, ok);
    if (!ok) return false;
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
    return true;
}

__device__ __noinline__ void fold_cell_ieee(const DevBlock *B, size_t ac, double e, double h, double d,
                                            double Ml, double Mr, double Nl, double Nr, double thr)
{
    const bool w = d >= thr;
    const double mc = 0.5 * (Ml + Mr);
    const double nc = 0.5 * (Nl + Nr);
    const double ds = np_max(d, thr);
    const double u = mc / ds, v = nc / ds;
    const double sp = sqrt(u * u + v * v);
    if (w) {
        B->acc_eta[ac] = np_max(B->acc_eta[ac], e);
        B->acc_speed[ac] = np_max(B->acc_speed[ac], sp);
        if (h < 0.0) B->acc_inund[ac] = np_max(B->acc_inund[ac], d);
    }
}

// One thread per interior column j, marching down rows [i0, i1) of a tile,
// unrolled so several rows' loads are in flight; M face i of row i+1 is
// carried in a register.
template <int W, int TPC, bool FOLD>
__global__ void __launch_bounds__(32 * W * TPC)
k_mass(StepArgs a, const Tile *__restrict__ tiles, int ntiles)
{
    if (stop_requested(a.err)) return;
    const int lt = threadIdx.x / (32 * W), ci = threadIdx.x % (32 * W);
    const int t = blockIdx.x * TPC + lt;
    if (t >= ntiles) return;
    const Tile tl = tiles[t];
    const DevBlock *B = a.blocks + tl.blk;
    const int nj = B->nj, ni = B->ni, P = B->P;
    const int j = tl.j0 + ci;
    if (j >= tl.j1 || j >= nj) return;
    const int iend = min(tl.i1, ni);
    if (tl.i0 >= iend) return;
    const int cur = a.cur;
    const double *__restrict__ eo = B->eta[cur];
    double *__restrict__ en = B->eta[cur ^ 1];
    const double *__restrict__ mo = B->m[cur];
    const double *__restrict__ no = B->n[cur];
    const double *__restrict__ hh = B->h;
    const double r = B->r, thr = a.thr;
    const bool fold = FOLD && (*a.acc_flag != 0);
    size_t row = (size_t)(tl.i0 + TS_G) * P + j + TS_G;
    double Mi = __ldg(mo + row);
#pragma unroll 4
    for (int i = tl.i0; i < iend; ++i, row += P) {
        const double Mi1 = __ldg(mo + row + P);
        const double Nj = __ldg(no + row), Nj1 = __ldg(no + row + 1);
        const double e0 = __ldg(eo + row), h = __ldg(hh + row);
        const double d = h + e0;
        if (fold) {
            // accumulate_outputs of the previous step (kernels.py:322-343):
            // its eta_new/m_new/n_new are this step's old buffers
            const size_t ac = (size_t)i * P + j;
            if (!fold_cell(B, ac, e0, h, d, Mi, Mi1, Nj, Nj1, thr))
                fold_cell_ieee(B, ac, e0, h, d, Mi, Mi1, Nj, Nj1, thr);
        }
        // update_mass (kernels.py:134-155); wet_old derived as h + eta_old >= thr
        const double div = r * (Mi1 - Mi) + r * (Nj1 - Nj);
        double e = e0 - div;
        if (!(d >= thr) && div != 0.0) e = np_max(e0, -h) - div;
        if (div != 0.0 && h + e < 0.0) e = -h;
        if (!isfinite(e)) report(a.err, B->order, 0, i, j);
        en[row] = e;
        Mi = Mi1;
    }
}

// ------------------------------------------------------ standalone fold
template <int W, int TPC>
__global__ void __launch_bounds__(32 * W * TPC)
k_accum(StepArgs a, const Tile *__restrict__ tiles, int ntiles)
{
    // a.cur names the buffer to read (the "new" role of kernels.py:327-335)
    const int lt = threadIdx.x / (32 * W), ci = threadIdx.x % (32 * W);
    const int t = blockIdx.x * TPC + lt;
    if (t >= ntiles) return;
    const Tile tl = tiles[t];
    const DevBlock *B = a.blocks + tl.blk;
    const int nj = B->nj, ni = B->ni, P = B->P;
    const int j = tl.j0 + ci;
    if (j >= tl.j1 || j >= nj) return;
    const int iend = min(tl.i1, ni);
    const double *eta = B->eta[a.cur], *m = B->m[a.cur], *n = B->n[a.cur];
    const double thr = a.thr;
#pragma unroll 4
    for (int i = tl.i0; i < iend; ++i) {
        const size_t row = (size_t)(i + TS_G) * P + j + TS_G, ac = (size_t)i * P + j;
        const double e = eta[row], h = B->h[row], d = h + e;
        const double Ml = m[row], Mr = m[row + P], Nl = n[row], Nr = n[row + 1];
        if (!fold_cell(B, ac, e, h, d, Ml, Mr, Nl, Nr, thr))
            fold_cell_ieee(B, ac, e, h, d, Ml, Mr, Nl, Nr, thr);
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
    if (wl && !wr) {                        // front_r (kernels.py:191-196)
        const double d_r = el + hr;
        active = d_r >= thr;
        df = d_r;
        gr = np_max(er, -hr) - el;
    } else if (!wl && wr) {                 // front_l (kernels.py:197-202)
        const double d_l = er + hl;
        active = d_l >= thr;
        df = d_l;
        gr = er - np_max(el, -hl);
    }
    F.dface = df;
    F.grad = gr;
    F.active = active;
    F.dsafe = np_max(df, thr);
}

// fadv = f0*f0/dsafe, fcross = f0*(qbar/dsafe) with one shared reciprocal
__device__ __forceinline__ void face_flux(Face &F, bool &ok)
{
    const double y = ts_rcp(F.dsafe);
    F.fa = ts_div(F.f0 * F.f0, F.dsafe, y, ok);
    F.fc = F.f0 * ts_div(F.qbar, F.dsafe, y, ok);
}

__device__ __noinline__ double2 face_flux_ieee(double f0, double qbar, double ds)
{
    return make_double2(f0 * f0 / ds, f0 * (qbar / ds));
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
    bool lok = true;
    const double s = ts_sqrt(m0 * m0 + q0 * q0, lok);
    const double den = du * du * ts_cbrt(du);
    const double fr = ts_div(kfric * s, den, ts_rcp(den), lok);
    const double numer = m0 - r * adv - grr * F.dface * F.grad;
    const double dn = 1.0 + fr;
    const double v = ts_div(numer, dn, ts_rcp(dn), lok);
    ok = ok && (lok || !F.active);
    return F.active ? v : 0.0;
}

__device__ __noinline__ double face_finish_ieee(double m0, double q0, double du, double dface, double grad,
                                                double adv, double kfric, double r, double grr)
{
    const double fr = kfric * sqrt(m0 * m0 + q0 * q0) / (du * du * ts_cbrt(du));
    const double numer = m0 - r * adv - grr * dface * grad;
    return numer / (1.0 + fr);
}

// One thread per column c in [j0-1, j1] of a tile; the march visits rows
// r = i0-1 .. i1: prelims of M face r and N row r, then (one row behind)
// the updates of M face r-1 and N row r-1.  FC_M and FA_N are exchanged
// across columns through a 3-slot shared ring (one __syncthreads per row);
// FA_M and FC_N (neighbours along x) stay in registers.  The next row's
// loads are issued before the current row's arithmetic.
template <int W, int TPC>
__global__ void __launch_bounds__(32 * W * TPC)
k_momentum(StepArgs a, const Tile *__restrict__ tiles, int ntiles, int T)
{
    constexpr int NT = 32 * W * TPC;
    __shared__ double sFC[3][NT];
    __shared__ double sFA[3][NT];
    if (stop_requested(a.err)) return;
    const int tid = threadIdx.x;
    const int lt = tid / (32 * W), ci = tid % (32 * W);
    const int t = blockIdx.x * TPC + lt;
    const bool tv = t < ntiles;
    Tile tl;
    if (tv) tl = tiles[t];
    else tl = Tile{0, 0, 0, 0, 0, 0};
    const DevBlock *B = a.blocks + tl.blk;
    const int ni = B->ni, nj = B->nj, P = B->P;
    const int c = tl.j0 - 1 + ci;
    const bool inTile = tv && c <= tl.j1;
    const bool colM = inTile && c <= nj;          // M window columns -1..nj
    const bool colN = inTile && c <= nj + 1;      // N window faces -1..nj+1
    const bool updM = tv && c >= tl.j0 && c < tl.j1 && c < nj;
    const bool updN = tv && c >= tl.j0 && c < tl.j1 && c <= nj;
    const int cur = a.cur;
    const double *__restrict__ eta = B->eta[cur ^ 1];
    const double *__restrict__ hh = B->h;
    const double *__restrict__ mo = B->m[cur];
    const double *__restrict__ no = B->n[cur];
    double *__restrict__ mn = B->m[cur ^ 1];
    double *__restrict__ nn = B->n[cur ^ 1];
    const double *__restrict__ nman = B->nman;
    const bool has_nman = B->has_nman != 0;
    const double thr = a.thr, r = B->r, grr = B->grr, kf = B->kf, dtg = B->dtg;
    const int order = B->order;
    const int i0 = tl.i0, i1 = tl.i1;

    // row r-1 of column c (carried), and the prefetched row r
    double e_p = 0.0, h_p = 0.0, D_p = 0.0, Nc_p = 0.0, Nc1_p = 0.0, Mc = 0.0, Mcl = 0.0;
    double e_n = 0.0, h_n = 0.0, el_n = 0.0, hl_n = 0.0, Nc_n = 0.0, Nc1_n = 0.0, Mn_n = 0.0, Mnl_n = 0.0;
    size_t rc = (size_t)(i0 - 2 + TS_G) * P + c + TS_G;
    if (colN) {
        e_p = __ldg(eta + rc);
        h_p = __ldg(hh + rc);
        Nc_p = __ldg(no + rc);
        Nc1_p = __ldg(no + rc + 1);
        Mc = __ldg(mo + rc + P);
        Mcl = __ldg(mo + rc + P - 1);
        rc += P;
        e_n = __ldg(eta + rc);
        h_n = __ldg(hh + rc);
        el_n = __ldg(eta + rc - 1);
        hl_n = __ldg(hh + rc - 1);
        Nc_n = __ldg(no + rc);
        Nc1_n = __ldg(no + rc + 1);
        Mn_n = __ldg(mo + rc + P);
        Mnl_n = __ldg(mo + rc + P - 1);
    }
    D_p = h_p + e_p;
    Face Mp{}, Np{};                 // centre faces of row r-1
    double faM_pp = 0.0;             // FA_M(r-2)
    double fcN_pp = 0.0;             // FC_N(r-2)
    for (int it = 0; it < T + 2; ++it) {
        const int rr = i0 - 1 + it;
        const int slot = it % 3, pslot = (it + 2) % 3;
        const bool rowOK = rr <= i1;
        const double e = e_n, h = h_n, el = el_n, hl = hl_n, Nc = Nc_n, Nc1 = Nc1_n, Mn = Mn_n, Mnl = Mnl_n;
        if (colN && rr + 1 <= i1) {            // prefetch row rr+1
            rc += P;
            e_n = __ldg(eta + rc);
            h_n = __ldg(hh + rc);
            el_n = __ldg(eta + rc - 1);
            hl_n = __ldg(hh + rc - 1);
            Nc_n = __ldg(no + rc);
            Nc1_n = __ldg(no + rc + 1);
            Mn_n = __ldg(mo + rc + P);
            Mnl_n = __ldg(mo + rc + P - 1);
        }
        const double D = h + e, Dl = hl + el;
        Face Mf{}, Nf{};
        const bool doM = colM && rowOK && rr <= ni + 1;
        const bool doN = colN && rowOK && rr <= ni;
        // M face rr, column c: cells (rr-1, c) | (rr, c)
        face_geom(Mf, e_p, e, h_p, h, D_p, D, Mc, 0.25 * ((Nc_p + Nc) + (Nc1_p + Nc1)), thr);
        // N face c of row rr: cells (rr, c-1) | (rr, c)
        face_geom(Nf, el, e, hl, h, Dl, D, Nc, 0.25 * ((Mcl + Mc) + (Mnl + Mn)), thr);
        bool ok = true;
        face_flux(Mf, ok);
        face_flux(Nf, ok);
        if (!ok) {
            const double2 fm = face_flux_ieee(Mf.f0, Mf.qbar, Mf.dsafe);
            const double2 fn = face_flux_ieee(Nf.f0, Nf.qbar, Nf.dsafe);
            Mf.fa = fm.x; Mf.fc = fm.y;
            Nf.fa = fn.x; Nf.fc = fn.y;
        }
        if (!doM) Mf = Face{};
        if (!doN) Nf = Face{};
        sFC[slot][tid] = Mf.fc;
        sFA[slot][tid] = Nf.fa;
        __syncthreads();
        if (it >= 2) {
            const int f = rr - 1;
            const bool dM = updM && f < i1, dN = updN && f < i1 && f < ni;
            const double advM = face_adv(Mp, faM_pp, Mf.fa, sFC[pslot][tid - 1], sFC[pslot][tid + 1]);
            const double advN = face_adv(Np, sFA[pslot][tid - 1], sFA[pslot][tid + 1], fcN_pp, Nf.fc);
            double kM = kf, kN = kf;
            const size_t fc = (size_t)(f + TS_G) * P + c + TS_G;
            if (has_nman && (dM || dN)) {
                const double nfM = 0.5 * (nman[fc - P] + nman[fc]);
                const double nfN = 0.5 * (nman[fc - 1] + nman[fc]);
                kM = dtg * nfM * nfM;
                kN = dtg * nfN * nfN;
            }
            bool ok2 = true;
            double vM = face_finish(Mp, advM, kM, r, grr, ok2);
            double vN = face_finish(Np, advN, kN, r, grr, ok2);
            if (!ok2) {
                vM = Mp.active ? face_finish_ieee(Mp.f0, Mp.qbar, Mp.dsafe, Mp.dface, Mp.grad, advM, kM, r, grr) : 0.0;
                vN = Np.active ? face_finish_ieee(Np.f0, Np.qbar, Np.dsafe, Np.dface, Np.grad, advN, kN, r, grr) : 0.0;
            }
            if (dM) {
                if (!isfinite(vM)) report(a.err, order, 1, f, c);
                mn[fc] = vM;
            }
            if (dN) {
                if (!isfinite(vN)) report(a.err, order, 2, f, c);
                nn[fc] = vN;
            }
        }
        faM_pp = Mp.fa;
        fcN_pp = Np.fc;
        Mp = Mf;
        Np = Nf;
        e_p = e;
        h_p = h;
        D_p = D;
        Nc_p = Nc;
        Nc1_p = Nc1;
        Mc = Mn;
        Mcl = Mnl;
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
void launch_mass(const StepArgs &a, const Tile *tiles, int ntiles, int W, int T, bool fold,
                 cudaStream_t s)
{
    (void)T;
    if (ntiles <= 0) return;
#define TS_MASS(WW)                                                                         \
    {                                                                                       \
        constexpr int TPC = tiles_per_cta<WW>();                                            \
        const int grid = (ntiles + TPC - 1) / TPC;                                          \
        if (fold) k_mass<WW, TPC, true><<<grid, 32 * WW * TPC, 0, s>>>(a, tiles, ntiles);   \
        else k_mass<WW, TPC, false><<<grid, 32 * WW * TPC, 0, s>>>(a, tiles, ntiles);       \
    }
    switch (W) {
    case 1: TS_MASS(1); break;
    case 2: TS_MASS(2); break;
    case 3: TS_MASS(3); break;
    default: TS_MASS(4); break;
    }
#undef TS_MASS
}

void launch_accumulate(const StepArgs &a, const Tile *tiles, int ntiles, int W, int T, cudaStream_t s)
{
    (void)T;
    if (ntiles <= 0) return;
#define TS_ACC(WW)                                                                          \
    {                                                                                       \
        constexpr int TPC = tiles_per_cta<WW>();                                            \
        k_accum<WW, TPC><<<(ntiles + TPC - 1) / TPC, 32 * WW * TPC, 0, s>>>(a, tiles, ntiles); \
    }
    switch (W) {
    case 1: TS_ACC(1); break;
    case 2: TS_ACC(2); break;
    case 3: TS_ACC(3); break;
    default: TS_ACC(4); break;
    }
#undef TS_ACC
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
