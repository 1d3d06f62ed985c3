// Shared device-side types for the nested-grid step.
//
// HBM layout: one arena per GPU; every owned block keeps the
// reference's ghosted BlockState arrays (kernels.py:39-62; halo g = 2) but
// with a common row pitch P = round_up(nj + 5, 4) doubles, so every row of
// every array starts 32-byte aligned and a tile of consecutive rows is one
// contiguous span.  Element (x, y) of an eta/h/nman array (cells x,y in
// [-2, n+2)) sits at (x+2)*P + (y+2); M face (fx, cy) at (fx+2)*P + cy+2;
// N (cx, fy) at (cx+2)*P + fy+2; accumulators (i, j) at i*P + j.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define TS_G 2

struct DevBlock {
    double *eta[2], *m[2], *n[2];
    double *h, *nman;
    double *acc_eta, *acc_speed, *acc_inund;
    int32_t ni, nj, P, order;       // order = global block index
    double r;                       // dt / dx                      (kernels.py:134, 242)
    double grr;                     // grav * r                     (kernels.py:243)
    double kf;                      // ((dt*grav)*n)*n, scalar n    (kernels.py:240)
    double dtg;                     // dt * grav
    int32_t has_nman, pad;
    // interior bathymetry as its 1-D depth profile (h = hprof[haxis ? j : i]),
    // or null: the mass kernel then reads ni or nj doubles instead of ni x nj
    const double *hprof;
    int32_t haxis, pad2;
};

// one unit of the march kernels: face rows [i0, i1) x output columns
// [j0, j1); also used as plain cell rectangles by the flat kernels (pad unused)
struct Tile {
    int32_t blk, i0, i1, j0, j1, pad;
};

// one restriction segment (coupling.EtaSegment + its link)
// mode 0: compute and write the parent cell; 1: compute into a buffer
// (srank < 0: the local stage; else rank srank's receive area); 2: write the
// parent cell from a buffer.  first = the segment's offset in that buffer.
struct RSeg {
    int32_t child, parent, ns, a, ring, pline, pa, count;
    int64_t first;
    int32_t mode, srank;
};

// one prolongation segment (coupling.FluxSegment + its link)
struct PSeg {
    int32_t parent, child, ns, a, cline, pline, pa, count;
    int64_t first;                  // offset (child faces) in its buffer
    int32_t mode, srank;            // as RSeg
};

// element copy: dst[dst_idx] = src[src_idx]; arr 0 eta, 1 m, 2 n (the
// "new" buffer of each), 3 h (setup); src_idx < 0 means "write 0"
// (reflective edge)
struct Copy {
    int32_t src_blk, dst_blk, src_idx, dst_idx;   // src_blk holds arr in bits 28..29
};

// one element of a merged exchange phase: every write of the
// phase with its value expressed in the phase's input state, so the phase's
// elements are independent and run as one launch
//   src: bits 0..27 block (kind 3: this rank), bits 28..29 kind:
//        0 copy, 1 zero, 2 mean of the 3x3 eta patch at sidx (restriction),
//        3 copy of receive-area slot sidx
//   dst: bits 0..27 block, or (bit 30 set) the rank whose receive-area slot
//        didx gets the value; bits 28..29 array (0 eta, 1 m, 2 n)
struct XOp {
    int32_t src, dst, sidx, didx;
};
#define TS_XDST_RECV 0x40000000

#define TS_NO_ERROR 0xffffffffffffffffULL

// first-error key: lexicographic (block order, what, i, j) so atomicMin
// reports the reference's first raising check (kernels.py:115-120;
// runner.py serial order); i, j biased by 4 (ghost indices are >= -2)
__host__ __device__ inline unsigned long long ts_err_key(int order, int what, long long i, long long j)
{
    return ((unsigned long long)order << 50) | ((unsigned long long)what << 48)
         | ((unsigned long long)(i + 4) << 24) | (unsigned long long)(j + 4);
}

// numpy scalar maximum (NaN propagating, first operand wins ties):
// (a >= b || isnan(a)) ? a : b
__host__ __device__ __forceinline__ double np_max(double a, double b)
{
    return (a >= b || a != a) ? a : b;
}

// np.sign: +1, -1, 0 for +-0, NaN for NaN
__host__ __device__ __forceinline__ double np_sign(double x)
{
    return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : (x == 0.0 ? 0.0 : x));
}

// ---- launchers (step_kernels.cu) ----
struct StepArgs {
    const DevBlock *blocks;
    int cur;                        // "old" buffer index
    double thr;
    unsigned long long *err;
    const int *acc_flag;            // fold previous step's outputs in K_mass
    int multi;                      // >1 rank: exchange kernels fence their peer stores
    double *const *recv;            // [n_ranks] receive areas of the cross-rank coupling
};

// inter-GPU phase barrier (one process per GPU): every rank bumps its epoch,
// stores it into each peer's flag slot over NVLink and spins until every
// peer's epoch reached its own (timeout -> error key what = 3)
// A rank's signal area is [n_ranks] peer epochs, its own epoch, then its
// error word: peer p's error word is peer_flags[p][n_ranks + 1].
struct BarrierArgs {
    unsigned long long *const *peer_flags;   // [n_ranks] peer signal areas (own at [rank])
    unsigned long long *my_flags;            // this rank's flag array, slot per peer
    unsigned long long *epoch;
    unsigned long long *err;
    int nranks, rank;
};
void launch_barrier(const BarrierArgs &b, cudaStream_t s);

void launch_mass(const StepArgs &a, const Tile *tiles, int ntiles, bool accumulate, cudaStream_t s);
void launch_accumulate(const StepArgs &a, const Tile *tiles, int ntiles, cudaStream_t s);
// lanes == 0: one tile per W warps (TPC tiles per CTA); lanes > 0: 128-thread
// CTAs (W = 4) holding 128 / lanes tiles of `lanes` threads each
// nman: some tile's block has per-cell Manning n
void launch_momentum(const StepArgs &a, const Tile *tiles, int ntiles, int W, int T, int lanes, bool nman,
                     cudaStream_t s);
int momentum_tiles_per_cta(int W, int lanes);
void launch_restrict(const StepArgs &a, const RSeg *segs, const int2 *chunks, int nchunks, double *stage,
                     cudaStream_t s);
void launch_prolong(const StepArgs &a, const PSeg *segs, const int2 *chunks, int nchunks, double *stage,
                    cudaStream_t s);
void launch_copies(const StepArgs &a, const Copy *c, int64_t n, bool serial, cudaStream_t s);
void launch_xops(const StepArgs &a, const XOp *ops, int64_t n, cudaStream_t s);
void launch_cbrt(const double *in, double *out, int64_t n, cudaStream_t s);
// h_ext of a block from a 1-D depth profile, ghosts edge-replicated
void launch_h_profile(const DevBlock &B, const double *prof, int axis, cudaStream_t s);
void launch_repitch(double *dst, int64_t dpitch, const double *src, int64_t spitch, int64_t rows, int64_t cols,
                    cudaStream_t s);
// many pitched <-> contiguous copies in one launch (batched host transfers)
struct Repitch {
    double *dst;
    const double *src;
    int64_t dpitch, spitch, rows, cols;
};
void launch_repitch_batch(const Repitch *jobs, int njobs, int64_t max_elems, cudaStream_t s);
