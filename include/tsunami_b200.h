/*
 * tsunami_b200.h — C ABI of the B200-native nested-grid shallow-water step.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/blockswe/, "blockswe"): the per-step body of
 * runner.Simulation (runner.py:193-365), the kernel layer (kernels.py) and
 * the per-step halves of the data-movement layer (coupling.py:278-340,
 * exchange.py:162-275).  The reference has no FFI of its own — its boundary
 * is a Python object API — so each entry point below names the reference
 * interface it replaces; INTEGRATION.md shows the ctypes binding a
 * maintainer would add to blockswe.
 *
 * Conventions
 *  - Plain C types only.  Block indices are positions in the reference's
 *    global block order, NestedGridSystem.all_blocks() (grid.py:82-84).
 *  - Host arrays use the reference's own BlockState layouts (kernels.py:
 *    39-62): C order, axis 0 = x, halo g = 2; eta/h (ni+4)x(nj+4),
 *    m (ni+5)x(nj+4), n (ni+4)x(nj+5); accumulators ni x nj.
 *  - Return codes: TS_OK, TS_ERR_NUMERICS (a non-finite field, the
 *    reference's NumericsError, kernels.py:115-120), TS_ERR_CUDA,
 *    TS_ERR_INVALID (bad argument: the reference's ValueError /
 *    GridStructureError).  ts_last_error() gives the message.
 *  - A handle is used by one host thread at a time; the library owns all
 *    device memory; inputs are copied at ts_create.
 */
#ifndef TSUNAMI_B200_H
#define TSUNAMI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 2

#define TS_OK 0
#define TS_ERR_NUMERICS 1
#define TS_ERR_CUDA 2
#define TS_ERR_INVALID 3

/* sides (exchange.py:37 order) and edge kinds (grid.py:102-119) */
#define TS_WEST 0
#define TS_EAST 1
#define TS_SOUTH 2
#define TS_NORTH 3
#define TS_REFLECTIVE 0
#define TS_RADIATION 1

/* one block: replaces BlockState construction (kernels.py:39-62),
 * set_initial_eta (kernels.py:97-101) and fill_bathymetry_halos
 * (exchange.py:281-300), whose results the caller passes in h_ext/nman_ext */
typedef struct ts_block_desc {
    int64_t block_id;          /* Block.block_id (grid.py:44) — for messages */
    int32_t ni, nj;            /* Block.ni / nj */
    int32_t owner;             /* rank (GPU) owning the block, plan.rank_of */
    int32_t level;             /* 0-based level index */
    double dx;                 /* GridLevel.dx */
    double manning;            /* scalar Block.manning_n (used if nman_ext == NULL) */
    const double *h_ext;       /* (ni+4)*(nj+4): BlockState.h_ext after fill_bathymetry_halos,
                                  or NULL with h_profile */
    const double *nman_ext;    /* NULL or (ni+4)*(nj+4): BlockState.n_ext (array case) */
    const double *eta0;        /* ni*nj interior initial level (runner.py:77-80) */
    /* Device-side bathymetry setup: a block whose depth
     * depends on one axis only (Block.h a broadcast view: the synthetic
     * slope / coastal-profile kinds, config.py:41-70) passes that 1-D
     * profile instead of h_ext; the device builds h_ext — edge replication
     * (kernels.py:108-112) and the siblings' strips (exchange.py:281-300,
     * applied at the first ts_run) — bit for bit. */
    const double *h_profile;   /* NULL, or ni values (h_axis 0) / nj values (h_axis 1) */
    int32_t h_axis;            /* 0: h[i, j] = h_profile[i]; 1: h[i, j] = h_profile[j] */
    int32_t pad_;
} ts_block_desc;

/* exchange.HaloEntry (exchange.py:62-101); entries are passed in the
 * reference's APPLY order (runner.py:178-186: receiver rank, sorted sender
 * rank, schedule order) so duplicate ghost writes resolve identically */
typedef struct ts_halo_entry {
    int32_t sender, receiver;  /* block indices */
    int32_t side;              /* sender's side facing the receiver */
    int32_t send_lo, send_hi;  /* HaloEntry.send_span */
    int32_t recv_lo, recv_hi;  /* HaloEntry.recv_span */
} ts_halo_entry;

/* coupling.EtaSegment (coupling.py:36-46) with its link's blocks */
typedef struct ts_eta_segment {
    int32_t parent, child;     /* block indices */
    int32_t side;
    int32_t child_lo, child_hi;      /* child_span */
    int32_t ring_start, parent_line;
    int32_t parent_lo, parent_hi;    /* parent_span */
} ts_eta_segment;

/* coupling.FluxSegment (coupling.py:49-59) with its link's blocks */
typedef struct ts_flux_segment {
    int32_t parent, child;
    int32_t side;
    int32_t child_lo, child_hi;
    int32_t child_face_line, parent_face_line;
    int32_t parent_lo, parent_hi;
} ts_flux_segment;

/* one apply_edge_flux call (kernels.py:274-306; runner.py:89-98, 116-117) */
typedef struct ts_edge {
    int32_t block, side, kind, lo, hi;
} ts_edge;

/* the whole configured system: replaces Simulation.__init__ (runner.py:59-102) */
typedef struct ts_desc {
    int32_t abi_version;       /* TS_ABI_VERSION */
    int32_t n_blocks;
    const ts_block_desc *blocks;
    double dt, gravity, wet_threshold;   /* SimulationConfig (grid.py:144-158) */
    int32_t n_halo;  const ts_halo_entry *halo;
    int32_t n_restrict; const ts_eta_segment *restrict_segs;
    int32_t n_prolong;  const ts_flux_segment *prolong_segs;
    int32_t n_edges; const ts_edge *edges;
    int32_t rank, n_ranks;     /* this process's rank / GPU count (1 GPU: 0, 1) */
    int32_t device;            /* CUDA device ordinal */
    int32_t tile_rows;         /* 0 = default */
} ts_desc;

typedef struct ts_handle ts_handle;

/* field codes for ts_get_field / ts_set_field (BlockState / OutputAccumulators) */
#define TS_ETA_OLD 0
#define TS_ETA_NEW 1
#define TS_M_OLD 2
#define TS_M_NEW 3
#define TS_N_OLD 4
#define TS_N_NEW 5
#define TS_H_EXT 6
#define TS_MAX_ETA 7
#define TS_MAX_SPEED 8
#define TS_MAX_INUNDATION 9

/* phase codes for ts_phase (runner.PHASE_SEQUENCE, runner.py:39-40, plus the
 * kernel-level calls of kernels.py) */
#define TS_PH_MASS 0        /* update_mass on every owned block (no accumulate) */
#define TS_PH_RESTRICT 1    /* restrict_eta + apply_restricted_eta */
#define TS_PH_HALO_ETA 2    /* pack/unpack_halo, eta phase */
#define TS_PH_MOMENTUM 3    /* update_momentum on every owned block, no edges */
#define TS_PH_EDGES 4       /* every ts_edge, in order */
#define TS_PH_PROLONG 5     /* prolong_flux + apply_prolonged_flux */
#define TS_PH_HALO_FLUX 6   /* pack/unpack_halo, flux phase */
#define TS_PH_OUTPUT 7      /* accumulate_outputs on every owned block */
#define TS_PH_SWAP 8        /* BlockState.swap */

const char *ts_last_error(void);
int ts_abi_version(void);

/* Simulation.__init__ (runner.py:59-102) */
int ts_create(const ts_desc *desc, ts_handle **out);
/* Simulation.run body for n steps (runner.py:193-365): mass, restrict,
 * halo-eta, momentum+edges, prolong, halo-flux, output, swap; the running
 * maxima are up to date on return.  Re-entrant across calls. */
int ts_run(ts_handle *h, int64_t n_steps);
/* one phase, for the kernel-level API and phase-order tests */
int ts_phase(ts_handle *h, int32_t phase);
/* BlockState / OutputAccumulators array access in the reference layout */
int ts_get_field(ts_handle *h, int32_t block, int32_t field, double *out, int64_t len);
int ts_set_field(ts_handle *h, int32_t block, int32_t field, const double *in, int64_t len);
/* BlockState.set_initial_eta (kernels.py:97-101): the ni*nj interior
 * initial level into both water-level buffers */
int ts_set_initial_eta(ts_handle *h, int32_t block, const double *eta0, int64_t len);
/* A fresh start on the same system, as constructing a new Simulation does
 * (runner.py:59-102; BlockState and OutputAccumulators start at zero,
 * kernels.py:39-62, 309-320): zero every owned block's water levels (both
 * buffers, ghosts included), fluxes and running maxima, clear the error
 * and the step count.  Bathymetry and Manning n are kept. */
int ts_reset(ts_handle *h);
/* Batched host->device copy of the setup inputs of n owned blocks: h_ext
 * ((ni+4)*(nj+4), as ts_set_field(TS_H_EXT); NULL leaves a block's
 * bathymetry as is) and the interior initial level (ni*nj, as
 * ts_set_initial_eta) — one synchronisation for all */
int ts_upload_inputs(ts_handle *h, int32_t n, const int32_t *blocks, const double *const *h_ext,
                     const double *const *eta0);
/* The device-side setup of ts_block_desc.h_profile for n owned blocks
 * again (a fresh run's bathymetry input): each 1-D depth profile (ni values
 * for axes[k] 0, nj for 1) expands to h_ext with edge replication; the
 * siblings' strips are copied before the next step */
int ts_upload_profiles(ts_handle *h, int32_t n, const int32_t *blocks, const double *const *profiles,
                       const int32_t *axes);
/* Batched device->host copy of nf fields of n owned blocks in the
 * reference layout (as ts_get_field): out[k * nf + f] receives field
 * fields[f] of block blocks[k] — one synchronisation for all */
int ts_download_fields(ts_handle *h, int32_t n, const int32_t *blocks, int32_t nf, const int32_t *fields,
                       double *const *out);
/* the first non-finite value of the failing step (kernels.py:115-120):
 * what = 0 water level, 1 x-flux, 2 y-flux; (i, j) local cell */
int ts_error_info(ts_handle *h, int32_t *block, int32_t *what, int64_t *i, int64_t *j);
/* per-routine device seconds of the last ts_run (runner.ROUTINES order:
 * mass, momentum, restrict, prolong, halo-eta, halo-flux, output) and total */
int ts_timings(ts_handle *h, double *routines7, double *total);
int64_t ts_steps_done(ts_handle *h);
/* device bytes held by the arena */
int64_t ts_device_bytes(ts_handle *h);
/* kernels launched per ts_run step (graph nodes) */
int32_t ts_launches_per_step(ts_handle *h);
/* enqueue a device barrier of all ranks on the library stream (collective;
 * no-op on one rank): work enqueued after it starts on every rank within
 * the barrier's latency, e.g. a timed region's start event */
int ts_device_barrier(ts_handle *h);
/* diagnostic: run ONE step (collective across ranks; the same state as
 * ts_run(1), end-of-run fold included) as a graph with an event after every
 * launch, the
 * width groups' march launches serialised; for launch k, labels[k] = kind * 16
 * + group and us[k] = device microseconds since the previous launch ended.
 * Kinds: 0 mass, 1 restrict (sources), 2 restrict (second pass), 3 halo-eta,
 * 4 barrier (label 64 eta, 65 second eta, 66 prolongation), 5 restrict
 * (received), 6 halo-eta after the received restriction, 7 march (group),
 * 8 edges, 9 prolong (sources), 10 prolong (second pass), 11 prolong
 * (received), 12 halo-flux, 13 merged eta phase, 14 merged flux phase (the
 * received values of a merged phase: labels 80 / 176).  *count = launches in the step (up to cap
 * reported). */
int ts_trace_step(ts_handle *h, int32_t *labels, float *us, int32_t cap, int32_t *count);
/* timing mode: every 8th graph-replayed step of ts_run records the mass,
 * momentum and whole-step boundaries into its own CUDA events (on the launch
 * stream; rebinding a launch's event nodes costs it ~9 us, so the steps in
 * between run untouched); ts_kernel_seconds returns their averages */
int ts_set_timing(ts_handle *h, int32_t on);
/* average device time (s) of the momentum kernel over the last ts_run's
 * timed graph replays, measured with events on the launch stream */
int ts_kernel_seconds(ts_handle *h, double *mass_s, double *momentum_s, double *step_s);
/* the CUDA stream (cudaStream_t) every kernel of the handle runs on, for
 * callers that bracket ts_run with their own events */
int ts_stream(ts_handle *h, void **stream);
void ts_destroy(ts_handle *h);

/* multi-GPU (one process per GPU): export this rank's arena/signal IPC
 * handles, then map every peer's before the first ts_run */
int ts_ipc_export(ts_handle *h, void *out, int64_t len);
int ts_ipc_import(ts_handle *h, int32_t peer_rank, const void *in, int64_t len);

/* page-locked host buffers (staging of the host<->device copies of the
 * public API at full PCIe rate); NULL on failure */
void *ts_host_alloc(int64_t bytes);
void ts_host_free(void *p);

/* the friction cube root (kernels.py:240-241 np.cbrt): host twin and device */
void ts_cbrt_host(const double *in, double *out, int64_t n);
int ts_cbrt_device(int32_t device, const double *in, double *out, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
