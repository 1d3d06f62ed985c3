// C ABI (include/tsunami_b200.h): device arena, exchange descriptors, the
// per-step CUDA graph and the run loop.  Replaces runner.Simulation's body
// (runner.py:59-365) for the blocks this process/GPU owns.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <type_traits>
#include <vector>

#include "../../include/tsunami_b200.h"
#include "cbrt.cuh"
#include "common.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(TS_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                             \
    } while (0)

// phase boundaries: 0 |mass| 1 |restrict| 2 |halo-eta| 3 |momentum| 4
// |edges| 5 |prolong| 6 |halo-flux| 7
constexpr int kPhaseEvents = 8;
// boundaries retargeted per step in timing mode: mass (0,1), momentum (3,4),
// whole step (0,7)
constexpr int kTimed[5] = {0, 1, 3, 4, 7};
constexpr int kTimingEvery = 8;           // timing mode: every 8th step is sampled
#ifndef TS_STEPS_PER_GRAPH
#define TS_STEPS_PER_GRAPH 4
#endif
constexpr int kStepsPerGraph = TS_STEPS_PER_GRAPH;   // ts_run launches steps in graphs of 4 (even)

template <typename S>
struct SegList {
    S *d = nullptr;
    int2 *ch = nullptr;       // (segment, first element) per CTA
    int nch = 0;
};

struct Group {
    int W = 0;                          // warps per tile; packed groups: warps per CTA
    int lanes = 0;                      // packed groups: threads per tile (nj + 3)
    int T = 64;                         // march rows per tile of this group
    std::vector<Tile> tiles;
    Tile *d = nullptr;
    // multi-GPU overlap: tiles[0, n_early) read no cell that the exchange
    // chain (peers' halo / restriction stores, the received restriction,
    // the halo copies that must follow it) writes, so they march while it
    // runs; tiles[n_early, size) march after it
    int n_early = 0;
    bool nman = false;                  // some block of the group has per-cell Manning n
};

}  // namespace

struct ts_handle {
    int device = 0, rank = 0, nranks = 1;
    cudaStream_t stream = nullptr;
    double dt = 0, g = 0, thr = 0;
    int nb = 0;
    std::vector<ts_block_desc> desc;      // pointers not retained
    std::vector<size_t> off;              // block offset inside its owner's arena
    std::vector<DevBlock> hb;             // host mirror of the device table
    DevBlock *d_blocks = nullptr;
    char *arena = nullptr;
    size_t arena_bytes = 0;
    int T = 64;                           // rows per march tile; T + 2 must be a multiple of 3
    // momentum march groups: [0, 4) one tile per W = 1..4 warps; then the
    // packed groups (tiles of nj + 3 threads side by side in a CTA)
    std::vector<Group> groups = std::vector<Group>(4);
    Tile *d_all = nullptr;                // every tile (flat mass / fold kernels)
    int n_all = 0;
    // the momentum launches of the column-width groups run as parallel
    // graph branches (the small groups fill the big one's tail)
    bool mom_par = true;
    cudaStream_t side[7] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[7] = {};
    // the late tiles' branches (multi-stream overlap of the eta exchange)
    cudaStream_t side2[7] = {};
    cudaEvent_t ev_fork2 = nullptr, ev_join2[7] = {};
    // contiguous device staging of host transfers (one 1-D copy + repitch
    // kernel instead of a row-by-row 2-D copy of narrow rows)
    double *d_io = nullptr;
    size_t io_len = 0;
    // batched transfers: one contiguous staging area for all owned blocks'
    // fields of a batch, and the repitch job list
    double *d_bulk = nullptr;
    size_t bulk_len = 0;
    Repitch *d_jobs = nullptr;
    size_t jobs_len = 0;
    // multi-GPU (one process per GPU): peer arenas mapped by CUDA IPC
    // [0, nranks): peers' epochs; [nranks]: own epoch; [nranks + 1]: the
    // error word (d_err), read by the peers at every phase barrier
    unsigned long long *d_sig = nullptr;
    std::vector<char *> peer_arena;
    std::vector<unsigned long long *> peer_sig;
    unsigned long long **d_peer_sig = nullptr;
    int imported = 0;
    bool x_restrict = false, x_halo = false, x_prolong = false;   // cross-rank traffic per phase
    // coupling segment lists: send = this rank's sources (direct, or into the
    // local stage / a peer's receive area), local = second pass of a two-pass
    // exchange, recv = cross-rank values received into this rank's area
    SegList<RSeg> r_send, r_local, r_recv;
    SegList<PSeg> p_send, p_local, p_recv;
    std::vector<size_t> recv_off;         // byte offset of every owner's receive area in its arena
    double **d_recv = nullptr;            // [n_ranks] receive-area bases (own + mapped peers)
    std::vector<double *> recv_base;
    bool r_two_pass = false;
    bool p_two_pass = false;
    Copy *d_heta = nullptr, *d_hflux = nullptr, *d_edge = nullptr;
    int64_t n_heta = 0, n_hflux = 0, n_edge = 0;
    // halo-eta copies whose source a peer's restriction writes: after the
    // received restriction (the reference's restriction-before-halo order),
    // with a second barrier when one of them crosses ranks
    Copy *d_heta2 = nullptr;
    int64_t n_heta2 = 0;
    bool x_halo2 = false;
    bool overlap = false;                 // the exchange chain runs beside the early march tiles
    cudaStream_t xs = nullptr;            // its stream
    cudaEvent_t ev_xfork = nullptr, ev_xjoin = nullptr;
    // device-built bathymetry: the siblings' h strips, copied once before
    // the first step (after every peer arena is mapped)
    Copy *d_hfill = nullptr;
    int64_t n_hfill = 0;
    bool h_fill_pending = false;
    bool edge_serial = false;
    double *d_stage = nullptr;
    unsigned long long *d_err = nullptr;  // = d_sig + nranks + 1
    int *d_accflag = nullptr;
    // step graphs per buffer parity; kept alive
    // because exec event-node updates refer to them
    cudaGraph_t graph[2] = {};
    cudaGraphExec_t gexec[2] = {};
    // kStepsPerGraph consecutive steps in one graph (starting at buffer
    // parity c): fewer graph-launch boundaries per step
    cudaGraph_t graph_multi[2] = {};
    cudaGraphExec_t gexec_multi[2] = {};
    cudaGraphNode_t ev_node_multi[2][kPhaseEvents] = {};
    cudaEvent_t ev[kPhaseEvents] = {};
    cudaEvent_t ev_first[kPhaseEvents] = {};    // the first step of a run (get_graph_first)
    cudaGraph_t graph_first[2] = {};
    cudaGraphExec_t gexec_first[2] = {};
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    int cur = 0;
    int64_t steps = 0;
    double routines[7] = {0};
    double total = 0;
    double mass_s = 0, mom_s = 0, step_s = 0;
    int launches = 0;
    bool timing = false;
    cudaGraphNode_t ev_node[2][kPhaseEvents] = {};
    std::vector<cudaEvent_t> pool;                    // 5 per timed step
    // merged exchange phases (build_merged): [0] eta sources, [1] eta
    // received, [2] flux sources, [3] flux received
    bool merged = false;
    bool mx_bar_eta = false, mx_bar_flux = false;
    XOp *d_mx[4] = {};
    int64_t n_mx[4] = {};
    double *d_mstage = nullptr;           // second-wave staging (recv slot [n_ranks])
    // per owned block: its 1-D depth profile on the device (DevBlock.hprof)
    std::vector<double *> hprof_buf;
    // ts_trace_step: an event after every launch of one captured step
    bool tracing = false;
    std::vector<cudaEvent_t> trace_ev;
    std::vector<int32_t> trace_label;
};

namespace {

StepArgs args_of(const ts_handle *h, int cur)
{
    StepArgs a;
    a.blocks = h->d_blocks;
    a.cur = cur;
    a.thr = h->thr;
    a.err = h->d_err;
    a.acc_flag = h->d_accflag;
    a.multi = h->nranks > 1;
    a.recv = h->d_recv;
    return a;
}


void barrier(ts_handle *h, cudaStream_t s)
{
    BarrierArgs b;
    b.peer_flags = h->d_peer_sig;
    b.my_flags = h->d_sig;
    b.epoch = h->d_sig + h->nranks;
    b.err = h->d_err;
    b.nranks = h->nranks;
    b.rank = h->rank;
    launch_barrier(b, s);
}

// The step body, in the reference's phase order (runner.py:352-365).  When
// `events` the phase boundaries are recorded (external event nodes when
// captured into a graph).
int enqueue_step(ts_handle *h, cudaStream_t s, int cur, bool events, int *nlaunch, cudaEvent_t *evs = nullptr)
{
    const StepArgs a = args_of(h, cur);
    if (!evs) evs = h->ev;
    int n = 0;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s, &cap));
    auto mark = [&](int k) -> int {
        if (!events) return 0;
        if (cap == cudaStreamCaptureStatusActive)
            CK(cudaEventRecordWithFlags(evs[k], s, cudaEventRecordExternal));
        else
            CK(cudaEventRecord(evs[k], s));
        return 0;
    };
    // ts_trace_step: an external event after every launch, labelled with
    // the launch's kind (TS_TRACE_* of the header) * 16 + its group
    auto tick = [&](cudaStream_t st, int label) -> int {
        if (!h->tracing) return 0;
        const size_t k = h->trace_label.size();
        if (k >= h->trace_ev.size()) return 0;
        CK(cudaEventRecordWithFlags(h->trace_ev[k], st, cudaEventRecordExternal));
        h->trace_label.push_back(label);
        return 0;
    };
    if (tick(s, -1)) return TS_ERR_CUDA;
    if (mark(0)) return TS_ERR_CUDA;
    if (h->n_all) { launch_mass(a, h->d_all, h->n_all, true, s); ++n; if (tick(s, 0)) return TS_ERR_CUDA; }
    if (mark(1)) return TS_ERR_CUDA;
    // multi-GPU phase barriers: only around phases with
    // cross-rank stores; each one orders this rank's peer stores before the
    // readers' next phase and keeps writers from overtaking readers
    // restriction: this rank's sources (direct / staged / into peers'
    // receive areas), the second pass of a two-pass exchange, then - once
    // every rank's stores have landed - the values received from peers
    // momentum launches of one tile range of every width group: the
    // largest on stream s, the others forked onto side streams (parallel
    // branches of the captured graph) and joined back
    auto march = [&](int which, cudaStream_t s) -> int {   // 0 all, 1 early, 2 late tiles
        int order[8], ng = 0;
        auto range = [&](const Group &g, int &lo, int &cnt) {
            lo = which == 2 ? g.n_early : 0;
            cnt = which == 0 ? (int)g.tiles.size() : (which == 1 ? g.n_early : (int)g.tiles.size() - g.n_early);
        };
        for (int k = 0; k < (int)h->groups.size() && ng < 8; ++k) {
            int lo, cnt;
            range(h->groups[k], lo, cnt);
            if (cnt > 0) order[ng++] = k;
        }
        auto work = [&](int k) {
            const Group &g = h->groups[k];
            int lo, cnt;
            range(g, lo, cnt);
            return (double)cnt * (g.lanes ? g.lanes : 32 * g.W);
        };
        for (int x = 1; x < ng; ++x)
            for (int y = x; y > 0 && work(order[y]) > work(order[y - 1]); --y)
                std::swap(order[y], order[y - 1]);
        const bool par = h->mom_par && ng > 1 && !h->tracing;
        cudaStream_t *side = which == 2 ? h->side2 : h->side;
        cudaEvent_t fork = which == 2 ? h->ev_fork2 : h->ev_fork;
        cudaEvent_t *join = which == 2 ? h->ev_join2 : h->ev_join;
        if (par) CK(cudaEventRecord(fork, s));
        for (int x = 0; x < ng; ++x) {
            Group &gr = h->groups[order[x]];
            int lo, cnt;
            range(gr, lo, cnt);
            cudaStream_t st = s;
            if (par && x > 0) {
                st = side[x - 1];
                CK(cudaStreamWaitEvent(st, fork, 0));
            }
            launch_momentum(a, gr.d + lo, cnt, gr.W, gr.T, gr.lanes, gr.nman, st);
            ++n;
            if (tick(st, 7 * 16 + order[x])) return TS_ERR_CUDA;
            if (par && x > 0) {
                CK(cudaEventRecord(join[x - 1], st));
                CK(cudaStreamWaitEvent(s, join[x - 1], 0));
            }
        }
        return TS_OK;
    };
    // the eta exchange chain: restriction (this rank's sources, the second
    // pass of a two-pass exchange), halo-eta, then - once every rank's
    // stores have landed - the values peers restricted into this rank's
    // blocks and the halo copies that read them
    auto chain = [&](cudaStream_t c) -> int {
        if (h->r_send.nch) { launch_restrict(a, h->r_send.d, h->r_send.ch, h->r_send.nch, h->d_stage, c); ++n; if (tick(c, 16)) return TS_ERR_CUDA; }
        if (h->r_local.nch) { launch_restrict(a, h->r_local.d, h->r_local.ch, h->r_local.nch, h->d_stage, c); ++n; if (tick(c, 32)) return TS_ERR_CUDA; }
        if (h->n_heta) { launch_copies(a, h->d_heta, h->n_heta, false, c); ++n; if (tick(c, 48)) return TS_ERR_CUDA; }
        if (h->x_restrict || h->x_halo) { barrier(h, c); ++n; if (tick(c, 64)) return TS_ERR_CUDA; }
        if (h->r_recv.nch) { launch_restrict(a, h->r_recv.d, h->r_recv.ch, h->r_recv.nch, h->d_stage, c); ++n; if (tick(c, 80)) return TS_ERR_CUDA; }
        if (h->n_heta2) { launch_copies(a, h->d_heta2, h->n_heta2, false, c); ++n; if (tick(c, 96)) return TS_ERR_CUDA; }
        if (h->x_halo2) { barrier(h, c); ++n; if (tick(c, 65)) return TS_ERR_CUDA; }
        CK(cudaGetLastError());
        return TS_OK;
    };
    if (h->merged) {
        // merged exchange phases (build_merged): one launch per phase, the
        // received values after the phase barrier
        if (h->n_mx[0]) { launch_xops(a, h->d_mx[0], h->n_mx[0], s); ++n; if (tick(s, 13 * 16)) return TS_ERR_CUDA; }
        if (mark(2)) return TS_ERR_CUDA;
        if (h->mx_bar_eta) { barrier(h, s); ++n; if (tick(s, 64)) return TS_ERR_CUDA; }
        if (h->n_mx[1]) { launch_xops(a, h->d_mx[1], h->n_mx[1], s); ++n; if (tick(s, 80)) return TS_ERR_CUDA; }
        if (mark(3)) return TS_ERR_CUDA;
        if (int rc = march(0, s)) return rc;
        if (mark(4)) return TS_ERR_CUDA;
        if (mark(5)) return TS_ERR_CUDA;
        if (h->n_mx[2]) { launch_xops(a, h->d_mx[2], h->n_mx[2], s); ++n; if (tick(s, 14 * 16)) return TS_ERR_CUDA; }
        if (mark(6)) return TS_ERR_CUDA;
        if (h->mx_bar_flux) { barrier(h, s); ++n; if (tick(s, 66)) return TS_ERR_CUDA; }
        if (h->n_mx[3]) { launch_xops(a, h->d_mx[3], h->n_mx[3], s); ++n; if (tick(s, 176)) return TS_ERR_CUDA; }
        if (mark(7)) return TS_ERR_CUDA;
        CK(cudaGetLastError());
        if (nlaunch) *nlaunch = n;
        return TS_OK;
    }
    if (h->overlap) {
        // DESIGN.md §5/§7: the chain and then the march of the tiles that
        // read a cell it writes ("late" tiles: parents' ring lines, ghost
        // strips) on their own stream, beside the march of every other tile
        // - the finest level is never a parent, so most of the step's march
        // overlaps the whole exchange (peer stores and barriers included)
        CK(cudaEventRecord(h->ev_xfork, s));
        CK(cudaStreamWaitEvent(h->xs, h->ev_xfork, 0));
        if (int rc = chain(h->xs)) return rc;
        if (mark(2)) return TS_ERR_CUDA;
        if (mark(3)) return TS_ERR_CUDA;
        if (int rc = march(2, h->xs)) return rc;
        CK(cudaEventRecord(h->ev_xjoin, h->xs));
        if (int rc = march(1, s)) return rc;
        CK(cudaStreamWaitEvent(s, h->ev_xjoin, 0));
    } else {
        if (int rc = chain(s)) return rc;
        if (mark(2)) return TS_ERR_CUDA;
        if (mark(3)) return TS_ERR_CUDA;
        if (int rc = march(0, s)) return rc;
    }
    if (mark(4)) return TS_ERR_CUDA;
    if (h->n_edge) { launch_copies(a, h->d_edge, h->n_edge, h->edge_serial, s); ++n; if (tick(s, 128)) return TS_ERR_CUDA; }
    if (mark(5)) return TS_ERR_CUDA;
    if (h->p_send.nch) { launch_prolong(a, h->p_send.d, h->p_send.ch, h->p_send.nch, h->d_stage, s); ++n; if (tick(s, 144)) return TS_ERR_CUDA; }
    if (h->p_local.nch) { launch_prolong(a, h->p_local.d, h->p_local.ch, h->p_local.nch, h->d_stage, s); ++n; if (tick(s, 160)) return TS_ERR_CUDA; }
    if (h->x_prolong) { barrier(h, s); ++n; if (tick(s, 66)) return TS_ERR_CUDA; }
    if (h->p_recv.nch) { launch_prolong(a, h->p_recv.d, h->p_recv.ch, h->p_recv.nch, h->d_stage, s); ++n; if (tick(s, 176)) return TS_ERR_CUDA; }
    if (mark(6)) return TS_ERR_CUDA;
    if (h->n_hflux) { launch_copies(a, h->d_hflux, h->n_hflux, false, s); ++n; if (tick(s, 192)) return TS_ERR_CUDA; }
    // "output" is folded into the next step's K_mass (and the end-of-run
    // flush); the swap is the parity flip of the caller
    if (mark(7)) return TS_ERR_CUDA;
    CK(cudaGetLastError());
    if (nlaunch) *nlaunch = n;
    return TS_OK;
}

int enqueue_flush(ts_handle *h, cudaStream_t s, int buf)
{
    const StepArgs a = args_of(h, buf);
    launch_accumulate(a, h->d_all, h->n_all, s);
    CK(cudaGetLastError());
    return TS_OK;
}

// capture (once) and return the executable step graph of a buffer parity
int get_graph(ts_handle *h, int c, cudaGraphExec_t *out)
{
    if (!h->gexec[c]) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        int nl = 0;
        int rc = enqueue_step(h, h->stream, c, true, &nl);
        cudaError_t e = cudaStreamEndCapture(h->stream, &g);
        if (rc) return rc;
        if (e != cudaSuccess) return fail(TS_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
        h->launches = nl;
        size_t nn = 0;
        CK(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(g, nodes.data(), &nn));
        CK(cudaGraphInstantiate(&h->gexec[c], g, 0));
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeEventRecord) continue;
            cudaEvent_t ev;
            CK(cudaGraphEventRecordNodeGetEvent(nd, &ev));
            for (int k = 0; k < kPhaseEvents; ++k)
                if (ev == h->ev[k]) h->ev_node[c][k] = nd;
        }
        h->graph[c] = g;
    }
    *out = h->gexec[c];
    return TS_OK;
}

// the first step of a run: phase events of its own (read once the run is
// done, so the host never waits in the middle of a run)
int get_graph_first(ts_handle *h, int c, cudaGraphExec_t *out)
{
    if (!h->gexec_first[c]) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_step(h, h->stream, c, true, nullptr, h->ev_first);
        cudaError_t e = cudaStreamEndCapture(h->stream, &g);
        if (rc) return rc;
        if (e != cudaSuccess) return fail(TS_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
        CK(cudaGraphInstantiate(&h->gexec_first[c], g, 0));
        h->graph_first[c] = g;
    }
    *out = h->gexec_first[c];
    return TS_OK;
}

// capture (once) kStepsPerGraph steps from parity c (phase events only in
// the first, so timing samples stay one per graph)
int get_graph_multi(ts_handle *h, int c, cudaGraphExec_t *out)
{
    if (!h->gexec_multi[c]) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        int rc = 0;
        for (int k = 0; k < kStepsPerGraph && !rc; ++k)
            rc = enqueue_step(h, h->stream, c ^ (k & 1), k == 0, nullptr);
        cudaError_t e = cudaStreamEndCapture(h->stream, &g);
        if (rc) return rc;
        if (e != cudaSuccess) return fail(TS_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
        CK(cudaGraphInstantiate(&h->gexec_multi[c], g, 0));
        size_t nn = 0;
        CK(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(g, nodes.data(), &nn));
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeEventRecord) continue;
            cudaEvent_t ev;
            CK(cudaGraphEventRecordNodeGetEvent(nd, &ev));
            for (int k = 0; k < kPhaseEvents; ++k)
                if (ev == h->ev[k]) h->ev_node_multi[c][k] = nd;
        }
        h->graph_multi[c] = g;
    }
    *out = h->gexec_multi[c];
    return TS_OK;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Reference-layout (row-major, unpadded) <-> pitched device array geometry
struct FieldGeom {
    double *ptr;
    int rows, cols;     // reference shape
    int pitch;          // device pitch (doubles)
};

int io_reserve(ts_handle *h, size_t n)
{
    if (n <= h->io_len) return TS_OK;
    CK(cudaStreamSynchronize(h->stream));
    if (h->d_io) CK(cudaFree(h->d_io));
    h->d_io = nullptr;
    h->io_len = 0;
    CK(cudaMalloc((void **)&h->d_io, n * 8));
    h->io_len = n;
    return TS_OK;
}

int field_geom(ts_handle *h, int b, int field, FieldGeom *g)
{
    if (b < 0 || b >= h->nb) return fail(TS_ERR_INVALID, "block index %d out of range", b);
    const DevBlock &B = h->hb[b];
    if (h->desc[b].owner != h->rank) return fail(TS_ERR_INVALID, "block %d is not owned by rank %d", b, h->rank);
    const int ni = B.ni, nj = B.nj, c = h->cur;
    g->pitch = B.P;
    switch (field) {
    case TS_ETA_OLD: *g = {B.eta[c], ni + 4, nj + 4, B.P}; break;
    case TS_ETA_NEW: *g = {B.eta[c ^ 1], ni + 4, nj + 4, B.P}; break;
    case TS_M_OLD: *g = {B.m[c], ni + 5, nj + 4, B.P}; break;
    case TS_M_NEW: *g = {B.m[c ^ 1], ni + 5, nj + 4, B.P}; break;
    case TS_N_OLD: *g = {B.n[c], ni + 4, nj + 5, B.P}; break;
    case TS_N_NEW: *g = {B.n[c ^ 1], ni + 4, nj + 5, B.P}; break;
    case TS_H_EXT: *g = {B.h, ni + 4, nj + 4, B.P}; break;
    case TS_MAX_ETA: *g = {B.acc_eta, ni, nj, B.P}; break;
    case TS_MAX_SPEED: *g = {B.acc_speed, ni, nj, B.P}; break;
    case TS_MAX_INUNDATION: *g = {B.acc_inund, ni, nj, B.P}; break;
    default: return fail(TS_ERR_INVALID, "unknown field %d", field);
    }
    return TS_OK;
}

// index helpers into the pitched arrays (x, y are local cell / face indices)
inline int32_t pidx(int P, int x, int y) { return (x + TS_G) * P + (y + TS_G); }

// exchange._strip_slices (exchange.py:162-182): (layer, along) -> (x, y)
void eta_strip_xy(int side, bool sending, int ni, int nj, int along, int layer, int *x, int *y)
{
    switch (side) {
    case TS_WEST: *x = sending ? layer : -2 + layer; *y = along; break;
    case TS_EAST: *x = sending ? ni - 2 + layer : ni + layer; *y = along; break;
    case TS_SOUTH: *y = sending ? layer : -2 + layer; *x = along; break;
    default: *y = sending ? nj - 2 + layer : nj + layer; *x = along; break;
    }
}

// exchange._face_strip (exchange.py:185-215): returns (x, y) and the array
// (1 = m, 2 = n)
void face_strip_xy(int side, bool sending, bool normal, int ni, int nj, int along, int layer,
                   int *x, int *y, int *arr)
{
    const bool x_side = side <= TS_EAST;
    const bool low = side == TS_WEST || side == TS_SOUTH;
    const int n_edge = x_side ? ni : nj;
    int across;
    if (normal) across = sending ? (low ? 1 + layer : n_edge - 2 + layer) : (low ? -2 + layer : n_edge + 1 + layer);
    else        across = sending ? (low ? layer : n_edge - 2 + layer) : (low ? -2 + layer : n_edge + layer);
    if (x_side) { *x = across; *y = along; *arr = normal ? 1 : 2; }
    else        { *x = along; *y = across; *arr = normal ? 2 : 1; }
}

const int kOpp[4] = {TS_EAST, TS_WEST, TS_NORTH, TS_SOUTH};

struct DstKey {
    int32_t blk, arr, idx;
    bool operator==(const DstKey &o) const { return blk == o.blk && arr == o.arr && idx == o.idx; }
};
struct DstHash {
    size_t operator()(const DstKey &k) const
    {
        return std::hash<long long>()(((long long)k.blk << 34) ^ ((long long)k.arr << 32) ^ (unsigned)k.idx);
    }
};

// keep the LAST writer of every destination (the reference applies entries
// in order, runner.py:178-186), preserving order among survivors
std::vector<Copy> dedup_last(const std::vector<Copy> &in)
{
    std::unordered_map<DstKey, size_t, DstHash> last;
    last.reserve(in.size() * 2);
    for (size_t k = 0; k < in.size(); ++k) {
        const int arr = (in[k].src_blk >> 28) & 3;
        last[{in[k].dst_blk, arr, in[k].dst_idx}] = k;
    }
    std::vector<Copy> out;
    out.reserve(last.size());
    for (size_t k = 0; k < in.size(); ++k) {
        const int arr = (in[k].src_blk >> 28) & 3;
        if (last[{in[k].dst_blk, arr, in[k].dst_idx}] == k) out.push_back(in[k]);
    }
    return out;
}

template <typename Tv>
int upload(Tv **dptr, const std::vector<Tv> &v)
{
    if (v.empty()) return TS_OK;
    CK(cudaMalloc((void **)dptr, v.size() * sizeof(Tv)));
    CK(cudaMemcpy(*dptr, v.data(), v.size() * sizeof(Tv), cudaMemcpyHostToDevice));
    return TS_OK;
}

// ---------------------------------------------------------------------------
// Merged exchange phases.  Each exchange phase of the
// reference is a sequence of element writes: the eta phase is restriction
// (every value packed from the phase's input, then applied; coupling.py:
// 278-315) followed by the halo copies in order (exchange.py:218-275); the
// flux phase is the edge rules in order (kernels.py:274-306), prolongation
// (packed, then applied; coupling.py:318-340) and the flux halo copies.
// Replaying that sequence on the host with every value kept as an
// expression in the phase's INPUT state (a copy of a cell written earlier in
// the phase becomes that write's expression) leaves one write per
// destination whose reads are all phase inputs.  When no read cell is also
// written (checked), the writes are independent: one launch per phase and
// rank, each element run by the rank holding its source data.  An element
// whose destination is another rank's interior cell (which that rank's own
// kernels write earlier in the step) goes through the receiver's receive
// area and is applied after the phase barrier; ghost cells are stored
// straight into the peer's arena.  Phases that do not pass the checks keep
// the launch-per-stage path.
struct XExpr {
    int kind;           // 0 copy, 1 zero, 2 mean9 (eta patch at idx)
    int blk, arr;
    int32_t idx;
};
struct XWrite {
    XExpr e;
    int blk, arr;
    int32_t idx;
    int wave = 0;       // 1: its destination is read by another write of the phase
};

inline long long xkey(int b, int arr, int32_t idx) { return ((long long)b << 34) ^ ((long long)arr << 32) ^ (uint32_t)idx; }

// open-addressing map from a cell key (>= 0) to a value, sized once.
// LOCAL: for xkey layouts (block and array above bit 32, the element index
// below) the index is added linearly, so a phase's writes, which walk rows
// and strips, probe neighbouring slots; otherwise a full 64-bit mix
template <typename V, bool LOCAL = false>
struct FlatMap {
    std::vector<long long> keys;
    std::vector<V> vals;
    size_t mask = 0;
    void init(size_t n)
    {
        size_t cap = 16;
        while (cap < 2 * n + 16) cap <<= 1;
        keys.assign(cap, -1);
        vals.assign(cap, V{});
        mask = cap - 1;
    }
    static size_t slot0(long long k)
    {
        if (LOCAL) {
            uint64_t y = (uint64_t)k >> 32;
            y *= 0xff51afd7ed558ccdULL;
            y ^= y >> 29;
            return (size_t)(y + ((uint64_t)k & 0xffffffffULL));
        }
        uint64_t x = (uint64_t)k;
        x ^= x >> 33;
        x *= 0xff51afd7ed558ccdULL;
        x ^= x >> 33;
        x *= 0xc4ceb9fe1a85ec53ULL;
        x ^= x >> 33;
        return (size_t)x;
    }
    const V *find(long long k) const
    {
        for (size_t i = slot0(k) & mask;; i = (i + 1) & mask) {
            if (keys[i] == k) return &vals[i];
            if (keys[i] < 0) return nullptr;
        }
    }
    V &operator[](long long k)
    {
        size_t i = slot0(k) & mask;
        while (keys[i] >= 0 && keys[i] != k) i = (i + 1) & mask;
        keys[i] = k;
        return vals[i];
    }
};

int build_merged(ts_handle *h, const ts_desc *d, const std::vector<Copy> &eta_all, const std::vector<Copy> &flux_all)
{
    h->merged = false;
    if (const char *f = getenv("TSUNAMI_B200_MERGED"))
        if (f[0] == '0') return TS_OK;
    if (h->overlap) return TS_OK;
    const auto t_start = std::chrono::steady_clock::now();
    auto owner = [&](int b) { return d->blocks[b].owner; };
    auto P_of = [&](int b) { return h->hb[b].P; };
    // interior cells: written by the owner's own mass (eta) / march (m, n)
    auto interior = [&](int b, int arr, int32_t idx) {
        const int P = P_of(b);
        const int x = idx / P - TS_G, y = idx % P - TS_G;
        const int ni = d->blocks[b].ni, nj = d->blocks[b].nj;
        if (arr == 0) return x >= 0 && x < ni && y >= 0 && y < nj;
        if (arr == 1) return x >= 0 && x <= ni && y >= 0 && y < nj;
        return x >= 0 && x < ni && y >= 0 && y <= nj;
    };
    auto reads = [&](const XExpr &e, std::vector<long long> &out) {
        out.clear();
        if (e.kind == 0) out.push_back(xkey(e.blk, e.arr, e.idx));
        else if (e.kind == 2) {
            const int P = P_of(e.blk);
            for (int dy = 0; dy < 3; ++dy)
                for (int dx = 0; dx < 3; ++dx) out.push_back(xkey(e.blk, 0, e.idx + dx * P + dy));
        }
    };
    struct Phase {
        FlatMap<XExpr, true> w;                    // cell -> its current expression
        std::vector<XWrite> seq;
        bool ok = true;
        std::string why;                           // the first check that failed (verbose)
    };
    auto cell_str = [&](long long k) {
        const int b = (int)(k >> 34), arr = (int)((k >> 32) & 3);
        const int32_t idx = (int32_t)(k & 0xffffffffLL);
        const int P = P_of(b);
        char buf[96];
        snprintf(buf, sizeof buf, "block %d %s (%d, %d)", b, arr == 0 ? "eta" : (arr == 1 ? "m" : "n"),
                 idx / P - TS_G, idx % P - TS_G);
        return std::string(buf);
    };
    std::vector<long long> rd;
    auto subst = [&](Phase &ph, const XExpr &e) {
        if (e.kind != 0) return e;
        const XExpr *it = ph.w.find(xkey(e.blk, e.arr, e.idx));
        return it ? *it : e;
    };
    // a packed stage: every expression against the state before the stage
    auto packed = [&](Phase &ph, const std::vector<XWrite> &stage) {
        std::vector<XWrite> v = stage;
        for (auto &x : v) {
            if (x.e.kind == 2) {
                reads(x.e, rd);
                for (long long k : rd)
                    if (ph.w.find(k) && ph.ok) {          // a mean over cells written earlier
                        ph.ok = false;
                        ph.why = "a ring mean reads " + cell_str(k) + ", written earlier in the phase";
                    }
            } else {
                x.e = subst(ph, x.e);
            }
        }
        for (auto &x : v) {
            ph.w[xkey(x.blk, x.arr, x.idx)] = x.e;
            ph.seq.push_back(x);
        }
    };
    auto sequential = [&](Phase &ph, const std::vector<XWrite> &stage) {
        for (XWrite x : stage) {
            x.e = subst(ph, x.e);
            ph.w[xkey(x.blk, x.arr, x.idx)] = x.e;
            ph.seq.push_back(x);
        }
    };
    auto copies = [&](const std::vector<Copy> &cs) {
        std::vector<XWrite> v;
        for (const Copy &c : cs) {
            const int arr = (c.src_blk >> 28) & 3, sb = c.src_blk & 0x0fffffff;
            XExpr e = c.src_idx < 0 ? XExpr{1, c.dst_blk, arr, 0} : XExpr{0, sb, arr, c.src_idx};
            v.push_back(XWrite{e, c.dst_blk, arr, c.dst_idx});
        }
        return v;
    };
    Phase pe, pf;
    {
        size_t ne = eta_all.size(), nf = flux_all.size();
        for (int k = 0; k < d->n_restrict; ++k) ne += std::max(0, d->restrict_segs[k].parent_hi - d->restrict_segs[k].parent_lo);
        for (int k = 0; k < d->n_prolong; ++k) nf += 3 * (size_t)std::max(0, d->prolong_segs[k].parent_hi - d->prolong_segs[k].parent_lo);
        for (int k = 0; k < d->n_edges; ++k) nf += (size_t)std::max(0, d->edges[k].hi - d->edges[k].lo);
        pe.w.init(ne);
        pe.seq.reserve(ne);
        pf.w.init(nf);
        pf.seq.reserve(nf);
    }
    {
        std::vector<XWrite> r;
        for (int k = 0; k < d->n_restrict; ++k) {
            const ts_eta_segment &sg = d->restrict_segs[k];
            const bool ns = sg.side >= TS_SOUTH;
            for (int p = 0; p < sg.parent_hi - sg.parent_lo; ++p) {
                const int x0 = ns ? sg.child_lo + 3 * p : sg.ring_start, y0 = ns ? sg.ring_start : sg.child_lo + 3 * p;
                const int x = ns ? sg.parent_lo + p : sg.parent_line, y = ns ? sg.parent_line : sg.parent_lo + p;
                r.push_back(XWrite{XExpr{2, sg.child, 0, pidx(P_of(sg.child), x0, y0)}, sg.parent, 0,
                                   pidx(P_of(sg.parent), x, y)});
            }
        }
        packed(pe, r);
        sequential(pe, copies(eta_all));
    }
    {
        std::vector<Copy> edges;
        for (int k = 0; k < d->n_edges; ++k) {
            const ts_edge &e = d->edges[k];
            const ts_block_desc &B = d->blocks[e.block];
            const int P = P_of(e.block);
            const bool xs = e.side <= TS_EAST;
            const int arr = xs ? 1 : 2;
            const int n_edge = xs ? B.ni : B.nj;
            const int edge = (e.side == TS_WEST || e.side == TS_SOUTH) ? 0 : n_edge;
            const int inner = (e.side == TS_WEST || e.side == TS_SOUTH) ? 1 : n_edge - 1;
            for (int a = e.lo; a < e.hi; ++a) {
                const int dst = xs ? pidx(P, edge, a) : pidx(P, a, edge);
                const int src = e.kind == TS_REFLECTIVE ? -1 : (xs ? pidx(P, inner, a) : pidx(P, a, inner));
                edges.push_back(Copy{e.block | (arr << 28), e.block, src, dst});
            }
        }
        sequential(pf, copies(edges));
        std::vector<XWrite> pr;
        for (int k = 0; k < d->n_prolong; ++k) {
            const ts_flux_segment &sg = d->prolong_segs[k];
            const bool ns = sg.side >= TS_SOUTH;
            const int arr = ns ? 2 : 1;
            for (int p = 0; p < sg.parent_hi - sg.parent_lo; ++p) {
                const int px = ns ? sg.parent_lo + p : sg.parent_face_line, py = ns ? sg.parent_face_line : sg.parent_lo + p;
                for (int u = 0; u < 3; ++u) {
                    const int a = sg.child_lo + 3 * p + u;
                    const int cx = ns ? a : sg.child_face_line, cy = ns ? sg.child_face_line : a;
                    pr.push_back(XWrite{XExpr{0, sg.parent, arr, pidx(P_of(sg.parent), px, py)}, sg.child, arr,
                                        pidx(P_of(sg.child), cx, cy)});
                }
            }
        }
        packed(pf, pr);
        sequential(pf, copies(flux_all));
    }
    // one write per destination (the last), then: no read cell is written
    auto finish = [&](Phase &ph) {
        FlatMap<size_t, true> last;
        last.init(ph.seq.size());
        for (size_t k = 0; k < ph.seq.size(); ++k) last[xkey(ph.seq[k].blk, ph.seq[k].arr, ph.seq[k].idx)] = k;
        std::vector<XWrite> out;
        out.reserve(ph.seq.size());
        for (size_t k = 0; k < ph.seq.size(); ++k)
            if (*last.find(xkey(ph.seq[k].blk, ph.seq[k].arr, ph.seq[k].idx)) == k) out.push_back(ph.seq[k]);
        // a destination that another write reads (a parent ring cell that a
        // coarser restriction averages: the reference's packed order reads it
        // before it is overwritten) is written in a second wave: its value is
        // computed with the first wave (every read sees the phase's input)
        // into a staging slot and stored after every read of the phase
        FlatMap<size_t, true> pos;
        pos.init(out.size());
        for (size_t k = 0; k < out.size(); ++k) pos[xkey(out[k].blk, out[k].arr, out[k].idx)] = k;
        for (auto &x : out) {
            reads(x.e, rd);
            for (long long k : rd)
                if (const size_t *p = pos.find(k)) out[*p].wave = 1;
        }
        ph.seq.swap(out);
    };
    finish(pe);
    finish(pf);
    if (!pe.ok || !pf.ok) {
        if (getenv("TSUNAMI_B200_VERBOSE"))
            fprintf(stderr, "[tsunami_b200] rank %d: exchange phases not mergeable (eta: %s; flux: %s)\n", h->rank,
                    pe.ok ? "ok" : pe.why.c_str(), pf.ok ? "ok" : pf.why.c_str());
        return TS_OK;
    }
    // receive slots in global order (every rank computes the same), eta
    // phase first; they must fit the areas sized by the per-segment path
    std::vector<size_t> cap(h->nranks, 0), cur(h->nranks, 0);
    {
        std::vector<size_t> relems(h->nranks, 0);
        for (int k = 0; k < d->n_restrict; ++k) {
            const ts_eta_segment &sg = d->restrict_segs[k];
            if (owner(sg.child) != owner(sg.parent)) relems[owner(sg.parent)] += sg.parent_hi - sg.parent_lo;
        }
        for (int k = 0; k < d->n_prolong; ++k) {
            const ts_flux_segment &sg = d->prolong_segs[k];
            if (owner(sg.parent) != owner(sg.child)) relems[owner(sg.child)] += 3 * (size_t)(sg.parent_hi - sg.parent_lo);
        }
        cap = relems;
    }
    std::vector<XOp> lists[4];
    bool cross[2] = {false, false}, recv_used = false;
    size_t n_stage = 0;
    auto emit = [&](Phase &ph, std::vector<XOp> &src_list, std::vector<XOp> &recv_list, int which) -> bool {
        // group the elements by kind so warps stay uniform
        std::stable_sort(ph.seq.begin(), ph.seq.end(), [](const XWrite &a, const XWrite &b) { return a.e.kind > b.e.kind; });
        for (const XWrite &x : ph.seq) {
            const int dst_owner = owner(x.blk);
            const int exec = x.e.kind == 1 ? dst_owner : owner(x.e.blk);
            const int32_t src = (x.e.kind == 1 ? 0 : x.e.blk) | (x.e.kind << 28);
            if (exec != dst_owner) cross[which] = true;
            if (x.wave && exec == dst_owner) {
                // second wave, local: staged, stored with the received values
                if (exec == h->rank) {
                    const int32_t slot = (int32_t)n_stage++;
                    src_list.push_back(XOp{src, TS_XDST_RECV | h->nranks | (x.arr << 28), x.e.idx, slot});
                    recv_list.push_back(XOp{h->nranks | (3 << 28), x.blk | (x.arr << 28), slot, x.idx});
                }
            } else if (exec != dst_owner && (x.wave || interior(x.blk, x.arr, x.idx))) {
                if (cur[dst_owner] >= cap[dst_owner]) {
                    if (getenv("TSUNAMI_B200_VERBOSE"))
                        fprintf(stderr, "[tsunami_b200] rank %d: merged exchange: receive area of rank %d full\n",
                                h->rank, dst_owner);
                    return false;
                }
                const int32_t slot = (int32_t)cur[dst_owner]++;
                recv_used = true;
                if (exec == h->rank)
                    src_list.push_back(XOp{src, TS_XDST_RECV | dst_owner | (x.arr << 28), x.e.idx, slot});
                if (dst_owner == h->rank)
                    recv_list.push_back(XOp{h->rank | (3 << 28), x.blk | (x.arr << 28), slot, x.idx});
            } else if (exec == h->rank) {
                src_list.push_back(XOp{src, x.blk | (x.arr << 28), x.e.idx, x.idx});
            }
        }
        return true;
    };
    if (!emit(pe, lists[0], lists[1], 0) || !emit(pf, lists[2], lists[3], 1)) return TS_OK;
    if (n_stage) {
        CK(cudaMalloc((void **)&h->d_mstage, n_stage * sizeof(double)));
        h->recv_base[h->nranks] = h->d_mstage;
        CK(cudaMemcpy(h->d_recv, h->recv_base.data(), h->recv_base.size() * sizeof(double *),
                      cudaMemcpyHostToDevice));
    }
    for (int q = 0; q < 4; ++q) {
        h->n_mx[q] = (int64_t)lists[q].size();
        if (int rc = upload(&h->d_mx[q], lists[q])) return rc;
    }
    // the eta barrier orders every cross-rank store of the step before the
    // receivers' march (flux-phase ghost stores included: the receivers
    // first read them in the next step's march); the flux barrier orders the
    // received values, and keeps a sender from refilling a receive area
    // before its owner has applied it
    h->mx_bar_eta = cross[0] || cross[1];
    h->mx_bar_flux = recv_used;
    h->merged = true;
    if (getenv("TSUNAMI_B200_VERBOSE"))
        fprintf(stderr, "[tsunami_b200] rank %d: merged exchange: eta %lld + %lld received, flux %lld + %lld "
                        "received, barriers eta %d flux %d (%.3f s)\n", h->rank, (long long)h->n_mx[0],
                (long long)h->n_mx[1], (long long)h->n_mx[2], (long long)h->n_mx[3], (int)h->mx_bar_eta,
                (int)h->mx_bar_flux,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
    return TS_OK;
}

// carve one block's arrays out of an arena region (same order and sizes on
// every rank; the Manning slot is always reserved so layouts agree without
// knowing a peer block's Manning representation)
// row pitch (doubles) of a block's ghosted arrays: nj + 4 columns (+1 N
// face), rounded to 32 bytes (64- or 128-byte rows measured slower: mass
// +9 us, prolongation +7 us per Kochi step)
#ifndef TS_PITCH_ALIGN
#define TS_PITCH_ALIGN 4
#endif
size_t pitch_of(int nj)
{
    return align_up((size_t)nj + 5, TS_PITCH_ALIGN);
}

// Ghosted arrays start TS_BASE_SHIFT doubles past a 256-byte boundary, so
// that with the 32-byte row pitch every row's interior (column g = 2 on)
// starts on a 32-byte sector: the kernels' interior row reads and writes
// then cover whole sectors (no partial-sector writes for L2 to fill from
// DRAM at the row ends).
#ifndef TS_BASE_SHIFT
#define TS_BASE_SHIFT 2
#endif

void place_block(DevBlock &B, char *p, bool with_nman)
{
    const size_t P = B.P;
    const size_t cell = (size_t)(B.ni + 4) * P + TS_BASE_SHIFT, mrows = (size_t)(B.ni + 5) * P + TS_BASE_SHIFT;
    const size_t acc = (size_t)B.ni * P;
    auto take = [&](size_t n) { double *q = (double *)p; p += align_up(n * 8, 256); return q; };
    auto take_g = [&](size_t n) { return take(n) + TS_BASE_SHIFT; };
    B.eta[0] = take_g(cell); B.eta[1] = take_g(cell);
    B.m[0] = take_g(mrows); B.m[1] = take_g(mrows);
    B.n[0] = take_g(cell); B.n[1] = take_g(cell);
    B.h = take_g(cell);
    double *nm = take_g(cell);
    B.nman = with_nman ? nm : nullptr;
    B.acc_eta = take(acc); B.acc_speed = take(acc); B.acc_inund = take(acc);
}

int create_impl(const ts_desc *d, ts_handle *h)
{
    // TSUNAMI_B200_VERBOSE: seconds spent in each part of the setup
    const bool verbose = getenv("TSUNAMI_B200_VERBOSE") != nullptr;
    auto t_prev = std::chrono::steady_clock::now();
    auto setup_mark = [&](const char *what) {
        if (!verbose) return;
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[tsunami_b200] setup: %s %.3f s\n", what, std::chrono::duration<double>(t - t_prev).count());
        t_prev = t;
    };
    if (!d) return fail(TS_ERR_INVALID, "null descriptor");
    if (d->abi_version != TS_ABI_VERSION)
        return fail(TS_ERR_INVALID, "ABI version %d, library is %d", d->abi_version, TS_ABI_VERSION);
    if (d->n_blocks <= 0 || !d->blocks) return fail(TS_ERR_INVALID, "system has no blocks");
    if (!(d->dt > 0)) return fail(TS_ERR_INVALID, "dt must be positive, got %g", d->dt);
    h->device = d->device;
    h->rank = d->rank;
    h->nranks = d->n_ranks > 0 ? d->n_ranks : 1;
    h->dt = d->dt;
    h->g = d->gravity;
    h->thr = d->wet_threshold;
    h->nb = d->n_blocks;
    if (d->tile_rows > 0) {
        if ((d->tile_rows + 2) % 3 != 0)
            return fail(TS_ERR_INVALID, "tile_rows + 2 must be a multiple of 3, got %d", d->tile_rows);
        h->T = d->tile_rows;
    }
    CK(cudaSetDevice(h->device));
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    for (auto &st : h->side) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    // the exchange chain and the late tiles on high-priority streams: their
    // CTAs are dispatched ahead of the early tiles' remaining ones
    {
        int lo = 0, hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CK(cudaStreamCreateWithPriority(&h->xs, cudaStreamNonBlocking, hi));
        for (auto &st : h->side2) CK(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
    }
    CK(cudaEventCreateWithFlags(&h->ev_fork2, cudaEventDisableTiming));
    for (auto &e : h->ev_join2) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_xfork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_xjoin, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    for (auto &e : h->ev_join) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : h->ev) CK(cudaEventCreate(&e));
    for (auto &e : h->ev_first) CK(cudaEventCreate(&e));
    CK(cudaEventCreate(&h->t0));
    CK(cudaEventCreate(&h->t1));

    setup_mark("start");
    // ---- arena: every rank computes the same per-owner layout for ALL
    // blocks, so a peer block's arrays are (peer arena base + offset) once
    // the peer's arena is mapped (ts_ipc_import)
    h->desc.assign(d->blocks, d->blocks + d->n_blocks);
    h->hb.assign(h->nb, DevBlock{});
    h->hprof_buf.assign(h->nb, nullptr);
    h->off.assign(h->nb, 0);
    std::vector<size_t> owner_total(h->nranks, 0);
    for (int b = 0; b < h->nb; ++b) {
        const ts_block_desc &bd = d->blocks[b];
        if (bd.ni < 1 || bd.nj < 1) return fail(TS_ERR_INVALID, "block %lld is %dx%d", (long long)bd.block_id, bd.ni, bd.nj);
        if (bd.owner < 0 || bd.owner >= h->nranks)
            return fail(TS_ERR_INVALID, "block %lld: owner %d outside [0, %d)", (long long)bd.block_id, bd.owner, h->nranks);
        if (bd.owner == h->rank && ((!bd.h_ext && !bd.h_profile) || !bd.eta0))
            return fail(TS_ERR_INVALID, "block %lld: missing h_ext/eta0", (long long)bd.block_id);
        if (bd.h_profile && bd.h_axis != 0 && bd.h_axis != 1)
            return fail(TS_ERR_INVALID, "block %lld: h_axis %d", (long long)bd.block_id, bd.h_axis);
        const size_t P = pitch_of(bd.nj);
        const size_t cell = (size_t)(bd.ni + 4) * P + TS_BASE_SHIFT, mrows = (size_t)(bd.ni + 5) * P + TS_BASE_SHIFT;
        const size_t acc = (size_t)bd.ni * P;
        size_t need = 0;
        need += 2 * align_up(cell * 8, 256) + 2 * align_up(mrows * 8, 256) + 2 * align_up(cell * 8, 256);
        need += 2 * align_up(cell * 8, 256);         // h and (reserved) Manning n
        need += 3 * align_up(acc * 8, 256);
        h->off[b] = owner_total[bd.owner];
        owner_total[bd.owner] += need;
    }
    // receive areas of the cross-rank coupling (restriction values, then
    // prolongation values, in global segment order), after the blocks
    {
        std::vector<size_t> relems(h->nranks, 0);
        for (int k = 0; k < d->n_restrict; ++k) {
            const ts_eta_segment &sg = d->restrict_segs[k];
            if (sg.parent < 0 || sg.parent >= h->nb || sg.child < 0 || sg.child >= h->nb) continue;
            const int op = d->blocks[sg.parent].owner;
            if (d->blocks[sg.child].owner != op && sg.parent_hi > sg.parent_lo) relems[op] += sg.parent_hi - sg.parent_lo;
        }
        for (int k = 0; k < d->n_prolong; ++k) {
            const ts_flux_segment &sg = d->prolong_segs[k];
            if (sg.parent < 0 || sg.parent >= h->nb || sg.child < 0 || sg.child >= h->nb) continue;
            const int oc = d->blocks[sg.child].owner;
            if (d->blocks[sg.parent].owner != oc && sg.parent_hi > sg.parent_lo) relems[oc] += 3 * (size_t)(sg.parent_hi - sg.parent_lo);
        }
        h->recv_off.assign(h->nranks, 0);
        for (int o = 0; o < h->nranks; ++o) {
            h->recv_off[o] = owner_total[o];
            owner_total[o] += align_up(relems[o] * 8, 256);
        }
    }
    const size_t total = owner_total[h->rank];
    h->arena_bytes = total;
    if (total) {
        CK(cudaMalloc((void **)&h->arena, total));
        CK(cudaMemset(h->arena, 0, total));
    }
    for (int b = 0; b < h->nb; ++b) {
        const ts_block_desc &bd = d->blocks[b];
        DevBlock &B = h->hb[b];
        B.ni = bd.ni;
        B.nj = bd.nj;
        B.P = (int)pitch_of(bd.nj);
        B.order = b;
        B.r = d->dt / bd.dx;
        B.grr = d->gravity * B.r;
        B.dtg = d->dt * d->gravity;
        B.kf = (B.dtg * bd.manning) * bd.manning;
        B.has_nman = bd.nman_ext ? 1 : 0;
        if (bd.owner != h->rank) continue;
        place_block(B, h->arena + h->off[b], B.has_nman != 0);
        const size_t P = B.P;
        // h_ext / n_ext with ghosts (kernels.py:53-62, exchange.py:281-300):
        // copied, or built on the device from a 1-D profile
        if (bd.h_ext) {
            CK(cudaMemcpy2D(B.h, P * 8, bd.h_ext, (size_t)(bd.nj + 4) * 8, (size_t)(bd.nj + 4) * 8,
                            bd.ni + 4, cudaMemcpyHostToDevice));
        } else {
            // the profile stays on the device: the mass kernel reads it
            // instead of the interior of h
            const int len = bd.h_axis == 0 ? bd.ni : bd.nj;
            double *prof = nullptr;
            CK(cudaMalloc((void **)&prof, (size_t)std::max(bd.ni, bd.nj) * 8));
            CK(cudaMemcpy(prof, bd.h_profile, (size_t)len * 8, cudaMemcpyHostToDevice));
            launch_h_profile(B, prof, bd.h_axis, h->stream);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(h->stream));
            h->hprof_buf[b] = prof;
            B.hprof = prof;
            B.haxis = bd.h_axis;
            h->h_fill_pending = true;
        }
        if (B.nman)
            CK(cudaMemcpy2D(B.nman, P * 8, bd.nman_ext, (size_t)(bd.nj + 4) * 8, (size_t)(bd.nj + 4) * 8,
                            bd.ni + 4, cudaMemcpyHostToDevice));
        // set_initial_eta: interior of BOTH buffers (kernels.py:97-101)
        for (int k = 0; k < 2; ++k)
            CK(cudaMemcpy2D(B.eta[k] + 2 * P + 2, P * 8, bd.eta0, (size_t)bd.nj * 8, (size_t)bd.nj * 8,
                            bd.ni, cudaMemcpyHostToDevice));
    }
    // host-transfer staging sized once for the largest owned field, so that
    // field uploads / downloads never reallocate (cudaFree synchronises the
    // device and, with peers mapped, costs far more)
    {
        size_t io = 0;
        for (int b = 0; b < h->nb; ++b)
            if (d->blocks[b].owner == h->rank)
                io = std::max(io, (size_t)(d->blocks[b].ni + 5) * (size_t)(d->blocks[b].nj + 5));
        if (io)
            if (int rc = io_reserve(h, io)) return rc;
    }
    CK(cudaMalloc((void **)&h->d_blocks, sizeof(DevBlock) * h->nb));
    CK(cudaMemcpy(h->d_blocks, h->hb.data(), sizeof(DevBlock) * h->nb, cudaMemcpyHostToDevice));
    // signal area: peers' epochs + own epoch + the error word (peers adopt
    // it at every barrier); its IPC handle is exported
    CK(cudaMalloc((void **)&h->d_sig, (h->nranks + 2) * sizeof(unsigned long long)));
    CK(cudaMemset(h->d_sig, 0, (h->nranks + 1) * sizeof(unsigned long long)));
    h->d_err = h->d_sig + h->nranks + 1;
    CK(cudaMemset(h->d_err, 0xff, sizeof(unsigned long long)));
    CK(cudaMalloc((void **)&h->d_accflag, sizeof(int)));
    CK(cudaMemset(h->d_accflag, 0, sizeof(int)));

    setup_mark("arena+upload");
    // ---- march tiles: faces [0, ni+1) x N faces [0, nj+1)
    for (int k = 0; k < 4; ++k) h->groups[k].W = k + 1;
    auto width_group = [](int nj, int &W, int &w) {
        if (nj + 3 <= 128) { W = (nj + 3 + 31) / 32; w = nj + 1; }
        else { W = 4; w = 126; }
    };
    // A block of nj + 3 <= 128 columns may instead share 128-thread CTAs
    // with tiles of its own width packed side by side (nj + 3 threads each)
    // when that keeps more threads busy: nj = 36 packs 3 tiles into 117 of
    // 128 threads instead of one tile into 39 of 64 (Kochi's 270 m level:
    // momentum 1.479 -> 1.458 ms).  384-thread CTAs (1 per SM) for nj = 48
    // (7 tiles, 93 %) and 160-thread CTAs (2 per SM, 3 tiles, 96 %) were
    // slower: occupancy matters more than idle lanes.  TSUNAMI_B200_PACK=0
    // disables packing.
    bool pack = true;
    if (const char *f = getenv("TSUNAMI_B200_PACK")) pack = atoi(f) != 0;
    std::vector<int> gid(h->nb, -1);
    for (int b = 0; b < h->nb; ++b) {
        if (d->blocks[b].owner != h->rank) continue;
        const int nj = d->blocks[b].nj, L = nj + 3;
        int W, w;
        width_group(nj, W, w);
        gid[b] = W - 1;
        if (!pack || L > 128) continue;
        const double u_std = (double)L / (32 * W), u_pack = (double)((128 / L) * L) / 128;
        if (u_pack <= u_std + 0.03) continue;
        int k = 4;
        for (; k < (int)h->groups.size(); ++k)
            if (h->groups[k].lanes == L) break;
        if (k == (int)h->groups.size()) {
            if (k >= 8) continue;                        // graph branches are bounded
            Group g;
            g.W = 4;
            g.lanes = L;
            h->groups.push_back(g);
        }
        gid[b] = k;
    }
    // rows per tile of each group: the longest of 124 / 94 / 64 / ... that
    // still gives the group three waves of CTAs (long tiles recompute fewer
    // halo rows: T + 2 rows per T; Kochi's 60/48-wide group at 124 rows:
    // momentum 1.460 -> 1.445 ms), shorter for small groups (a tile's march
    // latency is proportional to its rows, and a group's last wave of long
    // tiles would otherwise set the momentum phase's length)
    if (d->tile_rows <= 0) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
        std::vector<double> rows(h->groups.size(), 0.0);
        for (int b = 0; b < h->nb; ++b) {
            if (gid[b] < 0) continue;
            int W, w;
            width_group(d->blocks[b].nj, W, w);
            rows[gid[b]] += (double)(d->blocks[b].ni + 1) * ((d->blocks[b].nj + 1 + w - 1) / w);
        }
        for (int k = 0; k < (int)h->groups.size(); ++k) {
            Group &gr = h->groups[k];
            const int tpc = momentum_tiles_per_cta(gr.W, gr.lanes);
            const double want = 3.0 * sms * 3;          // three waves of 3 CTAs per SM
            gr.T = 16;
            for (int T : {124, 94, 64, 48, 32, 24})
                if (rows[k] / T / tpc >= want) { gr.T = T; break; }
        }
        // TSUNAMI_B200_TROWS="W:T,..." (tuning): rows per tile of the plain
        // W-warp group (W = 1..4; T + 2 a multiple of 3)
        if (const char *f = getenv("TSUNAMI_B200_TROWS")) {
            for (const char *q = f; *q;) {
                int W = 0, T = 0, used = 0;
                if (sscanf(q, "%d:%d%n", &W, &T, &used) != 2) break;
                if (W >= 1 && W <= 4 && T >= 4 && (T + 2) % 3 == 0) h->groups[W - 1].T = T;
                q += used;
                if (*q == ',') ++q;
            }
        }
    } else {
        for (auto &gr : h->groups) gr.T = h->T;
    }
    for (int b = 0; b < h->nb; ++b) {
        if (gid[b] < 0) continue;
        const int ni = d->blocks[b].ni, nj = d->blocks[b].nj;
        int W, w;
        width_group(nj, W, w);
        Group &gr = h->groups[gid[b]];
        gr.nman |= d->blocks[b].nman_ext != nullptr;
        const int T = gr.T;
        for (int j0 = 0; j0 < nj + 1; j0 += w) {
            const int j1 = std::min(j0 + w, nj + 1);
            for (int i0 = 0; i0 < ni + 1; i0 += T)
                gr.tiles.push_back(Tile{b, i0, std::min(i0 + T, ni + 1), j0, j1, 0});
        }
    }
    // (the march tiles are uploaded once the exchange tables below have
    // split them into early and late ones)
    {
        // cell tiles of the flat kernels (mass + fold, flush): about
        // mass_cells cells each, whole rows up to 1024 columns
        int target = 8192;
        if (const char *f = getenv("TSUNAMI_B200_MASS_CELLS")) target = std::max(256, atoi(f));
        std::vector<Tile> all;
        for (int b = 0; b < h->nb; ++b) {
            if (d->blocks[b].owner != h->rank) continue;
            const int ni = d->blocks[b].ni, nj = d->blocks[b].nj;
            const int cw = std::min(nj, 1024);
            const int R = std::max(1, target / cw);
            for (int j0 = 0; j0 < nj; j0 += cw)
                for (int i0 = 0; i0 < ni; i0 += R)
                    all.push_back(Tile{b, i0, std::min(i0 + R, ni), j0, std::min(j0 + cw, nj), 0});
        }
        h->n_all = (int)all.size();
        if (int rc = upload(&h->d_all, all)) return rc;
    }

    auto owned = [&](int b) { return b >= 0 && b < h->nb && d->blocks[b].owner == h->rank; };
    auto check_blk = [&](int b) { return b >= 0 && b < h->nb; };
    size_t stage_len = 0;

    setup_mark("tiles");
    // ---- coupling segments (coupling.py:278-340).  Pass 1 validates,
    // flags cross-rank traffic and detects whether any written element is
    // also read in the same exchange (then the reference's pack-all-then-
    // apply order needs two passes); pass 2 builds this rank's lists.
    std::vector<size_t> recv_cur(h->nranks, 0);      // elements, per receiving owner
    auto build_lists = [&](auto &send, auto &local, auto &recv, auto make, int nseg, auto geom,
                           bool two_pass, int mult) -> int {
        using S = typename std::decay<decltype(make(0, 0, 0, 0))>::type;
        std::vector<S> vs, vl, vr;
        int64_t stage_cur = 0;
        for (int k = 0; k < nseg; ++k) {
            int src, dst, count;
            geom(k, src, dst, count);
            if (count == 0) continue;
            const int os = d->blocks[src].owner, od = d->blocks[dst].owner;
            const int64_t n = (int64_t)mult * count;
            int64_t roff = -1;
            if (os != od) {
                roff = (int64_t)recv_cur[od];
                recv_cur[od] += (size_t)n;
            }
            if (os == h->rank) {
                if (os != od) vs.push_back(make(k, 1, od, roff));
                else if (two_pass) {
                    vs.push_back(make(k, 1, -1, stage_cur));
                    vl.push_back(make(k, 2, -1, stage_cur));
                    stage_cur += n;
                } else {
                    vs.push_back(make(k, 0, -1, 0));
                }
            } else if (od == h->rank) {
                vr.push_back(make(k, 2, h->rank, roff));
            }
        }
        stage_len = std::max(stage_len, (size_t)stage_cur);
        auto up = [&](auto &L, std::vector<S> &v) -> int {
            if (int rc = upload(&L.d, v)) return rc;
            std::vector<int2> ch;
            for (int q = 0; q < (int)v.size(); ++q)
                for (int o = 0; o < mult * v[q].count; o += 256) ch.push_back(make_int2(q, o));
            L.nch = (int)ch.size();
            return upload(&L.ch, ch);
        };
        if (int rc = up(send, vs)) return rc;
        if (int rc = up(local, vl)) return rc;
        return up(recv, vr);
    };
    {
        // two-pass detection: a restricted parent cell that another segment
        // reads (written cells in an open-addressing set, reads looked up)
        size_t nw = 0;
        for (int k = 0; k < d->n_restrict; ++k)
            nw += (size_t)std::max(0, d->restrict_segs[k].parent_hi - d->restrict_segs[k].parent_lo);
        FlatMap<char> written;
        written.init(nw);
        std::vector<long long> read;
        read.reserve(9 * nw);
        auto key = [](int b, int x, int y) { return ((long long)b << 42) ^ ((long long)(x + 8) << 21) ^ (long long)(y + 8); };
        for (int k = 0; k < d->n_restrict; ++k) {
            const ts_eta_segment &sg = d->restrict_segs[k];
            if (!check_blk(sg.parent) || !check_blk(sg.child) || sg.side < 0 || sg.side > 3)
                return fail(TS_ERR_INVALID, "bad restriction segment %d", k);
            const int count = sg.parent_hi - sg.parent_lo;
            if (count < 0 || sg.child_hi - sg.child_lo != 3 * count)
                return fail(TS_ERR_INVALID, "restriction segment %d: spans disagree", k);
            if (count == 0) continue;
            const bool ns = sg.side >= TS_SOUTH;
            if (d->blocks[sg.child].owner != d->blocks[sg.parent].owner) h->x_restrict = true;
            for (int p = 0; p < count; ++p) {
                written[key(sg.parent, ns ? sg.parent_lo + p : sg.parent_line, ns ? sg.parent_line : sg.parent_lo + p)] = 1;
                for (int u = 0; u < 3; ++u)
                    for (int v = 0; v < 3; ++v) {
                        const int x = ns ? sg.child_lo + 3 * p + u : sg.ring_start + u;
                        const int y = ns ? sg.ring_start + v : sg.child_lo + 3 * p + v;
                        read.push_back(key(sg.child, x, y));
                    }
            }
        }
        for (long long r : read)
            if (written.find(r)) { h->r_two_pass = true; break; }
        auto make = [&](int k, int mode, int srank, int64_t first) {
            const ts_eta_segment &sg = d->restrict_segs[k];
            return RSeg{sg.child, sg.parent, sg.side >= TS_SOUTH, sg.child_lo, sg.ring_start, sg.parent_line,
                        sg.parent_lo, sg.parent_hi - sg.parent_lo, first, mode, srank};
        };
        auto geom = [&](int k, int &src, int &dst, int &count) {
            const ts_eta_segment &sg = d->restrict_segs[k];
            src = sg.child; dst = sg.parent; count = sg.parent_hi - sg.parent_lo;
        };
        if (int rc = build_lists(h->r_send, h->r_local, h->r_recv, make, d->n_restrict, geom, h->r_two_pass, 1))
            return rc;
    }
    {
        size_t nw = 0;
        for (int k = 0; k < d->n_prolong; ++k)
            nw += 3 * (size_t)std::max(0, d->prolong_segs[k].parent_hi - d->prolong_segs[k].parent_lo);
        FlatMap<char> written;
        written.init(nw);
        std::vector<long long> read;
        read.reserve(nw / 3 + 1);
        auto key = [](int b, int arr, int x, int y) {
            return ((long long)b << 44) ^ ((long long)arr << 42) ^ ((long long)(x + 8) << 21) ^ (long long)(y + 8);
        };
        for (int k = 0; k < d->n_prolong; ++k) {
            const ts_flux_segment &sg = d->prolong_segs[k];
            if (!check_blk(sg.parent) || !check_blk(sg.child) || sg.side < 0 || sg.side > 3)
                return fail(TS_ERR_INVALID, "bad prolongation segment %d", k);
            const int count = sg.parent_hi - sg.parent_lo;
            if (count < 0 || sg.child_hi - sg.child_lo != 3 * count)
                return fail(TS_ERR_INVALID, "prolongation segment %d: spans disagree", k);
            if (count == 0) continue;
            const bool ns = sg.side >= TS_SOUTH;
            if (d->blocks[sg.child].owner != d->blocks[sg.parent].owner) h->x_prolong = true;
            const int arr = ns ? 2 : 1;
            for (int p = 0; p < count; ++p) {
                read.push_back(key(sg.parent, arr, ns ? sg.parent_lo + p : sg.parent_face_line,
                                   ns ? sg.parent_face_line : sg.parent_lo + p));
                for (int u = 0; u < 3; ++u) {
                    const int a = sg.child_lo + 3 * p + u;
                    written[key(sg.child, arr, ns ? a : sg.child_face_line, ns ? sg.child_face_line : a)] = 1;
                }
            }
        }
        for (long long r : read)
            if (written.find(r)) { h->p_two_pass = true; break; }
        auto make = [&](int k, int mode, int srank, int64_t first) {
            const ts_flux_segment &sg = d->prolong_segs[k];
            return PSeg{sg.parent, sg.child, sg.side >= TS_SOUTH, sg.child_lo, sg.child_face_line,
                        sg.parent_face_line, sg.parent_lo, sg.parent_hi - sg.parent_lo, first, mode, srank};
        };
        auto geom = [&](int k, int &src, int &dst, int &count) {
            const ts_flux_segment &sg = d->prolong_segs[k];
            src = sg.parent; dst = sg.child; count = sg.parent_hi - sg.parent_lo;
        };
        if (int rc = build_lists(h->p_send, h->p_local, h->p_recv, make, d->n_prolong, geom, h->p_two_pass, 3))
            return rc;
    }
    // receive-area bases: own now, peers' as their arenas are mapped
    // [n_ranks] is this rank's staging of the merged phases' second-wave writes
    h->recv_base.assign(h->nranks + 1, nullptr);
    if (h->arena) h->recv_base[h->rank] = (double *)(h->arena + h->recv_off[h->rank]);
    CK(cudaMalloc((void **)&h->d_recv, (h->nranks + 1) * sizeof(double *)));
    CK(cudaMemcpy(h->d_recv, h->recv_base.data(), (h->nranks + 1) * sizeof(double *), cudaMemcpyHostToDevice));
    if (stage_len) CK(cudaMalloc((void **)&h->d_stage, stage_len * sizeof(double)));

    setup_mark("coupling");
    // ---- halo strips (exchange.py:218-275) as deduplicated element copies
    std::vector<Copy> eta_all, flux_all;          // every rank's, for the merged phases
    {
        std::vector<Copy> eta, flux;
        for (int k = 0; k < d->n_halo; ++k) {
            const ts_halo_entry &e = d->halo[k];
            if (!check_blk(e.sender) || !check_blk(e.receiver) || e.side < 0 || e.side > 3)
                return fail(TS_ERR_INVALID, "bad halo entry %d", k);
            const int span = e.send_hi - e.send_lo;
            if (span < 0 || e.recv_hi - e.recv_lo != span)
                return fail(TS_ERR_INVALID, "halo entry %d: spans disagree", k);
            const ts_block_desc &S = d->blocks[e.sender], &R = d->blocks[e.receiver];
            if (S.owner != R.owner) h->x_halo = true;
            const int Ps = h->hb[e.sender].P, Pr = h->hb[e.receiver].P;
            const int rside = kOpp[e.side];
            for (int l = 0; l < 2; ++l)
                for (int a = 0; a < span; ++a) {
                    int sx, sy, rx, ry;
                    eta_strip_xy(e.side, true, S.ni, S.nj, e.send_lo + a, l, &sx, &sy);
                    eta_strip_xy(rside, false, R.ni, R.nj, e.recv_lo + a, l, &rx, &ry);
                    eta.push_back(Copy{e.sender, e.receiver, pidx(Ps, sx, sy), pidx(Pr, rx, ry)});
                }
            for (int normal = 1; normal >= 0; --normal) {
                const int len = normal ? span : span + 1;
                for (int l = 0; l < 2; ++l)
                    for (int a = 0; a < len; ++a) {
                        int sx, sy, sarr, rx, ry, rarr;
                        face_strip_xy(e.side, true, normal, S.ni, S.nj, e.send_lo + a, l, &sx, &sy, &sarr);
                        face_strip_xy(rside, false, normal, R.ni, R.nj, e.recv_lo + a, l, &rx, &ry, &rarr);
                        flux.push_back(Copy{e.sender | (sarr << 28), e.receiver, pidx(Ps, sx, sy), pidx(Pr, rx, ry)});
                    }
            }
        }
        eta = dedup_last(eta);
        flux = dedup_last(flux);
        eta_all = eta;
        flux_all = flux;
        // cells a peer's restriction writes (parent ring lines of a child
        // on another rank): a halo copy reading one must follow the
        // received restriction
        std::unordered_set<long long> xr;
        auto ckey = [](int b, long long idx) { return ((long long)b << 40) ^ idx; };
        for (int k = 0; k < d->n_restrict; ++k) {
            const ts_eta_segment &sg = d->restrict_segs[k];
            if (d->blocks[sg.child].owner == d->blocks[sg.parent].owner) continue;
            const bool ns = sg.side >= TS_SOUTH;
            const int Pp = h->hb[sg.parent].P;
            for (int q = 0; q < sg.parent_hi - sg.parent_lo; ++q)
                xr.insert(ckey(sg.parent, pidx(Pp, ns ? sg.parent_lo + q : sg.parent_line,
                                               ns ? sg.parent_line : sg.parent_lo + q)));
        }
        std::vector<Copy> eta_own, eta_own2, flux_own;
        for (auto &c : eta) {
            const int sb = c.src_blk & 0x0fffffff;
            const bool hazard = xr.count(ckey(sb, c.src_idx)) != 0;
            if (hazard && d->blocks[sb].owner != d->blocks[c.dst_blk].owner) h->x_halo2 = true;
            if (owned(sb)) (hazard ? eta_own2 : eta_own).push_back(c);
        }
        for (auto &c : flux) if (owned(c.src_blk & 0x0fffffff)) flux_own.push_back(c);
        h->n_heta = (int64_t)eta_own.size();
        h->n_heta2 = (int64_t)eta_own2.size();
        h->n_hflux = (int64_t)flux_own.size();
        if (int rc = upload(&h->d_heta, eta_own)) return rc;
        if (int rc = upload(&h->d_heta2, eta_own2)) return rc;
        // march tiles that read a cell the exchange chain writes on this
        // rank (peers' halo stores, received restriction values, the halo
        // copies after them) march after it; the others beside it
        {
            std::vector<std::vector<int>> late_rows(h->nb);
            auto mark_row = [&](int b, int x) { late_rows[b].push_back(x); };
            // every cell the chain writes into this rank's blocks: halo
            // destinations (own copies and peers' stores) and restricted
            // parent cells (whichever rank restricts them)
            for (auto &c : eta)
                if (owned(c.dst_blk)) mark_row(c.dst_blk, c.dst_idx / h->hb[c.dst_blk].P - TS_G);
            for (int k = 0; k < d->n_restrict; ++k) {
                const ts_eta_segment &sg = d->restrict_segs[k];
                if (!owned(sg.parent)) continue;
                const bool ns = sg.side >= TS_SOUTH;
                for (int q = 0; q < sg.parent_hi - sg.parent_lo; ++q) mark_row(sg.parent, ns ? sg.parent_lo + q : sg.parent_line);
            }
            for (auto &v : late_rows) {
                std::sort(v.begin(), v.end());
                v.erase(std::unique(v.begin(), v.end()), v.end());
            }
            // measured: Kochi-1.0 2.061 vs 2.062 ms at 1 GPU,
            // 0.763-0.770 vs 0.714 ms at 4 GPUs - the late tiles (every
            // parent level's) start only after the chain and finish after the
            // early ones; so opt-in (TSUNAMI_B200_OVERLAP=1)
            h->overlap = false;
            if (const char *f = getenv("TSUNAMI_B200_OVERLAP"))
                h->overlap = atoi(f) != 0 && (!eta.empty() || d->n_restrict > 0);
            for (auto &gr : h->groups) {
                std::vector<Tile> early, late;
                for (const Tile &t : gr.tiles) {
                    // a tile reads cell rows [i0 - 2, i1]
                    const auto &v = late_rows[t.blk];
                    auto it = std::lower_bound(v.begin(), v.end(), t.i0 - 2);
                    const bool is_late = h->overlap && it != v.end() && *it <= t.i1;
                    (is_late ? late : early).push_back(t);
                }
                gr.n_early = (int)early.size();
                gr.tiles = early;
                gr.tiles.insert(gr.tiles.end(), late.begin(), late.end());
                if (int rc = upload(&gr.d, gr.tiles)) return rc;
            }
        }
        // the same strips of h: fill_bathymetry_halos (exchange.py:281-300)
        // for device-built bathymetry (every rank whose blocks send)
        {
            bool any_profile = false;
            for (int b = 0; b < h->nb; ++b) any_profile |= d->blocks[b].h_profile != nullptr;
            std::vector<Copy> hf = eta_own;
            hf.insert(hf.end(), eta_own2.begin(), eta_own2.end());
            for (auto &c : hf) c.src_blk |= 3 << 28;
            h->n_hfill = (int64_t)hf.size();
            if (int rc = upload(&h->d_hfill, hf)) return rc;
            h->h_fill_pending = any_profile && h->n_hfill > 0;
        }
        if (int rc = upload(&h->d_hflux, flux_own)) return rc;
    }
    setup_mark("halos");
    // ---- outer-boundary edges (kernels.py:274-306)
    {
        std::vector<Copy> edges;
        std::unordered_set<long long> dsts;
        bool serial = false;
        for (int k = 0; k < d->n_edges; ++k) {
            const ts_edge &e = d->edges[k];
            if (!check_blk(e.block) || e.side < 0 || e.side > 3 || (e.kind != TS_REFLECTIVE && e.kind != TS_RADIATION))
                return fail(TS_ERR_INVALID, "bad edge %d", k);
            if (!owned(e.block)) continue;
            const ts_block_desc &B = d->blocks[e.block];
            const int P = h->hb[e.block].P;
            const bool xs = e.side <= TS_EAST;
            const int arr = xs ? 1 : 2;
            const int n_edge = xs ? B.ni : B.nj;
            const int edge = (e.side == TS_WEST || e.side == TS_SOUTH) ? 0 : n_edge;
            const int inner = (e.side == TS_WEST || e.side == TS_SOUTH) ? 1 : n_edge - 1;
            for (int a = e.lo; a < e.hi; ++a) {
                const int dst = xs ? pidx(P, edge, a) : pidx(P, a, edge);
                const int src = e.kind == TS_REFLECTIVE ? -1 : (xs ? pidx(P, inner, a) : pidx(P, a, inner));
                if (src >= 0 && dsts.count(((long long)e.block << 34) ^ ((long long)arr << 32) ^ (unsigned)src)) serial = true;
                dsts.insert(((long long)e.block << 34) ^ ((long long)arr << 32) ^ (unsigned)dst);
                edges.push_back(Copy{e.block | (arr << 28), e.block, src, dst});
            }
        }
        // a radiation source written by an earlier edge, or a repeated
        // destination, needs the reference's sequential order
        if (dsts.size() != edges.size()) serial = true;
        for (auto &c : edges)
            if (c.src_idx >= 0 && dsts.count(((long long)c.dst_blk << 34) ^ ((long long)((c.src_blk >> 28) & 3) << 32) ^ (unsigned)c.src_idx))
                serial = true;
        h->edge_serial = serial;
        h->n_edge = (int64_t)edges.size();
        if (int rc = upload(&h->d_edge, edges)) return rc;
    }
    setup_mark("edges");
    if (int rc = build_merged(h, d, eta_all, flux_all)) return rc;
    CK(cudaDeviceSynchronize());
    if (const char *f = getenv("TSUNAMI_B200_MOMPAR")) h->mom_par = f[0] == '1';
    h->peer_arena.assign(h->nranks, nullptr);
    h->peer_sig.assign(h->nranks, nullptr);
    h->peer_arena[h->rank] = h->arena;
    h->peer_sig[h->rank] = h->d_sig;
    CK(cudaMalloc((void **)&h->d_peer_sig, h->nranks * sizeof(unsigned long long *)));
    CK(cudaMemcpy(h->d_peer_sig, h->peer_sig.data(), h->nranks * sizeof(unsigned long long *),
                  cudaMemcpyHostToDevice));
    cudaGraphExec_t g;
    setup_mark("merged");
    return get_graph(h, 0, &g);
}

// one block's entry of the device table after a host-side change (ordered
// with the library stream's kernels)
int push_block_entry(ts_handle *h, int b)
{
    CK(cudaMemcpyAsync(h->d_blocks + b, &h->hb[b], sizeof(DevBlock), cudaMemcpyHostToDevice, h->stream));
    return TS_OK;
}

// a host write of a block's h_ext: its interior is no longer a 1-D profile
int drop_profile(ts_handle *h, int b)
{
    if (!h->hb[b].hprof) return TS_OK;
    h->hb[b].hprof = nullptr;
    return push_block_entry(h, b);
}

// the siblings' bathymetry strips of device-built h_ext, once, before the
// first step (peer arenas are mapped by then; the first step's halo-eta
// barrier orders them before any rank's momentum reads ghost h)
int fill_bathymetry(ts_handle *h)
{
    if (!h->h_fill_pending) return TS_OK;
    if (h->imported != h->nranks - 1) return TS_OK;       // ts_run reports the missing peers
    const StepArgs a = args_of(h, h->cur);
    launch_copies(a, h->d_hfill, h->n_hfill, false, h->stream);
    CK(cudaGetLastError());
    h->h_fill_pending = false;
    return TS_OK;
}

int check_error(ts_handle *h)
{
    unsigned long long key;
    CK(cudaMemcpy(&key, h->d_err, sizeof key, cudaMemcpyDeviceToHost));
    if (key == TS_NO_ERROR) return TS_OK;
    const int order = (int)(key >> 50), what = (int)((key >> 48) & 3);
    const long long i = (long long)((key >> 24) & 0xffffff) - 4, j = (long long)(key & 0xffffff) - 4;
    if (what == 3)
        return fail(TS_ERR_CUDA, "rank %d: peer rank %lld did not reach a phase barrier within 30 s", h->rank, i);
    static const char *names[3] = {"water level", "x-flux", "y-flux"};
    return fail(TS_ERR_NUMERICS, "non-finite %s in block %lld at local cell (%lld, %lld)", names[what],
                (long long)h->desc[order].block_id, i, j);
}

}  // namespace

extern "C" {

const char *ts_last_error(void) { return g_err.c_str(); }
int ts_abi_version(void) { return TS_ABI_VERSION; }

int ts_create(const ts_desc *desc, ts_handle **out)
{
    if (!out) return fail(TS_ERR_INVALID, "null output handle");
    *out = nullptr;
    ts_handle *h = new ts_handle();
    const auto t0 = std::chrono::steady_clock::now();
    int rc = create_impl(desc, h);
    if (getenv("TSUNAMI_B200_VERBOSE"))
        fprintf(stderr, "[tsunami_b200] rank %d: ts_create %.3f s\n", h->rank,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    if (rc) {
        std::string keep = g_err;
        ts_destroy(h);
        g_err = keep;
        return rc;
    }
    *out = h;
    return TS_OK;
}

int ts_run(ts_handle *h, int64_t n_steps)
{
    if (!h) return fail(TS_ERR_INVALID, "null handle");
    if (n_steps < 0) return fail(TS_ERR_INVALID, "negative step count");
    CK(cudaSetDevice(h->device));
    if (int rc = check_error(h)) return rc;
    if (n_steps == 0) return TS_OK;
    if (h->imported != h->nranks - 1)
        return fail(TS_ERR_INVALID, "rank %d: %d of %d peers mapped; call ts_ipc_import for every peer first",
                    h->rank, h->imported, h->nranks - 1);
    cudaStream_t s = h->stream;
    if (int rc = fill_bathymetry(h)) return rc;
    // the first step of every run folds nothing: the previous run ended with
    // the flush (or no step ran yet), and host writes made since then must
    // not reach the maxima (the reference folds only in a step's output
    // phase, kernels.py:322-343)
    CK(cudaMemsetAsync(h->d_accflag, 0, sizeof(int), s));
    CK(cudaEventRecord(h->t0, s));
    // first step: its phase events apportion the call's device time to the
    // routines (runner.ROUTINES)
    cudaGraphExec_t g;
    if (int rc = get_graph_first(h, h->cur, &g)) return rc;
    CK(cudaGraphLaunch(g, s));
    float ph[7] = {0};
    h->cur ^= 1;
    h->steps += 1;
    int64_t done = 1;
    CK(cudaMemsetAsync(h->d_accflag, 1, 1, s));
    const int64_t chunk = 256;
    double sum_mass = 0, sum_mom = 0, sum_step = 0;
    int64_t timed = 0;
    while (done < n_steps) {
        const int64_t n = std::min(chunk, n_steps - done);
        if (h->timing && h->pool.size() < (size_t)(5 * n)) {
            const size_t old = h->pool.size();
            h->pool.resize(5 * n);
            for (size_t k = old; k < h->pool.size(); ++k) CK(cudaEventCreate(&h->pool[k]));
        }
        // steps go out in graphs of kStepsPerGraph (single-step graphs for
        // the remainder); timing samples the first step of every
        // kTimingEvery-th step's graph: rebinding a launch's event nodes
        // costs it ~9 us of device time (measured), so the other launches
        // run their graph untouched
        int64_t ns = 0;
        for (int64_t k = 0; k < n;) {
            if (n - k >= kStepsPerGraph) {
                if (int rc = get_graph_multi(h, h->cur, &g)) return rc;
                const bool sample = h->timing && k % kTimingEvery == 0;
                if (sample)
                    for (int q = 0; q < 5; ++q)
                        CK(cudaGraphExecEventRecordNodeSetEvent(g, h->ev_node_multi[h->cur][kTimed[q]],
                                                                h->pool[5 * ns + q]));
                CK(cudaGraphLaunch(g, s));
                if (sample) {
                    for (int q = 0; q < 5; ++q)
                        CK(cudaGraphExecEventRecordNodeSetEvent(g, h->ev_node_multi[h->cur][kTimed[q]],
                                                                h->ev[kTimed[q]]));
                    ++ns;
                }
                k += kStepsPerGraph;       // an even count: the parity is unchanged
                continue;
            }
            if (int rc = get_graph(h, h->cur, &g)) return rc;
            const bool sample = h->timing && k % kTimingEvery == 0;
            if (sample)
                for (int q = 0; q < 5; ++q)
                    CK(cudaGraphExecEventRecordNodeSetEvent(g, h->ev_node[h->cur][kTimed[q]], h->pool[5 * ns + q]));
            CK(cudaGraphLaunch(g, s));
            if (sample) {     // leave the graph's own phase events in place
                for (int q = 0; q < 5; ++q)
                    CK(cudaGraphExecEventRecordNodeSetEvent(g, h->ev_node[h->cur][kTimed[q]], h->ev[kTimed[q]]));
                ++ns;
            }
            h->cur ^= 1;
            ++k;
        }
        h->steps += n;
        done += n;
        if (h->timing || done < n_steps) {
            CK(cudaStreamSynchronize(s));
            if (int rc = check_error(h)) return rc;
        }
        if (h->timing) {
            for (int64_t k = 0; k < ns; ++k) {
                float a = 0, b = 0, c = 0;
                CK(cudaEventElapsedTime(&a, h->pool[5 * k + 0], h->pool[5 * k + 1]));
                CK(cudaEventElapsedTime(&b, h->pool[5 * k + 2], h->pool[5 * k + 3]));
                CK(cudaEventElapsedTime(&c, h->pool[5 * k + 0], h->pool[5 * k + 4]));
                sum_mass += a; sum_mom += b; sum_step += c;
            }
            timed += ns;
        }
    }
    if (timed) {
        h->mass_s = sum_mass / timed / 1e3;
        h->mom_s = sum_mom / timed / 1e3;
        h->step_s = sum_step / timed / 1e3;
    }
    if (int rc = enqueue_flush(h, s, h->cur)) return rc;
    CK(cudaEventRecord(h->t1, s));
    CK(cudaStreamSynchronize(s));
    float tot = 0;
    CK(cudaEventElapsedTime(&tot, h->t0, h->t1));
    for (int k = 0; k < 7; ++k) CK(cudaEventElapsedTime(&ph[k], h->ev_first[k], h->ev_first[k + 1]));
    const double sum = ph[0] + ph[1] + ph[2] + ph[3] + ph[4] + ph[5] + ph[6];
    const double scale = sum > 0 ? (tot / 1e3) / sum : 0.0;
    // ROUTINES order: mass, momentum, restrict, prolong, halo-eta, halo-flux,
    // output.  momentum includes the edge rules like Simulation._momentum
    // (runner.py:111-117); output is fused into mass.
    h->routines[0] = ph[0] * scale;
    h->routines[1] = (ph[3] + ph[4]) * scale;
    h->routines[2] = ph[1] * scale;
    h->routines[3] = ph[5] * scale;
    h->routines[4] = ph[2] * scale;
    h->routines[5] = ph[6] * scale;
    h->routines[6] = 0.0;
    h->total = tot / 1e3;
    return check_error(h);
}

int ts_trace_step(ts_handle *h, int32_t *labels, float *us, int32_t cap, int32_t *count)
{
    if (!h) return fail(TS_ERR_INVALID, "null handle");
    if (cap < 0 || (cap > 0 && (!labels || !us)) || !count) return fail(TS_ERR_INVALID, "bad trace buffers");
    CK(cudaSetDevice(h->device));
    if (int rc = check_error(h)) return rc;
    if (h->imported != h->nranks - 1)
        return fail(TS_ERR_INVALID, "rank %d: %d of %d peers mapped; call ts_ipc_import for every peer first",
                    h->rank, h->imported, h->nranks - 1);
    if (int rc = fill_bathymetry(h)) return rc;
    while (h->trace_ev.size() < 96) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        h->trace_ev.push_back(e);
    }
    h->trace_label.clear();
    // as ts_run(1): the step folds nothing of the past (the previous run
    // ended with its fold) and its own maxima are folded after it
    CK(cudaMemsetAsync(h->d_accflag, 0, sizeof(int), h->stream));
    h->tracing = true;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue_step(h, h->stream, h->cur, false, nullptr);
    cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    h->tracing = false;
    if (rc) return rc;
    if (e != cudaSuccess) return fail(TS_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
    cudaGraphExec_t x;
    CK(cudaGraphInstantiate(&x, g, 0));
    CK(cudaGraphLaunch(x, h->stream));
    if (int rc2 = enqueue_flush(h, h->stream, h->cur ^ 1)) return rc2;
    CK(cudaStreamSynchronize(h->stream));
    CK(cudaGraphExecDestroy(x));
    CK(cudaGraphDestroy(g));
    h->cur ^= 1;
    h->steps += 1;
    const int n = (int)h->trace_label.size() - 1;
    *count = n;
    for (int k = 0; k < n && k < cap; ++k) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, h->trace_ev[k], h->trace_ev[k + 1]));
        labels[k] = h->trace_label[k + 1];
        us[k] = ms * 1e3f;
    }
    return check_error(h);
}

int ts_device_barrier(ts_handle *h)
{
    if (!h) return fail(TS_ERR_INVALID, "null handle");
    if (h->nranks < 2) return TS_OK;
    if (h->imported != h->nranks - 1)
        return fail(TS_ERR_INVALID, "rank %d: %d of %d peers mapped; call ts_ipc_import for every peer first",
                    h->rank, h->imported, h->nranks - 1);
    CK(cudaSetDevice(h->device));
    barrier(h, h->stream);
    CK(cudaGetLastError());
    return TS_OK;
}

int ts_set_timing(ts_handle *h, int32_t on)
{
    if (!h) return fail(TS_ERR_INVALID, "null handle");
    h->timing = on != 0;
    return TS_OK;
}

int ts_phase(ts_handle *h, int32_t phase)
{
    if (!h) return fail(TS_ERR_INVALID, "null handle");
    CK(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    if (int rc = fill_bathymetry(h)) return rc;
    const StepArgs a = args_of(h, h->cur);
    switch (phase) {
    case TS_PH_MASS: launch_mass(a, h->d_all, h->n_all, false, s); break;
    case TS_PH_RESTRICT:
        launch_restrict(a, h->r_send.d, h->r_send.ch, h->r_send.nch, h->d_stage, s);
        launch_restrict(a, h->r_local.d, h->r_local.ch, h->r_local.nch, h->d_stage, s);
        if (h->x_restrict) barrier(h, s);
        launch_restrict(a, h->r_recv.d, h->r_recv.ch, h->r_recv.nch, h->d_stage, s);
        break;
    case TS_PH_HALO_ETA:
        launch_copies(a, h->d_heta, h->n_heta, false, s);
        launch_copies(a, h->d_heta2, h->n_heta2, false, s);
        if (h->x_halo || h->x_halo2) barrier(h, s);
        break;
    case TS_PH_MOMENTUM:
        for (Group &gr : h->groups) {
            if (!gr.tiles.empty())
                launch_momentum(a, gr.d, (int)gr.tiles.size(), gr.W, gr.T, gr.lanes, gr.nman, s);
        }
        break;
    case TS_PH_EDGES: launch_copies(a, h->d_edge, h->n_edge, h->edge_serial, s); break;
    case TS_PH_PROLONG:
        launch_prolong(a, h->p_send.d, h->p_send.ch, h->p_send.nch, h->d_stage, s);
        launch_prolong(a, h->p_local.d, h->p_local.ch, h->p_local.nch, h->d_stage, s);
        if (h->x_prolong) barrier(h, s);
        launch_prolong(a, h->p_recv.d, h->p_recv.ch, h->p_recv.nch, h->d_stage, s);
        break;
    case TS_PH_HALO_FLUX: launch_copies(a, h->d_hflux, h->n_hflux, false, s); break;
    case TS_PH_OUTPUT:
        if (int rc = enqueue_flush(h, s, h->cur ^ 1)) return rc;
        break;
    case TS_PH_SWAP: h->cur ^= 1; return TS_OK;
    default: return fail(TS_ERR_INVALID, "unknown phase %d", phase);
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    return check_error(h);
}

int ts_get_field(ts_handle *h, int32_t block, int32_t field, double *out, int64_t len)
{
    if (!h || !out) return fail(TS_ERR_INVALID, "null argument");
    CK(cudaSetDevice(h->device));
    if (int rc = fill_bathymetry(h)) return rc;
    FieldGeom g;
    if (int rc = field_geom(h, block, field, &g)) return rc;
    if (len != (int64_t)g.rows * g.cols) return fail(TS_ERR_INVALID, "length %lld != %d x %d", (long long)len, g.rows, g.cols);
    CK(cudaSetDevice(h->device));
    if (field == TS_H_EXT)
        if (int rc = drop_profile(h, block)) return rc;
    if (int rc = io_reserve(h, (size_t)len)) return rc;
    launch_repitch(h->d_io, g.cols, g.ptr, g.pitch, g.rows, g.cols, h->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, h->d_io, (size_t)len * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return TS_OK;
}

int ts_set_field(ts_handle *h, int32_t block, int32_t field, const double *in, int64_t len)
{
    if (!h || !in) return fail(TS_ERR_INVALID, "null argument");
    CK(cudaSetDevice(h->device));
    if (int rc = fill_bathymetry(h)) return rc;
    FieldGeom g;
    if (int rc = field_geom(h, block, field, &g)) return rc;
    if (len != (int64_t)g.rows * g.cols) return fail(TS_ERR_INVALID, "length %lld != %d x %d", (long long)len, g.rows, g.cols);
    CK(cudaSetDevice(h->device));
    if (int rc = io_reserve(h, (size_t)len)) return rc;
    CK(cudaMemcpyAsync(h->d_io, in, (size_t)len * 8, cudaMemcpyHostToDevice, h->stream));
    launch_repitch(g.ptr, g.pitch, h->d_io, g.cols, g.rows, g.cols, h->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    return TS_OK;
}

int ts_set_initial_eta(ts_handle *h, int32_t block, const double *eta0, int64_t len)
{
    if (!h || !eta0) return fail(TS_ERR_INVALID, "null argument");
    FieldGeom g;
    if (int rc = field_geom(h, block, TS_ETA_OLD, &g)) return rc;
    const DevBlock &B = h->hb[block];
    if (len != (int64_t)B.ni * B.nj) return fail(TS_ERR_INVALID, "length %lld != %d x %d", (long long)len, B.ni, B.nj);
    CK(cudaSetDevice(h->device));
    if (int rc = io_reserve(h, (size_t)len)) return rc;
    CK(cudaMemcpyAsync(h->d_io, eta0, (size_t)len * 8, cudaMemcpyHostToDevice, h->stream));
    for (int k = 0; k < 2; ++k)
        launch_repitch(B.eta[k] + 2 * (size_t)B.P + 2, B.P, h->d_io, B.nj, B.ni, B.nj, h->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    return TS_OK;
}

void *ts_host_alloc(int64_t bytes)
{
    void *p = nullptr;
    if (bytes <= 0 || cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocPortable) != cudaSuccess) return nullptr;
    return p;
}

void ts_host_free(void *p)
{
    if (p) cudaFreeHost(p);
}

namespace {

int bulk_reserve(ts_handle *h, size_t elems, size_t njobs)
{
    if (elems > h->bulk_len) {
        CK(cudaStreamSynchronize(h->stream));
        if (h->d_bulk) CK(cudaFree(h->d_bulk));
        h->d_bulk = nullptr;
        h->bulk_len = 0;
        CK(cudaMalloc((void **)&h->d_bulk, elems * 8));
        h->bulk_len = elems;
    }
    if (njobs > h->jobs_len) {
        CK(cudaStreamSynchronize(h->stream));
        if (h->d_jobs) CK(cudaFree(h->d_jobs));
        h->d_jobs = nullptr;
        h->jobs_len = 0;
        CK(cudaMalloc((void **)&h->d_jobs, njobs * sizeof(Repitch)));
        h->jobs_len = njobs;
    }
    return TS_OK;
}

int run_jobs(ts_handle *h, const std::vector<Repitch> &jobs)
{
    if (jobs.empty()) return TS_OK;
    int64_t mx = 0;
    for (auto &j : jobs) mx = std::max(mx, j.rows * j.cols);
    CK(cudaMemcpyAsync(h->d_jobs, jobs.data(), jobs.size() * sizeof(Repitch), cudaMemcpyHostToDevice, h->stream));
    launch_repitch_batch(h->d_jobs, (int)jobs.size(), mx, h->stream);
    CK(cudaGetLastError());
    return TS_OK;
}

}  // namespace

int ts_reset(ts_handle *h)
{
    if (!h) return fail(TS_ERR_INVALID, "null handle");
    CK(cudaSetDevice(h->device));
    for (int b = 0; b < h->nb; ++b) {
        if (h->desc[b].owner != h->rank) continue;
        const DevBlock &B = h->hb[b];
        const size_t P = B.P, cell = (size_t)(B.ni + 4) * P, mrows = (size_t)(B.ni + 5) * P;
        const size_t acc = (size_t)B.ni * P;
        for (int k = 0; k < 2; ++k) {
            CK(cudaMemsetAsync(B.eta[k], 0, cell * 8, h->stream));
            CK(cudaMemsetAsync(B.m[k], 0, mrows * 8, h->stream));
            CK(cudaMemsetAsync(B.n[k], 0, cell * 8, h->stream));
        }
        for (double *a : {B.acc_eta, B.acc_speed, B.acc_inund}) CK(cudaMemsetAsync(a, 0, acc * 8, h->stream));
    }
    CK(cudaMemsetAsync(h->d_err, 0xff, sizeof(unsigned long long), h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->cur = 0;
    h->steps = 0;
    return TS_OK;
}

int ts_upload_inputs(ts_handle *h, int32_t n, const int32_t *blocks, const double *const *h_ext,
                     const double *const *eta0)
{
    if (!h || n < 0 || (n && (!blocks || !h_ext || !eta0))) return fail(TS_ERR_INVALID, "null argument");
    CK(cudaSetDevice(h->device));
    if (int rc = fill_bathymetry(h)) return rc;
    size_t total = 0;
    for (int k = 0; k < n; ++k) {
        FieldGeom g;
        if (int rc = field_geom(h, blocks[k], TS_H_EXT, &g)) return rc;
        if (!eta0[k]) return fail(TS_ERR_INVALID, "block %d: null input", blocks[k]);
        const DevBlock &B = h->hb[blocks[k]];
        total += (h_ext[k] ? (size_t)g.rows * g.cols : 0) + (size_t)B.ni * B.nj;
    }
    if (int rc = bulk_reserve(h, total, 3 * (size_t)n)) return rc;
    std::vector<Repitch> jobs;
    size_t off = 0;
    for (int k = 0; k < n; ++k) {
        const DevBlock &B = h->hb[blocks[k]];
        const size_t he = h_ext[k] ? (size_t)(B.ni + 4) * (B.nj + 4) : 0, ee = (size_t)B.ni * B.nj;
        double *sh = h->d_bulk + off, *se = sh + he;
        if (he) {                          // (NULL: bathymetry left as is, e.g. ts_upload_profiles)
            if (int rc = drop_profile(h, blocks[k])) return rc;
            CK(cudaMemcpyAsync(sh, h_ext[k], he * 8, cudaMemcpyHostToDevice, h->stream));
            jobs.push_back(Repitch{B.h, sh, B.P, B.nj + 4, B.ni + 4, B.nj + 4});
        }
        CK(cudaMemcpyAsync(se, eta0[k], ee * 8, cudaMemcpyHostToDevice, h->stream));
        // set_initial_eta: the interior of both water-level buffers
        for (int q = 0; q < 2; ++q)
            jobs.push_back(Repitch{B.eta[q] + 2 * (size_t)B.P + 2, se, B.P, B.nj, B.ni, B.nj});
        off += he + ee;
    }
    if (int rc = run_jobs(h, jobs)) return rc;
    CK(cudaStreamSynchronize(h->stream));
    return TS_OK;
}

int ts_upload_profiles(ts_handle *h, int32_t n, const int32_t *blocks, const double *const *profiles,
                       const int32_t *axes)
{
    if (!h || n < 0 || (n && (!blocks || !profiles || !axes))) return fail(TS_ERR_INVALID, "null argument");
    CK(cudaSetDevice(h->device));
    if (int rc = fill_bathymetry(h)) return rc;
    size_t total = 0;
    for (int k = 0; k < n; ++k) {
        FieldGeom g;
        if (int rc = field_geom(h, blocks[k], TS_H_EXT, &g)) return rc;
        if (!profiles[k] || (axes[k] != 0 && axes[k] != 1))
            return fail(TS_ERR_INVALID, "block %d: bad profile", blocks[k]);
        const DevBlock &B = h->hb[blocks[k]];
        total += axes[k] == 0 ? B.ni : B.nj;
    }
    (void)total;
    for (int k = 0; k < n; ++k) {
        const int b = blocks[k];
        DevBlock &B = h->hb[b];
        const size_t len = axes[k] == 0 ? B.ni : B.nj;
        if (!h->hprof_buf[b]) CK(cudaMalloc((void **)&h->hprof_buf[b], (size_t)std::max(B.ni, B.nj) * 8));
        CK(cudaMemcpyAsync(h->hprof_buf[b], profiles[k], len * 8, cudaMemcpyHostToDevice, h->stream));
        launch_h_profile(B, h->hprof_buf[b], axes[k], h->stream);
        B.hprof = h->hprof_buf[b];
        B.haxis = axes[k];
        if (int rc = push_block_entry(h, b)) return rc;
    }
    CK(cudaGetLastError());
    // the siblings' strips (exchange.py:281-300), once every rank's
    // profiles are expanded: before this rank's next step
    h->h_fill_pending = h->n_hfill > 0;
    if (h->nranks == 1) {
        if (int rc = fill_bathymetry(h)) return rc;
    }
    CK(cudaStreamSynchronize(h->stream));
    return TS_OK;
}

int ts_download_fields(ts_handle *h, int32_t n, const int32_t *blocks, int32_t nf, const int32_t *fields,
                       double *const *out)
{
    if (!h || n < 0 || nf < 0 || (n && nf && (!blocks || !fields || !out)))
        return fail(TS_ERR_INVALID, "null argument");
    CK(cudaSetDevice(h->device));
    if (int rc = fill_bathymetry(h)) return rc;
    std::vector<FieldGeom> geo((size_t)n * nf);
    size_t total = 0;
    for (int k = 0; k < n; ++k)
        for (int f = 0; f < nf; ++f) {
            FieldGeom &g = geo[(size_t)k * nf + f];
            if (int rc = field_geom(h, blocks[k], fields[f], &g)) return rc;
            if (!out[(size_t)k * nf + f]) return fail(TS_ERR_INVALID, "null output buffer");
            total += (size_t)g.rows * g.cols;
        }
    if (int rc = bulk_reserve(h, total, geo.size())) return rc;
    std::vector<Repitch> jobs;
    std::vector<size_t> offs;
    size_t off = 0;
    for (auto &g : geo) {
        jobs.push_back(Repitch{h->d_bulk + off, g.ptr, g.cols, g.pitch, g.rows, g.cols});
        offs.push_back(off);
        off += (size_t)g.rows * g.cols;
    }
    if (int rc = run_jobs(h, jobs)) return rc;
    for (size_t q = 0; q < geo.size(); ++q)
        CK(cudaMemcpyAsync(out[q], h->d_bulk + offs[q], (size_t)geo[q].rows * geo[q].cols * 8,
                           cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return TS_OK;
}

int ts_error_info(ts_handle *h, int32_t *block, int32_t *what, int64_t *i, int64_t *j)
{
    if (!h) return fail(TS_ERR_INVALID, "null handle");
    unsigned long long key;
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpy(&key, h->d_err, sizeof key, cudaMemcpyDeviceToHost));
    if (key == TS_NO_ERROR) {
        if (block) *block = -1;
        return TS_OK;
    }
    if (block) *block = (int32_t)(key >> 50);
    if (what) *what = (int32_t)((key >> 48) & 3);
    if (i) *i = (int64_t)((key >> 24) & 0xffffff) - 4;
    if (j) *j = (int64_t)(key & 0xffffff) - 4;
    return TS_OK;
}

int ts_timings(ts_handle *h, double *routines7, double *total)
{
    if (!h) return fail(TS_ERR_INVALID, "null handle");
    if (routines7) std::memcpy(routines7, h->routines, sizeof h->routines);
    if (total) *total = h->total;
    return TS_OK;
}

int64_t ts_steps_done(ts_handle *h) { return h ? h->steps : -1; }
int64_t ts_device_bytes(ts_handle *h) { return h ? (int64_t)h->arena_bytes : -1; }
int32_t ts_launches_per_step(ts_handle *h) { return h ? h->launches : -1; }

int ts_kernel_seconds(ts_handle *h, double *mass_s, double *momentum_s, double *step_s)
{
    if (!h) return fail(TS_ERR_INVALID, "null handle");
    if (mass_s) *mass_s = h->mass_s;
    if (momentum_s) *momentum_s = h->mom_s;
    if (step_s) *step_s = h->step_s;
    return TS_OK;
}

int ts_stream(ts_handle *h, void **stream)
{
    if (!h || !stream) return fail(TS_ERR_INVALID, "null argument");
    *stream = (void *)h->stream;
    return TS_OK;
}

void ts_destroy(ts_handle *h)
{
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (auto &g : h->gexec_multi)
        if (g) cudaGraphExecDestroy(g);
    for (auto &g : h->graph_multi)
        if (g) cudaGraphDestroy(g);
    for (auto &g : h->gexec)
        if (g) cudaGraphExecDestroy(g);
    for (auto &g : h->gexec_first)
        if (g) cudaGraphExecDestroy(g);
    for (auto &g : h->graph_first)
        if (g) cudaGraphDestroy(g);
    for (auto &e : h->ev_first)
        if (e) cudaEventDestroy(e);
    for (auto &g : h->graph)
        if (g) cudaGraphDestroy(g);
    for (auto &gr : h->groups) {
        cudaFree(gr.d);
    }
    cudaFree(h->d_all);
    for (auto *L : {&h->r_send, &h->r_local, &h->r_recv}) {
        cudaFree(L->d);
        cudaFree(L->ch);
    }
    for (auto *L : {&h->p_send, &h->p_local, &h->p_recv}) {
        cudaFree(L->d);
        cudaFree(L->ch);
    }
    cudaFree(h->d_recv);
    cudaFree(h->d_heta);
    cudaFree(h->d_hfill);
    cudaFree(h->d_hflux);
    cudaFree(h->d_edge);
    cudaFree(h->d_stage);
    cudaFree(h->d_io);
    cudaFree(h->d_bulk);
    cudaFree(h->d_jobs);
    cudaFree(h->d_accflag);
    cudaFree(h->d_blocks);
    for (int p = 0; p < (int)h->peer_arena.size(); ++p)
        if (p != h->rank) {
            if (h->peer_arena[p]) cudaIpcCloseMemHandle(h->peer_arena[p]);
            if (h->peer_sig[p]) cudaIpcCloseMemHandle(h->peer_sig[p]);
        }
    cudaFree(h->d_sig);
    cudaFree(h->d_peer_sig);
    cudaFree(h->arena);
    for (auto &e : h->ev)
        if (e) cudaEventDestroy(e);
    for (auto &e : h->pool) cudaEventDestroy(e);
    if (h->t0) cudaEventDestroy(h->t0);
    if (h->t1) cudaEventDestroy(h->t1);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    for (auto &e : h->ev_join)
        if (e) cudaEventDestroy(e);
    for (auto &st : h->side)
        if (st) cudaStreamDestroy(st);
    if (h->xs) cudaStreamDestroy(h->xs);
    for (auto &st : h->side2)
        if (st) cudaStreamDestroy(st);
    for (auto &e : h->ev_join2)
        if (e) cudaEventDestroy(e);
    if (h->ev_fork2) cudaEventDestroy(h->ev_fork2);
    if (h->ev_xfork) cudaEventDestroy(h->ev_xfork);
    if (h->ev_xjoin) cudaEventDestroy(h->ev_xjoin);
    cudaFree(h->d_heta2);
    for (auto *p : h->d_mx) cudaFree(p);
    cudaFree(h->d_mstage);
    for (double *p : h->hprof_buf) cudaFree(p);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

int ts_ipc_export(ts_handle *h, void *out, int64_t len)
{
    if (!h || !out) return fail(TS_ERR_INVALID, "null argument");
    if (len < (int64_t)(2 * sizeof(cudaIpcMemHandle_t) + 8)) return fail(TS_ERR_INVALID, "IPC blob too short");
    CK(cudaSetDevice(h->device));
    char *o = (char *)out;
    std::memset(o, 0, (size_t)len);
    if (h->arena) CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)o, h->arena));
    CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)(o + sizeof(cudaIpcMemHandle_t)), h->d_sig));
    const int64_t bytes = (int64_t)h->arena_bytes;
    std::memcpy(o + 2 * sizeof(cudaIpcMemHandle_t), &bytes, 8);
    return TS_OK;
}

int ts_ipc_import(ts_handle *h, int32_t peer, const void *in, int64_t len)
{
    if (!h || !in) return fail(TS_ERR_INVALID, "null argument");
    if (peer < 0 || peer >= h->nranks || peer == h->rank) return fail(TS_ERR_INVALID, "bad peer rank %d", peer);
    if (len < (int64_t)(2 * sizeof(cudaIpcMemHandle_t) + 8)) return fail(TS_ERR_INVALID, "IPC blob too short");
    CK(cudaSetDevice(h->device));
    const char *b = (const char *)in;
    int64_t bytes = 0;
    std::memcpy(&bytes, b + 2 * sizeof(cudaIpcMemHandle_t), 8);
    void *arena = nullptr, *sig = nullptr;
    if (bytes > 0) {
        cudaIpcMemHandle_t ha;
        std::memcpy(&ha, b, sizeof ha);
        CK(cudaIpcOpenMemHandle(&arena, ha, cudaIpcMemLazyEnablePeerAccess));
    }
    cudaIpcMemHandle_t hs;
    std::memcpy(&hs, b + sizeof(cudaIpcMemHandle_t), sizeof hs);
    CK(cudaIpcOpenMemHandle(&sig, hs, cudaIpcMemLazyEnablePeerAccess));
    h->peer_arena[peer] = (char *)arena;
    h->peer_sig[peer] = (unsigned long long *)sig;
    h->recv_base[peer] = arena ? (double *)((char *)arena + h->recv_off[peer]) : nullptr;
    CK(cudaMemcpy(h->d_recv, h->recv_base.data(), h->recv_base.size() * sizeof(double *), cudaMemcpyHostToDevice));
    for (int k = 0; k < h->nb; ++k)
        if (h->desc[k].owner == peer) place_block(h->hb[k], (char *)arena + h->off[k], false);
    CK(cudaMemcpy(h->d_blocks, h->hb.data(), sizeof(DevBlock) * h->nb, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_peer_sig, h->peer_sig.data(), h->nranks * sizeof(unsigned long long *),
                  cudaMemcpyHostToDevice));
    h->imported += 1;
    return TS_OK;
}

void ts_cbrt_host(const double *in, double *out, int64_t n)
{
    for (int64_t k = 0; k < n; ++k) out[k] = ts_cbrt(in[k]);
}

int ts_cbrt_device(int32_t device, const double *in, double *out, int64_t n)
{
    if (n <= 0) return TS_OK;
    CK(cudaSetDevice(device));
    double *d = nullptr;
    CK(cudaMalloc((void **)&d, 2 * n * sizeof(double)));
    CK(cudaMemcpy(d, in, n * sizeof(double), cudaMemcpyHostToDevice));
    launch_cbrt(d, d + n, n, 0);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, d + n, n * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaFree(d));
    return TS_OK;
}

}  // extern "C"
