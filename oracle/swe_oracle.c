/*
 * TEST INFRASTRUCTURE — CPU oracle for the nested-grid shallow-water step.
 *
 * A plain-C restatement of the reference's per-step algorithm
 * (/root/reference/pkg/src/blockswe/{kernels,coupling,exchange,runner}.py),
 * used ONLY by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs, and only as the checker.  It is never linked into
 * or called by the product (paper_2408_07609_b200/).
 *
 * Faithfulness rules:
 *  - same per-block ghosted layout as BlockState (kernels.py:39-62):
 *    eta/h/wet (ni+4)x(nj+4), m (ni+5)x(nj+4), n (ni+4)x(nj+5), C order,
 *    axis 0 = x (i), axis 1 = y (j, contiguous), halo g = 2;
 *  - an explicit wet array maintained exactly where the reference writes it
 *    (kernels.py:103-105, 155; exchange.py:255-257; coupling.py:315), so the
 *    product's derived-wet design is checked against it, not assumed;
 *  - the same evaluation order, no FMA contraction (built with
 *    -ffp-contract=off), numpy maximum/sign semantics, IEEE / and sqrt;
 *  - np.cbrt replaced by oracle_cbrt (cbrt_oracle.h) — the "cbrt-aligned"
 *    oracle; golden fixtures pin it to the reference run with the same cbrt.
 *  - exchange phases pack everything, then apply in the reference's apply
 *    order (runner.py:268-291), so overlapping reads/writes and duplicate
 *    ghost writes resolve exactly as in the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include "cbrt_oracle.h"

#define G 2

typedef struct {
    int64_t ni, nj;
    double *eta[2], *m[2], *n[2];
    uint8_t *wet;
    double *h;
    double *nman;       /* per-cell (ni+4)x(nj+4) or NULL for scalar */
    double nman_s;
    double dx;
    double *max_eta, *max_speed, *max_inund;   /* ni x nj */
    int64_t block_id;
} OBlock;

typedef struct {
    int64_t code;       /* 0 ok, 1 water level, 2 x-flux, 3 y-flux, 4/5 kernel fault x/y */
    int64_t block;      /* index into the block array */
    int64_t i, j;
    double value;
} OErr;

/* numpy scalar maximum: (a >= b || isnan(a)) ? a : b   (NaN propagating) */
static inline double np_max(double a, double b) { return (a >= b || a != a) ? a : b; }
/* np.sign: +1 / -1 / 0 (for +-0) / NaN */
static inline double np_sign(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : (x == 0.0 ? 0.0 : x)); }

int64_t oracle_threads(int64_t n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads((int)n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

void oracle_cbrt_array(const double *in, double *out, int64_t n)
{
    for (int64_t k = 0; k < n; ++k) out[k] = oracle_cbrt(in[k]);
}

/* ------------------------------------------------------------------ mass
 * kernels.py:123-155 */
int64_t oracle_mass(OBlock *b, int64_t cur, double dt, double thr, OErr *err)
{
    const int64_t ni = b->ni, nj = b->nj;
    const int64_t sc = nj + 4, sn = nj + 5;
    double *eo = b->eta[cur], *en = b->eta[1 - cur];
    double *m = b->m[cur], *n = b->n[cur];
    double *e = (double *)malloc(sizeof(double) * (size_t)(ni * nj > 0 ? ni * nj : 1));
    const double r = dt / b->dx;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ni; ++i) {
        for (int64_t j = 0; j < nj; ++j) {
            double div = r * (m[(G + i + 1) * sc + G + j] - m[(G + i) * sc + G + j])
                       + r * (n[(G + i) * sn + G + j + 1] - n[(G + i) * sn + G + j]);
            int64_t c = (G + i) * sc + G + j;
            double eta_old = eo[c], h = b->h[c];
            double v = eta_old - div;
            if (!b->wet[c] && div != 0.0) v = np_max(eta_old, -h) - div;
            if (div != 0.0 && h + v < 0.0) v = -h;
            e[i * nj + j] = v;
        }
    }
    for (int64_t k = 0; k < ni * nj; ++k) {
        if (!isfinite(e[k])) {
            err->code = 1; err->i = k / nj; err->j = k % nj;
            free(e);
            return 1;
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ni; ++i)
        for (int64_t j = 0; j < nj; ++j) {
            int64_t c = (G + i) * sc + G + j;
            double v = e[i * nj + j];
            en[c] = v;
            b->wet[c] = (b->h[c] + v >= thr);
        }
    free(e);
    return 0;
}

/* -------------------------------------------------------------- momentum
 * _momentum_axis, kernels.py:158-249.  Views are strided so the y-pass runs
 * the identical code on "transposed" arrays (kernels.py:265-269). */
typedef struct { double *p; int64_t rs, cs; } V2;
typedef struct { uint8_t *p; int64_t rs, cs; } W2;
#define AT(v, a, b) ((v).p[(int64_t)(a) * (v).rs + (int64_t)(b) * (v).cs])

static int64_t momentum_axis(V2 eta, V2 h, W2 wet, V2 nman, int nman_is_scalar, double nman_s,
                             V2 f_old, V2 f_new, V2 q_old, int64_t n, int64_t m,
                             double dx, double dt, double grav, double thr, OErr *err)
{
    const int64_t H = n + 3, W = m + 2;   /* faces -1..n+1, columns -1..m */
    const size_t N = (size_t)(H * W);
    double *dface = malloc(N * 8), *grad = malloc(N * 8), *dsafe = malloc(N * 8);
    double *fadv = malloc(N * 8), *fcross = malloc(N * 8), *f0 = malloc(N * 8), *qbar = malloc(N * 8);
    uint8_t *both = malloc(N), *active = malloc(N);
    int all_wet = 1;
    for (int64_t a = 0; a < H && all_wet; ++a)
        for (int64_t c = 0; c < W; ++c)
            if (!AT(wet, a, c + 1) || !AT(wet, a + 1, c + 1)) { all_wet = 0; break; }

#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < H; ++a) {
        for (int64_t c = 0; c < W; ++c) {
            size_t k = (size_t)(a * W + c);
            double el = AT(eta, a, c + 1), er = AT(eta, a + 1, c + 1);
            double hl = AT(h, a, c + 1), hr = AT(h, a + 1, c + 1);
            int wl = AT(wet, a, c + 1), wr = AT(wet, a + 1, c + 1);
            f0[k] = AT(f_old, a + 1, c + 1);
            qbar[k] = 0.25 * ((AT(q_old, a, c + 1) + AT(q_old, a + 1, c + 1))
                              + (AT(q_old, a, c + 2) + AT(q_old, a + 1, c + 2)));
            double df = 0.5 * ((hl + el) + (hr + er));
            double gr = er - el;
            int bo = 1, ac = 1;
            if (!all_wet) {
                bo = wl && wr;
                ac = bo;
                if (wl && !wr) {            /* front_r, kernels.py:191-196 */
                    double d_r = el + hr;
                    ac = (d_r >= thr);
                    df = d_r;
                    gr = np_max(er, -hr) - el;
                } else if (!wl && wr) {     /* front_l, kernels.py:197-202 */
                    double d_l = er + hl;
                    ac = (d_l >= thr);
                    df = d_l;
                    gr = er - np_max(el, -hl);
                }
            }
            dface[k] = df; grad[k] = gr; both[k] = (uint8_t)bo; active[k] = (uint8_t)ac;
        }
    }
    if (!all_wet) {                         /* kernels.py:206-211 */
        for (size_t k = 0; k < N; ++k)
            if (active[k] && dface[k] <= 0.0) {
                err->i = (int64_t)(k / (size_t)W) - 1; err->j = (int64_t)(k % (size_t)W) - 1;
                err->value = dface[k];
                free(dface); free(grad); free(dsafe); free(fadv); free(fcross); free(f0);
                free(qbar); free(both); free(active);
                return 1;
            }
    }
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)N; ++k) {
        double ds = np_max(dface[k], thr);
        dsafe[k] = ds;
        fadv[k] = f0[k] * f0[k] / ds;
        fcross[k] = f0[k] * (qbar[k] / ds);
    }
    const double r = dt / dx;
    const double dtg = dt * grav, gr_r = grav * r;
    const double kf = (dtg * nman_s) * nman_s;
#pragma omp parallel for schedule(static)
    for (int64_t fi = 0; fi <= n; ++fi) {
        const int64_t u = fi + 1;
        for (int64_t cj = 0; cj < m; ++cj) {
            const int64_t c = cj + 1;
            const size_t k = (size_t)(u * W + c);
            double m0 = f0[k], q0 = qbar[k];
            double adv = 0.5 * ((fadv[k + W] - fadv[k - W]) - np_sign(m0)
                                * ((fadv[k + W] + fadv[k - W]) - 2.0 * fadv[k]));
            adv = adv + 0.5 * ((fcross[k + 1] - fcross[k - 1]) - np_sign(q0)
                               * ((fcross[k + 1] + fcross[k - 1]) - 2.0 * fcross[k]));
            if (!all_wet) adv = adv * (both[k] ? 1.0 : 0.0);
            double fr;
            double du = dsafe[k];
            if (nman_is_scalar) {
                fr = kf * sqrt(m0 * m0 + q0 * q0) / (du * du * oracle_cbrt(du));
            } else {
                double nf = 0.5 * (AT(nman, u, c + 1) + AT(nman, u + 1, c + 1));
                fr = dtg * nf * nf * sqrt(m0 * m0 + q0 * q0) / (du * du * oracle_cbrt(du));
            }
            double numer = m0 - r * adv - gr_r * dface[k] * grad[k];
            double res;
            if (all_wet || active[k]) res = numer / (1.0 + fr);
            else res = 0.0;
            AT(f_new, u + 1, c + 1) = res;
        }
    }
    free(dface); free(grad); free(dsafe); free(fadv); free(fcross); free(f0);
    free(qbar); free(both); free(active);
    return 0;
}

static int first_nonfinite(const double *a, int64_t rows, int64_t cols, int64_t *i, int64_t *j)
{
    for (int64_t k = 0; k < rows * cols; ++k)
        if (!isfinite(a[k])) { *i = k / cols - G; *j = k % cols - G; return 1; }
    return 0;
}

/* update_momentum, kernels.py:252-271 */
int64_t oracle_momentum(OBlock *b, int64_t cur, double dt, double grav, double thr, OErr *err)
{
    const int64_t ni = b->ni, nj = b->nj;
    const int64_t sc = nj + 4, sm = nj + 4, sn = nj + 5;
    double *en = b->eta[1 - cur];
    int scal = (b->nman == NULL);
    V2 eta = {en, sc, 1}, h = {b->h, sc, 1}, nman = {b->nman, sc, 1};
    W2 wet = {b->wet, sc, 1};
    V2 mo = {b->m[cur], sm, 1}, mn = {b->m[1 - cur], sm, 1}, no = {b->n[cur], sn, 1};
    if (momentum_axis(eta, h, wet, nman, scal, b->nman_s, mo, mn, no, ni, nj,
                      b->dx, dt, grav, thr, err)) { err->code = 4; return 4; }
    V2 etaT = {en, 1, sc}, hT = {b->h, 1, sc}, nmanT = {b->nman, 1, sc};
    W2 wetT = {b->wet, 1, sc};
    V2 noT = {b->n[cur], 1, sn}, nnT = {b->n[1 - cur], 1, sn}, moT = {b->m[cur], 1, sm};
    if (momentum_axis(etaT, hT, wetT, nmanT, scal, b->nman_s, noT, nnT, moT, nj, ni,
                      b->dx, dt, grav, thr, err)) { err->code = 5; return 5; }
    if (first_nonfinite(b->m[1 - cur], ni + 5, nj + 4, &err->i, &err->j)) { err->code = 2; return 2; }
    if (first_nonfinite(b->n[1 - cur], ni + 4, nj + 5, &err->i, &err->j)) { err->code = 3; return 3; }
    return 0;
}

/* apply_edge_flux, kernels.py:274-306.  side: 0 west 1 east 2 south 3 north;
 * kind: 0 reflective 1 radiation */
void oracle_edge(OBlock *b, int64_t cur, int64_t side, int64_t kind, int64_t lo, int64_t hi)
{
    const int64_t ni = b->ni, nj = b->nj;
    if (side <= 1) {
        double *t = b->m[1 - cur];
        const int64_t s = nj + 4;
        int64_t edge = side == 0 ? G : G + ni, inner = side == 0 ? G + 1 : G + ni - 1;
        for (int64_t j = G + lo; j < G + hi; ++j)
            t[edge * s + j] = kind == 0 ? 0.0 : t[inner * s + j];
    } else {
        double *t = b->n[1 - cur];
        const int64_t s = nj + 5;
        int64_t edge = side == 2 ? G : G + nj, inner = side == 2 ? G + 1 : G + nj - 1;
        for (int64_t i = G + lo; i < G + hi; ++i)
            t[i * s + edge] = kind == 0 ? 0.0 : t[i * s + inner];
    }
}

/* accumulate_outputs, kernels.py:322-343 */
void oracle_accumulate(OBlock *b, int64_t cur, double thr)
{
    const int64_t ni = b->ni, nj = b->nj, sc = nj + 4, sm = nj + 4, sn = nj + 5;
    const double *eta = b->eta[1 - cur], *m = b->m[1 - cur], *n = b->n[1 - cur];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ni; ++i)
        for (int64_t j = 0; j < nj; ++j) {
            int64_t c = (G + i) * sc + G + j, a = i * nj + j;
            double e = eta[c], h = b->h[c], d = h + e;
            int w = d >= thr;
            if (w) b->max_eta[a] = np_max(b->max_eta[a], e);
            double mc = 0.5 * (m[(G + i) * sm + G + j] + m[(G + i + 1) * sm + G + j]);
            double nc = 0.5 * (n[(G + i) * sn + G + j] + n[(G + i) * sn + G + j + 1]);
            double ds = np_max(d, thr);
            double u = mc / ds, v = nc / ds;
            double sp = sqrt(u * u + v * v);
            if (w) b->max_speed[a] = np_max(b->max_speed[a], sp);
            if (w && h < 0.0) b->max_inund[a] = np_max(b->max_inund[a], d);
        }
}

/* ------------------------------------------------------------ exchanges */
enum { RS_CHILD, RS_PARENT, RS_SIDE, RS_A, RS_B, RS_RING, RS_PLINE, RS_PA, RS_PB, RS_OFF, RS_NF };
enum { PR_PARENT, PR_CHILD, PR_SIDE, PR_A, PR_B, PR_CLINE, PR_PLINE, PR_PA, PR_PB, PR_OFF, PR_NF };
enum { HE_SEND, HE_RECV, HE_SIDE, HE_SLO, HE_SHI, HE_RLO, HE_RHI, HE_EOFF, HE_FOFF, HE_NF };
enum { ED_BLK, ED_SIDE, ED_KIND, ED_LO, ED_HI, ED_NF };

/* coupling._ring_patch_means + restrict_eta, coupling.py:278-300 */
static void restrict_pack(OBlock *bl, int64_t cur, const int64_t *o, double *buf)
{
    OBlock *c = &bl[o[RS_CHILD]];
    const double *e = c->eta[1 - cur];
    const int64_t s = c->nj + 4, count = o[RS_PB] - o[RS_PA];
    const int ns = o[RS_SIDE] >= 2;   /* south/north */
    for (int64_t p = 0; p < count; ++p) {
        double acc = 0.0;
        for (int dy = 0; dy < 3; ++dy)
            for (int dx = 0; dx < 3; ++dx) {
                int64_t x, y;
                if (ns) { x = o[RS_A] + 3 * p + dx; y = o[RS_RING] + dy; }
                else    { x = o[RS_RING] + dx; y = o[RS_A] + 3 * p + dy; }
                acc += e[(G + x) * s + G + y];
            }
        buf[o[RS_OFF] + p] = acc * (1.0 / 9.0);
    }
}

/* apply_restricted_eta, coupling.py:303-315 */
static void restrict_apply(OBlock *bl, int64_t cur, const int64_t *o, const double *buf, double thr)
{
    OBlock *pb = &bl[o[RS_PARENT]];
    double *e = pb->eta[1 - cur];
    const int64_t s = pb->nj + 4, count = o[RS_PB] - o[RS_PA];
    const int ns = o[RS_SIDE] >= 2;
    for (int64_t p = 0; p < count; ++p) {
        int64_t x = ns ? o[RS_PA] + p : o[RS_PLINE];
        int64_t y = ns ? o[RS_PLINE] : o[RS_PA] + p;
        int64_t k = (G + x) * s + G + y;
        double v = buf[o[RS_OFF] + p];
        e[k] = v;
        pb->wet[k] = pb->h[k] + v >= thr;
    }
}

/* prolong_flux / apply_prolonged_flux, coupling.py:318-340 */
static void prolong_pack(OBlock *bl, int64_t cur, const int64_t *o, double *buf)
{
    OBlock *pb = &bl[o[PR_PARENT]];
    const int64_t count = o[PR_PB] - o[PR_PA];
    for (int64_t p = 0; p < count; ++p) {
        double v;
        if (o[PR_SIDE] >= 2) v = pb->n[1 - cur][(G + o[PR_PA] + p) * (pb->nj + 5) + G + o[PR_PLINE]];
        else                 v = pb->m[1 - cur][(G + o[PR_PLINE]) * (pb->nj + 4) + G + o[PR_PA] + p];
        buf[o[PR_OFF] + p] = v;
    }
}

static void prolong_apply(OBlock *bl, int64_t cur, const int64_t *o, const double *buf)
{
    OBlock *c = &bl[o[PR_CHILD]];
    const int64_t count = o[PR_PB] - o[PR_PA];
    for (int64_t p = 0; p < count; ++p)
        for (int k = 0; k < 3; ++k) {
            double v = buf[o[PR_OFF] + p];
            int64_t a = o[PR_A] + 3 * p + k;
            if (o[PR_SIDE] >= 2) c->n[1 - cur][(G + a) * (c->nj + 5) + G + o[PR_CLINE]] = v;
            else                 c->m[1 - cur][(G + o[PR_CLINE]) * (c->nj + 4) + G + a] = v;
        }
}

/* _strip_slices (exchange.py:162-182): element (layer, along) -> array index
 * of the eta-shaped array; layer 0 is the lower global coordinate. */
static int64_t eta_strip_index(const OBlock *b, int64_t side, int sending, int64_t along, int64_t layer)
{
    const int64_t s = b->nj + 4;
    int64_t x, y;
    switch (side) {
    case 0: x = sending ? layer : -2 + layer; y = along; break;                       /* west */
    case 1: x = sending ? b->ni - 2 + layer : b->ni + layer; y = along; break;         /* east */
    case 2: y = sending ? layer : -2 + layer; x = along; break;                       /* south */
    default: y = sending ? b->nj - 2 + layer : b->nj + layer; x = along; break;        /* north */
    }
    return (G + x) * s + G + y;
}

/* _face_strip (exchange.py:185-215).  normal: along cells, across faces;
 * tangential: along faces (span+1), across cells.  Returns the flat index
 * into m (x sides normal / s-n tangential) or n. */
static int64_t face_strip_index(const OBlock *b, int64_t side, int sending, int normal,
                                int64_t along, int64_t layer)
{
    const int x_side = side <= 1;
    const int low = (side == 0 || side == 2);
    const int64_t n_edge = x_side ? b->ni : b->nj;
    int64_t across;
    if (normal) {
        if (sending) across = low ? 1 + layer : n_edge - 2 + layer;
        else         across = low ? -2 + layer : n_edge + 1 + layer;
    } else {
        if (sending) across = low ? layer : n_edge - 2 + layer;
        else         across = low ? -2 + layer : n_edge + layer;
    }
    /* normal: x side -> m[across (face), along (cell j)];  s/n -> n[along (cell i), across (face)]
     * tangential: x side -> n[across (cell i), along (face j)]; s/n -> m[along (face i), across (cell j)] */
    if (x_side) {
        if (normal) return (G + across) * (b->nj + 4) + G + along;
        return (G + across) * (b->nj + 5) + G + along;
    }
    if (normal) return (G + along) * (b->nj + 5) + G + across;
    return (G + along) * (b->nj + 4) + G + across;
}

static const int64_t OPP[4] = {1, 0, 3, 2};

static void halo_pack(OBlock *bl, int64_t cur, const int64_t *o, int flux, double *buf)
{
    const OBlock *b = &bl[o[HE_SEND]];
    const int64_t side = o[HE_SIDE], lo = o[HE_SLO], span = o[HE_SHI] - o[HE_SLO];
    if (!flux) {
        const double *e = b->eta[1 - cur];
        for (int64_t l = 0; l < 2; ++l)
            for (int64_t k = 0; k < span; ++k)
                buf[o[HE_EOFF] + l * span + k] = e[eta_strip_index(b, side, 1, lo + k, l)];
        return;
    }
    const int x_side = side <= 1;
    const double *na = x_side ? b->m[1 - cur] : b->n[1 - cur];
    const double *ta = x_side ? b->n[1 - cur] : b->m[1 - cur];
    double *dst = buf + o[HE_FOFF];
    for (int64_t l = 0; l < 2; ++l)
        for (int64_t k = 0; k < span; ++k)
            dst[l * span + k] = na[face_strip_index(b, side, 1, 1, lo + k, l)];
    dst += 2 * span;
    for (int64_t l = 0; l < 2; ++l)
        for (int64_t k = 0; k <= span; ++k)
            dst[l * (span + 1) + k] = ta[face_strip_index(b, side, 1, 0, lo + k, l)];
}

static void halo_apply(OBlock *bl, int64_t cur, const int64_t *o, int flux, const double *buf, double thr)
{
    OBlock *b = &bl[o[HE_RECV]];
    const int64_t side = OPP[o[HE_SIDE]], lo = o[HE_RLO], span = o[HE_RHI] - o[HE_RLO];
    if (!flux) {
        double *e = b->eta[1 - cur];
        for (int64_t l = 0; l < 2; ++l)
            for (int64_t k = 0; k < span; ++k) {
                int64_t idx = eta_strip_index(b, side, 0, lo + k, l);
                e[idx] = buf[o[HE_EOFF] + l * span + k];
            }
        for (int64_t l = 0; l < 2; ++l)
            for (int64_t k = 0; k < span; ++k) {
                int64_t idx = eta_strip_index(b, side, 0, lo + k, l);
                b->wet[idx] = b->h[idx] + e[idx] >= thr;
            }
        return;
    }
    const int x_side = side <= 1;
    double *na = x_side ? b->m[1 - cur] : b->n[1 - cur];
    double *ta = x_side ? b->n[1 - cur] : b->m[1 - cur];
    const double *src = buf + o[HE_FOFF];
    for (int64_t l = 0; l < 2; ++l)
        for (int64_t k = 0; k < span; ++k)
            na[face_strip_index(b, side, 0, 1, lo + k, l)] = src[l * span + k];
    src += 2 * span;
    for (int64_t l = 0; l < 2; ++l)
        for (int64_t k = 0; k <= span; ++k)
            ta[face_strip_index(b, side, 0, 0, lo + k, l)] = src[l * (span + 1) + k];
}

/* ------------------------------------------------------------ step loop */
typedef struct {
    int64_t nblocks;
    OBlock *blocks;
    double dt, grav, thr;
    int64_t cur;
    int64_t n_restrict; const int64_t *restrict_ops;   /* pack order == apply order */
    int64_t n_prolong; const int64_t *prolong_ops;
    int64_t n_halo; const int64_t *halo_ops;           /* in reference apply order */
    int64_t n_edges; const int64_t *edge_ops;
    double *buf;                                       /* >= max phase payload */
    int64_t accumulate;                                /* 1: fold outputs each step */
} OSim;

/* Exchange phases are "pack all, then apply all" (runner.py:268-291;
 * exchange.py:308-351): a block that is both parent and child, or a strip
 * read and written in one phase, sees pre-phase values. */
static void phase_restrict(OSim *s)
{
    for (int64_t k = 0; k < s->n_restrict; ++k) restrict_pack(s->blocks, s->cur, s->restrict_ops + k * RS_NF, s->buf);
    for (int64_t k = 0; k < s->n_restrict; ++k) restrict_apply(s->blocks, s->cur, s->restrict_ops + k * RS_NF, s->buf, s->thr);
}

static void phase_halo(OSim *s, int flux)
{
    for (int64_t k = 0; k < s->n_halo; ++k) halo_pack(s->blocks, s->cur, s->halo_ops + k * HE_NF, flux, s->buf);
    for (int64_t k = 0; k < s->n_halo; ++k) halo_apply(s->blocks, s->cur, s->halo_ops + k * HE_NF, flux, s->buf, s->thr);
}

static void phase_prolong(OSim *s)
{
    for (int64_t k = 0; k < s->n_prolong; ++k) prolong_pack(s->blocks, s->cur, s->prolong_ops + k * PR_NF, s->buf);
    for (int64_t k = 0; k < s->n_prolong; ++k) prolong_apply(s->blocks, s->cur, s->prolong_ops + k * PR_NF, s->buf);
}

/* One phase at a time (for phase-level parity tests); phase codes follow
 * runner.PHASE_SEQUENCE (runner.py:39-40). */
int64_t oracle_phase(OSim *s, int64_t phase, OErr *err)
{
    memset(err, 0, sizeof(*err));
    switch (phase) {
    case 0:
        for (int64_t b = 0; b < s->nblocks; ++b)
            if (oracle_mass(&s->blocks[b], s->cur, s->dt, s->thr, err)) { err->block = b; return err->code; }
        return 0;
    case 1: phase_restrict(s); return 0;
    case 2: phase_halo(s, 0); return 0;
    case 3:
        for (int64_t b = 0; b < s->nblocks; ++b)
            if (oracle_momentum(&s->blocks[b], s->cur, s->dt, s->grav, s->thr, err)) { err->block = b; return err->code; }
        for (int64_t k = 0; k < s->n_edges; ++k) {
            const int64_t *o = s->edge_ops + k * ED_NF;
            oracle_edge(&s->blocks[o[ED_BLK]], s->cur, o[ED_SIDE], o[ED_KIND], o[ED_LO], o[ED_HI]);
        }
        return 0;
    case 4: phase_prolong(s); return 0;
    case 5: phase_halo(s, 1); return 0;
    case 6:
        for (int64_t b = 0; b < s->nblocks; ++b) oracle_accumulate(&s->blocks[b], s->cur, s->thr);
        return 0;
    case 7: s->cur ^= 1; return 0;
    }
    return -1;
}

/* Simulation._run_serial (runner.py:220-266); stops at the first error
 * (mass errors of a step precede its momentum errors; blocks in global
 * order), like the reference's first raising call. */
int64_t oracle_run(OSim *s, int64_t nsteps, OErr *err)
{
    for (int64_t step = 0; step < nsteps; ++step) {
        for (int64_t ph = 0; ph < 8; ++ph) {
            if (ph == 6 && !s->accumulate) continue;
            int64_t rc = oracle_phase(s, ph, err);
            if (rc) return rc;
        }
    }
    return 0;
}
