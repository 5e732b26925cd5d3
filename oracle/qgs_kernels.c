/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C float64 restatement of the reference QGS tile-raster kernels
 * (/root/reference/pkg/src/qgsplat/raster_kernels.py, intersect.py,
 * geodesic.py, surface.py).  It exists to check the sm_100a product path
 * and to serve as the host-core CPU baseline in bench.py; nothing in the
 * product package links or calls it.
 *
 * Arithmetic is written so that every floating-point operation happens in
 * the same order as the numba source (no FMA contraction: build with
 * -ffp-contract=off), which makes the results bit-identical to the
 * reference on the same inputs; tests/golden pins that.
 *
 * Layout: per-primitive arrays are row-major float64 (ohat P*3, M P*9,
 * wv P*3, sv P*3, lam P*2, alpha P, colors P*3, Nmat P*9), planar is u8,
 * pix_bbox is int64 P*4 (umin, umax, vmin, vmax, inclusive).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* intersect.py:20-28 */
#define QO_A_EPS 1e-6
#define QO_B_EPS 1e-12
#define QO_RHO_EPS 1e-12
#define QO_BR_QUAD 0
#define QO_BR_LINEAR 1
#define QO_BR_PLANAR 2
/* geodesic.py:16 */
#define QO_U_SERIES 1e-3
/* raster_kernels.py:26-37 */
#define QO_RING 8
#define QO_NG 33
enum { GS_OHAT = 0, GS_M = 3, GS_W = 12, GS_S = 15, GS_ALPHA = 18,
       GS_COLOR = 19, GS_NMAT = 22, GS_LAM = 31 };

typedef struct {
    int64_t P;
    const double *ohat, *M, *wv, *sv, *lam, *alpha, *colors, *Nmat;
    const uint8_t *planar;
    const int64_t *bbox;
} qo_prims;

typedef struct {
    int32_t resort, euclid;
    double t_clip, alpha_floor, alpha_clamp, t_term;
} qo_settings;

/* one ray/surface hit (intersect.py:58-115 return tuple) */
typedef struct {
    int valid, branch;
    double t, x, y, rho, cth, sth, a, l, sig, G;
} qo_hit;

/* one shaded fragment (raster_kernels.py:40-80 return tuple) */
typedef struct {
    qo_hit h;
    double abar, nc[3], K;
} qo_frag;

/* ---------------------------------------------------------------- scalars */

/* geodesic.py:23-31 */
double qo_arc_length(double a, double rho)
{
    double u = 2.0 * a * rho;
    if (fabs(u) < QO_U_SERIES) {
        double u2 = u * u;
        return rho * (1.0 + u2 / 6.0 - u2 * u2 / 40.0);
    }
    double r = sqrt(u * u + 1.0);
    return (log(r + u) + u * r) / (4.0 * a);
}

/* geodesic.py:34-48; out = (l, dl/da, dl/drho) */
void qo_arc_length_grad(double a, double rho, double *out)
{
    double u = 2.0 * a * rho;
    if (fabs(u) < QO_U_SERIES) {
        double u2 = u * u;
        out[0] = rho * (1.0 + u2 / 6.0 - u2 * u2 / 40.0);
        out[1] = rho * rho * (2.0 * u / 3.0 - u * u * u / 5.0);
        out[2] = 1.0 + u2 / 2.0 - u2 * u2 / 8.0;
        return;
    }
    double r = sqrt(u * u + 1.0);
    double l = (log(r + u) + u * r) / (4.0 * a);
    out[0] = l;
    out[1] = (rho * r - l) / a;
    out[2] = r;
}

/* geodesic.py:51-59 */
double qo_sigma_dir(double s1, double s2, double c, double s)
{
    double m = (s2 * c) * (s2 * c) + (s1 * s) * (s1 * s);
    return fabs(s1 * s2) / sqrt(m);
}

/* geodesic.py:62-71; out = (sigma, d/ds1, d/ds2, d/dc, d/ds) */
void qo_sigma_dir_grad(double s1, double s2, double c, double s, double *out)
{
    double m = (s2 * c) * (s2 * c) + (s1 * s) * (s1 * s);
    double sig = fabs(s1 * s2) / sqrt(m);
    out[0] = sig;
    out[1] = sig * (1.0 / s1 - s1 * s * s / m);
    out[2] = sig * (1.0 / s2 - s2 * c * c / m);
    out[3] = -sig * s2 * s2 * c / m;
    out[4] = -sig * s1 * s1 * s / m;
}

static inline void miss(qo_hit *h, int branch)
{
    h->valid = 0; h->branch = branch;
    h->t = h->x = h->y = h->rho = 0.0; h->cth = 1.0; h->sth = 0.0;
    h->a = h->l = 0.0; h->sig = 1.0; h->G = 0.0;
}

static inline void polar(double x, double y, double *rho, double *c, double *s)
{
    *rho = sqrt(x * x + y * y);
    if (*rho > QO_RHO_EPS) { *c = x / *rho; *s = y / *rho; }
    else { *c = 1.0; *s = 0.0; }
}

/* intersect.py:58-115: near-then-far 3-sigma selection on one local ray */
void qo_fragment_geometry(double w1, double w2, double iw3, double s1, double s2,
                          double s3, double ox, double oy, double oz, double dx,
                          double dy, double dz, int planar, int euclid,
                          double t_clip, qo_hit *h)
{
    if (planar) {
        if (fabs(dz) < QO_B_EPS) { miss(h, QO_BR_PLANAR); return; }
        double t = -oz / dz;
        if (t <= t_clip) { miss(h, QO_BR_PLANAR); return; }
        double x = ox + t * dx, y = oy + t * dy, rho, c, s;
        polar(x, y, &rho, &c, &s);
        double sig = qo_sigma_dir(s1, s2, c, s);
        double l = rho;
        if (l > 3.0 * sig) { miss(h, QO_BR_PLANAR); return; }
        h->valid = 1; h->branch = QO_BR_PLANAR;
        h->t = t; h->x = x; h->y = y; h->rho = rho; h->cth = c; h->sth = s;
        h->a = 0.0; h->l = l; h->sig = sig;
        h->G = exp(-(l * l) / (2.0 * sig * sig));
        return;
    }
    /* ray_coeffs, intersect.py:31-36 */
    double A = w1 * dx * dx + w2 * dy * dy;
    double B = 2.0 * (w1 * ox * dx + w2 * oy * dy) - iw3 * dz;
    double C = w1 * ox * ox + w2 * oy * oy - iw3 * oz;
    /* candidate_depths, intersect.py:39-55 */
    int cnt, branch;
    double roots[2] = {0.0, 0.0};
    if (fabs(A) < QO_A_EPS) {
        branch = QO_BR_LINEAR;
        if (fabs(B) < QO_B_EPS) cnt = 0;
        else { cnt = 1; roots[0] = -C / B; }
    } else {
        branch = QO_BR_QUAD;
        double disc = B * B - 4.0 * A * C;
        if (disc < 0.0) cnt = 0;
        else {
            double sa = A > 0.0 ? 1.0 : -1.0;
            double sq = sqrt(disc);
            roots[0] = (-B - sa * sq) / (2.0 * A);
            roots[1] = (-B + sa * sq) / (2.0 * A);
            cnt = disc == 0.0 ? 1 : 2;
        }
    }
    double s1s2 = s1 * s2;
    for (int k = 0; k < cnt; ++k) {
        double t = roots[k];
        if (t <= t_clip) continue;
        double x = ox + t * dx, y = oy + t * dy;
        /* euclidean 3-sigma ellipse pre-reject, intersect.py:100-102 */
        double m = (s2 * x) * (s2 * x) + (s1 * y) * (s1 * y);
        if (m > 9.0 * s1s2 * s1s2) continue;
        double rho, c, s;
        polar(x, y, &rho, &c, &s);
        double a = s3 * (w1 * c * c + w2 * s * s);
        double l = euclid ? rho : qo_arc_length(a, rho);
        double sig = qo_sigma_dir(s1, s2, c, s);
        if (l <= 3.0 * sig) {
            h->valid = 1; h->branch = branch;
            h->t = t; h->x = x; h->y = y; h->rho = rho; h->cth = c; h->sth = s;
            h->a = a; h->l = l; h->sig = sig;
            h->G = exp(-(l * l) / (2.0 * sig * sig));
            return;
        }
    }
    miss(h, branch);
}

/* ------------------------------------------------------------ shading */

static inline void local_dir(const double *M, double dx, double dy, double dz,
                             double *d)
{
    d[0] = M[0] * dx + M[1] * dy + M[2] * dz;
    d[1] = M[3] * dx + M[4] * dy + M[5] * dz;
    d[2] = M[6] * dx + M[7] * dy + M[8] * dz;
}

/* raster_kernels.py:40-80 */
static void shade(const qo_prims *pr, int64_t p, double dx, double dy, double dz,
                  const qo_settings *st, qo_frag *f)
{
    double dh[3];
    local_dir(pr->M + 9 * p, dx, dy, dz, dh);
    const double *wv = pr->wv + 3 * p, *sv = pr->sv + 3 * p, *oh = pr->ohat + 3 * p;
    qo_fragment_geometry(wv[0], wv[1], wv[2], sv[0], sv[1], sv[2], oh[0], oh[1],
                         oh[2], dh[0], dh[1], dh[2], pr->planar[p] == 1,
                         st->euclid, st->t_clip, &f->h);
    if (!f->h.valid) return;
    double abar = pr->alpha[p] * f->h.G;
    if (abar < st->alpha_floor) { f->h.valid = 0; return; }
    if (abar > st->alpha_clamp) abar = st->alpha_clamp;
    f->abar = abar;
    double nl[3];
    if (f->h.branch == QO_BR_PLANAR) {
        nl[0] = 0.0; nl[1] = 0.0; nl[2] = -1.0;
        f->K = 0.0;
    } else {
        double nx = 2.0 * wv[0] * f->h.x, ny = 2.0 * wv[1] * f->h.y, nz = -wv[2];
        double nrm = sqrt(nx * nx + ny * ny + nz * nz);
        nl[0] = nx / nrm; nl[1] = ny / nrm; nl[2] = nz / nrm;
        /* surface.py:27-32 */
        double l1 = pr->lam[2 * p], l2 = pr->lam[2 * p + 1], x = f->h.x, y = f->h.y;
        double den = 1.0 + 4.0 * l1 * l1 * x * x + 4.0 * l2 * l2 * y * y;
        f->K = 4.0 * l1 * l2 / (den * den);
    }
    const double *N = pr->Nmat + 9 * p;
    double c0 = N[0] * nl[0] + N[1] * nl[1] + N[2] * nl[2];
    double c1 = N[3] * nl[0] + N[4] * nl[1] + N[5] * nl[2];
    double c2 = N[6] * nl[0] + N[7] * nl[1] + N[8] * nl[2];
    if (c0 * dx + c1 * dy + c2 * dz > 0.0) { c0 = -c0; c1 = -c1; c2 = -c2; }
    f->nc[0] = c0; f->nc[1] = c1; f->nc[2] = c2;
}

/* ------------------------------------------------- per-pixel fragment stream
 *
 * Both passes walk the same emission sequence: fragments of the tile list in
 * order, staged through the 8-entry min-depth ring (raster_kernels.py:159-270,
 * 589-670).  The visitor gets each emitted fragment with its tile-list
 * position and returns 0 once the pixel has terminated.
 */
typedef struct { double t; int64_t pos; qo_frag f; } qo_entry;
typedef int (*qo_visit)(void *ctx, int64_t pos, int64_t prim, const qo_frag *f);

static int64_t pixel_stream(const qo_prims *pr, const int64_t *list, int64_t lo,
                            int64_t hi, int64_t u, int64_t v, const double *d,
                            const qo_settings *st, qo_visit visit, void *ctx,
                            qo_entry *ring)
{
    int64_t viol = 0, n = 0;
    double last_t = -1.0e300;
    int alive = 1;
#define QO_EMIT(POS, FR)                                                   \
    do {                                                                   \
        double et_ = (FR)->h.t;                                            \
        if (et_ < last_t - 1e-12) viol += 1;                               \
        if (et_ > last_t) last_t = et_;                                    \
        alive = visit(ctx, (POS), list[(POS)], (FR));                      \
    } while (0)
    for (int64_t i = lo; i < hi && alive; ++i) {
        int64_t p = list[i];
        const int64_t *bb = pr->bbox + 4 * p;
        if (u < bb[0] || u > bb[1] || v < bb[2] || v > bb[3]) continue;
        qo_frag f;
        shade(pr, p, d[0], d[1], d[2], st, &f);
        if (!f.h.valid) continue;
        if (!st->resort) { QO_EMIT(i, &f); continue; }
        if (n == QO_RING) {
            int jm = 0;
            for (int j = 1; j < n; ++j)
                if (ring[j].t < ring[jm].t) jm = j;
            if (f.h.t < ring[jm].t) {
                QO_EMIT(i, &f);
            } else {
                qo_entry out = ring[jm];
                ring[jm].t = f.h.t; ring[jm].pos = i; ring[jm].f = f;
                QO_EMIT(out.pos, &out.f);
            }
        } else {
            ring[n].t = f.h.t; ring[n].pos = i; ring[n].f = f;
            ++n;
        }
    }
    while (alive && n > 0) {
        int jm = 0;
        for (int j = 1; j < n; ++j)
            if (ring[j].t < ring[jm].t) jm = j;
        qo_entry out = ring[jm];
        --n;
        ring[jm] = ring[n];
        QO_EMIT(out.pos, &out.f);
    }
#undef QO_EMIT
    return viol;
}

/* ------------------------------------------------------------- forward */

typedef struct {
    const double *colors;
    double T, c[3], a, d, d2, n[3], k, dist, s0, s1, s2, median, t_term;
    int64_t nfrag;
} qo_fwd_px;

/* compositing of one emitted fragment, raster_kernels.py:194-215 */
static int fwd_visit(void *vctx, int64_t pos, int64_t p, const qo_frag *f)
{
    (void)pos;
    qo_fwd_px *c = (qo_fwd_px *)vctx;
    double t = f->h.t, w = f->abar * c->T;
    const double *col = c->colors + 3 * p;
    c->c[0] += w * col[0];
    c->c[1] += w * col[1];
    c->c[2] += w * col[2];
    c->a += w;
    c->d += w * t;
    c->d2 += w * t * t;
    c->n[0] += w * f->nc[0];
    c->n[1] += w * f->nc[1];
    c->n[2] += w * f->nc[2];
    c->k += w * f->K;
    c->dist += w * (t * t * c->s0 - 2.0 * t * c->s1 + c->s2);
    c->s0 += w;
    c->s1 += w * t;
    c->s2 += w * t * t;
    if (c->T > 0.5) c->median = t;
    c->T *= 1.0 - f->abar;
    c->nfrag += 1;
    return !(c->T < c->t_term);
}

/* forward_kernel, raster_kernels.py:83-286.  Output maps are (H, W[, 3]). */
void qo_forward(int64_t H, int64_t W, const double *dirs, const int64_t *tile_offsets,
                const int64_t *tile_prims, int64_t tiles_x, int64_t tiles_y,
                const qo_prims *pr, const qo_settings *st, double *o_color,
                double *o_alpha, double *o_depth, double *o_depthsq, double *o_median,
                double *o_normal, double *o_curv, double *o_dist, double *o_T,
                int64_t *o_nfrag, int64_t *o_viol, const int64_t *tile_list, int64_t n_list)
{
    /* tile_list (optional): process only these tiles (CPU-baseline sampling) */
    int64_t n_iter = tile_list ? n_list : tiles_x * tiles_y;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t it = 0; it < n_iter; ++it) {
        int64_t tile = tile_list ? tile_list[it] : it;
        int64_t ty = tile / tiles_x, tx = tile % tiles_x;
        int64_t v1 = ty * 16 + 16 < H ? ty * 16 + 16 : H;
        int64_t u1 = tx * 16 + 16 < W ? tx * 16 + 16 : W;
        int64_t viol = 0;
        qo_entry ring[QO_RING];
        for (int64_t v = ty * 16; v < v1; ++v)
            for (int64_t u = tx * 16; u < u1; ++u) {
                int64_t px = v * W + u;
                qo_fwd_px c;
                memset(&c, 0, sizeof c);
                c.colors = pr->colors;
                c.T = 1.0;
                c.t_term = st->t_term;
                viol += pixel_stream(pr, tile_prims, tile_offsets[tile],
                                     tile_offsets[tile + 1], u, v, dirs + 3 * px, st,
                                     fwd_visit, &c, ring);
                for (int j = 0; j < 3; ++j) {
                    o_color[3 * px + j] = c.c[j];
                    o_normal[3 * px + j] = c.n[j];
                }
                o_alpha[px] = c.a; o_depth[px] = c.d; o_depthsq[px] = c.d2;
                o_median[px] = c.median; o_curv[px] = c.k; o_dist[px] = c.dist;
                o_T[px] = c.T; o_nfrag[px] = c.nfrag;
            }
        o_viol[tile] = viol;
    }
}

/* ------------------------------------------------------------ backward */

typedef struct {
    const qo_prims *pr;
    const qo_settings *st;
    double *rows;          /* this tile's pair-gradient rows, NG per position */
    double *rows_abs;      /* optional: sums of |each fragment's contribution| (diagnostics) */
    int64_t px;            /* pixel index (diagnostics) */
    int64_t row0;          /* tile_offsets[tile] */
    double d[3];
    double T, pref, vtot, F0, F1, F2;
    double uc[3], ua, ut, un[3], uk, ud;
} qo_bwd_px;

/* diagnostics: per-fragment contributions of one primitive
 * (qo_set_diag_prim): rows of [pixel, t, 33 slot deltas] */
static int64_t diag_prim = -1, diag_n = 0, diag_max = 0;
static double *diag_buf = NULL;

void qo_set_diag_prim(int64_t prim, double *buf, int64_t max_rows)
{
    diag_prim = prim; diag_buf = buf; diag_max = max_rows; diag_n = 0;
}

int64_t qo_diag_rows(void) { return diag_n; }

/* _grad_fragment, raster_kernels.py:289-502 */
static int bwd_visit(void *vctx, int64_t pos, int64_t p, const qo_frag *f)
{
    qo_bwd_px *c = (qo_bwd_px *)vctx;
    const qo_prims *pr = c->pr;
    double *g = c->rows + (pos - c->row0) * QO_NG;
    double before[QO_NG];
    if (c->rows_abs || p == diag_prim)
        for (int j = 0; j < QO_NG; ++j) before[j] = g[j];
    const double *wv = pr->wv + 3 * p, *sv = pr->sv + 3 * p, *oh = pr->ohat + 3 * p;
    const double *N = pr->Nmat + 9 * p, *Mp = pr->M + 9 * p, *col = pr->colors + 3 * p;
    double w1 = wv[0], w2 = wv[1], iw3 = wv[2];
    double t = f->h.t, x = f->h.x, y = f->h.y, rho = f->h.rho, cth = f->h.cth;
    double sth = f->h.sth, a = f->h.a, l = f->h.l, sig = f->h.sig, G = f->h.G;
    double abar = f->abar;
    int branch = f->h.branch;
    double dx = c->d[0], dy = c->d[1], dz = c->d[2];

    double nlx, nly, nlz, K, nrm;
    if (branch == QO_BR_PLANAR) {
        nlx = 0.0; nly = 0.0; nlz = -1.0; K = 0.0; nrm = 1.0;
    } else {
        double nxu = 2.0 * w1 * x, nyu = 2.0 * w2 * y, nzu = -iw3;
        nrm = sqrt(nxu * nxu + nyu * nyu + nzu * nzu);
        nlx = nxu / nrm; nly = nyu / nrm; nlz = nzu / nrm;
        double l1 = pr->lam[2 * p], l2 = pr->lam[2 * p + 1];
        double den = 1.0 + 4.0 * l1 * l1 * x * x + 4.0 * l2 * l2 * y * y;
        K = 4.0 * l1 * l2 / (den * den);
    }
    double ncx = N[0] * nlx + N[1] * nly + N[2] * nlz;
    double ncy = N[3] * nlx + N[4] * nly + N[5] * nlz;
    double ncz = N[6] * nlx + N[7] * nly + N[8] * nlz;
    double flip = 1.0;
    if (ncx * dx + ncy * dy + ncz * dz > 0.0) {
        flip = -1.0; ncx = -ncx; ncy = -ncy; ncz = -ncz;
    }
    double T = c->T, w_i = abar * T;
    double V = c->uc[0] * col[0] + c->uc[1] * col[1] + c->uc[2] * col[2] + c->ua
               + c->ut * t + c->un[0] * ncx + c->un[1] * ncy + c->un[2] * ncz
               + c->uk * K + c->ud * (t * t * c->F0 - 2.0 * t * c->F1 + c->F2);
    c->pref += w_i * V;
    double g_abar = T * V - (c->vtot - c->pref) / (1.0 - abar);

    g[GS_COLOR + 0] += w_i * c->uc[0];
    g[GS_COLOR + 1] += w_i * c->uc[1];
    g[GS_COLOR + 2] += w_i * c->uc[2];
    double g_t = c->ut * w_i + c->ud * 2.0 * w_i * (t * c->F0 - c->F1);
    double gcx = w_i * c->un[0], gcy = w_i * c->un[1], gcz = w_i * c->un[2];
    double g_K = w_i * c->uk;

    double g_G;
    if (abar < c->st->alpha_clamp) {
        g[GS_ALPHA] += g_abar * G;
        g_G = g_abar * pr->alpha[p];
    } else {
        g_G = 0.0;
    }
    double g_l = g_G * G * (-l / (sig * sig));
    double g_sig = g_G * G * (l * l / (sig * sig * sig));
    double sg[5];
    qo_sigma_dir_grad(sv[0], sv[1], cth, sth, sg);
    g[GS_S + 0] += g_sig * sg[1];
    g[GS_S + 1] += g_sig * sg[2];
    double g_cth = g_sig * sg[3], g_sth = g_sig * sg[4];
    double g_x = 0.0, g_y = 0.0, g_rho = 0.0, g_a = 0.0;
    if (c->st->euclid || branch == QO_BR_PLANAR) {
        g_rho += g_l;
    } else {
        double lg[3];
        qo_arc_length_grad(a, rho, lg);
        g_a += g_l * lg[1];
        g_rho += g_l * lg[2];
    }
    double g_w1, g_w2, g_iw3;
    if (branch != QO_BR_PLANAR) {
        double s3 = sv[2];
        g[GS_S + 2] += g_a * (w1 * cth * cth + w2 * sth * sth);
        g_w1 = g_a * s3 * cth * cth;
        g_w2 = g_a * s3 * sth * sth;
        g_iw3 = 0.0;
        g_cth += g_a * 2.0 * s3 * w1 * cth;
        g_sth += g_a * 2.0 * s3 * w2 * sth;
        double l1 = pr->lam[2 * p], l2 = pr->lam[2 * p + 1];
        double den = 1.0 + 4.0 * l1 * l1 * x * x + 4.0 * l2 * l2 * y * y;
        double den3 = den * den * den;
        g[GS_LAM + 0] += g_K * (4.0 * l2 / (den * den) - 64.0 * l1 * l1 * l2 * x * x / den3);
        g[GS_LAM + 1] += g_K * (4.0 * l1 / (den * den) - 64.0 * l1 * l2 * l2 * y * y / den3);
        g_x += g_K * (-16.0 * K * l1 * l1 * x / den);
        g_y += g_K * (-16.0 * K * l2 * l2 * y / den);
        double g_nlx = flip * (N[0] * gcx + N[3] * gcy + N[6] * gcz);
        double g_nly = flip * (N[1] * gcx + N[4] * gcy + N[7] * gcz);
        double g_nlz = flip * (N[2] * gcx + N[5] * gcy + N[8] * gcz);
        g[GS_NMAT + 0] += flip * gcx * nlx;
        g[GS_NMAT + 1] += flip * gcx * nly;
        g[GS_NMAT + 2] += flip * gcx * nlz;
        g[GS_NMAT + 3] += flip * gcy * nlx;
        g[GS_NMAT + 4] += flip * gcy * nly;
        g[GS_NMAT + 5] += flip * gcy * nlz;
        g[GS_NMAT + 6] += flip * gcz * nlx;
        g[GS_NMAT + 7] += flip * gcz * nly;
        g[GS_NMAT + 8] += flip * gcz * nlz;
        double dot = nlx * g_nlx + nly * g_nly + nlz * g_nlz;
        double g_ntx = (g_nlx - nlx * dot) / nrm;
        double g_nty = (g_nly - nly * dot) / nrm;
        double g_ntz = (g_nlz - nlz * dot) / nrm;
        g_w1 += 2.0 * x * g_ntx;
        g_x += 2.0 * w1 * g_ntx;
        g_w2 += 2.0 * y * g_nty;
        g_y += 2.0 * w2 * g_nty;
        g_iw3 += -g_ntz;
    } else {
        g[GS_NMAT + 2] += -flip * gcx;
        g[GS_NMAT + 5] += -flip * gcy;
        g[GS_NMAT + 8] += -flip * gcz;
        g_w1 = 0.0; g_w2 = 0.0; g_iw3 = 0.0;
    }
    if (rho > 1e-12) {
        g_x += g_cth * sth * sth / rho - g_sth * cth * sth / rho;
        g_y += -g_cth * cth * sth / rho + g_sth * cth * cth / rho;
    }
    g_x += g_rho * cth;
    g_y += g_rho * sth;

    double dh[3];
    local_dir(Mp, dx, dy, dz, dh);
    double g_tt = g_t + g_x * dh[0] + g_y * dh[1];
    double g_o0 = g_x, g_o1 = g_y, g_o2 = 0.0;
    double g_d0 = g_x * t, g_d1 = g_y * t, g_d2 = 0.0;
    double ox = oh[0], oy = oh[1], oz = oh[2];
    if (branch == QO_BR_PLANAR) {
        g_o2 += -g_tt / dh[2];
        g_d2 += g_tt * oz / (dh[2] * dh[2]);
    } else {
        double A = w1 * dh[0] * dh[0] + w2 * dh[1] * dh[1];
        double B = 2.0 * (w1 * ox * dh[0] + w2 * oy * dh[1]) - iw3 * dh[2];
        double gA, gB, gC;
        if (branch == QO_BR_LINEAR) {
            gA = 0.0;
            gB = -g_tt * t / B;
            gC = -g_tt / B;
        } else {
            double q = 2.0 * A * t + B;
            gA = -g_tt * t * t / q;
            gB = -g_tt * t / q;
            gC = -g_tt / q;
        }
        g_w1 += gA * dh[0] * dh[0] + gB * 2.0 * ox * dh[0] + gC * ox * ox;
        g_w2 += gA * dh[1] * dh[1] + gB * 2.0 * oy * dh[1] + gC * oy * oy;
        g_iw3 += -gB * dh[2] - gC * oz;
        g_o0 += gB * 2.0 * w1 * dh[0] + gC * 2.0 * w1 * ox;
        g_o1 += gB * 2.0 * w2 * dh[1] + gC * 2.0 * w2 * oy;
        g_o2 += -gC * iw3;
        g_d0 += gA * 2.0 * w1 * dh[0] + gB * 2.0 * w1 * ox;
        g_d1 += gA * 2.0 * w2 * dh[1] + gB * 2.0 * w2 * oy;
        g_d2 += -gB * iw3;
    }
    g[GS_W + 0] += g_w1;
    g[GS_W + 1] += g_w2;
    g[GS_W + 2] += g_iw3;
    g[GS_OHAT + 0] += g_o0;
    g[GS_OHAT + 1] += g_o1;
    g[GS_OHAT + 2] += g_o2;
    g[GS_M + 0] += g_d0 * dx;
    g[GS_M + 1] += g_d0 * dy;
    g[GS_M + 2] += g_d0 * dz;
    g[GS_M + 3] += g_d1 * dx;
    g[GS_M + 4] += g_d1 * dy;
    g[GS_M + 5] += g_d1 * dz;
    g[GS_M + 6] += g_d2 * dx;
    g[GS_M + 7] += g_d2 * dy;
    g[GS_M + 8] += g_d2 * dz;
    if (c->rows_abs) {
        double *ga = c->rows_abs + (pos - c->row0) * QO_NG;
        for (int j = 0; j < QO_NG; ++j) ga[j] += fabs(g[j] - before[j]);
    }
    if (p == diag_prim && diag_buf) {
#pragma omp critical(qo_diag)
        {
            if (diag_n < diag_max) {
                double *r = diag_buf + diag_n * (QO_NG + 2);
                r[0] = (double)c->px; r[1] = t;
                for (int j = 0; j < QO_NG; ++j) r[2 + j] = g[j] - before[j];
            }
            diag_n++;
        }
    }

    c->T = T * (1.0 - abar);
    return !(c->T < c->st->t_term);
}

static void bwd_tile(int64_t tile, int64_t H, int64_t W, const double *dirs,
                     const int64_t *tile_offsets, const int64_t *tile_prims,
                     int64_t tiles_x, const qo_prims *pr, const qo_settings *st,
                     const double *f_color, const double *f_alpha, const double *f_depth,
                     const double *f_depthsq, const double *f_normal, const double *f_curv,
                     const double *f_dist, const double *u_color, const double *u_alpha,
                     const double *u_depth, const double *u_normal, const double *u_curv,
                     const double *u_dist, double *rows, double *rows_abs)
{
    int64_t ty = tile / tiles_x, tx = tile % tiles_x;
    int64_t v1 = ty * 16 + 16 < H ? ty * 16 + 16 : H;
    int64_t u1 = tx * 16 + 16 < W ? tx * 16 + 16 : W;
    qo_entry ring[QO_RING];
    for (int64_t v = ty * 16; v < v1; ++v)
        for (int64_t u = tx * 16; u < u1; ++u) {
            int64_t px = v * W + u;
            qo_bwd_px c;
            c.uc[0] = u_color[3 * px]; c.uc[1] = u_color[3 * px + 1];
            c.uc[2] = u_color[3 * px + 2];
            c.ua = u_alpha[px]; c.ut = u_depth[px];
            c.un[0] = u_normal[3 * px]; c.un[1] = u_normal[3 * px + 1];
            c.un[2] = u_normal[3 * px + 2];
            c.uk = u_curv[px]; c.ud = u_dist[px];
            /* raster_kernels.py:537-540: pixels without upstream are skipped */
            if (c.uc[0] == 0.0 && c.uc[1] == 0.0 && c.uc[2] == 0.0 && c.ua == 0.0 &&
                c.ut == 0.0 && c.un[0] == 0.0 && c.un[1] == 0.0 && c.un[2] == 0.0 &&
                c.uk == 0.0 && c.ud == 0.0)
                continue;
            c.pr = pr; c.st = st; c.rows = rows; c.rows_abs = rows_abs; c.px = px;
            c.row0 = tile_offsets[tile];
            c.d[0] = dirs[3 * px]; c.d[1] = dirs[3 * px + 1]; c.d[2] = dirs[3 * px + 2];
            c.F0 = f_alpha[px]; c.F1 = f_depth[px]; c.F2 = f_depthsq[px];
            c.vtot = c.uc[0] * f_color[3 * px] + c.uc[1] * f_color[3 * px + 1]
                     + c.uc[2] * f_color[3 * px + 2] + c.ua * c.F0 + c.ut * c.F1
                     + c.un[0] * f_normal[3 * px] + c.un[1] * f_normal[3 * px + 1]
                     + c.un[2] * f_normal[3 * px + 2] + c.uk * f_curv[px]
                     + c.ud * 2.0 * f_dist[px];
            c.T = 1.0;
            c.pref = 0.0;
            pixel_stream(pr, tile_prims, tile_offsets[tile], tile_offsets[tile + 1], u, v,
                         c.d, st, bwd_visit, &c, ring);
        }
}

/*
 * backward_kernel + merge_pair_grads (raster_kernels.py:505-681).  kg (P*33)
 * must be zeroed by the caller.  Tiles run in parallel in bounded chunks, each
 * with private pair rows; rows are then merged into kg in (tile, position)
 * order, which is exactly the reference's serial merge order.
 */
int qo_backward(int64_t H, int64_t W, const double *dirs, const int64_t *tile_offsets,
                const int64_t *tile_prims, int64_t tiles_x, int64_t tiles_y,
                const qo_prims *pr, const qo_settings *st, const double *f_color,
                const double *f_alpha, const double *f_depth, const double *f_depthsq,
                const double *f_normal, const double *f_curv, const double *f_dist,
                const double *u_color, const double *u_alpha, const double *u_depth,
                const double *u_normal, const double *u_curv, const double *u_dist,
                double *kg, const int64_t *tile_list, int64_t n_list, double *kg_abs)
{
    /* tile_list (optional, ascending): process only these tiles; all other
       tiles must have empty ranges (CPU-baseline sampling) */
    int64_t n_iter = tile_list ? n_list : tiles_x * tiles_y;
    int nthr = 1;
#ifdef _OPENMP
    nthr = omp_get_max_threads();
#endif
    int64_t chunk = 4 * (int64_t)nthr;
    for (int64_t k0 = 0; k0 < n_iter; k0 += chunk) {
        int64_t k1 = k0 + chunk < n_iter ? k0 + chunk : n_iter;
        int64_t t0 = tile_list ? tile_list[k0] : k0;
        int64_t t1 = tile_list ? tile_list[k1 - 1] + 1 : k1;
        int64_t base = tile_offsets[t0];
        int64_t n_rows = tile_offsets[t1] - base;
        double *rows = (double *)calloc((size_t)(n_rows > 0 ? n_rows : 1) * QO_NG,
                                        sizeof(double));
        if (!rows) return -1;
        double *rows_abs = NULL;
        if (kg_abs) {
            rows_abs = (double *)calloc((size_t)(n_rows > 0 ? n_rows : 1) * QO_NG, sizeof(double));
            if (!rows_abs) { free(rows); return -1; }
        }
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t it = k0; it < k1; ++it) {
            int64_t tile = tile_list ? tile_list[it] : it;
            bwd_tile(tile, H, W, dirs, tile_offsets, tile_prims, tiles_x, pr, st,
                     f_color, f_alpha, f_depth, f_depthsq, f_normal, f_curv, f_dist,
                     u_color, u_alpha, u_depth, u_normal, u_curv, u_dist,
                     rows + (tile_offsets[tile] - base) * QO_NG,
                     rows_abs ? rows_abs + (tile_offsets[tile] - base) * QO_NG : NULL);
        }
        for (int64_t i = 0; i < n_rows; ++i) {
            double *dst = kg + tile_prims[base + i] * QO_NG;
            const double *src = rows + i * QO_NG;
            for (int j = 0; j < QO_NG; ++j) dst[j] += src[j];
            if (kg_abs) {
                double *da = kg_abs + tile_prims[base + i] * QO_NG;
                const double *sa = rows_abs + i * QO_NG;
                for (int j = 0; j < QO_NG; ++j) da[j] += sa[j];
            }
        }
        free(rows);
        free(rows_abs);
    }
    return 0;
}

/* tile_sort_depths, raster_kernels.py:684-716 */
void qo_tile_keys(int64_t n, const int64_t *pair_tiles, const int64_t *pair_prims,
                  int64_t tiles_x, const qo_prims *pr, const double *vert_u,
                  const double *vert_v, const double *center_dist, double cx, double cy,
                  double fx, double fy, int64_t W, int64_t H, int euclid, double t_clip,
                  double *keys)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        int64_t p = pair_prims[i], tile = pair_tiles[i];
        int64_t ty = tile / tiles_x, tx = tile % tiles_x;
        int64_t ulo = tx * 16, uhi = (tx * 16 + 16 < W ? tx * 16 + 16 : W) - 1;
        int64_t vlo = ty * 16, vhi = (ty * 16 + 16 < H ? ty * 16 + 16 : H) - 1;
        int64_t iu = (int64_t)floor(vert_u[p]), iv = (int64_t)floor(vert_v[p]);
        iu = iu < ulo ? ulo : (iu > uhi ? uhi : iu);
        iv = iv < vlo ? vlo : (iv > vhi ? vhi : iv);
        double u = (double)iu, v = (double)iv;
        double ddx = (u + 0.5 - cx) / fx, ddy = (v + 0.5 - cy) / fy;
        double nrm = sqrt(ddx * ddx + ddy * ddy + 1.0);
        double dh[3];
        local_dir(pr->M + 9 * p, ddx / nrm, ddy / nrm, 1.0 / nrm, dh);
        const double *wv = pr->wv + 3 * p, *sv = pr->sv + 3 * p, *oh = pr->ohat + 3 * p;
        qo_hit h;
        qo_fragment_geometry(wv[0], wv[1], wv[2], sv[0], sv[1], sv[2], oh[0], oh[1],
                             oh[2], dh[0], dh[1], dh[2], pr->planar[p] == 1, euclid,
                             t_clip, &h);
        keys[i] = h.valid ? h.t : center_dist[p];
    }
}

int qo_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------ diagnostics
 * Per-pixel trace: every accepted candidate (tile-list order) and every
 * emitted fragment (compositing order) with its transmittance before it. */
typedef struct {
    qo_fwd_px px;
    int max, n;
    int64_t *prim;
    double *t, *abar, *T;
} qo_trace_ctx;

static int trace_visit(void *vctx, int64_t pos, int64_t p, const qo_frag *f)
{
    qo_trace_ctx *c = (qo_trace_ctx *)vctx;
    if (c->n < c->max) {
        c->prim[c->n] = p; c->t[c->n] = f->h.t; c->abar[c->n] = f->abar; c->T[c->n] = c->px.T;
    }
    c->n++;
    return fwd_visit(&c->px, pos, p, f);
}

int qo_trace_pixel(int64_t W, const double *dirs, const int64_t *tile_offsets,
                   const int64_t *tile_prims, int64_t tiles_x, const qo_prims *pr,
                   const qo_settings *st, int64_t u, int64_t v, int max,
                   int64_t *acc_prim, double *acc_t, double *acc_abar, int *n_acc,
                   int64_t *em_prim, double *em_t, double *em_abar, double *em_T)
{
    int64_t tile = (v / 16) * tiles_x + u / 16, px = v * W + u;
    const double *d = dirs + 3 * px;
    int na = 0;
    for (int64_t i = tile_offsets[tile]; i < tile_offsets[tile + 1]; ++i) {
        int64_t p = tile_prims[i];
        const int64_t *bb = pr->bbox + 4 * p;
        if (u < bb[0] || u > bb[1] || v < bb[2] || v > bb[3]) continue;
        qo_frag f;
        shade(pr, p, d[0], d[1], d[2], st, &f);
        if (!f.h.valid) continue;
        if (na < max) { acc_prim[na] = p; acc_t[na] = f.h.t; acc_abar[na] = f.abar; }
        na++;
    }
    *n_acc = na;
    qo_trace_ctx c;
    memset(&c, 0, sizeof c);
    c.px.colors = pr->colors; c.px.T = 1.0; c.px.t_term = st->t_term;
    c.max = max; c.prim = em_prim; c.t = em_t; c.abar = em_abar; c.T = em_T;
    qo_entry ring[QO_RING];
    pixel_stream(pr, tile_prims, tile_offsets[tile], tile_offsets[tile + 1], u, v, d, st,
                 trace_visit, &c, ring);
    return c.n;
}
