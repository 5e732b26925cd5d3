/*
 * qgs_b200 -- C ABI of the B200 (sm_100a) Quadratic Gaussian Splatting tile
 * rasterizer.
 *
 * The reference path is pure Python: qgsplat.rasterizer.prepare / forward /
 * backward (/root/reference/pkg/src/qgsplat/rasterizer.py:123,198,230) over
 * numba kernels (raster_kernels.py:83 forward_kernel, :505 backward_kernel,
 * :673 merge_pair_grads, :684 tile_sort_depths).  This library replaces that
 * path one stage per entry point; the Python drop-in
 * (paper_2411_16392_b200/rasterizer.py) binds it with ctypes.
 * shows the binding a qgsplat maintainer would add.
 *
 * Conventions
 *   - Every pointer is DEVICE memory unless stated; the caller owns and
 *     allocates all buffers (sizes come from the *_bytes queries).  The
 *     library never calls cudaMalloc and never synchronises the stream.
 *   - All calls are asynchronous on `stream` and return 0 on success or a
 *     negative QGS_E_* code; qgs_last_error() gives a thread-local message.
 *   - Per-primitive parameters are fp32; geometry that feeds integer
 *     outputs (screen boxes, tile sort keys) is computed in fp64 on device.
 */
#ifndef QGS_B200_H
#define QGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *qgs_stream_t; /* == cudaStream_t */

#define QGS_TILE 16          /* bounds.py:19 */
#define QGS_KG_STRIDE 16     /* floats per primitive in the kernel-gradient buffer */
#define QGS_AUX_PLANES 12    /* float64 planes per pixel kept for the backward */

enum {
    QGS_OK = 0,
    QGS_E_ARG = -1,          /* invalid argument / size */
    QGS_E_CUDA = -2,         /* a CUDA launch or API call failed */
    QGS_E_CAPACITY = -3,     /* a workspace is too small */
};

/* Pinhole camera (cameras.py:15-94).  center = -R_wc^T t_wc, computed by the
 * caller exactly as Camera.center does (cameras.py:48-51). */
typedef struct qgs_camera {
    double fx, fy, cx, cy;
    int32_t width, height;
    double R_wc[9];          /* row-major world->camera rotation */
    double t_wc[3];
    double center[3];
} qgs_camera;

/* RenderSettings (rasterizer.py:22-30). */
typedef struct qgs_settings {
    double background[3];
    double t_near_clip, alpha_floor, alpha_clamp, t_term;
    int32_t resort, euclidean_density;
    int32_t no_cull;         /* extension: 1 disables the forward's conic cull (the
                                results are identical either way; tests check it) */
    int32_t exact_decisions; /* extension: 1 re-makes every selection / alpha-floor
                                decision whose fp32 margin is inside its rounding band
                                in fp64 (the reference's float64 accepted set; slower) */
} qgs_settings;

/* Raw primitive parameters, PrimitiveSet layout (model.py:126-141), fp32. */
typedef struct qgs_params {
    const float *centers;      /* P*3 */
    const float *quats;        /* P*4, (w, x, y, z), not necessarily unit */
    const float *raw_scales;   /* P*3 */
    const float *raw_signs;    /* P*3 */
    const float *raw_opacity;  /* P */
    const float *sh;           /* P*3*sh_coeffs, channel-major per primitive */
    int32_t P;
    int32_t sh_coeffs;         /* (deg+1)^2 in {1, 4, 9, 16} */
} qgs_params;

/* Forward outputs, RenderTargets (rasterizer.py:61-74).  Maps are H*W
 * row-major (x3 interleaved for colour/normal). */
#define QGS_FRAG_PAGE 16        /* fragment slots per pixel per log page */
#define QGS_FRAG_MAX_PAGES 32   /* pages per raster warp: 512 fragments per pixel */

typedef struct qgs_targets {
    float *color;              /* color_raw + T * background */
    float *color_raw;
    float *alpha, *depth, *depth_sq, *depth_median;
    float *normal;
    float *curvature, *distortion, *transmittance;
    int32_t *n_fragments;      /* H*W */
    int32_t *violations;       /* per tile (tiles_x*tiles_y) */
    double *aux;               /* QGS_AUX_PLANES*H*W float64 blend sums; required by
                                  qgs_backward, may be NULL for a forward-only call */
    unsigned long long *counters; /* optional, accumulated (+=): [0] candidates inside
                                  the pixel box, [1] accepted fragments, [2] composited,
                                  [3] candidates left by the conic cull, [4] candidates
                                  passing the coarse fp32 test (5 entries) */
    /* Optional fragment log (frag_prim == NULL: none), written by the forward
     * and read by the backward instead of replaying the candidate tests.
     * Paged: a pool of pages, each QGS_FRAG_PAGE fragment slots deep for the
     * 32 pixels of one raster warp (an 8x4 block), slot (page, k, lane) at
     * ((page * QGS_FRAG_PAGE + k) * 32 + lane).  A raster warp takes pages
     * from the pool (atomically, *frag_pool_next) as its deepest pixel grows,
     * up to QGS_FRAG_MAX_PAGES; its page ids go to
     * frag_page_table[warp * QGS_FRAG_MAX_PAGES + i] and their number to
     * frag_page_count[warp] (-1: pool exhausted or a pixel deeper than
     * QGS_FRAG_PAGE * QGS_FRAG_MAX_PAGES -- the backward replays that block
     * with the full candidate test).  Warps are 8 per tile, tile-major.  So
     * memory scales with the fragments composited, not with pixels x cap. */
    int32_t *frag_prim;        /* pool: primitive of each logged fragment */
    double *frag_t;            /* pool: its float64 depth */
    float *frag_xy;            /* pool x2 (optional): its local hit point (x, y) as the
                                  forward shaded it, so the backward re-shades in fp32 */
    int32_t *frag_page_table;  /* n_warps * QGS_FRAG_MAX_PAGES */
    int32_t *frag_page_count;  /* n_warps */
    int32_t *frag_pool_next;   /* device counter: pages handed out (the forward zeroes it) */
    int32_t frag_pool_pages;   /* pool capacity in pages */
    int32_t *tile_order;       /* optional scratch of tiles_x*tiles_y ints: the forward
                                  fills it with the tiles by descending pair count and
                                  both raster kernels run the heaviest tiles first (NULL:
                                  natural order) */
} qgs_targets;

/* Upstream map gradients (rasterizer.py:230-250); NULL = all zero. */
typedef struct qgs_upstream {
    const float *color;        /* H*W*3 */
    const float *alpha, *depth;
    const float *normal;       /* H*W*3 */
    const float *curvature, *distortion;
} qgs_upstream;

/* Raw-parameter gradients, GradientBuffer (rasterizer.py:77-108); fp32,
 * ACCUMULATED (+=) so several views sum on device before one all-reduce. */
typedef struct qgs_grads {
    float *centers, *quats, *raw_scales, *raw_signs, *raw_opacity, *sh;
    float *screen_center;      /* P*2 */
} qgs_grads;

/* ---- stage 1: per-primitive preprocessing (rasterizer.py:124-158,
 *      bounds.py:272-292, sh.py:82-88).  Writes the per-primitive state into
 *      `prep` (qgs_prep_bytes(P) bytes) and the total (tile, primitive) pair
 *      count into *d_n_pairs (device int64) -- or -k when k primitives have
 *      non-finite raw scales/signs (model.py:37-38: the caller raises
 *      ParameterError from the one read it makes anyway; qgs_bin must not be
 *      called then). */
size_t qgs_prep_bytes(int32_t P);
int qgs_preprocess(const qgs_params *prims, const qgs_camera *cam,
                   const qgs_settings *st, void *prep, int64_t *d_n_pairs,
                   qgs_stream_t stream);
/* qgs_preprocess in two parts, together bit-identical to it: everything but
 * the SH colour (geometry, boxes, tile counts, pair offsets), then the colour
 * (sh.py:82-88) -- so that the SH coefficients (3/4 of the parameter bytes at
 * degree 3) can still be on their way from the host while the view is binned.
 * qgs_preprocess_color must run before qgs_forward. */
int qgs_preprocess_geometry(const qgs_params *prims, const qgs_camera *cam,
                            const qgs_settings *st, void *prep, int64_t *d_n_pairs,
                            qgs_stream_t stream);
int qgs_preprocess_color(const qgs_params *prims, const qgs_camera *cam, void *prep,
                         qgs_stream_t stream);

/* ---- stage 2: key duplication + per-tile (depth key, id) sort
 *      (rasterizer.py:159-181, raster_kernels.py:684-716).  tile_offsets has
 *      tiles_x*tiles_y+1 entries, tile_prims n_pairs entries; both
 *      bit-identical to the reference's np.lexsort((prim, key, tile)). */
size_t qgs_bin_workspace_bytes(int32_t P, int64_t n_pairs, int32_t n_tiles);
int qgs_bin(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
            int64_t n_pairs, void *workspace, size_t workspace_bytes,
            int32_t *tile_offsets, int32_t *tile_prims, qgs_stream_t stream);
/* Debug/parity: the float64 sort key of every sorted pair (same order as
 * tile_prims), recomputed from (tile, prim). */
int qgs_sorted_keys(const void *prep, int32_t P, const qgs_camera *cam,
                    const qgs_settings *st, const int32_t *tile_offsets,
                    const int32_t *tile_prims, int64_t n_pairs, double *keys,
                    qgs_stream_t stream);
/* Unit-level key kernel: keys of explicit (tile, prim) pairs from CALLER-GIVEN
 * float64 prepared arrays (the oracle's), for the bit-exact key test. */
int qgs_tile_keys_f64(int64_t n, const int64_t *pair_tiles, const int64_t *pair_prims,
                      int32_t tiles_x, const double *ohat, const double *M,
                      const double *wv, const double *sv, const uint8_t *planar,
                      const double *vert_u, const double *vert_v, const double *dist,
                      const qgs_camera *cam, const qgs_settings *st, double *keys,
                      qgs_stream_t stream);

/* ---- stage 3: forward raster (raster_kernels.py:83-286, rasterizer.py:198-227) */
int qgs_forward(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
                const int32_t *tile_offsets, const int32_t *tile_prims,
                const qgs_targets *out, qgs_stream_t stream);

/* ---- stage 4: backward raster (raster_kernels.py:289-681).  kg is
 *      P*QGS_KG_STRIDE floats, zeroed by the caller; slots: ohat 0-2,
 *      omega 3-5 (the skew part of the local-frame rotation accumulator X,
 *      g_R = R X, which replaces the reference's M and Nmat slots: the
 *      quaternion gradient sees only the skew part), w 6-8 and s 9-11 (with
 *      the lambda terms folded in), alpha 12, colour 13-15. */
int qgs_backward(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
                 const int32_t *tile_offsets, const int32_t *tile_prims,
                 const qgs_targets *fwd, const qgs_upstream *up, float *kg,
                 qgs_stream_t stream);

/* ---- stage 4, deterministic variant (RenderSettings.deterministic): the
 *      same kernel gradients, added to kg in a fixed order with fp64 sums --
 *      bitwise repeatable like the reference's serial merge
 *      (raster_kernels.py:673-681; pkg/tests/test_rasterizer_gradients.py:
 *      217-229).  Each composited fragment writes its slots to a row fixed
 *      by the forward (a scan of n_fragments in raster-warp order); rows are
 *      grouped per primitive by a stable radix sort and summed in row order.
 *      n_frags = the sum of fwd->n_fragments; workspace from
 *      qgs_backward_det_workspace_bytes. */
size_t qgs_backward_det_workspace_bytes(int32_t P, int64_t n_frags, const qgs_camera *cam);
int qgs_backward_deterministic(const void *prep, int32_t P, const qgs_camera *cam,
                               const qgs_settings *st, const int32_t *tile_offsets,
                               const int32_t *tile_prims, const qgs_targets *fwd,
                               const qgs_upstream *up, float *kg, int64_t n_frags,
                               void *workspace, size_t workspace_bytes, qgs_stream_t stream);

/* ---- stage 5: chain to raw parameters (rasterizer.py:270-334). */
int qgs_chain(const qgs_params *prims, const void *prep, const float *kg,
              const qgs_camera *cam, const qgs_grads *out, qgs_stream_t stream);

/* Per-primitive debug export of the prepared state (parity tests):
 * scales P*3 (f64), alphas P (f64), colors P*3 (f64), pix_bbox P*4 (i32),
 * planar P (u8). Any pointer may be NULL. */
int qgs_export_prep(const void *prep, int32_t P, double *scales, double *alphas,
                    double *colors, int32_t *pix_bbox, uint8_t *planar,
                    qgs_stream_t stream);

/* The rest of the reference's PreparedView (rasterizer.py:33-58, populated
 * at :124-195), recomputed on the device from the raw parameters with the
 * same fp64 device functions as qgs_preprocess (ohat, M, wv are the exact
 * values the raster kernels use).  Any pointer may be NULL.  Shapes:
 * R, M, Nmat P*9 (row-major 3x3), ohat, wv, view_dirs P*3, lam P*2,
 * view_dist P (f64); clamped, color_clamped P*3 (u8). */
typedef struct qgs_prep_export {
    double *R, *ohat, *M, *Nmat, *wv, *lam, *view_dirs, *view_dist;
    uint8_t *clamped, *color_clamped;
} qgs_prep_export;
int qgs_export_prep_geometry(const qgs_params *prims, const void *prep, const qgs_camera *cam,
                             const qgs_prep_export *out, qgs_stream_t stream);

/* PreparedView.dirs: unit camera-frame ray of every pixel centre
 * (cameras.py:53-59, the reference's operation order), H*W*3 f64. */
int qgs_pixel_dirs(const qgs_camera *cam, double *dirs, qgs_stream_t stream);

/* Diagnostics build counters (QGS_UTIL_COUNTERS; 0 entries otherwise): copies
 * and clears up to n of [float64 band re-decisions, near-tangent roots decided
 * by the fp64 closed form, candidates rejected by the coarse test's stage 1,
 * by its stage 2].  Returns the number copied. */
int qgs_diag_counters(unsigned long long *out, int n);

/* Diagnostics: replay one pixel's fragment stream (same device functions as
 * the raster kernels) and record up to `max` accepted candidates (tile-list
 * order) and emitted fragments (compositing order, with T before each).
 * counts[0] = accepted, counts[1] = emitted. */
int qgs_trace_pixel(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
                    const int32_t *tile_offsets, const int32_t *tile_prims, int32_t u, int32_t v,
                    int32_t max, int32_t *acc_prim, float *acc_t, float *acc_abar,
                    int32_t *em_prim, float *em_t, float *em_abar, double *em_T,
                    int32_t *counts, qgs_stream_t stream);

/* ---- Loss producers: the upstream maps for
 * qgs_backward, computed from the forward's maps in place.  They replace
 * qgsplat.losses (/root/reference/pkg/src/qgsplat/losses.py) and
 * qgsplat.ssim (ssim.py); the call sites are train.py:193-211.  All maps are
 * fp32, row-major (H, W[, C]); arithmetic is fp64; `values` is device fp64.
 * Gradient outputs are ACCUMULATED (+= weight * d loss / d map) and may be
 * NULL when only the value is wanted.  Workspace: qgs_loss_workspace_bytes.
 */
size_t qgs_loss_workspace_bytes(int32_t H, int32_t W, int32_t C);

/* losses.py:36-50 photometric (1-m) L1 + m (1 - SSIM), ssim.py:41-86 SSIM
 * (11x11 Gaussian, sigma 1.5, zero padding, crop mean).  C in [1, 4].
 * values[0] = loss, values[1] = L1 mean, values[2] = SSIM mean (0 when m = 0).
 * QGS_E_ARG when m > 0 and H or W < 11 (ssim.py:53-54). */
int qgs_loss_photometric(const float *render, const float *gt, int32_t H, int32_t W,
                         int32_t C, double lambda_ssim, double weight, float *d_render,
                         double *values, void *workspace, size_t workspace_bytes,
                         qgs_stream_t stream);

/* losses.py:53-56: values[0] = mean(distortion); d_dist += weight / (H W). */
int qgs_loss_distortion(const float *distortion, int32_t H, int32_t W, double weight,
                        float *d_dist, double *values, void *workspace,
                        size_t workspace_bytes, qgs_stream_t stream);

/* losses.py:59-89 depth_to_normal: N (H, W, 3) camera-frame normals from
 * central differences of the back-projected depth (distance along the unit
 * pixel ray), mask (H, W) u8.  Only intrinsics and size of `cam` are used. */
int qgs_depth_to_normal(const float *depth, const float *alpha, const qgs_camera *cam,
                        double alpha_thresh, float *N, uint8_t *mask, qgs_stream_t stream);

/* losses.py:97-113 curvature_guided_normal_consistency.  With depth != NULL
 * the pseudo ground truth (N, mask) is computed from depth / alpha on the fly
 * (depth_to_normal fused in; N and mask ignored), else read from N / mask.
 * values[0] = loss, values[1] = mask count. */
int qgs_loss_normal_consistency(const float *alpha, const float *normal, const float *curvature,
                                const float *depth, const float *N, const uint8_t *mask,
                                const qgs_camera *cam, double alpha_thresh, double eps_curvature,
                                int32_t guided, double weight, float *d_alpha, float *d_normal,
                                float *d_curvature, double *values, void *workspace,
                                size_t workspace_bytes, qgs_stream_t stream);

/* ---- Optimizer step and densification: Adam over
 * the six groups (optim.py:14-64) and clone / split / prune
 * (train.py:269-335) on the device.  Call sites: train.py:239-262.  Groups
 * are in PrimitiveSet order; state (Adam moments) is fp32 with the groups'
 * shapes; arithmetic is fp64. */
typedef struct qgs_groups {          /* a writable parameter-group set */
    float *centers, *quats, *raw_scales, *raw_signs, *raw_opacity, *sh;
    int32_t P;
    int32_t sh_coeffs;
} qgs_groups;

typedef struct qgs_adam_config {
    double lr[6];                    /* per group */
    double beta1, beta2, eps;        /* optim.py:15 defaults 0.9, 0.999, 1e-15 */
    int64_t t;                       /* the step number after the increment */
    const uint8_t *freeze[6];        /* per-element freeze masks or NULL (optim.py:24) */
} qgs_adam_config;

typedef struct qgs_densify_stats {   /* train.py:263-267, fp64 */
    double *grad_accum;              /* P */
    double *grad_count;              /* P */
    double *center_accum;            /* P*3 */
} qgs_densify_stats;

typedef struct qgs_densify_config {  /* config.py:24-43 */
    double grad_threshold, percent_dense, scene_extent, prune_opacity, clone_nudge;
    int64_t max_primitives;
} qgs_densify_config;

/* optim.py:23-47 Adam.step (non-finite gradient rows skip, counted into
 * *d_skipped; quaternions renormalised), fused with the densification
 * statistics of train.py:239-244 when stats != NULL. */
int qgs_adam_step(const qgs_groups *prims, const qgs_grads *grads, const qgs_groups *m,
                  const qgs_groups *v, const qgs_adam_config *cfg,
                  const qgs_densify_stats *stats, uint64_t *d_skipped, qgs_stream_t stream);

/* train.py:269-329 in two calls.  plan: decisions and the ordered
 * compaction offsets into `workspace`; d_counts (device int64[4]) = output
 * primitives, survivors, clones, split parents (the host reads d_counts[0]
 * to size the outputs).  apply: writes [survivors | clones | split + |
 * split -], opacity-pruned, with the survivors' Adam state and zero state
 * for the new primitives. */
size_t qgs_densify_workspace_bytes(int32_t P);
int qgs_densify_plan(const qgs_params *prims, const qgs_densify_stats *stats,
                     const qgs_densify_config *cfg, void *workspace, size_t workspace_bytes,
                     int64_t *d_counts, qgs_stream_t stream);
int qgs_densify_apply(const qgs_params *prims, const qgs_params *m, const qgs_params *v,
                      const qgs_densify_stats *stats, const qgs_densify_config *cfg,
                      const void *workspace, const qgs_groups *out, const qgs_groups *out_m,
                      const qgs_groups *out_v, qgs_stream_t stream);

/* train.py:332-335: opacity capped at `cap` (0.01), its Adam state zeroed. */
int qgs_reset_opacity(const qgs_groups *prims, const qgs_groups *m, const qgs_groups *v,
                      double cap, qgs_stream_t stream);

/* ---- Multi-view reprojection + NCC regulariser:
 * multiview.py:108-311, called at train.py:215-233.  Maps fp32: depth and
 * alpha (H, W), camera-frame normal (H, W, 3), the ground-truth photo
 * (H, W, image_channels) reduced to gray by its channel mean. */
typedef struct qgs_mv_maps {
    const float *depth, *alpha, *normal, *image;
    int32_t height, width, image_channels;
} qgs_mv_maps;

typedef struct qgs_mv_config {       /* multiview.py:17-23 */
    int32_t patch_size;              /* odd, <= 13; default 7 */
    double alpha_thresh, min_denom, ncc_eps;
    int32_t full_chain;
} qgs_mv_config;

typedef struct qgs_mv_grads {        /* upstream maps the loss accumulates into */
    float *depth, *alpha, *normal;   /* any may be NULL */
} qgs_mv_grads;

size_t qgs_multiview_workspace_bytes(int32_t H, int32_t W, int32_t Hn, int32_t Wn);
/* values (device fp64[4]) = loss, n_valid, mean reprojection error (px), mean
 * NCC (0, 0, 0, 1 when no pixel is valid).  up_ref / up_nbr (either may
 * be NULL) ACCUMULATE weight * the loss gradient w.r.t. each view's maps. */
int qgs_multiview_loss(const qgs_mv_maps *ref, const qgs_camera *cam_ref, const qgs_mv_maps *nbr,
                       const qgs_camera *cam_nbr, const qgs_mv_config *cfg, double weight,
                       const qgs_mv_grads *up_ref, const qgs_mv_grads *up_nbr, double *values,
                       void *workspace, size_t workspace_bytes, qgs_stream_t stream);

const char *qgs_last_error(void);
int qgs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QGS_B200_H */
