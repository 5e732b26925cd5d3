#include <algorithm>
// extern "C" entry points of libqgs_b200.so (declared in include/qgs_b200.h).
#include <cstdio>
#include <string>

#include "kernels.cuh"
#include "losses.cuh"
#include "optim.cuh"
#include "multiview.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

int cuda_fail(const char *where, cudaError_t e)
{
    return fail(QGS_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define QGS_CK(call)                                                     \
    do {                                                                 \
        cudaError_t e_ = (call);                                         \
        if (e_ != cudaSuccess) return cuda_fail(#call, e_);              \
    } while (0)
#define QGS_LAUNCHED(name)                                               \
    do {                                                                 \
        cudaError_t e_ = cudaGetLastError();                             \
        if (e_ != cudaSuccess) return cuda_fail(name, e_);               \
    } while (0)

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// prep = [PrepView arrays][scan block sums]
size_t scan_blocks(int32_t P) { return (size_t)cdiv(P > 0 ? P : 1, qgs::SCAN_ITEMS); }

int64_t *scan_sums_ptr(void *prep, int32_t P)
{
    return reinterpret_cast<int64_t *>(static_cast<char *>(prep) + qgs::prep_bytes(P));
}

struct BinWs {
    int *diff;
    int32_t *cursor;
    uint64_t *bucket, *tmp;
    double *rays;         // W*H*3 unit pixel rays (fp64) for the key kernel
    int32_t *order;       // tiles by descending pair count (sort schedule)
    qgs::HugeSort *huge;  // the huge tiles' buckets between the two sort stages
    size_t bytes;
};

BinWs bin_ws(void *base, int32_t tiles_x, int32_t tiles_y, int64_t n_pairs)
{
    char *b = static_cast<char *>(base);
    BinWs w;
    size_t o = 0;
    size_t ndiff = (size_t)(tiles_x + 1) * (tiles_y + 1);
    w.diff = reinterpret_cast<int *>(b + o);        o += qgs::align256(ndiff * sizeof(int));
    w.cursor = reinterpret_cast<int32_t *>(b + o);  o += qgs::align256((size_t)tiles_x * tiles_y * 4);
    w.bucket = reinterpret_cast<uint64_t *>(b + o); o += qgs::align256((size_t)n_pairs * 8);
    w.tmp = reinterpret_cast<uint64_t *>(b + o);    o += qgs::align256((size_t)n_pairs * 8);
    w.rays = reinterpret_cast<double *>(b + o);     o += qgs::align256((size_t)tiles_x * tiles_y * 256 * 24);
    w.order = reinterpret_cast<int32_t *>(b + o);   o += qgs::align256((size_t)tiles_x * tiles_y * 4);
    w.huge = reinterpret_cast<qgs::HugeSort *>(b + o); o += qgs::align256(qgs::huge_sort_bytes());
    w.bytes = o;
    return w;
}

int configure()
{
    QGS_CK(qgs::ensure_smem_attr(reinterpret_cast<const void *>(qgs::tile_sort_kernel),
                                 (int)qgs::sort_smem_bytes()));
    QGS_CK(qgs::ensure_smem_attr(reinterpret_cast<const void *>(qgs::tile_sort_chunks_kernel),
                                 (int)qgs::sort_smem_bytes()));
    return 0;
}

int check_cam(const qgs_camera *cam)
{
    if (!cam) return fail(QGS_E_ARG, "camera is NULL");
    if (cam->width <= 0 || cam->height <= 0 || cam->width > 32767 || cam->height > 32767)
        return fail(QGS_E_ARG, "image size must be in [1, 32767]");
    if (!(cam->fx > 0 && cam->fy > 0)) return fail(QGS_E_ARG, "focal lengths must be positive");
    return 0;
}

}  // namespace

extern "C" {

const char *qgs_last_error(void) { return g_err.c_str(); }

int qgs_diag_counters(unsigned long long *out, int n)
{
    if (!out || n < 0) return fail(QGS_E_ARG, "NULL argument");
    return qgs::diag_counters(out, n);
}
int qgs_version(void) { return 1; }

size_t qgs_prep_bytes(int32_t P)
{
    return qgs::prep_bytes(P) + qgs::align256(scan_blocks(P) * sizeof(int64_t));
}

static int preprocess_impl(const qgs_params *prims, const qgs_camera *cam, const qgs_settings *st,
                           void *prep, int64_t *d_n_pairs, qgs_stream_t stream, int with_color)
{
    if (!prims || !st || !prep || !d_n_pairs) return fail(QGS_E_ARG, "NULL argument");
    if (int rc = check_cam(cam)) return rc;
    if (prims->P < 0) return fail(QGS_E_ARG, "P < 0");
    if (prims->sh_coeffs != 1 && prims->sh_coeffs != 4 && prims->sh_coeffs != 9 &&
        prims->sh_coeffs != 16)
        return fail(QGS_E_ARG, "sh_coeffs must be 1, 4, 9 or 16");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int P = prims->P;
    qgs::PrepView pv = qgs::prep_view(prep, P);
    qgs::CamK ck = qgs::make_camk(*cam);
    if (P == 0) {
        QGS_CK(cudaMemsetAsync(d_n_pairs, 0, sizeof(int64_t), s));
        QGS_CK(cudaMemsetAsync(pv.pair_off, 0, sizeof(int64_t), s));
        return 0;
    }
    QGS_CK(cudaMemsetAsync(pv.nonfinite, 0, sizeof(int32_t), s));
    qgs::preprocess_kernel<<<cdiv(P, 128), 128, 0, s>>>(*prims, ck, pv, st->euclidean_density,
                                                         with_color);
    QGS_LAUNCHED("preprocess_kernel");
    const int nb = (int)scan_blocks(P);
    int64_t *sums = scan_sums_ptr(prep, P);
    qgs::scan_sums_kernel<<<nb, qgs::SCAN_THREADS, 0, s>>>(pv.ntiles, P, sums);
    qgs::scan_top_kernel<<<1, qgs::SCAN_THREADS, 0, s>>>(sums, nb, d_n_pairs, pv.pair_off, P,
                                                         pv.nonfinite);
    qgs::scan_out_kernel<<<nb, qgs::SCAN_THREADS, 0, s>>>(pv.ntiles, P, sums, pv.pair_off);
    QGS_LAUNCHED("scan kernels");
    return 0;
}

int qgs_preprocess(const qgs_params *prims, const qgs_camera *cam, const qgs_settings *st,
                   void *prep, int64_t *d_n_pairs, qgs_stream_t stream)
{
    return preprocess_impl(prims, cam, st, prep, d_n_pairs, stream, 1);
}

int qgs_preprocess_geometry(const qgs_params *prims, const qgs_camera *cam,
                            const qgs_settings *st, void *prep, int64_t *d_n_pairs,
                            qgs_stream_t stream)
{
    return preprocess_impl(prims, cam, st, prep, d_n_pairs, stream, 0);
}

int qgs_preprocess_color(const qgs_params *prims, const qgs_camera *cam, void *prep,
                         qgs_stream_t stream)
{
    if (!prims || !prep) return fail(QGS_E_ARG, "NULL argument");
    if (int rc = check_cam(cam)) return rc;
    if (prims->P < 0) return fail(QGS_E_ARG, "P < 0");
    if (prims->sh_coeffs != 1 && prims->sh_coeffs != 4 && prims->sh_coeffs != 9 &&
        prims->sh_coeffs != 16)
        return fail(QGS_E_ARG, "sh_coeffs must be 1, 4, 9 or 16");
    if (prims->P == 0) return 0;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    qgs::color_kernel<<<cdiv(prims->P, 128), 128, 0, s>>>(*prims, qgs::make_camk(*cam),
                                                          qgs::prep_view(prep, prims->P));
    QGS_LAUNCHED("color_kernel");
    return 0;
}

size_t qgs_bin_workspace_bytes(int32_t P, int64_t n_pairs, int32_t n_tiles)
{
    (void)P;
    // diff grid is at most (n_tiles + tiles_x + tiles_y + 1) entries; bound it by 2*n_tiles + 2*32768
    size_t ndiff = 2 * (size_t)n_tiles + 65538;
    return qgs::align256(ndiff * sizeof(int)) + qgs::align256((size_t)n_tiles * 4) +
           2 * qgs::align256((size_t)n_pairs * 8) + qgs::align256((size_t)n_tiles * 256 * 24) +
           qgs::align256((size_t)n_tiles * 4) + qgs::align256(qgs::huge_sort_bytes()) + 256;
}

int qgs_bin(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
            int64_t n_pairs, void *workspace, size_t workspace_bytes, int32_t *tile_offsets,
            int32_t *tile_prims, qgs_stream_t stream)
{
    if (!prep || !st || !tile_offsets) return fail(QGS_E_ARG, "NULL argument");
    if (int rc = check_cam(cam)) return rc;
    if (n_pairs < 0 || n_pairs > 0x7fffffffLL) return fail(QGS_E_ARG, "n_pairs out of int32 range");
    if (int rc = configure()) return rc;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    qgs::CamK ck = qgs::make_camk(*cam);
    qgs::SetK sk = qgs::make_setk(*st);
    const int n_tiles = ck.tiles_x * ck.tiles_y;
    BinWs ws = bin_ws(workspace, ck.tiles_x, ck.tiles_y, n_pairs);
    sk.pbits = 1;                                  // id bits of the sort composite
    while (sk.pbits < 31 && (1LL << sk.pbits) < (long long)P) ++sk.pbits;
    if (ws.bytes > workspace_bytes) return fail(QGS_E_CAPACITY, "bin workspace too small");
    qgs::PrepView pv = qgs::prep_view(const_cast<void *>(prep), P);
    QGS_CK(cudaMemsetAsync(ws.diff, 0, (size_t)(ck.tiles_x + 1) * (ck.tiles_y + 1) * sizeof(int), s));
    if (P > 0) {
        qgs::tile_diff_kernel<<<cdiv(P, 256), 256, 0, s>>>(pv.bbox, P, ck.tiles_x, ws.diff);
        QGS_LAUNCHED("tile_diff_kernel");
    }
    qgs::tile_offsets_kernel<<<1, 1024, 0, s>>>(ws.diff, ck.tiles_x, ck.tiles_y, tile_offsets,
                                                 ws.cursor);
    QGS_LAUNCHED("tile_offsets_kernel");
    if (n_pairs == 0) return 0;
    const int grid = (int)std::min<long long>(cdiv(n_pairs, 256), 148LL * 32);
    qgs::pixel_rays_kernel<<<cdiv((long long)ck.W * ck.H, 256), 256, 0, s>>>(ck, ws.rays);
    QGS_LAUNCHED("pixel_rays_kernel");
    qgs::pair_key_kernel<<<grid, 256, 0, s>>>(pv, P, n_pairs, ck, sk, ws.rays, ws.cursor, ws.bucket);
    QGS_LAUNCHED("pair_key_kernel");
    pv.rays = ws.rays;
    // largest tiles first: one CTA sorts a tile, so a 100K-entry tile started
    // last would be the kernel's tail
    qgs::tile_order_kernel<<<1, 1024, qgs::ORDER_SMEM, s>>>(tile_offsets, n_tiles, ws.order, 1);
    QGS_LAUNCHED("tile_order_kernel (sort)");
    QGS_CK(cudaMemsetAsync(&ws.huge->count, 0, sizeof(int), s));
    qgs::tile_sort_kernel<<<n_tiles, qgs::sort_threads(), qgs::sort_smem_bytes(), s>>>(
        tile_offsets, ws.bucket, ws.tmp, pv, ck, sk, tile_prims, ws.order, ws.huge);
    QGS_LAUNCHED("tile_sort_kernel");
    // the huge tiles' buckets, SORT_CHUNKS CTAs per tile (most CTAs exit at once)
    int cdev = 0, csms = 148;
    cudaGetDevice(&cdev);
    cudaDeviceGetAttribute(&csms, cudaDevAttrMultiProcessorCount, cdev);
    qgs::tile_sort_chunks_kernel<<<csms * 2, qgs::sort_threads(), qgs::sort_smem_bytes(), s>>>(
        tile_offsets, ws.tmp, pv, ck, sk, tile_prims, ws.huge);
    QGS_LAUNCHED("tile_sort_chunks_kernel");

    return 0;
}

int qgs_sorted_keys(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
                    const int32_t *tile_offsets, const int32_t *tile_prims, int64_t n_pairs,
                    double *keys, qgs_stream_t stream)
{
    (void)n_pairs;
    if (int rc = check_cam(cam)) return rc;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    qgs::CamK ck = qgs::make_camk(*cam);
    qgs::SetK sk = qgs::make_setk(*st);
    qgs::PrepView pv = qgs::prep_view(const_cast<void *>(prep), P);
    const int n_tiles = ck.tiles_x * ck.tiles_y;
    qgs::sorted_keys_kernel<<<n_tiles, 128, 0, s>>>(pv, tile_offsets, tile_prims, n_tiles, ck, sk,
                                                   keys);
    QGS_LAUNCHED("sorted_keys_kernel");
    return 0;
}

int qgs_tile_keys_f64(int64_t n, const int64_t *pair_tiles, const int64_t *pair_prims,
                      int32_t tiles_x, const double *ohat, const double *M, const double *wv,
                      const double *sv, const uint8_t *planar, const double *vert_u,
                      const double *vert_v, const double *dist, const qgs_camera *cam,
                      const qgs_settings *st, double *keys, qgs_stream_t stream)
{
    if (int rc = check_cam(cam)) return rc;
    if (n <= 0) return 0;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    qgs::CamK ck = qgs::make_camk(*cam);
    if (tiles_x != ck.tiles_x) return fail(QGS_E_ARG, "tiles_x does not match the camera");
    qgs::SetK sk = qgs::make_setk(*st);
    const int grid = (int)std::min<long long>(cdiv(n, 256), 148LL * 32);
    qgs::tile_keys_f64_kernel<<<grid, 256, 0, s>>>(n, pair_tiles, pair_prims, ohat, M, wv, sv,
                                                  planar, vert_u, vert_v, dist, ck, sk, keys);
    QGS_LAUNCHED("tile_keys_f64_kernel");
    return 0;
}

int qgs_forward(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
                const int32_t *tile_offsets, const int32_t *tile_prims, const qgs_targets *out,
                qgs_stream_t stream)
{
    if (!prep || !st || !out || !tile_offsets) return fail(QGS_E_ARG, "NULL argument");
    if (int rc = check_cam(cam)) return rc;
    if (int rc = configure()) return rc;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    qgs::CamK ck = qgs::make_camk(*cam);
    qgs::SetK sk = qgs::make_setk(*st);
    qgs::PrepView pv = qgs::prep_view(const_cast<void *>(prep), P);
    if (out->violations)
        QGS_CK(cudaMemsetAsync(out->violations, 0, sizeof(int32_t) * ck.tiles_x * ck.tiles_y, s));
    if (out->frag_prim) {
        if (!out->frag_t || !out->frag_page_table || !out->frag_page_count || !out->frag_pool_next)
            return fail(QGS_E_ARG, "fragment log: frag_t, page table, page count and pool "
                                   "counter are required with frag_prim");
        if (out->frag_pool_pages < 0) return fail(QGS_E_ARG, "frag_pool_pages < 0");
        QGS_CK(cudaMemsetAsync(out->frag_pool_next, 0, sizeof(int32_t), s));
    }
    if (out->tile_order) {
        qgs::tile_order_kernel<<<1, 1024, qgs::ORDER_SMEM, s>>>(tile_offsets, ck.tiles_x * ck.tiles_y,
                                                              out->tile_order, 0);
        QGS_LAUNCHED("tile_order_kernel");
    }
    const int n_slots = ck.tiles_x * ck.tiles_y * qgs::RASTER_BLOCKS_PER_TILE;
    const size_t fsm = qgs::FWD_WPC * qgs::fwd_smem_per_warp();
    QGS_CK(qgs::ensure_smem_attr(reinterpret_cast<const void *>(qgs::raster_fwd_exact_kernel), (int)fsm));
    QGS_CK(qgs::ensure_smem_attr(reinterpret_cast<const void *>(qgs::raster_fwd_kernel), (int)fsm));
    if (sk.exact)       // selection decisions inside their fp32 band re-made in float64
        qgs::raster_fwd_exact_kernel<<<n_slots / qgs::FWD_WPC, qgs::RASTER_THREADS * qgs::FWD_WPC,
                                       fsm, s>>>(pv.rec, pv.geo, pv.conic, tile_offsets,
                                                 tile_prims, ck, sk, *out);
    else
        qgs::raster_fwd_kernel<<<n_slots / qgs::FWD_WPC, qgs::RASTER_THREADS * qgs::FWD_WPC, fsm,
                                 s>>>(pv.rec, pv.geo, pv.conic, tile_offsets, tile_prims, ck, sk,
                                      *out);
    QGS_LAUNCHED("raster_fwd_kernel");
    return 0;
}

namespace {
int backward_impl(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
                  const int32_t *tile_offsets, const int32_t *tile_prims, const qgs_targets *fwd,
                  const qgs_upstream *up, float *kg, const qgs::DetRows &det, cudaStream_t s)
{
    qgs::CamK ck = qgs::make_camk(*cam);
    qgs::SetK sk = qgs::make_setk(*st);
    qgs::PrepView pv = qgs::prep_view(const_cast<void *>(prep), P);
    const int grid = ck.tiles_x * ck.tiles_y * qgs::RASTER_BLOCKS_PER_TILE;
    // blocks with a fragment log, then (a launch whose warps mostly exit at
    // once) the blocks without one
    const size_t bsm = qgs::BWD_WPC * qgs::bwd_smem_per_warp();
    QGS_CK(qgs::ensure_smem_attr(reinterpret_cast<const void *>(qgs::raster_bwd_det_kernel), (int)bsm));
    QGS_CK(qgs::ensure_smem_attr(reinterpret_cast<const void *>(qgs::raster_bwd_kernel), (int)bsm));
    if (det.rows)
        qgs::raster_bwd_det_kernel<<<grid / qgs::BWD_WPC, qgs::RASTER_THREADS * qgs::BWD_WPC, bsm,
                                     s>>>(pv.rec, pv.geo, tile_offsets, tile_prims, ck, sk, *fwd,
                                          *up, kg, det);
    else
        qgs::raster_bwd_kernel<<<grid / qgs::BWD_WPC, qgs::RASTER_THREADS * qgs::BWD_WPC, bsm, s>>>(
            pv.rec, pv.geo, tile_offsets, tile_prims, ck, sk, *fwd, *up, kg, det);
    {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int rgrid = std::min(sms * 4, (grid + 31) / 32);
        qgs::raster_bwd_replay_kernel<<<rgrid, qgs::RASTER_THREADS, qgs::bwd_smem_per_warp(), s>>>(
            pv.rec, pv.geo, tile_offsets, tile_prims, ck, sk, *fwd, *up, kg, det);
    }
    QGS_LAUNCHED("raster_bwd_kernel");
    return 0;
}

int backward_checks(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
                    const int32_t *tile_offsets, const qgs_targets *fwd, const qgs_upstream *up,
                    float *kg)
{
    if (!prep || !st || !fwd || !up || !tile_offsets || (!kg && P > 0))
        return fail(QGS_E_ARG, "NULL argument");
    if (P == 0) return 0;
    if (!fwd->aux) return fail(QGS_E_ARG, "backward needs the forward's aux planes");
    if (int rc = check_cam(cam)) return rc;
    return configure();
}
}  // namespace

int qgs_backward(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
                 const int32_t *tile_offsets, const int32_t *tile_prims, const qgs_targets *fwd,
                 const qgs_upstream *up, float *kg, qgs_stream_t stream)
{
    if (int rc = backward_checks(prep, P, cam, st, tile_offsets, fwd, up, kg)) return rc;
    if (P == 0) return 0;
    qgs::DetRows none{nullptr, nullptr, nullptr};
    return backward_impl(prep, P, cam, st, tile_offsets, tile_prims, fwd, up, kg, none,
                         reinterpret_cast<cudaStream_t>(stream));
}

size_t qgs_backward_det_workspace_bytes(int32_t P, int64_t n_frags, const qgs_camera *cam)
{
    if (!cam || P < 0 || n_frags < 0) return 0;
    const qgs::CamK ck = qgs::make_camk(*cam);
    return qgs::det_workspace_bytes(P, n_frags, ck.tiles_x * ck.tiles_y * qgs::RASTER_BLOCKS_PER_TILE);
}

int qgs_backward_deterministic(const void *prep, int32_t P, const qgs_camera *cam,
                               const qgs_settings *st, const int32_t *tile_offsets,
                               const int32_t *tile_prims, const qgs_targets *fwd,
                               const qgs_upstream *up, float *kg, int64_t n_frags,
                               void *workspace, size_t workspace_bytes, qgs_stream_t stream)
{
    if (int rc = backward_checks(prep, P, cam, st, tile_offsets, fwd, up, kg)) return rc;
    if (P == 0) return 0;
    if (!workspace || n_frags < 0 || n_frags > 0xffffffffLL)
        return fail(QGS_E_ARG, "deterministic backward: workspace / n_frags out of range");
    if (workspace_bytes < qgs_backward_det_workspace_bytes(P, n_frags, cam))
        return fail(QGS_E_CAPACITY, "deterministic backward workspace too small");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const qgs::CamK ck = qgs::make_camk(*cam);
    const int n_warps = ck.tiles_x * ck.tiles_y * qgs::RASTER_BLOCKS_PER_TILE;
    qgs::DetRows det;
    QGS_CK(qgs::det_prepare(ck, fwd->n_fragments, P, n_frags, workspace, workspace_bytes, det, s));
    if (int rc = backward_impl(prep, P, cam, st, tile_offsets, tile_prims, fwd, up, kg, det, s))
        return rc;
    QGS_CK(qgs::det_finish(P, n_frags, n_warps, workspace, kg, s));
    return 0;
}

int qgs_chain(const qgs_params *prims, const void *prep, const float *kg, const qgs_camera *cam,
              const qgs_grads *out, qgs_stream_t stream)
{
    (void)prep;
    if (!prims || !out) return fail(QGS_E_ARG, "NULL argument");
    if (int rc = check_cam(cam)) return rc;
    if (prims->P == 0) return 0;
    if (!kg) return fail(QGS_E_ARG, "NULL argument");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    qgs::CamK ck = qgs::make_camk(*cam);
    qgs::chain_kernel<<<cdiv(prims->P, 128), 128, 0, s>>>(*prims, ck, kg, *out);
    QGS_LAUNCHED("chain_kernel");
    return 0;
}

int qgs_trace_pixel(const void *prep, int32_t P, const qgs_camera *cam, const qgs_settings *st,
                    const int32_t *tile_offsets, const int32_t *tile_prims, int32_t u, int32_t v,
                    int32_t max, int32_t *acc_prim, float *acc_t, float *acc_abar,
                    int32_t *em_prim, float *em_t, float *em_abar, double *em_T,
                    int32_t *counts, qgs_stream_t stream)
{
    if (int rc = check_cam(cam)) return rc;
    if (u < 0 || v < 0 || u >= cam->width || v >= cam->height) return fail(QGS_E_ARG, "pixel outside image");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    qgs::CamK ck = qgs::make_camk(*cam);
    qgs::SetK sk = qgs::make_setk(*st);
    qgs::PrepView pv = qgs::prep_view(const_cast<void *>(prep), P);
    qgs::trace_pixel_kernel<<<1, 32, 0, s>>>(pv.rec, pv.geo, tile_offsets, tile_prims, ck, sk, u, v, max,
                                            acc_prim, acc_t, acc_abar, em_prim, em_t, em_abar,
                                            em_T, counts);
    QGS_LAUNCHED("trace_pixel_kernel");
    return 0;
}

int qgs_export_prep(const void *prep, int32_t P, double *scales, double *alphas, double *colors,
                    int32_t *pix_bbox, uint8_t *planar, qgs_stream_t stream)
{
    if (P == 0) return 0;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    qgs::PrepView pv = qgs::prep_view(const_cast<void *>(prep), P);
    qgs::export_prep_kernel<<<cdiv(P, 128), 128, 0, s>>>(pv, P, scales, alphas, colors, pix_bbox,
                                                        planar);
    QGS_LAUNCHED("export_prep_kernel");
    return 0;
}

int qgs_export_prep_geometry(const qgs_params *prims, const void *prep, const qgs_camera *cam,
                             const qgs_prep_export *out, qgs_stream_t stream)
{
    if (!prims || !prep || !out) return fail(QGS_E_ARG, "NULL argument");
    if (int rc = check_cam(cam)) return rc;
    if (prims->P == 0) return 0;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    qgs::PrepView pv = qgs::prep_view(const_cast<void *>(prep), prims->P);
    qgs::export_geom_kernel<<<cdiv(prims->P, 128), 128, 0, s>>>(*prims, qgs::make_camk(*cam), pv,
                                                               *out);
    QGS_LAUNCHED("export_geom_kernel");
    return 0;
}

int qgs_pixel_dirs(const qgs_camera *cam, double *dirs, qgs_stream_t stream)
{
    if (!dirs) return fail(QGS_E_ARG, "NULL argument");
    if (int rc = check_cam(cam)) return rc;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    qgs::CamK ck = qgs::make_camk(*cam);
    qgs::pixel_rays_kernel<<<cdiv((long long)ck.W * ck.H, 256), 256, 0, s>>>(ck, dirs);
    QGS_LAUNCHED("pixel_rays_kernel");
    return 0;
}

// ------------------------------------------------------------ losses

namespace {
int check_map(int32_t H, int32_t W)
{
    if (H <= 0 || W <= 0 || H > 32767 || W > 32767) return fail(QGS_E_ARG, "map size must be in [1, 32767]");
    return 0;
}
qgs::LossCam loss_cam(const qgs_camera &c)
{
    return qgs::LossCam{c.fx, c.fy, c.cx, c.cy, c.width, c.height};
}
}  // namespace

size_t qgs_loss_workspace_bytes(int32_t H, int32_t W, int32_t C)
{
    return qgs::loss_workspace_bytes(H, W, C);
}

int qgs_loss_photometric(const float *render, const float *gt, int32_t H, int32_t W, int32_t C,
                         double lambda_ssim, double weight, float *d_render, double *values,
                         void *workspace, size_t workspace_bytes, qgs_stream_t stream)
{
    if (int rc = check_map(H, W)) return rc;
    if (!render || !gt || !values || !workspace) return fail(QGS_E_ARG, "NULL argument");
    if (C < 1 || C > 4) return fail(QGS_E_ARG, "channels must be in [1, 4]");
    if (!(lambda_ssim >= 0.0 && lambda_ssim <= 1.0))
        return fail(QGS_E_ARG, "lambda_photo_ssim must lie in [0, 1]");
    if (lambda_ssim > 0.0 && (H < 11 || W < 11))
        return fail(QGS_E_ARG, "image smaller than the SSIM window");
    if (workspace_bytes < qgs::loss_workspace_bytes(H, W, C))
        return fail(QGS_E_CAPACITY, "loss workspace too small");
    cudaError_t e = qgs::photometric(render, gt, H, W, C, lambda_ssim, weight, d_render, values,
                                     workspace, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("qgs_loss_photometric", e);
    return 0;
}

int qgs_loss_distortion(const float *distortion, int32_t H, int32_t W, double weight,
                        float *d_dist, double *values, void *workspace, size_t workspace_bytes,
                        qgs_stream_t stream)
{
    if (int rc = check_map(H, W)) return rc;
    if (!distortion || !values || !workspace) return fail(QGS_E_ARG, "NULL argument");
    if (workspace_bytes < qgs::loss_workspace_bytes(H, W, 1))
        return fail(QGS_E_CAPACITY, "loss workspace too small");
    cudaError_t e = qgs::distortion(distortion, H, W, weight, d_dist, values, workspace,
                                    reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("qgs_loss_distortion", e);
    return 0;
}

int qgs_depth_to_normal(const float *depth, const float *alpha, const qgs_camera *cam,
                        double alpha_thresh, float *N, uint8_t *mask, qgs_stream_t stream)
{
    if (int rc = check_cam(cam)) return rc;
    if (!depth || !alpha || !N || !mask) return fail(QGS_E_ARG, "NULL argument");
    cudaError_t e = qgs::depth_to_normal(depth, alpha, loss_cam(*cam), alpha_thresh, N, mask,
                                         reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("qgs_depth_to_normal", e);
    return 0;
}

int qgs_loss_normal_consistency(const float *alpha, const float *normal, const float *curvature,
                                const float *depth, const float *N, const uint8_t *mask,
                                const qgs_camera *cam, double alpha_thresh, double eps_curvature,
                                int32_t guided, double weight, float *d_alpha, float *d_normal,
                                float *d_curvature, double *values, void *workspace,
                                size_t workspace_bytes, qgs_stream_t stream)
{
    if (int rc = check_cam(cam)) return rc;
    if (!alpha || !normal || !values || !workspace) return fail(QGS_E_ARG, "NULL argument");
    if (guided && !curvature) return fail(QGS_E_ARG, "guided consistency needs the curvature map");
    if (!depth && (!N || !mask)) return fail(QGS_E_ARG, "need depth, or N and mask");
    if (workspace_bytes < qgs::loss_workspace_bytes(cam->height, cam->width, 1))
        return fail(QGS_E_CAPACITY, "loss workspace too small");
    cudaError_t e = qgs::normal_consistency(alpha, normal, curvature, depth, N, mask,
                                            loss_cam(*cam), alpha_thresh, eps_curvature, guided,
                                            weight, d_alpha, d_normal, guided ? d_curvature : nullptr,
                                            values, workspace,
                                            reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("qgs_loss_normal_consistency", e);
    return 0;
}

// ---------------------------------------------------- optimizer / densify

namespace {
void group_ptrs(const qgs_groups &g, float *out[6])
{
    out[0] = g.centers; out[1] = g.quats; out[2] = g.raw_scales;
    out[3] = g.raw_signs; out[4] = g.raw_opacity; out[5] = g.sh;
}
void group_ptrs_ro(const qgs_params &g, const float *out[6])
{
    out[0] = g.centers; out[1] = g.quats; out[2] = g.raw_scales;
    out[3] = g.raw_signs; out[4] = g.raw_opacity; out[5] = g.sh;
}
void group_widths(int sh_coeffs, int w[6])
{
    w[0] = 3; w[1] = 4; w[2] = 3; w[3] = 3; w[4] = 1; w[5] = 3 * sh_coeffs;
}
bool sh_ok(int k) { return k == 1 || k == 4 || k == 9 || k == 16; }
}  // namespace

int qgs_adam_step(const qgs_groups *prims, const qgs_grads *grads, const qgs_groups *m,
                  const qgs_groups *v, const qgs_adam_config *cfg,
                  const qgs_densify_stats *stats, uint64_t *d_skipped, qgs_stream_t stream)
{
    if (!prims || !grads || !m || !v || !cfg || !d_skipped) return fail(QGS_E_ARG, "NULL argument");
    if (prims->P < 0 || !sh_ok(prims->sh_coeffs)) return fail(QGS_E_ARG, "bad parameter set");
    if (m->P != prims->P || v->P != prims->P || m->sh_coeffs != prims->sh_coeffs ||
        v->sh_coeffs != prims->sh_coeffs)
        return fail(QGS_E_ARG, "Adam state does not match the parameters");
    if (cfg->t < 1) return fail(QGS_E_ARG, "step number must be >= 1");
    qgs::AdamArgs a{};
    group_ptrs(*prims, a.p);
    group_ptrs(*m, a.m);
    group_ptrs(*v, a.v);
    const float *g[6] = {grads->centers, grads->quats, grads->raw_scales, grads->raw_signs,
                         grads->raw_opacity, grads->sh};
    for (int k = 0; k < 6; ++k) {
        a.g[k] = g[k];
        a.freeze[k] = cfg->freeze[k];
        a.lr[k] = cfg->lr[k];
        if (!a.p[k] || !a.m[k] || !a.v[k] || !a.g[k]) return fail(QGS_E_ARG, "NULL group");
    }
    group_widths(prims->sh_coeffs, a.w);
    a.b1 = cfg->beta1;
    a.b2 = cfg->beta2;
    a.b1c = 1.0 - pow(cfg->beta1, (double)cfg->t);   // optim.py:26-27
    a.b2c = 1.0 - pow(cfg->beta2, (double)cfg->t);
    a.eps = cfg->eps;
    if (stats) {
        if (!stats->grad_accum || !stats->grad_count || !stats->center_accum || !grads->screen_center)
            return fail(QGS_E_ARG, "statistics need every buffer and the screen-centre gradient");
        a.g_screen = grads->screen_center;
        a.grad_accum = stats->grad_accum;
        a.grad_count = stats->grad_count;
        a.center_accum = stats->center_accum;
    }
    a.skipped = reinterpret_cast<unsigned long long *>(d_skipped);
    a.P = prims->P;
    cudaError_t e = qgs::adam_step(a, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("qgs_adam_step", e);
    return 0;
}

size_t qgs_densify_workspace_bytes(int32_t P) { return qgs::densify_workspace_bytes(P < 0 ? 0 : P); }

int qgs_densify_plan(const qgs_params *prims, const qgs_densify_stats *stats,
                     const qgs_densify_config *cfg, void *workspace, size_t workspace_bytes,
                     int64_t *d_counts, qgs_stream_t stream)
{
    if (!prims || !stats || !cfg || !workspace || !d_counts) return fail(QGS_E_ARG, "NULL argument");
    if (prims->P < 0) return fail(QGS_E_ARG, "P < 0");
    if (workspace_bytes < qgs::densify_workspace_bytes(prims->P))
        return fail(QGS_E_CAPACITY, "densify workspace too small");
    qgs::DensifyArgs a{};
    a.raw_scales = prims->raw_scales;
    a.raw_signs = prims->raw_signs;
    a.raw_opacity = prims->raw_opacity;
    a.grad_accum = stats->grad_accum;
    a.grad_count = stats->grad_count;
    a.grad_threshold = cfg->grad_threshold;
    a.big_threshold = cfg->percent_dense * cfg->scene_extent;
    a.prune_opacity = cfg->prune_opacity;
    a.room = (long long)cfg->max_primitives - prims->P;
    a.P = prims->P;
    cudaError_t e = qgs::densify_plan(a, workspace, d_counts, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("qgs_densify_plan", e);
    return 0;
}

int qgs_densify_apply(const qgs_params *prims, const qgs_params *m, const qgs_params *v,
                      const qgs_densify_stats *stats, const qgs_densify_config *cfg,
                      const void *workspace, const qgs_groups *out, const qgs_groups *out_m,
                      const qgs_groups *out_v, qgs_stream_t stream)
{
    if (!prims || !m || !v || !stats || !cfg || !workspace || !out || !out_m || !out_v)
        return fail(QGS_E_ARG, "NULL argument");
    if (!sh_ok(prims->sh_coeffs) || out->sh_coeffs != prims->sh_coeffs)
        return fail(QGS_E_ARG, "sh_coeffs mismatch");
    qgs::ApplyArgs a{};
    group_ptrs_ro(*prims, a.src);
    group_ptrs_ro(*m, a.m_src);
    group_ptrs_ro(*v, a.v_src);
    group_ptrs(*out, a.dst);
    group_ptrs(*out_m, a.m_dst);
    group_ptrs(*out_v, a.v_dst);
    group_widths(prims->sh_coeffs, a.w);
    a.center_accum = stats->center_accum;
    a.clone_nudge = cfg->clone_nudge;
    a.P = prims->P;
    cudaError_t e = qgs::densify_apply(a, workspace, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("qgs_densify_apply", e);
    return 0;
}

int qgs_reset_opacity(const qgs_groups *prims, const qgs_groups *m, const qgs_groups *v,
                      double cap, qgs_stream_t stream)
{
    if (!prims || !m || !v) return fail(QGS_E_ARG, "NULL argument");
    cudaError_t e = qgs::reset_opacity(prims->raw_opacity, m->raw_opacity, v->raw_opacity,
                                       prims->P, cap, reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("qgs_reset_opacity", e);
    return 0;
}

// ------------------------------------------------------------ multiview

namespace {
// multiview.py:31-47 intrinsics and the relative transform X_b = R X_a + T
void mv_intrinsics(const qgs_camera &c, double K[9], double Kinv[9])
{
    const double k[9] = {c.fx, 0.0, c.cx, 0.0, c.fy, c.cy, 0.0, 0.0, 1.0};
    const double ki[9] = {1.0 / c.fx, 0.0, -c.cx / c.fx, 0.0, 1.0 / c.fy, -c.cy / c.fy, 0.0, 0.0, 1.0};
    for (int i = 0; i < 9; ++i) { K[i] = k[i]; Kinv[i] = ki[i]; }
}
void mv_relative(const qgs_camera &a, const qgs_camera &b, double R[9], double T[3])
{
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += b.R_wc[3 * i + k] * a.R_wc[3 * j + k];
            R[3 * i + j] = s;
        }
    for (int i = 0; i < 3; ++i)
        T[i] = b.t_wc[i] - (R[3 * i] * a.t_wc[0] + R[3 * i + 1] * a.t_wc[1] + R[3 * i + 2] * a.t_wc[2]);
}
}  // namespace

size_t qgs_multiview_workspace_bytes(int32_t H, int32_t W, int32_t Hn, int32_t Wn)
{
    return qgs::multiview_workspace_bytes(H, W, Hn, Wn);
}

int qgs_multiview_loss(const qgs_mv_maps *ref, const qgs_camera *cam_ref, const qgs_mv_maps *nbr,
                       const qgs_camera *cam_nbr, const qgs_mv_config *cfg, double weight,
                       const qgs_mv_grads *up_ref, const qgs_mv_grads *up_nbr, double *values,
                       void *workspace, size_t workspace_bytes, qgs_stream_t stream)
{
    if (!ref || !nbr || !cfg || !values || !workspace) return fail(QGS_E_ARG, "NULL argument");
    if (int rc = check_cam(cam_ref)) return rc;
    if (int rc = check_cam(cam_nbr)) return rc;
    const qgs_mv_maps *mm[2] = {ref, nbr};
    for (const qgs_mv_maps *m : mm) {
        if (!m->depth || !m->alpha || !m->normal || !m->image) return fail(QGS_E_ARG, "NULL map");
        if (m->height < 2 || m->width < 2) return fail(QGS_E_ARG, "maps must be at least 2x2");
        if (m->image_channels < 1 || m->image_channels > 4) return fail(QGS_E_ARG, "image channels in [1, 4]");
        if ((long long)m->height * m->width * 4 >= (1LL << 31)) return fail(QGS_E_ARG, "maps too large");
    }
    if (cfg->patch_size < 1 || cfg->patch_size % 2 == 0 || cfg->patch_size > qgs::multiview_max_patch())
        return fail(QGS_E_ARG, "patch_size must be odd and <= 13");
    if (workspace_bytes < qgs::multiview_workspace_bytes(ref->height, ref->width, nbr->height, nbr->width))
        return fail(QGS_E_CAPACITY, "multiview workspace too small");
    qgs::MvArgs a{};
    a.D_r = ref->depth; a.A_r = ref->alpha; a.N_r = ref->normal; a.I_r = ref->image;
    a.D_n = nbr->depth; a.A_n = nbr->alpha; a.N_n = nbr->normal; a.I_n = nbr->image;
    a.Cr = ref->image_channels; a.Cn = nbr->image_channels;
    a.H = ref->height; a.W = ref->width; a.Hn = nbr->height; a.Wn = nbr->width;
    a.fx_r = cam_ref->fx; a.fy_r = cam_ref->fy; a.cx_r = cam_ref->cx; a.cy_r = cam_ref->cy;
    a.fx_n = cam_nbr->fx; a.fy_n = cam_nbr->fy; a.cx_n = cam_nbr->cx; a.cy_n = cam_nbr->cy;
    mv_intrinsics(*cam_ref, a.K_r, a.K_r_inv);
    mv_intrinsics(*cam_nbr, a.K_n, a.K_n_inv);
    mv_relative(*cam_ref, *cam_nbr, a.R_rn, a.T_rn);
    mv_relative(*cam_nbr, *cam_ref, a.R_nr, a.T_nr);
    a.r = cfg->patch_size / 2;
    a.alpha_thresh = cfg->alpha_thresh;
    a.min_denom = cfg->min_denom;
    a.ncc_eps = cfg->ncc_eps;
    a.full_chain = cfg->full_chain;
    cudaError_t e = qgs::multiview(
        a, weight, up_ref ? up_ref->depth : nullptr, up_ref ? up_ref->alpha : nullptr,
        up_ref ? up_ref->normal : nullptr, up_nbr ? up_nbr->depth : nullptr,
        up_nbr ? up_nbr->alpha : nullptr, up_nbr ? up_nbr->normal : nullptr, values, workspace,
        reinterpret_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail("qgs_multiview_loss", e);
    return 0;
}

}  // extern "C"
