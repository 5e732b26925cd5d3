// Kernel declarations shared between the translation units and abi.cu.
#pragma once
#include "qgs_common.cuh"

namespace qgs {

// preprocess.cu
__global__ void preprocess_kernel(qgs_params prm, CamK cam, PrepView pv, int euclid, int with_color);
__global__ void color_kernel(qgs_params prm, CamK cam, PrepView pv);
__global__ void chain_kernel(qgs_params prm, CamK cam, const float *kg, qgs_grads out);
__global__ void export_prep_kernel(PrepView pv, int P, double *scales, double *alphas,
                                   double *colors, int32_t *bbox, uint8_t *planar);

// binning.cu
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = SCAN_THREADS * 4;
__global__ void scan_sums_kernel(const int32_t *in, int n, int64_t *sums);
__global__ void scan_top_kernel(int64_t *sums, int nb, int64_t *d_total, int64_t *out, int n,
                                const int32_t *nonfinite = nullptr);
__global__ void scan_out_kernel(const int32_t *in, int n, const int64_t *sums, int64_t *out);
__global__ void tile_diff_kernel(const int4 *bbox, int P, int tiles_x, int *diff);
__global__ void tile_offsets_kernel(int *diff, int tiles_x, int tiles_y, int32_t *tile_offsets,
                                    int32_t *cursor);
__global__ void pixel_rays_kernel(CamK cam, double *rays);
__global__ void export_geom_kernel(qgs_params prm, CamK cam, PrepView pv, qgs_prep_export o);
__global__ void pair_key_kernel(PrepView pv, int P, int64_t n_pairs, CamK cam, SetK st,
                                const double *rays, int32_t *cursor, uint64_t *bucket);
// tiles over SORT_HUGE entries: stage 1 (tile_sort_kernel) buckets them and
// records the buckets here; stage 2 (tile_sort_chunks_kernel) sorts the
// buckets with sort_chunks() CTAs per tile
constexpr int SORT_MAX_BUCKETS = 8192;
constexpr int SORT_MAX_HUGE = 512;
struct HugeTile {
    int tile, nb, shift, ns;          // ns: splitters (sample-sort buckets), -1: linear buckets
    uint32_t kmin, range;
    float dmin, dscale;               // linear buckets (BucketFn)
};
struct HugeSort {
    int count;
    int pad[7];
    HugeTile t[SORT_MAX_HUGE];
    __device__ int *bend_of(int h)    // bucket ends (+ splitters), SORT_MAX_BUCKETS ints per tile
    {
        return reinterpret_cast<int *>(this + 1) + (size_t)h * SORT_MAX_BUCKETS;
    }
};
__global__ void tile_sort_kernel(const int32_t *tile_offsets, uint64_t *keys, uint64_t *tmp,
                                 PrepView pv, CamK cam, SetK st, int32_t *tile_prims,
                                 const int32_t *order, HugeSort *huge);
__global__ void tile_sort_chunks_kernel(const int32_t *tile_offsets, const uint64_t *tmp,
                                        PrepView pv, CamK cam, SetK st, int32_t *tile_prims,
                                        const HugeSort *huge);
int sort_chunks();
size_t huge_sort_bytes();
__global__ void sorted_keys_kernel(PrepView pv, const int32_t *tile_offsets,
                                   const int32_t *tile_prims, int n_tiles, CamK cam, SetK st,
                                   double *keys);
__global__ void tile_keys_f64_kernel(int64_t n, const int64_t *pair_tiles,
                                     const int64_t *pair_prims, const double *ohat,
                                     const double *M, const double *wv, const double *sv,
                                     const uint8_t *planar, const double *vu, const double *vv,
                                     const double *dist, CamK cam, SetK st, double *keys);
size_t sort_smem_bytes();
int sort_threads();                 // binning.cu SORT_T

// det_reduce.cu (RenderSettings.deterministic): fragment (pixel, k) of the
// backward writes its kernel-gradient slots to row base[warp * 32 + lane] + k
struct DetRows {
    const int64_t *base;   // per raster-warp lane
    float *rows;           // [rows][KG]
    int32_t *prim;         // [rows]
};
size_t det_workspace_bytes(int P, int64_t n_frags, int n_warps);
cudaError_t det_prepare(const CamK &cam, const int32_t *n_frag, int P, int64_t n_frags, void *ws,
                        size_t ws_bytes, DetRows &out, cudaStream_t s);
cudaError_t det_finish(int P, int64_t n_frags, int n_warps, void *ws, float *kg, cudaStream_t s);

// raster.cu
__global__ void raster_fwd_kernel(const PrimRec *recs, const Geo64 *geo, const ConicRec *conics,
                                  const int32_t *tile_offsets,
                                  const int32_t *tile_prims, CamK cam, SetK st, qgs_targets out);
__global__ void raster_fwd_exact_kernel(const PrimRec *recs, const Geo64 *geo,
                                        const ConicRec *conics, const int32_t *tile_offsets,
                                        const int32_t *tile_prims, CamK cam, SetK st,
                                        qgs_targets out);
__global__ void raster_bwd_replay_kernel(const PrimRec *recs, const Geo64 *geo,
                                         const int32_t *tile_offsets, const int32_t *tile_prims,
                                         CamK cam, SetK st, qgs_targets fwd, qgs_upstream upst,
                                         float *kg, DetRows det);
__global__ void raster_bwd_kernel(const PrimRec *recs, const Geo64 *geo, const int32_t *tile_offsets,
                                  const int32_t *tile_prims, CamK cam, SetK st, qgs_targets fwd,
                                  qgs_upstream upst, float *kg, DetRows det);
__global__ void raster_bwd_det_kernel(const PrimRec *recs, const Geo64 *geo,
                                      const int32_t *tile_offsets, const int32_t *tile_prims,
                                      CamK cam, SetK st, qgs_targets fwd, qgs_upstream upst,
                                      float *kg, DetRows det);
__global__ void trace_pixel_kernel(const PrimRec *recs, const Geo64 *geo, const int32_t *tile_offsets,
                                   const int32_t *tile_prims, CamK cam, SetK st, int u, int v,
                                   int max, int *acc_prim, float *acc_t, float *acc_abar,
                                   int *em_prim, float *em_t, float *em_abar, double *em_T,
                                   int *counts);
__global__ void tile_order_kernel(const int32_t *tile_offsets, int n_tiles, int32_t *order,
                                  int heavy_only);
constexpr int ORDER_SMEM = 0;      // static shared memory only
constexpr int RASTER_THREADS = 32;   // one warp per 8x4 block, 8 blocks per tile
constexpr int RASTER_BLOCKS_PER_TILE = 8;
// raster warps per CTA (independent warps; a CTA of several puts a tile's
// blocks on one SM, where they share the L1 for the tile's list and records)
#ifndef QGS_FWD_WPC
#define QGS_FWD_WPC 8     // a tile per CTA: C3 forward 10.6 -> 10.0 ms (1, 2, 8 measured)
#endif
#ifndef QGS_BWD_WPC
#define QGS_BWD_WPC 4     // C3 backward 5.89 -> 5.80 ms (1, 4 measured)
#endif
constexpr int FWD_WPC = QGS_FWD_WPC;
constexpr int BWD_WPC = QGS_BWD_WPC;
size_t fwd_smem_per_warp();
int diag_counters(unsigned long long *out, int n);
size_t bwd_smem_per_warp();

}  // namespace qgs
