// K2-K4: tile binning, float64 sort keys and the per-tile (key, id) sort.
//
// Reference: rasterizer.py:150-181 (pair expansion, tile_sort_depths,
// np.lexsort((prim, key, tile)), bincount/cumsum) and raster_kernels.py:684-716.
//
// Pipeline (all stream-ordered, one host read of the pair count before it):
//   tile_diff_kernel    4 atomics per primitive into a 2D difference grid
//   tile_offsets_kernel 2D prefix sum -> per-tile counts -> tile_offsets
//   pair_key_kernel     one thread per (tile, primitive) pair: fp64 key
//                       (bit-identical to tile_sort_depths), composite
//                       (f32_rd(key) << 32 | prim) scattered into its tile
//                       bucket through a per-tile cursor
//   tile_sort_kernel    one CTA per tile: stable LSD radix sort of the bucket
//                       on the f32 key bits that vary inside the tile, then
//                       exact fix-up of equal-f32 runs by (fp64 key, prim id)
// The result equals lexsort((prim, key, tile)) exactly: within a tile the
// order is (key ascending, prim ascending), a total order.
//
// Compiled with -fmad=false (keys must round exactly as the reference).
#include "qgs_common.cuh"

namespace qgs {

// ------------------------------------------------------------- scan utils

constexpr int SCAN_T = 1024;

template <typename T>
__device__ T block_exclusive_scan(T v, T *s_warp, T &total)
{
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    T x = v;
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        T w = lane < nw ? s_warp[lane] : T(0);
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) s_warp[lane] = w;
    }
    __syncthreads();
    T base = wid > 0 ? s_warp[wid - 1] : T(0);
    total = s_warp[nw - 1];
    __syncthreads();
    return base + x - v;
}

// per-block sums of ntiles
__global__ void scan_sums_kernel(const int32_t *__restrict__ in, int n, int64_t *sums)
{
    __shared__ int64_t s_w[32];
    int64_t acc = 0;
    int base = blockIdx.x * SCAN_T * 4;
    for (int k = 0; k < 4; ++k) {
        int i = base + k * SCAN_T + threadIdx.x;
        if (i < n) acc += in[i];
    }
    int64_t tot;
    block_exclusive_scan<int64_t>(acc, s_w, tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// exclusive scan of the block sums (single block, any length)
__global__ void scan_top_kernel(int64_t *sums, int nb, int64_t *d_total, int64_t *out, int n)
{
    __shared__ int64_t s_w[32];
    int64_t carry = 0;
    for (int b0 = 0; b0 < nb; b0 += SCAN_T) {
        int i = b0 + threadIdx.x;
        int64_t v = i < nb ? sums[i] : 0;
        int64_t tot;
        int64_t ex = block_exclusive_scan<int64_t>(v, s_w, tot);
        if (i < nb) sums[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) { *d_total = carry; out[n] = carry; }
}

__global__ void scan_out_kernel(const int32_t *__restrict__ in, int n, const int64_t *sums,
                                int64_t *out)
{
    __shared__ int64_t s_w[32];
    int base = blockIdx.x * SCAN_T * 4;
    int i0 = base + threadIdx.x * 4;
    int32_t v[4];
    int64_t acc = 0;
    for (int k = 0; k < 4; ++k) { v[k] = (i0 + k < n) ? in[i0 + k] : 0; acc += v[k]; }
    int64_t tot;
    int64_t ex = block_exclusive_scan<int64_t>(acc, s_w, tot) + sums[blockIdx.x];
    for (int k = 0; k < 4; ++k) {
        if (i0 + k < n) out[i0 + k] = ex;
        ex += v[k];
    }
}

// ------------------------------------------------------- tile offsets

__global__ void tile_diff_kernel(const int4 *__restrict__ bbox, int P, int tiles_x, int *diff)
{
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    int4 b = bbox[p];
    if (b.x > b.y) return;
    int tx0 = b.x / TILE, tx1 = b.y / TILE, ty0 = b.z / TILE, ty1 = b.w / TILE;
    int stride = tiles_x + 1;
    atomicAdd(&diff[ty0 * stride + tx0], 1);
    atomicAdd(&diff[ty0 * stride + tx1 + 1], -1);
    atomicAdd(&diff[(ty1 + 1) * stride + tx0], -1);
    atomicAdd(&diff[(ty1 + 1) * stride + tx1 + 1], 1);
}

// single block: integrate the difference grid, write tile_offsets and cursors
__global__ void tile_offsets_kernel(int *diff, int tiles_x, int tiles_y, int32_t *tile_offsets,
                                    int32_t *cursor)
{
    __shared__ int s_w[32];
    int stride = tiles_x + 1;
    // prefix along x for each row, then along y for each column
    for (int ty = threadIdx.x; ty < tiles_y; ty += blockDim.x) {
        int run = 0;
        for (int tx = 0; tx < tiles_x; ++tx) { run += diff[ty * stride + tx]; diff[ty * stride + tx] = run; }
    }
    __syncthreads();
    for (int tx = threadIdx.x; tx < tiles_x; tx += blockDim.x) {
        int run = 0;
        for (int ty = 0; ty < tiles_y; ++ty) { run += diff[ty * stride + tx]; diff[ty * stride + tx] = run; }
    }
    __syncthreads();
    int n = tiles_x * tiles_y;
    int carry = 0;
    for (int t0 = 0; t0 < n; t0 += blockDim.x) {
        int t = t0 + threadIdx.x;
        int c = 0;
        if (t < n) { int ty = t / tiles_x, tx = t - ty * tiles_x; c = diff[ty * stride + tx]; }
        int tot;
        int ex = block_exclusive_scan<int>(c, s_w, tot);
        if (t < n) { tile_offsets[t] = carry + ex; cursor[t] = carry + ex; }
        carry += tot;
    }
    if (threadIdx.x == 0) tile_offsets[n] = carry;
}

// ------------------------------------------------------------- pair keys

__device__ inline uint32_t key_hi(double key)
{
    return __float_as_uint(__double2float_rd(key));
}

// One warp per primitive; lanes stride over the primitive's tiles.
__global__ void pair_key_kernel(PrepView pv, int P, int64_t n_pairs, CamK cam, SetK st,
                                int32_t *cursor, uint64_t *bucket)
{
    (void)n_pairs;
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < P; p += warps) {
        const int nt = pv.ntiles[p];
        if (nt == 0) continue;
        const int4 b = pv.bbox[p];
        const int tx0 = b.x / TILE, ty0 = b.z / TILE;
        const int ncols = b.y / TILE - tx0 + 1;
        const Geo64 &g = pv.geo[p];
        for (int local = lane; local < nt; local += 32) {
            const int row = local / ncols;
            const int tile = (ty0 + row) * cam.tiles_x + tx0 + (local - row * ncols);
            const double key = tile_key_geo(g, tile, cam, st.euclid != 0, st.t_clip);
            const int slot = atomicAdd(&cursor[tile], 1);
            bucket[slot] = ((uint64_t)key_hi(key) << 32) | (uint32_t)p;
        }
    }
}

// ------------------------------------------------------- per-tile sort

constexpr int SORT_T = 512;
constexpr int SORT_IPT = 16;
constexpr int SORT_W = SORT_T / 32;
constexpr int CHUNK = SORT_T * SORT_IPT;

struct SortSmem {
    uint64_t buf[CHUNK];             // single-chunk segments live here
    int warp_cnt[SORT_W][256];       // per-warp digit counts -> prefixes
    int base[256];                   // running output base per digit
    int hist[256];
    int scan_w[32];
    uint32_t kmin, kmax;
    int flag;
};

__device__ inline int warp_striped_index(int k)
{
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    return w * (32 * SORT_IPT) + k * 32 + lane;
}

// Stable rank of one chunk (items warp-striped), digits in [0,256), 256 =
// invalid.  On return, rank[k] = base[d] + (#items of digit d before it in
// this chunk); then base[d] advances by the chunk's digit counts.
__device__ void chunk_rank(SortSmem &sm, const int (&dig)[SORT_IPT], int (&rank)[SORT_IPT])
{
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned lt = (1u << lane) - 1u;
    for (int d = lane; d < 256; d += 32) sm.warp_cnt[w][d] = 0;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < SORT_IPT; ++k) {
        int d = dig[k];
        unsigned peers = __match_any_sync(0xffffffffu, d);
        int before = d < 256 ? sm.warp_cnt[w][d] : 0;
        rank[k] = before + __popc(peers & lt);
        __syncwarp();
        if (d < 256 && (peers & lt) == 0) sm.warp_cnt[w][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per-digit prefix over warps; warp prefix + running base
    for (int d = threadIdx.x; d < 256; d += SORT_T) {
        int run = sm.base[d];
        for (int ww = 0; ww < SORT_W; ++ww) {
            int c = sm.warp_cnt[ww][d];
            sm.warp_cnt[ww][d] = run;
            run += c;
        }
        sm.base[d] = run;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SORT_IPT; ++k)
        if (dig[k] < 256) rank[k] += sm.warp_cnt[w][dig[k]];
    __syncthreads();
}

__device__ void digit_base_from_hist(SortSmem &sm)
{
    __syncthreads();
    int v = threadIdx.x < 256 ? sm.hist[threadIdx.x] : 0;
    int tot;
    int ex = block_exclusive_scan<int>(v, sm.scan_w, tot);
    if (threadIdx.x < 256) sm.base[threadIdx.x] = ex;
    __syncthreads();
}

// (fp64 key, prim) ordering for an equal-f32 run, insertion sort (stable)
__device__ void fix_run(uint64_t *a, int len, int tile, const PrepView &pv, const CamK &cam,
                        const SetK &st)
{
    double kk[64];
    if (len > 64) {
        // long run of identical f32 keys (degenerate input): sort without caching
        for (int i = 1; i < len; ++i) {
            uint64_t x = a[i];
            double kx = tile_key_geo(pv.geo[(uint32_t)x], tile, cam, st.euclid != 0, st.t_clip);
            int j = i - 1;
            while (j >= 0) {
                uint32_t pj = (uint32_t)a[j];
                double kj = tile_key_geo(pv.geo[pj], tile, cam, st.euclid != 0, st.t_clip);
                if (kj > kx || (kj == kx && pj > (uint32_t)x)) { a[j + 1] = a[j]; --j; }
                else break;
            }
            a[j + 1] = x;
        }
        return;
    }
    for (int i = 0; i < len; ++i)
        kk[i] = tile_key_geo(pv.geo[(uint32_t)a[i]], tile, cam, st.euclid != 0, st.t_clip);
    for (int i = 1; i < len; ++i) {
        uint64_t x = a[i];
        double kx = kk[i];
        int j = i - 1;
        while (j >= 0 && (kk[j] > kx || (kk[j] == kx && (uint32_t)a[j] > (uint32_t)x))) {
            a[j + 1] = a[j]; kk[j + 1] = kk[j]; --j;
        }
        a[j + 1] = x; kk[j + 1] = kx;
    }
}

__device__ void fixup_and_emit(uint64_t *a, int n, int tile, const PrepView &pv, const CamK &cam,
                               const SetK &st, int32_t *out)
{
    for (int i = threadIdx.x; i < n; i += SORT_T) {
        uint32_t h = (uint32_t)(a[i] >> 32);
        bool head = (i == 0 || (uint32_t)(a[i - 1] >> 32) != h) && i + 1 < n &&
                    (uint32_t)(a[i + 1] >> 32) == h;
        if (head) {
            int j = i + 1;
            while (j < n && (uint32_t)(a[j] >> 32) == h) ++j;
            fix_run(a + i, j - i, tile, pv, cam, st);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += SORT_T) out[i] = (int32_t)(uint32_t)a[i];
}

__global__ void __launch_bounds__(SORT_T)
tile_sort_kernel(const int32_t *__restrict__ tile_offsets, uint64_t *keys, uint64_t *tmp,
                 PrepView pv, CamK cam, SetK st, int32_t *tile_prims)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem &sm = *reinterpret_cast<SortSmem *>(smem_raw);
    int tile = blockIdx.x;
    int start = tile_offsets[tile], n = tile_offsets[tile + 1] - start;
    if (n == 0) return;
    if (n == 1) {
        if (threadIdx.x == 0) tile_prims[start] = (int32_t)(uint32_t)keys[start];
        return;
    }
    uint64_t *src = keys + start, *dst = tmp + start;
    bool single = n <= CHUNK;
    // key range -> bits to sort
    if (threadIdx.x == 0) { sm.kmin = 0xffffffffu; sm.kmax = 0u; }
    __syncthreads();
    uint32_t lmin = 0xffffffffu, lmax = 0;
    for (int i = threadIdx.x; i < n; i += SORT_T) {
        uint64_t v = src[i];
        if (single) sm.buf[i] = v;
        uint32_t h = (uint32_t)(v >> 32);
        lmin = min(lmin, h); lmax = max(lmax, h);
    }
    atomicMin(&sm.kmin, lmin);
    atomicMax(&sm.kmax, lmax);
    __syncthreads();
    uint32_t diff = sm.kmin ^ sm.kmax;
    int bits = diff ? 32 - __clz(diff) : 0;

    for (int shift = 0; shift < bits; shift += 8) {
        // segment digit histogram -> base offsets
        for (int d = threadIdx.x; d < 256; d += SORT_T) sm.hist[d] = 0;
        __syncthreads();
        const uint64_t *in = single ? sm.buf : src;
        for (int i = threadIdx.x; i < n; i += SORT_T)
            atomicAdd(&sm.hist[(uint32_t)(in[i] >> (32 + shift)) & 0xffu], 1);
        digit_base_from_hist(sm);
        for (int c0 = 0; c0 < n; c0 += CHUNK) {
            uint64_t it[SORT_IPT];
            int dig[SORT_IPT], rank[SORT_IPT];
#pragma unroll
            for (int k = 0; k < SORT_IPT; ++k) {
                int idx = c0 + warp_striped_index(k);
                bool ok = idx < n;
                it[k] = ok ? in[idx] : 0ull;
                dig[k] = ok ? (int)((uint32_t)(it[k] >> (32 + shift)) & 0xffu) : 256;
            }
            chunk_rank(sm, dig, rank);   // ends with __syncthreads: all reads done
            uint64_t *out = single ? sm.buf : dst;
#pragma unroll
            for (int k = 0; k < SORT_IPT; ++k)
                if (dig[k] < 256) out[rank[k]] = it[k];
            __syncthreads();
        }
        if (!single) { uint64_t *t = src; src = dst; dst = t; }
    }
    if (single) {
        fixup_and_emit(sm.buf, n, tile, pv, cam, st, tile_prims + start);
    } else {
        __syncthreads();
        fixup_and_emit(src, n, tile, pv, cam, st, tile_prims + start);
    }
}

// -------------------------------------------------------- debug / unit

__global__ void sorted_keys_kernel(PrepView pv, const int32_t *tile_offsets,
                                   const int32_t *tile_prims, int n_tiles, CamK cam, SetK st,
                                   double *keys)
{
    int tile = blockIdx.x;
    if (tile >= n_tiles) return;
    for (int i = tile_offsets[tile] + threadIdx.x; i < tile_offsets[tile + 1]; i += blockDim.x)
        keys[i] = tile_key_geo(pv.geo[tile_prims[i]], tile, cam, st.euclid != 0, st.t_clip);
}

__global__ void tile_keys_f64_kernel(int64_t n, const int64_t *pair_tiles,
                                     const int64_t *pair_prims, const double *ohat,
                                     const double *M, const double *wv, const double *sv,
                                     const uint8_t *planar, const double *vu, const double *vv,
                                     const double *dist, CamK cam, SetK st, double *keys)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = pair_prims[i];
        keys[i] = tile_key64(ohat + 3 * p, M + 9 * p, wv + 3 * p, sv + 3 * p, planar[p] == 1,
                             vu[p], vv[p], dist[p], (int)pair_tiles[i], cam, st.euclid != 0,
                             st.t_clip);
    }
}

size_t sort_smem_bytes() { return sizeof(SortSmem); }

}  // namespace qgs
