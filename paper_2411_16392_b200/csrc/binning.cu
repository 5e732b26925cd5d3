// K2-K4: tile binning, float64 sort keys and the per-tile (key, id) sort.
//
// Reference: rasterizer.py:150-181 (pair expansion, tile_sort_depths,
// np.lexsort((prim, key, tile)), bincount/cumsum) and raster_kernels.py:684-716.
//
// Pipeline (all stream-ordered, one host read of the pair count before it):
//   tile_diff_kernel    4 atomics per primitive into a 2D difference grid
//   tile_offsets_kernel 2D prefix sum -> per-tile counts -> tile_offsets
//   pair_key_kernel     a warp per primitive, a lane per (tile, primitive)
//                       pair: fp64 key (bit-identical to tile_sort_depths),
//                       composite (fp64 key bits truncated to 64 - pbits | prim)
//                       scattered into its tile bucket through a per-tile cursor
//   tile_sort_kernel    one CTA per tile (heavy tiles first): bucket pass
//                       linear in depth, then every item ranks itself in its
//                       bucket by the composite, equal key prefixes by
//                       (fp64 key, prim id); tiles over SORT_HUGE entries
//                       finish in tile_sort_chunks_kernel
// The result equals lexsort((prim, key, tile)) exactly: within a tile the
// order is (key ascending, prim ascending), a total order.
//
// Compiled with -fmad=false (keys must round exactly as the reference).
#include <cuda_pipeline.h>

#include "kernels.cuh"

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
__global__ void scan_top_kernel(int64_t *sums, int nb, int64_t *d_total, int64_t *out, int n,
                                const int32_t *nonfinite)   // default nullptr (kernels.cuh)
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
    if (threadIdx.x == 0) {
        out[n] = carry;
        // the host's one read per view: the pair count, or -k when k
        // primitives have non-finite raw scales / signs
        const int bad = nonfinite ? *nonfinite : 0;
        *d_total = bad > 0 ? -(int64_t)bad : carry;
    }
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

// Sort composite of a (tile, primitive) pair: the float64 key's bit pattern
// (keys are positive, so bit order is value order) truncated to its top
// 64 - pbits bits, then the primitive id in the low pbits bits.  Ordering
// composites orders by (truncated key, id); entries whose truncated keys are
// equal are put in exact (fp64 key, id) order by the sort.
__device__ __forceinline__ uint64_t sort_composite(double key, int prim, int pbits)
{
    const uint64_t kb = (uint64_t)__double_as_longlong(key);
    return (kb >> pbits << pbits) | (uint64_t)(uint32_t)prim;
}
__device__ __forceinline__ int comp_prim(uint64_t x, int pbits)
{
    return (int)(x & ((1ull << pbits) - 1ull));
}
// 32-bit bucketing key of a composite: exponent (offset from 2^-63) and the
// top 23 mantissa bits of the float64 key -- monotone for keys in
// [2^-63, 2^448] (depths > t_clip, centre distances >= 1e-12)
__device__ __forceinline__ uint32_t sort_h(uint64_t x)
{
    return (uint32_t)((x >> 29) - (960ull << 23));
}

// unit ray of every pixel centre, fp64 (the key kernel's pixel rays)
__global__ void pixel_rays_kernel(CamK cam, double *rays)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cam.W * cam.H) return;
    const int v = i / cam.W, u = i - v * cam.W;
    double cx, cy, cz;
    pixel_ray64(cam, u, v, cx, cy, cz);
    rays[3 * (size_t)i] = cx;
    rays[3 * (size_t)i + 1] = cy;
    rays[3 * (size_t)i + 2] = cz;
}

// One warp per primitive; lanes stride over the primitive's tiles (row-major
// inside its box).  Per pair: the clamped vertex pixel of the tile, its ray
// from the table and the float64 key with the reference's operation order.
// (An fp32 pre-reject of rays that cannot hit the support was measured
// slower: most pairs' vertex-nearest pixel does hit.)
#ifndef QGS_KEY_PREFETCH
#define QGS_KEY_PREFETCH 1
#endif
#ifndef QGS_KEY_MIN_BLOCKS
#define QGS_KEY_MIN_BLOCKS 2     // 128 registers, no spills: 2.74 -> 2.60 ms at C3 (3 and 4 measured)
#endif
__global__ void __launch_bounds__(256, QGS_KEY_MIN_BLOCKS)
pair_key_kernel(PrepView pv, int P, int64_t n_pairs, CamK cam, SetK st,
                const double *__restrict__ rays, int32_t *cursor, uint64_t *bucket)
{
    (void)n_pairs;                 // bounds checks of the debug build only
    __shared__ KeyPrim s_kp[8];
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    const bool euclid = st.euclid != 0;
#if QGS_KEY_PREFETCH
    // The warp's next primitive is fetched while this one's keys are
    // computed: its Geo64 one double per lane (one coalesced 256-B read),
    // its box (lanes 0-3) and tile count (lane 4).  Without it every
    // primitive began with a chain of dependent loads (count, box, geometry
    // read by one lane, first ray) that ~7 key iterations could not hide.
    __shared__ double s_geo[8][32];
    static_assert(sizeof(Geo64) == 32 * sizeof(double), "one double per lane");
    double gv = 0.0;
    int meta = 0;
    auto fetch = [&](int q) {
        if (q < P) {
            gv = __ldg(reinterpret_cast<const double *>(pv.geo + q) + lane);
            meta = lane < 4 ? __ldg(reinterpret_cast<const int *>(pv.bbox + q) + lane)
                            : (lane == 4 ? __ldg(pv.ntiles + q) : 0);
        }
    };
    int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    fetch(p);
    for (; p < P; p += warps) {
        const double cur_gv = gv;
        const int cur_meta = meta;
        fetch(p + warps);
        const int nt = __shfl_sync(0xffffffffu, cur_meta, 4);
        if (nt == 0) continue;
        int4 b;
        b.x = __shfl_sync(0xffffffffu, cur_meta, 0);
        b.y = __shfl_sync(0xffffffffu, cur_meta, 1);
        b.z = __shfl_sync(0xffffffffu, cur_meta, 2);
        const int tx0 = b.x / TILE, ty0 = b.z / TILE;
        const int ncols = b.y / TILE - tx0 + 1;
        __syncwarp();
        s_geo[threadIdx.x >> 5][lane] = cur_gv;
        __syncwarp();
        const Geo64 &g = *reinterpret_cast<const Geo64 *>(s_geo[threadIdx.x >> 5]);
#else
    for (int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < P; p += warps) {
        const int nt = pv.ntiles[p];
        if (nt == 0) continue;
        const int4 b = pv.bbox[p];
        const int tx0 = b.x / TILE, ty0 = b.z / TILE;
        const int ncols = b.y / TILE - tx0 + 1;
        const Geo64 &g = pv.geo[p];
        __syncwarp();
#endif
        // per-primitive key constants in shared memory (broadcast reads)
        if (lane == 0) s_kp[threadIdx.x >> 5] = key_prim(g);
        __syncwarp();
        const KeyPrim &kp = s_kp[threadIdx.x >> 5];
        const long long iu_v = (long long)floor(g.vert_u), iv_v = (long long)floor(g.vert_v);
        int row = lane / ncols, col = lane - row * ncols;
        const int drow = 32 / ncols, dcol = 32 - drow * ncols;
        // software pipeline: the tile's cursor atomic and the next pair's
        // ray load are issued before the current key's fp64 work
        auto pixel_of = [&](int tx, int ty) -> size_t {
            const long long ulo = tx * TILE, uhi = min(cam.W, tx * TILE + TILE) - 1;
            const long long vlo = ty * TILE, vhi = min(cam.H, ty * TILE + TILE) - 1;
            const long long iu = iu_v < ulo ? ulo : (iu_v > uhi ? uhi : iu_v);
            const long long iv = iv_v < vlo ? vlo : (iv_v > vhi ? vhi : iv_v);
            return (size_t)iv * cam.W + iu;
        };
        double cx = 0.0, cy = 0.0, cz = 0.0;
        if (lane < nt) {
            const double *ray = rays + 3 * pixel_of(tx0 + col, ty0 + row);
            cx = ray[0]; cy = ray[1]; cz = ray[2];
        }
        for (int local = lane; local < nt; local += 32) {
            const int tile = (ty0 + row) * cam.tiles_x + tx0 + col;
            const int slot = atomicAdd(&cursor[tile], 1);
            col += dcol;
            row += drow;
            if (col >= ncols) { col -= ncols; ++row; }
            double nx = 0.0, ny = 0.0, nz = 0.0;
            if (local + 32 < nt) {
                const double *ray = rays + 3 * pixel_of(tx0 + col, ty0 + row);
                nx = ray[0]; ny = ray[1]; nz = ray[2];
            }
            const double key = key_from_ray_fast(kp, cx, cy, cz, euclid, st.t_clip);
            QGS_CHECK(slot >= 0 && slot < n_pairs);
            bucket[slot] = sort_composite(key, p, st.pbits);
            cx = nx; cy = ny; cz = nz;
        }
    }
}

// ------------------------------------------------------- per-tile sort
//
// One CTA per tile, two levels:
//   1. bucket (MSD) pass: the tile's depth range (the keys rounded to fp32)
//      cut linearly into nb buckets (nb ~ n/2, a power of two, <= 8192;
//      sample-sort buckets when a linear one exceeds SORT_SKEW items);
//      histogram, scan and an
//      unstable scatter (shared-memory cursors) into a staging array --
//      shared memory when the tile fits, else its slice of `tmp` (L2-resident
//      at these sizes).  Nothing downstream depends on the scatter order.
//   2. every item ranks itself inside its bucket by the composite (key
//      prefix, prim id) -- buckets hold a few items -- and items with equal
//      key prefixes by (fp64 key, prim) (rank_in_bucket), which gives exactly
//      lexsort((prim, key, tile)).  Tiles larger than shared memory are
//      staged in L2 and ranked in groups of whole buckets loaded into
//      shared memory (cut again into second-level buckets when they average
//      over QGS_SORT_L2_MIN items).
#ifndef QGS_SORT_T
#define QGS_SORT_T 512
#endif
#ifndef QGS_SORT_SMEM_ITEMS
#define QGS_SORT_SMEM_ITEMS 6144
#endif
#ifndef QGS_SORT_MIN_BLOCKS
#define QGS_SORT_MIN_BLOCKS 2
#endif
constexpr int SORT_T = QGS_SORT_T;
#ifndef QGS_SORT_IPT
#define QGS_SORT_IPT 8      // 2 4 6 8: C3 2.16 2.08 2.08 2.07 ms
#endif
constexpr int SORT_IPT = QGS_SORT_IPT;            // items per thread per register pass
constexpr int SORT_CHUNK = SORT_T * SORT_IPT;     // items per register pass
constexpr int SORT_SMEM_ITEMS = QGS_SORT_SMEM_ITEMS;   // staged in shared memory up to this
static_assert(SORT_MAX_BUCKETS == 8192, "kernels.cuh");
#ifndef QGS_SORT_L2_MIN
#define QGS_SORT_L2_MIN 12   // mean first-level bucket that takes the second level (6 8 12 16 never: 2.25 2.24 2.20 2.20 2.21 ms at C3)
#endif
constexpr int SORT_NB2 = 2048;                   // second-level buckets of a staged group
// one register pass of items c0 + k * SORT_T + threadIdx.x (k < SORT_IPT) of
// a[0, n): every load issued before any is used
__device__ __forceinline__ void load_chunk(uint64_t (&v)[SORT_IPT], const uint64_t *a, int c0, int n)
{
#pragma unroll
    for (int k = 0; k < SORT_IPT; ++k) {
        const int i = c0 + k * SORT_T + (int)threadIdx.x;
        v[k] = i < n ? a[i] : 0ull;
    }
}

// a staged group uses the head of buf; its second-level bucket counts the tail
constexpr int SORT_GROUP_ITEMS = SORT_SMEM_ITEMS - SORT_NB2 / 2;

#ifndef QGS_SORT_HUGE
#define QGS_SORT_HUGE 49152
#endif
constexpr int SORT_HUGE = QGS_SORT_HUGE;        // tiles over this many entries: multi-CTA stage 2
constexpr int SORT_CHUNKS = 16;                  // CTAs per huge tile in stage 2

struct SortSmem {
    uint64_t buf[SORT_SMEM_ITEMS];
    int bend[SORT_MAX_BUCKETS];   // counts -> start cursors -> (after the scatter) bucket ends
    int scan_w[32];
    uint32_t kmin, kmax;
    int maxcnt;
};

// the float64 key of a tied entry (pixel rays from the key kernel's table)
__device__ __noinline__ double key64_of(uint64_t v, int tile, const PrepView &pv,
                                        const CamK &cam, const SetK &st)
{
    return tile_key_geo(pv.geo[comp_prim(v, st.pbits)], tile, cam, st.euclid != 0, st.t_clip, pv.rays);
}

// Final position of composite x inside its bucket [b0, b1) of `a`: items
// with a smaller f32 key, plus items with the same f32 key that precede it in
// (fp64 key, prim) order.  Composites are distinct (prim ids are), and equal
// f32 keys are rare, so the fp64 keys are recomputed only for those.
// (the rare tie path, out of line: its fp64 key calls would otherwise set the
// register allocation -- and the spills -- of the whole sort kernel)
__device__ __noinline__ int rank_in_bucket(const uint64_t *a, int b0, int b1, uint64_t x,
                                           int tile, const PrepView &pv, const CamK &cam,
                                           const SetK &st)
{
    const int pb = st.pbits;
    const uint64_t h = x >> pb;
    const int p = comp_prim(x, pb);
    int r = 0;
    bool have = false;
    double kx = 0.0;
    for (int j = b0; j < b1; ++j) {
        const uint64_t y = a[j];
        const uint64_t hy = y >> pb;
        if (hy < h) {
            ++r;
        } else if (hy == h && y != x) {
            if (!have) { kx = key64_of(x, tile, pv, cam, st); have = true; }
            const double ky = key64_of(y, tile, pv, cam, st);
            r += (ky < kx || (ky == kx && comp_prim(y, pb) < p)) ? 1 : 0;
        }
    }
    return r;
}

// Emit the sorted order of buckets [g0, g1) whose items sit in a[0 .. ),
// bucket b at a[bucket_start(b) - base ...]: every item finds its own rank inside
// its bucket (buckets average a few items), item-parallel over the CTA.
// Ends with __syncthreads.
__device__ __forceinline__ int bucket_start(const SortSmem &sm, int d)
{
    return d == 0 ? 0 : sm.bend[d - 1];
}

// Bucket of a composite: the tile's key range cut linearly in depth -- the
// float64 key (low bits: the id) rounded to fp32, (f - dmin) * dscale,
// truncated and clamped -- or, for tiles whose depths cluster so that a
// linear cut leaves buckets of hundreds of items, the number of sample
// splitters <= its sort_h (a sample sort's buckets, balanced whatever the
// distribution).  Both are monotone in the composite (rounding, subtraction
// and scaling by a positive factor never reverse an order; fminf sends inf
// and NaN to the last bucket), so bucket order is key order.  (Linear in
// sort_h -- the top 32 bits of the key's bit pattern, log-like across
// octaves -- left 9.6 items per rank at C3; linear in depth 6.2,
// tools/sort_stats.py.)
constexpr int SORT_SPLIT = 4095;                 // most splitters (a sample of 4096)
#ifndef QGS_SORT_SKEW
#define QGS_SORT_SKEW 128
#endif
constexpr int SORT_SKEW = QGS_SORT_SKEW;         // largest linear bucket tolerated
__device__ __forceinline__ float key_f32(uint64_t x)
{
    return __double2float_rn(__longlong_as_double((long long)x));
}
struct BucketFn {
    float dmin, dscale;                          // linear buckets
    int nbm1;                                    // last bucket
    const uint32_t *sp;                          // sorted splitters, or nullptr
    int ns;                                      // number of splitters
    __device__ __forceinline__ float pos(uint64_t x) const { return (key_f32(x) - dmin) * dscale; }
    __device__ __forceinline__ int operator()(uint64_t x) const
    {
        if (!sp) return __float2int_rz(fminf(pos(x), (float)nbm1));
        const uint32_t h = sort_h(x);
        int lo = 0, hi = ns;                     // upper_bound(sp, h)
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sp[mid] <= h) lo = mid + 1; else hi = mid;
        }
        return lo;
    }
};

// rank of x among its bucket a[b0, b1): composite compare, with the exact
// (fp64 key, prim) order only when an equal f32 key is present
__device__ __forceinline__ int rank_fast(const uint64_t *a, int b0, int b1, uint64_t x, int tile,
                                         const PrepView &pv, const CamK &cam, const SetK &st)
{
    // y has x's key prefix and another id  <=>  0 < (y ^ x) < 2^pbits
    const uint64_t pm1 = (1ull << st.pbits) - 1ull;
    int r = 0;
    bool eq = false;
#pragma unroll 4
    for (int j = b0; j < b1; ++j) {
        const uint64_t y = a[j];
        r += y < x ? 1 : 0;
        eq |= ((y ^ x) - 1ull) < pm1;
    }
    return eq ? rank_in_bucket(a, b0, b1, x, tile, pv, cam, st) : r;
}

__device__ void sort_buckets(SortSmem &sm, const uint64_t *a, int base, int g0, int g1,
                             const BucketFn &bf, int tile, const PrepView &pv,
                             const CamK &cam, const SetK &st, int32_t *out)
{
    const int i0 = bucket_start(sm, g0) - base, i1 = bucket_start(sm, g1) - base;
    for (int i = i0 + threadIdx.x; i < i1; i += SORT_T) {
        const uint64_t x = a[i];
        const int d = bf(x);
        const int b0 = bucket_start(sm, d), b1 = sm.bend[d];
        const int r = b1 - b0 == 1 ? 0 : rank_fast(a, b0 - base, b1 - base, x, tile, pv, cam, st);
        QGS_CHECK(r >= 0 && r < b1 - b0);
        out[b0 + r] = comp_prim(x, st.pbits);
    }
    __syncthreads();
}

// Second level: the group's key interval [glo, ghi) (from the
// first-level bucket bounds) cut linearly into SORT_NB2 buckets;
// histogram from the L2 slice, scatter into shared memory, rank.
// First-level buckets of big tiles hold tens to hundreds of
// items, too many for the quadratic in-bucket rank.
// The second-level bucket: linear in the first level's depth coordinate
// over the group's buckets [g0, g1), or (sample-sort first level) linear in
// sort_h over the group's key interval [glo, ghi).
struct SubFn {
    const BucketFn &bf;
    float g0, s2f;
    uint32_t glo;
    int s2;
    __device__ __forceinline__ int operator()(uint64_t x) const
    {
        if (!bf.sp) return __float2int_rz(fminf((bf.pos(x) - g0) * s2f, (float)(SORT_NB2 - 1)));
        return (int)((sort_h(x) - glo) >> s2);
    }
};

__device__ __noinline__ void sort_group_l2(SortSmem &sm, const uint64_t *stage, int base, int cnt,
                                           const BucketFn &bf, int g0, int g1, uint64_t glo,
                                           uint64_t ghi, int tile, const PrepView &pv,
                                           const CamK &cam, const SetK &st, int32_t *out)
{
    int *bend2 = reinterpret_cast<int *>(sm.buf + SORT_GROUP_ITEMS);
    int s2 = 0;
    if (bf.sp)
        while (((ghi - glo - 1) >> s2) >= (uint64_t)SORT_NB2) ++s2;
    const SubFn bf2{bf, (float)g0, (float)SORT_NB2 / (float)(g1 - g0), (uint32_t)glo, s2};
    for (int d = threadIdx.x; d < SORT_NB2; d += SORT_T) bend2[d] = 0;
    __syncthreads();
    for (int c0 = 0; c0 < cnt; c0 += SORT_CHUNK) {
        uint64_t v[SORT_IPT];
        load_chunk(v, stage + base, c0, cnt);
#pragma unroll
        for (int k = 0; k < SORT_IPT; ++k)
            if (c0 + k * SORT_T + (int)threadIdx.x < cnt) atomicAdd(&bend2[bf2(v[k])], 1);
    }
    __syncthreads();
    {
        constexpr int PER = SORT_NB2 / SORT_T;
        int c[PER], sum = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) { c[q] = bend2[threadIdx.x * PER + q]; sum += c[q]; }
        int tot;
        int ex = block_exclusive_scan<int>(sum, sm.scan_w, tot);
#pragma unroll
        for (int q = 0; q < PER; ++q) { bend2[threadIdx.x * PER + q] = ex; ex += c[q]; }
    }
    __syncthreads();
    for (int c0 = 0; c0 < cnt; c0 += SORT_CHUNK) {
        uint64_t v[SORT_IPT];
        load_chunk(v, stage + base, c0, cnt);
#pragma unroll
        for (int k = 0; k < SORT_IPT; ++k)
            if (c0 + k * SORT_T + (int)threadIdx.x < cnt) sm.buf[atomicAdd(&bend2[bf2(v[k])], 1)] = v[k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += SORT_T) {
        const uint64_t x = sm.buf[i];
        const int d = bf2(x);
        const int b0 = d == 0 ? 0 : bend2[d - 1], b1 = bend2[d];
        const int r = b1 - b0 == 1 ? 0 : rank_fast(sm.buf, b0, b1, x, tile, pv, cam, st);
        out[base + b0 + r] = comp_prim(x, st.pbits);
    }
    __syncthreads();
}

__device__ __forceinline__ void sort_groups(SortSmem &sm, const uint64_t *stage, int c0, int c1, int nb,
                                         const BucketFn &bf, uint32_t kmin, uint32_t range,
                                         int shift, int tile, const PrepView &pv, const CamK &cam,
                                         const SetK &st, int32_t *out);

__global__ void __launch_bounds__(SORT_T, QGS_SORT_MIN_BLOCKS)
tile_sort_kernel(const int32_t *__restrict__ tile_offsets, uint64_t *keys, uint64_t *tmp,
                 PrepView pv, CamK cam, SetK st, int32_t *tile_prims, const int32_t *order,
                 HugeSort *huge)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem &sm = *reinterpret_cast<SortSmem *>(smem_raw);
    const int tile = order ? order[blockIdx.x] : (int)blockIdx.x;
    const int start = tile_offsets[tile], n = tile_offsets[tile + 1] - start;
    if (n == 0) return;
    const int lane = threadIdx.x & 31;
    const uint64_t *src = keys + start;
    int32_t *out = tile_prims + start;
    if (n == 1) {
        if (threadIdx.x == 0) out[0] = comp_prim(src[0], st.pbits);
        return;
    }
    uint64_t *stage = n <= SORT_SMEM_ITEMS ? sm.buf : tmp + start;
    const bool regs = n <= SORT_CHUNK;     // one register pass holds the whole tile

    // key range
    if (threadIdx.x == 0) { sm.kmin = 0xffffffffu; sm.kmax = 0u; sm.maxcnt = 0; }
    uint64_t it[SORT_IPT];
    uint32_t lmin = 0xffffffffu, lmax = 0u;
    for (int c0 = 0; c0 < n; c0 += SORT_CHUNK) {
#pragma unroll
        for (int k = 0; k < SORT_IPT; ++k) {
            const int i = c0 + k * SORT_T + threadIdx.x;
            it[k] = i < n ? src[i] : 0ull;
            if (i < n) {
                const uint32_t h = sort_h(it[k]);
                lmin = min(lmin, h); lmax = max(lmax, h);
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
        lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    }
    int nb = 64;
    while (nb < SORT_MAX_BUCKETS && nb * 2 < n) nb <<= 1;
    for (int d = threadIdx.x; d < nb; d += SORT_T) sm.bend[d] = 0;
    __syncthreads();
    if (lane == 0) { atomicMin(&sm.kmin, lmin); atomicMax(&sm.kmax, lmax); }
    __syncthreads();
    const uint32_t kmin = sm.kmin, range = sm.kmax - sm.kmin;
    int shift = 0;
    while ((range >> shift) >= (uint32_t)nb) ++shift;
    // the key range as fp32 depths: composites below / above every key of the tile
    const float dmin = key_f32(((uint64_t)kmin + (960ull << 23)) << 29);
    const float rf = key_f32(((uint64_t)sm.kmax + (960ull << 23) + 1ull) << 29) - dmin;
    BucketFn bf{dmin, rf > 0.f ? fminf((float)nb / rf, 1e30f) : 0.f, nb - 1, nullptr, 0};

    // histogram (a tile over one register pass: the chunk's SORT_IPT loads
    // are all issued before the first use -- load, use, load, use left one
    // L2 read in flight per thread)
    for (int c0 = 0; c0 < n; c0 += SORT_CHUNK) {
        if (!regs) load_chunk(it, src, c0, n);
#pragma unroll
        for (int k = 0; k < SORT_IPT; ++k) {
            const int i = c0 + k * SORT_T + threadIdx.x;
            if (i < n) atomicAdd(&sm.bend[bf(it[k])], 1);
        }
    }
    __syncthreads();
    {
        int mx = 0;
        for (int d = threadIdx.x; d < nb; d += SORT_T) mx = max(mx, sm.bend[d]);
        mx = __reduce_max_sync(0xffffffffu, mx);
        if (lane == 0) atomicMax(&sm.maxcnt, mx);
    }
    __syncthreads();
    if (sm.maxcnt > SORT_SKEW && n >= 512) {
        // depths cluster: sample-sort buckets instead.  S evenly spaced keys
        // (S a power of two <= n / 2, <= 4096) are sorted in shared memory
        // (bitonic), the S - 1 upper ones become splitters (kept in the
        // upper half of bend) and the histogram is redone.
        int S = 256;
        while (S < SORT_SPLIT + 1 && 4 * S <= n) S <<= 1;
        uint32_t *smp = reinterpret_cast<uint32_t *>(sm.buf);
        for (int i = threadIdx.x; i < S; i += SORT_T)
            smp[i] = sort_h(src[(size_t)i * n / S]);
        __syncthreads();
        for (int k = 2; k <= S; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < S; i += SORT_T) {
                    const int l = i ^ j;
                    if (l > i) {
                        const uint32_t a = smp[i], b = smp[l];
                        const bool up = (i & k) == 0;
                        if ((a > b) == up) { smp[i] = b; smp[l] = a; }
                    }
                }
                __syncthreads();
            }
        uint32_t *sp = reinterpret_cast<uint32_t *>(sm.bend) + SORT_MAX_BUCKETS / 2 + 1;
        for (int i = threadIdx.x; i < S - 1; i += SORT_T) sp[i] = smp[i + 1];
        nb = S;
        bf.ns = S - 1;
        for (int d = threadIdx.x; d < nb; d += SORT_T) sm.bend[d] = 0;
        __syncthreads();
        bf.sp = sp;
        for (int i = threadIdx.x; i < n; i += SORT_T) atomicAdd(&sm.bend[bf(src[i])], 1);
        __syncthreads();
    }
    // exclusive scan of the bucket counts (nb <= 8192 = 16 per thread; the
    // thread's counts are re-read from shared memory rather than held in 16
    // registers -- the kernel runs at 64 and spilled)
    {
        constexpr int PER = SORT_MAX_BUCKETS / SORT_T;
        int sum = 0;
#pragma unroll 4
        for (int q = 0; q < PER; ++q) {
            const int d = threadIdx.x * PER + q;
            sum += d < nb ? sm.bend[d] : 0;
        }
        int tot;
        int ex = block_exclusive_scan<int>(sum, sm.scan_w, tot);
#pragma unroll 4
        for (int q = 0; q < PER; ++q) {
            const int d = threadIdx.x * PER + q;
            if (d < nb) {
                const int c = sm.bend[d];
                sm.bend[d] = ex;
                ex += c;
            }
        }
    }
    __syncthreads();
    // scatter into buckets
    for (int c0 = 0; c0 < n; c0 += SORT_CHUNK) {
        if (!regs) load_chunk(it, src, c0, n);
#pragma unroll
        for (int k = 0; k < SORT_IPT; ++k) {
            const int i = c0 + k * SORT_T + threadIdx.x;
            if (i < n) {
                const int pos = atomicAdd(&sm.bend[bf(it[k])], 1);
                stage[pos] = it[k];
            }
        }
    }
    __syncthreads();

    if (n <= SORT_SMEM_ITEMS) {
        sort_buckets(sm, stage, 0, 0, nb, bf, tile, pv, cam, st, out);
    } else {
        // groups of consecutive buckets that fit in shared memory: one
        // coalesced bulk load from the L2 staging slice, then warps sort
        // their buckets out of shared memory.  A tile over SORT_HUGE entries
        // hands its buckets to tile_sort_chunks_kernel instead (SORT_CHUNKS
        // CTAs per tile: one CTA would be the kernel's tail -- C4's largest
        // tiles hold 391K entries).
        if (n > SORT_HUGE && huge) {
            __shared__ int s_h;
            if (threadIdx.x == 0) {
                const int h = atomicAdd(&huge->count, 1);
                s_h = h;
                if (h < SORT_MAX_HUGE) {
                    HugeTile &t = huge->t[h];
                    t.tile = tile; t.nb = nb; t.kmin = kmin; t.range = range; t.shift = shift;
                    t.ns = bf.sp ? bf.ns : -1;
                    t.dmin = bf.dmin; t.dscale = bf.dscale;
                }
            }
            __syncthreads();
            if (s_h < SORT_MAX_HUGE) {
                int *dst = huge->bend_of(s_h);
                for (int d = threadIdx.x; d < SORT_MAX_BUCKETS; d += SORT_T) dst[d] = sm.bend[d];
                return;
            }
        }
        sort_groups(sm, stage, 0, nb, nb, bf, kmin, range, shift, tile, pv, cam, st, out);
    }
}

// The buckets [c0, c1) of a tile, staged in L2 (`stage`), in groups that fit
// in shared memory (see tile_sort_kernel); sm.bend holds the bucket ends.
__device__ __forceinline__ void sort_groups(SortSmem &sm, const uint64_t *stage, int c0, int c1, int nb,
                                         const BucketFn &bf, uint32_t kmin, uint32_t range,
                                         int shift, int tile, const PrepView &pv, const CamK &cam,
                                         const SetK &st, int32_t *out)
{
        (void)shift;
        auto lo_of = [&](int d) -> uint64_t {     // sample-sort buckets only
            if (d == 0) return kmin;
            return d > bf.ns ? (uint64_t)kmin + range + 1 : (uint64_t)bf.sp[d - 1];
        };
        int g0 = c0;
        while (g0 < c1) {
            const int base = bucket_start(sm, g0);
            // last bucket end within SORT_GROUP_ITEMS of base (binary search)
            int lo = g0 + 1, hi = c1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (sm.bend[mid - 1] - base <= SORT_GROUP_ITEMS) lo = mid; else hi = mid - 1;
            }
            int g1 = lo;
            if (sm.bend[g1 - 1] - base > SORT_GROUP_ITEMS) {
                // one degenerate bucket larger than shared memory: rank it in place
                const int b1 = sm.bend[g1 - 1];
                for (int i = base + threadIdx.x; i < b1; i += SORT_T) {
                    const uint64_t x = stage[i];
                    out[base + rank_in_bucket(stage, base, b1, x, tile, pv, cam, st)] =
                        comp_prim(x, st.pbits);
                }
                __syncthreads();
                g0 = g1;
                continue;
            }
            const int cnt = sm.bend[g1 - 1] - base;
            if (cnt <= QGS_SORT_L2_MIN * (g1 - g0)) {
                // first-level buckets already small: rank in them directly
                for (int i = threadIdx.x; i < cnt; i += SORT_T)
                    __pipeline_memcpy_async(&sm.buf[i], &stage[base + i], sizeof(uint64_t));
                __pipeline_commit();
                __pipeline_wait_prior(0);
                __syncthreads();
                sort_buckets(sm, sm.buf, base, g0, g1, bf, tile, pv, cam, st, out);
                g0 = g1;
                continue;
            }
            sort_group_l2(sm, stage, base, cnt, bf, g0, g1, bf.sp ? lo_of(g0) : 0ull,
                          bf.sp ? lo_of(g1) : 0ull, tile, pv, cam, st, out);
            g0 = g1;
        }
}

// second stage of the tiles over SORT_HUGE entries: CTA (h, j) sorts chunk j
// of huge tile h's buckets (first stage: tile_sort_kernel)
__global__ void __launch_bounds__(SORT_T, QGS_SORT_MIN_BLOCKS)
tile_sort_chunks_kernel(const int32_t *__restrict__ tile_offsets, const uint64_t *tmp, PrepView pv,
                        CamK cam, SetK st, int32_t *tile_prims, const HugeSort *huge)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SortSmem &sm = *reinterpret_cast<SortSmem *>(smem_raw);
    // a persistent grid over the (huge tile, chunk) items: the count is only
    // known on the device, and a grid sized for the maximum cost 0.15 ms of
    // empty CTAs per view when there is no huge tile
    const int n_items = min(huge->count, SORT_MAX_HUGE) * SORT_CHUNKS;
    for (int w = (int)blockIdx.x; w < n_items; w += (int)gridDim.x) {
    const int h = w / SORT_CHUNKS, j = w % SORT_CHUNKS;
    const HugeTile t = huge->t[h];
    const int start = tile_offsets[t.tile];
    const int *src = const_cast<HugeSort *>(huge)->bend_of(h);
    for (int d = threadIdx.x; d < SORT_MAX_BUCKETS; d += SORT_T) sm.bend[d] = src[d];
    __syncthreads();
    BucketFn bf{t.dmin, t.dscale, t.nb - 1, nullptr, 0};
    if (t.ns >= 0) {
        bf.sp = reinterpret_cast<const uint32_t *>(sm.bend) + SORT_MAX_BUCKETS / 2 + 1;
        bf.ns = t.ns;
    }
    const int c0 = (int)((long long)t.nb * j / SORT_CHUNKS);
    const int c1 = (int)((long long)t.nb * (j + 1) / SORT_CHUNKS);
    if (c0 < c1)
        sort_groups(sm, tmp + start, c0, c1, t.nb, bf, t.kmin, t.range, t.shift, t.tile, pv, cam,
                    st, tile_prims + start);
    __syncthreads();                    // sm.bend is reloaded by the next item
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
int sort_chunks() { return SORT_CHUNKS; }
size_t huge_sort_bytes() { return sizeof(HugeSort) + (size_t)SORT_MAX_HUGE * SORT_MAX_BUCKETS * sizeof(int); }
int sort_threads() { return SORT_T; }

}  // namespace qgs
