// Deterministic backward reduction (RenderSettings.deterministic).
//
// The reference merges its per-(tile, pair) gradient rows serially in a
// fixed order (raster_kernels.py:9-11, 673-681), so its backward is bitwise
// repeatable (pkg/tests/test_rasterizer_gradients.py:217-229).  The default
// GPU backward reduces with fp32 vector atomics, whose order varies.  This
// mode replaces the atomics by a fixed-order reduction:
//
//   1. det_counts_kernel: every pixel's composited-fragment count in raster
//      warp order (warp = 8x4 block, tile-major; lane = pixel in the block);
//      an exclusive scan gives each pixel a base row, so fragment k of a
//      pixel owns row base + k -- a position fixed by the forward alone.
//   2. The backward kernel writes each fragment's 16 kernel-gradient slots
//      to its row (and the primitive id beside it) instead of adding them.
//   3. A stable radix sort of (primitive id, row) groups the rows of each
//      primitive in row order.  Each primitive's segment is cut into chunks
//      whose length depends on the segment length alone (256 rows, ~sqrt(n)
//      for long segments); a warp per chunk sums its rows in fp64 (fixed lane
//      assignment, one fixed shuffle), then the chunk sums of a primitive are
//      added in chunk order and the rounded total goes to kg.  (A warp per
//      whole primitive left the screen-sized primitives of C4 -- 10^5-10^6
//      rows each -- as a 90 ms serial tail.)
//
// Same bits on every run, and fp64 accumulation instead of fp32 atomics.
#include <algorithm>

#include <cub/cub.cuh>

#include "kernels.cuh"

namespace qgs {

__global__ void det_counts_kernel(CamK cam, const int32_t *__restrict__ n_frag, int n_slots,
                                  int32_t *__restrict__ counts)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_slots) return;
    const int rw = i >> 5, lane = i & 31;
    const int tile = rw >> 3, blk = rw & 7;
    const int ty = tile / cam.tiles_x, tx = tile - ty * cam.tiles_x;
    const int u = tx * TILE + (blk & 1) * 8 + (lane & 7);
    const int v = ty * TILE + (blk >> 1) * 4 + (lane >> 3);
    counts[i] = (u < cam.W && v < cam.H) ? n_frag[v * cam.W + u] : 0;
}

__global__ void det_iota_kernel(int64_t n, uint32_t *out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint32_t)i;
}

// first sorted position of each primitive (lower bound), P + 1 entries
__global__ void det_bounds_kernel(const uint32_t *__restrict__ keys, int64_t n, int P,
                                  int64_t *__restrict__ start)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > P) return;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < (uint32_t)p) lo = mid + 1;
        else hi = mid;
    }
    start[p] = lo;
}

// rows per chunk of a primitive's sorted segment: a function of its length only
__device__ __forceinline__ int64_t det_chunk_rows(int64_t len)
{
    const int64_t r = (int64_t)sqrt((double)len);
    return r > 256 ? (r + 31) & ~(int64_t)31 : 256;
}

__global__ void det_nchunks_kernel(const int64_t *__restrict__ start, int P,
                                   int32_t *__restrict__ nchunk)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > P) return;
    int32_t n = 0;
    if (p < P) {
        const int64_t len = start[p + 1] - start[p];
        if (len > 0) n = (int32_t)((len + det_chunk_rows(len) - 1) / det_chunk_rows(len));
    }
    nchunk[p] = n;
}

// chunk -> primitive map (chunks of a primitive are consecutive)
__global__ void det_owner_kernel(const int64_t *__restrict__ coff, int P, int32_t *__restrict__ owner)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    for (int64_t c = coff[p]; c < coff[p + 1]; ++c) owner[c] = p;
}

// warp per chunk: lane l sums slot (l & 15) over the chunk's rows half
// (l >> 4), (l >> 4) + 2, ... in fp64; the halves combine by one shuffle
__global__ void det_chunk_kernel(const int64_t *__restrict__ start, const int64_t *__restrict__ coff,
                                 const int32_t *__restrict__ owner, const uint32_t *__restrict__ order,
                                 const float *__restrict__ rows, int P, double *__restrict__ part)
{
    const int64_t n_chunks = coff[P];
    const int lane = threadIdx.x & 31, slot = lane & 15, half = lane >> 4;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < n_chunks;
         c += warps) {
        const int p = owner[c];
        const int64_t s0 = start[p], len = start[p + 1] - s0, cr = det_chunk_rows(len);
        const int64_t a = s0 + (c - coff[p]) * cr, b = min(a + cr, s0 + len);
        double s = 0.0;
#pragma unroll 4
        for (int64_t j = a + half; j < b; j += 2) s += (double)rows[(size_t)order[j] * KG + slot];
        s += __shfl_down_sync(0xffffffffu, s, 16);
        if (half == 0) part[(size_t)c * KG + slot] = s;
    }
}

// half-warp per primitive: the chunk sums in chunk order
__global__ void det_combine_kernel(const int64_t *__restrict__ coff, const double *__restrict__ part,
                                   int P, float *__restrict__ kg)
{
    const int p = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 4);
    const int slot = threadIdx.x & 15;
    if (p >= P) return;
    const int64_t c0 = coff[p], c1 = coff[p + 1];
    if (c1 == c0) return;
    double s = 0.0;
    for (int64_t c = c0; c < c1; ++c) s += part[(size_t)c * KG + slot];
    kg[(size_t)p * KG + slot] += (float)s;
}

namespace {
inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }
inline int cdiv64(int64_t a, int b) { return (int)((a + b - 1) / b); }

struct DetWs {
    int32_t *counts;
    int64_t *base;
    float *rows;
    uint32_t *prim, *prim_sorted, *idx, *idx_sorted;
    int64_t *start;
    int32_t *nchunk, *owner;
    int64_t *coff;
    double *part;
    void *temp;
    size_t temp_bytes;
    size_t bytes;
};

// chunks of all segments: at most n_frags / 256 + one partial chunk per primitive
inline int64_t max_chunks(int P, int64_t n_frags) { return n_frags / 256 + (int64_t)P + 1; }

size_t cub_temp_bytes(int P, int64_t n_frags, int n_slots)
{
    size_t a = 0, b = 0, c = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (const int32_t *)nullptr, (int64_t *)nullptr, n_slots);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (const int32_t *)nullptr, (int64_t *)nullptr, P + 1);
    a = a > c ? a : c;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (int64_t)(n_frags > 0 ? n_frags : 1));
    return a > b ? a : b;
}

DetWs det_ws(void *base, int P, int64_t n_frags, int n_slots)
{
    DetWs w;
    char *b = static_cast<char *>(base);
    size_t o = 0;
    const size_t nf = (size_t)(n_frags > 0 ? n_frags : 1);
    w.counts = reinterpret_cast<int32_t *>(b + o);      o += al((size_t)n_slots * 4);
    w.base = reinterpret_cast<int64_t *>(b + o);        o += al((size_t)n_slots * 8);
    w.rows = reinterpret_cast<float *>(b + o);          o += al(nf * KG * 4);
    w.prim = reinterpret_cast<uint32_t *>(b + o);       o += al(nf * 4);
    w.prim_sorted = reinterpret_cast<uint32_t *>(b + o); o += al(nf * 4);
    w.idx = reinterpret_cast<uint32_t *>(b + o);        o += al(nf * 4);
    w.idx_sorted = reinterpret_cast<uint32_t *>(b + o); o += al(nf * 4);
    w.start = reinterpret_cast<int64_t *>(b + o);       o += al(((size_t)P + 1) * 8);
    w.nchunk = reinterpret_cast<int32_t *>(b + o);      o += al(((size_t)P + 1) * 4);
    w.coff = reinterpret_cast<int64_t *>(b + o);        o += al(((size_t)P + 1) * 8);
    const size_t nc = (size_t)max_chunks(P, n_frags);
    w.owner = reinterpret_cast<int32_t *>(b + o);       o += al(nc * 4);
    w.part = reinterpret_cast<double *>(b + o);         o += al(nc * KG * 8);
    w.temp_bytes = cub_temp_bytes(P, n_frags, n_slots);
    w.temp = b + o;                                     o += al(w.temp_bytes);
    w.bytes = o;
    return w;
}
}  // namespace

size_t det_workspace_bytes(int P, int64_t n_frags, int n_warps)
{
    return det_ws(nullptr, P, n_frags, n_warps * 32).bytes;
}

// stage 1 (before the backward kernel): per-pixel base rows
cudaError_t det_prepare(const CamK &cam, const int32_t *n_frag, int P, int64_t n_frags,
                        void *ws, size_t ws_bytes, DetRows &out, cudaStream_t s)
{
    const int n_slots = cam.tiles_x * cam.tiles_y * 8 * 32;
    DetWs w = det_ws(ws, P, n_frags, n_slots);
    if (w.bytes > ws_bytes) return cudaErrorInvalidValue;
    det_counts_kernel<<<cdiv64(n_slots, 256), 256, 0, s>>>(cam, n_frag, n_slots, w.counts);
    size_t tb = w.temp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(w.temp, tb, w.counts, w.base, n_slots, s);
    if (e != cudaSuccess) return e;
    out.base = w.base;
    out.rows = w.rows;
    out.prim = reinterpret_cast<int32_t *>(w.prim);
    return cudaGetLastError();
}

// stage 3 (after the backward kernel): fixed-order per-primitive sums into kg
cudaError_t det_finish(int P, int64_t n_frags, int n_warps, void *ws, float *kg, cudaStream_t s)
{
    DetWs w = det_ws(ws, P, n_frags, n_warps * 32);
    if (n_frags > 0) {
        det_iota_kernel<<<cdiv64(n_frags, 256), 256, 0, s>>>(n_frags, w.idx);
        int bits = 1;
        while (bits < 32 && (1ll << bits) < (long long)P) ++bits;
        size_t tb = w.temp_bytes;
        cudaError_t e = cub::DeviceRadixSort::SortPairs(w.temp, tb, w.prim, w.prim_sorted, w.idx,
                                                        w.idx_sorted, n_frags, 0, bits, s);
        if (e != cudaSuccess) return e;
    }
    det_bounds_kernel<<<cdiv64((int64_t)P + 1, 256), 256, 0, s>>>(w.prim_sorted, n_frags, P,
                                                                  w.start);
    det_nchunks_kernel<<<cdiv64((int64_t)P + 1, 256), 256, 0, s>>>(w.start, P, w.nchunk);
    size_t tb = w.temp_bytes;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(w.temp, tb, w.nchunk, w.coff, P + 1, s);
    if (e != cudaSuccess) return e;
    det_owner_kernel<<<cdiv64(P, 256), 256, 0, s>>>(w.coff, P, w.owner);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nc = max_chunks(P, n_frags);
    const int grid = (int)std::min<int64_t>(cdiv64(nc * 32, 256), (int64_t)sms * 16);
    det_chunk_kernel<<<grid, 256, 0, s>>>(w.start, w.coff, w.owner, w.idx_sorted, w.rows, P, w.part);
    det_combine_kernel<<<cdiv64((int64_t)P * 16, 256), 256, 0, s>>>(w.coff, w.part, P, kg);
    return cudaGetLastError();
}

}  // namespace qgs
