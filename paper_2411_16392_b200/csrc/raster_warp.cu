// K5 forward and K6 backward raster kernels, one warp per 8x4 pixel block.
//
// Reference: raster_kernels.py:83-286 (forward_kernel), :289-502
// (_grad_fragment), :505-670 (backward_kernel), :673-681 (merge).
//
// Work unit = one warp = one 8x4 block of a 16x16 tile (8 blocks per tile).
// Warps never synchronise with each other: a forward CTA holds the 8 warps of
// one tile (a backward CTA 4), only so that they share the SM's L1 for the
// tile's list, boxes and records; each warp stops as soon as its own 32
// pixels have terminated.  Tiles run heaviest first (tile_order_kernel).
//
// Forward, per block:
//   pass 0  the tile's depth-sorted list streamed 32 entries per window, one
//           per lane: culled pixel box against the block, then the screen
//           conic test on all 32 pixels; survivors queue up in stream order
//   batch   WB = 4 queued entries at a time: records staged in shared memory
//           (8 lanes per 128-byte record), fp64 geometry heads by cp.async
//   pass 1  coarse fp32 test (shade.cuh: coarse_stage1/2) of each pixel's
//           culled-in candidates
//   pass 2  set bits in stream order: fp64 depth refinement + exact
//           selection + alpha floor (MODE_EXACT: decisions inside their fp32
//           band re-made in fp64), the 8-entry min-depth ring, fp64
//           compositing of emitted fragments
//   log     every composited fragment (prim, fp64 depth, fp32 local hit
//           point) appended to the paged fragment log
//
// Transmittance, blend weights and the eleven blend sums are fp64: the
// backward's suffix sums (vtot - prefix, the front-to-back rewrite of
// raster_kernels.py:340) are exact to ~1e-15.
//
// Backward: each pixel's logged fragments re-shaded in fp32 from the logged
// hit point (grazing rays from the fp64 geometry), 16 kernel-level gradient
// slots per fragment (ohat, the rotation accumulator's skew part, w, s,
// alpha, colour), reduced across lanes that emitted the same primitive
// (match_any + padded shared-memory transpose) into 16-byte vector atomics --
// or, deterministic mode, written to rows for det_reduce.cu.  Blocks without
// a log are replayed by a separate kernel with the forward's candidate test.
#include <cuda_pipeline.h>

#include "kernels.cuh"
#include "shade.cuh"

namespace qgs {

// minimum resident warps per SM the register allocation must allow
#ifndef QGS_FWD_LIST_PREFETCH
#define QGS_FWD_LIST_PREFETCH 1
#endif
#ifndef QGS_FWD_EXACT_MIN_BLOCKS
#define QGS_FWD_EXACT_MIN_BLOCKS 16   // the fp64 band code needs the registers (measured: 18 -> 16 is -4 %)
#endif
#ifndef QGS_BWD_MIN_BLOCKS
#define QGS_BWD_MIN_BLOCKS 20
#endif
#ifndef QGS_FWD_MIN_BLOCKS
#define QGS_FWD_MIN_BLOCKS 18
#endif

#ifndef QGS_WB
#define QGS_WB 4
#endif
#ifndef QGS_UTIL_COUNTERS
#define QGS_UTIL_COUNTERS 0        // diagnostics build: lane utilisation of passes 1 and 2
#endif
#ifndef QGS_FWD_RAY_REGS
#define QGS_FWD_RAY_REGS 1    // fp64 pixel ray in registers instead of shared memory
#endif
constexpr int WB = QGS_WB;    // queued entries per batch (4, 8 or 16: smem per warp vs batch overhead; 4 measured best)
constexpr unsigned FULL = 0xffffffffu;

// Geo64 head read by the exact test (ohat, M, wv: its first 15 doubles)
struct __align__(16) GeoHead {
    double v[16];
};
static_assert(offsetof(Geo64, wv) + 3 * sizeof(double) <= sizeof(GeoHead), "GeoHead covers ohat, M, wv");

#ifndef QGS_FWD_STAGE_GEO
#define QGS_FWD_STAGE_GEO 1
#endif
#ifndef QGS_PAY_XY
#define QGS_PAY_XY 1
#endif
#ifndef QGS_FWD_COMPOSITE_VEC
#define QGS_FWD_COMPOSITE_VEC 1
#endif
constexpr int PAYN = QGS_PAY_XY ? 3 : 5;


struct FwdSmem {
#if QGS_FWD_STAGE_GEO
    GeoHead geoh[WB];
#endif
    PrimRec rec[WB];
    int qprim[WB + 32];       // culled-in entries waiting for the coarse/exact passes
    uint32_t qmask[WB + 32];  // their conic & box & alive pixel masks
    int aprim[64];            // box-overlapping entries waiting for the conic test
    uint32_t amask[64];       // their box & alive pixel masks
    double ring_t[RING][32];  // per-lane ring, [slot][lane]: conflict-free
    int ring_p[RING][32];
#if !QGS_FWD_RAY_REGS
    double d64[3][32];        // fp64 pixel ray (only the exact path reads it)
#endif
    // fp64 blend sums, touched once per composited fragment (the backward's
    // suffix sums vtot - prefix need them: fp32 colour / normal / curvature
    // sums were measured to triple the gradient violations at C2)
    double acc[11][32];
    float pay[RING][PAYN][32];   // ring payload (see Pay)
    int pages[QGS_FRAG_MAX_PAGES];  // fragment-log pages of this warp
    union {
        float tfirst[WB][32];    // pass 1 -> pass 2: first coarse root that survived
        uint32_t boxw[32];       // work counters only (between batches): window box masks
    };
};

// Ring payload of an accepted fragment.  QGS_PAY_XY: (abar, local hit x, y)
// -- compositing re-derives the camera normal and curvature from them and
// the primitive's record (3 floats per slot keep shared memory per warp, the
// forward's occupancy limiter, low); else (abar, camera normal, curvature).
struct Pay {
    float v[PAYN];
};

// (tile, block) of schedule slot `slot` (default: this warp of this CTA)
// and the lane's pixel
__device__ __forceinline__ void block_pixel(int tiles_x, const int32_t *order, int &tile, int &blk,
                                            int &u, int &v, int slot = -1)
{
    if (slot < 0) slot = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
    tile = order ? order[slot >> 3] : (slot >> 3);
    blk = slot & 7;
    const int ty = tile / tiles_x, tx = tile - ty * tiles_x;
    const int lane = threadIdx.x & 31;
    u = tx * TILE + (blk & 1) * 8 + (lane & 7);
    v = ty * TILE + (blk >> 1) * 4 + (lane >> 3);
}

// stage records list[b0 .. b0+nb) into shared memory; returns lane's prim id
__device__ __forceinline__ int load_batch32(PrimRec *srec, int *sprim,
                                            const PrimRec *__restrict__ recs,
                                            const int32_t *__restrict__ list, int b0, int nb)
{
    const int lane = threadIdx.x & 31;
    const int my = lane < nb ? list[b0 + lane] : 0;
    if (lane < WB) sprim[lane] = my;
    const float4 *src = reinterpret_cast<const float4 *>(recs);
    float4 *dst = reinterpret_cast<float4 *>(srec);
#pragma unroll
    for (int it = 0; it < WB / 4; ++it) {
        const int j = it * 4 + (lane >> 3), q = lane & 7;
        const int pj = __shfl_sync(FULL, my, j);
        if (j < nb) dst[j * 8 + q] = __ldg(src + (size_t)pj * 8 + q);
    }
    __syncwarp();
    return my;
}

// stage the records of queued entries ids[0 .. nb) into shared memory
// (8 lanes per 128-byte record, coalesced)
__device__ __forceinline__ void load_batch_ids(PrimRec *srec, const PrimRec *__restrict__ recs,
                                               const int *ids, int nb)
{
    const int lane = threadIdx.x & 31;
    const float4 *src = reinterpret_cast<const float4 *>(recs);
    float4 *dst = reinterpret_cast<float4 *>(srec);
#pragma unroll
    for (int it = 0; it < WB / 4; ++it) {
        const int j = it * 4 + (lane >> 3), q = lane & 7;
        if (j < nb) dst[j * 8 + q] = __ldg(src + (size_t)ids[j] * 8 + q);
    }
    __syncwarp();
}

// lane mask of this block covered by an inclusive pixel box (packed words)
__device__ __forceinline__ uint32_t block_lanes(uint32_t bb_u, uint32_t bb_v, int bu, int bv)
{
    int c0 = max((int)(bb_u & 0xffffu) - bu, 0), c1 = min((int)(bb_u >> 16) - bu, 7);
    int r0 = max((int)(bb_v & 0xffffu) - bv, 0), r1 = min((int)(bb_v >> 16) - bv, 3);
    if (c0 > c1 || r0 > r1) return 0u;
    uint32_t cols = (0xffu >> (7 - c1)) & (0xffu << c0);
    uint32_t rows = (0xffffffffu >> (8 * (3 - r1))) & (0xffffffffu << (8 * r0));
    return (cols * 0x01010101u) & rows;
}

// Conic cull (ConicRec): mask of block pixels in rows [r0, r0 + NR) whose
// centre lies inside the primitive's bounding-ellipsoid outline.
template <int NR>
__device__ __forceinline__ uint32_t conic_rows(const ConicRec &q, int bu, int bv, int r0)
{
    const float U0 = (float)bu - conic_uc(q), vc = conic_vc(q);
    uint32_t m = 0u;
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
        const int r = r0 + rr;
        const float V = (float)(bv + r) - vc;
        const float QV = fmaf(fmaf(q.C, V, q.E), V, q.F);
        const float BVD = fmaf(q.B, V, q.D);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const float U = U0 + (float)c;
            const float Q = fmaf(fmaf(q.A, U, BVD), U, QV);
            m |= (Q <= 0.f ? 1u : 0u) << (8 * r + c);
        }
    }
    return m;
}

#ifndef QGS_BWD_VEC_LOADS
#define QGS_BWD_VEC_LOADS 1
#endif
#ifndef QGS_RED_SETS
#define QGS_RED_SETS 8
#endif
#ifndef QGS_RED_SINGLES
#define QGS_RED_SINGLES 1
#endif
#ifndef QGS_RED_RANKS
#define QGS_RED_RANKS 1       // group leaders listed by rank in shared memory (no 8-step scan)
#endif
#ifndef QGS_RING_TREE
#define QGS_RING_TREE 1       // full-ring minimum as a 3-level tree (same slot as the scan)
#endif

__device__ __forceinline__ PrimRec load_rec(const PrimRec *p)
{
    PrimRec r;
    const float4 *src = reinterpret_cast<const float4 *>(p);
    float4 *dst = reinterpret_cast<float4 *>(&r);
#pragma unroll
    for (int q = 0; q < 8; ++q) dst[q] = __ldg(src + q);
    return r;
}

// ohat, M, wv (the first 15 doubles) with 16-byte loads; the rest is unset
__device__ __forceinline__ Geo64 load_geo_head(const Geo64 *p)
{
    Geo64 g;
    const double2 *src = reinterpret_cast<const double2 *>(p);
    double2 *dst = reinterpret_cast<double2 *>(&g);
#pragma unroll
    for (int q = 0; q < 8; ++q) dst[q] = __ldg(src + q);
    return g;
}

// Per-lane ring view into shared memory.
struct Ring {
    double *t;   // &ring_t[0][lane], stride 32
    int *p;
    int n;
};

// minimum of a full ring, first slot among equal minima (the reference's
// strict-< scan, raster_kernels.py:160-164).  A tree (left subtree = lower
// slots, right replaces left only when strictly smaller) gives the same slot
// as the linear scan with a 3-deep instead of an 8-deep compare chain.
// Depths in the ring are never NaN (confirm_root rejects !(t > t_clip)).
__device__ __forceinline__ void ring_min(const Ring &R, int n, double &m, int &jm)
{
#if QGS_RING_TREE
    static_assert(RING == 8, "tree minimum of 8 slots");
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = k < n ? R.t[k * 32] : __longlong_as_double(0x7ff0000000000000LL);  // empty: +inf
    int i[8] = {0, 1, 2, 3, 4, 5, 6, 7};
#pragma unroll
    for (int w = 1; w < 8; w <<= 1)
#pragma unroll
        for (int k = 0; k < 8; k += 2 * w) {
            const bool r = v[k + w] < v[k];
            v[k] = r ? v[k + w] : v[k];
            i[k] = r ? i[k + w] : i[k];
        }
    m = v[0];
    jm = i[0];
#else
    m = R.t[0];
    jm = 0;
    for (int k = 1; k < n; ++k) {
        const double tk = R.t[k * 32];
        if (tk < m) { m = tk; jm = k; }
    }
#endif
}
__device__ __forceinline__ void ring_min_full(const Ring &R, double &m, int &jm)
{
    ring_min(R, RING, m, jm);
}

// push an accepted fragment; true with (et, ep) when one is emitted
// (raster_kernels.py:159-226: first minimum, strict <, emit incoming if nearer)
__device__ __forceinline__ bool ring_push(Ring &R, double t, int prim, double &et, int &ep)
{
    if (R.n < RING) {
        QGS_CHECK(R.n >= 0);
        R.t[R.n * 32] = t;
        R.p[R.n * 32] = prim;
        R.n++;
        return false;
    }
    double m;
    int jm;
    ring_min_full(R, m, jm);
    if (t < m) { et = t; ep = prim; return true; }
    et = m;
    ep = R.p[jm * 32];
    R.t[jm * 32] = t;
    R.p[jm * 32] = prim;
    return true;
}

// drain one entry (raster_kernels.py:227-270: first minimum, swap with last)
__device__ __forceinline__ void ring_pop(Ring &R, double &et, int &ep)
{
    double m;
    int jm;
    ring_min(R, R.n, m, jm);
    et = m;
    ep = R.p[jm * 32];
    R.n--;
    R.t[jm * 32] = R.t[R.n * 32];
    R.p[jm * 32] = R.p[R.n * 32];
}

// forward ring with payload (same ordering rule as ring_push / ring_pop)
__device__ __forceinline__ bool ring_push_pay(Ring &R, float (*pay)[PAYN][32], int lane, double t,
                                              int prim, const Pay &in, double &et, int &ep,
                                              Pay &out)
{
    if (R.n < RING) {
        R.t[R.n * 32] = t;
        R.p[R.n * 32] = prim;
#pragma unroll
        for (int f = 0; f < PAYN; ++f) pay[R.n][f][lane] = in.v[f];
        R.n++;
        return false;
    }
    double m;
    int jm;
    ring_min_full(R, m, jm);
    if (t < m) { et = t; ep = prim; out = in; return true; }
    et = m;
    ep = R.p[jm * 32];
#pragma unroll
    for (int f = 0; f < PAYN; ++f) out.v[f] = pay[jm][f][lane];
    R.t[jm * 32] = t;
    R.p[jm * 32] = prim;
#pragma unroll
    for (int f = 0; f < PAYN; ++f) pay[jm][f][lane] = in.v[f];
    return true;
}

__device__ __forceinline__ void ring_pop_pay(Ring &R, float (*pay)[PAYN][32], int lane, double &et,
                                             int &ep, Pay &out)
{
    double m;
    int jm;
    ring_min(R, R.n, m, jm);
    et = m;
    ep = R.p[jm * 32];
#pragma unroll
    for (int f = 0; f < PAYN; ++f) out.v[f] = pay[jm][f][lane];
    R.n--;
    R.t[jm * 32] = R.t[R.n * 32];
    R.p[jm * 32] = R.p[R.n * 32];
#pragma unroll
    for (int f = 0; f < PAYN; ++f) pay[jm][f][lane] = pay[R.n][f][lane];
}

enum { A_C0 = 0, A_A = 3, A_D = 4, A_D2 = 5, A_N0 = 6, A_K = 9, A_DIST = 10 };

// row stride of the backward's reduction buffer: 20 floats (80 B) puts the
// 16-byte stores of 8 consecutive lanes in distinct bank groups (16 would
// put every other lane on the same banks)
constexpr int KGP = KG + 4;

struct BwdSmem {
    PrimRec rec[WB];        // replay path
    int prim[WB];
    double ring_t[RING][32];
    int ring_p[RING][32];
    float red[1][33][KGP];  // row 32 stays zero (padding reads of the group sums)
    int lead[32];           // reduction: lane of the r-th group leader
};

struct Cfg {
    float t_clip, alpha_floor, alpha_clamp;
    double alpha_clamp64, t_term;
    bool euclid, resort;
};

__device__ __forceinline__ Cfg make_cfg(const SetK &st)
{
    Cfg c;
    c.t_clip = (float)st.t_clip;
    c.alpha_floor = (float)st.alpha_floor;
    c.alpha_clamp = (float)st.alpha_clamp;
    c.alpha_clamp64 = st.alpha_clamp;
    c.t_term = st.t_term;
    c.euclid = st.euclid != 0;
    c.resort = st.resort != 0;
    return c;
}

// exact candidate test (raster_kernels.py:121-130, 58-63); t = fp64 depth
template <int M>
__device__ __forceinline__ bool accept(const PrimRec &r, const Geo64 &g, const double d64[3],
                                       float dx, float dy, float dz, const Cfg &c, double &t)
{
    Hit h;
    if (!hit_refined<M>(r, g, d64, dx, dy, dz, c.euclid, c.t_clip, h)) return false;
    if (!alpha_pass<M>(r, &g, d64, h, c.euclid, c.alpha_floor)) return false;
    t = h.t64;
    return true;
}

// ring step for an accepted fragment; returns whether one is emitted
__device__ __forceinline__ bool ring_step(const Cfg &c, Ring &R, double t, int prim, double &et,
                                          int &ep)
{
    if (!c.resort) { et = t; ep = prim; return true; }
    return ring_push(R, t, prim, et, ep);
}

struct Frag {
    Hit h;
    float abar;
    double abar64;
    bool clamped;
    float nl[3], nc[3], K, inrm, flip;
};

// re-shade an emitted fragment at its fp64 depth (raster_kernels.py:40-80)
__device__ __forceinline__ void finish_frag(const PrimRec &r, float dx, float dy, float dz,
                                            const Cfg &c, Frag &f);

__device__ __forceinline__ void shade_emitted(const PrimRec &r, const Geo64 &g, const double d64[3],
                                              float dx, float dy, float dz, double t64,
                                              const Cfg &c, Frag &f)
{
    double dh[3];
    local_dir64(g, d64, dh);
    shade_at(r, g, dh, t64, c.euclid, f.h);
    finish_frag(r, dx, dy, dz, c, f);
}

// weight, alpha and the camera-frame normal of a shaded fragment
__device__ __forceinline__ void finish_frag(const PrimRec &r, float dx, float dy, float dz,
                                            const Cfg &c, Frag &f)
{
    f.h.G = QGS_EXPF(-(f.h.l * f.h.l) / (2.f * f.h.sig * f.h.sig));
    float abar = r.alpha * f.h.G;
    f.clamped = abar > c.alpha_clamp;
    f.abar = f.clamped ? c.alpha_clamp : abar;
    f.abar64 = f.clamped ? c.alpha_clamp64 : (double)abar;
    normal_curv32(r, f.h, dx, dy, dz, f.nl, f.nc, f.K, f.inrm, f.flip);
}

// ================================================================ forward

// One raster block (schedule slot `slot`) of the forward.  M = MODE_FAST:
// fp32 decisions; MODE_EXACT (settings.exact_decisions): decisions inside
// their fp32 rounding band re-made in fp64 (shade.cuh).  Two kernels so
// that the fast one carries no fp64 selection code.  (Measured and
// rejected: an fp32 pass that hands blocks with band cases to a float64
// fix-up pass -- ~15 % of C3's blocks meet one, and the fix-up's tail cost
// more than the exact kernel's register pressure.)
template <int M>
__device__ __forceinline__ void fwd_block(const PrimRec *__restrict__ recs,
                                          const Geo64 *__restrict__ geo,
                                          const ConicRec *__restrict__ conics,
                                          const int32_t *__restrict__ tile_offsets,
                                          const int32_t *__restrict__ tile_prims, const CamK &cam,
                                          const SetK &st, const qgs_targets &out, int slot)
{
    // one FwdSmem per warp (dynamic shared memory: QGS_FWD_WPC warps per CTA)
    extern __shared__ __align__(16) unsigned char raster_smem[];
    FwdSmem &sm = reinterpret_cast<FwdSmem *>(raster_smem)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    int tile, blk, u, v;
    block_pixel(cam.tiles_x, out.tile_order, tile, blk, u, v, slot);
    const int rw = (tile << 3) | blk;                // raster warp id (fragment-log row)
    const int bu = u - (lane & 7), bv = v - (lane >> 3);
    const bool inside = u < cam.W && v < cam.H;
    const Cfg c = make_cfg(st);
    const bool cull = st.no_cull == 0;
    float dx, dy, dz;
    double ray64[3] = {0.0, 0.0, 1.0};
    if (inside) pixel_dir64(cam, u, v, ray64);
#if !QGS_FWD_RAY_REGS
    sm.d64[0][lane] = ray64[0]; sm.d64[1][lane] = ray64[1]; sm.d64[2][lane] = ray64[2];
#endif
    dx = (float)ray64[0]; dy = (float)ray64[1]; dz = (float)ray64[2];
#pragma unroll
    for (int k = 0; k < 11; ++k) sm.acc[k][lane] = 0.0;

    double T = 1.0;
    float median = 0.f;
    double last_t = -1.0e300;
    int nfrag = 0, viol = 0;
    unsigned n_box = 0, n_acc = 0, n_cand = 0, n_coarse = 0;
#if QGS_UTIL_COUNTERS
    unsigned long long u_p1 = 0, u_p2 = 0;        // diagnostics: pass-1 / pass-2 lane slots
#endif
    Ring R{&sm.ring_t[0][lane], &sm.ring_p[0][lane], 0};
    bool alive = inside;
    // paged fragment log (qgs_targets): warp-uniform page count, pages taken
    // from the pool before each batch for the depth the batch can reach
    bool log_on = out.frag_prim != nullptr && out.frag_t != nullptr;
    int npages = 0;
    auto ensure_pages = [&](int extra) {     // warp-uniform call
        if (!log_on) return;
        const int need = (__reduce_max_sync(FULL, (unsigned)nfrag) + extra + QGS_FRAG_PAGE - 1) /
                         QGS_FRAG_PAGE;
        if (need <= npages) return;
        if (need > QGS_FRAG_MAX_PAGES) { log_on = false; return; }
        int base = 0;
        if (lane == 0) base = atomicAdd(out.frag_pool_next, need - npages);
        base = __shfl_sync(FULL, base, 0);
        if (base + (need - npages) > out.frag_pool_pages) { log_on = false; return; }
        QGS_CHECK(need <= QGS_FRAG_MAX_PAGES && base >= 0);
        if (lane < need - npages) sm.pages[npages + lane] = base + lane;
        npages = need;
        __syncwarp();
    };

    auto composite = [&](int ep, double t, const Pay &f) {
#if QGS_FWD_COMPOSITE_VEC
        const PrimRec r = load_rec(recs + ep);      // all 8 lines of the record in flight
#else
        const PrimRec &r = recs[ep];
#endif
        if (t < last_t - 1e-12) viol++;
        if (t > last_t) last_t = t;
        const float fabar = f.v[0];
#if QGS_PAY_XY
        float n0, n1, n2, fK;
        {
            Hit hh;
            hh.x = f.v[1];
            hh.y = f.v[2];
            hh.branch = (r.flags & 1u) ? BR_PLANAR : BR_QUAD;
            float nl[3], nc[3], inrm, flip;
            normal_curv32(r, hh, dx, dy, dz, nl, nc, fK, inrm, flip);
            n0 = nc[0]; n1 = nc[1]; n2 = nc[2];
        }
#else
        const float n0 = f.v[1], n1 = f.v[2], n2 = f.v[3], fK = f.v[4];
#endif
        const double abar64 = fabar < 0.f ? c.alpha_clamp64 : (double)fabar;  // <0: clamped
        const double w = abar64 * T;
        double *a = &sm.acc[0][lane];            // stride 32 doubles per sum
        const double aa = a[A_A * 32], ad = a[A_D * 32], ad2 = a[A_D2 * 32];
        a[(A_C0 + 0) * 32] += w * (double)r.col[0];
        a[(A_C0 + 1) * 32] += w * (double)r.col[1];
        a[(A_C0 + 2) * 32] += w * (double)r.col[2];
        a[A_DIST * 32] += w * (t * t * aa - 2.0 * t * ad + ad2);   // sums before this fragment
        a[A_A * 32] = aa + w;
        a[A_D * 32] = ad + w * t;
        a[A_D2 * 32] = ad2 + w * t * t;
        a[(A_N0 + 0) * 32] += w * (double)n0;
        a[(A_N0 + 1) * 32] += w * (double)n1;
        a[(A_N0 + 2) * 32] += w * (double)n2;
        a[A_K * 32] += w * (double)fK;
        if (T > 0.5) median = (float)t;
        T *= 1.0 - abar64;
        if (log_on) {
            QGS_CHECK(nfrag / QGS_FRAG_PAGE < npages);
            QGS_CHECK(sm.pages[nfrag / QGS_FRAG_PAGE] < out.frag_pool_pages);
            const size_t o = ((size_t)sm.pages[nfrag / QGS_FRAG_PAGE] * QGS_FRAG_PAGE +
                              (nfrag % QGS_FRAG_PAGE)) * 32 + lane;
            out.frag_prim[o] = ep;
            out.frag_t[o] = t;
#if QGS_PAY_XY
            if (out.frag_xy) reinterpret_cast<float2 *>(out.frag_xy)[o] = make_float2(f.v[1], f.v[2]);
#endif
        }
        nfrag++;
        if (T < c.t_term) alive = false;
    };

    // Batch of up to WB queued entries: stage their records, run the coarse
    // test on each pixel's culled-in candidates (pass 1), then the exact
    // test, ring and compositing in stream order (pass 2).  (Measured and
    // rejected: one loop with one call site per phase -- this body is
    // inlined at three -- halves the kernel's code and its instruction-cache
    // stalls, but runs 15 % slower.)
    auto run_batch = [&](int nb) {
        ensure_pages(nb);                        // each entry emits at most one fragment per pixel
        load_batch_ids(sm.rec, recs, sm.qprim, nb);
        // geometry heads for the exact pass, copied asynchronously under pass 1
#if QGS_FWD_STAGE_GEO
        {
            const char *gsrc = reinterpret_cast<const char *>(geo);
            char *gdst = reinterpret_cast<char *>(sm.geoh);
#pragma unroll
            for (int it = 0; it < WB / 4; ++it) {
                const int j = it * 4 + (lane >> 3), q = lane & 7;
                if (j < nb)
                    __pipeline_memcpy_async(gdst + j * sizeof(GeoHead) + 16 * q,
                                            gsrc + (size_t)sm.qprim[j] * sizeof(Geo64) + 16 * q, 16);
            }
            __pipeline_commit();
        }
#endif
        uint32_t cand = 0u;
        for (int j = 0; j < nb; ++j) cand |= ((sm.qmask[j] >> lane) & 1u) << j;
        if (!alive) cand = 0u;

        // pass 1 (two candidates per iteration: their branch-free stage-1
        // chains interleave, which hides the SQRT/RCP latencies)
        uint32_t bits = 0u, margb = 0u, secb = 0u;
        uint32_t uni = __reduce_or_sync(FULL, cand);
        while (uni) {
            const int j = __ffs(uni) - 1;
            uni &= uni - 1;
            const int j1 = uni ? __ffs(uni) - 1 : j;
            uni &= uni - 1;
#if QGS_UTIL_COUNTERS
            u_p1 += (j1 != j) ? 2 : 1;
#endif
            const bool a0 = (cand >> j) & 1u, a1 = j1 != j && ((cand >> j1) & 1u);
            if (!(a0 || a1)) continue;
            float r0[2], r1[2], hx0, hy0, hx1, hy1;
#if QGS_UTIL_COUNTERS
            bool ok0 = true, ok1 = true;
            unsigned s0 = coarse_stage1(sm.rec[j], dx, dy, dz, c.t_clip, r0, hx0, hy0, &ok0);
            unsigned s1 = coarse_stage1(sm.rec[j1], dx, dy, dz, c.t_clip, r1, hx1, hy1, &ok1);
            // [1] is reused here (near-tangent roots are counted in the exact pass)
            if (a0 && !ok0) atomicAdd(&qgs_diag[1], 1ull << 32);
            if (a1 && !ok1) atomicAdd(&qgs_diag[1], 1ull << 32);
#else
            unsigned s0 = coarse_stage1(sm.rec[j], dx, dy, dz, c.t_clip, r0, hx0, hy0);
            unsigned s1 = coarse_stage1(sm.rec[j1], dx, dy, dz, c.t_clip, r1, hx1, hy1);
#endif
            s0 = a0 ? s0 : 0u;
            s1 = a1 ? s1 : 0u;
#if QGS_UTIL_COUNTERS
            // [2]: candidates the stage-1 test rejects (no root, behind the
            // clip, or outside the widened ellipse); [3]: rejected by stage 2
            if (a0 && !s0) atomicAdd(&qgs_diag[2], 1ull);
            if (a1 && !s1) atomicAdd(&qgs_diag[2], 1ull);
#endif
            if (s0) {
                const unsigned p = (s0 & CR_MARGINAL) ? s0 : coarse_stage2(sm.rec[j], c.euclid, s0, r0, hx0, hy0);
#if QGS_UTIL_COUNTERS
                if (!p) atomicAdd(&qgs_diag[3], 1ull);
#endif
                if (p) {
                    bits |= 1u << j;
                    if (p & CR_MARGINAL) margb |= 1u << j;
                    else sm.tfirst[j][lane] = (p & 1u) ? r0[0] : r0[1];
                    if ((p & 3u) == 3u) secb |= 1u << j;
                }
            }
            if (s1) {
                const unsigned p = (s1 & CR_MARGINAL) ? s1 : coarse_stage2(sm.rec[j1], c.euclid, s1, r1, hx1, hy1);
#if QGS_UTIL_COUNTERS
                if (!p) atomicAdd(&qgs_diag[3], 1ull);
#endif
                if (p) {
                    bits |= 1u << j1;
                    if (p & CR_MARGINAL) margb |= 1u << j1;
                    else sm.tfirst[j1][lane] = (p & 1u) ? r1[0] : r1[1];
                    if ((p & 3u) == 3u) secb |= 1u << j1;
                }
            }
        }
        if (out.counters) { n_cand += __popc(cand); n_coarse += __popc(bits); }

#if QGS_FWD_STAGE_GEO
        __pipeline_wait_prior(0);
        __syncwarp();
#endif

        // pass 2: exact test, ring and compositing in stream order
#if QGS_FWD_RAY_REGS
        const double d[3] = {ray64[0], ray64[1], ray64[2]};
#else
        const double d[3] = {sm.d64[0][lane], sm.d64[1][lane], sm.d64[2][lane]};
#endif
        auto exact = [&](int j, Hit &h) -> bool {
#if QGS_FWD_STAGE_GEO
            const Geo64 &gh = *reinterpret_cast<const Geo64 *>(&sm.geoh[j]);   // head only
#else
            const Geo64 &gh = geo[sm.qprim[j]];
#endif
            const PrimRec &r = sm.rec[j];
            const Geo64 *gfull = geo + sm.qprim[j];
            return hit_exact_from<M>(r, gh, gfull, d, dx, dy, dz, c.euclid, c.t_clip,
                                     sm.tfirst[j][lane], (secb >> j) & 1u, (margb >> j) & 1u, h) &&
                   alpha_pass<M>(r, gfull, d, h, c.euclid, c.alpha_floor);
        };
        auto accept_one = [&](int j, const Hit &h) {
            const int p = sm.qprim[j];
            const PrimRec &r = sm.rec[j];
            const float abar = r.alpha * h.G;
            n_acc++;
            // fragment payload now, so compositing never re-shades (raster_kernels.py:58-80)
            Pay pin;
            pin.v[0] = abar > c.alpha_clamp ? -c.alpha_clamp : abar;
#if QGS_PAY_XY
            pin.v[1] = h.x;
            pin.v[2] = h.y;
#else
            {
                float nl[3], nc[3], K, inrm, flip;
                normal_curv32(r, h, dx, dy, dz, nl, nc, K, inrm, flip);
                pin.v[1] = nc[0]; pin.v[2] = nc[1]; pin.v[3] = nc[2]; pin.v[4] = K;
            }
#endif
            double et;
            int ep;
            Pay pout;
            bool emit;
            if (!c.resort) { et = h.t64; ep = p; pout = pin; emit = true; }
            else emit = ring_push_pay(R, sm.pay, lane, h.t64, p, pin, et, ep, pout);
            if (emit) composite(ep, et, pout);
        };
#if QGS_UTIL_COUNTERS
        u_p2 += __reduce_max_sync(FULL, alive ? (unsigned)__popc(bits) : 0u);
#endif
        while (bits && alive) {
            const int j = __ffs(bits) - 1;
            bits &= bits - 1;
            Hit h;
            if (exact(j, h)) accept_one(j, h);
        }
        __syncwarp();
    };

    // Pass 0, two levels, both in stream order.  (a) The tile's depth-sorted
    // list is streamed 32 entries per window, one per lane: the entry's
    // culled pixel box (ConicRec) against the block and the live pixels;
    // overlapping entries join queue A.  (b) Every 32 entries of queue A are
    // conic-tested on all 32 block pixels, one entry per lane; entries that
    // keep a pixel join queue B, and every WB entries of queue B run as one
    // batch.
    const int start = tile_offsets[tile], end = tile_offsets[tile + 1];
    int qn = 0, an = 0;
    auto drain_b = [&]() {
        while (qn >= WB) {
            run_batch(WB);
            qn -= WB;
            // shift the queue down by WB (overlapping ranges: read, sync, write)
            int qp = 0;
            uint32_t qm = 0u;
            if (lane < qn) { qp = sm.qprim[WB + lane]; qm = sm.qmask[WB + lane]; }
            __syncwarp();
            if (lane < qn) { sm.qprim[lane] = qp; sm.qmask[lane] = qm; }
            __syncwarp();
            if (!__any_sync(FULL, alive)) { qn = 0; an = 0; return false; }
        }
        return true;
    };
    auto conic_pass = [&](int na) {            // queue A entries [0, na) -> queue B
        const uint32_t live = __ballot_sync(FULL, alive);
        uint32_t m = 0u;
        int pj = 0;
        if (lane < na) {
            pj = sm.aprim[lane];
            m = sm.amask[lane] & live;
            if (m && cull) m &= conic_rows<4>(conics[pj], bu, bv, 0);
        }
        const uint32_t keep = __ballot_sync(FULL, m != 0u);
        if (m) {
            const int pos = qn + __popc(keep & ((1u << lane) - 1u));
            QGS_CHECK(pos < WB + 32);
            sm.qprim[pos] = pj;
            sm.qmask[pos] = m;
        }
        qn += __popc(keep);
        __syncwarp();
    };
#if QGS_FWD_LIST_PREFETCH
    // list windows software-pipelined: the ids of window w+2 and the culled
    // boxes of window w+1 are in flight while window w is processed
    auto ld_id = [&](int b) { return b + lane < end ? __ldg(tile_prims + b + lane) : 0; };
    auto ld_bb = [&](int b, int p) {
        return (cull && b + lane < end) ? __ldg(reinterpret_cast<const uint2 *>(&conics[p].bb_u))
                                        : make_uint2(0u, 0u);
    };
    int id1 = ld_id(start), id2 = ld_id(start + 32);
    uint2 bb1 = ld_bb(start, id1);
#endif
    for (int b0 = start; b0 < end; b0 += 32) {
        const uint32_t live = __ballot_sync(FULL, alive);
        if (!live) break;
        const int nb = min(32, end - b0);
        int pj = 0;
        uint32_t bm = 0u;
#if QGS_FWD_LIST_PREFETCH
        const int pcur = id1;
        const uint2 bcur = bb1;
        id1 = id2;
        bb1 = ld_bb(b0 + 32, id1);
        id2 = ld_id(b0 + 64);
#endif
        if (lane < nb) {
#if QGS_FWD_LIST_PREFETCH
            pj = pcur;
            if (cull) {
                bm = block_lanes(bcur.x, bcur.y, bu, bv);
            } else {
#else
            pj = tile_prims[b0 + lane];
            if (cull) {
                const uint2 bb = *reinterpret_cast<const uint2 *>(&conics[pj].bb_u);
                bm = block_lanes(bb.x, bb.y, bu, bv);
            } else {
#endif
                bm = block_lanes(recs[pj].bb_u, recs[pj].bb_v, bu, bv);
            }
            if (out.counters)                  // algorithmic work: the reference's pixel box
                sm.boxw[lane] = cull ? block_lanes(recs[pj].bb_u, recs[pj].bb_v, bu, bv) : bm;
            bm &= live;
        }
        if (out.counters) {
            __syncwarp();
            for (int j = 0; j < nb; ++j) n_box += alive ? (sm.boxw[j] >> lane) & 1u : 0u;
            __syncwarp();
        }
        const uint32_t keep = __ballot_sync(FULL, bm != 0u);
        if (bm) {
            const int pos = an + __popc(keep & ((1u << lane) - 1u));
            QGS_CHECK(pos < 64);
            sm.aprim[pos] = pj;
            sm.amask[pos] = bm;
        }
        an += __popc(keep);
        __syncwarp();
        if (an >= 32) {
            conic_pass(32);
            an -= 32;
            if (lane < an) { sm.aprim[lane] = sm.aprim[32 + lane]; sm.amask[lane] = sm.amask[32 + lane]; }
            __syncwarp();
            if (!drain_b()) break;
        }
    }
    if (an > 0 && __any_sync(FULL, alive)) {
        conic_pass(an);
        drain_b();
    }
    if (qn > 0 && __any_sync(FULL, alive)) run_batch(qn);

    ensure_pages(RING);                      // the drain emits at most RING more
    while (alive && R.n > 0) {               // raster_kernels.py:227-270
        double et;
        int ep;
        Pay pout;
        ring_pop_pay(R, sm.pay, lane, et, ep, pout);
        composite(ep, et, pout);
    }
    if (out.frag_page_count) {
        if (lane < npages) out.frag_page_table[(size_t)rw * QGS_FRAG_MAX_PAGES + lane] = sm.pages[lane];
        if (lane == 0) out.frag_page_count[rw] = (out.frag_prim && log_on) ? npages : -1;
    }

    if (inside) {
        const int W = cam.W, npx = cam.W * cam.H, px = v * W + u;
        const double ac0 = sm.acc[A_C0][lane], ac1 = sm.acc[A_C0 + 1][lane],
                     ac2 = sm.acc[A_C0 + 2][lane], aa = sm.acc[A_A][lane],
                     ad = sm.acc[A_D][lane], ad2 = sm.acc[A_D2][lane],
                     an0 = sm.acc[A_N0][lane], an1 = sm.acc[A_N0 + 1][lane],
                     an2 = sm.acc[A_N0 + 2][lane], ak = sm.acc[A_K][lane],
                     adist = sm.acc[A_DIST][lane];
        out.color_raw[3 * px + 0] = (float)ac0;
        out.color_raw[3 * px + 1] = (float)ac1;
        out.color_raw[3 * px + 2] = (float)ac2;
        out.color[3 * px + 0] = (float)(ac0 + T * st.bg[0]);
        out.color[3 * px + 1] = (float)(ac1 + T * st.bg[1]);
        out.color[3 * px + 2] = (float)(ac2 + T * st.bg[2]);
        out.alpha[px] = (float)aa;
        out.depth[px] = (float)ad;
        out.depth_sq[px] = (float)ad2;
        out.depth_median[px] = median;
        out.normal[3 * px + 0] = (float)an0;
        out.normal[3 * px + 1] = (float)an1;
        out.normal[3 * px + 2] = (float)an2;
        out.curvature[px] = (float)ak;
        out.distortion[px] = (float)adist;
        out.transmittance[px] = (float)T;
        out.n_fragments[px] = nfrag;
        if (out.aux) {
            double *a = out.aux;
            a[(AX_C0 + 0) * (size_t)npx + px] = ac0;
            a[(AX_C0 + 1) * (size_t)npx + px] = ac1;
            a[(AX_C0 + 2) * (size_t)npx + px] = ac2;
            a[AX_A * (size_t)npx + px] = aa;
            a[AX_D * (size_t)npx + px] = ad;
            a[AX_D2 * (size_t)npx + px] = ad2;
            a[(AX_N0 + 0) * (size_t)npx + px] = an0;
            a[(AX_N0 + 1) * (size_t)npx + px] = an1;
            a[(AX_N0 + 2) * (size_t)npx + px] = an2;
            a[AX_K * (size_t)npx + px] = ak;
            a[AX_DIST * (size_t)npx + px] = adist;
            a[AX_T * (size_t)npx + px] = T;
        }
    }
    // per-tile violations and the work counters
    for (int o = 16; o; o >>= 1) {
        viol += __shfl_xor_sync(FULL, viol, o);
        n_box += __shfl_xor_sync(FULL, n_box, o);
        n_acc += __shfl_xor_sync(FULL, n_acc, o);
        n_cand += __shfl_xor_sync(FULL, n_cand, o);
        n_coarse += __shfl_xor_sync(FULL, n_coarse, o);
        nfrag += __shfl_xor_sync(FULL, nfrag, o);
    }
    if (lane == 0) {
        if (out.violations) atomicAdd(&out.violations[tile], viol);
        if (out.counters) {
            atomicAdd(&out.counters[0], (unsigned long long)n_box);
            atomicAdd(&out.counters[1], (unsigned long long)n_acc);
            atomicAdd(&out.counters[2], (unsigned long long)nfrag);
            atomicAdd(&out.counters[3], (unsigned long long)n_cand);
            atomicAdd(&out.counters[4], (unsigned long long)n_coarse);
#if QGS_UTIL_COUNTERS
            atomicAdd(&out.counters[5], 32ull * u_p1);     // lane slots of pass 1 (per candidate)
            atomicAdd(&out.counters[6], 32ull * u_p2);     // lane slots of pass 2
#endif
        }
    }
}

__global__ void __launch_bounds__(32 * FWD_WPC, QGS_FWD_MIN_BLOCKS / FWD_WPC)
raster_fwd_kernel(const PrimRec *__restrict__ recs, const Geo64 *__restrict__ geo,
                  const ConicRec *__restrict__ conics, const int32_t *__restrict__ tile_offsets,
                  const int32_t *__restrict__ tile_prims, CamK cam, SetK st, qgs_targets out)
{
    fwd_block<MODE_FAST>(recs, geo, conics, tile_offsets, tile_prims, cam, st, out, -1);
}

#ifdef QGS_FWD_EXACT_MAXNREG
__global__ void __maxnreg__(QGS_FWD_EXACT_MAXNREG)
#else
__global__ void __launch_bounds__(32 * FWD_WPC, QGS_FWD_EXACT_MIN_BLOCKS / FWD_WPC)
#endif
raster_fwd_exact_kernel(const PrimRec *__restrict__ recs, const Geo64 *__restrict__ geo,
                        const ConicRec *__restrict__ conics, const int32_t *__restrict__ tile_offsets,
                        const int32_t *__restrict__ tile_prims, CamK cam, SetK st, qgs_targets out)
{
    fwd_block<MODE_EXACT>(recs, geo, conics, tile_offsets, tile_prims, cam, st, out, -1);
}

// =============================================================== backward

struct Up {
    float c0, c1, c2, a, d, n0, n1, n2, k, dist;
};

// _grad_fragment (raster_kernels.py:289-502) for one emitted fragment, fp32,
// with Nmat^T folded into the M slots and lambda into the s / w slots.
__device__ __forceinline__ void frag_grad(const PrimRec &r, const Frag &f, float dx, float dy,
                                          float dz, float w, float g_abar, float tdev,
                                          const Up &up, bool euclid, float g[KG])
{
    const Hit &h = f.h;
    const float t = h.t, x = h.x, y = h.y, rho = h.rho, cth = h.cth, sth = h.sth;
    g[KG_COLOR + 0] = w * up.c0;
    g[KG_COLOR + 1] = w * up.c1;
    g[KG_COLOR + 2] = w * up.c2;
    float g_t = up.d * w + up.dist * 2.f * w * tdev;
    float gcx = w * up.n0, gcy = w * up.n1, gcz = w * up.n2;
    float g_K = w * up.k;
    float g_G = 0.f;
    g[KG_ALPHA] = 0.f;
    if (!f.clamped) {
        g[KG_ALPHA] = g_abar * h.G;
        g_G = g_abar * r.alpha;
    }
    const float sig = h.sig, l = h.l;
    const float isig2 = 1.f / (sig * sig);
    const float g_l = g_G * h.G * (-l * isig2);
    const float g_sig = g_G * h.G * (l * l * isig2 / sig);
    // sigma(s1, s2, cth, sth) (geodesic.py:62-71)
    const float s1 = r.s1, s2 = r.s2, s3 = r.s3;
    const float m = fmaf(s2 * cth, s2 * cth, (s1 * sth) * (s1 * sth));
    const float im = 1.f / m;
    g[KG_S + 0] = g_sig * sig * (1.f / s1 - s1 * sth * sth * im);
    g[KG_S + 1] = g_sig * sig * (1.f / s2 - s2 * cth * cth * im);
    float g_cth = g_sig * (-sig * s2 * s2 * cth * im);
    float g_sth = g_sig * (-sig * s1 * s1 * sth * im);
    float g_x = 0.f, g_y = 0.f, g_rho = 0.f, g_a = 0.f;
    if (euclid || h.branch == BR_PLANAR) {
        g_rho = g_l;
    } else {
        float dla, dlr;
        arc32_grad(h.a, rho, l, dla, dlr);
        g_a = g_l * dla;
        g_rho = g_l * dlr;
    }
    float g_w1 = 0.f, g_w2 = 0.f, g_iw3 = 0.f;
    float g_nl[3];            // d L / d (local unit normal), = flip * M * g_nc
    {
        const float fl = f.flip;
        g_nl[0] = fl * fmaf(r.M[0], gcx, fmaf(r.M[1], gcy, r.M[2] * gcz));
        g_nl[1] = fl * fmaf(r.M[3], gcx, fmaf(r.M[4], gcy, r.M[5] * gcz));
        g_nl[2] = fl * fmaf(r.M[6], gcx, fmaf(r.M[7], gcy, r.M[8] * gcz));
    }
    if (h.branch != BR_PLANAR) {
        const float w1 = r.w1, w2 = r.w2;
        float gs3 = g_a * fmaf(w1 * cth, cth, w2 * sth * sth);
        g_w1 = g_a * s3 * cth * cth;
        g_w2 = g_a * s3 * sth * sth;
        g_cth += g_a * 2.f * s3 * w1 * cth;
        g_sth += g_a * 2.f * s3 * w2 * sth;
        // curvature K(lam1, lam2, x, y) (surface.py:27-32)
        const float l1 = r.lam1, l2 = r.lam2;
        const float den = 1.f + 4.f * (l1 * l1 * x * x + l2 * l2 * y * y);
        const float iden = 1.f / den, iden2 = iden * iden, iden3 = iden2 * iden;
        const float g_l1 = g_K * (4.f * l2 * iden2 - 64.f * l1 * l1 * l2 * x * x * iden3);
        const float g_l2 = g_K * (4.f * l1 * iden2 - 64.f * l1 * l2 * l2 * y * y * iden3);
        g_x += g_K * (-16.f * f.K * l1 * l1 * x * iden);
        g_y += g_K * (-16.f * f.K * l2 * l2 * y * iden);
        // lambda_k = s3 w_k folded in (rasterizer.py:290-293)
        gs3 += g_l1 * w1 + g_l2 * w2;
        g_w1 += g_l1 * s3;
        g_w2 += g_l2 * s3;
        g[KG_S + 2] = gs3;
        // through the normalisation of ntilde = (2 w1 x, 2 w2 y, -iw3)
        const float dot = fmaf(f.nl[0], g_nl[0], fmaf(f.nl[1], g_nl[1], f.nl[2] * g_nl[2]));
        const float g_ntx = (g_nl[0] - f.nl[0] * dot) * f.inrm;
        const float g_nty = (g_nl[1] - f.nl[1] * dot) * f.inrm;
        const float g_ntz = (g_nl[2] - f.nl[2] * dot) * f.inrm;
        g_w1 += 2.f * x * g_ntx;
        g_x += 2.f * w1 * g_ntx;
        g_w2 += 2.f * y * g_nty;
        g_y += 2.f * w2 * g_nty;
        g_iw3 += -g_ntz;
    } else {
        g[KG_S + 2] = 0.f;
    }
    // polar coordinates of the hit
    if (rho > 1e-12f) {
        const float ir = 1.f / rho;
        g_x += (g_cth * sth * sth - g_sth * cth * sth) * ir;
        g_y += (-g_cth * cth * sth + g_sth * cth * cth) * ir;
    }
    g_x += g_rho * cth;
    g_y += g_rho * sth;
    // Hit point x = ohat + t dhat and the root t(ohat, dhat, w): the
    // reference's gA dh^2 + gB 2 o dh + gC o^2 (raster_kernels.py:464-482)
    // collapses exactly to the point form k x^2 with k = -g_tt / F'(t); the
    // point form keeps fp32 accuracy (the polynomial form cancels terms
    // ~|o|^2 down to ~x^2).
    const float hx = h.dhx, hy = h.dhy, hz = h.dhz;
    const float g_tt = g_t + g_x * hx + g_y * hy;
    const float k = -g_tt / h.q;
    float go[3], dl[3] = {0.f, 0.f, 0.f};   // d L / d ohat; dhat term beyond t * go
    if (h.branch == BR_PLANAR) {
        go[0] = g_x; go[1] = g_y; go[2] = k;     // F = oz + t dhz
    } else {
        const float w1 = r.w1, w2 = r.w2, iw3 = r.iw3;
        go[0] = g_x + k * 2.f * w1 * x;
        go[1] = g_y + k * 2.f * w2 * y;
        go[2] = -k * iw3;
        if (h.branch == BR_LINEAR) {
            // t = -C/B ignores A: dhat gets t*(2 w o) instead of t*(2 w x)
            g_w1 += k * (x * x - t * t * hx * hx);
            g_w2 += k * (y * y - t * t * hy * hy);
            dl[0] = -k * t * t * 2.f * w1 * hx;
            dl[1] = -k * t * t * 2.f * w2 * hy;
        } else {
            g_w1 += k * x * x;
            g_w2 += k * y * y;
        }
        g_iw3 += -k * h.z;
    }
    g[KG_W + 0] = g_w1;
    g[KG_W + 1] = g_w2;
    g[KG_W + 2] = g_iw3;
    g[KG_OHAT + 0] = go[0];
    g[KG_OHAT + 1] = go[1];
    g[KG_OHAT + 2] = go[2];
    // The chain's rotation gradient is g_R = R X with the local-frame
    // accumulator X = x_loc (x) g_ohat + dhat (x) dl + g_nl (x) nl (no
    // cancellation between the ohat and M = R^T R_cw paths, which are each
    // ~|eye - c| / |x| larger than it).  The quaternion gradient of R(q/|q|)
    // sees only the skew part of X (its symmetric part moves along q, which
    // the normalisation projects out), so only
    // omega = (X12 - X21, X20 - X02, X01 - X10) = x_loc x g_ohat + dhat x dl + g_nl x nl
    // is accumulated.
    const float xl[3] = {x, y, h.z}, dh3[3] = {hx, hy, hz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int j = (a + 1) % 3, b = (a + 2) % 3;
        g[KG_ROT + a] = fmaf(xl[j], go[b], -xl[b] * go[j]) + fmaf(dh3[j], dl[b], -dh3[b] * dl[j]) +
                        fmaf(g_nl[j], f.nl[b], -g_nl[b] * f.nl[j]);
    }
    (void)dx; (void)dy; (void)dz;
}

// Sum the slots of lanes that emitted the same primitive and add each sum to
// the primitive's kernel-gradient row.  A lane alone with its primitive adds
// its row directly (four 16-byte vector atomics, red.global.add.v4.f32);
// larger groups put their rows in shared memory and are served eight at a
// time: lane = 4 * set + q sums float4 slot q (slots 4q .. 4q+3) of the
// set-th group over its members and issues one vector atomic, so a group
// costs four atomics whatever its size.  The groups' leaders are listed by
// rank in shared memory (QGS_RED_RANKS): a lane set reads its leader instead
// of an 8-step find-first-set scan per round (backward 5.71 -> 5.38 ms).
__device__ __forceinline__ void warp_accumulate(float (*red)[33][KGP], int *lead, bool emit,
                                                int prim, const float g[KG],
                                                float *__restrict__ kg)
{
    const int lane = threadIdx.x & 31, w = 0;   // red: this warp's own buffer
    const unsigned key = emit ? (unsigned)prim : 0xffffffffu;
    const unsigned peers = __match_any_sync(FULL, key);
#if QGS_RED_SINGLES
    // a lane alone with its primitive adds its row directly
    const bool single = emit && peers == (1u << lane);
    if (single) {
        float4 *dst = reinterpret_cast<float4 *>(kg + (size_t)prim * KG);
#pragma unroll
        for (int q = 0; q < KG / 4; ++q)
            atomicAdd(dst + q, make_float4(g[4 * q], g[4 * q + 1], g[4 * q + 2], g[4 * q + 3]));
    }
    const bool shared_grp = emit && !single;
#else
    const bool shared_grp = emit;
#endif
    if (shared_grp) {
        float4 *dst = reinterpret_cast<float4 *>(red[w][lane]);
#pragma unroll
        for (int q = 0; q < KG / 4; ++q) dst[q] = make_float4(g[4 * q], g[4 * q + 1], g[4 * q + 2], g[4 * q + 3]);
    }
    const bool is_leader = shared_grp && (peers & ((1u << lane) - 1u)) == 0;
    unsigned leaders = __ballot_sync(FULL, is_leader);
#if QGS_RED_RANKS
    if (is_leader) lead[__popc(leaders & ((1u << lane) - 1u))] = lane;
#endif
    __syncwarp();
#if QGS_RED_SETS == 16
    // sixteen sets of 2 lanes, each lane two float4 slots (q, q + 2)
    const int set = lane >> 1, q = lane & 1;
    constexpr int NSET = 16;
#else
    // eight sets of 4 lanes, each lane one float4 slot
    const int set = lane >> 2, q = lane & 3;
    constexpr int NSET = 8;
#endif
    const float4 (*red4)[KGP / 4] = reinterpret_cast<const float4 (*)[KGP / 4]>(red[w]);
#if QGS_RED_RANKS
    const int n_lead = __popc(leaders);
    for (int base = 0; base < n_lead; base += NSET) {
        // leaders base .. base + NSET - 1 in lane order, one per lane set
        const int ld = base + set < n_lead ? lead[base + set] : -1;
#else
    while (leaders) {
        // the NSET lowest pending leaders (warp-uniform), one per lane set
        int ld = -1;
#pragma unroll
        for (int k = 0; k < NSET; ++k) {
            const int lk = leaders ? __ffs(leaders) - 1 : -1;
            ld = set == k ? lk : ld;
            leaders &= leaders - 1;
        }
#endif
        const unsigned grp = __shfl_sync(FULL, peers, ld < 0 ? 0 : ld);
        const int gp = __shfl_sync(FULL, prim, ld < 0 ? 0 : ld);
        if (ld >= 0) {
#if QGS_RED_SETS == 16
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
            for (unsigned mm = grp; mm; mm &= mm - 1) {
                const int i0 = __ffs(mm) - 1;
                const float4 x = red4[i0][q], y = red4[i0][q + 2];
                a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
                b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
            }
            float4 *dst = reinterpret_cast<float4 *>(kg + (size_t)gp * KG);
            atomicAdd(dst + q, a);
            atomicAdd(dst + q + 2, b);
#else
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
            for (unsigned mm = grp; mm;) {             // two independent partial sums
                const int i0 = __ffs(mm) - 1; mm &= mm - 1;
                const int i1 = mm ? __ffs(mm) - 1 : 32; mm &= mm - 1;
                const float4 x = red4[i0][q], y = red4[i1][q];
                a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
                b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
            }
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
            atomicAdd(reinterpret_cast<float4 *>(kg + (size_t)gp * KG) + q, a);
#endif
        }
    }
    __syncwarp();
}

// One raster block of the backward.  REPLAY = false: blocks with a fragment
// log (the hot kernel: no candidate-test code in it); true: blocks without
// one, replayed with the forward's candidate test (EXACT: the forward's
// decision mode).  DET: write rows for the deterministic reduction
// (det_reduce.cu) instead of atomics.
template <bool EXACT, bool DET, bool REPLAY>
__device__ __forceinline__ void bwd_block(const PrimRec *__restrict__ recs,
                                          const Geo64 *__restrict__ geo,
                                          const int32_t *__restrict__ tile_offsets,
                                          const int32_t *__restrict__ tile_prims, const CamK &cam,
                                          const SetK &st, const qgs_targets &fwd,
                                          const qgs_upstream &upst, float *__restrict__ kg,
                                          const DetRows &det, int slot = -1)
{
    // one BwdSmem per warp (dynamic shared memory: QGS_BWD_WPC warps per CTA;
    // the replay kernel: one warp per CTA)
    extern __shared__ __align__(16) unsigned char raster_smem[];
    BwdSmem &sm = reinterpret_cast<BwdSmem *>(raster_smem)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    if (lane < KG) sm.red[0][32][lane] = 0.f;        // zero row for padded group sums
    __syncwarp();
    int tile, blk, u, v;
    block_pixel(cam.tiles_x, fwd.tile_order, tile, blk, u, v, slot);
    const int rw = (tile << 3) | blk;                // raster warp id (fragment-log row)
    const bool inside = u < cam.W && v < cam.H;
    const Cfg c = make_cfg(st);
    const int npx = cam.W * cam.H, px = inside ? v * cam.W + u : 0;

    Up up = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (inside) {
        if (upst.color) { up.c0 = upst.color[3 * px]; up.c1 = upst.color[3 * px + 1]; up.c2 = upst.color[3 * px + 2]; }
        if (upst.alpha) up.a = upst.alpha[px];
        if (upst.depth) up.d = upst.depth[px];
        if (upst.normal) { up.n0 = upst.normal[3 * px]; up.n1 = upst.normal[3 * px + 1]; up.n2 = upst.normal[3 * px + 2]; }
        if (upst.curvature) up.k = upst.curvature[px];
        if (upst.distortion) up.dist = upst.distortion[px];
    }
    // raster_kernels.py:537-540: pixels without upstream contribute nothing
    const bool has_up = up.c0 != 0.f || up.c1 != 0.f || up.c2 != 0.f || up.a != 0.f ||
                        up.d != 0.f || up.n0 != 0.f || up.n1 != 0.f || up.n2 != 0.f ||
                        up.k != 0.f || up.dist != 0.f;
    // colour gradient reaches the composited colour incl. background
    // (rasterizer.py:246-250): u_alpha -= u_color . bg
    const double ua64 = (double)up.a - ((double)up.c0 * st.bg[0] + (double)up.c1 * st.bg[1] +
                                        (double)up.c2 * st.bg[2]);
    up.a = (float)ua64;

    double d64[3] = {0.0, 0.0, 1.0};
    if (inside) pixel_dir64(cam, u, v, d64);
    const float dx = (float)d64[0], dy = (float)d64[1], dz = (float)d64[2];
    double F0 = 0, F1 = 0, F2 = 0, vtot = 0;
    if (inside && has_up) {
        const double *a = fwd.aux;
        F0 = a[AX_A * (size_t)npx + px];
        F1 = a[AX_D * (size_t)npx + px];
        F2 = a[AX_D2 * (size_t)npx + px];
        vtot = (double)up.c0 * a[(AX_C0 + 0) * (size_t)npx + px] +
               (double)up.c1 * a[(AX_C0 + 1) * (size_t)npx + px] +
               (double)up.c2 * a[(AX_C0 + 2) * (size_t)npx + px] + ua64 * F0 +
               (double)up.d * F1 + (double)up.n0 * a[(AX_N0 + 0) * (size_t)npx + px] +
               (double)up.n1 * a[(AX_N0 + 1) * (size_t)npx + px] +
               (double)up.n2 * a[(AX_N0 + 2) * (size_t)npx + px] +
               (double)up.k * a[AX_K * (size_t)npx + px] +
               (double)up.dist * 2.0 * a[AX_DIST * (size_t)npx + px];
    }
    double T = 1.0, pref = 0.0;
    Ring R{&sm.ring_t[0][lane], &sm.ring_p[0][lane], 0};
    bool alive = inside && has_up;

    // deterministic mode: this pixel's k-th fragment owns row det_base + k
    const int64_t det_base = DET ? det.base[(size_t)rw * 32 + lane] : 0;
    int kf = 0;
#if QGS_DEBUG_CHECKS
    const int nf_of_pixel = inside ? fwd.n_fragments[px] : 0;
#endif
    // replay: the pixel stops after the forward's fragment count (its
    // termination decision may have been made on the float64 transmittance)
    int n_left = 0;
    if (REPLAY && alive) {
        n_left = fwd.n_fragments[px];
        alive = n_left > 0;
    }
    auto emit_grad = [&](bool emit, int ep, double t, bool have_xy, float lx, float ly,
                         const PrimRec *staged) {
        float g[KG];
        if (emit) {
            Frag f;
#if QGS_BWD_VEC_LOADS
            // whole records in flight at once (16-byte loads) rather than
            // field by field as the arithmetic reaches them
            const PrimRec r = staged ? *staged : load_rec(recs + ep);
#else
            const PrimRec &r = staged ? *staged : recs[ep];
#endif
            if (have_xy && shade_from_log(r, lx, ly, t, dx, dy, dz, c.euclid, f.h)) {
                finish_frag(r, dx, dy, dz, c, f);      // logged hit point: fp32 re-shade
            } else {
#if QGS_BWD_VEC_LOADS
                const Geo64 gh = load_geo_head(geo + ep);
#else
                const Geo64 &gh = geo[ep];
#endif
                shade_emitted(r, gh, d64, dx, dy, dz, t, c, f);
            }
            const double w = f.abar64 * T;
            // the upstream-weighted value of the fragment, summed as a balanced
            // tree (a 4-deep instead of a 10-deep float64 dependency chain)
            const double V =
                (((double)up.c0 * r.col[0] + (double)up.c1 * r.col[1]) +
                 ((double)up.c2 * r.col[2] + ua64)) +
                (((double)up.d * t + (double)up.n0 * f.nc[0]) +
                 ((double)up.n1 * f.nc[1] + (double)up.n2 * f.nc[2])) +
                ((double)up.k * f.K + (double)up.dist * (t * t * F0 - 2.0 * t * F1 + F2));
            pref += w * V;
            const float g_abar = (float)(T * V) - (float)(vtot - pref) / (float)(1.0 - f.abar64);
            frag_grad(r, f, dx, dy, dz, (float)w, g_abar, (float)(t * F0 - F1), up, c.euclid, g);
            T *= 1.0 - f.abar64;
            if (REPLAY ? --n_left == 0 : T < c.t_term) alive = false;
        }
        if (DET) {
            if (emit) {
                float4 *dst = reinterpret_cast<float4 *>(det.rows + (size_t)(det_base + kf) * KG);
#pragma unroll
                for (int q = 0; q < KG / 4; ++q)
                    dst[q] = make_float4(g[4 * q], g[4 * q + 1], g[4 * q + 2], g[4 * q + 3]);
                QGS_CHECK(ep >= 0 && kf < nf_of_pixel);
                det.prim[det_base + kf] = ep;
                kf++;
            }
            return;
        }
        warp_accumulate(sm.red, sm.lead, emit, ep, g, kg);
    };

    // Fragment log written by the forward: the composited sequence of every
    // pixel, so no candidate is re-tested and no ring is replayed.
    {
        const int np = (fwd.frag_prim && fwd.frag_t && fwd.frag_page_count)
                           ? fwd.frag_page_count[rw] : -1;
        if (REPLAY && np >= 0) return;            // the log kernel has it
        if (!REPLAY && np < 0) return;            // the replay kernel has it
        if (!REPLAY) {
            const int nf = alive ? fwd.n_fragments[px] : 0;
            const int nf_max = __reduce_max_sync(FULL, nf);
            // lane i holds the warp's i-th page id
            QGS_CHECK(np <= QGS_FRAG_MAX_PAGES && nf_max <= np * QGS_FRAG_PAGE);
            const int my_page = lane < np ? fwd.frag_page_table[(size_t)rw * QGS_FRAG_MAX_PAGES + lane] : 0;
            auto slot = [&](int k) {
                const int pg = __shfl_sync(FULL, my_page, k / QGS_FRAG_PAGE);
                return ((size_t)pg * QGS_FRAG_PAGE + (k % QGS_FRAG_PAGE)) * 32 + lane;
            };
            const float2 *xy = reinterpret_cast<const float2 *>(fwd.frag_xy);
            const bool have_xy = xy != nullptr;
            int np_ = -1;
            double nt_ = 0.0;
            float2 nxy = make_float2(0.f, 0.f);
            if (nf_max > 0) {
                const size_t o = slot(0);
                if (0 < nf) {
                    np_ = fwd.frag_prim[o]; nt_ = fwd.frag_t[o];
                    if (have_xy) nxy = xy[o];
                }
            }
            for (int k = 0; k < nf_max; ++k) {
                const bool emit = k < nf;
                const int ep = np_;
                const double et = nt_;
                const float2 exy = nxy;
                if (k + 1 < nf_max) {            // prefetch the next fragment
                    const size_t o = slot(k + 1);
                    if (k + 1 < nf) {
                        np_ = fwd.frag_prim[o];
                        nt_ = fwd.frag_t[o];
                        if (have_xy) nxy = xy[o];
                    }
                }
                emit_grad(emit, ep, et, have_xy, exy.x, exy.y, nullptr);
            }
            return;
        }
    }

    // No log (or the block's log overflowed its pages): replay the block's
    // stream with the full candidate test -- the same inline functions as the
    // forward, so the same accepted set, fp64 depths and ring decisions.
    const int start = tile_offsets[tile], end = tile_offsets[tile + 1];
    for (int b0 = start; b0 < end; b0 += WB) {
        if (!__any_sync(FULL, alive)) break;
        const int nb = min(WB, end - b0);
        load_batch32(sm.rec, sm.prim, recs, tile_prims, b0, nb);
        for (int j = 0; j < nb; ++j) {
            if (!__any_sync(FULL, alive)) break;
            double et = 0.0;
            int ep = -1;
            bool emit = false;
            if (alive && in_box(sm.rec[j], u, v)) {
                const int p = sm.prim[j];
                double t = 0.0;
                if (accept<EXACT ? MODE_EXACT : MODE_FAST>(sm.rec[j], geo[p], d64, dx, dy, dz, c, t))
                    emit = ring_step(c, R, t, p, et, ep);
            }
            if (__any_sync(FULL, emit)) emit_grad(emit, ep, et, false, 0.f, 0.f, nullptr);
        }
        __syncwarp();
    }
    while (__any_sync(FULL, alive && R.n > 0)) {
        double et = 0.0;
        int ep = -1;
        bool emit = alive && R.n > 0;
        if (emit) ring_pop(R, et, ep);
        emit_grad(emit, ep, et, false, 0.f, 0.f, nullptr);
    }
}

__global__ void __launch_bounds__(32 * BWD_WPC, QGS_BWD_MIN_BLOCKS / BWD_WPC)
raster_bwd_kernel(const PrimRec *__restrict__ recs, const Geo64 *__restrict__ geo,
                  const int32_t *__restrict__ tile_offsets,
                  const int32_t *__restrict__ tile_prims, CamK cam, SetK st, qgs_targets fwd,
                  qgs_upstream upst, float *__restrict__ kg, DetRows det)
{
    bwd_block<false, false, false>(recs, geo, tile_offsets, tile_prims, cam, st, fwd, upst, kg, det);
}

// blocks without a fragment log (rare: a page pool that ran dry, or a
// forward called without a log): replayed with the forward's decision mode.
// A small persistent grid scans the slots 32 at a time (page count < 0).
template <bool DET>
__device__ __forceinline__ void bwd_replay_slots(const PrimRec *__restrict__ recs,
                                                 const Geo64 *__restrict__ geo,
                                                 const int32_t *__restrict__ tile_offsets,
                                                 const int32_t *__restrict__ tile_prims,
                                                 const CamK &cam, const SetK &st,
                                                 const qgs_targets &fwd, const qgs_upstream &upst,
                                                 float *__restrict__ kg, const DetRows &det)
{
    const int lane = threadIdx.x & 31;
    const int n_slots = cam.tiles_x * cam.tiles_y * 8;
    const bool logged = fwd.frag_prim && fwd.frag_t && fwd.frag_page_count;
    for (int base = blockIdx.x * 32; base < n_slots; base += gridDim.x * 32) {
        // slot -> tile's raster warp id: the page count is indexed by warp id
        int rw = -1;
        if (base + lane < n_slots) {
            const int t = fwd.tile_order ? fwd.tile_order[(base + lane) >> 3] : (base + lane) >> 3;
            rw = (t << 3) | ((base + lane) & 7);
        }
        unsigned todo = __ballot_sync(FULL, rw >= 0 && (!logged || fwd.frag_page_count[rw] < 0));
        while (todo) {
            const int k = __ffs(todo) - 1;
            todo &= todo - 1;
            if (st.exact)
                bwd_block<true, DET, true>(recs, geo, tile_offsets, tile_prims, cam, st, fwd, upst,
                                           kg, det, base + k);
            else
                bwd_block<false, DET, true>(recs, geo, tile_offsets, tile_prims, cam, st, fwd,
                                            upst, kg, det, base + k);
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(32, 8)
raster_bwd_replay_kernel(const PrimRec *__restrict__ recs, const Geo64 *__restrict__ geo,
                         const int32_t *__restrict__ tile_offsets,
                         const int32_t *__restrict__ tile_prims, CamK cam, SetK st,
                         qgs_targets fwd, qgs_upstream upst, float *__restrict__ kg, DetRows det)
{
    if (det.rows) bwd_replay_slots<true>(recs, geo, tile_offsets, tile_prims, cam, st, fwd, upst, kg, det);
    else bwd_replay_slots<false>(recs, geo, tile_offsets, tile_prims, cam, st, fwd, upst, kg, det);
}

// deterministic mode (det_reduce.cu): rows instead of atomics
__global__ void __launch_bounds__(32 * BWD_WPC, QGS_BWD_MIN_BLOCKS / BWD_WPC)
raster_bwd_det_kernel(const PrimRec *__restrict__ recs, const Geo64 *__restrict__ geo,
                      const int32_t *__restrict__ tile_offsets,
                      const int32_t *__restrict__ tile_prims, CamK cam, SetK st, qgs_targets fwd,
                      qgs_upstream upst, float *__restrict__ kg, DetRows det)
{
    bwd_block<false, true, false>(recs, geo, tile_offsets, tile_prims, cam, st, fwd, upst, kg, det);
}

size_t fwd_smem_per_warp() { return sizeof(FwdSmem); }

// diagnostics build (QGS_UTIL_COUNTERS): copy and clear the device counters
int diag_counters(unsigned long long *out, int n)
{
#if QGS_UTIL_COUNTERS
    if (n > 4) n = 4;
    if (cudaMemcpyFromSymbol(out, qgs_diag, sizeof(unsigned long long) * n) != cudaSuccess) return -1;
    const unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(qgs_diag, z, sizeof(z));
    return n;
#else
    (void)out; (void)n;
    return 0;
#endif
}
size_t bwd_smem_per_warp() { return sizeof(BwdSmem); }

// ===================================================== raster schedule
// tiles by descending pair count (ties by tile), so the raster kernels start
// the longest tiles first; one CTA, bitonic sort of (~count, tile) in smem
// Schedules (one CTA): tiles grouped by pair count -- quarter-octave bins,
// largest first, index order inside a bin (a stable counting sort; the
// schedule only has to put long tiles early, not order them exactly).
// heavy_only: only tiles over 4x the mean count move to the front; the
// rest keep their natural order (memory locality of the sort).
constexpr int ORDER_BINS = 129;                 // 128 count bins + "unranked"
__global__ void __launch_bounds__(1024)
tile_order_kernel(const int32_t *__restrict__ tile_offsets, int n_tiles, int32_t *order,
                  int heavy_only)
{
    __shared__ int hist[ORDER_BINS], run[ORDER_BINS];
    __shared__ int wcnt[32][ORDER_BINS];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double heavy = 4.0 * (double)tile_offsets[n_tiles] / (double)max(n_tiles, 1);
    auto bin_of = [&](int t) {
        const int cnt = tile_offsets[t + 1] - tile_offsets[t];
        if (heavy_only && !((double)cnt > heavy)) return ORDER_BINS - 1;
        const int key = (int)floorf(4.f * __log2f((float)cnt + 1.f));
        return max(0, 127 - min(key, 127));
    };
    for (int b = threadIdx.x; b < ORDER_BINS; b += blockDim.x) { hist[b] = 0; run[b] = 0; }
    for (int b = threadIdx.x; b < 32 * ORDER_BINS; b += blockDim.x) (&wcnt[0][0])[b] = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) atomicAdd(&hist[bin_of(t)], 1);
    __syncthreads();
    if (threadIdx.x == 0) {                     // exclusive scan of the bins
        int acc = 0;
        for (int b = 0; b < ORDER_BINS; ++b) { const int c = hist[b]; hist[b] = acc; acc += c; }
    }
    __syncthreads();
    for (int c0 = 0; c0 < n_tiles; c0 += blockDim.x) {
        const int t = c0 + threadIdx.x;
        const bool ok = t < n_tiles;
        const int b = ok ? bin_of(t) : ORDER_BINS;   // ORDER_BINS: no tile
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const int r = __popc(peers & ((1u << lane) - 1u));
        if (ok && r == 0) wcnt[w][b] = __popc(peers);
        __syncthreads();
        if (ok) {
            int pre = 0;
            for (int k = 0; k < w; ++k) pre += wcnt[k][b];
            order[hist[b] + run[b] + pre + r] = t;
        }
        __syncthreads();
        for (int bb = threadIdx.x; bb < ORDER_BINS; bb += blockDim.x) {
            int tot = 0;
            for (int k = 0; k < 32; ++k) { tot += wcnt[k][bb]; wcnt[k][bb] = 0; }
            run[bb] += tot;
        }
        __syncthreads();
    }
}

// ============================================================ diagnostics
// Single-thread replay of one pixel's stream with the same inline functions:
// records every accepted candidate and every emitted fragment (with T before).
__global__ void trace_pixel_kernel(const PrimRec *__restrict__ recs, const Geo64 *__restrict__ geo,
                                   const int32_t *__restrict__ tile_offsets,
                                   const int32_t *__restrict__ tile_prims, CamK cam, SetK st,
                                   int u, int v, int max, int *acc_prim, float *acc_t,
                                   float *acc_abar, int *em_prim, float *em_t, float *em_abar,
                                   double *em_T, int *counts)
{
    __shared__ double ring_t[RING][32];
    __shared__ int ring_p[RING][32];
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const Cfg c = make_cfg(st);
    double d[3];
    pixel_dir64(cam, u, v, d);
    const float dx = (float)d[0], dy = (float)d[1], dz = (float)d[2];
    const int tile = (v / TILE) * cam.tiles_x + u / TILE;
    Ring R{&ring_t[0][0], &ring_p[0][0], 0};
    double T = 1.0;
    int na = 0, ne = 0;
    bool alive = true;
    auto record = [&](int ep, double et) {
        Frag f;
        shade_emitted(recs[ep], geo[ep], d, dx, dy, dz, et, c, f);
        if (ne < max) { em_prim[ne] = ep; em_t[ne] = (float)et; em_abar[ne] = f.abar; em_T[ne] = T; }
        ne++;
        T *= 1.0 - f.abar64;
        if (T < c.t_term) alive = false;
    };
    for (int i = tile_offsets[tile]; i < tile_offsets[tile + 1] && alive; ++i) {
        const int p = tile_prims[i];
        const PrimRec &r = recs[p];
        double t;
        if (in_box(r, u, v) && (st.exact ? accept<MODE_EXACT>(r, geo[p], d, dx, dy, dz, c, t)
                                         : accept<MODE_FAST>(r, geo[p], d, dx, dy, dz, c, t))) {
            if (na < max) {
                Frag f;
                shade_emitted(r, geo[p], d, dx, dy, dz, t, c, f);
                acc_prim[na] = p; acc_t[na] = (float)t; acc_abar[na] = f.abar;
            }
            na++;
            double et;
            int ep;
            bool emit;
            if (!c.resort) { et = t; ep = p; emit = true; }
            else emit = ring_push(R, t, p, et, ep);
            if (emit) record(ep, et);
        }
    }
    while (alive && R.n > 0) {
        double et;
        int ep;
        ring_pop(R, et, ep);
        record(ep, et);
    }
    counts[0] = na;
    counts[1] = ne;
}


}  // namespace qgs
