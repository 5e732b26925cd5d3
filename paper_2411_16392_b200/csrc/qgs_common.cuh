// Shared device code for the sm_100a QGS tile rasterizer.
//
// Per-primitive state lives in one caller-owned "prep" buffer:
//   Geo64[P]   float64 geometry (feeds screen boxes and tile sort keys; these
//              integer/ordering outputs must be bit-identical to the reference)
//   PrimRec[P] 128-byte fp32 record consumed by the raster kernels
//   int4[P]    inclusive pixel box (umin, umax, vmin, vmax); empty = (0,-1,0,-1)
//   int32[P]   tiles covered;  int64[P+1] exclusive scan = pair offsets
#pragma once

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <set>
#include <utility>
#include <cuda_runtime.h>

#include "../../include/qgs_b200.h"

// Device bounds checks of the debug build (libqgs_b200_debug.so, built with
// -DQGS_DEBUG_CHECKS=1 by build.py; tests/test_debug_checks.py runs every
// path under it): a failed check traps the kernel (cudaErrorLaunchFailure /
// illegal instruction), which the host reports.  compute-sanitizer is not
// available on the GPU pool, so these are the memory-safety net.
#ifndef QGS_DEBUG_CHECKS
#define QGS_DEBUG_CHECKS 0
#endif
#if QGS_DEBUG_CHECKS
#define QGS_CHECK(cond)                                                                  \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            printf("QGS_CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);        \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define QGS_CHECK(cond) do { } while (0)
#endif

namespace qgs {

// Raise a kernel's dynamic shared-memory limit once per (kernel, device):
// cudaFuncSetAttribute applies to the current device only, so a process that
// uses several GPUs needs it on each.  Thread-safe; returns the CUDA status.
inline cudaError_t ensure_smem_attr(const void *func, int bytes)
{
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({func, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({func, dev});
    return e;
}


constexpr int TILE = 16;            // bounds.py:19
constexpr int RING = 8;             // raster_kernels.py:26 BUFFER_SIZE
constexpr int KG = QGS_KG_STRIDE;   // kernel-gradient floats per primitive
constexpr int AUX = QGS_AUX_PLANES;

// kernel-gradient slots (raster_kernels.py:29-37 with M, Nmat folded into the
// 3-vector omega and lambda into s / w; 16 floats = four 16-byte vectors)
enum { KG_OHAT = 0, KG_ROT = 3, KG_W = 6, KG_S = 9, KG_ALPHA = 12, KG_COLOR = 13 };
// fp64 aux planes written by the forward for the backward
enum { AX_C0 = 0, AX_A = 3, AX_D = 4, AX_D2 = 5, AX_N0 = 6, AX_K = 9, AX_DIST = 10, AX_T = 11 };
enum { BR_QUAD = 0, BR_LINEAR = 1, BR_PLANAR = 2 };

struct Geo64 {            // 32 doubles, 256 B
    double ohat[3];
    double M[9];          // local-from-camera rotation R^T R_cw (row-major)
    double wv[3];         // w1, w2, iw3
    double sv[3];         // activated signed scales
    double vert_u, vert_v, dist;
    double alpha;
    double col[3];
    double planar;        // 1.0 / 0.0
    double pad[6];
};

struct __align__(16) PrimRec {   // 32 floats, 128 B
    float M[9];           // 0-8
    float ox, oy, oz;     // 9-11
    float w1, w2, iw3;    // 12-14
    float s1, s2, s3;     // 15-17
    float lam1, lam2;     // 18-19
    float alpha;          // 20
    float C;              // 21 ray-quadric constant term, rounded once from fp64
    float col[3];         // 22-24
    uint32_t bb_u;        // 25 umin | umax << 16
    uint32_t bb_v;        // 26 vmin | vmax << 16
    uint32_t flags;       // 27 bit0 planar
    float s12;            // 28 |s1 s2|
    float ell9;           // 29 9 (s1 s2)^2
    float pad[2];
};
static_assert(sizeof(PrimRec) == 128, "PrimRec must be 128 B");
static_assert(sizeof(Geo64) == 256, "Geo64 must be 256 B");

// Screen-space cull of one primitive: the pixel-centre conic of the outline
// of an ellipsoid that contains every point the selection rule can accept
// (preprocess.cu: bounding_conic).  Pixel (u, v) with U = u - uc, V = v - vc
// can only be accepted if  A U^2 + B U V + C V^2 + D U + E V + F <= 0
// (F carries the fp32 evaluation margin; all zero with F = -1 = no cull).
struct __align__(16) ConicRec {   // 32 B
    float A, B, C, D, E, F;
    uint32_t bb_u, bb_v;  // the inclusive pixel box (as PrimRec); origin = its centre
};
static_assert(sizeof(ConicRec) == 32, "ConicRec must be 32 B");

__host__ __device__ inline float conic_uc(const ConicRec &q)
{
    return 0.5f * (float)((q.bb_u & 0xffffu) + (q.bb_u >> 16));
}
__host__ __device__ inline float conic_vc(const ConicRec &q)
{
    return 0.5f * (float)((q.bb_v & 0xffffu) + (q.bb_v >> 16));
}

struct PrepView {
    Geo64 *geo;
    PrimRec *rec;
    ConicRec *conic;
    const double *rays;   // optional W*H*3 fp64 pixel-ray table (binning workspace)
    int4 *bbox;
    int32_t *ntiles;
    int64_t *pair_off;    // P+1
    int32_t *nonfinite;   // primitives with non-finite raw scales / signs (model.py:37-38)
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

__host__ __device__ inline PrepView prep_view(void *base, int32_t P)
{
    char *b = static_cast<char *>(base);
    PrepView v;
    v.rays = nullptr;
    size_t o = 0;
    v.geo = reinterpret_cast<Geo64 *>(b + o);      o += align256(sizeof(Geo64) * (size_t)P);
    v.rec = reinterpret_cast<PrimRec *>(b + o);    o += align256(sizeof(PrimRec) * (size_t)P);
    v.conic = reinterpret_cast<ConicRec *>(b + o); o += align256(sizeof(ConicRec) * (size_t)P);
    v.bbox = reinterpret_cast<int4 *>(b + o);      o += align256(sizeof(int4) * (size_t)P);
    v.ntiles = reinterpret_cast<int32_t *>(b + o); o += align256(sizeof(int32_t) * (size_t)P);
    v.pair_off = reinterpret_cast<int64_t *>(b + o); o += align256(sizeof(int64_t) * ((size_t)P + 1));
    v.nonfinite = reinterpret_cast<int32_t *>(b + o);
    return v;
}

__host__ __device__ inline size_t prep_bytes(int32_t P)
{
    return align256(sizeof(Geo64) * (size_t)P) + align256(sizeof(PrimRec) * (size_t)P) +
           align256(sizeof(ConicRec) * (size_t)P) +
           align256(sizeof(int4) * (size_t)P) + align256(sizeof(int32_t) * (size_t)P) +
           align256(sizeof(int64_t) * ((size_t)P + 1)) + 256 + 256;
}

// Camera / settings as kernel arguments (by value).
struct CamK {
    double fx, fy, cx, cy;
    int W, H, tiles_x, tiles_y;
    double Rwc[9], twc[3], eye[3];
};

struct SetK {
    double bg[3];
    double t_clip, alpha_floor, alpha_clamp, t_term;
    int resort, euclid, no_cull, exact;
    int pbits;            // bits of the primitive id in the sort composite (qgs_bin)
};

inline CamK make_camk(const qgs_camera &c)
{
    CamK k;
    k.fx = c.fx; k.fy = c.fy; k.cx = c.cx; k.cy = c.cy;
    k.W = c.width; k.H = c.height;
    k.tiles_x = (c.width + TILE - 1) / TILE;
    k.tiles_y = (c.height + TILE - 1) / TILE;
    for (int i = 0; i < 9; ++i) k.Rwc[i] = c.R_wc[i];
    for (int i = 0; i < 3; ++i) { k.twc[i] = c.t_wc[i]; k.eye[i] = c.center[i]; }
    return k;
}

inline SetK make_setk(const qgs_settings &s)
{
    SetK k;
    for (int i = 0; i < 3; ++i) k.bg[i] = s.background[i];
    k.t_clip = s.t_near_clip; k.alpha_floor = s.alpha_floor;
    k.alpha_clamp = s.alpha_clamp; k.t_term = s.t_term;
    k.resort = s.resort; k.euclid = s.euclidean_density; k.no_cull = s.no_cull;
    k.exact = s.exact_decisions;
    k.pbits = 32;
    return k;
}

// ----------------------------------------------------------------- fp64
// These follow the reference operation order exactly (intersect.py:31-115,
// geodesic.py:23-31,51-59).  Translation units that use them are compiled
// with -fmad=false so nothing is contracted into an FMA.

__device__ inline double arc_length64(double a, double rho)
{
    double u = 2.0 * a * rho;
    if (fabs(u) < 1e-3) {
        double u2 = u * u;
        return rho * (1.0 + u2 / 6.0 - u2 * u2 / 40.0);
    }
    double r = sqrt(u * u + 1.0);
    return (log(r + u) + u * r) / (4.0 * a);
}

__device__ inline double sigma_dir64(double s1, double s2, double c, double s)
{
    double m = (s2 * c) * (s2 * c) + (s1 * s) * (s1 * s);
    return fabs(s1 * s2) / sqrt(m);
}

// arc length of z = a r^2 over [0, rho] in fp32 (series below |u| = 0.3,
// log form above: |u| + r >= 1.34, so __logf keeps ~1e-6 relative)
__device__ inline float arc_length32(float a, float rho)
{
    float u = 2.f * a * rho;
    if (fabsf(u) < 0.3f) {
        float u2 = u * u;
        return rho * (1.f + u2 * (1.f / 6.f + u2 * (-1.f / 40.f + u2 * (1.f / 112.f - u2 * (5.f / 1152.f)))));
    }
    float r = sqrtf(u * u + 1.f);
    return __fdividef(copysignf(__logf(fabsf(u) + r), u) + u * r, 4.f * a);   // |u| + r >= 1.34
}

// The 3-sigma test l <= 3 sigma(theta) at local (x, y) (intersect.py:104-112,
// geodesic.py:23-31,51-59).  Decided in fp32 when the margin exceeds 1e-4
// relative (the fp32 evaluation is good to ~1e-6), else by the reference's
// own float64 expressions -- so the decision is always the float64 one.
__device__ inline bool within_3sigma64(double x, double y, double s1, double s2, double s3,
                                       double w1, double w2, bool euclid)
{
    {
        const float xf = (float)x, yf = (float)y;
        const float r2 = xf * xf + yf * yf;
        if (r2 > 1e-18f) {
            // approximate rsqrt / reciprocal / log: ~1e-6 relative, far inside the band
            const float ir = rsqrtf(r2), rho = r2 * ir, c = xf * ir, sn = yf * ir;
            const float a = (float)s3 * ((float)w1 * c * c + (float)w2 * sn * sn);
            const float l = euclid ? rho : arc_length32(a, rho);
            const float f1 = (float)s1, f2 = (float)s2;
            const float m = (f2 * c) * (f2 * c) + (f1 * sn) * (f1 * sn);
            const float isig = m * rsqrtf(m) * __frcp_rn(fabsf(f1 * f2));   // 1 / sigma
            const float q = l * isig * (1.f / 3.f);
            if (q < 1.f - 1e-4f) return true;
            if (q > 1.f + 1e-4f) return false;
        }
    }
    double rho = sqrt(x * x + y * y), c = 1.0, s = 0.0;
    if (rho > 1e-12) { c = x / rho; s = y / rho; }
    double a = s3 * (w1 * c * c + w2 * s * s);
    double l = euclid ? rho : arc_length64(a, rho);
    double sig = sigma_dir64(s1, s2, c, s);
    return l <= 3.0 * sig;
}

// fragment_geometry restricted to what the sort key needs: (valid, t).
__device__ inline bool hit_depth64(const double *wv, const double *sv, const double *oh,
                                   double dx, double dy, double dz, bool planar, bool euclid,
                                   double t_clip, double &t_out)
{
    if (planar) {
        if (fabs(dz) < 1e-12) return false;
        double t = -oh[2] / dz;
        if (t <= t_clip) return false;
        double x = oh[0] + t * dx, y = oh[1] + t * dy;
        if (!within_3sigma64(x, y, sv[0], sv[1], 0.0, 0.0, 0.0, true)) return false;
        t_out = t;
        return true;
    }
    double w1 = wv[0], w2 = wv[1], iw3 = wv[2], ox = oh[0], oy = oh[1], oz = oh[2];
    double A = w1 * dx * dx + w2 * dy * dy;
    double B = 2.0 * (w1 * ox * dx + w2 * oy * dy) - iw3 * dz;
    double C = w1 * ox * ox + w2 * oy * oy - iw3 * oz;
    double r0 = 0.0, r1 = 0.0;
    int cnt;
    if (fabs(A) < 1e-6) {
        if (fabs(B) < 1e-12) cnt = 0;
        else { cnt = 1; r0 = -C / B; }
    } else {
        double disc = B * B - 4.0 * A * C;
        if (disc < 0.0) cnt = 0;
        else {
            double sa = A > 0.0 ? 1.0 : -1.0;
            double sq = sqrt(disc);
            r0 = (-B - sa * sq) / (2.0 * A);
            r1 = (-B + sa * sq) / (2.0 * A);
            cnt = disc == 0.0 ? 1 : 2;
        }
    }
    double s1 = sv[0], s2 = sv[1], s3 = sv[2], s1s2 = s1 * s2;
    for (int k = 0; k < cnt; ++k) {
        double t = k == 0 ? r0 : r1;
        if (t <= t_clip) continue;
        double x = ox + t * dx, y = oy + t * dy;
        double m = (s2 * x) * (s2 * x) + (s1 * y) * (s1 * y);
        if (m > 9.0 * s1s2 * s1s2) continue;
        if (within_3sigma64(x, y, s1, s2, s3, w1, w2, euclid)) { t_out = t; return true; }
    }
    return false;
}

// tile_sort_depths (raster_kernels.py:684-716) for one (tile, primitive).
// unit camera ray of pixel centre (u, v), cameras.py:53-59 operation order
__device__ inline void pixel_ray64(const CamK &cam, int u, int v, double &cx, double &cy,
                                   double &cz)
{
    double ddx = ((double)u + 0.5 - cam.cx) / cam.fx, ddy = ((double)v + 0.5 - cam.cy) / cam.fy;
    double nrm = sqrt(ddx * ddx + ddy * ddy + 1.0);
    cx = ddx / nrm; cy = ddy / nrm; cz = 1.0 / nrm;
}

// tile_sort_depths' key for one unit camera ray (cx, cy, cz): the depth of
// the selected hit, else the centre distance (raster_kernels.py:700-716)
__device__ inline double key_from_ray64(const double *ohat, const double *M, const double *wv,
                                        const double *sv, bool planar, double dist, double cx,
                                        double cy, double cz, bool euclid, double t_clip)
{
    double dx = M[0] * cx + M[1] * cy + M[2] * cz;
    double dy = M[3] * cx + M[4] * cy + M[5] * cz;
    double dz = M[6] * cx + M[7] * cy + M[8] * cz;
    double t;
    if (hit_depth64(wv, sv, ohat, dx, dy, dz, planar, euclid, t_clip, t)) return t;
    return dist;
}

// hit_depth64 / key_from_ray64 with the per-primitive subexpressions hoisted
// (identical operations in identical order, so bit-identical keys) and the
// far root's division done only when the near root is rejected.
struct KeyPrim {
    double M[9], ohat[3], w1, w2, iw3, s1, s2, s3;
    double w1ox, w2oy, C, lim, dist;
    bool planar;
};

__device__ inline KeyPrim key_prim(const Geo64 &g)
{
    KeyPrim k;
    for (int i = 0; i < 9; ++i) k.M[i] = g.M[i];
    for (int i = 0; i < 3; ++i) k.ohat[i] = g.ohat[i];
    k.w1 = g.wv[0]; k.w2 = g.wv[1]; k.iw3 = g.wv[2];
    k.s1 = g.sv[0]; k.s2 = g.sv[1]; k.s3 = g.sv[2];
    const double ox = k.ohat[0], oy = k.ohat[1], oz = k.ohat[2];
    k.w1ox = k.w1 * ox;
    k.w2oy = k.w2 * oy;
    k.C = k.w1 * ox * ox + k.w2 * oy * oy - k.iw3 * oz;
    const double s1s2 = k.s1 * k.s2;
    k.lim = 9.0 * s1s2 * s1s2;
    k.dist = g.dist;
    k.planar = g.planar != 0.0;
    return k;
}

#ifndef QGS_KEY_SHARED_RCP
#define QGS_KEY_SHARED_RCP 1
#endif
// n / b correctly rounded from y = RN(1/b) (__drcp_rn): q = n y, then the FMA
// correction q + (n - b q) y (Markstein: exact for y = RN(1/b) and q within
// an ulp, barring over/underflow, which these magnitudes never reach) -- for
// several quotients with one divisor, bit-identical to the divisions
__device__ __forceinline__ double div_rcp(double n, double b, double y)
{
    const double q = n * y;
    return __fma_rn(__fma_rn(-b, q, n), y, q);
}
__device__ inline double key_from_ray_fast(const KeyPrim &k, double cx, double cy, double cz,
                                           bool euclid, double t_clip)
{
    const double dx = k.M[0] * cx + k.M[1] * cy + k.M[2] * cz;
    const double dy = k.M[3] * cx + k.M[4] * cy + k.M[5] * cz;
    const double dz = k.M[6] * cx + k.M[7] * cy + k.M[8] * cz;
    const double ox = k.ohat[0], oy = k.ohat[1];
    if (k.planar) {
        if (fabs(dz) < 1e-12) return k.dist;
        const double t = -k.ohat[2] / dz;
        if (t <= t_clip) return k.dist;
        const double x = ox + t * dx, y = oy + t * dy;
        return within_3sigma64(x, y, k.s1, k.s2, 0.0, 0.0, 0.0, true) ? t : k.dist;
    }
    const double A = k.w1 * dx * dx + k.w2 * dy * dy;
    const double B = 2.0 * (k.w1ox * dx + k.w2oy * dy) - k.iw3 * dz;
    auto try_root = [&](double t) -> bool {
        if (t <= t_clip) return false;
        const double x = ox + t * dx, y = oy + t * dy;
        const double m = (k.s2 * x) * (k.s2 * x) + (k.s1 * y) * (k.s1 * y);
        if (m > k.lim) return false;
        return within_3sigma64(x, y, k.s1, k.s2, k.s3, k.w1, k.w2, euclid);
    };
    if (fabs(A) < 1e-6) {
        if (fabs(B) < 1e-12) return k.dist;
        const double t = -k.C / B;
        return try_root(t) ? t : k.dist;
    }
    const double disc = B * B - 4.0 * A * k.C;
    if (disc < 0.0) return k.dist;
    const double sa = A > 0.0 ? 1.0 : -1.0;
    const double sq = sqrt(disc);
#if QGS_KEY_SHARED_RCP
    // both roots divide by 2A: one correctly rounded reciprocal (div_rcp),
    // bit-identical to the reference's divisions (checked in the debug build)
    const double den = 2.0 * A;
    const double y = __drcp_rn(den);
    auto qdiv = [&](double n) { return div_rcp(n, den, y); };
#else
    auto qdiv = [&](double n) { return n / (2.0 * A); };
#endif
    const double t0 = qdiv(-B - sa * sq);
    QGS_CHECK(t0 == (-B - sa * sq) / (2.0 * A) || t0 != t0);
    if (try_root(t0)) return t0;
    if (disc == 0.0) return k.dist;
    const double t1 = qdiv(-B + sa * sq);
    QGS_CHECK(t1 == (-B + sa * sq) / (2.0 * A) || t1 != t1);
    return try_root(t1) ? t1 : k.dist;
}

// `dirtab` (optional): the W*H*3 table of pixel_ray64, bit-identical.
__device__ inline double tile_key64(const double *ohat, const double *M, const double *wv,
                                    const double *sv, bool planar, double vu, double vv,
                                    double dist, int tile, const CamK &cam, bool euclid,
                                    double t_clip, const double *dirtab = nullptr)
{
    int ty = tile / cam.tiles_x, tx = tile - ty * cam.tiles_x;
    long long ulo = tx * TILE, uhi = min(cam.W, tx * TILE + TILE) - 1;
    long long vlo = ty * TILE, vhi = min(cam.H, ty * TILE + TILE) - 1;
    long long iu = (long long)floor(vu), iv = (long long)floor(vv);
    iu = iu < ulo ? ulo : (iu > uhi ? uhi : iu);
    iv = iv < vlo ? vlo : (iv > vhi ? vhi : iv);
    double cx, cy, cz;
    if (dirtab) {
        const double *d = dirtab + 3 * ((size_t)iv * cam.W + iu);
        cx = d[0]; cy = d[1]; cz = d[2];
    } else {
        pixel_ray64(cam, (int)iu, (int)iv, cx, cy, cz);
    }
    return key_from_ray64(ohat, M, wv, sv, planar, dist, cx, cy, cz, euclid, t_clip);
}

__device__ inline double tile_key_geo(const Geo64 &g, int tile, const CamK &cam, bool euclid,
                                      double t_clip, const double *dirtab = nullptr)
{
    return tile_key64(g.ohat, g.M, g.wv, g.sv, g.planar != 0.0, g.vert_u, g.vert_v, g.dist,
                      tile, cam, euclid, t_clip, dirtab);
}


}  // namespace qgs
