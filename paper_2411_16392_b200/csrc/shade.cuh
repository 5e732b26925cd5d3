// Raster-side shading of one (pixel ray, primitive) pair.
//
// Selection rule of fragment_geometry (intersect.py:58-115) and _shade
// (raster_kernels.py:40-80).  Two stages:
//
//  1. Coarse fp32 test on every candidate: roots of A t^2 + B t + C (C
//     precomputed per primitive in fp64) and the 3-sigma test with a 5%
//     margin.  This polynomial form cancels badly (terms ~ w |o|^2 ~ 1e3-1e4
//     summing to ~1 at the hit), so it only decides which roots are worth a
//     precise look.
//  2. Refinement in fp64 of each root that passes: two fp64
//     Newton steps on the POINT-evaluated implicit function
//     F(x) = w1 x^2 + w2 y^2 - iw3 z at x = ohat + t dhat (no cancellation),
//     giving the depth t64 to ~1e-15.  The hit point is re-derived from t64
//     in fp64 (shade_at), rounded once to fp32, and the exact selection
//     (t > t_clip, ellipse pre-reject, l <= 3 sigma) and the Gaussian weight
//     are evaluated from it.
//
// shade_at(t64) is also what re-shades an emitted fragment, so candidate
// time and emission time see bit-identical values.  The ring orders by t64,
// matching the reference's float64 depth order except at exact ties.
#pragma once

#include "qgs_common.cuh"

// the Gaussian weight and the arc length's log: accurate by default
#ifndef QGS_FAST_EXPLOG
#define QGS_FAST_EXPLOG 0
#endif
#if QGS_FAST_EXPLOG
#define QGS_EXPF __expf
#define QGS_LOGF __logf
#else
#define QGS_EXPF expf
#define QGS_LOGF logf
#endif
#ifndef QGS_NEWTON64
#define QGS_NEWTON64 2      // fp64 Newton steps refining an accepted root
#endif
#ifndef QGS_NEWTON_RCP64
#define QGS_NEWTON_RCP64 1  // derivative inverse from rcp.approx.f64 (C3 forward -1.6 %)
#endif

namespace qgs {

struct Hit {
    double t64;
    float t, x, y, z, rho, cth, sth, a, l, sig, G;
    float q;                  // dt-denominator: F'(t) (quad), B (linear), dhz (planar)
    float dhx, dhy, dhz;
    int branch;
};

// Decision modes of the candidate test: MODE_FAST fp32 decisions; MODE_EXACT
// (settings.exact_decisions) re-makes band cases in fp64.
enum { MODE_FAST = 0, MODE_EXACT = 1 };

// arc length of z = a r^2 over [0, rho]; series below |u| = 0.3 (error < 1e-8)
__device__ __forceinline__ float arc32(float a, float rho)
{
    float u = 2.f * a * rho;
    if (fabsf(u) < 0.3f) {
        float u2 = u * u;
        return rho * (1.f + u2 * (1.f / 6.f + u2 * (-1.f / 40.f + u2 * (1.f / 112.f - u2 * (5.f / 1152.f)))));
    }
    float r = sqrtf(fmaf(u, u, 1.f));
    float as = copysignf(QGS_LOGF(fabsf(u) + r), u);
    return (as + u * r) / (4.f * a);
}

// (dl/da, dl/drho) on the same branch
__device__ __forceinline__ void arc32_grad(float a, float rho, float l, float &dla, float &dlr)
{
    float u = 2.f * a * rho;
    if (fabsf(u) < 0.3f) {
        float u2 = u * u;
        float fp = u * (1.f / 3.f + u2 * (-1.f / 10.f + u2 * (3.f / 56.f - u2 * (5.f / 144.f))));
        dla = 2.f * rho * rho * fp;
        dlr = 1.f + u2 * (0.5f + u2 * (-0.125f + u2 * (1.f / 16.f - u2 * (5.f / 128.f))));
        return;
    }
    float r = sqrtf(fmaf(u, u, 1.f));
    dla = (rho * r - l) / a;
    dlr = r;
}

// polar coordinates, curvature coefficient, geodesic length and sigma at a
// local point; returns the 3-sigma test (factor `k` widens it)
__device__ __forceinline__ bool eval_point(const PrimRec &r, float x, float y, bool planar,
                                           bool euclid, float k, Hit &h)
{
    float rho = sqrtf(fmaf(x, x, y * y));
    float c = 1.f, s = 0.f;
    if (rho > 1e-12f) { float ir = 1.f / rho; c = x * ir; s = y * ir; }
    float a = planar ? 0.f : r.s3 * fmaf(r.w1 * c, c, r.w2 * s * s);
    float l = (planar || euclid) ? rho : arc32(a, rho);
    float sc = r.s2 * c, ss = r.s1 * s;
    float sig = r.s12 * rsqrtf(fmaf(sc, sc, ss * ss));
    h.x = x; h.y = y; h.rho = rho; h.cth = c; h.sth = s; h.a = a; h.l = l; h.sig = sig;
    return l <= k * 3.f * sig;
}

__device__ __forceinline__ bool ellipse_out(const PrimRec &r, float x, float y, float k)
{
    float ex = r.s2 * x, ey = r.s1 * y;
    return fmaf(ex, ex, ey * ey) > k * r.ell9;
}

// Exact evaluation at a given fp64 depth (candidate confirmation and
// re-shading of emitted fragments).  dh64 = M d in fp64.
__device__ __forceinline__ void shade_at(const PrimRec &r, const Geo64 &g, const double dh[3],
                                         double t64, bool euclid, Hit &h)
{
    const bool planar = (r.flags & 1u) != 0;
    double x = g.ohat[0] + t64 * dh[0];
    double y = g.ohat[1] + t64 * dh[1];
    h.z = (float)(g.ohat[2] + t64 * dh[2]);
    h.t64 = t64;
    h.t = (float)t64;
    h.dhx = (float)dh[0]; h.dhy = (float)dh[1]; h.dhz = (float)dh[2];
    if (planar) {
        h.branch = BR_PLANAR;
        h.q = (float)dh[2];
    } else {
        double w1 = g.wv[0], w2 = g.wv[1], iw3 = g.wv[2];
        double A = w1 * dh[0] * dh[0] + w2 * dh[1] * dh[1];
        double Fp = 2.0 * (w1 * x * dh[0] + w2 * y * dh[1]) - iw3 * dh[2];
        if (fabs(A) < 1e-6) { h.branch = BR_LINEAR; h.q = (float)(Fp - 2.0 * A * t64); }
        else { h.branch = BR_QUAD; h.q = (float)Fp; }
    }
    eval_point(r, (float)x, (float)y, planar, euclid, 1.f, h);
}

// fp32 re-shade guard: a logged fragment whose root derivative F'(t) is
// below this fraction of its terms (a grazing ray) re-shades from the
// float64 geometry; the root gradient dt = -g / F'(t) amplifies F's fp32
// cancellation error by its inverse (the near-tangent
// fragments under 1e-2 carry the gradient error)
#ifndef QGS_LOG_Q_GUARD
#define QGS_LOG_Q_GUARD 1e-2f
#endif

// Re-shading of a logged fragment in fp32: the forward's fp32 hit point
// (x, y) makes rho, theta, l, sigma -- hence G and alpha -- bit-identical to
// the forward's; dh, z and the root derivative q are re-derived in fp32
// (gradient-only quantities, ~1e-6 relative except q on grazing rays).
// Returns false when the fp32 root derivative q is ill-conditioned (a
// grazing ray: |q| below QGS_LOG_Q_GUARD of its terms) or |A| is too close to the
// linear-branch threshold to trust the fp32 branch; the caller then re-shades
// that fragment from the float64 geometry.
__device__ __forceinline__ bool shade_from_log(const PrimRec &r, float x, float y, double t64,
                                               float dx, float dy, float dz, bool euclid, Hit &h)
{
    bool ok = true;
    const bool planar = (r.flags & 1u) != 0;
    const float hx = fmaf(r.M[0], dx, fmaf(r.M[1], dy, r.M[2] * dz));
    const float hy = fmaf(r.M[3], dx, fmaf(r.M[4], dy, r.M[5] * dz));
    const float hz = fmaf(r.M[6], dx, fmaf(r.M[7], dy, r.M[8] * dz));
    h.t64 = t64;
    h.t = (float)t64;
    h.dhx = hx; h.dhy = hy; h.dhz = hz;
    if (planar) {
        h.branch = BR_PLANAR;
        h.q = hz;
        h.z = 0.f;
    } else {
        const float a1 = r.w1 * hx * hx, a2 = r.w2 * hy * hy;
        const float A = a1 + a2;
        const float t1 = r.w1 * x * hx, t2 = r.w2 * y * hy, t3 = r.iw3 * hz;
        const float Fp = 2.f * (t1 + t2) - t3;
        // q well conditioned, and the linear-branch decision |A| < 1e-6
        // (made in float64 by the forward) not within fp32 reach of a flip
        // (A cancels on hyperbolic patches: its fp32 error is ~1e-7 of |a1| + |a2|)
        ok = fabsf(Fp) >= QGS_LOG_Q_GUARD * (2.f * (fabsf(t1) + fabsf(t2)) + fabsf(t3)) &&
             fabsf(fabsf(A) - 1e-6f) > 1e-6f * (fabsf(a1) + fabsf(a2)) + 1e-12f;
        if (fabsf(A) < 1e-6f) {
            h.branch = BR_LINEAR;
            h.q = Fp - 2.f * A * h.t;
            h.z = fmaf(h.t, hz, r.oz);
        } else {
            h.branch = BR_QUAD;
            h.q = Fp;
            h.z = r.s3 * fmaf(r.w1 * x, x, r.w2 * y * y);   // on the quadric
        }
    }
    eval_point(r, x, y, planar, euclid, 1.f, h);
    return ok;
}

__device__ __forceinline__ void local_dir64(const Geo64 &g, const double d[3], double dh[3])
{
    dh[0] = g.M[0] * d[0] + g.M[1] * d[1] + g.M[2] * d[2];
    dh[1] = g.M[3] * d[0] + g.M[4] * d[1] + g.M[5] * d[2];
    dh[2] = g.M[6] * d[0] + g.M[7] * d[1] + g.M[8] * d[2];
}

// fp64 Newton on the point-evaluated implicit function starting at t0.
// Linear branch (|A| < 1e-6, intersect.py:42-45) solves B t + C = 0 exactly
// like the reference (the A t^2 term is removed from F); planar solves
// oz + t dhz = 0.
__device__ __forceinline__ double refine_depth(const Geo64 &g, const double dh[3], bool planar,
                                               float t0)
{
    const double ox = g.ohat[0], oy = g.ohat[1], oz = g.ohat[2];
    double t = (double)t0;
    if (planar) {
        float idz = 1.f / (float)dh[2];
        for (int it = 0; it < 2; ++it) t -= (oz + t * dh[2]) * (double)idz;
        return t;
    }
    const double w1 = g.wv[0], w2 = g.wv[1], iw3 = g.wv[2];
    const double A = w1 * dh[0] * dh[0] + w2 * dh[1] * dh[1];
    const double Alin = fabs(A) < 1e-6 ? A : 0.0;   // removed on the linear branch
    // two steps of the approximate-derivative Newton (each contracts the
    // error by >= 1e6 plus the quadratic term) take the coarse root's <= 1e-4
    // to full precision; a third was measured to change nothing
    constexpr int NEWTON64 = QGS_NEWTON64;
#pragma unroll
    for (int it = 0; it < NEWTON64; ++it) {
        double x = ox + t * dh[0], y = oy + t * dh[1], z = oz + t * dh[2];
        double F = w1 * x * x + w2 * y * y - iw3 * z - Alin * t * t;
        double Fp = 2.0 * (w1 * x * dh[0] + w2 * y * dh[1]) - iw3 * dh[2] - 2.0 * Alin * t;
#if QGS_NEWTON_RCP64
        double rf;      // ~2^-20 reciprocal straight from the fp64 MUFU (no conversions)
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rf) : "d"(Fp));
        t -= F * rf;
#else
        t -= F * (double)(1.f / (float)Fp);
#endif
    }
    return t;
}

// Exact-decision mode (settings.exact_decisions): a selection or alpha-floor
// decision whose fp32 margin lies inside these relative bands is re-made in
// fp64 with the reference's expressions, so the accepted set is the float64
// one; the default mode keeps the fp32 decisions (no fp64 code in the hot
// kernels -- DESIGN.md section 6 has the parity and cost of both).
constexpr float SEL_BAND = 1e-5f;          // ellipse pre-reject, l <= 3 sigma
constexpr float FLOOR_BAND = 1e-4f;        // alpha G >= alpha_floor

// The reference's float64 selection at depth t64 (intersect.py:90-113:
// ellipse pre-reject, l <= 3 sigma; raster_kernels.py:58-60: alpha floor)
// from the primitive's float64 geometry in global memory.  Bit 0: the root
// is selected; bit 1: and its weight passes the floor.  Out of line.
#ifndef QGS_UTIL_COUNTERS
#define QGS_UTIL_COUNTERS 0
#endif
#if QGS_UTIL_COUNTERS
// diagnostics build: [0] exact64 calls (band cases), [1] near-tangent roots
// decided by the fp64 closed form; read by tools/lane_util_fwd.py
__device__ unsigned long long qgs_diag[4];
#endif

static __device__ __noinline__ unsigned exact64(const Geo64 *gp, const double dh[3], double t64,
                                                bool planar, bool euclid, double floor)
{
#if QGS_UTIL_COUNTERS
    atomicAdd(&qgs_diag[0], 1ull);
#endif
    const Geo64 &g = *gp;
    const double x = g.ohat[0] + t64 * dh[0], y = g.ohat[1] + t64 * dh[1];
    const double s1 = g.sv[0], s2 = g.sv[1], s3 = g.sv[2];
    if (!planar) {
        const double s1s2 = s1 * s2;
        const double m = (s2 * x) * (s2 * x) + (s1 * y) * (s1 * y);
        if (m > 9.0 * s1s2 * s1s2) return 0u;
    }
    const double rho = sqrt(x * x + y * y);
    double c = 1.0, s = 0.0;
    if (rho > 1e-12) { c = x / rho; s = y / rho; }
    const double a = planar ? 0.0 : s3 * (g.wv[0] * c * c + g.wv[1] * s * s);
    const double l = (planar || euclid) ? rho : arc_length64(a, rho);
    const double sig = sigma_dir64(s1, s2, c, s);
    if (!(l <= 3.0 * sig)) return 0u;
    const double G = exp(-(l * l) / (2.0 * sig * sig));
    return 1u | (g.alpha * G < floor ? 0u : 2u);
}

// exact selection + weight at an fp64 depth; false if the root is rejected.
// `gfull`: the primitive's complete Geo64 in global memory (EXACT band cases).
template <int M>
__device__ __forceinline__ bool confirm_root(const PrimRec &r, const Geo64 &g, const Geo64 *gfull,
                                             const double dh[3], double t64, bool planar,
                                             bool euclid, float t_clip, Hit &h)
{
    if (!(t64 > (double)t_clip)) return false;
    shade_at(r, g, dh, t64, euclid, h);
    if (M == MODE_FAST) {
        if (!planar && ellipse_out(r, h.x, h.y, 1.f)) return false;
        if (!(h.l <= 3.f * h.sig)) return false;
    } else {
        bool pass = true, near = false;
        if (!planar) {
            const float ex = r.s2 * h.x, ey = r.s1 * h.y;
            const float m = fmaf(ex, ex, ey * ey);
            pass = m <= r.ell9;
            near = fabsf(m - r.ell9) <= SEL_BAND * r.ell9;
        }
        const float lim = 3.f * h.sig;
        pass = pass && h.l <= lim;
        near = near || fabsf(h.l - lim) <= SEL_BAND * lim;
        if (near) pass = (exact64(gfull, dh, t64, planar, euclid, 0.0) & 1u) != 0u;
        if (!pass) return false;
    }
    h.G = QGS_EXPF(-(h.l * h.l) / (2.f * h.sig * h.sig));
    return true;
}

// the alpha floor on a selected hit (raster_kernels.py:58-60); fp64 inside
// its band in MODE_EXACT
template <int M>
__device__ __forceinline__ bool alpha_pass(const PrimRec &r, const Geo64 *gfull, const double d64[3],
                                           Hit &h, bool euclid, float floor)
{
    const float ab = r.alpha * h.G;
    if (M != MODE_EXACT || fabsf(ab - floor) > FLOOR_BAND * floor) return ab >= floor;
    double dh[3];
    dh[0] = gfull->M[0] * d64[0] + gfull->M[1] * d64[1] + gfull->M[2] * d64[2];
    dh[1] = gfull->M[3] * d64[0] + gfull->M[4] * d64[1] + gfull->M[5] * d64[2];
    dh[2] = gfull->M[6] * d64[0] + gfull->M[7] * d64[1] + gfull->M[8] * d64[2];
    return (exact64(gfull, dh, h.t64, h.branch == BR_PLANAR, euclid, (double)floor) & 2u) != 0u;
}

// Near-tangent rays: the fp32 discriminant is within its rounding band of
// zero, so the roots come from the reference's own fp64 closed form
// (intersect.py:39-55).  Out of line and a leaf (geometry by pointer, the
// local ray by value, the roots back in registers): the caller confirms the
// roots with the same inline code as every other candidate.
struct Roots2 {
    double r0, r1;
    int cnt;
};

static __device__ __noinline__ Roots2 marginal_roots(const Geo64 *gp, double dh0, double dh1,
                                                     double dh2)
{
#if QGS_UTIL_COUNTERS
    atomicAdd(&qgs_diag[1], 1ull);
#endif
    const Geo64 &g = *gp;
    const double w1 = g.wv[0], w2 = g.wv[1], iw3 = g.wv[2];
    const double ox = g.ohat[0], oy = g.ohat[1], oz = g.ohat[2];
    const double A = w1 * dh0 * dh0 + w2 * dh1 * dh1;
    const double B = 2.0 * (w1 * ox * dh0 + w2 * oy * dh1) - iw3 * dh2;
    const double C = w1 * ox * ox + w2 * oy * oy - iw3 * oz;
    Roots2 rr{0.0, 0.0, 0};
    if (fabs(A) < 1e-6) {
        if (fabs(B) < 1e-12) return rr;
        rr.r0 = -C / B;
        rr.cnt = 1;
    } else {
        const double disc = B * B - 4.0 * A * C;
        if (disc < 0.0) return rr;
        const double sa = A > 0.0 ? 1.0 : -1.0, sq = sqrt(disc);
        rr.r0 = (-B - sa * sq) / (2.0 * A);
        rr.r1 = (-B + sa * sq) / (2.0 * A);
        rr.cnt = disc == 0.0 ? 1 : 2;
    }
    return rr;
}

// Coarse fp32 stage (the per-candidate hot path).  Returns a mask: bit k set
// when root k (0 near, 1 far) passes the widened tests, CR_MARGINAL when the
// discriminant is inside its fp32 rounding band (decided later in fp64).
// Uses approximate reciprocal / sqrt / log: it only has to be conservative.
constexpr unsigned CR_MARGINAL = 4u;

__device__ __forceinline__ float arc32_fast(float a, float rho)
{
    float u = 2.f * a * rho;
    if (fabsf(u) < 0.3f) {
        float u2 = u * u;
        return rho * (1.f + u2 * (1.f / 6.f + u2 * (-1.f / 40.f + u2 * (1.f / 112.f))));
    }
    float r = sqrtf(fmaf(u, u, 1.f));
    float as = copysignf(__logf(fabsf(u) + r), u);
    return __fdividef(as + u * r, 4.f * a);
}

constexpr float COARSE_K = 1.05f;         // margin on the 3-sigma tests

// Stage 1, branch-free (selects only) so that two candidates interleave:
// roots of the ray quadric and the widened ellipse pre-reject of both roots.
// Returns bit k = root k survives, CR_MARGINAL = near-tangent (fp64 decides).
__device__ __forceinline__ unsigned coarse_stage1(const PrimRec &r, float dx, float dy, float dz,
                                                  float t_clip, float roots[2], float &hx,
                                                  float &hy, bool *has_root = nullptr)
{
    const bool planar = (r.flags & 1u) != 0;
    hx = fmaf(r.M[0], dx, fmaf(r.M[1], dy, r.M[2] * dz));
    hy = fmaf(r.M[3], dx, fmaf(r.M[4], dy, r.M[5] * dz));
    const float hz = fmaf(r.M[6], dx, fmaf(r.M[7], dy, r.M[8] * dz));
    const float A = fmaf(r.w1 * hx, hx, r.w2 * hy * hy);
    const float B = 2.f * fmaf(r.w1 * r.ox, hx, r.w2 * r.oy * hy) - r.iw3 * hz;
    const float C = r.C, AC4 = 4.f * A * C;
    const float disc = fmaf(B, B, -AC4);
    const bool lin = fabsf(A) < 1e-6f;
    const bool quad = !planar && !lin;
    // fp32 rounding of disc is ~1e-7 max(B^2, |4AC|); inside a 1e-5 band the
    // sign is decided in fp64
    const bool marg = quad && fabsf(disc) <= 1e-5f * fmaxf(B * B, fabsf(AC4));
    const float q = -0.5f * (B + copysignf(sqrtf(fmaxf(disc, 0.f)), B));
    // one reciprocal serves the first root of every branch
    const float den = planar ? hz : (lin ? B : A);
    const float num = planar ? -r.oz : (lin ? -C : q);
    const float ta = __fdividef(num, den);
    const float tb = __fdividef(C, q);
    const float t0 = quad ? fminf(ta, tb) : ta;
    const float t1 = quad ? fmaxf(ta, tb) : ta;
    const bool ok = planar ? fabsf(hz) >= 1e-12f : (lin ? fabsf(B) >= 1e-12f : disc >= 0.f);
    const float lim = (COARSE_K * COARSE_K) * r.ell9;
    const float x0 = fmaf(t0, hx, r.ox), y0 = fmaf(t0, hy, r.oy);
    const float x1 = fmaf(t1, hx, r.ox), y1 = fmaf(t1, hy, r.oy);
    const float m0 = fmaf(r.s2 * x0, r.s2 * x0, (r.s1 * y0) * (r.s1 * y0));
    const float m1 = fmaf(r.s2 * x1, r.s2 * x1, (r.s1 * y1) * (r.s1 * y1));
    const float tmin = t_clip * 0.99f;
    const bool in0 = ok && t0 > tmin && (planar || m0 <= lim);
    const bool in1 = ok && quad && t1 > tmin && m1 <= lim;
    roots[0] = t0;
    roots[1] = t1;
    if (has_root) *has_root = ok;          // diagnostics only
    return marg ? CR_MARGINAL : ((in0 ? 1u : 0u) | (in1 ? 2u : 0u));
}

// Stage 2: widened geodesic 3-sigma test of the roots that survived stage 1.
__device__ __forceinline__ unsigned coarse_stage2(const PrimRec &r, bool euclid, unsigned in,
                                                  const float roots[2], float hx, float hy)
{
    const bool planar = (r.flags & 1u) != 0;
    unsigned pass = 0u;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (!(in & (1u << k))) continue;
        const float t = roots[k];
        float x = fmaf(t, hx, r.ox), y = fmaf(t, hy, r.oy);
        float rho2 = fmaf(x, x, y * y);
        float ir = rsqrtf(fmaxf(rho2, 1e-30f));
        float rho = rho2 * ir;
        float c = rho > 1e-12f ? x * ir : 1.f, s = rho > 1e-12f ? y * ir : 0.f;
        float a = planar ? 0.f : r.s3 * fmaf(r.w1 * c, c, r.w2 * s * s);
        float l = (planar || euclid) ? rho : arc32_fast(a, rho);
        float sc = r.s2 * c, ss = r.s1 * s;
        float sig = r.s12 * rsqrtf(fmaf(sc, sc, ss * ss));
        if (l <= COARSE_K * 3.f * sig) pass |= 1u << k;
    }
    return pass;
}

__device__ __forceinline__ unsigned coarse_roots(const PrimRec &r, float dx, float dy, float dz,
                                                 bool euclid, float t_clip, float roots[2],
                                                 float &hx, float &hy, float &hz)
{
    hz = 0.f;
    const unsigned in = coarse_stage1(r, dx, dy, dz, t_clip, roots, hx, hy);
    if (in == 0u || (in & CR_MARGINAL)) return in;
    return coarse_stage2(r, euclid, in, roots, hx, hy);
}

// Exact test of a candidate whose coarse stage already ran: `t_first` is the
// first root that survived it, `second` whether root 1 survived too,
// `marginal` the near-tangent flag.  Same decisions as hit_refined.
template <int M>
__device__ __forceinline__ bool hit_exact_from(const PrimRec &r, const Geo64 &g,
                                               const Geo64 *gfull, const double d64[3],
                                               float dx, float dy,
                                               float dz, bool euclid, float t_clip,
                                               float t_first, bool second, bool marginal,
                                               Hit &h)
{
    const bool planar = (r.flags & 1u) != 0;     // (near-tangent rays are never planar)
    double dh[3];
    local_dir64(g, d64, dh);
    if (planar && fabs(dh[2]) < 1e-12) return false;
    double ta, tb = 0.0;
    bool hb;
    if (marginal) {
        const Roots2 rr = marginal_roots(&g, dh[0], dh[1], dh[2]);
        if (rr.cnt == 0) return false;
        ta = rr.r0;
        tb = rr.r1;
        hb = rr.cnt == 2;
    } else {
        ta = refine_depth(g, dh, planar, t_first);
        hb = second;
    }
    if (confirm_root<M>(r, g, gfull, dh, ta, planar, euclid, t_clip, h)) return true;
    if (!hb) return false;
    if (!marginal) {
        float roots[2], hx, hy;
        coarse_stage1(r, dx, dy, dz, t_clip, roots, hx, hy);
        tb = refine_depth(g, dh, planar, roots[1]);
    }
    return confirm_root<M>(r, g, gfull, dh, tb, planar, euclid, t_clip, h);
}

// Full candidate test: coarse fp32 roots, fp64 refinement, exact selection.
// Returns the selected hit (valid, before the alpha floor) or false.
template <int M>
__device__ __forceinline__ bool hit_refined(const PrimRec &r, const Geo64 &g, const double d64[3],
                                            float dx, float dy, float dz, bool euclid,
                                            float t_clip, Hit &h)
{
    float roots[2], hx, hy, hz;
    const unsigned pass = coarse_roots(r, dx, dy, dz, euclid, t_clip, roots, hx, hy, hz);
    if (pass == 0u) return false;
    const bool planar = (r.flags & 1u) != 0;
    double dh[3];
    local_dir64(g, d64, dh);
    if (pass & CR_MARGINAL) {
        const Roots2 rr = marginal_roots(&g, dh[0], dh[1], dh[2]);
        for (int k = 0; k < rr.cnt; ++k)
            if (confirm_root<M>(r, g, &g, dh, k == 0 ? rr.r0 : rr.r1, false, euclid, t_clip, h))
                return true;
        return false;
    }
    if (planar && fabs(dh[2]) < 1e-12) return false;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (!(pass & (1u << k))) continue;
        double t64 = refine_depth(g, dh, planar, roots[k]);
        if (confirm_root<M>(r, g, &g, dh, t64, planar, euclid, t_clip, h)) return true;
    }
    return false;
}

// camera-frame camera-facing normal and Gaussian curvature at a hit
__device__ __forceinline__ void normal_curv32(const PrimRec &r, const Hit &h, float dx, float dy,
                                              float dz, float nl[3], float nc[3], float &K,
                                              float &inrm, float &flip)
{
    if (h.branch == BR_PLANAR) {
        nl[0] = 0.f; nl[1] = 0.f; nl[2] = -1.f; K = 0.f; inrm = 1.f;
    } else {
        float nx = 2.f * r.w1 * h.x, ny = 2.f * r.w2 * h.y, nz = -r.iw3;
        inrm = rsqrtf(fmaf(nx, nx, fmaf(ny, ny, nz * nz)));
        nl[0] = nx * inrm; nl[1] = ny * inrm; nl[2] = nz * inrm;
        float l1x = r.lam1 * h.x, l2y = r.lam2 * h.y;
        float den = 1.f + 4.f * fmaf(l1x, l1x, l2y * l2y);
        K = 4.f * r.lam1 * r.lam2 / (den * den);
    }
    // Nmat = M^T (camera-from-local)
    nc[0] = fmaf(r.M[0], nl[0], fmaf(r.M[3], nl[1], r.M[6] * nl[2]));
    nc[1] = fmaf(r.M[1], nl[0], fmaf(r.M[4], nl[1], r.M[7] * nl[2]));
    nc[2] = fmaf(r.M[2], nl[0], fmaf(r.M[5], nl[1], r.M[8] * nl[2]));
    flip = 1.f;
    if (fmaf(nc[0], dx, fmaf(nc[1], dy, nc[2] * dz)) > 0.f) {
        flip = -1.f; nc[0] = -nc[0]; nc[1] = -nc[1]; nc[2] = -nc[2];
    }
}

// camera-frame unit ray of pixel (u, v) in fp64 with the reference's
// operation order (cameras.py:53-59), no FMA contraction
__device__ __forceinline__ void pixel_dir64(const CamK &cam, int u, int v, double d[3])
{
    double a = __ddiv_rn(__dsub_rn(__dadd_rn((double)u, 0.5), cam.cx), cam.fx);
    double b = __ddiv_rn(__dsub_rn(__dadd_rn((double)v, 0.5), cam.cy), cam.fy);
    double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), 1.0));
    d[0] = __ddiv_rn(a, n); d[1] = __ddiv_rn(b, n); d[2] = __ddiv_rn(1.0, n);
}

__device__ __forceinline__ bool in_box(const PrimRec &r, int u, int v)
{
    int umin = (int)(r.bb_u & 0xffffu), umax = (int)(r.bb_u >> 16);
    int vmin = (int)(r.bb_v & 0xffffu), vmax = (int)(r.bb_v >> 16);
    return u >= umin && u <= umax && v >= vmin && v <= vmax;
}

}  // namespace qgs
