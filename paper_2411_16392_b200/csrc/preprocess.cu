// K1 per-primitive preprocessing and K7 chain-to-raw-parameters.
//
// One thread per primitive, float64 throughout; this translation unit is
// compiled with -fmad=false so products and sums round exactly as the
// reference's numpy expressions do (rasterizer.py:124-158, bounds.py:167-292,
// model.py:29-110, sh.py:22-99).  Outputs: the fp64 geometry used by the sort
// keys, the 128-byte fp32 raster record, the inclusive pixel box and the
// number of 16x16 tiles the box covers.
#include "qgs_common.cuh"

namespace qgs {

__device__ inline double sign0(double v) { return v < 0.0 ? -1.0 : 1.0; }

// quat_to_rot (model.py:70-87), normalised (w, x, y, z) -> row-major R
__device__ inline void quat_rot(const float *q4, double R[9], double qn[4], double &norm)
{
    double w = q4[0], x = q4[1], y = q4[2], z = q4[3];
    norm = sqrt(w * w + x * x + y * y + z * z);
    {   // four quotients, one divisor: one reciprocal (div_rcp, bit-identical)
        const double in = __drcp_rn(norm);
        QGS_CHECK(div_rcp(w, norm, in) == w / norm && div_rcp(z, norm, in) == z / norm);
        w = div_rcp(w, norm, in); x = div_rcp(x, norm, in);
        y = div_rcp(y, norm, in); z = div_rcp(z, norm, in);
    }
    qn[0] = w; qn[1] = x; qn[2] = y; qn[3] = z;
    R[0] = 1 - 2 * (y * y + z * z);
    R[1] = 2 * (x * y - w * z);
    R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);
    R[4] = 1 - 2 * (x * x + z * z);
    R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);
    R[7] = 2 * (y * z + w * x);
    R[8] = 1 - 2 * (x * x + y * y);
}

// activate_scales (model.py:29-45)
__device__ inline void activate(const float *rs, const float *rg, double s[3], bool clamped[3])
{
    for (int k = 0; k < 3; ++k) {
        s[k] = tanh((double)rg[k]) * exp((double)rs[k]);
        clamped[k] = false;
    }
    for (int k = 0; k < 2; ++k)
        if (fabs(s[k]) < 1e-4) { clamped[k] = true; s[k] = sign0(s[k]) * 1e-4; }
}

// real SH basis, degrees 0..3 (sh.py:22-46)
__device__ inline void sh_basis(int K, double x, double y, double z, double Y[16])
{
    const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    Y[0] = C0;
    if (K > 1) { Y[1] = -C1 * y; Y[2] = C1 * z; Y[3] = -C1 * x; }
    if (K > 4) {
        Y[4] = 1.0925484305920792 * x * y;
        Y[5] = -1.0925484305920792 * y * z;
        Y[6] = 0.31539156525252005 * (2 * z * z - x * x - y * y);
        Y[7] = -1.0925484305920792 * x * z;
        Y[8] = 0.5462742152960396 * (x * x - y * y);
    }
    if (K > 9) {
        Y[9] = -0.5900435899266435 * y * (3 * x * x - y * y);
        Y[10] = 2.890611442640554 * x * y * z;
        Y[11] = -0.4570457994644658 * y * (4 * z * z - x * x - y * y);
        Y[12] = 0.3731763325901154 * z * (2 * z * z - 3 * x * x - 3 * y * y);
        Y[13] = -0.4570457994644658 * x * (4 * z * z - x * x - y * y);
        Y[14] = 1.445305721320277 * z * (x * x - y * y);
        Y[15] = -0.5900435899266435 * x * (x * x - 3 * y * y);
    }
}

// d basis / d dir (sh.py:49-79), J[k][3]
__device__ inline void sh_basis_jac(int K, double x, double y, double z, double J[16][3])
{
    const double C1 = 0.4886025119029199;
    for (int k = 0; k < K; ++k) J[k][0] = J[k][1] = J[k][2] = 0.0;
    if (K > 1) { J[1][1] = -C1; J[2][2] = C1; J[3][0] = -C1; }
    if (K > 4) {
        const double a = 1.0925484305920792, b = -1.0925484305920792, c = 0.31539156525252005,
                     d = -1.0925484305920792, e = 0.5462742152960396;
        J[4][0] = a * y; J[4][1] = a * x;
        J[5][1] = b * z; J[5][2] = b * y;
        J[6][0] = -2 * c * x; J[6][1] = -2 * c * y; J[6][2] = 4 * c * z;
        J[7][0] = d * z; J[7][2] = d * x;
        J[8][0] = 2 * e * x; J[8][1] = -2 * e * y;
    }
    if (K > 9) {
        const double c0 = -0.5900435899266435, c1 = 2.890611442640554, c2 = -0.4570457994644658,
                     c3 = 0.3731763325901154, c4 = -0.4570457994644658, c5 = 1.445305721320277,
                     c6 = -0.5900435899266435;
        J[9][0] = 6 * c0 * x * y; J[9][1] = c0 * (3 * x * x - 3 * y * y);
        J[10][0] = c1 * y * z; J[10][1] = c1 * x * z; J[10][2] = c1 * x * y;
        J[11][0] = -2 * c2 * x * y; J[11][1] = c2 * (4 * z * z - x * x - 3 * y * y);
        J[11][2] = 8 * c2 * y * z;
        J[12][0] = -6 * c3 * x * z; J[12][1] = -6 * c3 * y * z;
        J[12][2] = c3 * (6 * z * z - 3 * x * x - 3 * y * y);
        J[13][0] = c4 * (4 * z * z - 3 * x * x - y * y); J[13][1] = -2 * c4 * x * y;
        J[13][2] = 8 * c4 * x * z;
        J[14][0] = 2 * c5 * x * z; J[14][1] = -2 * c5 * y * z; J[14][2] = c5 * (x * x - y * y);
        J[15][0] = c6 * (3 * x * x - 3 * y * y); J[15][1] = -6 * c6 * x * y;
    }
}

// inline solve_radius_for_sigma (geodesic.py:80-91 as bounds.py:177-178)
__device__ inline double support_radius(double a, double sig)
{
    return 14.0 * sig / (6.0 + sqrt(36.0 + 112.0 * a * sig));
}

// pixel AABB of 8 local corners (bounds.py:234-269); returns false when empty
__device__ inline void project_box(const double cs[8][3], const double R[9], const double c[3],
                                   const CamK &cam, long long box[4])
{
    bool any = false, all = true;
    double umin = 1e18, vmin = 1e18, umax = -1e18, vmax = -1e18;
    for (int k = 0; k < 8; ++k) {
        double w0 = R[0] * cs[k][0] + R[1] * cs[k][1] + R[2] * cs[k][2] + c[0];
        double w1 = R[3] * cs[k][0] + R[4] * cs[k][1] + R[5] * cs[k][2] + c[1];
        double w2 = R[6] * cs[k][0] + R[7] * cs[k][1] + R[8] * cs[k][2] + c[2];
        double X = w0 * cam.Rwc[0] + w1 * cam.Rwc[1] + w2 * cam.Rwc[2] + cam.twc[0];
        double Y = w0 * cam.Rwc[3] + w1 * cam.Rwc[4] + w2 * cam.Rwc[5] + cam.twc[1];
        double Z = w0 * cam.Rwc[6] + w1 * cam.Rwc[7] + w2 * cam.Rwc[8] + cam.twc[2];
        if (Z > 1e-6) {
            any = true;
            // both coordinates divide by Z: one reciprocal (div_rcp)
            const double iz = __drcp_rn(Z);
            double u = div_rcp(cam.fx * X, Z, iz) + cam.cx, v = div_rcp(cam.fy * Y, Z, iz) + cam.cy;
            QGS_CHECK(u == cam.fx * X / Z + cam.cx && v == cam.fy * Y / Z + cam.cy);
            umin = fmin(umin, u); umax = fmax(umax, u);
            vmin = fmin(vmin, v); vmax = fmax(vmax, v);
        } else {
            all = false;
        }
    }
    double lu = fmin(fmax(floor(umin - 0.5), 0.0), (double)(cam.W - 1));
    double hu = fmin(fmax(ceil(umax - 0.5), 0.0), (double)(cam.W - 1));
    double lv = fmin(fmax(floor(vmin - 0.5), 0.0), (double)(cam.H - 1));
    double hv = fmin(fmax(ceil(vmax - 0.5), 0.0), (double)(cam.H - 1));
    box[0] = (long long)lu; box[1] = (long long)hu; box[2] = (long long)lv; box[3] = (long long)hv;
    if (any && !all) { box[0] = 0; box[1] = cam.W - 1; box[2] = 0; box[3] = cam.H - 1; }
    if (!any || box[0] > box[1] || box[2] > box[3]) { box[0] = 0; box[1] = -1; box[2] = 0; box[3] = -1; }
}

// tight_bboxes_batch for one primitive (bounds.py:272-292)
__device__ inline void tight_box(const double s[3], const double R[9], const double c[3],
                                 const CamK &cam, long long out[4])
{
    double m1 = fabs(s[0]), m2 = fabs(s[1]), m3 = fabs(s[2]);
    double a0 = s[2] * sign0(s[0]) / (s[0] * s[0]);
    double a1 = s[2] * sign0(s[1]) / (s[1] * s[1]);
    bool flat = m3 < 1e-6;
    double big = fmax(m1, m2), small = fmin(m1, m2);
    // loose support box
    double amin = a0 * a1 < 0 ? 0.0 : fmin(fabs(a0), fabs(a1));
    double amax = fmax(fabs(a0), fabs(a1));
    double r1 = flat ? 3.0 * m1 : support_radius(amin, 3.0 * m1);
    double r2 = flat ? 3.0 * m2 : support_radius(amin, 3.0 * m2);
    double zb = fmax(0.0, (21.0 * big - 6.0 * support_radius(amax, 3.0 * small)) / 4.0);
    double zlo = flat ? 0.0 : ((a0 < 0 || a1 < 0) ? -zb : 0.0);
    double zhi = flat ? 0.0 : ((a0 > 0 || a1 > 0) ? zb : 0.0);
    double cs[8][3];
    int k = 0;
    for (int ex = -1; ex <= 1; ex += 2)
        for (int ey = -1; ey <= 1; ey += 2)
            for (int ez = 0; ez < 2; ++ez) {
                cs[k][0] = ex * r1; cs[k][1] = ey * r2; cs[k][2] = ez ? zhi : zlo;
                ++k;
            }
    long long loose[4];
    project_box(cs, R, c, cam, loose);
    // tangent-plane frustum (elliptic case)
    bool ok = (m3 >= 1e-6) && (a0 * a1 > 0) && (fmin(fabs(a0), fabs(a1)) >= 1e-9);
    for (int j = 0; j < 4; ++j) out[j] = loose[j];
    if (!ok) {
        if (out[0] > out[1] || out[2] > out[3]) { out[0] = 0; out[1] = -1; out[2] = 0; out[3] = -1; }
        return;
    }
    double zs = a0 > 0 ? 1.0 : -1.0;
    double A0 = fabs(a0), A1 = fabs(a1);
    double q1 = support_radius(A0, 3.0 * m1), q2 = support_radius(A1, 3.0 * m2);
    double zb2 = fmax(0.0, (21.0 * big - 6.0 * support_radius(fmax(A0, A1), 3.0 * small)) / 4.0);
    double h = fmax(zb2, fmax(A0 * (q1 * q1), A1 * (q2 * q2)));
    double e1 = (h / A0 + q1 * q1) / (2.0 * q1), e2 = (h / A1 + q2 * q2) / (2.0 * q2);
    k = 0;
    for (int ex = -1; ex <= 1; ex += 2)
        for (int ey = -1; ey <= 1; ey += 2) {
            cs[k][0] = ex * q1 / 2; cs[k][1] = ey * q2 / 2; cs[k][2] = 0.0;
            cs[k + 4][0] = ex * e1; cs[k + 4][1] = ey * e2; cs[k + 4][2] = zs * h;
            ++k;
        }
    long long fr[4];
    project_box(cs, R, c, cam, fr);
    bool live_l = loose[0] <= loose[1];
    if (live_l && fr[0] <= fr[1]) {
        out[0] = max(loose[0], fr[0]); out[1] = min(loose[1], fr[1]);
        out[2] = max(loose[2], fr[2]); out[3] = min(loose[3], fr[3]);
    }
    if (live_l && (fr[0] > fr[1] || fr[2] > fr[3])) { out[0] = 0; out[1] = -1; out[2] = 0; out[3] = -1; }
    if (out[0] > out[1] || out[2] > out[3]) { out[0] = 0; out[1] = -1; out[2] = 0; out[3] = -1; }
}

// Bounding ellipsoid of everything the selection rule can accept
// (intersect.py:58-115), in the primitive's local frame: centre (0, 0, zc),
// semi-axes ax, ay, az.  A hit at local (x, y, z) on the quadric passes the
// 3-sigma test l <= 3 sigma(theta), and the arc length l is at least the
// chord from the vertex, sqrt(rho^2 + z^2), while sigma(theta) <= max|s_i|:
//   E1: (x/3s1)^2 + (y/3s2)^2 + (z/3 smax)^2 <= rho^2/(9 sigma^2) + z^2/(9 sigma^2) <= 1.
// Independently rho <= l <= 3 sigma(theta) puts (x, y) in the ellipse
// (x/3s1)^2 + (y/3s2)^2 <= 1, on which z = s3 (w1 x^2 + w2 y^2) lies in
// [zlo, zhi]; for 0 < lam < 1 the cylinder-slab is inside
//   E2: lam (x/3s1)^2 + lam (y/3s2)^2 + (1 - lam) ((z - zc)/h)^2 <= 1.
// E2 is the only one in Euclidean-density mode (no chord bound) and for
// planar primitives (h = 0: the disk itself); otherwise the smaller volume.
__device__ inline void bounding_ellipsoid(const double s[3], bool planar, bool euclid,
                                          double &zc, double ax[3])
{
    const double m1 = fabs(s[0]), m2 = fabs(s[1]), smax = fmax(m1, m2);
    if (planar) { zc = 0.0; ax[0] = 3.0 * m1; ax[1] = 3.0 * m2; ax[2] = 0.0; return; }
    // range of w1 x^2 + w2 y^2 = sgn(s1)(x/s1)^2 + sgn(s2)(y/s2)^2 on the ellipse: [lo, hi] * 9
    const double g1 = s[0] < 0.0 ? -1.0 : 1.0, g2 = s[1] < 0.0 ? -1.0 : 1.0;
    const double lo = fmin(0.0, fmin(g1, g2)), hi = fmax(0.0, fmax(g1, g2));
    double z0 = 9.0 * s[2] * (s[2] >= 0.0 ? lo : hi), z1 = 9.0 * s[2] * (s[2] >= 0.0 ? hi : lo);
    if (!euclid) { z0 = fmax(z0, -3.0 * smax); z1 = fmin(z1, 3.0 * smax); }
    const double h = 0.5 * (z1 - z0);
    const double lam = 0.75;
    // volumes: E1 27 m1 m2 smax, E2 9 m1 m2 h / (lam sqrt(1 - lam))
    if (!euclid && 27.0 * smax <= 9.0 * h / (lam * sqrt(1.0 - lam))) {
        zc = 0.0; ax[0] = 3.0 * m1; ax[1] = 3.0 * m2; ax[2] = 3.0 * smax;
        return;
    }
    zc = 0.5 * (z0 + z1);
    const double il = 1.0 / sqrt(lam);
    ax[0] = 3.0 * m1 * il; ax[1] = 3.0 * m2 * il; ax[2] = h / sqrt(1.0 - lam);
}

// 0.1% slack on every axis: the linear-branch root (|A| < 1e-6, t = -C/B)
// sits A t^2 ~ 1e-5 off the quadric, and fp64 rounding
__device__ inline void pad_axes(double ax[3]) { for (int k = 0; k < 3; ++k) ax[k] *= 1.001; }

// Pixel-centre conic bounding the screen footprint of the bounding ellipsoid
// E (centre mc, camera-frame axes Ri scaled by ax).  A pixel whose ray line
// misses E cannot be accepted.  Non-planar E: the line through the eye along
// d meets E iff (d.A c)^2 - (d.A d)(c.A c - 1) >= 0 (A = E's shape matrix, c
// its centre): exact for any E position once the eye is outside E, also for
// an E that straddles the camera plane (its footprint is then a hyperbola,
// left unbounded).  Planar E (a disk): the outline of the dual quadric,
// C* = Mq Mq^T - m m^T, point conic = adj(C*), for a disk in front of the
// camera.  The conic is taken about pixel-centre origin (u0, v0), normalised,
// and widened by its fp32 evaluation margin; an elliptic footprint also
// tightens the pixel box.  No cull (F = -1) when neither form applies.
__device__ inline ConicRec bounding_conic(const double s[3], bool planar, bool euclid,
                                          const double R[9], const double c[3],
                                          const CamK &cam, const long long box[4])
{
    ConicRec q;
    q.A = q.B = q.C = q.D = q.E = 0.f;
    q.F = -1.f;
    if (box[0] > box[1]) { q.bb_u = 0xffffu; q.bb_v = 0xffffu; return q; }
    q.bb_u = (uint32_t)box[0] | ((uint32_t)box[1] << 16);
    q.bb_v = (uint32_t)box[2] | ((uint32_t)box[3] << 16);
    double zc, ax[3];
    bounding_ellipsoid(s, planar, euclid, zc, ax);
    pad_axes(ax);
    // centre and axes in camera coordinates
    double cw[3], Ri[3][3], mc[3];
    for (int i = 0; i < 3; ++i) cw[i] = c[i] + zc * R[3 * i + 2];
    for (int i = 0; i < 3; ++i) {
        mc[i] = cam.Rwc[3 * i] * cw[0] + cam.Rwc[3 * i + 1] * cw[1] + cam.Rwc[3 * i + 2] * cw[2] + cam.twc[i];
        for (int k = 0; k < 3; ++k)
            Ri[i][k] = cam.Rwc[3 * i] * R[k] + cam.Rwc[3 * i + 1] * R[3 + k] + cam.Rwc[3 * i + 2] * R[6 + k];
    }
    const bool disk = !(ax[2] > 0.0);
    double K[3][3];                       // quadratic form on camera rays d: >= 0 possible hit
    if (!disk) {
        double A[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double acc = 0.0;
                for (int k = 0; k < 3; ++k) acc += Ri[i][k] * Ri[j][k] / (ax[k] * ax[k]);
                A[i][j] = acc;
            }
        double ac[3];
        for (int i = 0; i < 3; ++i) ac[i] = A[i][0] * mc[0] + A[i][1] * mc[1] + A[i][2] * mc[2];
        const double cac = ac[0] * mc[0] + ac[1] * mc[1] + ac[2] * mc[2];
        const double gamma = cac - 1.0;
        if (!(gamma > 1e-6 * cac)) return q;        // eye inside E: every line hits
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) K[i][j] = ac[i] * ac[j] - gamma * A[i][j];
    } else {
        // disk: dual-quadric outline, in front of the camera plane only
        double Mc[3][3];
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k) Mc[i][k] = Ri[i][k] * ax[k];
        const double zr = sqrt(Mc[2][0] * Mc[2][0] + Mc[2][1] * Mc[2][1]);
        if (!(mc[2] - zr > 1e-6 * fmax(mc[2], 1e-30))) return q;
        double D[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                D[i][j] = Mc[i][0] * Mc[j][0] + Mc[i][1] * Mc[j][1] - mc[i] * mc[j];
        // adjugate = point conic (up to sign); orient: the centre ray must be inside
        double P[3][3];
        P[0][0] = D[1][1] * D[2][2] - D[1][2] * D[2][1];
        P[0][1] = P[1][0] = D[0][2] * D[2][1] - D[0][1] * D[2][2];
        P[0][2] = P[2][0] = D[0][1] * D[1][2] - D[0][2] * D[1][1];
        P[1][1] = D[0][0] * D[2][2] - D[0][2] * D[2][0];
        P[1][2] = P[2][1] = D[0][2] * D[1][0] - D[0][0] * D[1][2];
        P[2][2] = D[0][0] * D[1][1] - D[0][1] * D[1][0];
        double at_c = 0.0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) at_c += mc[i] * P[i][j] * mc[j];
        const double sg = at_c > 0.0 ? 1.0 : -1.0;    // make the centre ray positive
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) K[i][j] = sg * P[i][j];
    }
    // Normalised pixel conic about pixel-centre origin (u0, v0): Q(U, V) =
    // A U^2 + B U V + C V^2 + D U + E V + F <= 0 possible, U = (pixel centre u) - u0
    double Q6[6];
    auto conic_about = [&](double u0, double v0) -> bool {
        // d = T (U, V, 1): u' = (U + u0 - cx) / fx, v' = (V + v0 - cy) / fy
        const double T[3][3] = {{1.0 / cam.fx, 0.0, (u0 - cam.cx) / cam.fx},
                                {0.0, 1.0 / cam.fy, (v0 - cam.cy) / cam.fy},
                                {0.0, 0.0, 1.0}};
        double KT[3][3], Kp[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                KT[i][j] = K[i][0] * T[0][j] + K[i][1] * T[1][j] + K[i][2] * T[2][j];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                Kp[i][j] = T[0][i] * KT[0][j] + T[1][i] * KT[1][j] + T[2][i] * KT[2][j];
        const double nrm = fmax(fabs(Kp[0][0]), fabs(Kp[1][1]));
        if (!(nrm > 0.0) || !isfinite(nrm)) return false;
        const double k = -1.0 / nrm;
        Q6[0] = Kp[0][0] * k; Q6[1] = 2.0 * Kp[0][1] * k; Q6[2] = Kp[1][1] * k;
        Q6[3] = 2.0 * Kp[0][2] * k; Q6[4] = 2.0 * Kp[1][2] * k; Q6[5] = Kp[2][2] * k;
        return true;
    };
    // 1. about the reference box centre; an ellipse tightens the box to its
    //    own pixel bounds (centre from grad Q = 0, half extents
    //    sqrt(-Q(c) C / det), sqrt(-Q(c) A / det)) plus one pixel each side
    double uc = (double)conic_uc(q), vc = (double)conic_vc(q);
    if (!conic_about(uc + 0.5, vc + 0.5)) return q;
    {
        const double A = Q6[0], B = Q6[1], C = Q6[2], Dd = Q6[3], E = Q6[4], F = Q6[5];
        const double det2 = 4.0 * A * C - B * B;
        if (A > 0.0 && C > 0.0 && det2 > 0.0) {
            const double U0 = (B * E - 2.0 * C * Dd) / det2, V0 = (B * Dd - 2.0 * A * E) / det2;
            const double kq = -(A * U0 * U0 + B * U0 * V0 + C * V0 * V0 + Dd * U0 + E * V0 + F);
            if (!(kq > 0.0)) {                           // empty footprint
                q.bb_u = 0xffffu; q.bb_v = 0xffffu;
                return q;
            }
            const double hu = sqrt(kq * 4.0 * C / det2), hv = sqrt(kq * 4.0 * A / det2);
            const double lo_u = floor(uc + U0 - hu) - 1.0, hi_u = ceil(uc + U0 + hu) + 1.0;
            const double lo_v = floor(vc + V0 - hv) - 1.0, hi_v = ceil(vc + V0 + hv) + 1.0;
            if (isfinite(lo_u) && isfinite(hi_u) && isfinite(lo_v) && isfinite(hi_v)) {
                const long long b0 = max(box[0], (long long)fmax(lo_u, -1.0));
                const long long b1 = min(box[1], (long long)fmin(hi_u, 1e9));
                const long long b2 = max(box[2], (long long)fmax(lo_v, -1.0));
                const long long b3 = min(box[3], (long long)fmin(hi_v, 1e9));
                if (b0 > b1 || b2 > b3) {        // nothing in the reference box can be accepted
                    q.bb_u = 0xffffu; q.bb_v = 0xffffu;
                    return q;
                }
                q.bb_u = (uint32_t)b0 | ((uint32_t)b1 << 16);
                q.bb_v = (uint32_t)b2 | ((uint32_t)b3 << 16);
            }
        }
    }
    // 2. the conic about the final box's centre, with the fp32 margin
    uc = (double)conic_uc(q); vc = (double)conic_vc(q);
    if (!conic_about(uc + 0.5, vc + 0.5)) {
        q.bb_u = (uint32_t)box[0] | ((uint32_t)box[1] << 16);      // no cull after all
        q.bb_v = (uint32_t)box[2] | ((uint32_t)box[3] << 16);
        return q;
    }
    const double hu = 0.5 * (double)((q.bb_u >> 16) - (q.bb_u & 0xffffu)) + 1.0;
    const double hv = 0.5 * (double)((q.bb_v >> 16) - (q.bb_v & 0xffffu)) + 1.0;
    const double mag = fabs(Q6[0]) * hu * hu + fabs(Q6[1]) * hu * hv + fabs(Q6[2]) * hv * hv +
                       fabs(Q6[3]) * hu + fabs(Q6[4]) * hv + fabs(Q6[5]);
    q.A = (float)Q6[0]; q.B = (float)Q6[1]; q.C = (float)Q6[2]; q.D = (float)Q6[3]; q.E = (float)Q6[4];
    q.F = (float)(Q6[5] - 2e-5 * mag);
    if (!isfinite(q.A + q.B + q.C + q.D + q.E + q.F)) {
        q.A = q.B = q.C = q.D = q.E = 0.f;
        q.F = -1.f;
        q.bb_u = (uint32_t)box[0] | ((uint32_t)box[1] << 16);
        q.bb_v = (uint32_t)box[2] | ((uint32_t)box[3] << 16);
    }
    return q;
}

#ifndef QGS_PRE_MIN_BLOCKS
#define QGS_PRE_MIN_BLOCKS 1
#endif
#ifndef QGS_CHAIN_MIN_BLOCKS
#define QGS_CHAIN_MIN_BLOCKS 1
#endif
// SH colour of primitive p seen along the unit direction vd (sh.py:82-88)
__device__ __forceinline__ void sh_colour(const qgs_params &prm, int p, const double vd[3],
                                          double col[3])
{
    int K = prm.sh_coeffs;
    double Y[16];
    sh_basis(K, vd[0], vd[1], vd[2], Y);
    const float *shp = prm.sh + (size_t)p * 3 * K;
    for (int ch = 0; ch < 3; ++ch) {
        double acc = 0.0;
        for (int k = 0; k < K; ++k) acc += (double)shp[ch * K + k] * Y[k];
        acc = acc + 0.5;
        col[ch] = acc < 0 ? 0.0 : acc;
    }
}

// with_color = 0: everything but the SH colour (left 0; color_kernel fills it
// in once the coefficients are on the device -- their upload, ~3/4 of the
// parameter bytes at SH degree 3, then overlaps the binning)
__global__ void __launch_bounds__(128, QGS_PRE_MIN_BLOCKS)
preprocess_kernel(qgs_params prm, CamK cam, PrepView pv, int euclid, int with_color)
{
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= prm.P) return;
    const float *cf = prm.centers + 3 * p;
    double c[3] = {cf[0], cf[1], cf[2]};
    double s[3];
    bool clamped[3];
    activate(prm.raw_scales + 3 * p, prm.raw_signs + 3 * p, s, clamped);
    {   // model.py:37-38 (ParameterError): counted here, raised by the host
        // from the pair-count read it makes anyway (no extra sync)
        bool fin = true;
        for (int k = 0; k < 3; ++k)
            fin = fin && isfinite(prm.raw_scales[3 * p + k]) && isfinite(prm.raw_signs[3 * p + k]);
        if (!fin) atomicAdd(pv.nonfinite, 1);
    }
    double alpha = 1.0 / (1.0 + exp(-(double)prm.raw_opacity[p]));
    double R[9], qn[4], qnorm;
    quat_rot(prm.quats + 4 * p, R, qn, qnorm);
    bool planar = fabs(s[2]) < 1e-6;
    double w1 = sign0(s[0]) / (s[0] * s[0]);
    double w2 = sign0(s[1]) / (s[1] * s[1]);
    double iw3 = planar ? 0.0 : 1.0 / s[2];
    double lam1 = s[2] * w1, lam2 = s[2] * w2;
    double e[3] = {cam.eye[0] - c[0], cam.eye[1] - c[1], cam.eye[2] - c[2]};
    Geo64 g;
    for (int i = 0; i < 3; ++i) g.ohat[i] = R[0 + i] * e[0] + R[3 + i] * e[1] + R[6 + i] * e[2];
    // M = R^T R_cw, R_cw = R_wc^T  ->  M[i][k] = sum_j R[j][i] Rwc[k][j]
    for (int i = 0; i < 3; ++i)
        for (int kk = 0; kk < 3; ++kk)
            g.M[3 * i + kk] = R[0 + i] * cam.Rwc[3 * kk + 0] + R[3 + i] * cam.Rwc[3 * kk + 1] +
                              R[6 + i] * cam.Rwc[3 * kk + 2];
    g.wv[0] = w1; g.wv[1] = w2; g.wv[2] = iw3;
    g.sv[0] = s[0]; g.sv[1] = s[1]; g.sv[2] = s[2];
    double v[3] = {c[0] - cam.eye[0], c[1] - cam.eye[1], c[2] - cam.eye[2]};
    double dist = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    dist = fmax(dist, 1e-12);
    g.dist = dist;
    const double idist = __drcp_rn(dist);
    double vd[3] = {div_rcp(v[0], dist, idist), div_rcp(v[1], dist, idist), div_rcp(v[2], dist, idist)};
    QGS_CHECK(vd[0] == v[0] / dist && vd[1] == v[1] / dist && vd[2] == v[2] / dist);
    // SH colour (sh.py:82-88)
    if (with_color) sh_colour(prm, p, vd, g.col);
    else g.col[0] = g.col[1] = g.col[2] = 0.0;
    g.alpha = alpha;
    g.planar = planar ? 1.0 : 0.0;
    // projected vertex (cameras.py:73-79)
    double X = c[0] * cam.Rwc[0] + c[1] * cam.Rwc[1] + c[2] * cam.Rwc[2] + cam.twc[0];
    double Yc = c[0] * cam.Rwc[3] + c[1] * cam.Rwc[4] + c[2] * cam.Rwc[5] + cam.twc[1];
    double Z = c[0] * cam.Rwc[6] + c[1] * cam.Rwc[7] + c[2] * cam.Rwc[8] + cam.twc[2];
    const double iZ = __drcp_rn(Z);
    g.vert_u = div_rcp(cam.fx * X, Z, iZ) + cam.cx;
    g.vert_v = div_rcp(cam.fy * Yc, Z, iZ) + cam.cy;
    QGS_CHECK(g.vert_u == cam.fx * X / Z + cam.cx && g.vert_v == cam.fy * Yc / Z + cam.cy);
    for (int i = 0; i < 6; ++i) g.pad[i] = 0.0;
    pv.geo[p] = g;

    long long box[4];
    tight_box(s, R, c, cam, box);
    pv.bbox[p] = make_int4((int)box[0], (int)box[1], (int)box[2], (int)box[3]);
    int nt = 0;
    if (box[0] <= box[1])
        nt = (int)((box[1] / TILE - box[0] / TILE + 1) * (box[3] / TILE - box[2] / TILE + 1));
    pv.ntiles[p] = nt;

    PrimRec r;
    for (int i = 0; i < 9; ++i) r.M[i] = (float)g.M[i];
    r.ox = (float)g.ohat[0]; r.oy = (float)g.ohat[1]; r.oz = (float)g.ohat[2];
    r.w1 = (float)w1; r.w2 = (float)w2; r.iw3 = (float)iw3;
    r.s1 = (float)s[0]; r.s2 = (float)s[1]; r.s3 = (float)s[2];
    r.lam1 = (float)lam1; r.lam2 = (float)lam2;
    r.alpha = (float)alpha;
    r.C = (float)(w1 * g.ohat[0] * g.ohat[0] + w2 * g.ohat[1] * g.ohat[1] - iw3 * g.ohat[2]);
    for (int ch = 0; ch < 3; ++ch) r.col[ch] = (float)g.col[ch];
    if (box[0] <= box[1]) {
        r.bb_u = (uint32_t)box[0] | ((uint32_t)box[1] << 16);
        r.bb_v = (uint32_t)box[2] | ((uint32_t)box[3] << 16);
    } else {
        r.bb_u = 0xffffu; r.bb_v = 0xffffu;   // umin > umax: never inside
    }
    r.flags = planar ? 1u : 0u;
    double s12 = fabs(s[0] * s[1]);
    r.s12 = (float)s12;
    r.ell9 = (float)(9.0 * s12 * s12);
    r.pad[0] = r.pad[1] = 0.f;
    pv.rec[p] = r;
    pv.conic[p] = bounding_conic(s, planar, euclid != 0, R, c, cam, box);
}

// the SH colour of every primitive (preprocess_kernel's with_color part, the
// same operations): Geo64.col and PrimRec.col
__global__ void __launch_bounds__(128)
color_kernel(qgs_params prm, CamK cam, PrepView pv)
{
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= prm.P) return;
    const float *cf = prm.centers + 3 * p;
    double c[3] = {cf[0], cf[1], cf[2]};
    double v[3] = {c[0] - cam.eye[0], c[1] - cam.eye[1], c[2] - cam.eye[2]};
    double dist = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    dist = fmax(dist, 1e-12);
    const double idist = __drcp_rn(dist);
    double vd[3] = {div_rcp(v[0], dist, idist), div_rcp(v[1], dist, idist), div_rcp(v[2], dist, idist)};
    QGS_CHECK(vd[0] == v[0] / dist && vd[1] == v[1] / dist && vd[2] == v[2] / dist);
    double col[3];
    sh_colour(prm, p, vd, col);
    for (int ch = 0; ch < 3; ++ch) {
        pv.geo[p].col[ch] = col[ch];
        pv.rec[p].col[ch] = (float)col[ch];
    }
}

// ------------------------------------------------------------- K7 chain

__global__ void __launch_bounds__(128, QGS_CHAIN_MIN_BLOCKS)
chain_kernel(qgs_params prm, CamK cam, const float *__restrict__ kg,
                             qgs_grads out)
{
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= prm.P) return;
    const float *g = kg + (size_t)p * KG;
    double gk[KG];
    bool any = false;
    for (int i = 0; i < KG; ++i) { gk[i] = g[i]; any |= g[i] != 0.f; }
    if (!any) return;   // no fragment of this primitive was composited

    const float *cf = prm.centers + 3 * p;
    double c[3] = {cf[0], cf[1], cf[2]};
    double s[3];
    bool clamped[3];
    activate(prm.raw_scales + 3 * p, prm.raw_signs + 3 * p, s, clamped);
    double alpha = 1.0 / (1.0 + exp(-(double)prm.raw_opacity[p]));
    double R[9], qn[4], qnorm;
    quat_rot(prm.quats + 4 * p, R, qn, qnorm);
    bool planar = fabs(s[2]) < 1e-6;
    double w1 = sign0(s[0]) / (s[0] * s[0]);
    double w2 = sign0(s[1]) / (s[1] * s[1]);

    // w_k = sign(s_k)/s_k^2, iw3 = 1/s3  (rasterizer.py:294-297)
    double gs0 = gk[KG_S + 0] + gk[KG_W + 0] * (-2.0 * w1 / s[0]);
    double gs1 = gk[KG_S + 1] + gk[KG_W + 1] * (-2.0 * w2 / s[1]);
    double gs2 = gk[KG_S + 2] + (planar ? 0.0 : gk[KG_W + 2] * (-1.0 / (s[2] * s[2])));
    double gsv[3] = {gs0, gs1, gs2};
    for (int k = 0; k < 3; ++k) {
        double th = tanh((double)prm.raw_signs[3 * p + k]);
        double ex = exp((double)prm.raw_scales[3 * p + k]);
        out.raw_scales[3 * p + k] += clamped[k] ? 0.f : (float)(gsv[k] * (th * ex));
        out.raw_signs[3 * p + k] += clamped[k] ? 0.f : (float)(gsv[k] * ((1.0 - th * th) * ex));
    }
    out.raw_opacity[p] += (float)(gk[KG_ALPHA] * alpha * (1.0 - alpha));

    // rotation (rasterizer.py:308-311): the reference's g_R equals R X with
    // X = sum x_loc (x) g_ohat + dhat (x) dl + g_nl (x) nl
    // (= R^T [R_cw g_M^T + (eye - c) g_ohat^T + R_cw g_Nmat]).  The raster
    // kernel accumulates only omega = vee(X - X^T); the symmetric part of X
    // changes nothing below (it moves R along q, which the normalisation
    // projects out), so X is replaced by its skew part (X - X^T) / 2.
    const double om0 = gk[KG_ROT + 0], om1 = gk[KG_ROT + 1], om2 = gk[KG_ROT + 2];
    const double Xs[9] = {0.0, 0.5 * om2, -0.5 * om1,
                          -0.5 * om2, 0.0, 0.5 * om0,
                          0.5 * om1, -0.5 * om0, 0.0};
    double gR[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double acc = 0.0;
            for (int j = 0; j < 3; ++j) acc += R[3 * a + j] * Xs[3 * j + b];
            gR[3 * a + b] = acc;
        }
    // quat_rot_backward (model.py:90-110)
    double w = qn[0], x = qn[1], y = qn[2], z = qn[3];
    const double dW[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0};
    const double dX[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x};
    const double dY[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y};
    const double dZ[9] = {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0};
    double gu[4] = {0, 0, 0, 0};
    for (int i = 0; i < 9; ++i) {
        gu[0] += gR[i] * dW[i]; gu[1] += gR[i] * dX[i];
        gu[2] += gR[i] * dY[i]; gu[3] += gR[i] * dZ[i];
    }
    double dq = gu[0] * qn[0] + gu[1] * qn[1] + gu[2] * qn[2] + gu[3] * qn[3];
    const double iqn = __drcp_rn(qnorm);
    for (int i = 0; i < 4; ++i) out.quats[4 * p + i] += (float)div_rcp(gu[i] - qn[i] * dq, qnorm, iqn);

    // centres through ohat and the SH view direction
    double gc[3];
    for (int i = 0; i < 3; ++i)
        gc[i] = -(R[3 * i + 0] * gk[KG_OHAT + 0] + R[3 * i + 1] * gk[KG_OHAT + 1] +
                  R[3 * i + 2] * gk[KG_OHAT + 2]);
    double v[3] = {c[0] - cam.eye[0], c[1] - cam.eye[1], c[2] - cam.eye[2]};
    double dist = fmax(sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]), 1e-12);
    const double idist = __drcp_rn(dist);
    double vd[3] = {div_rcp(v[0], dist, idist), div_rcp(v[1], dist, idist), div_rcp(v[2], dist, idist)};
    QGS_CHECK(vd[0] == v[0] / dist && vd[1] == v[1] / dist && vd[2] == v[2] / dist);
    int K = prm.sh_coeffs;
    double Y[16], J[16][3];
    sh_basis(K, vd[0], vd[1], vd[2], Y);
    sh_basis_jac(K, vd[0], vd[1], vd[2], J);
    const float *shp = prm.sh + (size_t)p * 3 * K;
    float *gsh = out.sh + (size_t)p * 3 * K;
    double gdir[3] = {0, 0, 0};
    for (int ch = 0; ch < 3; ++ch) {
        double raw = 0.0;
        for (int k = 0; k < K; ++k) raw += (double)shp[ch * K + k] * Y[k];
        raw += 0.5;
        double gcol = raw < 0 ? 0.0 : gk[KG_COLOR + ch];
        if (gcol == 0.0) continue;
        for (int k = 0; k < K; ++k) {
            gsh[ch * K + k] += (float)(gcol * Y[k]);
            for (int d = 0; d < 3; ++d) gdir[d] += gcol * shp[ch * K + k] * J[k][d];
        }
    }
    double dd = gdir[0] * vd[0] + gdir[1] * vd[1] + gdir[2] * vd[2];
    for (int i = 0; i < 3; ++i) gc[i] += div_rcp(gdir[i] - vd[i] * dd, dist, idist);
    for (int i = 0; i < 3; ++i) out.centers[3 * p + i] += (float)gc[i];

    // screen-space centre gradient (rasterizer.py:323-333)
    double X = c[0] * cam.Rwc[0] + c[1] * cam.Rwc[1] + c[2] * cam.Rwc[2] + cam.twc[0];
    double Yc = c[0] * cam.Rwc[3] + c[1] * cam.Rwc[4] + c[2] * cam.Rwc[5] + cam.twc[1];
    double Z = c[0] * cam.Rwc[6] + c[1] * cam.Rwc[7] + c[2] * cam.Rwc[8] + cam.twc[2];
    double Zs = fabs(Z) < 1e-9 ? 1e-9 : Z;
    const double Zs2 = Zs * Zs, iZs = __drcp_rn(Zs), iZs2 = __drcp_rn(Zs2);
    double gu_s = 0.0, gv_s = 0.0;
    for (int i = 0; i < 3; ++i) {
        double Ju = cam.fx * (div_rcp(cam.Rwc[i], Zs, iZs) - div_rcp(X * cam.Rwc[6 + i], Zs2, iZs2));
        double Jv = cam.fy * (div_rcp(cam.Rwc[3 + i], Zs, iZs) - div_rcp(Yc * cam.Rwc[6 + i], Zs2, iZs2));
        QGS_CHECK(Ju == cam.fx * (cam.Rwc[i] / Zs - X * cam.Rwc[6 + i] / (Zs * Zs)));
        gu_s += Ju * gc[i];
        gv_s += Jv * gc[i];
    }
    out.screen_center[2 * p + 0] += (float)(gu_s * (2.0 / cam.W));
    out.screen_center[2 * p + 1] += (float)(gv_s * (2.0 / cam.H));
}

// ------------------------------------------------------------- exports

__global__ void export_prep_kernel(PrepView pv, int P, double *scales, double *alphas,
                                   double *colors, int32_t *bbox, uint8_t *planar)
{
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const Geo64 &g = pv.geo[p];
    if (scales) for (int i = 0; i < 3; ++i) scales[3 * p + i] = g.sv[i];
    if (alphas) alphas[p] = g.alpha;
    if (colors) for (int i = 0; i < 3; ++i) colors[3 * p + i] = g.col[i];
    if (bbox) {
        int4 b = pv.bbox[p];
        bbox[4 * p] = b.x; bbox[4 * p + 1] = b.y; bbox[4 * p + 2] = b.z; bbox[4 * p + 3] = b.w;
    }
    if (planar) planar[p] = g.planar != 0.0 ? 1 : 0;
}

// the rest of PreparedView (rasterizer.py:124-147), same fp64 functions
__global__ void export_geom_kernel(qgs_params prm, CamK cam, PrepView pv, qgs_prep_export o)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= prm.P) return;
    const Geo64 &g = pv.geo[p];
    double s[3];
    bool clamped[3];
    activate(prm.raw_scales + 3 * p, prm.raw_signs + 3 * p, s, clamped);
    double R[9], qn[4], qnorm;
    quat_rot(prm.quats + 4 * p, R, qn, qnorm);
    if (o.R) for (int i = 0; i < 9; ++i) o.R[9 * (size_t)p + i] = R[i];
    if (o.ohat) for (int i = 0; i < 3; ++i) o.ohat[3 * (size_t)p + i] = g.ohat[i];
    if (o.M) for (int i = 0; i < 9; ++i) o.M[9 * (size_t)p + i] = g.M[i];
    if (o.wv) for (int i = 0; i < 3; ++i) o.wv[3 * (size_t)p + i] = g.wv[i];
    if (o.lam) { o.lam[2 * (size_t)p] = g.sv[2] * g.wv[0]; o.lam[2 * (size_t)p + 1] = g.sv[2] * g.wv[1]; }
    if (o.clamped) for (int i = 0; i < 3; ++i) o.clamped[3 * (size_t)p + i] = clamped[i] ? 1 : 0;
    if (o.Nmat)      // Nmat = R_wc R (rasterizer.py:140-141)
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k)
                o.Nmat[9 * (size_t)p + 3 * i + k] = cam.Rwc[3 * i + 0] * R[0 + k] +
                                                    cam.Rwc[3 * i + 1] * R[3 + k] +
                                                    cam.Rwc[3 * i + 2] * R[6 + k];
    const float *cf = prm.centers + 3 * p;
    const double v[3] = {(double)cf[0] - cam.eye[0], (double)cf[1] - cam.eye[1],
                         (double)cf[2] - cam.eye[2]};
    double dist = fmax(sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]), 1e-12);
    const double vd[3] = {v[0] / dist, v[1] / dist, v[2] / dist};
    if (o.view_dist) o.view_dist[p] = dist;
    if (o.view_dirs) for (int i = 0; i < 3; ++i) o.view_dirs[3 * (size_t)p + i] = vd[i];
    if (o.color_clamped) {   // sh.py:86-88: colour + 0.5 < 0 before the clamp
        const int K = prm.sh_coeffs;
        double Y[16];
        sh_basis(K, vd[0], vd[1], vd[2], Y);
        const float *shp = prm.sh + (size_t)p * 3 * K;
        for (int ch = 0; ch < 3; ++ch) {
            double acc = 0.0;
            for (int k = 0; k < K; ++k) acc += (double)shp[ch * K + k] * Y[k];
            o.color_clamped[3 * (size_t)p + ch] = (acc + 0.5) < 0 ? 1 : 0;
        }
    }
}

}  // namespace qgs
