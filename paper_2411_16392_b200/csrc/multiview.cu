// Multi-view reprojection + NCC regulariser on the device (SURVEY.md 8(f)
// row 3): multiview.py:108-311, the second rasterizer consumer of a training
// step (train.py:215-233).
//
// One thread per reference pixel does the whole per-pixel chain of the
// reference in fp64: the plane homography H_rn from the rendered depth /
// alpha / normal, the warp of the k x k patch into the neighbour view, the
// bilinear samples of the neighbour's depth/alpha ratio, normal and gray
// image, the forward-backward reprojection error through H_nr, NCC, and the
// adjoint of all of it.  Every gradient is linear in the 1 / n_valid factor
// of the mean, so the kernel accumulates unscaled gradients (reference-pixel
// terms written in place, neighbour terms scattered bilinearly with fp64
// atomics) and per-CTA partial sums; a finishing CTA folds the sums in a
// fixed order and the apply kernels scale by weight / n_valid into the fp32
// upstream maps.  The warped patch's gray samples are cached in shared
// memory (fp64, one column per thread); the gradient loop recomputes the
// warp and the sample derivatives rather than keeping 5 x k^2 values.  One
// reciprocal per dehomogenised point.
#include "multiview.cuh"
#include "qgs_common.cuh"

namespace qgs {

namespace {

constexpr int MV_T = 64;
#ifndef QGS_MV_CACHE_A
#define QGS_MV_CACHE_A 1            // cache the reference patch's gray samples too
#endif
#ifndef QGS_MV_MINB
#define QGS_MV_MINB 4               // shared memory allows 4 CTAs anyway: no register cap, no spills
#endif
constexpr int MV_NCACHE = QGS_MV_CACHE_A ? 2 : 1;
constexpr int MV_MAX_KP = 169;                   // patch <= 13 (shared-memory cache, 173 KB)

__device__ __forceinline__ double gray_at(const float *img, int C, int W, int x, int y)
{
    const int i = y * W + x;                    // maps are < 2^31 / 4 elements (ABI check)
    if (C == 1) return (double)img[i];
    const float *p = img + i * C;
    double s = 0.0;
    for (int c = 0; c < C; ++c) s += (double)p[c];
    return s / (double)C;                       // multiview.py:26-28 img.mean(axis=2)
}

// multiview.py:50-74 _bilerp: clipped corner, value and the two derivatives
struct Corner {
    int x0, y0;
    double ax, ay;
};

__device__ __forceinline__ Corner corner(double fx, double fy, int W, int H)
{
    Corner c;
    const double flx = floor(fx), fly = floor(fy);
    long long x0 = isfinite(flx) ? (long long)flx : 0, y0 = isfinite(fly) ? (long long)fly : 0;
    x0 = x0 < 0 ? 0 : (x0 > W - 2 ? W - 2 : x0);
    y0 = y0 < 0 ? 0 : (y0 > H - 2 ? H - 2 : y0);
    c.x0 = (int)x0;
    c.y0 = (int)y0;
    c.ax = fx - (double)x0;
    c.ay = fy - (double)y0;
    return c;
}

__device__ __forceinline__ void lerp4(double v00, double v01, double v10, double v11, const Corner &c,
                                      double &val, double &dx, double &dy)
{
    const double top = v00 * (1 - c.ax) + v01 * c.ax;
    const double bot = v10 * (1 - c.ax) + v11 * c.ax;
    val = top * (1 - c.ay) + bot * c.ay;
    dx = (v01 - v00) * (1 - c.ay) + (v11 - v10) * c.ay;
    dy = bot - top;
}

__device__ __forceinline__ double ratio_at(const MvArgs &a, int x, int y)
{
    const size_t p = (size_t)y * a.Wn + x;
    return (double)a.D_n[p] / fmax((double)a.A_n[p], 1e-6);
}

// 3x3 products in the reference's einsum order: sum over (j, k), j outer
__device__ __forceinline__ void triple(const double *A, const double *Mid, const double *B, double *out)
{
    for (int i = 0; i < 3; ++i)
        for (int l = 0; l < 3; ++l) {
            double s = 0.0;
            for (int j = 0; j < 3; ++j)
                for (int k = 0; k < 3; ++k) s += A[3 * i + j] * Mid[3 * j + k] * B[3 * k + l];
            out[3 * i + l] = s;
        }
}

// "ji,njk,lk->nil": A^T G B^T
__device__ __forceinline__ void triple_t(const double *A, const double *G, const double *B, double *out)
{
    for (int i = 0; i < 3; ++i)
        for (int l = 0; l < 3; ++l) {
            double s = 0.0;
            for (int j = 0; j < 3; ++j)
                for (int k = 0; k < 3; ++k) s += A[3 * j + i] * G[3 * j + k] * B[3 * l + k];
            out[3 * i + l] = s;
        }
}

struct Warp {
    double px, py, z;            // dehomogenised point and its z
    double hx, hy;               // homogeneous pixel (u + 0.5 + ox, v + 0.5 + oy)
};

__device__ __forceinline__ Warp warp_point(const double *H, double hx, double hy)
{
    Warp w;
    w.hx = hx;
    w.hy = hy;
    const double q0 = H[0] * hx + H[1] * hy + H[2];
    const double q1 = H[3] * hx + H[4] * hy + H[5];
    double z = H[6] * hx + H[7] * hy + H[8];
    w.z = z;
    if (fabs(z) < 1e-12) z = 1e-12;
    const double iz = 1.0 / z;
    w.px = q0 * iz;
    w.py = q1 * iz;
    return w;
}

__global__ void __launch_bounds__(MV_T, QGS_MV_MINB)
multiview_kernel(MvArgs a)
{
    __shared__ double red[MV_T / 32][4];
    extern __shared__ double sbk[];                  // [2][Kp][MV_T] patch samples: warped, reference
    const int W = a.W, H = a.H, r = a.r, k = 2 * r + 1, Kp = k * k;
    const int u = blockIdx.x * 32 + (threadIdx.x & 31);
    const int v = blockIdx.y * (MV_T / 32) + (threadIdx.x >> 5);
    const bool in = u < W && v < H;
    const size_t px = in ? (size_t)v * W + u : 0;
    double s_cnt = 0.0, s_term = 0.0, s_err = 0.0, s_ncc = 0.0;
    double gr_n[3] = {0.0, 0.0, 0.0}, gr_d = 0.0, gr_a = 0.0;
    bool keep = false;

    // multiview.py:137-141 candidates
    double A = 0.0, D = 0.0, N0 = 0.0, N1 = 0.0, N2 = 0.0, ln = 0.0;
    if (in && u >= r && u < W - r && v >= r && v < H - r) {
        A = a.A_r[px];
        D = a.D_r[px];
        N0 = a.N_r[3 * px]; N1 = a.N_r[3 * px + 1]; N2 = a.N_r[3 * px + 2];
        ln = sqrt(N0 * N0 + N1 * N1 + N2 * N2);
        keep = A > a.alpha_thresh && D > 0.0 && ln > 1e-9;
    }
    double dir[3], X[3], n[3], den = 0.0, tbar = 0.0, Hrn[9];
    if (keep) {
        // cameras.py:53-59 pixel ray, multiview.py:150-158
        const double ax = ((double)u + 0.5 - a.cx_r) / a.fx_r, ay = ((double)v + 0.5 - a.cy_r) / a.fy_r;
        const double dn = sqrt(ax * ax + ay * ay + 1.0);
        dir[0] = ax / dn; dir[1] = ay / dn; dir[2] = 1.0 / dn;
        tbar = D / A;
        for (int i = 0; i < 3; ++i) X[i] = tbar * dir[i];
        n[0] = N0 / ln; n[1] = N1 / ln; n[2] = N2 / ln;
        den = n[0] * X[0] + n[1] * X[1] + n[2] * X[2];
        keep = fabs(den) > a.min_denom;
    }
    Warp wc{};
    if (keep) {
        double Mid[9];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) Mid[3 * i + j] = a.R_rn[3 * i + j] + a.T_rn[i] * (n[j] / den);
        triple(a.K_n, Mid, a.K_r_inv, Hrn);
        // every warped patch point in front of the neighbour and inside its
        // frame; the gray samples of the warped patch go to the cache
        int ox = -r, oy = -r;
        for (int q = 0; q < Kp && keep; ++q) {
            const Warp w = warp_point(Hrn, (double)u + 0.5 + ox, (double)v + 0.5 + oy);
#if QGS_MV_CACHE_A
            sbk[(Kp + q) * MV_T + threadIdx.x] = gray_at(a.I_r, a.Cr, W, u + ox, v + oy);
#endif
            if (++ox > r) { ox = -r; ++oy; }
            keep = w.z > 1e-9 && w.px > 0.6 && w.px < a.Wn - 0.6 && w.py > 0.6 && w.py < a.Hn - 0.6;
            if (q == Kp / 2) wc = w;
            const Corner c = corner(w.px - 0.5, w.py - 0.5, a.Wn, a.Hn);
            double b, bx, by;
            lerp4(gray_at(a.I_n, a.Cn, a.Wn, c.x0, c.y0), gray_at(a.I_n, a.Cn, a.Wn, c.x0 + 1, c.y0),
                  gray_at(a.I_n, a.Cn, a.Wn, c.x0, c.y0 + 1),
                  gray_at(a.I_n, a.Cn, a.Wn, c.x0 + 1, c.y0 + 1), c, b, bx, by);
            sbk[q * MV_T + threadIdx.x] = b;
        }
    }
    // neighbour plane at the warped centre (multiview.py:189-218)
    double tb_n = 0, dtb_x = 0, dtb_y = 0, nn_raw[3], dnn_x[3], dnn_y[3], lnn = 0, nn[3];
    double dir_n[3], X_n[3], den_n = 0, mnorm = 0, Hnr[9], p_b[2], z_b = 0, e[2], err = 0;
    Corner cc{};
    if (keep) {
        const double fxc = wc.px - 0.5, fyc = wc.py - 0.5;
        cc = corner(fxc, fyc, a.Wn, a.Hn);
        lerp4(ratio_at(a, cc.x0, cc.y0), ratio_at(a, cc.x0 + 1, cc.y0), ratio_at(a, cc.x0, cc.y0 + 1),
              ratio_at(a, cc.x0 + 1, cc.y0 + 1), cc, tb_n, dtb_x, dtb_y);
        double an_s, d0, d1;
        const size_t p00 = (size_t)cc.y0 * a.Wn + cc.x0;
        lerp4(a.A_n[p00], a.A_n[p00 + 1], a.A_n[p00 + a.Wn], a.A_n[p00 + a.Wn + 1], cc, an_s, d0, d1);
        for (int c = 0; c < 3; ++c)
            lerp4(a.N_n[3 * p00 + c], a.N_n[3 * (p00 + 1) + c], a.N_n[3 * (p00 + a.Wn) + c],
                  a.N_n[3 * (p00 + a.Wn + 1) + c], cc, nn_raw[c], dnn_x[c], dnn_y[c]);
        lnn = sqrt(nn_raw[0] * nn_raw[0] + nn_raw[1] * nn_raw[1] + nn_raw[2] * nn_raw[2]);
        keep = an_s > a.alpha_thresh && lnn > 1e-9 && tb_n > 0.0;
        if (keep) {
            for (int c = 0; c < 3; ++c) nn[c] = nn_raw[c] / fmax(lnn, 1e-12);
            const double m0 = (wc.px - a.cx_n) / a.fx_n, m1 = (wc.py - a.cy_n) / a.fy_n;
            mnorm = sqrt(m0 * m0 + m1 * m1 + 1.0);
            dir_n[0] = m0 / mnorm; dir_n[1] = m1 / mnorm; dir_n[2] = 1.0 / mnorm;
            for (int c = 0; c < 3; ++c) X_n[c] = tb_n * dir_n[c];
            den_n = nn[0] * X_n[0] + nn[1] * X_n[1] + nn[2] * X_n[2];
            keep = fabs(den_n) > a.min_denom;
        }
        if (keep) {
            double Mid[9];
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) Mid[3 * i + j] = a.R_nr[3 * i + j] + a.T_nr[i] * (nn[j] / den_n);
            triple(a.K_r, Mid, a.K_n_inv, Hnr);
            const double q0 = Hnr[0] * wc.px + Hnr[1] * wc.py + Hnr[2];
            const double q1 = Hnr[3] * wc.px + Hnr[4] * wc.py + Hnr[5];
            z_b = Hnr[6] * wc.px + Hnr[7] * wc.py + Hnr[8];
            keep = z_b > 1e-9;
            p_b[0] = q0 / z_b;
            p_b[1] = q1 / z_b;
            e[0] = p_b[0] - ((double)u + 0.5);
            e[1] = p_b[1] - ((double)v + 0.5);
            err = sqrt(e[0] * e[0] + e[1] * e[1]);
        }
    }
    // NCC between the reference patch and the warped neighbour patch
    // (multiview.py:222-235); the patch loops recompute the warp
    auto sample_b = [&](int ox, int oy, Warp &w, double &b, double &bx, double &by) {
        w = warp_point(Hrn, (double)u + 0.5 + ox, (double)v + 0.5 + oy);
        const Corner c = corner(w.px - 0.5, w.py - 0.5, a.Wn, a.Hn);
        lerp4(gray_at(a.I_n, a.Cn, a.Wn, c.x0, c.y0), gray_at(a.I_n, a.Cn, a.Wn, c.x0 + 1, c.y0),
              gray_at(a.I_n, a.Cn, a.Wn, c.x0, c.y0 + 1), gray_at(a.I_n, a.Cn, a.Wn, c.x0 + 1, c.y0 + 1),
              c, b, bx, by);
    };
#if QGS_MV_CACHE_A
    const double *ak = sbk + (size_t)Kp * MV_T + threadIdx.x;
    auto sample_a = [&](int q) { return ak[q * MV_T]; };
#else
    auto sample_a = [&](int q) { return gray_at(a.I_r, a.Cr, W, u + q % k - r, v + q / k - r); };
#endif
    const double *bk = sbk + threadIdx.x;
    if (keep) {
        double sa = 0.0, sb = 0.0;
        for (int q = 0; q < Kp; ++q) {
            sa += sample_a(q);
            sb += bk[q * MV_T];
        }
        const double ma = sa / Kp, mb = sb / Kp;
        double Va = 0.0, Vb = 0.0, Scc = 0.0;
        for (int q = 0; q < Kp; ++q) {
            const double ca = sample_a(q) - ma, cb = bk[q * MV_T] - mb;
            Va += ca * ca;
            Vb += cb * cb;
            Scc += ca * cb;
        }
        const double sq = sqrt(Va * Vb);
        const double denom = fmax(sq, a.ncc_eps);
        const double ncc = Scc / denom;
        s_cnt = 1.0;
        s_term = err + 1.0 - ncc;
        s_err = err;
        s_ncc = ncc;

        // ---- backward with kf = 1 (scaled by 1 / n_valid when applied)
        double gH[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        const double live = sq > a.ncc_eps ? 1.0 : 0.0;
        const double coef = live * Scc * Va / (denom * denom * denom);
        double md = 0.0;
        for (int q = 0; q < Kp; ++q) md += (sample_a(q) - ma) / denom - coef * (bk[q * MV_T] - mb);
        md /= Kp;
        for (int q = 0, ox = -r, oy = -r; q < Kp; ++q) {
            Warp w;
            double b, bx, by;
            sample_b(ox, oy, w, b, bx, by);
            if (++ox > r) { ox = -r; ++oy; }
            const double dd = (sample_a(q) - ma) / denom - coef * (b - mb);
            const double gb = -1.0 * (dd - md);
            const double gx = gb * bx, gy = gb * by;
            const double iz = 1.0 / (fabs(w.z) < 1e-12 ? 1e-12 : w.z);
            const double gq[3] = {gx * iz, gy * iz, -(gx * w.px + gy * w.py) * iz};
            const double ph[3] = {w.hx, w.hy, 1.0};
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) gH[3 * i + j] += gq[i] * ph[j];
        }
        if (a.full_chain) {
            // reprojection term (multiview.py:258-296)
            const double safe = fmax(err, 1e-12);
            const double gpb[2] = {e[0] / safe, e[1] / safe};
            const double gqb[3] = {gpb[0] / z_b, gpb[1] / z_b,
                                   -(gpb[0] * p_b[0] + gpb[1] * p_b[1]) / z_b};
            const double pch[3] = {wc.px, wc.py, 1.0};
            double gHnr[9];
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) gHnr[3 * i + j] = gqb[i] * pch[j];
            double gpc[2];
            for (int j = 0; j < 2; ++j)
                gpc[j] = Hnr[j] * gqb[0] + Hnr[3 + j] * gqb[1] + Hnr[6 + j] * gqb[2];
            double gMid[9];
            triple_t(a.K_r, gHnr, a.K_n_inv, gMid);
            double gw[3];
            for (int j = 0; j < 3; ++j)
                gw[j] = a.T_nr[0] * gMid[j] + a.T_nr[1] * gMid[3 + j] + a.T_nr[2] * gMid[6 + j];
            const double s_n = gw[0] * nn[0] + gw[1] * nn[1] + gw[2] * nn[2];
            double gnn[3], gXn[3], gdir[3];
            for (int c = 0; c < 3; ++c) {
                gnn[c] = gw[c] / den_n - (s_n / (den_n * den_n)) * X_n[c];
                gXn[c] = -(s_n / (den_n * den_n)) * nn[c];
            }
            const double gtb = gXn[0] * dir_n[0] + gXn[1] * dir_n[1] + gXn[2] * dir_n[2];
            for (int c = 0; c < 3; ++c) gdir[c] = gXn[c] * tb_n;
            const double dg = dir_n[0] * gdir[0] + dir_n[1] * gdir[1] + dir_n[2] * gdir[2];
            const double gm0 = (gdir[0] - dir_n[0] * dg) / mnorm, gm1 = (gdir[1] - dir_n[1] * dg) / mnorm;
            gpc[0] += gm0 / a.fx_n;
            gpc[1] += gm1 / a.fy_n;
            const double ng = nn[0] * gnn[0] + nn[1] * gnn[1] + nn[2] * gnn[2];
            double gnr[3];
            for (int c = 0; c < 3; ++c) gnr[c] = (gnn[c] - nn[c] * ng) / fmax(lnn, 1e-12);
            gpc[0] += (gnr[0] * dnn_x[0] + gnr[1] * dnn_x[1] + gnr[2] * dnn_x[2]) + gtb * dtb_x;
            gpc[1] += (gnr[0] * dnn_y[0] + gnr[1] * dnn_y[1] + gnr[2] * dnn_y[2]) + gtb * dtb_y;
            // bilinear scatter of the sampled values' gradients (multiview.py:77-88)
            const double w00 = (1 - cc.ax) * (1 - cc.ay), w01 = cc.ax * (1 - cc.ay),
                         w10 = (1 - cc.ax) * cc.ay, w11 = cc.ax * cc.ay;
            const size_t p00 = (size_t)cc.y0 * a.Wn + cc.x0;
            const size_t pp[4] = {p00, p00 + 1, p00 + a.Wn, p00 + a.Wn + 1};
            const double ww[4] = {w00, w01, w10, w11};
            const size_t npn = (size_t)a.Hn * a.Wn;
            for (int t = 0; t < 4; ++t) {
                atomicAdd(a.g_nbr + pp[t], gtb * ww[t]);
                for (int c = 0; c < 3; ++c) atomicAdd(a.g_nbr + (1 + c) * npn + pp[t], gnr[c] * ww[t]);
            }
            const double z = fabs(wc.z) < 1e-12 ? 1e-12 : wc.z;
            const double gqc[3] = {gpc[0] / z, gpc[1] / z, -(gpc[0] * wc.px + gpc[1] * wc.py) / z};
            const double ph[3] = {wc.hx, wc.hy, 1.0};
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) gH[3 * i + j] += gqc[i] * ph[j];
        }
        // H_rn chain into the reference plane (multiview.py:298-310)
        double gMid[9];
        triple_t(a.K_n, gH, a.K_r_inv, gMid);
        double gw[3];
        for (int j = 0; j < 3; ++j)
            gw[j] = a.T_rn[0] * gMid[j] + a.T_rn[1] * gMid[3 + j] + a.T_rn[2] * gMid[6 + j];
        const double s_r = gw[0] * n[0] + gw[1] * n[1] + gw[2] * n[2];
        double gn[3], gX[3];
        for (int c = 0; c < 3; ++c) {
            gn[c] = gw[c] / den - (s_r / (den * den)) * X[c];
            gX[c] = -(s_r / (den * den)) * n[c];
        }
        const double gtbar = gX[0] * dir[0] + gX[1] * dir[1] + gX[2] * dir[2];
        const double ngn = n[0] * gn[0] + n[1] * gn[1] + n[2] * gn[2];
        for (int c = 0; c < 3; ++c) gr_n[c] = (gn[c] - n[c] * ngn) / ln;
        gr_d = gtbar / A;
        gr_a = -gtbar * tbar / A;
    }
    if (in) {
        const size_t np_ = (size_t)H * W;
        a.g_ref[px] = gr_d;
        a.g_ref[np_ + px] = gr_a;
        for (int c = 0; c < 3; ++c) a.g_ref[(2 + c) * np_ + px] = gr_n[c];
    }
    // per-CTA partial sums (count, loss terms, error, ncc)
    double s[4] = {s_cnt, s_term, s_err, s_ncc};
    for (int j = 0; j < 4; ++j)
        for (int o = 16; o; o >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
    if ((threadIdx.x & 31) == 0)
        for (int j = 0; j < 4; ++j) red[threadIdx.x >> 5][j] = s[j];
    __syncthreads();
    if (threadIdx.x == 0) {
        const int blk = blockIdx.y * gridDim.x + blockIdx.x;
        for (int j = 0; j < 4; ++j) {
            double t = 0.0;
            for (int w = 0; w < MV_T / 32; ++w) t += red[w][j];
            a.partial[4 * blk + j] = t;
        }
    }
}

// values: [value, n_valid, warp_px, ncc]; scal[0] = 1 / n_valid (0 when none)
__global__ void mv_finish_kernel(const double *partial, int nblk, double *values, double *scal)
{
    __shared__ double red[8][4];
    double s[4] = {0, 0, 0, 0};
    for (int i = threadIdx.x; i < nblk; i += blockDim.x)
        for (int j = 0; j < 4; ++j) s[j] += partial[4 * i + j];
    for (int j = 0; j < 4; ++j)
        for (int o = 16; o; o >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
    if ((threadIdx.x & 31) == 0)
        for (int j = 0; j < 4; ++j) red[threadIdx.x >> 5][j] = s[j];
    __syncthreads();
    if (threadIdx.x != 0) return;
    double t[4] = {0, 0, 0, 0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        for (int j = 0; j < 4; ++j) t[j] += red[w][j];
    const double nv = t[0];
    if (nv > 0.0) {
        values[0] = t[1] / nv;
        values[1] = nv;
        values[2] = t[2] / nv;
        values[3] = t[3] / nv;
        scal[0] = 1.0 / nv;
    } else {
        values[0] = 0.0; values[1] = 0.0; values[2] = 0.0; values[3] = 1.0;
        scal[0] = 0.0;
    }
}

__global__ void mv_apply_ref_kernel(const double *g, int npx, const double *scal, double weight,
                                    float *d_depth, float *d_alpha, float *d_normal)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npx) return;
    const double s = weight * scal[0];
    if (d_depth) d_depth[i] = (float)((double)d_depth[i] + s * g[i]);
    if (d_alpha) d_alpha[i] = (float)((double)d_alpha[i] + s * g[(size_t)npx + i]);
    if (d_normal)
        for (int c = 0; c < 3; ++c)
            d_normal[3 * (size_t)i + c] = (float)((double)d_normal[3 * (size_t)i + c] + s * g[(2 + c) * (size_t)npx + i]);
}

// multiview.py:290-296: the ratio's gradient into the neighbour's depth and alpha
__global__ void mv_apply_nbr_kernel(const double *g, int npx, const float *D_n, const float *A_n,
                                    const double *scal, double weight, float *d_depth,
                                    float *d_alpha, float *d_normal)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npx) return;
    const double s = weight * scal[0];
    const double gr = g[i], A = (double)A_n[i];
    const bool big = A > 1e-6;
    const double am = fmax(A, 1e-6);
    if (d_depth && big) d_depth[i] = (float)((double)d_depth[i] + s * (gr / am));
    if (d_alpha && big) d_alpha[i] = (float)((double)d_alpha[i] + s * (-gr * (double)D_n[i] / (am * am)));
    if (d_normal)
        for (int c = 0; c < 3; ++c)
            d_normal[3 * (size_t)i + c] = (float)((double)d_normal[3 * (size_t)i + c] + s * g[(1 + c) * (size_t)npx + i]);
}

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }
inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

int multiview_max_patch() { return 13; }

size_t multiview_workspace_bytes(int H, int W, int Hn, int Wn)
{
    const size_t nblk = (size_t)cdiv(W, 32) * cdiv(H, MV_T / 32);
    return al((size_t)H * W * 5 * 8) + al((size_t)Hn * Wn * 4 * 8) + al(nblk * 4 * 8) + al(64);
}

cudaError_t multiview(MvArgs a, double weight, float *ref_depth, float *ref_alpha,
                      float *ref_normal, float *nbr_depth, float *nbr_alpha, float *nbr_normal,
                      double *values, void *ws, cudaStream_t s)
{
    char *w = static_cast<char *>(ws);
    const dim3 grid(cdiv(a.W, 32), cdiv(a.H, MV_T / 32));
    const int nblk = grid.x * grid.y;
    a.g_ref = reinterpret_cast<double *>(w);
    w += al((size_t)a.H * a.W * 5 * 8);
    a.g_nbr = reinterpret_cast<double *>(w);
    w += al((size_t)a.Hn * a.Wn * 4 * 8);
    a.partial = reinterpret_cast<double *>(w);
    w += al((size_t)nblk * 4 * 8);
    double *scal = reinterpret_cast<double *>(w);
    cudaMemsetAsync(a.g_nbr, 0, (size_t)a.Hn * a.Wn * 4 * 8, s);
    const int Kp = (2 * a.r + 1) * (2 * a.r + 1);
    const size_t smem = (size_t)MV_NCACHE * Kp * MV_T * sizeof(double);
    {
        const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(multiview_kernel),
                                               (int)(MV_NCACHE * MV_MAX_KP * MV_T * sizeof(double)));
        if (e != cudaSuccess) return e;
    }
    multiview_kernel<<<grid, MV_T, smem, s>>>(a);
    mv_finish_kernel<<<1, 256, 0, s>>>(a.partial, nblk, values, scal);
    const int npr = a.H * a.W, npn = a.Hn * a.Wn;
    if (ref_depth || ref_alpha || ref_normal)
        mv_apply_ref_kernel<<<cdiv(npr, 256), 256, 0, s>>>(a.g_ref, npr, scal, weight, ref_depth,
                                                           ref_alpha, ref_normal);
    if (nbr_depth || nbr_alpha || nbr_normal)
        mv_apply_nbr_kernel<<<cdiv(npn, 256), 256, 0, s>>>(a.g_nbr, npn, a.D_n, a.A_n, scal, weight,
                                                           nbr_depth, nbr_alpha, nbr_normal);
    return cudaGetLastError();
}

}  // namespace qgs
