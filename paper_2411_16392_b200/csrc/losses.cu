// Loss producers on the device: the maps the
// rasterizer backward consumes as upstream gradients, built in place from the
// forward's maps without leaving HBM.
//
//   photometric  losses.py:36-50 over ssim.py:41-86 (11x11 Gaussian SSIM)
//   distortion   losses.py:53-56
//   depth->normal + curvature-guided normal consistency  losses.py:59-113
//
// Everything is computed in fp64 from the fp32 maps (B200 runs fp64 at half
// the fp32 rate and these kernels are HBM/latency bound), so values and
// gradients follow the reference's float64 numpy to rounding.  Reductions are
// per-CTA partial sums finished by one CTA in a fixed order: deterministic.
//
// SSIM tiles: a CTA owns a 32x32 output tile of one channel and stages the
// 42x42 input window (zero outside the image, the reference's
// correlate1d(mode="constant")) in shared memory, blurs along rows of the
// image first and columns second (ssim.py:29-31 order), and keeps the five
// moment maps in registers for the per-pixel SSIM and its three adjoint maps
// (stored fp32 between the passes: the gradient they make is stored fp32).
// The gradient pass blurs the adjoint maps the same way (the Gaussian is
// symmetric, so the adjoint of the blur is the blur, ssim.py:1-7).
#include "losses.cuh"

#include <type_traits>

namespace qgs {

namespace {

constexpr int SS_T = 32;                 // output tile edge
constexpr int SS_R = 5;                  // window radius (WINDOW 11)
constexpr int SS_E = SS_T + 2 * SS_R;    // staged edge (42)
constexpr int SS_THREADS = 256;
#ifndef QGS_SSIM_ADJ_F32
#define QGS_SSIM_ADJ_F32 1          // adjoint maps in fp32 (the gradient is stored fp32 anyway): -6 %
#endif
using AdjT = std::conditional<QGS_SSIM_ADJ_F32, float, double>::type;
constexpr int SS_VB = 4;                 // outputs per thread along a blur (register run)
constexpr double SS_C1 = 0.01 * 0.01;    // ssim.py:15
constexpr double SS_C2 = 0.03 * 0.03;    // ssim.py:16

// ssim.py:19-23: normalised Gaussian taps, sigma 1.5 (a kernel parameter:
// constant-bank broadcast, no per-device symbol upload)
struct Gauss {
    double k[2 * SS_R + 1];
};

Gauss make_gauss()
{
    Gauss g;
    double s = 0.0;
    for (int i = 0; i <= 2 * SS_R; ++i) {
        const double xx = (double)(i - SS_R);
        g.k[i] = exp(-(xx * xx) / (2 * 1.5 * 1.5));
        s += g.k[i];
    }
    for (int i = 0; i <= 2 * SS_R; ++i) g.k[i] /= s;
    return g;
}

struct SsimSmem {
    double in[3][SS_E][SS_E];            // staged inputs (x, y) / adjoint maps
    double vb[5][SS_T][SS_E];            // after the first (row-axis) blur
};

__device__ __forceinline__ double block_sum(double v, double *red)
{
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < nw; ++i) s += red[i];
    return s;                            // valid on thread 0
}

// Moments (ux, uy, uxx, uyy, uxy) of one channel over a 32x32 tile, the
// SSIM map, the masked adjoint maps (M d_ux, M d_uxx, M d_uxy; ssim.py:71-78)
// and per-CTA partial sums of S over the crop and |x - y| over the tile.
__global__ void __launch_bounds__(SS_THREADS)
ssim_moments_kernel(const float *__restrict__ x, const float *__restrict__ y, int H, int W,
                    int C, int with_ssim, double inv_valid, Gauss gk, AdjT *__restrict__ adj,
                    double *__restrict__ partial)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SsimSmem &sm = *reinterpret_cast<SsimSmem *>(smem_raw);
    __shared__ double red[SS_THREADS / 32];
    const int c = blockIdx.z;
    const int u0 = blockIdx.x * SS_T, v0 = blockIdx.y * SS_T;
    const int blk = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;

    // L1 over the tile (the staged centre only)
    double l1 = 0.0;
    for (int i = threadIdx.x; i < SS_T * SS_T; i += SS_THREADS) {
        const int u = u0 + (i & (SS_T - 1)), v = v0 + (i >> 5);
        if (u < W && v < H) {
            const size_t p = ((size_t)v * W + u) * C + c;
            l1 += fabs((double)x[p] - (double)y[p]);
        }
    }
    double s_sum = 0.0;
    if (with_ssim) {
        for (int i = threadIdx.x; i < SS_E * SS_E; i += SS_THREADS) {
            const int r = i / SS_E, q = i - r * SS_E;
            const int v = v0 - SS_R + r, u = u0 - SS_R + q;
            double xv = 0.0, yv = 0.0;
            if (u >= 0 && u < W && v >= 0 && v < H) {
                const size_t p = ((size_t)v * W + u) * C + c;
                xv = (double)x[p];
                yv = (double)y[p];
            }
            sm.in[0][r][q] = xv;
            sm.in[1][r][q] = yv;
        }
        __syncthreads();
        // first blur: along image rows (axis 0), for every staged column;
        // a thread slides down SS_VB output rows of one column, so each
        // staged value is read once per run instead of once per tap
        for (int it = threadIdx.x; it < SS_E * (SS_T / SS_VB); it += SS_THREADS) {
            const int q = it % SS_E, r0 = (it / SS_E) * SS_VB;
            double xs[SS_VB + 2 * SS_R], ys[SS_VB + 2 * SS_R];
#pragma unroll
            for (int k = 0; k < SS_VB + 2 * SS_R; ++k) {
                xs[k] = sm.in[0][r0 + k][q];
                ys[k] = sm.in[1][r0 + k][q];
            }
#pragma unroll
            for (int o = 0; o < SS_VB; ++o) {
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
#pragma unroll
                for (int k = 0; k <= 2 * SS_R; ++k) {
                    const double g = gk.k[k];
                    const double xv = xs[o + k], yv = ys[o + k];
                    a0 += g * xv;
                    a1 += g * yv;
                    a2 += g * (xv * xv);
                    a3 += g * (yv * yv);
                    a4 += g * (xv * yv);
                }
                sm.vb[0][r0 + o][q] = a0; sm.vb[1][r0 + o][q] = a1; sm.vb[2][r0 + o][q] = a2;
                sm.vb[3][r0 + o][q] = a3; sm.vb[4][r0 + o][q] = a4;
            }
        }
        __syncthreads();
        // second blur along axis 1: SS_VB consecutive outputs of a row per thread
        for (int it = threadIdx.x; it < SS_T * (SS_T / SS_VB); it += SS_THREADS) {
            const int r = it / (SS_T / SS_VB), q0 = (it % (SS_T / SS_VB)) * SS_VB;
            double mm[5][SS_VB];
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                double vs[SS_VB + 2 * SS_R];
#pragma unroll
                for (int k = 0; k < SS_VB + 2 * SS_R; ++k) vs[k] = sm.vb[j][r][q0 + k];
#pragma unroll
                for (int o = 0; o < SS_VB; ++o) {
                    double a = 0.0;
#pragma unroll
                    for (int k = 0; k <= 2 * SS_R; ++k) a += gk.k[k] * vs[o + k];
                    mm[j][o] = a;
                }
            }
#pragma unroll
          for (int o = 0; o < SS_VB; ++o) {
            const int q = q0 + o;
            const int u = u0 + q, v = v0 + r;
            const double m[5] = {mm[0][o], mm[1][o], mm[2][o], mm[3][o], mm[4][o]};
            if (u >= W || v >= H) continue;          // this pixel only
            const double ux = m[0], uy = m[1];
            const double vx = m[2] - ux * ux, vy = m[3] - uy * uy, vxy = m[4] - ux * uy;
            const double A1 = 2 * ux * uy + SS_C1, A2 = 2 * vxy + SS_C2;
            const double B1 = ux * ux + uy * uy + SS_C1, B2 = vx + vy + SS_C2;
            const bool crop = u >= SS_R && u < W - SS_R && v >= SS_R && v < H - SS_R;
            double d0 = 0.0, d1 = 0.0, d2 = 0.0;
            if (crop) {
                s_sum += (A1 * A2) / (B1 * B2);
                // ssim.py:73-78 (S as a function of ux, uxx, uxy)
                const double dux = (2 * uy * B1 - A1 * 2 * ux) / (B1 * B1) * (A2 / B2)
                                 + (A1 / B1) * (-2 * uy * B2 - A2 * (-2 * ux)) / (B2 * B2);
                const double duxx = (A1 / B1) * (-A2 / (B2 * B2));
                const double duxy = (A1 / B1) * (2 / B2);
                d0 = inv_valid * dux;
                d1 = inv_valid * duxx;
                d2 = inv_valid * duxy;
            }
            const size_t p = (((size_t)c * H + v) * W + u) * 3;
            adj[p] = (AdjT)d0;
            adj[p + 1] = (AdjT)d1;
            adj[p + 2] = (AdjT)d2;
          }
        }
    }
    const double t_l1 = block_sum(l1, red);
    const double t_s = block_sum(s_sum, red);
    if (threadIdx.x == 0) {
        partial[2 * blk] = t_l1;
        partial[2 * blk + 1] = t_s;
    }
}

// d render += weight * ((1 - m) sign(x - y) / size - m dSSIM/dx)
// (losses.py:43-48), dSSIM/dx = blur(M d_ux) + 2 x blur(M d_uxx) + y blur(M d_uxy)
// (ssim.py:79-80).
__global__ void __launch_bounds__(SS_THREADS)
ssim_grad_kernel(const float *__restrict__ x, const float *__restrict__ y, int H, int W, int C,
                 int with_ssim, double l1_scale, double m_ssim, double weight, Gauss gk,
                 const AdjT *__restrict__ adj, float *__restrict__ d_render)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SsimSmem &sm = *reinterpret_cast<SsimSmem *>(smem_raw);
    const int c = blockIdx.z;
    const int u0 = blockIdx.x * SS_T, v0 = blockIdx.y * SS_T;
    if (with_ssim) {
        for (int i = threadIdx.x; i < SS_E * SS_E; i += SS_THREADS) {
            const int r = i / SS_E, q = i - r * SS_E;
            const int v = v0 - SS_R + r, u = u0 - SS_R + q;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0;
            if (u >= 0 && u < W && v >= 0 && v < H) {
                const size_t p = (((size_t)c * H + v) * W + u) * 3;
                a0 = (double)adj[p]; a1 = (double)adj[p + 1]; a2 = (double)adj[p + 2];
            }
            sm.in[0][r][q] = a0;
            sm.in[1][r][q] = a1;
            sm.in[2][r][q] = a2;
        }
        __syncthreads();
        for (int it = threadIdx.x; it < SS_E * (SS_T / SS_VB); it += SS_THREADS) {
            const int q = it % SS_E, r0 = (it / SS_E) * SS_VB;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                double vs[SS_VB + 2 * SS_R];
#pragma unroll
                for (int k = 0; k < SS_VB + 2 * SS_R; ++k) vs[k] = sm.in[j][r0 + k][q];
#pragma unroll
                for (int o = 0; o < SS_VB; ++o) {
                    double a = 0.0;
#pragma unroll
                    for (int k = 0; k <= 2 * SS_R; ++k) a += gk.k[k] * vs[o + k];
                    sm.vb[j][r0 + o][q] = a;
                }
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < SS_T * SS_T; i += SS_THREADS) {
        const int r = i >> 5, q = i & (SS_T - 1);
        const int u = u0 + q, v = v0 + r;
        if (u >= W || v >= H) continue;
        const size_t p = ((size_t)v * W + u) * C + c;
        const double xv = (double)x[p], yv = (double)y[p];
        const double diff = xv - yv;
        const double sg = diff > 0.0 ? 1.0 : (diff < 0.0 ? -1.0 : 0.0);
        double g = sg * l1_scale;
        if (with_ssim) {
            double b0 = 0.0, b1 = 0.0, b2 = 0.0;
#pragma unroll
            for (int k = 0; k <= 2 * SS_R; ++k) {
                const double g = gk.k[k];
                b0 += g * sm.vb[0][r][q + k];
                b1 += g * sm.vb[1][r][q + k];
                b2 += g * sm.vb[2][r][q + k];
            }
            g = g - m_ssim * (b0 + 2 * xv * b1 + yv * b2);
        }
        d_render[p] = (float)((double)d_render[p] + weight * g);
    }
}

// ------------------------------------------------ distortion (losses.py:53-56)
__global__ void __launch_bounds__(256)
distortion_kernel(const float *__restrict__ dmap, size_t n, double grad, float *__restrict__ d_dist,
                  double *__restrict__ partial)
{
    __shared__ double red[8];
    double s = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        s += (double)dmap[i];
        if (d_dist) d_dist[i] = (float)((double)d_dist[i] + grad);
    }
    const double t = block_sum(s, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// ---------------------------- depth -> normal (losses.py:59-89)
__device__ __forceinline__ void cam_dir(const LossCam &k, int u, int v, double &dx, double &dy,
                                        double &dz)
{
    // cameras.py:53-59
    const double a = ((double)u + 0.5 - k.cx) / k.fx, b = ((double)v + 0.5 - k.cy) / k.fy;
    const double n = sqrt(a * a + b * b + 1.0);
    dx = a / n; dy = b / n; dz = 1.0 / n;
}

struct DepthNormal {
    double n[3];
    bool valid;
};

__device__ __forceinline__ bool pix_ok(const float *depth, const float *alpha, int W, int u, int v,
                                       double thresh)
{
    const size_t p = (size_t)v * W + u;
    return (double)alpha[p] > thresh && (double)depth[p] > 0.0;
}

__device__ DepthNormal depth_normal_at(const float *__restrict__ depth,
                                       const float *__restrict__ alpha, const LossCam &k, int u,
                                       int v, double thresh)
{
    DepthNormal r{{0.0, 0.0, 0.0}, false};
    const int W = k.W, H = k.H;
    if (u < 1 || v < 1 || u > W - 2 || v > H - 2) return r;
    const bool ok = pix_ok(depth, alpha, W, u, v, thresh) && pix_ok(depth, alpha, W, u + 1, v, thresh)
                    && pix_ok(depth, alpha, W, u - 1, v, thresh)
                    && pix_ok(depth, alpha, W, u, v + 1, thresh)
                    && pix_ok(depth, alpha, W, u, v - 1, thresh);
    double P[4][3];
    const int du[4] = {1, -1, 0, 0}, dv[4] = {0, 0, 1, -1};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double ax, ay, az;
        cam_dir(k, u + du[j], v + dv[j], ax, ay, az);
        const double d = (double)depth[(size_t)(v + dv[j]) * W + u + du[j]];
        P[j][0] = d * ax; P[j][1] = d * ay; P[j][2] = d * az;
    }
    const double ex = P[0][0] - P[1][0], ey = P[0][1] - P[1][1], ez = P[0][2] - P[1][2];
    const double fx = P[2][0] - P[3][0], fy = P[2][1] - P[3][1], fz = P[2][2] - P[3][2];
    double nx = ey * fz - ez * fy, ny = ez * fx - ex * fz, nz = ex * fy - ey * fx;
    const double nn = sqrt(nx * nx + ny * ny + nz * nz);
    if (!(ok && nn > 1e-12)) return r;
    const double inv = fmax(nn, 1e-12);
    nx /= inv; ny /= inv; nz /= inv;
    double cx, cy, cz;
    cam_dir(k, u, v, cx, cy, cz);
    if (nx * cx + ny * cy + nz * cz > 0.0) { nx = -nx; ny = -ny; nz = -nz; }
    r.n[0] = nx; r.n[1] = ny; r.n[2] = nz;
    r.valid = true;
    return r;
}

__global__ void __launch_bounds__(256)
depth_normal_kernel(const float *__restrict__ depth, const float *__restrict__ alpha, LossCam k,
                    double thresh, float *__restrict__ N, uint8_t *__restrict__ mask)
{
    const int u = blockIdx.x * 32 + (threadIdx.x & 31), v = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (u >= k.W || v >= k.H) return;
    const DepthNormal dn = depth_normal_at(depth, alpha, k, u, v, thresh);
    const size_t p = (size_t)v * k.W + u;
    N[3 * p] = (float)dn.n[0];
    N[3 * p + 1] = (float)dn.n[1];
    N[3 * p + 2] = (float)dn.n[2];
    mask[p] = dn.valid ? 1 : 0;
}

// ---------------- curvature-guided normal consistency (losses.py:97-113)
// pass 0: per-CTA partial sums of (mask, mask * lambda_K * ln);
// pass 1: the gradients, scaled by 1 / count from the finished sums.
template <bool FROM_DEPTH>
__global__ void __launch_bounds__(256)
normal_consistency_kernel(const float *__restrict__ alpha, const float *__restrict__ normal,
                          const float *__restrict__ curv, const float *__restrict__ depth,
                          const float *__restrict__ Nin, const uint8_t *__restrict__ mask_in,
                          LossCam k, double thresh, double eps, int guided, int pass,
                          double weight, const double *__restrict__ scal, float *d_alpha,
                          float *d_normal, float *d_curv, double *__restrict__ partial)
{
    __shared__ double red[8];
    const int u = blockIdx.x * 32 + (threadIdx.x & 31), v = blockIdx.y * 8 + (threadIdx.x >> 5);
    const bool in = u < k.W && v < k.H;
    double m = 0.0, N0 = 0.0, N1 = 0.0, N2 = 0.0;
    size_t p = 0;
    if (in) {
        p = (size_t)v * k.W + u;
        if (FROM_DEPTH) {
            const DepthNormal dn = depth_normal_at(depth, alpha, k, u, v, thresh);
            m = dn.valid ? 1.0 : 0.0;
            N0 = dn.n[0]; N1 = dn.n[1]; N2 = dn.n[2];
        } else {
            m = mask_in[p] ? 1.0 : 0.0;
            N0 = (double)Nin[3 * p]; N1 = (double)Nin[3 * p + 1]; N2 = (double)Nin[3 * p + 2];
        }
    }
    double lam = 1.0, dlam = 0.0, ln = 0.0, K = 0.0;
    if (in) {
        ln = (double)alpha[p] - ((double)normal[3 * p] * N0 + (double)normal[3 * p + 1] * N1
                                 + (double)normal[3 * p + 2] * N2);
        if (guided) {
            K = (double)curv[p];
            lam = 1.0 / (1.0 + fabs(K) + eps);                    // losses.py:92-94
            const double sg = K > 0.0 ? 1.0 : (K < 0.0 ? -1.0 : 0.0);
            dlam = -sg * lam * lam;
        }
    }
    if (pass == 0) {
        const double tm = block_sum(m, red);
        const double tv = block_sum(m * lam * ln, red);
        if (threadIdx.x == 0) {
            const int blk = blockIdx.y * gridDim.x + blockIdx.x;
            partial[2 * blk] = tm;
            partial[2 * blk + 1] = tv;
        }
        return;
    }
    if (!in) return;
    const double count = scal[0];
    const double ml = m * lam / count;
    if (d_alpha) d_alpha[p] = (float)((double)d_alpha[p] + weight * ml);
    if (d_normal) {
        d_normal[3 * p] = (float)((double)d_normal[3 * p] + weight * (-ml * N0));
        d_normal[3 * p + 1] = (float)((double)d_normal[3 * p + 1] + weight * (-ml * N1));
        d_normal[3 * p + 2] = (float)((double)d_normal[3 * p + 2] + weight * (-ml * N2));
    }
    if (d_curv) d_curv[p] = (float)((double)d_curv[p] + weight * (m * dlam * ln / count));
}

// One CTA folds the partial sums in index order (deterministic) and writes
// the loss values (and, for the normal loss, the count the gradients use).
__global__ void __launch_bounds__(256)
loss_finish_kernel(const double *__restrict__ partial, int nblk, int kind, double a, double b,
                   double c, double *__restrict__ values, double *__restrict__ scal)
{
    __shared__ double red[8];
    double s0 = 0.0, s1 = 0.0;
    const int stride = kind == LOSS_DISTORTION ? 1 : 2;
    // fixed assignment of partials to threads and a fixed tree: same order every call
    for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
        s0 += partial[stride * i];
        if (stride == 2) s1 += partial[stride * i + 1];
    }
    const double t0 = block_sum(s0, red);
    const double t1 = block_sum(s1, red);
    if (threadIdx.x != 0) return;
    if (kind == LOSS_PHOTOMETRIC) {
        // a = 1 / size, b = lambda_ssim, c = n_valid (ssim.py:83 total / n_valid)
        const double l1 = t0 * a;
        const double s = b > 0.0 ? t1 / c : 0.0;
        values[1] = l1;
        values[2] = s;
        values[0] = b > 0.0 ? (1.0 - b) * l1 + b * (1.0 - s) : l1;
    } else if (kind == LOSS_DISTORTION) {
        values[0] = t0 * a;
    } else {
        const double count = fmax(t0, 1.0);
        scal[0] = count;
        values[0] = t1 / count;
        values[1] = t0;
    }
}

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }
inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace

size_t loss_workspace_bytes(int H, int W, int C)
{
    const size_t ssim_blocks = (size_t)cdiv(W, SS_T) * cdiv(H, SS_T) * (C > 0 ? C : 1);
    const size_t nblk = ssim_blocks > (size_t)cdiv(W, 32) * cdiv(H, 8) ? ssim_blocks
                                                                        : (size_t)cdiv(W, 32) * cdiv(H, 8);
    return al((size_t)H * W * (C > 0 ? C : 1) * 3 * sizeof(double)) +
           al(nblk * 2 * sizeof(double)) + al(8 * sizeof(double));
}

cudaError_t photometric(const float *render, const float *gt, int H, int W, int C,
                        double lambda_ssim, double weight, float *d_render, double *values,
                        void *ws, cudaStream_t s)
{
    static const Gauss gk = make_gauss();
    char *w = static_cast<char *>(ws);
    AdjT *adj = reinterpret_cast<AdjT *>(w);
    double *partial = reinterpret_cast<double *>(w + al((size_t)H * W * C * 3 * sizeof(double)));
    const dim3 grid(cdiv(W, SS_T), cdiv(H, SS_T), C);
    const int nblk = grid.x * grid.y * grid.z;
    const int with_ssim = lambda_ssim > 0.0 ? 1 : 0;
    const double n_valid = (double)(H - 2 * SS_R) * (double)(W - 2 * SS_R) * C;
    const double size = (double)H * W * C;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(ssim_moments_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(SsimSmem));
        cudaFuncSetAttribute(ssim_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(SsimSmem));
        attr = true;
    }
    const size_t smem = with_ssim ? sizeof(SsimSmem) : 0;
    ssim_moments_kernel<<<grid, SS_THREADS, smem, s>>>(render, gt, H, W, C, with_ssim,
                                                       1.0 / n_valid, gk, adj, partial);
    loss_finish_kernel<<<1, 256, 0, s>>>(partial, nblk, LOSS_PHOTOMETRIC, 1.0 / size, lambda_ssim,
                                         n_valid, values, nullptr);
    if (d_render)
        ssim_grad_kernel<<<grid, SS_THREADS, smem, s>>>(render, gt, H, W, C, with_ssim,
                                                        (1.0 - lambda_ssim) / size, lambda_ssim,
                                                        weight, gk, adj, d_render);
    return cudaGetLastError();
}

cudaError_t distortion(const float *dmap, int H, int W, double weight, float *d_dist,
                       double *values, void *ws, cudaStream_t s)
{
    const size_t n = (size_t)H * W;
    double *partial = static_cast<double *>(ws);
    const int nblk = 148 * 4;
    distortion_kernel<<<nblk, 256, 0, s>>>(dmap, n, weight / (double)n, d_dist, partial);
    loss_finish_kernel<<<1, 256, 0, s>>>(partial, nblk, LOSS_DISTORTION, 1.0 / (double)n, 0.0,
                                         0.0, values, nullptr);
    return cudaGetLastError();
}

cudaError_t depth_to_normal(const float *depth, const float *alpha, const LossCam &k,
                            double thresh, float *N, uint8_t *mask, cudaStream_t s)
{
    const dim3 grid(cdiv(k.W, 32), cdiv(k.H, 8));
    depth_normal_kernel<<<grid, 256, 0, s>>>(depth, alpha, k, thresh, N, mask);
    return cudaGetLastError();
}

cudaError_t normal_consistency(const float *alpha, const float *normal, const float *curv,
                               const float *depth, const float *N, const uint8_t *mask,
                               const LossCam &k, double thresh, double eps, int guided,
                               double weight, float *d_alpha, float *d_normal, float *d_curv,
                               double *values, void *ws, cudaStream_t s)
{
    const dim3 grid(cdiv(k.W, 32), cdiv(k.H, 8));
    const int nblk = grid.x * grid.y;
    double *partial = static_cast<double *>(ws);
    double *scal = reinterpret_cast<double *>(static_cast<char *>(ws) +
                                              al((size_t)nblk * 2 * sizeof(double)));
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
            loss_finish_kernel<<<1, 256, 0, s>>>(partial, nblk, LOSS_NORMAL, 0.0, 0.0, 0.0, values,
                                                 scal);
            if (!d_alpha && !d_normal && !d_curv) break;
        }
        if (depth)
            normal_consistency_kernel<true><<<grid, 256, 0, s>>>(
                alpha, normal, curv, depth, nullptr, nullptr, k, thresh, eps, guided, pass, weight,
                scal, d_alpha, d_normal, d_curv, partial);
        else
            normal_consistency_kernel<false><<<grid, 256, 0, s>>>(
                alpha, normal, curv, nullptr, N, mask, k, thresh, eps, guided, pass, weight, scal,
                d_alpha, d_normal, d_curv, partial);
    }
    return cudaGetLastError();
}

}  // namespace qgs
