// Optimizer step and densification on the device:
// the step that follows the gradient all-reduce (train.py:239-262) and the
// clone / split / prune pass (train.py:269-330), over the six fp32 parameter
// groups resident in HBM.
//
//   adam_kernel         optim.py:23-47 Adam.step, fused with the
//                       densification statistics of train.py:239-244
//   densify_flags       train.py:270-290 (mean gradient, room, split / clone)
//   radix select        train.py:278-284 top-`room` by (-mean, index)
//   densify_apply       train.py:292-329 (survivors, nudged clones, split
//                       children, opacity prune) as ONE ordered compaction
//   reset_opacity       train.py:332-335
//
// Adam: a CTA owns 256 consecutive primitives.  Each thread first checks its
// primitive's gradient row for non-finite values (one bad primitive must not
// poison the others, optim.py:28-33) and folds the screen-centre gradient
// norm and the centre gradient into the statistics; then the CTA walks each
// group's contiguous element range with coalesced loads and updates
// (m, v, param) in fp64 arithmetic from fp32 storage; last, every thread
// renormalises its quaternion.
#include "optim.cuh"

namespace qgs {

namespace {

constexpr int AD_T = 256;

__global__ void __launch_bounds__(AD_T)
adam_kernel(AdamArgs a)
{
    __shared__ int bad[AD_T];
    __shared__ int nbad;
    const int p0 = blockIdx.x * AD_T;
    const int np = min(AD_T, a.P - p0);
    const int i = p0 + threadIdx.x;
    if (threadIdx.x == 0) nbad = 0;
    bad[threadIdx.x] = 0;
    __syncthreads();
    // non-finite rows: coalesced sweep of the block's gradient slice
    for (int g = 0; g < 6; ++g) {
        const int w = a.w[g];
        const float *src = a.g[g] + (size_t)p0 * w;
        const float iw = 1.f / (float)w;
        for (int e = threadIdx.x; e < np * w; e += AD_T)
            if (!isfinite(src[e])) bad[(int)(((float)e + 0.5f) * iw)] = 1;
    }
    __syncthreads();
    if (threadIdx.x < np) {
        if (bad[threadIdx.x]) atomicAdd(&nbad, 1);
        if (a.grad_accum) {
            // train.py:240-244 (before the step; the raw, unmasked gradients)
            const double gx = a.g_screen[2 * (size_t)i], gy = a.g_screen[2 * (size_t)i + 1];
            const double gn = sqrt(gx * gx + gy * gy);
            if (gn > 0.0) {
                a.grad_accum[i] += gn;
                a.grad_count[i] += 1.0;
            }
            for (int k = 0; k < 3; ++k) a.center_accum[3 * (size_t)i + k] += (double)a.g[0][3 * (size_t)i + k];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && nbad) atomicAdd(a.skipped, (unsigned long long)nbad);
    const double ib1c = 1.0 / a.b1c, ib2c = 1.0 / a.b2c;   // bias corrections as products
    for (int g = 0; g < 6; ++g) {
        const int w = a.w[g];
        const float iw = 1.f / (float)w;        // row of element e: (e + 0.5) / w is >= 0.5 / w from any integer
        const size_t e0 = (size_t)p0 * w;
        const int ne = np * w;
        const double lr = a.lr[g];
#pragma unroll 4
        for (int e = threadIdx.x; e < ne; e += AD_T) {
            const size_t idx = e0 + e;
            double grad = bad[(int)(((float)e + 0.5f) * iw)] ? 0.0 : (double)a.g[g][idx];
            if (a.freeze[g] && a.freeze[g][idx]) grad = 0.0;
            const double m = a.b1 * (double)a.m[g][idx] + (1.0 - a.b1) * grad;
            const double v = a.b2 * (double)a.v[g][idx] + (1.0 - a.b2) * grad * grad;
            const double mhat = m * ib1c, vhat = v * ib2c;
            a.m[g][idx] = (float)m;
            a.v[g][idx] = (float)v;
            a.p[g][idx] = (float)((double)a.p[g][idx] - lr * mhat / (sqrt(vhat) + a.eps));
        }
    }
    __syncthreads();
    if (threadIdx.x < np) {
        // optim.py:46-47: keep quaternions unit
        float *q = a.p[1] + 4 * (size_t)i;
        const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
        const double n = sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
        q[0] = (float)(q0 / n); q[1] = (float)(q1 / n); q[2] = (float)(q2 / n); q[3] = (float)(q3 / n);
    }
}

// model.py:29-45 activated |s1|, |s2| (the in-plane scales, floored at S_MIN)
__device__ __forceinline__ void inplane_scales(const float *rs, const float *rg, size_t i,
                                               double &s0, double &s1)
{
    double s[2];
    for (int k = 0; k < 2; ++k) {
        double v = tanh((double)rg[3 * i + k]) * exp((double)rs[3 * i + k]);
        if (fabs(v) < 1e-4) v = (v < 0.0 ? -1.0 : 1.0) * 1e-4;
        s[k] = v;
    }
    s0 = s[0];
    s1 = s[1];
}

enum { F_DENSIFY = 1, F_BIG = 2, F_ALIVE = 4 };

__global__ void densify_flags_kernel(DensifyArgs a, uint8_t *flags, uint64_t *keys,
                                     unsigned long long *n_densify)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.P) return;
    const double cnt = a.grad_count[i];
    const double mean = cnt > 0.0 ? a.grad_accum[i] / fmax(cnt, 1.0) : 0.0;
    const bool dens = mean > a.grad_threshold;
    double s0, s1;
    inplane_scales(a.raw_scales, a.raw_signs, i, s0, s1);
    const bool big = fmax(fabs(s0), fabs(s1)) > a.big_threshold;
    // model.py:55-56 sigmoid; train.py:326-327 prune (children share the parent's opacity)
    const double alpha = 1.0 / (1.0 + exp(-(double)a.raw_opacity[i]));
    const bool alive = alpha >= a.prune_opacity;
    flags[i] = (dens ? F_DENSIFY : 0) | (big ? F_BIG : 0) | (alive ? F_ALIVE : 0);
    keys[i] = (uint64_t)__double_as_longlong(mean);     // mean >= 0: bit order is value order
    if (dens) atomicAdd(n_densify, 1ull);
}

// Radix select of the room-th largest key (8-bit digits, most significant
// first).  st[0] = prefix, st[1] = remaining rank, st[2] = active (selection
// needed: 0 < room < count), st[3] = room.
__global__ void radix_hist_kernel(const uint64_t *__restrict__ keys, int P, int shift,
                                  const unsigned long long *st, unsigned long long *hist)
{
    __shared__ unsigned int h[256];
    if (!st[2]) return;
    for (int b = threadIdx.x; b < 256; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const uint64_t prefix = st[0];
    const uint64_t hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        if ((k & hi_mask) == (prefix & hi_mask)) atomicAdd(&h[(k >> shift) & 255], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < 256; b += blockDim.x)
        if (h[b]) atomicAdd(&hist[b], (unsigned long long)h[b]);
}

__global__ void radix_pick_kernel(int shift, unsigned long long *st, unsigned long long *hist)
{
    if (threadIdx.x != 0 || !st[2]) return;
    unsigned long long rem = st[1];
    for (int b = 255; b >= 0; --b) {
        const unsigned long long c = hist[b];
        if (c >= rem) {
            st[0] |= (unsigned long long)b << shift;
            break;
        }
        rem -= c;
    }
    st[1] = rem;
    for (int b = 0; b < 256; ++b) hist[b] = 0;
}

// before the passes: decide whether a selection is needed (train.py:275-284)
__global__ void room_kernel(const unsigned long long *n_densify, long long room,
                            unsigned long long *st, unsigned long long *hist)
{
    if (threadIdx.x != 0) return;
    st[0] = 0;
    st[1] = room > 0 ? (unsigned long long)room : 0;
    st[2] = (room > 0 && *n_densify > (unsigned long long)room) ? 1 : 0;
    st[3] = room > 0 ? (unsigned long long)room : 0;
    st[4] = room <= 0 ? 1 : 0;                         // no room: densify nothing
    for (int b = 0; b < 256; ++b) hist[b] = 0;
}

__global__ void ties_kernel(const uint64_t *__restrict__ keys, int P, const unsigned long long *st,
                            int32_t *eq)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    eq[i] = (st[2] && keys[i] == st[0]) ? 1 : 0;
}

// final flags and the three category indicators (kept survivor / clone / split)
__global__ void categories_kernel(int P, const uint64_t *__restrict__ keys, const int64_t *eq_rank,
                                  const unsigned long long *st, uint8_t *flags, int32_t *c_surv,
                                  int32_t *c_clone, int32_t *c_split)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    uint8_t f = flags[i];
    bool dens = (f & F_DENSIFY) != 0;
    if (st[4]) dens = false;
    if (st[2]) {
        // the top `room` by (-mean, index): key above the threshold, or equal
        // to it and among the first st[1] such indices
        const uint64_t k = keys[i];
        dens = k > st[0] || (k == st[0] && eq_rank[i] < (int64_t)st[1]);
    }
    const bool big = (f & F_BIG) != 0, alive = (f & F_ALIVE) != 0;
    const bool split = dens && big, clone = dens && !big;
    f = (uint8_t)((f & ~F_DENSIFY) | (dens ? F_DENSIFY : 0));
    flags[i] = f;
    c_surv[i] = (!split && alive) ? 1 : 0;
    c_clone[i] = (clone && alive) ? 1 : 0;
    c_split[i] = (split && alive) ? 1 : 0;
}

__device__ __forceinline__ void copy_row(const float *src, float *dst, size_t i, size_t o, int w)
{
    for (int k = 0; k < w; ++k) dst[o * w + k] = src[i * w + k];
}

__device__ __forceinline__ void zero_row(float *dst, size_t o, int w)
{
    for (int k = 0; k < w; ++k) dst[o * w + k] = 0.f;
}

// One thread per input primitive writes its surviving copy (with its Adam
// state), its nudged clone and its two split children (zero state) at the
// scanned offsets: [survivors | clones | split + | split -], each in index
// order, opacity-pruned -- the order of PrimitiveSet.concatenate followed by
// select(keep) (train.py:292-329).
__global__ void densify_apply_kernel(ApplyArgs a, const uint8_t *__restrict__ flags,
                                     const int64_t *__restrict__ o_surv,
                                     const int64_t *__restrict__ o_clone,
                                     const int64_t *__restrict__ o_split)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.P) return;
    const uint8_t f = flags[i];
    const bool dens = f & F_DENSIFY, big = f & F_BIG, alive = f & F_ALIVE;
    if (!alive) return;
    const bool split = dens && big, clone = dens && !big;
    const int64_t S = o_surv[a.P], C = o_clone[a.P], Sp = o_split[a.P];
    if (!split) {
        const size_t o = (size_t)o_surv[i];
        for (int g = 0; g < 6; ++g) {
            copy_row(a.src[g], a.dst[g], i, o, a.w[g]);
            copy_row(a.m_src[g], a.m_dst[g], i, o, a.w[g]);
            copy_row(a.v_src[g], a.v_dst[g], i, o, a.w[g]);
        }
    }
    if (!dens) return;
    double s0, s1;
    inplane_scales(a.src[2], a.src[3], i, s0, s1);
    const float *c = a.src[0] + 3 * (size_t)i;
    auto emit = [&](size_t o, double cx, double cy, double cz, int axis) {
        for (int g = 0; g < 6; ++g) {
            copy_row(a.src[g], a.dst[g], i, o, a.w[g]);
            zero_row(a.m_dst[g], o, a.w[g]);
            zero_row(a.v_dst[g], o, a.w[g]);
        }
        a.dst[0][3 * o] = (float)cx;
        a.dst[0][3 * o + 1] = (float)cy;
        a.dst[0][3 * o + 2] = (float)cz;
        if (axis >= 0)
            a.dst[2][3 * o + axis] = (float)((double)a.src[2][3 * (size_t)i + axis] - log(2.0));
    };
    if (clone) {
        // train.py:297-304: step against the accumulated centre gradient
        const double gx = a.center_accum[3 * (size_t)i], gy = a.center_accum[3 * (size_t)i + 1],
                     gz = a.center_accum[3 * (size_t)i + 2];
        const double n = sqrt(gx * gx + gy * gy + gz * gz);
        double dx = 0.0, dy = 0.0, dz = 0.0;
        if (n > 1e-12) {
            const double inv = fmax(n, 1e-12);
            dx = -gx / inv; dy = -gy / inv; dz = -gz / inv;
        }
        const double st = a.clone_nudge * fmin(fabs(s0), fabs(s1));
        emit((size_t)(S + o_clone[i]), (double)c[0] + dx * st, (double)c[1] + dy * st,
             (double)c[2] + dz * st, -1);
    } else {
        // train.py:307-318: children at +- half the larger in-plane axis
        const int axis = fabs(s1) > fabs(s0) ? 1 : 0;
        const double sa = fabs(axis ? s1 : s0);
        const float *q = a.src[1] + 4 * (size_t)i;
        double w = q[0], x = q[1], y = q[2], z = q[3];
        const double qn = sqrt(w * w + x * x + y * y + z * z);
        w /= qn; x /= qn; y /= qn; z /= qn;
        // model.py:70-87 column `axis` of R
        double ax, ay, az;
        if (axis == 0) {
            ax = 1 - 2 * (y * y + z * z); ay = 2 * (x * y + w * z); az = 2 * (x * z - w * y);
        } else {
            ax = 2 * (x * y - w * z); ay = 1 - 2 * (x * x + z * z); az = 2 * (y * z + w * x);
        }
        const double ox = 0.5 * sa * ax, oy = 0.5 * sa * ay, oz = 0.5 * sa * az;
        const size_t o = (size_t)(S + C + o_split[i]);
        emit(o, (double)c[0] + ox, (double)c[1] + oy, (double)c[2] + oz, axis);
        emit(o + (size_t)Sp, (double)c[0] - ox, (double)c[1] - oy, (double)c[2] - oz, axis);
    }
}

__global__ void reset_opacity_kernel(float *raw_opacity, float *m, float *v, int P, double cap)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const double alpha = 1.0 / (1.0 + exp(-(double)raw_opacity[i]));
    const double y = fmin(alpha, cap);
    raw_opacity[i] = (float)log(y / (1.0 - y));        // model.py:59-60
    m[i] = 0.f;
    v[i] = 0.f;
}

// [kept total, survivors, clones, split parents]
__global__ void counts_kernel(const int64_t *tot, int64_t *out)
{
    if (threadIdx.x != 0) return;
    out[0] = tot[0] + tot[1] + 2 * tot[2];
    out[1] = tot[0];
    out[2] = tot[1];
    out[3] = tot[2];
}

inline size_t al(size_t x) { return (x + 255) & ~(size_t)255; }
inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

struct DensWs {
    uint8_t *flags;
    uint64_t *keys;
    int32_t *c[3];        // survivor / clone / split indicators (c[0] doubles as the tie flags)
    int64_t *o[3];        // their exclusive scans (P + 1)
    int64_t *sums;        // scan block sums
    int64_t *tot;         // scan totals [3]
    int64_t *eq_rank;     // tie ranks (P + 1)
    unsigned long long *st, *hist, *n_densify;
    size_t bytes;
};

DensWs carve(void *base, int P)
{
    DensWs w{};
    char *p = static_cast<char *>(base);
    size_t off = 0;
    auto take = [&](size_t n) { char *r = p ? p + off : nullptr; off += al(n); return r; };
    const size_t nb = (size_t)cdiv(P > 0 ? P : 1, SCAN_ITEMS);
    w.flags = reinterpret_cast<uint8_t *>(take((size_t)P));
    w.keys = reinterpret_cast<uint64_t *>(take((size_t)P * 8));
    for (int k = 0; k < 3; ++k) w.c[k] = reinterpret_cast<int32_t *>(take((size_t)P * 4));
    for (int k = 0; k < 3; ++k) w.o[k] = reinterpret_cast<int64_t *>(take((size_t)(P + 1) * 8));
    w.eq_rank = reinterpret_cast<int64_t *>(take((size_t)(P + 1) * 8));
    w.sums = reinterpret_cast<int64_t *>(take(nb * 8));
    w.tot = reinterpret_cast<int64_t *>(take(4 * 8));
    w.st = reinterpret_cast<unsigned long long *>(take(8 * 8));
    w.hist = reinterpret_cast<unsigned long long *>(take(256 * 8));
    w.n_densify = reinterpret_cast<unsigned long long *>(take(8));
    w.bytes = off;
    return w;
}

void scan(const int32_t *in, int n, int64_t *sums, int64_t *total, int64_t *out, cudaStream_t s)
{
    const int nb = cdiv(n > 0 ? n : 1, SCAN_ITEMS);
    scan_sums_kernel<<<nb, SCAN_THREADS, 0, s>>>(in, n, sums);
    scan_top_kernel<<<1, SCAN_THREADS, 0, s>>>(sums, nb, total, out, n);
    scan_out_kernel<<<nb, SCAN_THREADS, 0, s>>>(in, n, sums, out);
}

}  // namespace

cudaError_t adam_step(const AdamArgs &a, cudaStream_t s)
{
    if (a.P > 0) adam_kernel<<<cdiv(a.P, AD_T), AD_T, 0, s>>>(a);
    return cudaGetLastError();
}

size_t densify_workspace_bytes(int P) { return carve(nullptr, P).bytes; }

cudaError_t densify_plan(const DensifyArgs &a, void *ws, int64_t *d_counts, cudaStream_t s)
{
    DensWs w = carve(ws, a.P);
    const int P = a.P;
    const int g = cdiv(P > 0 ? P : 1, 256);
    cudaMemsetAsync(w.n_densify, 0, 8, s);
    if (P > 0) densify_flags_kernel<<<g, 256, 0, s>>>(a, w.flags, w.keys, w.n_densify);
    room_kernel<<<1, 32, 0, s>>>(w.n_densify, a.room, w.st, w.hist);
    for (int shift = 56; shift >= 0; shift -= 8) {
        radix_hist_kernel<<<148 * 2, 256, 0, s>>>(w.keys, P, shift, w.st, w.hist);
        radix_pick_kernel<<<1, 32, 0, s>>>(shift, w.st, w.hist);
    }
    if (P > 0) ties_kernel<<<g, 256, 0, s>>>(w.keys, P, w.st, w.c[0]);
    scan(w.c[0], P, w.sums, w.tot + 3, w.eq_rank, s);
    if (P > 0)
        categories_kernel<<<g, 256, 0, s>>>(P, w.keys, w.eq_rank, w.st, w.flags, w.c[0], w.c[1],
                                            w.c[2]);
    for (int k = 0; k < 3; ++k) scan(w.c[k], P, w.sums, w.tot + k, w.o[k], s);
    counts_kernel<<<1, 32, 0, s>>>(w.tot, d_counts);
    return cudaGetLastError();
}

cudaError_t densify_apply(const ApplyArgs &a, const void *ws, cudaStream_t s)
{
    DensWs w = carve(const_cast<void *>(ws), a.P);
    if (a.P > 0)
        densify_apply_kernel<<<cdiv(a.P, 128), 128, 0, s>>>(a, w.flags, w.o[0], w.o[1], w.o[2]);
    return cudaGetLastError();
}

cudaError_t reset_opacity(float *raw_opacity, float *m, float *v, int P, double cap, cudaStream_t s)
{
    if (P > 0) reset_opacity_kernel<<<cdiv(P, 256), 256, 0, s>>>(raw_opacity, m, v, P, cap);
    return cudaGetLastError();
}

}  // namespace qgs
