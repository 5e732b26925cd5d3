// Optimizer step and densification (optim.cu): host launchers called by abi.cu.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace qgs {

// groups in PrimitiveSet order: centers, quats, raw_scales, raw_signs, raw_opacity, sh
struct AdamArgs {
    float *p[6];
    const float *g[6];
    float *m[6];
    float *v[6];
    const uint8_t *freeze[6];      // per element, NULL = none
    int w[6];                      // floats per primitive
    double lr[6];
    double b1, b2, b1c, b2c, eps;
    const float *g_screen;         // (P, 2) screen-centre gradient
    double *grad_accum, *grad_count, *center_accum;   // NULL: no statistics
    unsigned long long *skipped;
    int P;
};

struct DensifyArgs {
    const float *raw_scales, *raw_signs, *raw_opacity;
    const double *grad_accum, *grad_count;
    double grad_threshold, big_threshold, prune_opacity;
    long long room;
    int P;
};

struct ApplyArgs {
    const float *src[6];
    const float *m_src[6];
    const float *v_src[6];
    float *dst[6];
    float *m_dst[6];
    float *v_dst[6];
    int w[6];
    const double *center_accum;
    double clone_nudge;
    int P;
};

cudaError_t adam_step(const AdamArgs &a, cudaStream_t s);
size_t densify_workspace_bytes(int P);
// d_counts (device int64[4]): kept total, survivors, clones, split parents
cudaError_t densify_plan(const DensifyArgs &a, void *ws, int64_t *d_counts, cudaStream_t s);
cudaError_t densify_apply(const ApplyArgs &a, const void *ws, cudaStream_t s);
cudaError_t reset_opacity(float *raw_opacity, float *m, float *v, int P, double cap,
                          cudaStream_t s);

}  // namespace qgs
