// Loss producers (losses.cu): host launchers called by abi.cu.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace qgs {

enum { LOSS_PHOTOMETRIC = 0, LOSS_DISTORTION = 1, LOSS_NORMAL = 2 };

// pinhole intrinsics for the camera-frame pixel rays (cameras.py:53-59)
struct LossCam {
    double fx, fy, cx, cy;
    int W, H;
};

size_t loss_workspace_bytes(int H, int W, int C);

// values: [loss, l1, ssim mean]; d_render (may be NULL) += weight * dloss/drender
cudaError_t photometric(const float *render, const float *gt, int H, int W, int C,
                        double lambda_ssim, double weight, float *d_render, double *values,
                        void *ws, cudaStream_t s);
// values: [loss]; d_dist (may be NULL) += weight / (H W)
cudaError_t distortion(const float *dmap, int H, int W, double weight, float *d_dist,
                       double *values, void *ws, cudaStream_t s);
cudaError_t depth_to_normal(const float *depth, const float *alpha, const LossCam &k,
                            double thresh, float *N, uint8_t *mask, cudaStream_t s);
// values: [loss, mask count]; N and mask come from depth (when depth != NULL)
// or from the N / mask arguments
cudaError_t normal_consistency(const float *alpha, const float *normal, const float *curv,
                               const float *depth, const float *N, const uint8_t *mask,
                               const LossCam &k, double thresh, double eps, int guided,
                               double weight, float *d_alpha, float *d_normal, float *d_curv,
                               double *values, void *ws, cudaStream_t s);

}  // namespace qgs
