// Multi-view reprojection + NCC loss (multiview.cu): host launcher called by abi.cu.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace qgs {

struct MvArgs {
    const float *D_r, *A_r, *N_r, *I_r;   // reference maps (depth, alpha, normal, photo)
    const float *D_n, *A_n, *N_n, *I_n;   // neighbour maps
    int Cr, Cn;                           // photo channels
    int H, W, Hn, Wn;
    double fx_r, fy_r, cx_r, cy_r, fx_n, fy_n, cx_n, cy_n;
    double K_r[9], K_n[9], K_r_inv[9], K_n_inv[9];
    double R_rn[9], T_rn[3], R_nr[9], T_nr[3];
    int r;                                // patch radius
    double alpha_thresh, min_denom, ncc_eps;
    int full_chain;
    double *g_ref, *g_nbr, *partial;      // set by the launcher (workspace)
};

size_t multiview_workspace_bytes(int H, int W, int Hn, int Wn);
int multiview_max_patch();        // largest odd patch the shared-memory cache holds
// values (device fp64[4]): loss, n_valid, mean warp error (px), mean NCC
cudaError_t multiview(MvArgs a, double weight, float *ref_depth, float *ref_alpha,
                      float *ref_normal, float *nbr_depth, float *nbr_alpha, float *nbr_normal,
                      double *values, void *ws, cudaStream_t s);

}  // namespace qgs
