// FP32 FMA and SFU (MUFU) throughput microbenchmarks for the roofline
// denominators (MEASURED_PEAKS.json carries only HBM and bf16 GEMM).
// Built into paper_2411_16392_b200/lib/libqgs_peaks.so by build.py; bench.py
// calls qgs_peaks() once per run.
#include <cuda_runtime.h>

#include <cstdio>

namespace {

constexpr int ITERS = 4096;
constexpr int CHAINS = 8;

__global__ void __launch_bounds__(256) ffma_kernel(float *out, float a, float b)
{
    float x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fmaf(x[c], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 1234.5f) out[0] = s;   // keep the work
}

__global__ void __launch_bounds__(256) mufu_kernel(float *out, float a)
{
    float x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-6f + c * 1e-3f;
    for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            float y;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[c]));
            x[c] = y * a;   // FMUL keeps the value bounded; MUFU is the limiter
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 1234.5f) out[0] = s;
}

}  // namespace

extern "C" int qgs_peaks(int device, double *fp32_tflops, double *mufu_tops, int *sms,
                         int *clock_khz)
{
    if (cudaSetDevice(device) != cudaSuccess) return -1;
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
    *sms = prop.multiProcessorCount;
    *clock_khz = clk;
    float *buf;
    if (cudaMalloc(&buf, 16) != cudaSuccess) return -2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = prop.multiProcessorCount * 8, threads = 256;
    float best_f = 1e30f, best_m = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        ffma_kernel<<<blocks, threads>>>(buf, 0.999f, 1e-4f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best_f) best_f = ms;
        cudaEventRecord(e0);
        mufu_kernel<<<blocks, threads>>>(buf, 0.5f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best_m) best_m = ms;
    }
    const double thr = (double)blocks * threads;
    *fp32_tflops = 2.0 * ITERS * CHAINS * thr / (best_f * 1e-3) / 1e12;
    *mufu_tops = (double)(ITERS / 4) * CHAINS * thr / (best_m * 1e-3) / 1e12;
    cudaFree(buf);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
