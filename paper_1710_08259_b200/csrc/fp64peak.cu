// fp64peak.cu — FP64 FMA throughput microbenchmark (the FP64 roofline denominator
// SURVEY.md §8(d) asks to be measured; MEASURED_PEAKS.json has no FP64 figure).
#include <cuda_runtime.h>

#include "nauticle_gpu.h"

namespace {

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void k_dfma(double* out, double a, double b) {
    double x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = __fma_rn(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

}  // namespace

extern "C" double nau_fp64_peak_tflops(int device) {
    cudaSetDevice(device);
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    double* out = nullptr;
    cudaMalloc(&out, sizeof(double));
    const int threads = 256;
    const int blocks = prop.multiProcessorCount * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 2.0 * kChains * (double)kIters * threads * (double)blocks;
    return flops / (best * 1e-3) / 1e12;
}
