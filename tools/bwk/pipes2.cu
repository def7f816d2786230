// Packed-FP32 pipe probe: independent FFMA2 / FADD2 chains against scalar
// FFMA, lanes (fp32 operations) per SM per clock, timed with CUDA events.
// Tells whether Blackwell's f32x2 instructions double the FP32 lane rate or
// only halve the issue slots (the range compression's ceiling depends on it).
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_2506_23568_b200/csrc/common.cuh"
using namespace hhsar;

template <int K>
__global__ void ffma2_k(float *out, int iters) {
    f2x a[K];
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = pk2(threadIdx.x * 1e-9f + k, k * 0.5f);
    const f2x b = pk2(1.0000001f, 0.9999999f), c = pk2(1e-7f, 2e-7f);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < K; ++k) a[k] = fma2(a[k], b, c);
    float s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += lo2(a[k]) + hi2(a[k]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int K>
__global__ void fadd2_k(float *out, int iters) {
    f2x a[K];
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = pk2(threadIdx.x * 1e-9f + k, k * 0.5f);
    const f2x c = pk2(1e-7f, 2e-7f);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < K; ++k) a[k] = add2(a[k], c);
    float s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += lo2(a[k]) + hi2(a[k]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// half scalar FFMA, half FFMA2 (mixed issue)
template <int K>
__global__ void mix_k(float *out, int iters) {
    f2x a[K];
    float b[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        a[k] = pk2(threadIdx.x * 1e-9f + k, k * 0.5f);
        b[k] = k * 0.25f;
    }
    const f2x m = pk2(1.0000001f, 0.9999999f), c = pk2(1e-7f, 2e-7f);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            a[k] = fma2(a[k], m, c);
            b[k] = fmaf(b[k], 1.0000001f, 1e-7f);
        }
    float s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += lo2(a[k]) + hi2(a[k]) + b[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int K>
__global__ void ffma_k(float *out, int iters) {
    float a[K];
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = threadIdx.x * 1e-9f + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int k = 0; k < K; ++k) a[k] = fmaf(a[k], 1.0000001f, 1e-7f);
    float s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += a[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float *d;
    cudaMalloc(&d, sizeof(float) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](const char *name, void (*kern)(float *, int), double lanes_per_iter,
                    double instr_per_iter) {
        kern<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double thr = (double)blocks * threads * iters;
        const double s = ms * 1e-3 * sms * 1.965e9;
        printf("%-22s %6.1f fp32 lanes/clk/SM  %5.2f warp-instr/clk/SM\n", name,
               thr * lanes_per_iter / s, thr * instr_per_iter / 32.0 / s);
    };
    time("FFMA (8 chains)", ffma_k<8>, 8, 8);
    time("FFMA2 (8 chains)", ffma2_k<8>, 16, 8);
    time("FADD2 (8 chains)", fadd2_k<8>, 16, 8);
    time("FFMA2+FFMA (4+4)", mix_k<4>, 12, 8);
    return 0;
}
