// Streaming ceiling probe for the range-compression traffic pattern: each CTA
// reads one n_f-sample row and writes one 4 n_f-bin row (no arithmetic).
#include <cuda_runtime.h>
#include <cstdint>
__global__ void __launch_bounds__(256) rw14(const float2 *__restrict__ in, float2 *__restrict__ out, int n_f) {
    const int64_t row = blockIdx.x;
    float2 v[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) v[r] = __ldcs(in + row * n_f + threadIdx.x + r * 256);
    float2 *o = out + row * 4 * n_f;
#pragma unroll
    for (int r = 0; r < 16; ++r) __stcs(o + threadIdx.x + r * 256, v[r & 3]);
}
extern "C" int bw_rw14(const void *in, void *out, int64_t n_el, int n_f) {
    rw14<<<(unsigned)n_el, 256>>>((const float2 *)in, (float2 *)out, n_f);
    return (int)cudaGetLastError();
}
