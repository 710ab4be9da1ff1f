// ffma2_probe.cu -- FP32 FMA throughput on this GPU: scalar FFMA vs packed
// FFMA2 (fma.rn.f32x2, sm_100), 8 independent chains per thread, full SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma2_probe tools/ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__global__ void scalar(float* out, int iters) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-7f + i;
    const float a = 0.9999f, b = 1e-6f;
    for (int k = 0; k < iters; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5f) out[0] = s;
}
__global__ void packed(float* out, int iters) {
    u64 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (u64)(threadIdx.x + i) * 0x0001000100010001ull;
    const u64 a = 0x3f7ff9723f7ff972ull, b = 0x358637bd358637bdull;
    for (int k = 0; k < iters; ++k)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma2(x[i], a, b);
    u64 s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= x[i];
    if (s == 12345) out[0] = (float)s;
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 4);
    const int iters = 1 << 16, threads = 1024, blocks = sms * 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) scalar<<<blocks, threads>>>(out, iters);
            else packed<<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fmas = (double)blocks * threads * iters * 8 * (mode ? 2 : 1);
        printf("{\"probe\": \"%s\", \"ms\": %.3f, \"tflops\": %.2f}\n", mode ? "ffma2" : "ffma", ms, 2 * fmas / ms / 1e9);
    }
    return 0;
}
