// dmma_probe.cu — is FP64 mma.sync (DMMA) a separate pipe from DFMA on this GPU?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
// Runs DFMA-only, DMMA-only and mixed warps; if mixed throughput exceeds the
// better of the two alone, the pipes overlap.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// mode 0: DFMA only, 1: DMMA only, 2: even warps DFMA / odd warps DMMA
__global__ void probe(double* out, int iters, int mode) {
    const int warp = threadIdx.x >> 5;
    const bool use_mma = mode == 1 || (mode == 2 && (warp & 1));
    double x[8], d[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-9 + i; d[i][0] = d[i][1] = i; }
    const double a = 0.999999, b = 1e-7;
    if (use_mma) {
        for (int k = 0; k < iters; ++k) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(d[i][0], d[i][1], a, b);
        }
    } else {
        for (int k = 0; k < iters; ++k) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i] + d[i][0] + d[i][1];
    if (s == 1234.5) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 16);
    const int iters = 2048, threads = 512;
    for (int mode = 0; mode < 3; ++mode) {
        probe<<<sms, threads>>>(d, iters, mode);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<sms, threads>>>(d, iters, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warps = (double)sms * threads / 32;
        // DFMA warp-instr = 32 FMA; DMMA m8n8k4 = 8*8*4 = 256 FMA
        double fma_dfma = 0, fma_dmma = 0;
        if (mode == 0) fma_dfma = warps * iters * 8 * 32.0;
        if (mode == 1) fma_dmma = warps * iters * 8 * 256.0;
        if (mode == 2) { fma_dfma = warps / 2 * iters * 8 * 32.0; fma_dmma = warps / 2 * iters * 8 * 256.0; }
        printf("mode %d (%s): %.3f ms  DFMA %.2f TFLOP/s  DMMA %.2f TFLOP/s  total %.2f TFLOP/s\n", mode,
               mode == 0 ? "DFMA only" : mode == 1 ? "DMMA only" : "mixed", ms, 2 * fma_dfma / ms / 1e9,
               2 * fma_dmma / ms / 1e9, 2 * (fma_dfma + fma_dmma) / ms / 1e9);
    }
    return 0;
}
