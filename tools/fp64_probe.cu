// fp64_probe.cu — measure DFMA latency and per-SM throughput on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe tools/fp64_probe.cu && ./fp64_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain(double* out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-9 + i;
    long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (double)(t1 - t0) / iters;   // cycles per iteration
    if (s == 12345.0) out[0] = s;
}

template <int ILP>
void run(int blocks, int threads, const char* tag) {
    double* d;
    cudaMalloc(&d, 16);
    const int iters = 4096;
    chain<ILP><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chain<ILP><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double flops = 2.0 * ILP * (double)iters * blocks * threads;
    printf("%-28s ILP=%2d blocks=%4d threads=%4d: %.2f cyc/iter (thread 0)  %.2f TFLOP/s\n", tag, ILP, blocks, threads,
           h[1], flops / (ms * 1e-3) / 1e12);
    cudaFree(d);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<1>(1, 32, "latency (1 warp, chain)");
    run<4>(1, 32, "1 warp ILP4");
    run<8>(1, 32, "1 warp ILP8");
    run<16>(1, 32, "1 warp ILP16");
    run<8>(1, 128, "4 warps ILP8 (1/SMSP)");
    run<16>(1, 128, "4 warps ILP16");
    run<8>(1, 256, "8 warps ILP8");
    run<4>(sms, 256, "full chip 8 warps ILP4");
    run<8>(sms, 256, "full chip 8 warps ILP8");
    run<16>(sms, 256, "full chip 8 warps ILP16");
    run<8>(sms, 512, "full chip 16 warps ILP8");
    run<8>(sms * 2, 512, "full chip 32 warps ILP8");
    return 0;
}
