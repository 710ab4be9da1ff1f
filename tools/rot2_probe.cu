// rot2_probe.cu — FP64 issue rate of the register-group math patterns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rot2_probe tools/rot2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void rot2_mul(const double2 m00, const double2 m01, const double2 m10, const double2 m11,
                                         double2& u, double2& v) {
    double2 a, b;
    a.x = fma(m00.x, u.x, fma(-m00.y, u.y, fma(m01.x, v.x, -m01.y * v.y)));
    a.y = fma(m00.x, u.y, fma(m00.y, u.x, fma(m01.x, v.y, m01.y * v.x)));
    b.x = fma(m10.x, u.x, fma(-m10.y, u.y, fma(m11.x, v.x, -m11.y * v.y)));
    b.y = fma(m10.x, u.y, fma(m10.y, u.x, fma(m11.x, v.y, m11.y * v.x)));
    u = a;
    v = b;
}

// mode 0: DFMA only; 1: DMUL only; 2: rot2 on 16 register amplitudes, 4 bits
__global__ void probe(double* out, int iters, int mode, const double2* mats) {
    double2 a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = make_double2(threadIdx.x * 1e-9 + j, j * 0.5);
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    const double c0 = 0.999999, c1 = 1e-7;
    if (mode == 0) {
        for (int k = 0; k < iters; ++k)
#pragma unroll
            for (int r = 0; r < 16; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = fma(x[i], c0, c1);
    } else if (mode == 1) {
        for (int k = 0; k < iters; ++k)
#pragma unroll
            for (int r = 0; r < 16; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = x[i] * c0;
    } else {
        __shared__ double2 sm[16];
        if (threadIdx.x < 16) sm[threadIdx.x] = mats[threadIdx.x];
        __syncthreads();
        for (int k = 0; k < iters; ++k) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double2 m00 = sm[4 * r], m01 = sm[4 * r + 1], m10 = sm[4 * r + 2], m11 = sm[4 * r + 3];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (!((j >> r) & 1)) rot2_mul(m00, m01, m10, m11, a[j], a[j | (1 << r)]);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += a[j].x + a[j].y;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    double2* m;
    cudaMalloc(&d, 16);
    cudaMalloc(&m, 16 * sizeof(double2));
    double2 hm[16];
    for (int i = 0; i < 16; ++i) hm[i] = make_double2(0.6 + 0.01 * i, 0.3 - 0.01 * i);
    cudaMemcpy(m, hm, sizeof(hm), cudaMemcpyHostToDevice);
    const int iters = 256;
    const char* names[3] = {"DFMA", "DMUL", "rot2 (16 amps, 4 bits)"};
    for (int warps : {8, 16}) {
        for (int mode = 0; mode < 3; ++mode) {
            probe<<<sms, warps * 32>>>(d, iters, mode, m);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            probe<<<sms, warps * 32>>>(d, iters, mode, m);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double threads = (double)sms * warps * 32;
            // flops: DFMA 2/instr, DMUL 1/instr, rot2: 4 bits x 8 pairs x 28 flops
            double flops = mode == 0 ? threads * iters * 128 * 2.0 : mode == 1 ? threads * iters * 128.0
                                                                               : threads * iters * 4 * 8 * 28.0;
            double instr = mode == 2 ? threads * iters * 4 * 8 * 16.0 : threads * iters * 128.0;
            printf("%2d warps/SM %-24s %.3f ms  %.2f TFLOP/s  %.2f FP64 warp-instr/clk/SM (at 1.965 GHz)\n", warps,
                   names[mode], ms, flops / ms / 1e9, instr / 32 / (ms * 1e-3) / sms / 1.965e9);
        }
    }
    return 0;
}
