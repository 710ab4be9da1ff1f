// Microbenchmark of one register group's cost components (complex128, R = 4):
// 16 amplitudes per thread, 4 fused 2x2 matrices per shared-memory round trip,
// 256 threads per CTA, 64 KiB tile, 2 CTAs per SM (the product configuration).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/group_micro tools/group_micro.cu
//   tools/group_micro [groups]
//
// Variants:
//   0  product-like: descriptors (combo / tcol / matrix ids) + matrices from smem each group, __syncwarp
//   1  matrices + offsets in registers (no descriptor loads), __syncwarp
//   2  as 1 with __syncthreads
//   3  as 1 with no synchronisation (timing only)
//   4  registers only: no shared-memory round trip (the math's own rate)
//   5  as 0 but matrices from smem only (offsets precomputed per thread), __syncwarp
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void rot2(const double2 m00, const double2 m01, const double2 m10, const double2 m11,
                                     double2& a, double2& b) {
    const double2 x = a, y = b;
    a.x = m00.x * x.x - m00.y * x.y + m01.x * y.x - m01.y * y.y;
    a.y = m00.x * x.y + m00.y * x.x + m01.x * y.y + m01.y * y.x;
    b.x = m10.x * x.x - m10.y * x.y + m11.x * y.x - m11.y * y.y;
    b.y = m10.x * x.y + m10.y * x.x + m11.x * y.y + m11.y * y.x;
}

struct Desc { uint32_t combo[16]; uint32_t tcol[8]; int32_t mat[4]; int32_t pad[4]; };

template <int V>
__global__ void __launch_bounds__(256, 2) micro(double2* out, const double2* mats_g, const Desc* desc_g, int groups) {
    extern __shared__ __align__(16) unsigned char smem[];
    double2* tile = reinterpret_cast<double2*>(smem);
    Desc* sd = reinterpret_cast<Desc*>(smem + 65536);
    double2* sm = reinterpret_cast<double2*>(smem + 65536 + 8 * sizeof(Desc));
    const int tid = threadIdx.x;
    for (int i = tid; i < 4096; i += 256) tile[i] = make_double2(1e-3 * i, 0.5);
    for (int i = tid; i < 8 * (int)sizeof(Desc) / 4; i += 256)
        reinterpret_cast<uint32_t*>(sd)[i] = reinterpret_cast<const uint32_t*>(desc_g)[i];
    for (int i = tid; i < 64; i += 256) sm[i] = mats_g[i];
    __syncthreads();
    const double2 r00 = sm[0], r01 = sm[1], r10 = sm[2], r11 = sm[3];
    // per-thread bases of the two alternating patterns (register bits 0..3 / 8..11)
    uint32_t bA = 0, bB = 0;
    for (int m = 0; m < 8; ++m) if ((tid >> m) & 1) { bA ^= sd[0].tcol[m]; bB ^= sd[1].tcol[m]; }
    double2 a[16];
    if (V == 4)
        for (int j = 0; j < 16; ++j) a[j] = tile[(tid * 16 + j) & 4095];
    for (int g = 0; g < groups; ++g) {
        if (V == 0) {
            const Desc& D = sd[g & 7];
            const int4 mi = *reinterpret_cast<const int4*>(D.mat);
            uint32_t base = 0;
#pragma unroll
            for (int m = 0; m < 8; ++m) if ((tid >> m) & 1) base ^= D.tcol[m];
            uint32_t off[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 c = reinterpret_cast<const uint4*>(D.combo)[q];
                off[4 * q] = base ^ c.x; off[4 * q + 1] = base ^ c.y; off[4 * q + 2] = base ^ c.z; off[4 * q + 3] = base ^ c.w;
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = *reinterpret_cast<const double2*>(smem + off[j]);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int m = r == 0 ? mi.x : r == 1 ? mi.y : r == 2 ? mi.z : mi.w;
                const double2* M = sm + m * 4;
                const double2 m00 = M[0], m01 = M[1], m10 = M[2], m11 = M[3];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (!((j >> r) & 1)) rot2(m00, m01, m10, m11, a[j], a[j | (1 << r)]);
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) *reinterpret_cast<double2*>(smem + off[j]) = a[j];
            __syncwarp();
        } else if (V == 5) {
            const Desc& D = sd[g & 7];
            const int4 mi = *reinterpret_cast<const int4*>(D.mat);
            uint32_t off[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) off[j] = (g & 1) ? (bB ^ (uint32_t)(j << 8) * 16) : (bA ^ (uint32_t)j * 16);
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = *reinterpret_cast<const double2*>(smem + off[j]);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int m = r == 0 ? mi.x : r == 1 ? mi.y : r == 2 ? mi.z : mi.w;
                const double2* M = sm + m * 4;
                const double2 m00 = M[0], m01 = M[1], m10 = M[2], m11 = M[3];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (!((j >> r) & 1)) rot2(m00, m01, m10, m11, a[j], a[j | (1 << r)]);
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) *reinterpret_cast<double2*>(smem + off[j]) = a[j];
            __syncwarp();
        } else if (V == 4) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (!((j >> r) & 1)) rot2(r00, r01, r10, r11, a[j], a[j | (1 << r)]);
        } else {
            uint32_t off[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) off[j] = (g & 1) ? (bB ^ (uint32_t)(j << 8) * 16) : (bA ^ (uint32_t)j * 16);
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = *reinterpret_cast<const double2*>(smem + off[j]);
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (!((j >> r) & 1)) rot2(r00, r01, r10, r11, a[j], a[j | (1 << r)]);
#pragma unroll
            for (int j = 0; j < 16; ++j) *reinterpret_cast<double2*>(smem + off[j]) = a[j];
            if (V == 1) __syncwarp();
            if (V == 2) __syncthreads();
        }
    }
    if (V == 4) {
        double2 s = make_double2(0, 0);
        for (int j = 0; j < 16; ++j) { s.x += a[j].x; s.y += a[j].y; }
        out[blockIdx.x * 256 + tid] = s;
    } else {
        __syncthreads();
        out[blockIdx.x * 256 + tid] = tile[tid];
    }
}

static int g_force_per_sm = 0;   // argv[2]: CTAs per SM (0 = occupancy)

template <int V>
int run(int groups, double2* out, const double2* mats, const Desc* desc, int sms) {
    const size_t smem = 65536 + 8 * sizeof(Desc) + 64 * sizeof(double2);
    CK(cudaFuncSetAttribute(micro<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, micro<V>, 256, smem));
    if (g_force_per_sm > 0 && g_force_per_sm < per_sm) per_sm = g_force_per_sm;
    const int blocks = per_sm * sms;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    micro<V><<<blocks, 256, smem>>>(out, mats, desc, groups / 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    micro<V><<<blocks, 256, smem>>>(out, mats, desc, groups);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = (double)blocks * 256 * groups * 4 * 8 * 28;
    printf("variant %d: %d CTAs/SM, %.3f ms, %.2f TFLOP/s (2x2 complex updates, 28 flops per pair)\n", V, per_sm, ms,
           flops / ms / 1e9);
    return 0;
}

int main(int argc, char** argv) {
    const int groups = argc > 1 ? atoi(argv[1]) : 4000;
    g_force_per_sm = argc > 2 ? atoi(argv[2]) : 0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2* out;
    double2* mats;
    Desc* desc;
    CK(cudaMalloc(&out, 4096 * 256 * sizeof(double2)));
    CK(cudaMalloc(&mats, 64 * sizeof(double2)));
    CK(cudaMalloc(&desc, 8 * sizeof(Desc)));
    double2 hm[64];
    for (int i = 0; i < 16; ++i) {   // rotation-like unitary matrices (values stay bounded)
        const double c = cos(0.1 * (i + 1)), s = sin(0.1 * (i + 1));
        hm[4 * i] = make_double2(c, 0.0);
        hm[4 * i + 1] = make_double2(0.0, -s);
        hm[4 * i + 2] = make_double2(0.0, -s);
        hm[4 * i + 3] = make_double2(c, 0.0);
    }
    Desc hd[8];
    for (int d = 0; d < 8; ++d) {
        // register bits = 4 tile bits, thread bits = the other 8 (bank-friendly: lane bits at 16-byte stride)
        const int rb = (d & 1) ? 8 : 0;   // register bits 0..3 or 8..11
        int tb[8], n = 0;
        for (int b = 0; b < 12; ++b) if (b < rb || b >= rb + 4) tb[n++] = b;
        for (int j = 0; j < 16; ++j) hd[d].combo[j] = (uint32_t)(j << rb) * 16;
        // lanes must spread over the eight 16-byte bank groups: XOR-swizzle the
        // first three lane bits into slot bits 0..2 when those are register bits
        for (int m = 0; m < 8; ++m) hd[d].tcol[m] = ((1u << tb[m]) ^ (rb == 0 && m < 3 ? 1u << m : 0u)) * 16;
        for (int r = 0; r < 4; ++r) hd[d].mat[r] = (4 * d + r) % 16;
    }
    CK(cudaMemcpy(mats, hm, sizeof(hm), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(desc, hd, sizeof(hd), cudaMemcpyHostToDevice));
    if (run<4>(groups, out, mats, desc, sms) || run<3>(groups, out, mats, desc, sms) ||
        run<1>(groups, out, mats, desc, sms) || run<2>(groups, out, mats, desc, sms) ||
        run<5>(groups, out, mats, desc, sms) || run<0>(groups, out, mats, desc, sms))
        return 1;
    return 0;
}
