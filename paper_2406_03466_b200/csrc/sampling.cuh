// sampling.cuh — counts mode (reference backend.py:140-157) on the device.
//
// The reference samples with numpy: edges = cumsum(probs) (sequential
// additions), u = Generator(PCG64(seed)).random(shots), draws =
// searchsorted(edges, u, side="right") clamped to 2^n - 1, counts =
// bincount(draws).  Here: the cumsum runs sequentially per state (same
// addition order as numpy), the PCG64 128-bit LCG with XSL-RR output is
// restated exactly (each thread jumps ahead to its block of draws), the
// inverse CDF is a binary search, and draws are tallied with integer atomics
// (order-independent), then compacted in ascending outcome order.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace qvb {

struct U128 {
    uint64_t hi, lo;
};

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
    return r;
}
__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
    return r;
}

// numpy's PCG64: state <- state * M + inc, output XSL-RR of the new state
__device__ __forceinline__ U128 pcg_mult() { return U128{2549297995355413924ull, 4865540595714422341ull}; }

struct Pcg64 {
    U128 state, inc;
    __device__ __forceinline__ uint64_t next() {
        state = add128(mul128(state, pcg_mult()), inc);
        const uint64_t x = state.hi ^ state.lo;
        const unsigned rot = (unsigned)(state.hi >> 58);
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    __device__ __forceinline__ double next_double() {   // Generator.random(): (next >> 11) * 2^-53
        return (double)(next() >> 11) * (1.0 / 9007199254740992.0);
    }
    // jump ahead by `delta` steps (Brown's LCG skip, O(log delta))
    __device__ void advance(uint64_t delta) {
        U128 acc_mult = {0, 1}, acc_plus = {0, 0}, cur_mult = pcg_mult(), cur_plus = inc;
        while (delta) {
            if (delta & 1) {
                acc_mult = mul128(acc_mult, cur_mult);
                acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
            }
            cur_plus = mul128(add128(cur_mult, U128{0, 1}), cur_plus);
            cur_mult = mul128(cur_mult, cur_mult);
            delta >>= 1;
        }
        state = add128(mul128(acc_mult, state), acc_plus);
    }
};

// edges = cumsum(p) in place, one thread per state, sequential (numpy order).
__global__ void cumsum_kernel(double* __restrict__ probs, int64_t dim, int64_t nstates) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nstates) return;
    double* p = probs + s * dim;
    double acc = 0.0;
    for (int64_t i = 0; i < dim; ++i) {
        acc += p[i];
        p[i] = acc;
    }
}

// One CTA per circuit: `shots` draws split into contiguous blocks per thread.
// rows[c] = row of edges of circuit c; hist[c] = 2^n uint32 counters.
__global__ void sample_kernel(const double* __restrict__ edges, const int64_t* __restrict__ edge_row,
                              const uint64_t* __restrict__ rng, int64_t shots, int64_t dim,
                              unsigned* __restrict__ hist, int64_t c0) {
    const int64_t c = c0 + blockIdx.x;
    const double* e = edges + edge_row[c] * dim;
    unsigned* h = hist + (int64_t)blockIdx.x * dim;
    const int64_t per = (shots + blockDim.x - 1) / blockDim.x;
    const int64_t j0 = (int64_t)threadIdx.x * per;
    const int64_t j1 = j0 + per < shots ? j0 + per : shots;
    if (j0 >= j1) return;
    Pcg64 g;
    g.state = U128{rng[4 * c], rng[4 * c + 1]};
    g.inc = U128{rng[4 * c + 2], rng[4 * c + 3]};
    g.advance((uint64_t)j0);
    for (int64_t j = j0; j < j1; ++j) {
        const double u = g.next_double();
        // searchsorted(side="right"): number of edges <= u
        int64_t lo = 0, hi = dim;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (e[mid] <= u) lo = mid + 1;
            else hi = mid;
        }
        const int64_t idx = lo < dim ? lo : dim - 1;
        atomicAdd(h + idx, 1u);
    }
}

// Compact one circuit's histogram to (index, count) pairs, ascending:
// out row = [m, idx_0, cnt_0, ..., idx_{m-1}, cnt_{m-1}].
__global__ void compact_counts_kernel(const unsigned* __restrict__ hist, int64_t dim, double* __restrict__ out,
                                      int64_t row_len, int64_t c0) {
    __shared__ int64_t base[1024 + 1];
    const unsigned* h = hist + (int64_t)blockIdx.x * dim;
    double* row = out + (c0 + blockIdx.x) * row_len;
    const int64_t per = (dim + blockDim.x - 1) / blockDim.x;
    const int64_t i0 = (int64_t)threadIdx.x * per;
    const int64_t i1 = i0 + per < dim ? i0 + per : dim;
    int64_t nz = 0;
    for (int64_t i = i0; i < i1; ++i) nz += h[i] != 0;
    base[threadIdx.x + 1] = nz;
    __syncthreads();
    if (threadIdx.x == 0) {
        base[0] = 0;
        for (unsigned t = 1; t <= blockDim.x; ++t) base[t] += base[t - 1];
        row[0] = (double)base[blockDim.x];
    }
    __syncthreads();
    int64_t at = base[threadIdx.x];
    for (int64_t i = i0; i < i1; ++i)
        if (h[i]) {
            row[1 + 2 * at] = (double)i;
            row[2 + 2 * at] = (double)h[i];
            ++at;
        }
}

}  // namespace qvb
