// kernels.cuh — sm_100a state-vector kernels.
//
// pass_kernel: one HBM sweep of a plan pass over a batch of states.  A CTA
//   owns one tile (2^k amplitudes spread over the pass's k index bits), stages
//   it in shared memory with 128-bit coalesced loads, applies the pass's
//   register groups (16 amplitudes per thread, up to four fused 2x2 matrices
//   per group, CNOTs folded into the slot map at plan time so they cost no
//   data movement), and writes the tile back -- or, on a state's last pass,
//   reduces it (norm, support probabilities, Pauli terms, JS loss) without
//   writing it.  Replaces the per-gate full sweeps of the reference
//   (pkg/src/qvirt/kernels.py:18-70) and its reductions (:73-94).
//
// All reductions are fixed-shape trees in FP64 with no atomics, so a result
// depends only on the circuit, never on its position in a launch or on the GPU.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "plan.hpp"

namespace qvb {

enum EpiFlags : int {
    F_STORE = 1,       // write the tile back
    F_NORM = 2,        // multi-tile: per-tile sum |a|^2 -> partial
    F_SUPPORT = 4,     // multi-tile: |a|^2 at support indices -> sup_out (unnormalised)
    F_SINGLE = 8,      // whole state is one tile: epilogue computed in-kernel
    F_S_SUPPORT = 16,  // single: normalised support probabilities + norm
    F_S_JS = 32,       // single: JS loss
    F_S_FULL = 64,     // single: all normalised probabilities
    F_S_PAULI = 128,   // single: Pauli terms
};

struct LaunchEntry {
    const void* in;     // nullptr: the input is |0...0>
    void* out;          // nullptr: no store
    const void* mats;   // matrix table of this state (slot 0)
    int64_t rslot;      // result slot (outputs)
    int64_t pslot;      // partial-sum slot (multi-tile norm partials)
    int64_t pad;
};

struct EpiArgs {
    int flags;
    int n;
    int64_t ntiles;
    double* partial;           // [rslot * ntiles + tile]
    const int32_t* sup_off;    // multi-tile support CSR over tiles [ntiles + 1]
    const int32_t* sup_local;
    const int32_t* sup_pos;
    double* sup_out;           // [rslot * (S + 1) + pos]
    int64_t S;
    const uint64_t* support;   // [S] (single tile)
    const double* target;      // [S]
    double* js_out;            // [rslot]
    double* full_out;          // [rslot << n]
    const int64_t* term_off;   // [rslot] .. [rslot + 1]
    const uint64_t* t_flip;
    const uint64_t* t_phase;
    double* pauli_out;         // [term]
};

template <typename T> struct Cx;
template <> struct Cx<double> { typedef double2 V; };
template <> struct Cx<float> { typedef float2 V; };

template <typename T, typename V>
__device__ __forceinline__ void rot2(const T* __restrict__ m, V& u, V& v) {
    const T m00r = m[0], m00i = m[1], m01r = m[2], m01i = m[3];
    const T m10r = m[4], m10i = m[5], m11r = m[6], m11i = m[7];
    V a, b;
    a.x = fma(m00r, u.x, fma(-m00i, u.y, fma(m01r, v.x, -m01i * v.y)));
    a.y = fma(m00r, u.y, fma(m00i, u.x, fma(m01r, v.y, m01i * v.x)));
    b.x = fma(m10r, u.x, fma(-m10i, u.y, fma(m11r, v.x, -m11i * v.y)));
    b.y = fma(m10r, u.y, fma(m10i, u.x, fma(m11r, v.y, m11i * v.x)));
    u = a;
    v = b;
}

// Deterministic block sum: xor-butterfly inside each warp (lane 0's value is
// used), then warp totals added in warp order by every thread.
__device__ __forceinline__ double block_sum(double v, double* sred) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sred[warp] = v;
    __syncthreads();
    double t = 0.0;
    const int nw = blockDim.x >> 5;
    for (int w = 0; w < nw; ++w) t += sred[w];
    return t;
}

__device__ __forceinline__ double js_term(double p, double q) {
    // reference ddcl.py:53-60: m = (p+q)/2; zero-numerator terms contribute nothing
    const double m = 0.5 * (p + q);
    double r = 0.0;
    if (p > 0.0) r += 0.5 * p * log(p / m);
    if (q > 0.0) r += 0.5 * q * log(q / m);
    return r;
}

template <typename T, int NT>
__global__ void __launch_bounds__(NT, 2) pass_kernel(const PassDesc pd, const GroupDesc* __restrict__ gdesc,
                                                  const LaunchEntry* __restrict__ ent, int nstates, EpiArgs ep) {
    typedef typename Cx<T>::V V;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int k = pd.k;
    const int tb = k - kRegBits;          // thread bits
    const int nt = 1 << tb;               // active threads
    V* tile = reinterpret_cast<V*>(smem_raw);
    GroupDesc* sg = reinterpret_cast<GroupDesc*>(smem_raw + (sizeof(V) << k));
    T* smat = reinterpret_cast<T*>(sg + pd.ng);
    double* sred = reinterpret_cast<double*>(smat + (size_t)pd.nm * 8);

    const int tid = threadIdx.x;
    const int64_t bid = blockIdx.x;
    const int y = (int)(bid % nstates);
    const int64_t x = bid / nstates;
    const LaunchEntry e = ent[y];

    {   // stage groups and this state's matrices
        const uint32_t* gsrc = reinterpret_cast<const uint32_t*>(gdesc + pd.g0);
        uint32_t* gdst = reinterpret_cast<uint32_t*>(sg);
        for (int i = tid; i < pd.ng * 16; i += blockDim.x) gdst[i] = gsrc[i];
        const T* msrc = reinterpret_cast<const T*>(e.mats) + (size_t)pd.m0 * 8;
        for (int i = tid; i < pd.nm * 8; i += blockDim.x) smat[i] = msrc[i];
    }
    uint64_t outer = 0;
    for (int j = 0; j < pd.n_outer; ++j)
        if ((x >> j) & 1) outer |= 1ull << pd.obits[j];

    const bool active = tid < nt;
    uint32_t tslot = 0;
    uint64_t tg = 0;
    for (int j = 0; j < tb; ++j)
        if ((tid >> j) & 1) { tslot ^= pd.swz[j]; tg |= 1ull << pd.sbits[j]; }
    const bool gen = e.in == nullptr;
    const bool zero_tile = gen && x != 0;
    if (active) {
        if (gen) {
#pragma unroll
            for (int it = 0; it < 16; ++it) {
                V v;
                v.x = (x == 0 && tid == 0 && it == 0) ? T(1) : T(0);
                v.y = T(0);
                tile[tslot ^ pd.swz_hi[it]] = v;
            }
        } else {
            const V* __restrict__ in = reinterpret_cast<const V*>(e.in);
            V r[16];
#pragma unroll
            for (int it = 0; it < 16; ++it) r[it] = __ldcs(in + (outer | tg | pd.g_hi[it]));
#pragma unroll
            for (int it = 0; it < 16; ++it) tile[tslot ^ pd.swz_hi[it]] = r[it];
        }
    }
    __syncthreads();

    if (!zero_tile) {
        for (int g = 0; g < pd.ng; ++g) {
            if (active) {
                const GroupDesc& G = sg[g];
                uint32_t base = 0;
                for (int m = 0; m < tb; ++m)
                    if ((tid >> m) & 1) base ^= G.tcol[m];
                V a[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) a[j] = tile[base ^ G.combo[j]];
#pragma unroll
                for (int r = 0; r < kRegBits; ++r) {
                    const int mi = G.mat[r];
                    if (mi >= 0) {
                        const T* M = smat + mi * 8;
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (!((j >> r) & 1)) rot2<T, V>(M, a[j], a[j | (1 << r)]);
                    }
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) tile[base ^ G.combo[j]] = a[j];
            }
            __syncthreads();
        }
    }

    // ---- store / reduce -------------------------------------------------
    uint32_t fslot = 0;
    for (int j = 0; j < tb; ++j)
        if ((tid >> j) & 1) fslot ^= pd.fin[j];
    double acc = 0.0;
    if (active) {
        V* __restrict__ out = reinterpret_cast<V*>(e.out);
        const bool store = (ep.flags & F_STORE) && out != nullptr;
#pragma unroll
        for (int it = 0; it < 16; ++it) {
            const V v = tile[fslot ^ pd.fin_hi[it]];
            if (store) __stcs(out + (outer | tg | pd.g_hi[it]), v);
            acc += (double)v.x * (double)v.x + (double)v.y * (double)v.y;
        }
    }
    if (!(ep.flags & (F_NORM | F_SINGLE | F_SUPPORT))) return;

    if (ep.flags & F_NORM) {
        const double s = block_sum(acc, sred);
        if (tid == 0) ep.partial[e.pslot * ep.ntiles + x] = s;
    }
    if (ep.flags & F_SUPPORT) {
        const int32_t lo = ep.sup_off[x], hi = ep.sup_off[x + 1];
        double* row = ep.sup_out + e.rslot * (ep.S + 1);
        for (int32_t i = lo + tid; i < hi; i += blockDim.x) {
            const uint32_t slot = apply_cols(pd.fin, k, (uint32_t)ep.sup_local[i]);
            const V v = tile[slot];
            row[ep.sup_pos[i]] = (double)v.x * (double)v.x + (double)v.y * (double)v.y;
        }
    }
    if (!(ep.flags & F_SINGLE)) return;

    // ---- single-tile epilogue: the tile is the whole state ----------------
    const double total = block_sum(acc, sred);
    const int64_t dim = 1ll << ep.n;
    if (ep.flags & F_S_FULL) {
        double* row = ep.full_out + (e.rslot << ep.n);
        if (active) {
#pragma unroll
            for (int it = 0; it < 16; ++it) {
                const uint32_t i = (uint32_t)tid | ((uint32_t)it << tb);
                if (i < dim) {
                    const V v = tile[fslot ^ pd.fin_hi[it]];
                    row[i] = ((double)v.x * (double)v.x + (double)v.y * (double)v.y) / total;
                }
            }
        }
    }
    if (ep.flags & (F_S_SUPPORT | F_S_JS)) {
        double* row = (ep.flags & F_S_SUPPORT) ? ep.sup_out + e.rslot * (ep.S + 1) : nullptr;
        double jsum = 0.0, qsum = 0.0;
        for (int64_t s = tid; s < ep.S; s += blockDim.x) {
            const uint64_t idx = ep.support[s];
            double q = 0.0;
            if (idx < (uint64_t)dim) {
                const V v = tile[apply_cols(pd.fin, k, (uint32_t)idx)];
                q = ((double)v.x * (double)v.x + (double)v.y * (double)v.y) / total;
            }
            if (row) row[s] = q;
            if (ep.flags & F_S_JS) { jsum += js_term(ep.target[s], q); qsum += q; }
        }
        if (row && tid == 0) row[ep.S] = total;
        if (ep.flags & F_S_JS) {
            const double J = block_sum(jsum, sred);
            const double Q = block_sum(qsum, sred);
            if (tid == 0) ep.js_out[e.rslot] = J + 0.5 * 0.69314718055994530942 * (1.0 - Q);
        }
    }
    if (ep.flags & F_S_PAULI) {
        const int64_t t0 = ep.term_off[e.rslot], t1 = ep.term_off[e.rslot + 1];
        for (int64_t t = t0; t < t1; ++t) {
            const uint64_t F = ep.t_flip[t], PH = ep.t_phase[t];
            const uint32_t fF = apply_cols(pd.fin, k, (uint32_t)F);
            double ar = 0.0, ai = 0.0;
            if (active) {
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const uint32_t i = (uint32_t)tid | ((uint32_t)it << tb);
                    const uint32_t sl = fslot ^ pd.fin_hi[it];
                    const V a = tile[sl];
                    const V b = tile[sl ^ fF];
                    // conj(b) * a
                    const double tr = (double)b.x * (double)a.x + (double)b.y * (double)a.y;
                    const double ti = (double)b.x * (double)a.y - (double)b.y * (double)a.x;
                    if (__popcll((uint64_t)i & PH) & 1) { ar -= tr; ai -= ti; }
                    else { ar += tr; ai += ti; }
                }
            }
            const double R = block_sum(ar, sred);
            const double I = block_sum(ai, sred);
            if (tid == 0) {
                const int ny = __popcll(ep.t_flip[t] & ep.t_phase[t]) & 3;   // Y factors flip and carry phase
                double val;
                switch (ny) {
                    case 0: val = R; break;
                    case 1: val = -I; break;
                    case 2: val = -R; break;
                    default: val = I; break;
                }
                ep.pauli_out[t] = val;
            }
        }
    }
}

// Multi-tile norm / support finalisation: one CTA per result slot.
// slots[2*b] = result slot, slots[2*b+1] = partial slot.
__global__ void finalize_dist_kernel(const int64_t* __restrict__ slots, int64_t ntiles, const double* __restrict__ partial,
                                     double* __restrict__ sup_out, int64_t S, const double* __restrict__ target,
                                     double* __restrict__ js_out, int want_js) {
    __shared__ double sred[32];
    const int64_t r = slots[2 * blockIdx.x], ps = slots[2 * blockIdx.x + 1];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < ntiles; i += blockDim.x) acc += partial[ps * ntiles + i];
    const double total = block_sum(acc, sred);
    double* row = sup_out + r * (S + 1);
    double jsum = 0.0, qsum = 0.0;
    for (int64_t s = threadIdx.x; s < S; s += blockDim.x) {
        const double q = row[s] / total;
        row[s] = q;
        if (want_js) { jsum += js_term(target[s], q); qsum += q; }
    }
    if (threadIdx.x == 0) row[S] = total;
    if (want_js) {
        const double J = block_sum(jsum, sred);
        const double Q = block_sum(qsum, sred);
        if (threadIdx.x == 0) js_out[r] = J + 0.5 * 0.69314718055994530942 * (1.0 - Q);
    }
}

// Multi-tile Pauli term: reads the stored state once.  Block b owns a fixed
// range of pair indices; partial sums are combined by finalize_pauli_kernel.
template <typename T>
__global__ void __launch_bounds__(256) pauli_sweep_kernel(const typename Cx<T>::V* __restrict__ st, int n, uint64_t F,
                                                           uint64_t PH, int64_t per_block, double2* __restrict__ partial) {
    typedef typename Cx<T>::V V;
    __shared__ double sred[32];
    double ar = 0.0, ai = 0.0;
    const int64_t j0 = (int64_t)blockIdx.x * per_block;
    if (F == 0) {
        for (int64_t j = j0 + threadIdx.x; j < j0 + per_block; j += blockDim.x) {
            const V a = st[j];
            const double p = (double)a.x * (double)a.x + (double)a.y * (double)a.y;
            if (__popcll((uint64_t)j & PH) & 1) ar -= p; else ar += p;
        }
    } else {
        const int pb = __ffsll((long long)F) - 1;
        const uint64_t lowm = (1ull << pb) - 1;
        for (int64_t j = j0 + threadIdx.x; j < j0 + per_block; j += blockDim.x) {
            const uint64_t i = (((uint64_t)j & ~lowm) << 1) | ((uint64_t)j & lowm);
            const uint64_t i2 = i ^ F;
            const V a = st[i], b = st[i2];
            const double tr = (double)b.x * (double)a.x + (double)b.y * (double)a.y;
            const double ti = (double)b.x * (double)a.y - (double)b.y * (double)a.x;
            // term(i) = conj(b) a s(i); term(i2) = conj(a) b s(i2) = conj(term(i)) * s(i) s(i2)
            const double si = (__popcll(i & PH) & 1) ? -1.0 : 1.0;
            const double s2 = (__popcll(i2 & PH) & 1) ? -1.0 : 1.0;
            ar += si * tr + s2 * tr;
            ai += si * ti - s2 * ti;
        }
    }
    const double R = block_sum(ar, sred);
    const double I = block_sum(ai, sred);
    if (threadIdx.x == 0) partial[blockIdx.x] = make_double2(R, I);
}

__global__ void finalize_pauli_kernel(const double2* __restrict__ partial, int64_t nblocks, int ny, double* __restrict__ out) {
    __shared__ double sred[32];
    double ar = 0.0, ai = 0.0;
    for (int64_t i = threadIdx.x; i < nblocks; i += blockDim.x) { ar += partial[i].x; ai += partial[i].y; }
    const double R = block_sum(ar, sred);
    const double I = block_sum(ai, sred);
    if (threadIdx.x == 0) {
        double val;
        switch (ny & 3) {
            case 0: val = R; break;
            case 1: val = -I; break;
            case 2: val = -R; break;
            default: val = I; break;
        }
        *out = val;
    }
}

}  // namespace qvb

namespace qvb {
// Multi-tile full distribution: p_i / total for a stored state.
template <typename T>
__global__ void full_probs_kernel(const typename Cx<T>::V* __restrict__ st, int64_t dim, const double* __restrict__ total,
                                  double* __restrict__ out) {
    typedef typename Cx<T>::V V;
    const double t = *total;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x) {
        const V a = st[i];
        out[i] = ((double)a.x * (double)a.x + (double)a.y * (double)a.y) / t;
    }
}
}  // namespace qvb
