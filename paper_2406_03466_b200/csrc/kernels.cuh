// kernels.cuh — sm_100a state-vector kernels.
//
// pass_kernel: one HBM sweep of a plan pass over a batch of states.  CTAs are
//   persistent per state: a CTA stages the pass's group descriptors and its
//   state's fused matrices once, then walks tiles (2^k amplitudes spread over
//   the pass's k index bits).  Per tile it stages the amplitudes in shared
//   memory with 128-bit coalesced loads, applies the register groups (16
//   amplitudes per thread, up to four fused 2x2 matrices per group; CNOTs were
//   folded into the slot maps at plan time so they move no data), and writes
//   the tile back -- or, on a state's last pass, reduces it (norm, support
//   probabilities, Pauli terms, JS loss) without writing it.  Replaces the
//   per-gate full sweeps of the reference (pkg/src/qvirt/kernels.py:18-70) and
//   its reductions (:73-94).
//
// All reductions are fixed-shape trees in FP64 with no atomics, so a result
// depends only on the circuit, never on its position in a launch or the GPU.
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
    F_PAIR = 256,      // multi-tile: shift-pair epilogue over (Psi0 = aux, Xi = this tile)
    F_MT_PAULI = 512,  // multi-tile: per-tile partial sums of the state's Pauli terms assigned to this sweep
};

struct LaunchEntry {
    const void* in;     // nullptr: the input is |0...0>
    void* out;          // nullptr: no store
    const void* mats;   // matrix table of this state (slot 0)
    int64_t rslot;      // result slot (outputs)
    int64_t pslot;      // partial-sum slot (multi-tile norm partials)
    const void* aux;    // F_PAIR: the unshifted output state Psi0
};

struct EpiArgs {
    int flags;
    int n;
    int64_t ntiles;
    double* partial;           // [pslot * ntiles + tile]
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
    double* pair_sup;          // F_PAIR: [(rslot * S + pos) * 4 + {|Psi0|^2, |Xi|^2, Im(Psi0 conj Xi), Re(..)}]
    // F_MT_PAULI: term t of state rslot (term_off) is evaluated by the launch
    // whose `sweep` equals t_sweep[t]; t_fslot = physical slot offset of the
    // term's flip mask in that pass's final layout, t_phloc its phase mask in
    // logical tile bits, t_phout its phase mask on the outer bits
    int sweep;
    const int32_t* t_sweep;
    const uint32_t* t_fslot;
    const uint32_t* t_phloc;
    const uint64_t* t_phout;
    double2* pauli_partial;    // [t * ntiles + tile]
};


template <typename T> struct Cx;
template <> struct Cx<double> { typedef double2 V; };
template <> struct Cx<float> { typedef float2 V; };

// (u, v) <- [[m00, m01], [m10, m11]] (u, v) with m00 REAL (the host removes
// each fused matrix's global phase, normalise_phase in qvb200.cu): 4
// multiplies + 10 FMAs per pair instead of 4 + 12.
template <typename V>
__device__ __forceinline__ void rot2(const V m00, const V m01, const V m10, const V m11, V& u, V& v) {
    V a, b;
    a.x = fma(m00.x, u.x, fma(m01.x, v.x, -m01.y * v.y));
    a.y = fma(m00.x, u.y, fma(m01.x, v.y, m01.y * v.x));
    b.x = fma(m10.x, u.x, fma(-m10.y, u.y, fma(m11.x, v.x, -m11.y * v.y)));
    b.y = fma(m10.x, u.y, fma(m10.y, u.x, fma(m11.x, v.y, m11.y * v.x)));
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

// Two deterministic block sums in one pass (8 warps at most per block here).
__device__ __forceinline__ double2 block_sum2(double a, double b, double* sred) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, off);
        b += __shfl_xor_sync(0xffffffffu, b, off);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) { sred[2 * warp] = a; sred[2 * warp + 1] = b; }
    __syncthreads();
    double2 t = make_double2(0.0, 0.0);
    const int nw = blockDim.x >> 5;
    for (int w = 0; w < nw; ++w) { t.x += sred[2 * w]; t.y += sred[2 * w + 1]; }
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

template <typename V>
__device__ __forceinline__ double norm2(const V v) {
    return (double)v.x * (double)v.x + (double)v.y * (double)v.y;
}

__host__ __device__ constexpr int pass_threads(int tb) { return tb >= 5 ? (1 << tb) : 32; }

// Ampere-style async global->shared copies (LDGSTS): the next tile streams in
// while the current one is computed.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// TB = tile bits - 4 = log2(active threads).  Work items are (state, tile)
// pairs, state fastest: item w = tile * nstates + state.  Persistent CTA c
// takes items c, c + G, c + 2G, ... (G = grid size = one full wave), so CTAs
// running at the same time touch the same tile of different states -- a
// shared trunk input is then read once from HBM and reused from L2.
//
// MODE 0: single-tile launches (every epilogue, incl. the whole-state F_SINGLE
// ones).  MODE 1 / 2: multi-tile launches -- 1 stores (F_STORE, F_NORM,
// F_SUPPORT) and defers the global stores behind the next tile's load issue,
// 2 is the shift-pair epilogue (F_PAIR).  Separate instantiations keep each
// variant's register footprint to what it uses.  Multi-tile passes that only
// store run on tma_pass_kernel (tma_pass.cuh) when their layout allows; this
// kernel covers the rest (first passes that zero-fill fresh bits, generated
// |0...0> inputs, every reducing epilogue) with the same arithmetic.
template <typename T, int TB, int MODE>
__global__ void __launch_bounds__(pass_threads(TB), TB >= 9 ? 1 : TB == 8 ? (sizeof(T) == 4 ? 3 : 2) : 4)
pass_kernel(const PassDesc pd, const GroupDesc* __restrict__ gdesc, const LaunchEntry* __restrict__ ent,
            int nstates, int unused, EpiArgs ep) {
    typedef typename Cx<T>::V V;
    constexpr bool MT = MODE != 0;
    constexpr bool PAIR = MODE != 1;
    constexpr bool PLAIN = MODE != 2;
    constexpr int NT = 1 << TB;             // active threads (TB < 5: a partial warp)
    constexpr int R = reg_bits(sizeof(T) == 8 ? 0 : 1);   // register bits per group
    constexpr int NA = 1 << R;                           // amplitudes per thread
    constexpr int K = TB + R;
    constexpr size_t TILE = sizeof(V) << K;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GroupDesc* sg = reinterpret_cast<GroupDesc*>(smem_raw + TILE);
    V* smat = reinterpret_cast<V*>(sg + pd.ng);                            // 4 complex per matrix
    double* sred = reinterpret_cast<double*>(smat + (size_t)pd.nm * 4);
    uint64_t* otab = reinterpret_cast<uint64_t*>(sred + 32);   // MT: 4 x 256 outer-offset tables
    (void)unused;

    const int tid = threadIdx.x;
    const int64_t ntiles = ep.ntiles;
    const int items = (int)(ntiles * nstates);   // < 2^31 (host-checked)
    const int G = gridDim.x;
    {   // stage the pass's group descriptors (once per CTA)
        const uint4* gsrc = reinterpret_cast<const uint4*>(gdesc + pd.g0);
        uint4* gdst = reinterpret_cast<uint4*>(sg);
        for (int i = tid; i < pd.ng * 8; i += blockDim.x) gdst[i] = gsrc[i];
    }
    if constexpr (MT) {   // outer offset of tile x = OR of 4 byte-indexed tables (n - k <= 32)
        for (int idx = tid; idx < 1024; idx += blockDim.x) {
            const int b = idx >> 8, v = idx & 255;
            uint64_t o = 0;
            for (int j = 0; j < 8; ++j)
                if (((v >> j) & 1) && 8 * b + j < pd.n_outer) o |= 1ull << pd.obits[8 * b + j];
            otab[idx] = o;
        }
        __syncthreads();
    }
    const bool active = tid < NT;
    // per-thread parts of the load / store maps (tile-independent)
    uint32_t tslot = 0, fslot = 0;
    uint64_t tg = 0;
#pragma unroll
    for (int j = 0; j < TB; ++j)
        if ((tid >> j) & 1) { tslot ^= pd.swz[j]; fslot ^= pd.fin[j]; tg |= 1ull << pd.sbits[j]; }
    auto outer_of = [&](int x) -> uint64_t {
        if constexpr (MT) {
            return otab[x & 255] | otab[256 + ((x >> 8) & 255)] | otab[512 + ((x >> 16) & 255)] |
                   otab[768 + ((x >> 24) & 255)];
        } else {
            uint64_t o = 0;
            for (int j = 0; j < pd.n_outer; ++j)
                if ((x >> j) & 1) o |= 1ull << pd.obits[j];
            return o;
        }
    };
    // item w = x * nstates + y (state fastest); CTA items advance by G = gx * nstates + gy
    const int gx = G / nstates;
    const int gy = (int)(G % nstates);
    auto src_of = [&](int xx, int yy) -> const V* {   // this thread's first source amplitude of an item
        const V* in = reinterpret_cast<const V*>(ent[yy].in);
        return (in == nullptr || !active) ? nullptr : in + (outer_of(xx) | tg);
    };
    auto load_src = [&](int w) -> const V* { return src_of(w / nstates, w % nstates); };
    // slots whose local index has a `fresh` bit hold amplitudes no earlier
    // pass wrote (exactly zero): they are zero-filled instead of loaded
    const bool t_fresh = (tid & pd.fresh) != 0;
    const uint32_t hi_fresh = pd.fresh >> TB;
    auto issue_from = [&](const V* src, unsigned char* dst) {   // NA async 8/16-byte copies per thread
        if (src == nullptr) return;
#pragma unroll
        for (int it = 0; it < NA; ++it) {
            unsigned char* d = dst + (size_t)(tslot ^ pd.swz_hi[it]) * sizeof(V);
            if (t_fresh || (it & hi_fresh)) *reinterpret_cast<V*>(d) = V{T(0), T(0)};
            else cp_async<sizeof(V)>(d, src + pd.g_hi[it]);
        }
    };
    auto issue_load = [&](int w, unsigned char* dst) { issue_from(load_src(w), dst); };
    if (blockIdx.x < items) issue_load(blockIdx.x, smem_raw);
    cp_async_commit();

    int cur_y = -1;
    LaunchEntry e;
    int i = 0;
    int x = (int)blockIdx.x / nstates;
    int y = (int)blockIdx.x % nstates;
    for (int w = blockIdx.x; w < items; w += G, ++i) {
        int xn = x + gx;   // the next item's coordinates
        int yn = y + gy;
        if (yn >= nstates) { yn -= nstates; ++xn; }
        if (y != cur_y) {   // stage this state's matrices (the previous item is finished)
            e = ent[y];
            const V* msrc = reinterpret_cast<const V*>(e.mats) + (size_t)pd.m0 * 4;
            for (int q = tid; q < pd.nm * 4; q += blockDim.x) smat[q] = msrc[q];
            cur_y = y;
        }
        const bool gen = e.in == nullptr;
        V* __restrict__ out = reinterpret_cast<V*>(e.out);
        const bool store = (ep.flags & F_STORE) && out != nullptr;
        unsigned char* tileb = smem_raw;
        const uint64_t outer = outer_of(x);
        const bool zero_tile = gen && x != 0;
        // ---- load (or generate |0...0>) ------------------------------------
        if (gen) {
            if (active) {
#pragma unroll
                for (int it = 0; it < NA; ++it) {
                    V v;
                    v.x = (x == 0 && tid == 0 && it == 0) ? T(1) : T(0);
                    v.y = T(0);
                    *reinterpret_cast<V*>(tileb + ((size_t)(tslot ^ pd.swz_hi[it]) * sizeof(V))) = v;
                }
            }
        }
        cp_async_wait<0>();   // this item's tile has landed (issued by the previous item)
        __syncthreads();
        const V* next_src = (w + G < items) ? src_of(xn, yn) : nullptr;
        // ---- register groups --------------------------------------------------
        if (!zero_tile) {
            // the tile buffer's byte offset (a multiple of 2^16 > every slot
            // offset) is folded into the XOR base: one address op per amplitude
            const uint32_t boff = (uint32_t)(tileb - smem_raw);
            for (int g = 0; g < pd.ng; ++g) {
                if (active) {
                    const GroupDesc& G = sg[g];
                    const int4 mats = *reinterpret_cast<const int4*>(G.mat);
                    // first matrix in flight before the amplitudes
                    V m00, m01, m10, m11;
                    if (mats.x >= 0) {
                        const V* M = smat + mats.x * 4;
                        m00 = M[0]; m01 = M[1]; m10 = M[2]; m11 = M[3];
                    }
                    uint32_t base = boff;
#pragma unroll
                    for (int m = 0; m < TB; ++m)
                        if ((tid >> m) & 1) base ^= G.tcol[m];
                    uint32_t off[NA];
#pragma unroll
                    for (int q = 0; q < NA / 4; ++q) {
                        const uint4 c = reinterpret_cast<const uint4*>(G.combo)[q];
                        off[4 * q] = base ^ c.x;
                        off[4 * q + 1] = base ^ c.y;
                        off[4 * q + 2] = base ^ c.z;
                        off[4 * q + 3] = base ^ c.w;
                    }
                    V a[NA];
#pragma unroll
                    for (int j = 0; j < NA; ++j) a[j] = *reinterpret_cast<const V*>(smem_raw + off[j]);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int mi = r == 0 ? mats.x : r == 1 ? mats.y : r == 2 ? mats.z : mats.w;
                        if (mi >= 0) {
                            if (r > 0) {
                                const V* M = smat + mi * 4;
                                m00 = M[0]; m01 = M[1]; m10 = M[2]; m11 = M[3];
                            }
#pragma unroll
                            for (int j = 0; j < NA; ++j)
                                if (!((j >> r) & 1)) rot2<V>(m00, m01, m10, m11, a[j], a[j | (1 << r)]);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < NA; ++j) *reinterpret_cast<V*>(smem_raw + off[j]) = a[j];
                }
                // warp-local segment: the next group reads only what this warp wrote
                if (g + 1 < pd.ng && !sg[g + 1].cta_sync) __syncwarp();
                else __syncthreads();
            }
        }
        // ---- store / reduce ----------------------------------------------------
        // Every shared-memory read of this tile (the thread's own amplitudes
        // into `vals`, support / Pauli / pair epilogues) happens before the
        // closing barrier; the next item's load is then issued before this
        // item's global stores, so its latency overlaps the store phase.
        double acc = 0.0;
        V vals[NA];
        if (ep.flags & F_SUPPORT) {
            const int32_t lo = ep.sup_off[x], hi = ep.sup_off[x + 1];
            double* row = ep.sup_out + e.rslot * (ep.S + 1);
            for (int32_t i = lo + tid; i < hi; i += blockDim.x) {
                const uint32_t slot = apply_cols(pd.fin, K, (uint32_t)ep.sup_local[i]);
                row[ep.sup_pos[i]] = norm2(*reinterpret_cast<const V*>(tileb + (size_t)slot * sizeof(V)));
            }
        }
        if (MT && PLAIN && (ep.flags & F_MT_PAULI)) {
            // Pauli terms of this state whose flip bits lie in this pass's
            // tile: sum_i conj(a[i ^ F]) a[i] (-1)^{|i & PH|} over the tile's
            // amplitudes (reference kernels.py:73-87), read-only: every term
            // of the sweep from one pass over the state
            const int64_t t0 = ep.term_off[e.rslot], t1 = ep.term_off[e.rslot + 1];
            for (int64_t t = t0; t < t1; ++t) {
                if (ep.t_sweep[t] != ep.sweep) continue;   // uniform across the block
                const uint32_t fF = ep.t_fslot[t], PHl = ep.t_phloc[t];
                double ar = 0.0, ai = 0.0;
                if (active) {
#pragma unroll
                    for (int it = 0; it < NA; ++it) {
                        const uint32_t l = (uint32_t)tid | ((uint32_t)it << TB);
                        const uint32_t sl = fslot ^ pd.fin_hi[it];
                        const V a = *reinterpret_cast<const V*>(tileb + (size_t)sl * sizeof(V));
                        const V b = *reinterpret_cast<const V*>(tileb + (size_t)(sl ^ fF) * sizeof(V));
                        const double tr = (double)b.x * (double)a.x + (double)b.y * (double)a.y;
                        const double ti = (double)b.x * (double)a.y - (double)b.y * (double)a.x;
                        if (__popc(l & PHl) & 1) { ar -= tr; ai -= ti; }
                        else { ar += tr; ai += ti; }
                    }
                }
                const double2 sum = block_sum2(ar, ai, sred);
                if (tid == 0) {
                    const double sg = (__popcll(outer & ep.t_phout[t]) & 1) ? -1.0 : 1.0;
                    ep.pauli_partial[t * ntiles + x] = make_double2(sg * sum.x, sg * sum.y);
                }
            }
        }
        if (PAIR && (ep.flags & F_PAIR)) {
            // shift pair: this tile holds Xi, `aux` the unshifted output Psi0.
            // Per tile: sum |Psi0|^2, sum |Xi|^2, sum Im(Psi0 conj(Xi)); per
            // support index the same three terms (finalize_pair_kernel forms
            // p(t +- pi/2) = |Psi0 -+ i Xi|^2 / 2 from them).
            const V* __restrict__ aux = reinterpret_cast<const V*>(e.aux);
            double accB = 0.0, accC = 0.0, accD = 0.0;
            if (active) {
                const V* __restrict__ src = aux + (outer | tg);
#pragma unroll
                for (int it = 0; it < NA; ++it) {
                    const V v = *reinterpret_cast<const V*>(tileb + (size_t)(fslot ^ pd.fin_hi[it]) * sizeof(V));
                    const V u = __ldcs(src + pd.g_hi[it]);
                    acc += norm2(u);
                    accB += norm2(v);
                    accC += (double)u.y * (double)v.x - (double)u.x * (double)v.y;   // Im(u conj v)
                    accD += (double)u.x * (double)v.x + (double)u.y * (double)v.y;   // Re(u conj v)
                }
            }
            const double A = block_sum(acc, sred);
            const double B = block_sum(accB, sred);
            const double C = block_sum(accC, sred);
            const double D = block_sum(accD, sred);
            if (tid == 0) {
                double* p = ep.partial + (e.pslot * ntiles + x) * 4;
                p[0] = A;
                p[1] = B;
                p[2] = C;
                p[3] = D;
            }
            const int32_t lo = ep.sup_off[x], hi = ep.sup_off[x + 1];
            for (int32_t q = lo + tid; q < hi; q += blockDim.x) {
                const uint32_t loc = (uint32_t)ep.sup_local[q];
                const V v = *reinterpret_cast<const V*>(tileb + (size_t)apply_cols(pd.fin, K, loc) * sizeof(V));
                uint64_t gidx = outer;
                for (int j = 0; j < K; ++j)
                    if ((loc >> j) & 1u) gidx |= 1ull << pd.sbits[j];
                const V u = aux[gidx];
                double* row = ep.pair_sup + (e.rslot * ep.S + ep.sup_pos[q]) * 4;
                row[0] = norm2(u);
                row[1] = norm2(v);
                row[2] = (double)u.y * (double)v.x - (double)u.x * (double)v.y;
                row[3] = (double)u.x * (double)v.x + (double)u.y * (double)v.y;
            }
        } else if (PLAIN && active) {
#pragma unroll
            for (int it = 0; it < NA; ++it) {
                vals[it] = *reinterpret_cast<const V*>(tileb + (size_t)(fslot ^ pd.fin_hi[it]) * sizeof(V));
                acc += norm2(vals[it]);
            }
            if constexpr (!MT) {
                if (store) {
                    V* __restrict__ dst = out + (outer | tg);
#pragma unroll
                    for (int it = 0; it < NA; ++it) __stcs(dst + pd.g_hi[it], vals[it]);
                }
            }
        }
        if (!MT && (ep.flags & F_NORM)) {
            const double s = block_sum(acc, sred);
            if (tid == 0) ep.partial[e.pslot * ntiles + x] = s;
        }
        if (!MT && (ep.flags & F_SINGLE)) {
            // the tile is the whole state (ntiles == 1)
            const double total = block_sum(acc, sred);
            const int64_t dim = 1ll << ep.n;
            if ((ep.flags & F_S_FULL) && active) {
                double* row = ep.full_out + (e.rslot << ep.n);
#pragma unroll
                for (int it = 0; it < NA; ++it) {
                    const uint32_t i = (uint32_t)tid | ((uint32_t)it << TB);
                    if (i < dim)
                        row[i] = norm2(*reinterpret_cast<const V*>(tileb + (size_t)(fslot ^ pd.fin_hi[it]) * sizeof(V))) / total;
                }
            }
            if (ep.flags & (F_S_SUPPORT | F_S_JS)) {
                double* row = (ep.flags & F_S_SUPPORT) ? ep.sup_out + e.rslot * (ep.S + 1) : nullptr;
                double jsum = 0.0, qsum = 0.0;
                for (int64_t s = tid; s < ep.S; s += blockDim.x) {
                    const uint64_t idx = ep.support[s];
                    double q = 0.0;
                    if (idx < (uint64_t)dim)
                        q = norm2(*reinterpret_cast<const V*>(tileb + (size_t)apply_cols(pd.fin, K, (uint32_t)idx) * sizeof(V))) / total;
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
                    const uint32_t fF = apply_cols(pd.fin, K, (uint32_t)F);
                    double ar = 0.0, ai = 0.0;
                    if (active) {
#pragma unroll
                        for (int it = 0; it < NA; ++it) {
                            const uint32_t i = (uint32_t)tid | ((uint32_t)it << TB);
                            const uint32_t sl = fslot ^ pd.fin_hi[it];
                            const V a = *reinterpret_cast<const V*>(tileb + (size_t)sl * sizeof(V));
                            const V b = *reinterpret_cast<const V*>(tileb + (size_t)(sl ^ fF) * sizeof(V));
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
                        const int ny = __popcll(F & PH) & 3;   // Y factors both flip and carry phase
                        ep.pauli_out[t] = ny == 0 ? R : ny == 1 ? -I : ny == 2 ? -R : I;
                    }
                }
            }
        }
        if (MT && PLAIN && store && active && !(ep.flags & F_PAIR)) {   // first half before the barrier
            V* __restrict__ dst = out + (outer | tg);
#pragma unroll
            for (int it = 0; it < NA / 2; ++it) __stcs(dst + pd.g_hi[it], vals[it]);
        }
        __syncthreads();   // the next tile overwrites the shared tile
        issue_from(next_src, smem_raw);
        cp_async_commit();
        if (MT && PLAIN && store && active && !(ep.flags & F_PAIR)) {
            V* __restrict__ dst = out + (outer | tg);
#pragma unroll
            for (int it = NA / 2; it < NA; ++it) __stcs(dst + pd.g_hi[it], vals[it]);
        }
        if (MT && (ep.flags & F_NORM)) {   // sred is outside the tile: safe beside the next load
            const double s = block_sum(acc, sred);
            if (tid == 0) ep.partial[e.pslot * ntiles + x] = s;
        }
        x = xn;
        y = yn;
    }
}

// Multi-tile norm / support finalisation: one CTA per result slot.
// slots[2*b] = result slot, slots[2*b+1] = partial slot.
__global__ void finalize_dist_kernel(const int64_t* __restrict__ slots, int64_t ntiles, const double* __restrict__ partial,
                                     double* __restrict__ sup_out, int64_t S, const double* __restrict__ target,
                                     double* __restrict__ js_out, int want_js, int unit_norm) {
    __shared__ double sred[32];
    const int64_t r = slots[2 * blockIdx.x], ps = slots[2 * blockIdx.x + 1];
    double acc = 0.0;
    if (!unit_norm)
        for (int64_t i = threadIdx.x; i < ntiles; i += blockDim.x) acc += partial[ps * ntiles + i];
    // light-cone runs do not sweep the norm: a unitary circuit keeps it at 1
    const double total = unit_norm ? 1.0 : block_sum(acc, sred);
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

// Per-circuit targets (QV_RES_TARGET_ROWS): one CTA per circuit, its unique
// state's normalised support row against its own target row, summed in the
// order finalize_dist_kernel uses (the same loss for equal targets).
__global__ void js_rows_kernel(const double* __restrict__ sup_out, const int64_t* __restrict__ urow,
                               const double* __restrict__ trows, int64_t S, double* __restrict__ js) {
    __shared__ double sred[32];
    const double* row = sup_out + urow[blockIdx.x] * (S + 1);
    const double* t = trows + (int64_t)blockIdx.x * S;
    double jsum = 0.0, qsum = 0.0;
    for (int64_t s = threadIdx.x; s < S; s += blockDim.x) {
        const double q = row[s];
        jsum += js_term(t[s], q);
        qsum += q;
    }
    const double J = block_sum(jsum, sred);
    const double Q = block_sum(qsum, sred);
    if (threadIdx.x == 0) js[blockIdx.x] = J + 0.5 * 0.69314718055994530942 * (1.0 - Q);
}

// Shift-pair finalisation: one CTA per shifted gate.  With A = sum|Psi0|^2,
// B = sum|Xi|^2, C = sum Im(Psi0 conj Xi), the two shifted distributions are
// q+-(s) = (a_s + b_s -+ 2 c_s) / (A + B -+ 2 C)  (psi+- = (Psi0 -+ i Xi)/sqrt2),
// and each JS loss is formed with the support + remainder identity.
// slots[2*b] = result slot, slots[2*b+1] = partial slot; out[2r], out[2r+1].
__global__ void finalize_pair_kernel(const int64_t* __restrict__ slots, int64_t ntiles, const double* __restrict__ partial,
                                     const double* __restrict__ pair_sup, int64_t S, const double* __restrict__ target,
                                     double* __restrict__ out, int unit_norm, const double* __restrict__ delta) {
    __shared__ double sred[32];
    const int64_t r = slots[2 * blockIdx.x], ps = slots[2 * blockIdx.x + 1];
    // the device Xi carries an extra global phase e^{i delta_r} relative to
    // Psi0 (per-matrix phase normalisation): Psi0 conj(Xi_true) = z e^{-i delta}
    // for the computed z, so Im(Psi0 conj Xi_true) = Im z cos delta - Re z sin delta
    const double cd = cos(delta[r]), sd = sin(delta[r]);
    double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
    for (int64_t i = threadIdx.x; i < ntiles; i += blockDim.x) {
        const double* p = partial + (ps * ntiles + i) * 4;
        a += p[0];
        b += p[1];
        c += p[2];
        d += p[3];
    }
    double A = block_sum(a, sred), B = block_sum(b, sred);
    double C = block_sum(c, sred) * cd - block_sum(d, sred) * sd;
    if (unit_norm) {   // light-cone run: |Psi0| = |Xi| = 1 and Im<Psi0|Xi> = 0 exactly
        A = 1.0;
        B = 1.0;
        C = 0.0;
    }
    const double tp = A + B - 2.0 * C, tm = A + B + 2.0 * C;
    double jp = 0.0, jm = 0.0, sp = 0.0, sm = 0.0;
    for (int64_t s = threadIdx.x; s < S; s += blockDim.x) {
        const double* q = pair_sup + (r * S + s) * 4;
        const double im = q[2] * cd - q[3] * sd;
        const double qp = (q[0] + q[1] - 2.0 * im) / tp;
        const double qm = (q[0] + q[1] + 2.0 * im) / tm;
        jp += js_term(target[s], qp);
        jm += js_term(target[s], qm);
        sp += qp;
        sm += qm;
    }
    const double JP = block_sum(jp, sred), JM = block_sum(jm, sred);
    const double SP = block_sum(sp, sred), SM = block_sum(sm, sred);
    if (threadIdx.x == 0) {
        out[2 * r] = JP + 0.5 * 0.69314718055994530942 * (1.0 - SP);
        out[2 * r + 1] = JM + 0.5 * 0.69314718055994530942 * (1.0 - SM);
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
            const double p = norm2(st[j]);
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
            // term(i) = conj(b) a s(i); term(i2) = conj(a) b s(i2) = conj(term(i)) s(i) s(i2)
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
        const int q = ny & 3;
        *out = q == 0 ? R : q == 1 ? -I : q == 2 ? -R : I;
    }
}

// F_MT_PAULI finalisation: one CTA per term; fixed-order tree over the
// per-tile partials, then the i^ny factor (kernels.py:87).
__global__ void finalize_pauli_mt_kernel(const int64_t* __restrict__ terms, int64_t ntiles,
                                         const double2* __restrict__ partial, const uint64_t* __restrict__ flip,
                                         const uint64_t* __restrict__ phase, double* __restrict__ out) {
    __shared__ double sred[32];
    const int64_t t = terms[blockIdx.x];
    double ar = 0.0, ai = 0.0;
    for (int64_t i = threadIdx.x; i < ntiles; i += blockDim.x) {
        const double2 p = partial[t * ntiles + i];
        ar += p.x;
        ai += p.y;
    }
    const double R = block_sum(ar, sred);
    const double I = block_sum(ai, sred);
    if (threadIdx.x == 0) {
        const int ny = __popcll(flip[t] & phase[t]) & 3;   // Y factors both flip and carry phase
        out[t] = ny == 0 ? R : ny == 1 ? -I : ny == 2 ? -R : I;
    }
}

// Multi-tile full distribution: p_i / total for a stored state.
template <typename T>
__global__ void full_probs_kernel(const typename Cx<T>::V* __restrict__ st, int64_t dim, const double* __restrict__ total,
                                  double* __restrict__ out) {
    const double t = *total;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = norm2(st[i]) / t;
}

}  // namespace qvb
