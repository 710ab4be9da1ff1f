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
    double* pair_sup;          // F_PAIR: [(rslot * S + pos) * 3 + {|Psi0|^2, |Xi|^2, Im(Psi0 conj Xi)}]
    long long* trace;          // QV_TRACE builds only: per-phase clock64() of CTA 0
};

#ifdef QV_TRACE
// trace[(item * 64 + event) * 16 + warp]: event 0 item start, 1 tile resident,
// 2 + 2g group g math done, 3 + 2g group g synchronised, 62 store done
// CTA 0 records warps 0..7 and, for 256-thread CTAs, CTA gridDim/2 (usually
// its partner on the same SM) records into warp slots 8..15; event 63 = %smid
#define QV_MARK(ev)                                                                                \
    do {                                                                                           \
        const int qv_slot = (blockIdx.x == 0) ? (int)(threadIdx.x >> 5)                            \
                            : (blockIdx.x == gridDim.x / 2 && blockDim.x <= 256) ? 8 + (int)(threadIdx.x >> 5) : -1; \
        if (ep.trace && qv_slot >= 0 && (threadIdx.x & 31) == 0 && i < 8 && qv_slot < 16) {       \
            long long qv_t;                                                                        \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(qv_t));                              \
            ep.trace[((i) * 64 + (ev)) * 16 + qv_slot] = qv_t;                                     \
            unsigned qv_sm;                                                                        \
            asm volatile("mov.u32 %0, %%smid;" : "=r"(qv_sm));                                     \
            ep.trace[((i) * 64 + 63) * 16 + qv_slot] = qv_sm;                                      \
        }                                                                                          \
    } while (0)
#else
#define QV_MARK(ev) \
    do {            \
    } while (0)
#endif

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
// DB (double buffer): two tile buffers; the next item's tile streams in with
// cp.async while the current one is computed and written back, so HBM, the
// shared-memory pipe and the FP64 pipe work concurrently inside one CTA.
//
// MODE 0: single-tile launches (every epilogue, incl. the whole-state F_SINGLE
// ones).  MODE 1 / 2: multi-tile launches -- 1 stores (F_STORE, F_NORM,
// F_SUPPORT) and defers the global stores behind the next tile's load issue,
// 2 is the shift-pair epilogue (F_PAIR).  Separate instantiations keep each
// variant's register footprint to what it uses.
#ifndef QV_L2_PREFETCH
#define QV_L2_PREFETCH 0
#endif
// diagnostic builds only (timing breakdowns; results are wrong)
#ifndef QV_RING_SLEEP_NS
#define QV_RING_SLEEP_NS 200
#endif
#ifndef QV_RING_TOKEN
#define QV_RING_TOKEN 1
#endif
#ifndef QV_DIAG_NO_MATH
#define QV_DIAG_NO_MATH 0
#endif
#ifndef QV_DIAG_NO_GROUPS
#define QV_DIAG_NO_GROUPS 0
#endif
template <typename T, int TB, bool DB, int MODE>
#ifndef QV_TB9_MIN_BLOCKS
#define QV_TB9_MIN_BLOCKS 1
#endif
#ifndef QV_C128_TB8_MIN_BLOCKS
#define QV_C128_TB8_MIN_BLOCKS 2   // complex128 at 12 tile bits: two CTAs per SM (128 registers)
#endif
#ifndef QV_C64_TB8_MIN_BLOCKS
#define QV_C64_TB8_MIN_BLOCKS 3   // complex64 at 12 tile bits: three CTAs per SM (<= 85 registers)
#endif
__global__ void __launch_bounds__(pass_threads(TB), (DB ? (sizeof(T) == 4 && TB == 8 ? QV_C64_TB8_MIN_BLOCKS : 1)
                                                     : TB >= 9 ? QV_TB9_MIN_BLOCKS
                                                     : TB == 8 ? (sizeof(T) == 4 ? QV_C64_TB8_MIN_BLOCKS : QV_C128_TB8_MIN_BLOCKS) : 4))
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
    GroupDesc* sg = reinterpret_cast<GroupDesc*>(smem_raw + TILE * (DB ? 2 : 1));
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
        QV_MARK(0);
        if (y != cur_y) {   // stage this state's matrices (the previous item is finished)
            e = ent[y];
            const V* msrc = reinterpret_cast<const V*>(e.mats) + (size_t)pd.m0 * 4;
            for (int q = tid; q < pd.nm * 4; q += blockDim.x) smat[q] = msrc[q];
            cur_y = y;
        }
        const bool gen = e.in == nullptr;
        V* __restrict__ out = reinterpret_cast<V*>(e.out);
        const bool store = (ep.flags & F_STORE) && out != nullptr;
        unsigned char* tileb = smem_raw + ((DB && (i & 1)) ? TILE : 0);
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
        QV_MARK(1);
        // the next item's source; optionally (QV_L2_PREFETCH) an L2 prefetch of
        // its tile, one thread per 128-byte row, so its cp.async at the end of
        // this item would hit L2.  Measured on B200: 2-state launches 7 % faster,
        // full gradients (38 states per launch) 3 % slower -- off by default.
        const V* next_src = (!DB && w + G < items) ? src_of(xn, yn) : nullptr;
        if constexpr (MT && QV_L2_PREFETCH) {
            constexpr int ROW = 128 / sizeof(V);
            if (next_src != nullptr && (tid & (ROW - 1)) == 0) {
#pragma unroll
                for (int it = 0; it < NA; ++it) {
#if QV_L2_PREFETCH == 2   // bulk form: the TMA unit moves the 128-byte row into L2
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;\n" ::"l"(next_src + pd.g_hi[it])
                                 : "memory");
#else
                    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(next_src + pd.g_hi[it]));
#endif
                }
            }
        }
        if (DB && w + G < items) {   // stream the next item's tile in behind this one's math
            issue_from(src_of(xn, yn), smem_raw + ((i & 1) ? 0 : TILE));
            cp_async_commit();
        }
        // ---- register groups --------------------------------------------------
        if (!zero_tile && !QV_DIAG_NO_GROUPS) {
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
                    for (int r = 0; r < (QV_DIAG_NO_MATH ? 0 : R); ++r) {   // diagnostic builds skip the math
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
                    if (g < 29) QV_MARK(2 + 2 * g);
#pragma unroll
                    for (int j = 0; j < NA; ++j) *reinterpret_cast<V*>(smem_raw + off[j]) = a[j];
                }
                // warp-local segment: the next group reads only what this warp wrote
                if (g + 1 < pd.ng && !sg[g + 1].cta_sync) __syncwarp();
                else __syncthreads();
                if (g < 29) QV_MARK(3 + 2 * g);
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
        QV_MARK(62);
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
        if (!DB) {
            issue_from(next_src, smem_raw);
            cp_async_commit();
        }
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

// ---------------------------------------------------------------------------
// Ring pass kernel (multi-tile, complex128): one 512-thread CTA per SM made of
// two 256-thread teams that share a ring of three tile buffers.  Item i of the
// CTA (items c, c + G, c + 2G, ...) belongs to team i mod 2 and lives in buffer
// i mod 3; the team that finishes item i issues the cp.async load of item i + 3
// into the buffer it just drained, and an mbarrier per buffer (256 arrivals,
// cp.async.mbarrier.arrive.noinc) tells the other team when it has landed.
// Each team therefore finds its next tile resident when it gets there, while
// the two teams' compute and store phases interleave on the SM -- the load
// latency the two-CTA layout exposes is hidden without a fourth buffer.
// Within a team the register-group code and every reduction order are those
// of pass_kernel (team-local named barriers instead of __syncthreads), so the
// results are bitwise identical.
__device__ __forceinline__ void team_sync(int team) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + team), "r"(256) : "memory");
}
__device__ __forceinline__ double team_sum(double v, double* sred, int team, int t) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    team_sync(team);
    if ((t & 31) == 0) sred[t >> 5] = v;
    team_sync(team);
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += sred[w];
    return s;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
// arrives once this thread's earlier cp.async copies have landed
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n"
                 ::"r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
// waits that may last a whole compute phase back off with __nanosleep so
// the spinning warps leave the issue slots to the computing team
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (true) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
        if (done) break;
        __nanosleep(QV_RING_SLEEP_NS);
    }
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

template <typename T, int MODE>   // MODE 1: store (F_STORE / F_NORM / F_SUPPORT), 2: shift pair (F_PAIR)
__global__ void __launch_bounds__(512, 1)
ring_pass_kernel(const PassDesc pd, const GroupDesc* __restrict__ gdesc, const LaunchEntry* __restrict__ ent,
                 int nstates, int unused, EpiArgs ep) {
    typedef typename Cx<T>::V V;
    constexpr int R = reg_bits(sizeof(T) == 8 ? 0 : 1);
    constexpr int NA = 1 << R;
    constexpr int TB = 8;                       // 256 threads per team
    constexpr int K = TB + R;
    constexpr size_t TILE = sizeof(V) << K;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + 3 * TILE);              // 3 mbarriers
    uint64_t* tok = full + 3;                                                         // 2 compute tokens
    double* sred_all = reinterpret_cast<double*>(full + 6);                          // 2 x 8
    uint64_t* otab = reinterpret_cast<uint64_t*>(sred_all + 16);                     // 4 x 256 outer offsets
    LaunchEntry* steam = reinterpret_cast<LaunchEntry*>(otab + 1024);                // per-team item entry
    GroupDesc* sg = reinterpret_cast<GroupDesc*>(steam + 2);
    V* smat_all = reinterpret_cast<V*>(sg + pd.ng);                                  // 2 x nm x 4
    (void)unused;

    const int team = threadIdx.x >> 8;
    const int t = threadIdx.x & 255;
    double* sred = sred_all + 8 * team;
    V* smat = smat_all + (size_t)team * pd.nm * 4;
    const int64_t ntiles = ep.ntiles;
    const int items = (int)(ntiles * nstates);   // < 2^31 (host-checked)
    const int G = gridDim.x;
    const int c = blockIdx.x;
    {
        const uint4* gsrc = reinterpret_cast<const uint4*>(gdesc + pd.g0);
        uint4* gdst = reinterpret_cast<uint4*>(sg);
        for (int i = threadIdx.x; i < pd.ng * 8; i += blockDim.x) gdst[i] = gsrc[i];
        if (threadIdx.x < 5) mbar_init(full + threadIdx.x, 256);   // full[0..2], tok[0..1]
        for (int idx = threadIdx.x; idx < 1024; idx += blockDim.x) {
            const int b = idx >> 8, v = idx & 255;
            uint64_t o = 0;
            for (int j = 0; j < 8; ++j)
                if (((v >> j) & 1) && 8 * b + j < pd.n_outer) o |= 1ull << pd.obits[8 * b + j];
            otab[idx] = o;
        }
    }
    __syncthreads();
    uint32_t tslot = 0, fslot = 0;
    uint64_t tg = 0;
#pragma unroll
    for (int j = 0; j < TB; ++j)
        if ((t >> j) & 1) { tslot ^= pd.swz[j]; fslot ^= pd.fin[j]; tg |= 1ull << pd.sbits[j]; }
    auto outer_of = [&](int x) -> uint64_t {
        return otab[x & 255] | otab[256 + ((x >> 8) & 255)] | otab[512 + ((x >> 16) & 255)] |
               otab[768 + ((x >> 24) & 255)];
    };
    auto src_of = [&](int xx, int yy) -> const V* {
        const V* in = reinterpret_cast<const V*>(ent[yy].in);
        return in == nullptr ? nullptr : in + (outer_of(xx) | tg);
    };
    auto load_src = [&](int w) -> const V* { return src_of(w / nstates, w % nstates); };
    // item coordinates advance by multiples of G: (x, y) += (kG / nstates, kG % nstates) with carry
    const int g2x = 2 * G / nstates, g3x = 3 * G / nstates;
    const int g2y = 2 * G % nstates, g3y = 3 * G % nstates;
    // this thread's share of item i's tile -> buffer i % 3, then one arrival
    const bool t_fresh = (t & pd.fresh) != 0;   // zero-filled slots (see pass_kernel)
    const uint32_t hi_fresh = pd.fresh >> TB;
    auto load_item = [&](const V* src, int i) {
        unsigned char* dst = smem_raw + (size_t)(i % 3) * TILE;
        if (src != nullptr) {
#pragma unroll
            for (int it = 0; it < NA; ++it) {
                unsigned char* d = dst + (size_t)(tslot ^ pd.swz_hi[it]) * sizeof(V);
                if (t_fresh || (it & hi_fresh)) *reinterpret_cast<V*>(d) = V{T(0), T(0)};
                else cp_async<sizeof(V)>(d, src + pd.g_hi[it]);
            }
        }
        mbar_arrive_cp_async(full + i % 3);
    };
    // prologue: item i's load is issued by team (i + 1) mod 2 (the team of item i - 3)
    for (int i = 0; i < 3; ++i)
        if (c + i * G < items && ((i + 1) & 1) == team) load_item(load_src(c + i * G), i);

    // The item's LaunchEntry is uniform across a team: it lives in shared
    // memory (steam[team]) rather than in every thread's registers, which
    // keeps the register-group loop free of spills.
    int cur_y = -1;
    int x = (c + team * G) / nstates;
    int y = (c + team * G) % nstates;
    for (int i = team; c + i * G < items; i += 2) {
        QV_MARK(0);
        unsigned char* tileb = smem_raw + (size_t)(i % 3) * TILE;
        if (y != cur_y) {
            const V* msrc = reinterpret_cast<const V*>(ent[y].mats) + (size_t)pd.m0 * 4;
            for (int q = t; q < pd.nm * 4; q += 256) smat[q] = msrc[q];
            if (t == 0) steam[team] = ent[y];
            cur_y = y;
        }
        const bool gen = ent[y].in == nullptr;
        const bool zero_tile = gen && x != 0;
        mbar_wait(full + i % 3, (unsigned)((i / 3) & 1));   // this item's tile has landed
        if (gen) {
#pragma unroll
            for (int it = 0; it < NA; ++it) {
                V v;
                v.x = (x == 0 && t == 0 && it == 0) ? T(1) : T(0);
                v.y = T(0);
                *reinterpret_cast<V*>(tileb + ((size_t)(tslot ^ pd.swz_hi[it]) * sizeof(V))) = v;
            }
        }
        team_sync(team);
        QV_MARK(1);
        // Compute token (QV_RING_TOKEN): the teams' register-group phases
        // alternate A0 B0 A1 B1 ..., so one team computes while the other
        // stores and its next tile streams in (without it the two teams -- like
        // every CTA of a plain launch -- fall into lock-step: all compute, then
        // all stream).  tok[tau] completes when the other team's previous
        // compute phase ends.
        const int m_item = i >> 1;   // this team's item counter
        if (QV_RING_TOKEN) {
            if (team == 0 && m_item >= 1) mbar_wait_sleep(tok + 0, (unsigned)((m_item - 1) & 1));
            if (team == 1) mbar_wait_sleep(tok + 1, (unsigned)(m_item & 1));
        }
        // ---- register groups (as pass_kernel) --------------------------------
        if (!zero_tile) {
            const uint32_t boff = (uint32_t)(tileb - smem_raw);
            for (int g = 0; g < pd.ng; ++g) {
                const GroupDesc& GD = sg[g];
                const int4 mats = *reinterpret_cast<const int4*>(GD.mat);
                V m00, m01, m10, m11;
                if (mats.x >= 0) {
                    const V* M = smat + mats.x * 4;
                    m00 = M[0]; m01 = M[1]; m10 = M[2]; m11 = M[3];
                }
                uint32_t base = boff;
#pragma unroll
                for (int m = 0; m < TB; ++m)
                    if ((t >> m) & 1) base ^= GD.tcol[m];
                uint32_t off[NA];
#pragma unroll
                for (int q = 0; q < NA / 4; ++q) {
                    const uint4 cc = reinterpret_cast<const uint4*>(GD.combo)[q];
                    off[4 * q] = base ^ cc.x;
                    off[4 * q + 1] = base ^ cc.y;
                    off[4 * q + 2] = base ^ cc.z;
                    off[4 * q + 3] = base ^ cc.w;
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
                if (g < 29) QV_MARK(2 + 2 * g);
#pragma unroll
                for (int j = 0; j < NA; ++j) *reinterpret_cast<V*>(smem_raw + off[j]) = a[j];
                if (g + 1 < pd.ng && !sg[g + 1].cta_sync) __syncwarp();
                else team_sync(team);
                if (g < 29) QV_MARK(3 + 2 * g);
            }
        }
        if (QV_RING_TOKEN) mbar_arrive(tok + (1 - team));   // hand the FP64 pipe to the other team
        // ---- store / reduce: every shared-memory read before the team barrier
        int x3 = x + g3x;   // item i + 3 (loaded by this team for the other one)
        int y3 = y + g3y;
        if (y3 >= nstates) { y3 -= nstates; ++x3; }
        const V* next_src = (c + (i + 3) * G < items) ? src_of(x3, y3) : nullptr;
        const LaunchEntry& e = steam[team];   // read before the closing team barrier only
        const uint64_t outer = outer_of(x);
        V* __restrict__ out = reinterpret_cast<V*>(e.out);
        const bool store = (ep.flags & F_STORE) && out != nullptr;
        const int64_t pslot = e.pslot;
        double acc = 0.0;
        V vals[NA];
        if (MODE == 1 && (ep.flags & F_SUPPORT)) {
            const int32_t lo = ep.sup_off[x], hi = ep.sup_off[x + 1];
            double* row = ep.sup_out + e.rslot * (ep.S + 1);
            for (int32_t q = lo + t; q < hi; q += 256) {
                const uint32_t slot = apply_cols(pd.fin, K, (uint32_t)ep.sup_local[q]);
                row[ep.sup_pos[q]] = norm2(*reinterpret_cast<const V*>(tileb + (size_t)slot * sizeof(V)));
            }
        }
        if (MODE == 2) {
            const V* __restrict__ aux = reinterpret_cast<const V*>(e.aux);
            double accB = 0.0, accC = 0.0, accD = 0.0;
            const V* __restrict__ src = aux + (outer | tg);
#pragma unroll
            for (int it = 0; it < NA; ++it) {
                const V v = *reinterpret_cast<const V*>(tileb + (size_t)(fslot ^ pd.fin_hi[it]) * sizeof(V));
                const V u = __ldcs(src + pd.g_hi[it]);
                acc += norm2(u);
                accB += norm2(v);
                accC += (double)u.y * (double)v.x - (double)u.x * (double)v.y;
                accD += (double)u.x * (double)v.x + (double)u.y * (double)v.y;
            }
            const double A = team_sum(acc, sred, team, t);
            const double B = team_sum(accB, sred, team, t);
            const double C = team_sum(accC, sred, team, t);
            const double D = team_sum(accD, sred, team, t);
            if (t == 0) {
                double* p = ep.partial + (pslot * ntiles + x) * 4;
                p[0] = A;
                p[1] = B;
                p[2] = C;
                p[3] = D;
            }
            const int32_t lo = ep.sup_off[x], hi = ep.sup_off[x + 1];
            for (int32_t q = lo + t; q < hi; q += 256) {
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
        } else {
#pragma unroll
            for (int it = 0; it < NA; ++it) {
                vals[it] = *reinterpret_cast<const V*>(tileb + (size_t)(fslot ^ pd.fin_hi[it]) * sizeof(V));
                acc += norm2(vals[it]);
            }
        }
        QV_MARK(62);
        team_sync(team);   // the buffer is drained: item i + 3 streams into it
        if (c + (i + 3) * G < items) load_item(next_src, i + 3);
        if (MODE == 1 && store) {
            V* __restrict__ dst = out + (outer | tg);
#pragma unroll
            for (int it = 0; it < NA; ++it) __stcs(dst + pd.g_hi[it], vals[it]);
        }
        if (MODE == 1 && (ep.flags & F_NORM)) {
            const double s = team_sum(acc, sred, team, t);
            if (t == 0) ep.partial[pslot * ntiles + x] = s;
        }
        x += g2x;   // this team's next item, i + 2
        y += g2y;
        if (y >= nstates) { y -= nstates; ++x; }
    }
    cp_async_wait<0>();   // loads issued for the other team complete before this thread exits
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

// Multi-tile full distribution: p_i / total for a stored state.
template <typename T>
__global__ void full_probs_kernel(const typename Cx<T>::V* __restrict__ st, int64_t dim, const double* __restrict__ total,
                                  double* __restrict__ out) {
    const double t = *total;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = norm2(st[i]) / t;
}

}  // namespace qvb
