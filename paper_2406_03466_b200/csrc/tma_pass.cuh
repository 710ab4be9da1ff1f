// tma_pass.cuh — warp-specialised, TMA-fed pass kernel for multi-tile states.
//
// One persistent CTA per SM walks the (state, tile) items of one plan pass,
// state fastest (the same item order as pass_kernel, so co-running CTAs share
// a trunk tile through L2).  Roles:
//
//   warp 8, lane 0  -- producer.  Per item: one cp.async.bulk.tensor load of
//                      the tile (a box of the <= 5-D tensor view of the state
//                      batch that the planner chose, TmaLayout) plus a 1-D
//                      cp.async.bulk of the item's fused matrices into the
//                      item's stage, both completing on the stage's `full`
//                      mbarrier; once the compute warps release the stage
//                      (`done`), one cp.async.bulk.tensor store of the tile
//                      back to HBM, and after its shared-memory reads retire
//                      (bulk wait_group.read) the load of item i + STAGES.
//   warps 0-7       -- compute.  The register groups of pass_kernel (same
//                      descriptors, same rot2 arithmetic order, so every
//                      amplitude is bitwise identical to the pass_kernel
//                      result), named barrier 1 between groups that need it;
//                      the last group writes in the TMA box layout.
//
// The compute warps issue no global loads or stores: HBM streaming is done by
// the TMA unit behind the FP64 math of the previous / next tiles, which is
// what the round-1 LDGSTS kernel could not overlap.
// Replaces, for the bulk of a gradient's passes, the reference's per-gate
// sweeps (pkg/src/qvirt/kernels.py:18-70).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "plan.hpp"

namespace qvb {

constexpr int kTmaTeamThreads = 256;       // 2^(12 - 4): one register group covers a 12-bit tile
// (complex64 tiles are 13 bits: one team of 2^(13 - 4) = 512 threads)
// One team: 8 compute warps + a producer warp (288 threads).  Two teams: 16
// compute warps and no producer warp (512 threads, 128 registers each -- a
// 17th warp would cut every warp's register share, allocated in 4-warp
// units, to 96); the team that finishes an item issues its store and the
// load that reuses the stage (see tma_pass_kernel).
// With PWG (two teams + a producer warpgroup: 640 threads) the launch gets
// 96 registers per thread; the producer warpgroup gives most of its share back
// (setmaxnreg 24) and the compute warpgroups take 112 -- within the CTA's
// pool of 96 x 640 (asking for more than the pool holds never returns).
// Two teams on tiles of 2^tbits register groups, tbits > 8 (complex64, 13-bit
// tiles): each team keeps 256 threads, every thread holding 2^(tbits - 8)
// register groups of the tile ("sub-batches").
__host__ __device__ constexpr int tma_threads(int teams, bool pwg = false, int tbits = 8) {
    return teams == 1 ? (1 << tbits) + 32 : 2 * (1 << (tbits < 8 ? tbits : 8)) + (pwg ? 128 : 0);
}
constexpr int kPwgComputeRegs = 112, kPwgProducerRegs = 24;
static_assert(2 * kTmaTeamThreads * kPwgComputeRegs + 128 * kPwgProducerRegs <= 96 * 640, "setmaxnreg pool");
constexpr int kTmaMatBytes = 4096;         // per-stage matrix area (<= 64 complex128 matrices)

// Per-launch constants of the TMA kernel (passed by value).
struct TmaArgs {
    int32_t ndim;             // index dimensions (shared-memory order); dimension ndim = state slot
    int32_t lo[4];            // lowest global bit of each dimension
    uint32_t cmask[4];        // coordinate mask of each dimension (span bits)
    int32_t elems0;           // tensor elements per amplitude in dimension 0 (2 for complex128)
    uint32_t wcombo[16];      // last group: TMA-layout byte offset of register j
    uint32_t wtcol[9];        // last group: TMA-layout byte offset of thread bit m
    uint64_t gwcombo[16];     // last group, direct stores: global amplitude offset of register j
    uint64_t gwtcol[9];       // last group, direct stores: global amplitude offset of thread bit m
    const unsigned char* base;   // state-slot array (the tensor's base address)
    uint64_t state_bytes;
    uint32_t tile_bytes, mat_bytes;
    uint32_t tmat_off;        // direct stores: byte offset of the teams' matrix buffers
    uint32_t ent_off;         // byte offset of the launch's (in, out, mats) table in shared memory
    uint32_t flam[9];         // first group: initial logical tile index of thread bit m
    uint32_t fmu[4];          // first group: initial logical tile index of register bit r
    int32_t pieces;           // a tile moves as `pieces` boxes split along the outermost box dimension
    int32_t piece_step;       // coordinate step between pieces along dimension ndim - 1
    long long* trace;         // QV_TMA_TRACE builds only (tools/tma_trace.py), else null
};

// QV_TMA_TRACE (diagnostic build, libqvb200_trace.so): %clock64 of each phase
// of the first kTraceItems items of each team of CTAs 0..kTraceCtas-1:
// trace[((cta * 2 + team) * kTraceItems + item) * 16 + event], event 0 = wait
// for the tile starts, 1 = tile resident, 2 + g = group g done, 12 = store
// issued, 13 = next load issued, 14 = item done.
constexpr int kTraceCtas = 4, kTraceItems = 64;
#ifndef QV_TMA_DIAG_NOMATH
#define QV_TMA_DIAG_NOMATH 0   // diagnostic builds only: skip the 2x2 math (wrong results)
#endif
#ifndef QV_TMA_DIAG_NOHBM
#define QV_TMA_DIAG_NOHBM 0    // diagnostic builds only: no tile loads / stores (wrong results)
#endif
#ifdef QV_TMA_TRACE
#define TMA_MARK(item, ev)                                                                             \
    do {                                                                                             \
        if (ta.trace && blockIdx.x < kTraceCtas && (item) / TEAMS < kTraceItems && tid == 0) {     \
            long long t_;                                                                            \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_));                                       \
            ta.trace[((blockIdx.x * 2 + team) * kTraceItems + (item) / TEAMS) * 16 + (ev)] = t_;    \
        }                                                                                            \
    } while (0)
#else
#define TMA_MARK(item, ev) \
    do {                   \
    } while (0)
#endif

template <int STAGES>
struct TmaSmem {   // byte offsets inside dynamic shared memory
    __host__ __device__ static constexpr uint32_t full(uint32_t tile) { return STAGES * (tile + kTmaMatBytes); }
    __host__ __device__ static constexpr uint32_t done(uint32_t tile) { return full(tile) + 16 * STAGES; }
    __host__ __device__ static constexpr uint32_t tok(uint32_t tile) { return done(tile) + 8 * STAGES; }
    __host__ __device__ static constexpr uint32_t groups(uint32_t tile) { return (tok(tile) + 16 + 127) & ~127u; }
    // per group, each team thread's slot base (XOR of its thread-bit columns)
    __host__ __device__ static constexpr uint32_t bases(uint32_t tile, int ng) { return groups(tile) + 128u * ng; }
    // per group, its four register-bit columns (combo[1], [2], [4], [8])
    __host__ __device__ static constexpr uint32_t rcols(uint32_t tile, int ng, int team_threads) {
        return bases(tile, ng) + 4u * team_threads * ng;
    }
    __host__ __device__ static constexpr uint32_t bytes(uint32_t tile, int ng, int team_threads) {
        return rcols(tile, ng, team_threads) + 16u * ng;
    }
};
// Item i's tile lands on full barrier full_of(i) = (stage, (i / STAGES) mod 2)
// and completes its phase full_parity(i).  Two barriers per stage: the items
// sharing one barrier are then 2*STAGES apart -- an even distance, so with
// two teams they all belong to the same team, which consumes them in order;
// a team can never wait on a barrier two phases ahead (a parity wait would
// then see the PREVIOUS phase as done and read a stage still being loaded).
template <int STAGES>
__device__ __forceinline__ uint32_t full_of(int i) { return (uint32_t)(i % STAGES + STAGES * ((i / STAGES) & 1)); }
template <int STAGES>
__device__ __forceinline__ uint32_t full_parity(int i) { return (uint32_t)((i / (2 * STAGES)) & 1); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        " WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const void* tmap, int32_t c0, int32_t c1, int32_t c2,
                                            int32_t c3, int32_t c4, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_store_5d(const void* tmap, int32_t c0, int32_t c1, int32_t c2, int32_t c3,
                                             int32_t c4, uint32_t src) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group"
        " [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(tmap),
        "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(src)
        : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// wait until at most n (0..3) of this thread's bulk groups still read shared memory
__device__ __forceinline__ void bulk_wait_read(int n) {
    switch (n) {
        case 0: asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); break;
        case 1: asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); break;
        case 2: asm volatile("cp.async.bulk.wait_group.read 2;\n" ::: "memory"); break;
        default: asm volatile("cp.async.bulk.wait_group.read 3;\n" ::: "memory"); break;
    }
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
template <int TT>
__device__ __forceinline__ void team_sync(int team) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + team), "n"(TT) : "memory");
}

// TEAMS compute teams of 8 warps each take alternate items (team t: items
// t, t + TEAMS, ...), so one team's shared-memory round trips and barriers
// overlap the other team's FP64 math (with a single team the FP64 pipe sat
// idle through every load / barrier phase: 46 % busy, ncu).
//
// Stage protocol: item i lives in stage i % STAGES.  Its tile + matrices
// arrive on full barrier full_of(i) (one expect_tx arrival + the TMA
// transaction bytes).  Two ways to give the stage back:
//  * DIRECT (default, TEAMS = 2): at the item's start the team copies the
//    item's matrices into its own double buffer; the last register group,
//    once every thread of the team has read its amplitudes, releases the
//    stage -- an elected thread issues the load of item i + STAGES into it
//    right away -- and then stores its registers straight to HBM
//    (st.global.cs, gwcombo / gwtcol: the final positions as global offsets).
//    With two teams computing on two of the three stages, the third stage's
//    turnaround (store read-out + next load) was what starved them (11 % of
//    warp samples waiting on `full`, ncu); this shortens it to the load alone.
//  * TMA store: the last group writes the tile back in the TMA box layout and
//    one bulk-tensor store sends it; once the store has read the stage, the
//    load of item i + STAGES is issued (by the producer warp for TEAMS = 1,
//    signalled by done[], or by an elected thread of the team for TEAMS = 2).
//
// ALT (two teams that never block on the TMA: producer warpgroup or direct
// stores): the teams take turns on the FP64 pipe -- math phase k of team 1
// waits for team 0's phase k, team 0's phase k + 1 for team 1's phase k
// (two mbarriers, one arrival per thread after its math) -- so each team's
// shared-memory loads, stores and barriers run under the other team's math
// instead of in phase with it (both teams computing at once doubled every
// group's time, QV_TMA_TRACE).
// CM (complex64, two teams): the launch's matrix tables live in constant
// memory (c_tma_mats, gathered per launch) and are read with LDC instead of
// broadcast shared loads -- 32q x 4L complex64 4.67 -> 4.55 s (same box);
// for complex128 the eight LDC.64 per matrix cost more than they save.
constexpr int kTmaConstBytes = 65536;
#ifndef QV_TMA_PACKED
#define QV_TMA_PACKED 1
#endif
__constant__ uint4 c_tma_mats[kTmaConstBytes / 16];
template <typename V>
__global__ void gather_cmats_kernel(const LaunchEntry* __restrict__ ent, int m0, int nm, V* __restrict__ out) {
    const V* src = reinterpret_cast<const V*>(ent[blockIdx.x].mats) + (size_t)m0 * 4;
    for (int q = threadIdx.x; q < nm * 4; q += blockDim.x) out[(size_t)blockIdx.x * nm * 4 + q] = src[q];
}
// complex64: each matrix as the seven packed FFMA2 operand pairs (+1 pad),
// (m00.x, m00.x), (m01.x, m01.x), (-m01.y, m01.y), (m10.x, m10.x),
// (-m10.y, m10.y), (m11.x, m11.x), (-m11.y, m11.y) -- 64 B per matrix
constexpr int kPackedMatBytes = 64;
__global__ void gather_cmats_packed_kernel(const LaunchEntry* __restrict__ ent, int m0, int nm, float2* __restrict__ out) {
    const float2* src = reinterpret_cast<const float2*>(ent[blockIdx.x].mats) + (size_t)m0 * 4;
    for (int q = threadIdx.x; q < nm; q += blockDim.x) {
        const float2 a = src[4 * q], b = src[4 * q + 1], c = src[4 * q + 2], d = src[4 * q + 3];
        float2* o = out + ((size_t)blockIdx.x * nm + q) * 8;
        o[0] = make_float2(a.x, a.x);
        o[1] = make_float2(b.x, b.x);
        o[2] = make_float2(-b.y, b.y);
        o[3] = make_float2(c.x, c.x);
        o[4] = make_float2(-c.y, c.y);
        o[5] = make_float2(d.x, d.x);
        o[6] = make_float2(-d.y, d.y);
        o[7] = make_float2(0.f, 0.f);
    }
}
typedef unsigned long long f2p;
__device__ __forceinline__ f2p f2_fma(f2p a, f2p b, f2p c) {
    f2p d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2p f2_mul(f2p a, f2p b) {
    f2p d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2p f2_swap(f2p a) {
    f2p d;
    asm("{\n\t.reg .f32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\tmov.b64 %0, {hi, lo};\n\t}" : "=l"(d) : "l"(a));
    return d;
}
// rot2 on packed (x, y) lanes: lane by lane the scalar rot2's FMA sequence
__device__ __forceinline__ void rot2_packed(const f2p* M, float2& u2, float2& v2) {
    f2p u = *reinterpret_cast<const f2p*>(&u2), v = *reinterpret_cast<const f2p*>(&v2);
    const f2p us = f2_swap(u), vs = f2_swap(v);
    f2p a = f2_mul(M[2], vs);
    a = f2_fma(M[1], v, a);
    a = f2_fma(M[0], u, a);
    f2p b = f2_mul(M[6], vs);
    b = f2_fma(M[5], v, b);
    b = f2_fma(M[4], us, b);
    b = f2_fma(M[3], u, b);
    *reinterpret_cast<f2p*>(&u2) = a;
    *reinterpret_cast<f2p*>(&v2) = b;
}

template <typename T, int TBITS, int STAGES, int TEAMS, bool DIRECT, bool PWG, bool ALT, bool CM = false>
__global__ void __launch_bounds__(tma_threads(TEAMS, PWG, TBITS), 1)
tma_pass_kernel(const __grid_constant__ CUtensorMap tmap, const PassDesc pd, const TmaArgs ta,
                const GroupDesc* __restrict__ gdesc, const LaunchEntry* __restrict__ ent, int nstates, int64_t ntiles) {
    static_assert(!DIRECT || TEAMS > 1, "direct stores are issued by the teams themselves");
    static_assert(!PWG || (TEAMS == 2 && !DIRECT), "the producer warpgroup serves two teams with bulk stores");
    static_assert(!ALT || TEAMS == 2, "alternating math needs two teams");
    constexpr bool PRODUCER_THREAD = TEAMS == 1 || PWG;
    constexpr bool PACKED = CM && sizeof(T) == 4 && QV_TMA_PACKED;   // complex64 FFMA2 from packed constant operands   // a thread outside the teams stores and reloads stages
    typedef typename Cx<T>::V V;
    constexpr int R = reg_bits(sizeof(T) == 8 ? 0 : 1);
    constexpr int NA = 1 << R;
    constexpr int TB = TBITS;
    // threads of a team: with one team, one register group per thread covers
    // the tile; two teams keep 256 threads and SUB groups per thread
    constexpr int SUB = (TEAMS == 2 && TB > 8) ? 1 << (TB - 8) : 1;
    constexpr int TT = (1 << TB) / SUB;
    constexpr int TTB = TB - (SUB == 2 ? 1 : SUB == 4 ? 2 : 0);   // log2(TT)
    static_assert(SUB <= 2 && (1 << TTB) == TT, "at most two sub-batches per thread");
    static_assert(SUB == 1 || (!DIRECT && !PWG && !ALT), "sub-batches: bulk stores by the team");
    constexpr int COMPUTE = TEAMS * TT;
    extern __shared__ __align__(1024) unsigned char tma_smem[];
    unsigned char* smem_raw = tma_smem;
    const uint32_t TILE = ta.tile_bytes;
    const uint32_t sbase = smem_u32(smem_raw);
    GroupDesc* sg = reinterpret_cast<GroupDesc*>(smem_raw + TmaSmem<STAGES>::groups(TILE));
    const uint32_t full0 = sbase + TmaSmem<STAGES>::full(TILE);
    const uint32_t done0 = sbase + TmaSmem<STAGES>::done(TILE);
    const uint32_t tok0 = sbase + TmaSmem<STAGES>::tok(TILE);

    const int items = (int)(ntiles * nstates);
    const int G = gridDim.x;
    const int my_items = (int)blockIdx.x < items ? (items - 1 - (int)blockIdx.x) / G + 1 : 0;

    // per stage: the resident item's store coordinates (TMA store) or its
    // output base pointer (direct stores); written by the thread that issues
    // the item's load, before the arrival that releases them with the tile
    __shared__ int32_t soc[STAGES][5];
    __shared__ V* sout[STAGES];
    int32_t lc0 = 0, lc1 = 0, lc2 = 0, lc3 = 0, lc4 = 0;   // load coordinates of the item being issued
    uint32_t lbar = 0;                                      // and its full barrier
    // the launch's per-state constants, staged once (matrix table, output
    // pointer, input / output state slot): the thread that issues a load
    // never waits on a global read or divides in the middle of an item
    const uint64_t* sent = reinterpret_cast<const uint64_t*>(smem_raw + ta.ent_off);
    // Coordinates as five scalars (dimension `ndim` is the state slot):
    // written out per dimension so nothing is indexed at run time and the
    // issuing thread never touches local memory.
    auto coord = [&](int d, uint64_t o, int32_t slot) -> int32_t {
        int32_t v = d < ta.ndim ? (int32_t)((o >> ta.lo[d & 3]) & ta.cmask[d & 3]) : 0;
        if (d == 0) v *= ta.elems0;
        return d == ta.ndim ? slot : v;
    };
    auto issue_load = [&](int i) {
        const int w = (int)blockIdx.x + i * G;
        const int x = w / nstates, y = w - x * nstates;
        const void* mats = reinterpret_cast<const void*>(sent[3 * y]);
        void* out = reinterpret_cast<void*>(sent[3 * y + 1]);
        const uint64_t slots = sent[3 * y + 2];
        const int32_t in_slot = (int32_t)(uint32_t)slots, out_slot = (int32_t)(slots >> 32);
        uint64_t o = 0;   // outer offset of tile x (light-cone restricted passes list fewer bits)
        for (int j = 0; j < pd.n_outer; ++j)
            if ((x >> j) & 1) o |= 1ull << pd.obits[j];
        const int s = i % STAGES;
        soc[s][0] = coord(0, o, out_slot);
        soc[s][1] = coord(1, o, out_slot);
        soc[s][2] = coord(2, o, out_slot);
        soc[s][3] = coord(3, o, out_slot);
        soc[s][4] = coord(4, o, out_slot);
        sout[s] = reinterpret_cast<V*>(out) + o;
        lc0 = coord(0, o, in_slot);
        lc1 = coord(1, o, in_slot);
        lc2 = coord(2, o, in_slot);
        lc3 = coord(3, o, in_slot);
        lc4 = coord(4, o, in_slot);
        const uint32_t bar = full0 + 8 * full_of<STAGES>(i);
        lbar = bar;
        if (QV_TMA_DIAG_NOHBM) {
            mbar_arrive(bar);
            return;
        }
        if constexpr (CM) {
            (void)mats;
            mbar_expect_tx(bar, TILE);
        } else {
            mbar_expect_tx(bar, TILE + ta.mat_bytes);
            bulk_load(sbase + STAGES * TILE + s * kTmaMatBytes, reinterpret_cast<const V*>(mats) + (size_t)pd.m0 * 4,
                      ta.mat_bytes, bar);
        }
        lbar = bar;
    };
    // The tile as `pieces` boxes (split along the outermost box dimension,
    // contiguous in shared memory): a stage's store and the load that reuses
    // it overlap piece by piece -- piece q of the next item loads as soon as
    // piece q of the last one has been read out.
    const uint32_t PIECE = TILE / (uint32_t)ta.pieces;
    const int pdim = ta.ndim - 1;   // the dimension pieces step along
    auto load_piece = [&](int s, int q) {
        if (QV_TMA_DIAG_NOHBM) return;
        const int32_t dq = q * ta.piece_step;
        tma_load_5d(sbase + s * TILE + q * PIECE, &tmap, lc0 + (pdim == 0 ? dq : 0), lc1 + (pdim == 1 ? dq : 0),
                    lc2 + (pdim == 2 ? dq : 0), lc3 + (pdim == 3 ? dq : 0), lc4, lbar);
    };
    auto store_piece = [&](int s, int q) {
        if (QV_TMA_DIAG_NOHBM) return;
        const int32_t dq = q * ta.piece_step;
        tma_store_5d(&tmap, soc[s][0] + (pdim == 0 ? dq : 0), soc[s][1] + (pdim == 1 ? dq : 0),
                     soc[s][2] + (pdim == 2 ? dq : 0), soc[s][3] + (pdim == 3 ? dq : 0), soc[s][4],
                     sbase + s * TILE + q * PIECE);
        bulk_commit();
    };
    // store the item in stage s, then load item `next` (if any) into it
    auto turn_stage = [&](int s, int next) {
        for (int q = 0; q < ta.pieces; ++q) store_piece(s, q);
        if (next < my_items) {
            issue_load(next);
            for (int q = 0; q < ta.pieces; ++q) {
                bulk_wait_read(ta.pieces - 1 - q);   // piece q of the store has left shared memory
                load_piece(s, q);
            }
        }
    };
    {
        const uint4* gsrc = reinterpret_cast<const uint4*>(gdesc + pd.g0);
        uint4* gdst = reinterpret_cast<uint4*>(sg);
        for (int i = threadIdx.x; i < pd.ng * 8; i += blockDim.x) gdst[i] = gsrc[i];
        uint64_t* se = reinterpret_cast<uint64_t*>(smem_raw + ta.ent_off);
        for (int y = threadIdx.x; y < nstates; y += blockDim.x) {
            const uint64_t in_slot = (uint64_t)((const unsigned char*)ent[y].in - ta.base) / ta.state_bytes;
            const uint64_t out_slot = (uint64_t)((const unsigned char*)ent[y].out - ta.base) / ta.state_bytes;
            se[3 * y] = reinterpret_cast<uint64_t>(ent[y].mats);
            se[3 * y + 1] = reinterpret_cast<uint64_t>(ent[y].out);
            se[3 * y + 2] = (uint32_t)in_slot | (out_slot << 32);
        }
        __syncthreads();
        // slot bases of every group for each team thread (one conflict-free
        // LDS per group instead of TTB descriptor reads and XORs)
        uint32_t* sb = reinterpret_cast<uint32_t*>(smem_raw + TmaSmem<STAGES>::bases(TILE, pd.ng));
        for (int j = threadIdx.x; j < pd.ng * TT; j += blockDim.x) {
            const int g = j / TT, t = j % TT;
            uint32_t b = 0;
            for (int m = 0; m < TTB; ++m)
                if ((t >> m) & 1) b ^= sg[g].tcol[m];
            sb[j] = b;
        }
        uint4* sr = reinterpret_cast<uint4*>(smem_raw + TmaSmem<STAGES>::rcols(TILE, pd.ng, TT));
        for (int g = threadIdx.x; g < pd.ng; g += blockDim.x)
            sr[g] = make_uint4(sg[g].combo[1], sg[g].combo[2], sg[g].combo[4], sg[g].combo[8]);
        if (threadIdx.x == 0) {
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(full0 + 8 * s, 1);
                mbar_init(full0 + 8 * (STAGES + s), 1);
                mbar_init(done0 + 8 * s, TT / 32);   // one arrival per warp
            }
            mbar_init(tok0, TT / 32);
            mbar_init(tok0 + 8, TT / 32);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            fence_proxy_async_smem();
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmap) : "memory");
            for (int i = 0; i < STAGES && i < my_items; ++i) {
                issue_load(i);
                for (int q = 0; q < ta.pieces; ++q) load_piece(i % STAGES, q);
            }
        }
    }
    __syncthreads();

    if (threadIdx.x >= COMPUTE) {
        // ------------------------------- producer (TEAMS == 1 or PWG)
        if constexpr (PWG) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kPwgProducerRegs) : "memory");
        if (threadIdx.x != COMPUTE) return;
        for (int j = 0; j < my_items; ++j) {
            const int s = j % STAGES;
            mbar_wait(done0 + 8 * s, (uint32_t)((j / STAGES) & 1));
            turn_stage(s, j + STAGES);
        }
        bulk_wait0();   // every store has completed before the CTA retires
        return;
    }

    // ---------------------------------------------------------------- compute
    if constexpr (PWG) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kPwgComputeRegs) : "memory");
    const int team = TEAMS == 1 ? 0 : (int)(threadIdx.x / TT);
    const int tid = (int)(threadIdx.x % TT);
    // ALT: math phases of this team so far, and how many each team has in total
    int phase = 0;
    const int phases0 = ((my_items + 1) / 2) * pd.ng, phases1 = (my_items / 2) * pd.ng;
    uint32_t wbase = 0, flt = 0;
    uint64_t gbase = 0;
#pragma unroll
    for (int m = 0; m < TTB; ++m)
        if ((tid >> m) & 1) {
            wbase ^= ta.wtcol[m];
            flt ^= ta.flam[m];
            if constexpr (DIRECT) gbase ^= ta.gwtcol[m];
        }
    const uint32_t* sbases = reinterpret_cast<const uint32_t*>(smem_raw + TmaSmem<STAGES>::bases(TILE, pd.ng));
    const uint4* srcols = reinterpret_cast<const uint4*>(smem_raw + TmaSmem<STAGES>::rcols(TILE, pd.ng, TT));
    for (int i = team; i < my_items; i += TEAMS) {
        const int s = i % STAGES;
        TMA_MARK(i, 0);
        mbar_wait(full0 + 8 * full_of<STAGES>(i), full_parity<STAGES>(i));
        TMA_MARK(i, 1);
        const uint32_t boff = s * TILE;   // a multiple of 2^15 >= every slot offset
        const V* smat = CM ? reinterpret_cast<const V*>(c_tma_mats) + (size_t)(((int)blockIdx.x + i * G) % nstates) * pd.nm * 4
                           : reinterpret_cast<const V*>(smem_raw + STAGES * TILE + s * kTmaMatBytes);
        const f2p* cpk = reinterpret_cast<const f2p*>(c_tma_mats) + (size_t)(((int)blockIdx.x + i * G) % nstates) * pd.nm * 8;
        (void)cpk;
        V* __restrict__ out = nullptr;
        if constexpr (DIRECT) {
            // the stage is released before the last group's math: its
            // matrices move to this team's buffer (double-buffered by item,
            // so a slow warp of the previous item never sees them change)
            out = sout[s];
            V* tm = reinterpret_cast<V*>(smem_raw + ta.tmat_off + (size_t)(2 * team + ((i / TEAMS) & 1)) * ta.mat_bytes);
            for (int q = tid; q < pd.nm * 4; q += TT) tm[q] = smat[q];
            team_sync<TT>(team);
            smat = tm;
        }
        for (int g = 0; g < pd.ng; ++g) {
            const GroupDesc& GD = sg[g];
            const int4 mats = *reinterpret_cast<const int4*>(GD.mat);
            V m00, m01, m10, m11;
            if (!PACKED && mats.x >= 0) {
                const V* M = smat + mats.x * 4;
                m00 = M[0]; m01 = M[1]; m10 = M[2]; m11 = M[3];
            }
            const uint32_t base = boff ^ sbases[g * TT + tid];
            // sub-batch h of this thread: virtual thread tid + h * TT
            const uint32_t hcol = SUB > 1 ? GD.tcol[TTB < 10 ? TTB : 0] : 0u;
            // slot of register j = base ^ combo[j]; combo is the XOR of the
            // four register-bit columns combo[1], [2], [4], [8]
            const uint4 rcv = srcols[g];
            const uint32_t rc0 = rcv.x, rc1 = rcv.y, rc2 = rcv.z, rc3 = rcv.w;
            auto off = [&](int h, int j) -> uint32_t {
                return base ^ (h ? hcol : 0u) ^ ((j & 1) ? rc0 : 0u) ^ ((j & 2) ? rc1 : 0u) ^ ((j & 4) ? rc2 : 0u) ^
                       ((j & 8) ? rc3 : 0u);
            };
            V a[SUB][NA];
#ifndef QV_TMA_DIAG_NOSMEM
#define QV_TMA_DIAG_NOSMEM 0   // diagnostic builds only: registers instead of the group's smem round trip
#endif
#pragma unroll
            for (int h = 0; h < SUB; ++h) {
                if (QV_TMA_DIAG_NOSMEM && g > 0) {
#pragma unroll
                    for (int j = 0; j < NA; ++j) a[h][j] = V{T(j + tid), T(g)};
                } else {
#pragma unroll
                    for (int j = 0; j < NA; ++j) a[h][j] = *reinterpret_cast<const V*>(smem_raw + off(h, j));
                }
            }
            if (g == 0 && pd.fresh) {
                // slots whose initial index has a bit no earlier pass touched
                // hold amplitude 0 (the box brought whatever HBM had there)
#pragma unroll
                for (int h = 0; h < SUB; ++h)
#pragma unroll
                    for (int j = 0; j < NA; ++j) {
                        const uint32_t l = flt ^ (h ? ta.flam[TTB < 9 ? TTB : 0] : 0u) ^ ((j & 1) ? ta.fmu[0] : 0u) ^
                                           ((j & 2) ? ta.fmu[1] : 0u) ^ ((j & 4) ? ta.fmu[2] : 0u) ^
                                           ((j & 8) ? ta.fmu[3] : 0u);
                        if (l & pd.fresh) a[h][j] = V{T(0), T(0)};
                    }
            }
            const bool last = g + 1 == pd.ng;
            // read before the math: after the group's 16 shared stores this
            // load would wait behind them in the MIO queue
            const bool next_cta_sync = !last && sg[g + 1].cta_sync;
            if (DIRECT && last) {
                // every thread of the team has read the stage: hand it to the
                // load of item i + STAGES
                team_sync<TT>(team);
                if (tid == 0 && i + STAGES < my_items) {
                    issue_load(i + STAGES);
                    for (int q = 0; q < ta.pieces; ++q) load_piece(s, q);
                }
            }
            if constexpr (ALT) {   // this team's turn on the FP64 pipe
                if (team == 0 && phase >= 1 && phase <= phases1) mbar_wait(tok0, (uint32_t)((phase - 1) & 1));
                if (team == 1 && phase < phases0) mbar_wait(tok0 + 8, (uint32_t)(phase & 1));
            }
            if constexpr (PACKED) {
                // complex64 + constant matrices: packed FFMA2 operands straight from LDC
#pragma unroll
                for (int r = 0; r < (QV_TMA_DIAG_NOMATH ? 0 : R); ++r) {
                    const int mi = r == 0 ? mats.x : r == 1 ? mats.y : r == 2 ? mats.z : mats.w;
                    if (mi >= 0) {
                        const f2p* M = cpk + (size_t)mi * 8;
                        f2p pm[7];
#pragma unroll
                        for (int e = 0; e < 7; ++e) pm[e] = M[e];
#pragma unroll
                        for (int h = 0; h < SUB; ++h)
#pragma unroll
                            for (int j = 0; j < NA; ++j)
                                if (!((j >> r) & 1)) rot2_packed(pm, a[h][j], a[h][j | (1 << r)]);
                    }
                }
            } else {
#pragma unroll
            for (int r = 0; r < (QV_TMA_DIAG_NOMATH ? 0 : R); ++r) {
                const int mi = r == 0 ? mats.x : r == 1 ? mats.y : r == 2 ? mats.z : mats.w;
                if (mi >= 0) {
                    if (r > 0) {
                        const V* M = smat + mi * 4;
                        m00 = M[0]; m01 = M[1]; m10 = M[2]; m11 = M[3];
                    }
#pragma unroll
                    for (int h = 0; h < SUB; ++h)
#pragma unroll
                        for (int j = 0; j < NA; ++j)
                            if (!((j >> r) & 1)) rot2<V>(m00, m01, m10, m11, a[h][j], a[h][j | (1 << r)]);
                }
            }
            }
            if constexpr (ALT) {   // hand the FP64 pipe to the other team
                // one arrival per warp (256 arrivals on one word serialise)
                __syncwarp();
                if ((tid & 31) == 0) {
                    if (team == 0 && phase < phases0) mbar_arrive(tok0 + 8);
                    if (team == 1) mbar_arrive(tok0);
                }
                ++phase;
            }
            if (g < 10) TMA_MARK(i, 2 + g);
            if (!last && QV_TMA_DIAG_NOSMEM) {
                // diagnostic: keep the results live without the smem store
                if (a[0][0].x == T(-12345.678)) *reinterpret_cast<V*>(smem_raw + off(0, 0)) = a[0][1];
                if (!next_cta_sync) __syncwarp();
                else team_sync<TT>(team);
            } else if (!last) {
                // re-read the register-bit columns (volatile: the slot offsets
                // are recomputed here instead of being held -- or spilled --
                // across the group's math)
                const volatile uint4* vc = srcols + g;
                const uint32_t sc0 = vc->x, sc1 = vc->y, sc2 = vc->z, sc3 = vc->w;
                const uint32_t sh = SUB > 1 ? reinterpret_cast<const volatile uint32_t*>(GD.tcol)[TTB < 10 ? TTB : 0] : 0u;
#pragma unroll
                for (int h = 0; h < SUB; ++h)
#pragma unroll
                    for (int j = 0; j < NA; ++j)
                        *reinterpret_cast<V*>(smem_raw + (base ^ (h ? sh : 0u) ^ ((j & 1) ? sc0 : 0u) ^
                                                          ((j & 2) ? sc1 : 0u) ^ ((j & 4) ? sc2 : 0u) ^
                                                          ((j & 8) ? sc3 : 0u))) = a[h][j];
                if (!next_cta_sync) __syncwarp();
                else team_sync<TT>(team);
            } else if constexpr (DIRECT) {
                TMA_MARK(i, 12);
#pragma unroll
                for (int j = 0; j < NA; ++j) __stcs(out + (gbase ^ ta.gwcombo[j]), a[0][j]);
                TMA_MARK(i, 13);
            } else {
                // every thread of the team has read its amplitudes before any
                // is rewritten in the TMA box layout
                team_sync<TT>(team);
#pragma unroll
                for (int h = 0; h < SUB; ++h)
#pragma unroll
                    for (int j = 0; j < NA; ++j)
                        *reinterpret_cast<V*>(smem_raw + (boff ^ wbase ^ (h ? ta.wtcol[TTB < 9 ? TTB : 0] : 0u) ^
                                                          ta.wcombo[j])) = a[h][j];
            }
        }
        if constexpr (!DIRECT) {
            fence_proxy_async_smem();   // generic-proxy writes -> visible to the TMA store
            if constexpr (PRODUCER_THREAD) {
                __syncwarp();   // the warp's fenced writes, then one arrival per warp
                if ((tid & 31) == 0) mbar_arrive(done0 + 8 * s);
            } else {
                team_sync<TT>(team);
                TMA_MARK(i, 12);
                if (tid == 0) turn_stage(s, i + STAGES);
                TMA_MARK(i, 13);
            }
        }
    }
    if constexpr (!PRODUCER_THREAD && !DIRECT) {
        if (tid == 0) bulk_wait0();   // this team's stores have completed
    }
}

}  // namespace qvb
