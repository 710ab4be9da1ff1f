// plan.hpp — circuit topology -> fused ops -> HBM passes -> register groups.
//
// A *topology* is a gate list without angles (kinds + qubits).  Everything in
// a plan depends on the topology only, never on angles or on which other
// circuits share a batch, so every circuit's arithmetic is a function of the
// circuit alone: results are bitwise independent of how a batch is split
// across virtual QPUs / GPUs (the reference's serial-equivalence law,
// pkg/src/qvirt/pool.py:10-14).
//
// Index convention (reference kernels.py:3-7): qubit q <-> amplitude index
// bit b = n-1-q.  Internally everything is expressed in bits.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace qvb {

constexpr int kRegBits = 4;          // max register bits per group (descriptor capacity)
constexpr int kGroupAmps = 1 << kRegBits;

// Register bits per group (amplitudes per thread = 2^R).  4 for both
// precisions: 16 amplitudes and up to four 2x2 matrices per shared-memory
// round trip.  (Measured on B200: R = 3 at complex128 -- 512 threads per tile,
// twice the warps -- was 20% slower than R = 4 because every group then pays
// its round trip for only three matrices.)
#ifndef QV_C128_REG_BITS
#define QV_C128_REG_BITS 4
#endif
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr int reg_bits(int precision) { return precision == 0 ? QV_C128_REG_BITS : 4; }
// Widest tile (multi-tile registers): 64 KiB for both precisions -- 2^12
// complex128 / 2^13 complex64 amplitudes, three of them in the TMA kernel's
// shared-memory ring.  (complex128 at 13 bits, 128 KiB, leaves room for no
// ring; 11 bits needs 28 passes instead of 23 for 28q x 8L.  complex64 at 13
// bits: 13 passes instead of 17 for 32q x 4L.)
#ifndef QV_C128_TILE_BITS
#define QV_C128_TILE_BITS 12
#endif
#ifndef QV_C64_TILE_BITS
#define QV_C64_TILE_BITS 13
#endif
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr int max_tile_bits(int precision) { return precision == 0 ? QV_C128_TILE_BITS : QV_C64_TILE_BITS; }
constexpr int kMaxTileBits = 13;     // 2^13 amplitudes (64 KiB at complex64, 128 KiB c128)
constexpr int kMaxQubits = 40;

enum GateKind : uint8_t { G_H = 0, G_X = 1, G_CNOT = 2, G_RY = 3, G_RZ = 4, G_MEASURE = 5, G_RX = 6, G_CZ = 7 };

inline bool is_rotation(uint8_t k) { return k == G_RY || k == G_RZ || k == G_RX; }
inline bool is_two_qubit(uint8_t k) { return k == G_CNOT || k == G_CZ; }

struct Topology {
    int n = 0;
    std::vector<uint8_t> kind;
    std::vector<int32_t> q0, q1;
    std::string key() const;         // exact identity of the topology (n + gate list)
};

// A fused operation: a maximal run of 1-qubit gates on one bit (MAT1, the
// matrix is the ordered product of its gates) or one CNOT.  `gates` holds
// topology gate indices; -1 stands for a constant Hadamard (CZ lowering).
struct FusedOp {
    bool cnot = false;
    int b0 = 0;       // MAT1: bit; CNOT: control bit
    int b1 = -1;      // CNOT: target bit
    std::vector<int32_t> gates;
};

// Device descriptor of one register group: a thread loads 16 amplitudes from
// physical shared-memory slots base(tid) ^ combo[j], applies up to 4 2x2
// matrices on register bits 0..3 and stores them back.  Slots are stored as
// BYTE offsets for the state's amplitude size so the kernel XORs them
// straight into a shared-memory address.
//
// Thread bits 0..4 are the lanes of a warp, bits 5.. the warp index.  The
// planner keeps the warp-index bits of consecutive groups equal and untouched
// by their matrices and CNOT targets wherever it can ("warp-local segments"):
// every warp then reads back exactly the amplitudes it wrote, and the groups
// are separated by __syncwarp instead of a CTA barrier (`cta_sync` = 0).
struct alignas(16) GroupDesc {
    uint32_t combo[16];  // byte offset of register index j
    uint32_t tcol[11];   // byte offset of thread bit m (tile bits - 4 of them)
    int32_t cta_sync;    // 1: a CTA barrier must precede this group
    int32_t mat[4];      // matrix index within the pass (-1 = identity)
};
static_assert(sizeof(GroupDesc) == 128, "GroupDesc layout");

// Device descriptor of one pass (one HBM sweep over every tile of a state).
struct alignas(16) PassDesc {
    int32_t k;           // tile bits (logical local bits 0..k-1)
    int32_t n_outer;     // n - k outer (tile-index) bits
    int32_t g0, ng;      // group range in the plan's group array
    int32_t m0, nm;      // matrix slot range in a circuit's matrix table
    uint32_t fresh;      // logical local bits no earlier pass touched: amplitudes there are 0, loaded as zeros
    int32_t pad1;
    uint8_t sbits[16];   // logical local bit j -> global index bit
    uint8_t obits[40];   // outer bit j -> global index bit
    uint16_t swz[16];    // physical slot column of logical bit j at load time
    uint16_t fin[16];    // physical slot column of logical bit j at store time
    uint16_t swz_hi[16]; // physical slot of (it << (k-4)), it = 0..15, at load
    uint16_t fin_hi[16]; // same at store
    uint64_t g_hi[16];   // global offset of (it << (k-4))
};

struct PassPlan {
    std::vector<int> S;      // global bits in the tile, ascending (size k)
    std::vector<int> ops;    // fused-op indices applied, program order
    int n_groups = 0;
    int n_mats = 0;
};

// Tensor-memory-accelerator layout of a multi-tile pass (tma_pass.cuh).
//
// The state batch is viewed as a <= 5-D tensor: each index dimension is one
// "piece" of the pass's tile bits (a run of consecutive global bits, <= 8 of
// them so the box stays <= 256 elements) together with the outer bits above
// it up to the next piece; the last dimension is the state slot.  A tile is
// then ONE box of that tensor, and the box lands in shared memory in piece
// order (dimension 0 = the low `coalesce` bits, a 128-byte row) under TMA's
// 128-byte swizzle (16-byte chunk ^= row mod 8).  The planner picks the pieces
// and their order (which tile bits sit in the swizzled row positions) to
// minimise shared-memory bank wavefronts of the pass's register groups, and
// the pass's groups are built on that layout, so the TMA load needs no
// re-layout.  CNOTs folded into the slot maps leave the tile permuted at the
// end of the pass; the LAST register group therefore writes its amplitudes
// back in the TMA layout (wcombo / wtcol) and the TMA store reads the same
// box layout.
struct TmaLayout {
    int32_t ok = 0;             // the pass can run on the TMA kernel
    int32_t ndim = 0;           // index dimensions, shared-memory order (<= 4)
    int32_t lo[4] = {0, 0, 0, 0};    // lowest global bit of each dimension
    int32_t span[4] = {0, 0, 0, 0};  // global bits the dimension covers
    int32_t box[4] = {0, 0, 0, 0};   // tile bits of the dimension (box = 2^box)
    uint32_t wcombo[16] = {0};  // last group: byte offset of register j in the TMA layout
    uint32_t wtcol[11] = {0};   // last group: byte offset of thread bit m in the TMA layout
    // the same registers' final positions as global amplitude offsets (OR of
    // 1 << sbits): the last group can store straight from registers to HBM
    uint64_t gwcombo[16] = {0};
    uint64_t gwtcol[11] = {0};
    int32_t coalesced = 0;      // lanes 0..c-1 of the last group write one contiguous 128-byte row
    // initial logical tile index of the FIRST group's thread bit m / register
    // bit r: a register whose index has a `fresh` bit (never touched before
    // this pass: the amplitude is 0) is zero-filled as it is read, so passes
    // with fresh bits also run on the TMA kernel (the box still loads them)
    uint32_t flam[11] = {0};
    uint32_t fmu[4] = {0};
    int64_t wavefronts = 0;     // bank model of the chosen layout (tools / tests)
};

struct Plan {
    int n = 0;
    int k = 0;               // tile bits
    int precision = 0;       // 0 = complex128, 1 = complex64
    bool single_tile = false;
    std::vector<FusedOp> ops;
    std::vector<int> mat_op;         // matrix slot -> fused op (slots ordered pass by pass)
    std::vector<PassPlan> passes;
    std::vector<PassDesc> pdesc;
    std::vector<TmaLayout> tma;      // per pass
    std::vector<GroupDesc> groups;
    int n_slots() const { return (int)mat_op.size(); }
};

// Tile bits used for a register of n qubits at a precision.
int tile_bits_for(int n, int precision);

// Build the full plan (fusion, pass selection, groups, descriptors).
// `max_tile_bits` > 0 overrides the precision's tile size (tests use small
// tiles to exercise the multi-tile planner on registers a CPU can check).
Plan build_plan(const Topology& topo, int precision, int max_tile_bits = 0);

// Fused 2x2 matrices of every slot for one circuit: out[slot*8 + 0..7] =
// (m00.re, m00.im, m01.re, m01.im, m10.re, m10.im, m11.re, m11.im).
// `angles` is indexed by topology gate index.
void circuit_matrices(const Plan& plan, const Topology& topo, const double* angles, double* out);

// Matrix of one slot with the generator Pauli of rotation gate `pauli_gate`
// (a topology gate index inside that slot) inserted just before the gate.
void slot_matrix_with_pauli(const Plan& plan, const Topology& topo, const double* angles, int slot,
                            int32_t pauli_gate, double* out8);

// Slot holding topology gate g (-1 if g is not a one-qubit gate of the plan).
std::vector<int> slot_of_gates(const Plan& plan, const Topology& topo);

// Light cone of a support-restricted output (SUPPORT / JS results, shift
// pairs): per pass, the global bits its tile index ranges over and the local
// bits it is the first to touch (zero-filled instead of loaded); `reach` =
// bits any pass touches (support indices outside it have amplitude 0).
struct LightCone {
    std::vector<uint64_t> outer_free;
    std::vector<uint32_t> fresh;
    uint64_t reach = 0;
};
LightCone light_cone(const Plan& plan, const uint64_t* support, int64_t S);

// The pass restricted to the tiles whose outer bits outside `free` are zero.
PassDesc restrict_pass(const PassDesc& pd, uint64_t free, uint32_t fresh);

// Low index bits every tile holds (a 128-byte row): 3 for complex128, 4 for complex64.
int tile_low_bits(int precision);

// A read-only pass (no register groups, identity slot layout) over the tile
// bit set `S` (k bits, including the low bits): the multi-tile Pauli sweeps.
PassDesc readonly_pass(const Plan& plan, uint64_t S);

#ifdef __CUDACC__
#define QV_HD __host__ __device__
#else
#define QV_HD
#endif

// Physical slot of a logical local index under a column map.
QV_HD inline uint32_t apply_cols(const uint16_t* cols, int k, uint32_t idx) {
    uint32_t r = 0;
    for (int j = 0; j < k; ++j)
        if ((idx >> j) & 1u) r ^= cols[j];
    return r;
}

}  // namespace qvb
