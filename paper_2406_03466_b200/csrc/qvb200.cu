// qvb200.cu — executor runtime and the C ABI declared in include/qvb200.h.
//
// One `Engine` per qv_handle: a CUDA device, a stream, a plan cache keyed by
// circuit topology, grow-only device buffers and the prefix-sharing scheduler.
//
// Scheduler (large registers, state in HBM).  A parameter-shift batch
// (reference gradients.py:33-46) is 2*N_theta copies of one circuit that each
// differ in one angle.  Every circuit is a fixed sequence of plan passes whose
// inputs are the previous pass's output and this circuit's fused matrices, so
// two circuits whose matrices agree on passes [0, p) have bit-identical states
// after pass p-1.  The scheduler keeps one "trunk" state (the prefix shared by
// the most circuits), branches every circuit off the trunk at the first pass
// where it differs, and runs the branches in batches on work buffers.  The
// arithmetic each circuit sees is exactly what it would see alone, so results
// stay bitwise independent of batch composition and device (pool.py:10-14),
// while the number of HBM sweeps drops to sum_c (P - branch_pass_c).
#include <chrono>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <utility>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "kernels.cuh"
#include "plan.hpp"
#include "sampling.cuh"
#include "tma_pass.cuh"
#include "qvb200.h"

namespace qvb {

struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ArgError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CircuitError : std::runtime_error {
    int64_t index;
    CircuitError(int64_t i, const std::string& m) : std::runtime_error(m), index(i) {}
};

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <typename X>
struct DevBuf {
    X* p = nullptr;
    size_t cap = 0;
    X* get(size_t n) {
        if (n == 0) n = 1;
        if (n > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            CK(cudaMalloc(&p, n * sizeof(X)));
            cap = n;
        }
        return p;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct CachedPlan {
    Topology topo;
    Plan plan;
    DevBuf<GroupDesc> d_groups;
};


// Hash of a matrix table, 8 bytes a step (candidates are confirmed with
// memcmp, so only the spread matters; a byte-wise FNV-1a cost ~10 ms per 1 024
// circuits of 20q x 6L).
uint64_t hash_words(const void* data, size_t bytes, uint64_t h = 1469598103934665603ull) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    size_t i = 0;
    for (; i + 8 <= bytes; i += 8) {
        uint64_t w;
        std::memcpy(&w, p + i, 8);
        h = (h ^ w) * 0x9e3779b97f4a7c15ull;
        h ^= h >> 29;
    }
    for (; i < bytes; ++i) { h ^= p[i]; h *= 1099511628211ull; }
    return h;
}

struct Engine {
    int device = 0;
    int precision = 0;
    uint64_t budget = 0;           // caller's cap on state memory (0: what the device has free)
    cudaStream_t stream = nullptr;
    std::mutex mu;
    std::string err;
    int64_t err_circuit = -1;
    double stats[18] = {0};   // [16] host ms of the call, [17] host ms before the first launch
    std::chrono::steady_clock::time_point t_entry;
    double host_ms() const {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_entry).count();
    }
    std::unordered_map<std::string, std::unique_ptr<CachedPlan>> plans;

    DevBuf<unsigned char> d_states;
    DevBuf<unsigned char> d_mats;
    DevBuf<LaunchEntry> d_entries;
    DevBuf<double> d_partial;
    DevBuf<double2> d_partial2;
    DevBuf<double> d_sup_out, d_js_out, d_full_out, d_pauli_out, d_target, d_delta, d_cstage;
    DevBuf<uint64_t> d_support, d_tflip, d_tphase;
    DevBuf<int64_t> d_term_off, d_slots;
    DevBuf<int32_t> d_sup_off, d_sup_local, d_sup_pos, d_tsweep;
    DevBuf<uint32_t> d_tfslot, d_tphloc;
    DevBuf<uint64_t> d_tphout;
    std::vector<cudaEvent_t> events;
    size_t events_used = 0;
    // pinned staging for host->device copies: a call's inputs are copied into
    // it and sent with truly asynchronous cudaMemcpyAsync (pageable sources
    // would each be staged synchronously by the driver).  Reset per call;
    // every call ends with a stream synchronisation.
    unsigned char* pinned = nullptr;
    size_t pinned_cap = 0, pinned_used = 0;

    unsigned char* stage(size_t bytes) {
        const size_t need = (bytes + 255) & ~(size_t)255;
        if (pinned_used + need > pinned_cap) {
            CK(cudaStreamSynchronize(stream));   // pending copies may still read the old buffer
            if (pinned) CK(cudaFreeHost(pinned));
            pinned_cap = std::max<size_t>({need, 2 * pinned_cap, (size_t)1 << 20});
            CK(cudaMallocHost(reinterpret_cast<void**>(&pinned), pinned_cap));
            pinned_used = 0;
        }
        unsigned char* at = pinned + pinned_used;
        pinned_used += need;
        return at;
    }
    struct Timed {
        cudaEvent_t start, stop;
        bool tma;
        double bytes;
        int m0, nm, nstates;   // pass (first matrix slot, matrices) and states of the launch
        int64_t ntiles;
    };
    std::vector<Timed> timed;   // pass-kernel launches of this call

    // Bytes available for state buffers now: the caller's cap, or this
    // engine's current state allocation plus 90 % of what the device has
    // free less 1 GiB for tables (other engines in the process, e.g. the
    // other precision, have taken their share by then).
    uint64_t state_budget() {
        if (budget) return budget;
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        const double avail = 0.9 * (double)free_b - (double)(1ull << 30);
        return d_states.cap + (uint64_t)std::max(0.0, avail);
    }

    size_t amp_bytes() const { return precision == 0 ? 16 : 8; }
    size_t mat_scalar_bytes() const { return precision == 0 ? 8 : 4; }

    cudaEvent_t next_event() {
        if (events_used == events.size()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            events.push_back(e);
        }
        return events[events_used++];
    }
};

// Host<->device copies of a call, counted for the e2e byte figures (stats[9], [10]).
inline void h2d(Engine& E, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    unsigned char* staged = E.stage(bytes);
    std::memcpy(staged, src, bytes);
    CK(cudaMemcpyAsync(dst, staged, bytes, cudaMemcpyHostToDevice, E.stream));
    E.stats[9] += (double)bytes;
}
inline void d2h(Engine& E, void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, E.stream));
    CK(cudaStreamSynchronize(E.stream));
    E.stats[10] += (double)bytes;
}

// ---------------------------------------------------------------------------
namespace {

// Global-phase normalisation of a fused 2x2 matrix (m00, m01, m10, m11 as
// re/im pairs): multiply by e^{-i arg m00} so that m00 is real and >= 0.
// Probabilities and Pauli expectations do not see global phases, and a real
// m00 lets the kernel's 2x2 update use 14 FP64 instructions per amplitude
// pair instead of 16.  Returns the removed phase arg(m00).
double normalise_phase(double* m) {
    const double r = std::hypot(m[0], m[1]);
    if (r == 0.0) return 0.0;
    const double c = m[0] / r, s = m[1] / r;   // e^{i theta}
    for (int e = 2; e < 8; e += 2) {
        const double re = m[e], im = m[e + 1];
        m[e] = re * c + im * s;                 // (re + i im) e^{-i theta}
        m[e + 1] = im * c - re * s;
    }
    m[0] = r;
    m[1] = 0.0;
    return std::atan2(s, c);
}

struct Request {   // one qv_execute call, validated
    const qv_circuits* c;
    const qv_results* r;
    int n;
    int64_t C;
};

void validate(const Request& q) {
    const qv_circuits* c = q.c;
    if (c->n_qubits < 1 || c->n_qubits > kMaxQubits) throw ArgError("n_qubits must be in 1.." + std::to_string(kMaxQubits));
    if (c->n_circuits < 1) throw ArgError("empty batch");
    if (!c->kinds || !c->q0 || !c->q1 || !c->angles) throw ArgError("null gate arrays");
    if (!c->uniform && !c->gate_offsets) throw ArgError("gate_offsets required when uniform = 0");
    const int n = c->n_qubits;
    auto check_gate = [&](int64_t ci, uint8_t k, int32_t a, int32_t b, double ang) {
        if (k > QV_GATE_CZ) throw CircuitError(ci, "unsupported gate kind " + std::to_string(k));
        if (k == QV_GATE_MEASURE_ALL) return;
        if (a < 0 || a >= n) throw CircuitError(ci, "gate targets qubit " + std::to_string(a) + " on " + std::to_string(n) + " qubits");
        if (k == QV_GATE_CNOT || k == QV_GATE_CZ) {
            if (b < 0 || b >= n) throw CircuitError(ci, "gate targets qubit " + std::to_string(b) + " on " + std::to_string(n) + " qubits");
            if (a == b) throw CircuitError(ci, "repeated qubit index in two-qubit gate");
        }
        if ((k == QV_GATE_RY || k == QV_GATE_RZ || k == QV_GATE_RX) && !std::isfinite(ang))
            throw CircuitError(ci, "non-finite angle");
    };
    if (c->uniform) {
        if (c->n_gates < 0) throw ArgError("n_gates < 0");
        for (int64_t g = 0; g < c->n_gates; ++g) {
            const uint8_t k = c->kinds[g];
            if (k > QV_GATE_CZ || k == QV_GATE_MEASURE_ALL) { check_gate(0, k, c->q0[g], c->q1[g], 0.0); continue; }
            check_gate(0, k, c->q0[g], c->q1[g], 0.0);
            if (k == QV_GATE_RY || k == QV_GATE_RZ || k == QV_GATE_RX)
                for (int64_t ci = 0; ci < q.C; ++ci)
                    if (!std::isfinite(c->angles[ci * c->n_gates + g])) throw CircuitError(ci, "non-finite angle");
        }
    } else {
        for (int64_t ci = 0; ci < q.C; ++ci) {
            const int64_t g0 = c->gate_offsets[ci], g1 = c->gate_offsets[ci + 1];
            if (g1 < g0) throw ArgError("gate_offsets must be non-decreasing");
            for (int64_t g = g0; g < g1; ++g) check_gate(ci, c->kinds[g], c->q0[g], c->q1[g], c->angles[g]);
        }
    }
    const qv_results* r = q.r;
    if (r->kind < QV_OUT_PAULI || r->kind > QV_OUT_COUNTS) throw ArgError("unknown result kind");
    if (r->flags & ~QV_RES_TARGET_ROWS) throw ArgError("unknown result flags");
    if ((r->flags & QV_RES_TARGET_ROWS) && r->kind != QV_OUT_JS) throw ArgError("target rows are a JS option");
    const uint64_t full = n >= 64 ? ~0ull : ((1ull << n) - 1);
    if (r->kind == QV_OUT_PAULI) {
        if (!r->term_offsets || !r->xmask || !r->ymask || !r->zmask) throw ArgError("null Pauli arrays");
        for (int64_t ci = 0; ci < q.C; ++ci) {
            const int64_t t0 = r->term_offsets[ci], t1 = r->term_offsets[ci + 1];
            if (t1 < t0) throw ArgError("term_offsets must be non-decreasing");
            for (int64_t t = t0; t < t1; ++t) {
                const uint64_t x = r->xmask[t], y = r->ymask[t], z = r->zmask[t];
                if ((x | y | z) & ~full) throw CircuitError(ci, "term acts on a qubit beyond the register");
                if ((x & y) | (x & z) | (y & z)) throw ArgError("overlapping Pauli masks");
            }
        }
    } else if (r->kind == QV_OUT_SUPPORT || r->kind == QV_OUT_JS) {
        if (r->support_count < 0 || (r->support_count > 0 && !r->support)) throw ArgError("bad support");
        if (r->kind == QV_OUT_JS && r->support_count > 0 && !r->target) throw ArgError("JS needs target probabilities");
        for (int64_t s = 0; s < r->support_count; ++s) {
            if (r->support[s] & ~full) throw ArgError("support index beyond the register");
            if (s && r->support[s] <= r->support[s - 1]) throw ArgError("support must be sorted and unique");
        }
    } else if (r->kind == QV_OUT_FULL) {
        if (n > 24) throw ArgError("full distributions are limited to 24 qubits");
    } else if (r->kind == QV_OUT_COUNTS) {
        if (n > 24) throw ArgError("counts mode is limited to 24 qubits");
        if (r->shots < 1) throw ArgError("shots must be positive");
        if (!r->rng_state) throw ArgError("counts mode needs one PCG64 state per circuit");
    }
}

int64_t output_size(const qv_circuits* c, const qv_results* r) {
    switch (r->kind) {
        case QV_OUT_PAULI: return r->term_offsets ? r->term_offsets[c->n_circuits] : -1;
        case QV_OUT_SUPPORT: return (int64_t)c->n_circuits * (r->support_count + 1);
        case QV_OUT_FULL: return (int64_t)c->n_circuits << c->n_qubits;
        case QV_OUT_JS: return c->n_circuits;
        case QV_OUT_COUNTS: return r->shots > 0 ? (int64_t)c->n_circuits * (2 * r->shots + 1) : -1;
        default: return -1;
    }
}

template <typename F>
void parallel_for(int64_t count, int64_t grain, F fn) {
    // a thread per `grain` items at most: spawning costs ~20 us a thread, more
    // than a small batch's whole fusion
    const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t nthr = std::min<int64_t>(std::min<int64_t>(hw, 16), std::max<int64_t>(1, count / std::max<int64_t>(1, grain)));
    if (nthr <= 1) { for (int64_t i = 0; i < count; ++i) fn(i); return; }
    std::vector<std::thread> th;
    std::atomic<int64_t> next(0);
    for (int64_t t = 0; t < nthr; ++t)
        th.emplace_back([&]() {
            for (;;) {
                const int64_t i0 = next.fetch_add(8);
                if (i0 >= count) break;
                for (int64_t i = i0; i < std::min(count, i0 + 8); ++i) fn(i);
            }
        });
    for (auto& t : th) t.join();
}

}  // namespace

// ---------------------------------------------------------------------------
struct GroupRun {
    Engine& E;
    const Request& q;
    CachedPlan& cp;
    std::vector<int64_t> circuits;          // batch indices in this topology group
    std::vector<const double*> angle_rows;  // per circuit, indexed by topology gate
    double* out;                            // caller output

    // unique states
    std::vector<int64_t> uniq_of;            // per circuit -> unique id
    std::vector<int64_t> uniq_rep;           // unique -> representative circuit (local index)
    std::vector<double> hmats;               // [C][slots*8] double
    size_t slots8 = 0;

    template <typename T>
    void run();
};

template <typename T>
using PassFn = void (*)(const PassDesc, const GroupDesc*, const LaunchEntry*, int, int, EpiArgs);

template <typename T, int... TBs>
constexpr std::array<PassFn<T>, sizeof...(TBs)> pass_table(std::integer_sequence<int, TBs...>) {
    return {{&pass_kernel<T, TBs, 0>...}};
}
// TB = tile bits - 4: 0..8 for complex128 (k <= 12), 0..9 for complex64 (k <= 13)
template <typename T>
const std::array<PassFn<T>, 10>& pass_kernels() {
    static const std::array<PassFn<T>, 10> table = pass_table<T>(std::make_integer_sequence<int, 10>{});
    return table;
}
template <typename T>
constexpr int multi_tile_tb() {
    return max_tile_bits(sizeof(T) == 8 ? 0 : 1) - reg_bits(sizeof(T) == 8 ? 0 : 1);
}
// multi-tile launches (widest tile): deferred stores / shift-pair epilogue
template <typename T>
PassFn<T> pass_kernel_multi(bool pair) {
    return pair ? &pass_kernel<T, multi_tile_tb<T>(), 2> : &pass_kernel<T, multi_tile_tb<T>(), 1>;
}

// TMA pass kernel: stages in flight per CTA (one CTA per SM).  complex128
// tiles are 64 KiB (3 stages), complex64 tiles 32 KiB (5 stages).
template <typename T>
constexpr int tma_stages() {   // 64 KiB tiles: 3 stages, 32 KiB: 5
    return (sizeof(typename Cx<T>::V) << max_tile_bits(sizeof(T) == 8 ? 0 : 1)) >= 65536 ? 3 : 5;
}
typedef void (*TmaFn)(const CUtensorMap, const PassDesc, const TmaArgs, const GroupDesc*, const LaunchEntry*, int,
                      int64_t);
// Compute teams per CTA (QVB200_TMA_TEAMS = 1 or 2, default 2).
int tma_teams() {
    static const int t = getenv("QVB200_TMA_TEAMS") ? std::max(1, std::min(2, atoi(getenv("QVB200_TMA_TEAMS")))) : 2;
    return t;
}
// The last register group writes the tile back in the TMA box layout for one
// bulk-tensor store (default), or stores its registers straight to HBM
// (QVB200_TMA_DIRECT=1, two teams).  Same arithmetic, same results.
// Measured on B200, 28q x 8L gradient: bulk stores 32.9-33.2 s, direct
// register stores 36.7-36.9 s (the stage turnaround they save costs less
// than 16 st.global.v2.f64 per thread per tile from the compute warps).
bool tma_direct() {
    static const bool d = getenv("QVB200_TMA_DIRECT") && std::string(getenv("QVB200_TMA_DIRECT")) == "1";
    return d;
}
// Two teams: the thread of the team that stored a stage reloads it (complex128
// default), or a producer warpgroup does (complex64 default); QVB200_TMA_PWG =
// 0 / 1 forces either.  Measured on B200: 28q x 8L complex128 gradient 33.3-
// 33.6 s (team thread) vs 34.4-35.2 s (producer warpgroup: both teams then
// run their groups in phase); 32q x 4L complex64 6.55-6.72 s vs 6.39 s.
bool tma_pwg(int precision) {
    static const char* env = getenv("QVB200_TMA_PWG");
    if (env) return std::string(env) == "1";
    return precision == 1;
}
// QVB200_TMA_ALT=1: the two teams take turns on the FP64 pipe (producer
// -- measured).
bool tma_cmats() {
    static const bool c = !(getenv("QVB200_TMA_CMATS") && std::string(getenv("QVB200_TMA_CMATS")) == "0");
    return c;
}
bool tma_alt() {
    static const bool a = getenv("QVB200_TMA_ALT") && std::string(getenv("QVB200_TMA_ALT")) == "1";
    return a;
}
template <typename T>
TmaFn tma_kernel(int teams, bool direct, bool pwg, bool alt, bool cm = false) {
    constexpr int ST = tma_stages<T>();
    constexpr int TBI = multi_tile_tb<T>();
    if constexpr (TBI != 8) {   // 8 K-amplitude tiles: one 512-thread team + the producer warp, or two
                                // 256-thread teams holding two register groups per thread
        if (teams == 1) return &tma_pass_kernel<T, TBI, ST, 1, false, false, false>;
        return cm ? &tma_pass_kernel<T, TBI, ST, 2, false, false, false, true>
                  : &tma_pass_kernel<T, TBI, ST, 2, false, false, false>;
    } else {
        if (teams == 1) return &tma_pass_kernel<T, 8, ST, 1, false, false, false>;
        if (direct)
            return alt ? &tma_pass_kernel<T, 8, ST, 2, true, false, true> : &tma_pass_kernel<T, 8, ST, 2, true, false, false>;
        if (pwg)
            return alt ? &tma_pass_kernel<T, 8, ST, 2, false, true, true> : &tma_pass_kernel<T, 8, ST, 2, false, true, false>;
        return alt ? &tma_pass_kernel<T, 8, ST, 2, false, false, true> : &tma_pass_kernel<T, 8, ST, 2, false, false, false>;
    }
}
constexpr size_t kTmaSmemCap = 226 * 1024;   // 227 KiB per block less the kernel's static stage table

template <typename T>
void set_kernel_attributes() {
    for (auto fn : pass_kernels<T>())
        CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (bool pair : {false, true})
        CK(cudaFuncSetAttribute(pass_kernel_multi<T>(pair), cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    for (int teams : {1, 2})
        for (bool direct : {false, true})
            for (bool pwg : {false, true})
                for (bool alt : {false, true})
                    for (bool cm : {false, true})
                        CK(cudaFuncSetAttribute(tma_kernel<T>(teams, direct, pwg, alt, cm),
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmemCap));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, []() {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// The state slots of a run (trunk / Psi0 / work states): one allocation, so
// one tensor map per pass covers every state of a launch.
struct StateArena {
    const unsigned char* base = nullptr;
    uint64_t state_bytes = 0;
    int64_t slots = 0;
};

// QVB200_TMA=0 disables the TMA kernel (A/B measurements; the arithmetic, and
// so every result, is the same either way).
bool tma_enabled() {
    static const bool on = !(getenv("QVB200_TMA") && std::string(getenv("QVB200_TMA")) == "0");
    return on;
}

// QVB200_LAUNCH_LOG=<file>: append one line per pass launch of every call
// (kernel, first matrix slot, matrices, states, tiles, ms, algorithmic bytes)
// -- the per-pass roofline breakdown in profiles/ comes from this.
void log_launches(Engine& E) {
    static const char* path = getenv("QVB200_LAUNCH_LOG");
    if (!path) return;
    FILE* f = fopen(path, "a");
    if (!f) return;
    for (auto& t : E.timed) {
        float x = 0.f;
        cudaEventElapsedTime(&x, t.start, t.stop);
        fprintf(f, "%s %d %d %d %lld %.6f %.0f\n", t.tma ? "tma" : "pass", t.m0, t.nm, t.nstates,
                (long long)t.ntiles, x, t.bytes);
    }
    fclose(f);
}

// Launches one pass over a batch of states; `bytes` = its algorithmic HBM
// traffic (stats[4]; stats[14] / [15] = time and bytes of TMA launches).
template <typename T>
void launch_pass(Engine& E, const PassDesc& pd, const GroupDesc* d_groups, const LaunchEntry* d_ent, int nstates,
                 int64_t ntiles, const EpiArgs& ep, bool generated, const TmaLayout* tl = nullptr,
                 const StateArena* arena = nullptr, double bytes = 0.0) {
    typedef typename Cx<T>::V V;
    const int tb = pd.k - reg_bits(sizeof(T) == 8 ? 0 : 1);
    const bool multi = ntiles > 1 && tb == multi_tile_tb<T>();
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, E.device));
    cudaEvent_t e0 = E.next_event(), e1 = E.next_event();
    // ---- TMA kernel: pure store passes of multi-tile states -----------------
    const size_t tile_bytes = sizeof(V) << pd.k;
    const size_t mat_bytes = (size_t)pd.nm * 4 * sizeof(V);
    constexpr int ST = tma_stages<T>();
    const int teams = tma_teams();
    const bool direct = teams > 1 && multi_tile_tb<T>() == 8 && tma_direct();
    const bool pwg = teams > 1 && multi_tile_tb<T>() == 8 && !direct && tma_pwg(E.precision);
    const bool alt = teams > 1 && multi_tile_tb<T>() == 8 && tma_alt();
    const int team_threads = teams == 1 ? (1 << multi_tile_tb<T>()) : 256;
    const size_t tmat_off = (TmaSmem<ST>::bytes((uint32_t)tile_bytes, pd.ng, team_threads) + 127) & ~(size_t)127;
    const size_t ent_off = tmat_off + (direct ? 4 * mat_bytes : 0);
    const size_t tma_smem = ent_off + (size_t)nstates * 3 * sizeof(uint64_t);
    if (tl && tl->ok && arena && arena->base && multi && tb == multi_tile_tb<T>() && ep.flags == F_STORE &&
        !generated && pd.ng >= 1 && mat_bytes <= (size_t)kTmaMatBytes && tma_smem <= kTmaSmemCap && tma_enabled() &&
        encode_tiled()) {
        TmaArgs ta;
        std::memset(&ta, 0, sizeof(ta));
        ta.ndim = tl->ndim;
        const int elems0 = sizeof(V) / 8;   // 8-byte tensor elements per amplitude
        cuuint64_t gdim[5], gstride[4];
        cuuint32_t box[5], estride[5] = {1, 1, 1, 1, 1};
        for (int d = 0; d < tl->ndim; ++d) {
            ta.lo[d] = tl->lo[d];
            ta.cmask[d] = (uint32_t)((1ull << tl->span[d]) - 1);
            gdim[d] = (cuuint64_t)1 << tl->span[d];
            box[d] = 1u << tl->box[d];
            if (d > 0) gstride[d - 1] = ((cuuint64_t)sizeof(V)) << tl->lo[d];
        }
        gdim[0] *= elems0;
        box[0] *= elems0;
        // QVB200_TMA_PIECES = 2 / 4 moves a tile as that many boxes along its
        // outermost box dimension, so a stage's store read-out and the next
        // load overlap piece by piece.  Measured on B200: 28q x 8L gradient
        // 33.66 s (4 pieces) vs 33.69 s (1), 32q x 4L complex64 7.62 s vs
        // 6.70 s -- whole-tile boxes by default.
        static const int max_pieces = getenv("QVB200_TMA_PIECES") ? std::max(1, atoi(getenv("QVB200_TMA_PIECES"))) : 1;
        int pieces = 1;
        if (tl->ndim > 1)
            while (pieces < max_pieces && pieces * 2 <= (int)box[tl->ndim - 1] && pieces * 2 <= 4) pieces *= 2;
        box[tl->ndim - 1] /= pieces;
        ta.elems0 = elems0;
        gdim[tl->ndim] = (cuuint64_t)arena->slots;
        box[tl->ndim] = 1;
        gstride[tl->ndim - 1] = arena->state_bytes;
        for (int d = tl->ndim + 1; d < 5; ++d) {
            gdim[d] = 1;
            box[d] = 1;
            gstride[d - 1] = arena->state_bytes * (cuuint64_t)arena->slots;
        }
        CUtensorMap tmap;
        const CUresult rc = encode_tiled()(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, (void*)arena->base, gdim, gstride,
                                           box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (rc != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)rc) + ")");
        for (int j = 0; j < 16; ++j) {
            ta.wcombo[j] = tl->wcombo[j];
            ta.gwcombo[j] = tl->gwcombo[j];
        }
        for (int m = 0; m < 9; ++m) {
            ta.wtcol[m] = tl->wtcol[m];
            ta.gwtcol[m] = tl->gwtcol[m];
        }
        for (int m = 0; m < 9; ++m) ta.flam[m] = tl->flam[m];
        for (int r = 0; r < 4; ++r) ta.fmu[r] = tl->fmu[r];
        ta.tmat_off = (uint32_t)tmat_off;
        ta.ent_off = (uint32_t)ent_off;
        ta.pieces = pieces;
        ta.piece_step = (int32_t)box[tl->ndim - 1];
        ta.base = arena->base;
        ta.state_bytes = arena->state_bytes;
        ta.tile_bytes = (uint32_t)tile_bytes;
        ta.mat_bytes = (uint32_t)mat_bytes;
        const int64_t items = ntiles * nstates;
        if (items >= (1ll << 31)) throw ArgError("launch has too many (state, tile) items");
        const int64_t blocks = std::min<int64_t>(items, sms);
        ta.trace = nullptr;
#ifdef QV_TMA_TRACE
        // trace the QVB200_TMA_TRACE_LAUNCH-th TMA launch of the process into
        // $QVB200_TMA_TRACE (raw int64: a header, then the clock table)
        static int tma_launch_no = 0;
        static const int want = getenv("QVB200_TMA_TRACE_LAUNCH") ? atoi(getenv("QVB200_TMA_TRACE_LAUNCH")) : 5;
        long long* d_trace = nullptr;
        const size_t trace_n = (size_t)kTraceCtas * 2 * kTraceItems * 16;
        const bool do_trace = getenv("QVB200_TMA_TRACE") && tma_launch_no++ == want;
        if (do_trace) {
            CK(cudaMalloc(&d_trace, trace_n * sizeof(long long)));
            CK(cudaMemsetAsync(d_trace, 0, trace_n * sizeof(long long), E.stream));
            ta.trace = d_trace;
        }
#endif
        // complex64 two-team launches read their matrices from constant
        // memory when the launch's tables fit (QVB200_TMA_CMATS=0 disables)
        const size_t cm_bytes = (size_t)nstates * pd.nm * (QV_TMA_PACKED ? kPackedMatBytes : 4 * sizeof(V));
        const bool cm = multi_tile_tb<T>() != 8 && teams == 2 && tma_cmats() && cm_bytes <= (size_t)kTmaConstBytes;
        if (cm) {
            V* stage = reinterpret_cast<V*>(E.d_cstage.get(kTmaConstBytes / sizeof(double)));
            if (QV_TMA_PACKED)
                gather_cmats_packed_kernel<<<(unsigned)nstates, 64, 0, E.stream>>>(d_ent, pd.m0, pd.nm,
                                                                                 reinterpret_cast<float2*>(stage));
            else
                gather_cmats_kernel<V><<<(unsigned)nstates, 64, 0, E.stream>>>(d_ent, pd.m0, pd.nm, stage);
            CK(cudaGetLastError());
            CK(cudaMemcpyToSymbolAsync(c_tma_mats, stage, cm_bytes, 0, cudaMemcpyDeviceToDevice, E.stream));
            E.stats[0] += 1;
        }
        CK(cudaEventRecord(e0, E.stream));
        tma_kernel<T>(teams, direct, pwg, alt, cm)<<<(unsigned)blocks, tma_threads(teams, pwg, multi_tile_tb<T>()), tma_smem, E.stream>>>(
            tmap, pd, ta, d_groups, d_ent, nstates, ntiles);
        CK(cudaGetLastError());
#ifdef QV_TMA_TRACE
        if (do_trace) {
            std::vector<long long> h(trace_n);
            CK(cudaStreamSynchronize(E.stream));
            CK(cudaMemcpy(h.data(), d_trace, trace_n * sizeof(long long), cudaMemcpyDeviceToHost));
            cudaFree(d_trace);
            if (FILE* f = fopen(getenv("QVB200_TMA_TRACE"), "wb")) {
                const long long hdr[8] = {pd.nm, pd.ng, nstates, (long long)ntiles, blocks, teams, ta.pieces, kTraceItems};
                fwrite(hdr, sizeof(long long), 8, f);
                fwrite(h.data(), sizeof(long long), h.size(), f);
                fclose(f);
            }
        }
#endif
        CK(cudaEventRecord(e1, E.stream));
        E.timed.push_back({e0, e1, true, bytes, pd.m0, pd.nm, nstates, ntiles});
        E.stats[0] += 1;
        E.stats[4] += bytes;
        E.stats[12] += 1;
        E.stats[15] += bytes;
        E.stats[11] += (double)nstates * (double)ntiles * (double)(1ll << pd.k) * 14.0 * pd.nm;
        return;
    }
    // ---- pass_kernel ---------------------------------------------------------
    const size_t smem = tile_bytes + (size_t)pd.ng * sizeof(GroupDesc) + (size_t)pd.nm * 4 * sizeof(V) +
                        32 * sizeof(double) + (multi ? 8192 : 0);
    const int threads = pass_threads(tb);
    PassFn<T> fn = multi ? pass_kernel_multi<T>((ep.flags & F_PAIR) != 0) : pass_kernels<T>()[tb];
    // persistent CTAs: enough per state to fill every SM at full occupancy
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
    per_sm = std::max(per_sm, 1);
    const int64_t slots = (int64_t)per_sm * sms;
    const int64_t blocks = std::min<int64_t>(ntiles * nstates, slots);   // exactly one persistent wave
    if (ntiles * nstates + 4 * blocks >= (1ll << 31)) throw ArgError("launch has too many (state, tile) items");
    EpiArgs e2 = ep;
    e2.ntiles = ntiles;
    CK(cudaEventRecord(e0, E.stream));
    fn<<<(unsigned)blocks, threads, smem, E.stream>>>(pd, d_groups, d_ent, nstates, 0, e2);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, E.stream));
    E.timed.push_back({e0, e1, false, bytes, pd.m0, pd.nm, nstates, ntiles});
    E.stats[0] += 1;
    E.stats[4] += bytes;
    // algorithmic FP64/FP32 work: 2^(n-1) pairs x 28 flops per fused 2x2
    // matrix (a |0> input only computes tile 0 of a multi-tile state)
    const double amps = generated ? (double)(1ll << pd.k) : (double)ntiles * (double)(1ll << pd.k);
    E.stats[11] += (double)nstates * amps * 14.0 * pd.nm;
}

// Support indices bucketed by the tile of the last pass that holds them
// (CSR over tiles) with their logical local index inside the tile; sets
// ep.sup_off / sup_local / sup_pos.  Requires ep.S and ep.ntiles.
// Indices with a bit outside `reach` are left out (their amplitude is 0).
void upload_support_csr(Engine& E, const PassDesc& last, const uint64_t* support, EpiArgs& ep,
                        uint64_t reach = ~0ull) {
    const int64_t ntiles = ep.ntiles, S = ep.S;
    std::vector<int32_t> cnt(ntiles + 1, 0), local(S), tile_of(S, -1);
    for (int64_t s = 0; s < S; ++s) {
        const uint64_t g = support[s];
        if (g & ~reach) continue;
        uint32_t loc = 0;
        uint64_t tl = 0;
        for (int j = 0; j < last.k; ++j)
            if ((g >> last.sbits[j]) & 1) loc |= 1u << j;
        for (int j = 0; j < last.n_outer; ++j)
            if ((g >> last.obits[j]) & 1) tl |= 1ull << j;
        local[s] = (int32_t)loc;
        tile_of[s] = (int32_t)tl;
        cnt[tl + 1]++;
    }
    for (int64_t t = 0; t < ntiles; ++t) cnt[t + 1] += cnt[t];
    std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1), sl(S), sp(S);
    for (int64_t s = 0; s < S; ++s) {
        if (tile_of[s] < 0) continue;
        const int32_t at = fill[tile_of[s]]++;
        sl[at] = local[s];
        sp[at] = (int32_t)s;
    }
    int32_t* doff = E.d_sup_off.get(ntiles + 1);
    int32_t* dloc = E.d_sup_local.get(S);
    int32_t* dpos = E.d_sup_pos.get(S);
    h2d(E, doff, cnt.data(), (ntiles + 1) * 4);
    if (S > 0) {
        h2d(E, dloc, sl.data(), S * 4);
        h2d(E, dpos, sp.data(), S * 4);
    }
    ep.sup_off = doff;
    ep.sup_local = dloc;
    ep.sup_pos = dpos;
}

template <typename T>
void GroupRun::run() {
    typedef typename Cx<T>::V V;
    const Plan& plan = cp.plan;
    const Topology& topo = cp.topo;
    const int n = q.n;
    const int64_t C = (int64_t)circuits.size();
    const int slots = plan.n_slots();
    slots8 = (size_t)slots * 8;
    const qv_results* R = q.r;
    const bool rows = R->kind == QV_OUT_JS && (R->flags & QV_RES_TARGET_ROWS);
    const int P = (int)plan.pdesc.size();

    // 1. fused matrices per circuit (host, FP64)
    hmats.assign((size_t)C * slots8, 0.0);
    // Circuits in chunks of 16, in batch order: a slot whose gates carry the
    // same angles (bit for bit) as in the previous circuit of the chunk copies
    // that circuit's matrix -- a shift table changes one angle per circuit, so
    // most slots skip the trig and the products.  One thread per >= 64 K gates.
    const int64_t gates = std::max<int64_t>(1, (int64_t)topo.kind.size());
    const int64_t chunk = 16, nchunks = (C + chunk - 1) / chunk;
    parallel_for(nchunks, std::max<int64_t>(1, 65536 / (gates * chunk)), [&](int64_t ch) {
        for (int64_t i = ch * chunk; i < std::min(C, (ch + 1) * chunk); ++i) {
            double* m = hmats.data() + (size_t)i * slots8;
            const bool has_prev = i > ch * chunk;
            for (int sl = 0; sl < slots; ++sl) {
                bool same = has_prev;
                if (same)
                    for (int32_t ref : plan.ops[plan.mat_op[sl]].gates)
                        if (ref >= 0 && std::memcmp(&angle_rows[i][ref], &angle_rows[i - 1][ref], sizeof(double))) {
                            same = false;
                            break;
                        }
                if (same) {
                    std::memcpy(m + (size_t)sl * 8, m - slots8 + (size_t)sl * 8, 8 * sizeof(double));
                } else {
                    slot_matrix_with_pauli(plan, topo, angle_rows[i], sl, -1, m + (size_t)sl * 8);
                    normalise_phase(m + (size_t)sl * 8);
                }
            }
        }
    });

    // 2. deduplicate identical circuits (same topology + same matrices)
    uniq_of.assign(C, -1);
    uniq_rep.clear();
    {
        std::unordered_map<uint64_t, std::vector<int64_t>> seen;
        for (int64_t i = 0; i < C; ++i) {
            const double* row = hmats.data() + (size_t)i * slots8;
            const uint64_t h = hash_words(row, slots8 * sizeof(double));
            auto& cand = seen[h];
            int64_t u = -1;
            for (int64_t j : cand) {
                if (!std::memcmp(row, hmats.data() + (size_t)uniq_rep[j] * slots8, slots8 * sizeof(double))) { u = j; break; }
            }
            if (u < 0) { u = (int64_t)uniq_rep.size(); uniq_rep.push_back(i); cand.push_back(u); }
            uniq_of[i] = u;
        }
    }
    const int64_t U = (int64_t)uniq_rep.size();
    E.stats[3] += (double)U;

    // 3. matrices of unique states on the device (precision of the state)
    std::vector<T> umats((size_t)U * slots8);
    for (int64_t u = 0; u < U; ++u) {
        const double* src = hmats.data() + (size_t)uniq_rep[u] * slots8;
        for (size_t j = 0; j < slots8; ++j) umats[(size_t)u * slots8 + j] = (T)src[j];
    }
    T* d_mats = reinterpret_cast<T*>(E.d_mats.get(std::max<size_t>(1, umats.size()) * sizeof(T)));
    if (!umats.empty()) h2d(E, d_mats, umats.data(), umats.size() * sizeof(T));

    // 4. result plumbing per unique state
    EpiArgs ep;
    std::memset(&ep, 0, sizeof(ep));
    ep.n = n;
    ep.S = (R->kind == QV_OUT_SUPPORT || R->kind == QV_OUT_JS) ? R->support_count : 0;
    std::vector<int64_t> term_off_u;     // per unique: offsets into unique-term arrays
    std::vector<int64_t> uterm_src;      // unique term -> caller term index
    if (R->kind == QV_OUT_PAULI) {
        std::vector<std::vector<int64_t>> per_u(U);
        for (int64_t i = 0; i < C; ++i) {
            const int64_t ci = circuits[i];
            for (int64_t t = R->term_offsets[ci]; t < R->term_offsets[ci + 1]; ++t) per_u[uniq_of[i]].push_back(t);
        }
        term_off_u.push_back(0);
        for (int64_t u = 0; u < U; ++u) {
            for (int64_t t : per_u[u]) uterm_src.push_back(t);
            term_off_u.push_back((int64_t)uterm_src.size());
        }
        const int64_t NTm = (int64_t)uterm_src.size();
        std::vector<uint64_t> fl(NTm), ph(NTm);
        for (int64_t j = 0; j < NTm; ++j) {
            const int64_t t = uterm_src[j];
            fl[j] = R->xmask[t] | R->ymask[t];
            ph[j] = R->ymask[t] | R->zmask[t];
        }
        uint64_t* dfl = E.d_tflip.get(NTm);
        uint64_t* dph = E.d_tphase.get(NTm);
        int64_t* dto = E.d_term_off.get(U + 1);
        if (NTm) {
            h2d(E, dfl, fl.data(), NTm * 8);
            h2d(E, dph, ph.data(), NTm * 8);
        }
        h2d(E, dto, term_off_u.data(), (U + 1) * 8);
        ep.term_off = dto;
        ep.t_flip = dfl;
        ep.t_phase = dph;
        ep.pauli_out = E.d_pauli_out.get(NTm);
    }
    if (ep.S > 0) {
        uint64_t* dsu = E.d_support.get(ep.S);
        h2d(E, dsu, R->support, ep.S * 8);
        ep.support = dsu;
        if (R->kind == QV_OUT_JS && !rows) {
            double* dta = E.d_target.get(ep.S);
            h2d(E, dta, R->target, ep.S * 8);
            ep.target = dta;
        }
    }
    // QV_RES_TARGET_ROWS: circuit i's own target row and its unique state's
    // support row; the losses are formed after the last pass (js_rows_kernel)
    double* d_trows = nullptr;
    int64_t* d_urow = nullptr;
    if (rows && ep.S > 0) {
        d_trows = E.d_target.get((size_t)C * ep.S);
        bool contiguous = true;
        for (int64_t i = 1; i < C && contiguous; ++i) contiguous = circuits[i] == circuits[0] + i;
        if (contiguous) {
            h2d(E, d_trows, R->target + (size_t)circuits[0] * ep.S, (size_t)C * ep.S * 8);
        } else {
            std::vector<double> t((size_t)C * ep.S);
            for (int64_t i = 0; i < C; ++i)
                std::memcpy(t.data() + (size_t)i * ep.S, R->target + (size_t)circuits[i] * ep.S, ep.S * 8);
            h2d(E, d_trows, t.data(), t.size() * 8);
        }
        d_urow = E.d_term_off.get(std::max<int64_t>(1, C));
        h2d(E, d_urow, uniq_of.data(), C * 8);
    }
    ep.sup_out = E.d_sup_out.get((size_t)U * (ep.S + 1));
    ep.js_out = E.d_js_out.get(rows ? std::max(U, C) : U);
    // full distributions (FULL) and the CDF rows counts mode samples from (COUNTS)
    const bool probs = R->kind == QV_OUT_FULL || R->kind == QV_OUT_COUNTS;
    if (probs) ep.full_out = E.d_full_out.get((size_t)U << n);

    const size_t state_bytes = sizeof(V) << n;
    cudaEvent_t call0 = E.next_event();
    CK(cudaEventRecord(call0, E.stream));
    if (E.stats[17] == 0.0) E.stats[17] = E.host_ms();

    if (plan.single_tile) {
        // whole register in one CTA's shared memory: one launch for the batch
        std::vector<LaunchEntry> ents(U);
        for (int64_t u = 0; u < U; ++u) ents[u] = {nullptr, nullptr, d_mats + (size_t)u * slots8, u, 0, 0};
        LaunchEntry* dent = E.d_entries.get(U);
        h2d(E, dent, ents.data(), U * sizeof(LaunchEntry));
        ep.flags = F_SINGLE;
        if (R->kind == QV_OUT_PAULI) ep.flags |= F_S_PAULI;
        if (R->kind == QV_OUT_SUPPORT || rows) ep.flags |= F_S_SUPPORT;
        if (R->kind == QV_OUT_JS && !rows) ep.flags |= F_S_JS;
        if (probs) ep.flags |= F_S_FULL;
        ep.ntiles = 1;
        if (U > 0x7fffffffll) throw ArgError("batch too large");
        launch_pass<T>(E, plan.pdesc[0], cp.d_groups.p, dent, (int)U, 1, ep, false);
        E.stats[1] += (double)U;
        E.stats[2] += (double)C;
    } else {
        const int k = plan.k;
        const int64_t ntiles = 1ll << (n - k);
        (void)k;
        const bool dist = R->kind == QV_OUT_SUPPORT || R->kind == QV_OUT_JS;
        // support-restricted outputs run every pass on its light cone only;
        // the state norm is then not swept (unitary circuits keep it at 1)
        std::vector<PassDesc> rpd(plan.pdesc.begin(), plan.pdesc.end());
        std::vector<int64_t> rtiles(P, ntiles);
        uint64_t reach = ~0ull;
        if (dist) {
            const LightCone lc = light_cone(plan, R->support, ep.S);
            for (int p = 0; p < P; ++p) {
                rpd[p] = restrict_pass(plan.pdesc[p], lc.outer_free[p], lc.fresh[p]);
                rtiles[p] = 1ll << rpd[p].n_outer;
            }
            reach = lc.reach;
        }
        const bool unit_norm = rtiles[P - 1] < ntiles;
        ep.ntiles = rtiles[P - 1];
        if (ep.S > 0) {
            upload_support_csr(E, rpd[P - 1], R->support, ep, reach);
            // support indices outside the reach are never written: zero rows first
            CK(cudaMemsetAsync(ep.sup_out, 0, (size_t)U * (ep.S + 1) * sizeof(double), E.stream));
        }
        // ---- Pauli outputs: every term evaluated read-only inside a pass.
        // Term t is assigned, from its flip mask alone (so a circuit's values
        // never depend on its batch), to sweep 0 = the state's last pass when
        // its flip bits lie in that pass's tile (nothing is stored then), else
        // to a read-only sweep over the first canonical window of tile bits
        // (low bits + a run of k - c consecutive bits, windows overlapping by
        // one bit) that holds its flip bits, else to a sweep of its own bits;
        // -1 (a per-term pauli_sweep_kernel) only when its flip bits do not
        // fit one tile.  MC-VQE's nearest-neighbour terms need at most two
        // sweeps per state instead of one state read per term.
        const bool pauli = R->kind == QV_OUT_PAULI;
        std::vector<int32_t> t_sweep;
        std::vector<uint64_t> sweep_mask;   // sweep s >= 1 -> tile bit set sweep_mask[s - 1]
        bool need_store_last = !dist;       // the final state is stored for later reads
        const int64_t NT_all = pauli ? (int64_t)uterm_src.size() : 0;
        if (pauli && NT_all * ntiles <= ((int64_t)1 << 27)) {
            const int c = tile_low_bits(E.precision);
            const uint64_t low = (1ull << c) - 1;
            uint64_t s_last = 0;
            for (int b : plan.passes[P - 1].S) s_last |= 1ull << b;
            auto fill = [&](uint64_t m) {   // pad with the lowest other bits up to k
                for (int b = 0; b < n && __builtin_popcountll(m) < k; ++b) m |= 1ull << b;
                return m;
            };
            std::vector<uint64_t> windows;
            for (int start = c; start < n; start += k - c - 1) {
                uint64_t w = low;
                for (int b = start; b < std::min(n, start + k - c); ++b) w |= 1ull << b;
                windows.push_back(fill(w));
                if (start + k - c >= n) break;
            }
            auto sweep_of = [&](uint64_t m) {
                auto it = std::find(sweep_mask.begin(), sweep_mask.end(), m);
                if (it != sweep_mask.end()) return (int32_t)(it - sweep_mask.begin()) + 1;
                sweep_mask.push_back(m);
                return (int32_t)sweep_mask.size();
            };
            t_sweep.assign(NT_all, -1);
            need_store_last = false;
            for (int64_t j = 0; j < NT_all; ++j) {
                const int64_t t = uterm_src[j];
                const uint64_t F = R->xmask[t] | R->ymask[t];
                if (!(F & ~s_last)) { t_sweep[j] = 0; continue; }
                need_store_last = true;
                int32_t sw = -1;
                for (uint64_t w : windows)
                    if (!(F & ~w)) { sw = sweep_of(w); break; }
                if (sw < 0 && __builtin_popcountll(F | low) <= k) sw = sweep_of(fill(F | low));
                t_sweep[j] = sw;
            }
        }
        const bool fused_pauli = !t_sweep.empty();
        const int n_sweeps = (int)sweep_mask.size();
        for (uint64_t m : sweep_mask) {
            rpd.push_back(readonly_pass(plan, m));
            rtiles.push_back(ntiles);
        }
        if (fused_pauli) {
            // per term: flip / phase masks in the tile bits of its sweep's pass
            std::vector<uint32_t> fslot(NT_all, 0), phloc(NT_all, 0);
            std::vector<uint64_t> phout(NT_all, 0);
            for (int64_t j = 0; j < NT_all; ++j) {
                if (t_sweep[j] < 0) continue;
                const PassDesc& pd = t_sweep[j] == 0 ? rpd[P - 1] : rpd[P - 1 + t_sweep[j]];
                const int64_t t = uterm_src[j];
                const uint64_t F = R->xmask[t] | R->ymask[t], PH = R->ymask[t] | R->zmask[t];
                uint32_t fl = 0, pl = 0;
                uint64_t in_tile = 0;
                for (int q = 0; q < pd.k; ++q) {
                    in_tile |= 1ull << pd.sbits[q];
                    if ((F >> pd.sbits[q]) & 1) fl |= 1u << q;
                    if ((PH >> pd.sbits[q]) & 1) pl |= 1u << q;
                }
                fslot[j] = apply_cols(pd.fin, pd.k, fl);
                phloc[j] = pl;
                phout[j] = PH & ~in_tile;
            }
            int32_t* dsw = E.d_tsweep.get(NT_all);
            uint32_t* dfs = E.d_tfslot.get(NT_all);
            uint32_t* dpl = E.d_tphloc.get(NT_all);
            uint64_t* dpo = E.d_tphout.get(NT_all);
            h2d(E, dsw, t_sweep.data(), NT_all * 4);
            h2d(E, dfs, fslot.data(), NT_all * 4);
            h2d(E, dpl, phloc.data(), NT_all * 4);
            h2d(E, dpo, phout.data(), NT_all * 8);
            ep.t_sweep = dsw;
            ep.t_fslot = dfs;
            ep.t_phloc = dpl;
            ep.t_phout = dpo;
            ep.pauli_partial = E.d_partial2.get((size_t)std::max<int64_t>(1, NT_all * ntiles));
        }
        const bool need_state_out = need_store_last;   // full distributions / unfused Pauli terms read the stored state

        // pass signatures per unique state
        std::vector<std::vector<uint64_t>> sig(U, std::vector<uint64_t>(P));
        for (int64_t u = 0; u < U; ++u)
            for (int p = 0; p < P; ++p)
                sig[u][p] = hash_words(umats.data() + (size_t)u * slots8 + (size_t)plan.pdesc[p].m0 * 8,
                                  (size_t)plan.pdesc[p].nm * 8 * sizeof(T), 0x9e3779b97f4a7c15ull + p);
        auto same_pass = [&](int64_t a, int64_t b, int p) {
            if (sig[a][p] != sig[b][p]) return false;
            const size_t off = (size_t)plan.pdesc[p].m0 * 8, len = (size_t)plan.pdesc[p].nm * 8 * sizeof(T);
            return !std::memcmp(umats.data() + (size_t)a * slots8 + off, umats.data() + (size_t)b * slots8 + off, len);
        };

        // memory: trunk + W work states
        const bool need_trunk = P > 1 && U > 1;
        const uint64_t avail_states = E.state_budget() / state_bytes;
        if (avail_states < (need_trunk ? 2u : 1u))
            throw ArgError("a " + std::to_string(n) + "-qubit state (" + std::to_string(state_bytes >> 20) +
                           " MiB) does not fit the memory budget");
        int64_t W = (int64_t)avail_states - (need_trunk ? 1 : 0);
        W = std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(W, 64), U));
        unsigned char* base = E.d_states.get((size_t)(W + (need_trunk ? 1 : 0)) * state_bytes);
        V* trunk = need_trunk ? reinterpret_cast<V*>(base) : nullptr;
        auto work = [&](int64_t b) { return reinterpret_cast<V*>(base + (size_t)((need_trunk ? 1 : 0) + b) * state_bytes); };
        double* partial = E.d_partial.get((size_t)W * ntiles);
        StateArena arena{base, state_bytes, W + (need_trunk ? 1 : 0)};

        // ---- build the whole launch schedule on the host -----------------
        enum LKind { L_PASS, L_FINAL_DIST, L_FULL, L_PAULI, L_FINAL_PAULI };
        struct L {
            LKind kind;
            int pass;
            size_t off;     // entries (L_PASS) / slot pairs (L_FINAL_DIST)
            int count;      // states
            int flags;
            V* state;       // L_FULL / L_PAULI
            int64_t u, j;   // unique id / unique term (L_PASS: Pauli sweep id)
            double bytes;
        };
        std::vector<L> sched;
        std::vector<LaunchEntry> ents;
        std::vector<int64_t> slots_tab;

        auto run_chains = [&](const std::vector<int64_t>& D, int p) {
            for (size_t b0 = 0; b0 < D.size(); b0 += (size_t)W) {
                const int nb = (int)std::min<size_t>((size_t)W, D.size() - b0);
                for (int pp = p; pp < P; ++pp) {
                    const bool lastp = pp == P - 1;
                    const size_t off = ents.size();
                    for (int b = 0; b < nb; ++b) {
                        const int64_t u = D[b0 + b];
                        const void* in = pp == p ? (p == 0 ? nullptr : (const void*)trunk) : (const void*)work(b);
                        void* o = (lastp && !need_state_out) ? nullptr : (void*)work(b);
                        ents.push_back({in, o, d_mats + (size_t)u * slots8, u, b, 0});
                    }
                    int flags = F_STORE;
                    if (lastp && dist) flags = unit_norm ? F_SUPPORT : F_NORM | F_SUPPORT;
                    if (lastp && probs) flags = F_STORE | F_NORM;
                    if (lastp && fused_pauli) flags = F_MT_PAULI | (need_state_out ? F_STORE : 0);
                    // algorithmic bytes: each state's write, and its read -- except
                    // that a chain's first pass reads the shared trunk once for
                    // all nb states (the others hit it in L2)
                    const double rd = (pp == p && p == 0) ? 0.0 : (pp == p ? 1.0 / nb : 1.0);
                    const double wr = (flags & F_STORE) ? 1.0 : 0.0;
                    const double frac = (double)rtiles[pp] / (double)ntiles;
                    sched.push_back({L_PASS, pp, off, nb, flags, nullptr, 0, 0, nb * (double)state_bytes * frac * (rd + wr)});
                }
                for (int sw = 1; sw <= n_sweeps; ++sw) {   // read-only Pauli sweeps of the stored states
                    const size_t off = ents.size();
                    for (int b = 0; b < nb; ++b)
                        ents.push_back({(const void*)work(b), nullptr, d_mats + (size_t)D[b0 + b] * slots8, D[b0 + b], b, 0});
                    sched.push_back({L_PASS, P - 1 + sw, off, nb, F_MT_PAULI, nullptr, 0, sw, nb * (double)state_bytes});
                }
                if (fused_pauli) {   // every swept term of the batch: fixed-order sum over tiles
                    const size_t off = slots_tab.size();
                    int count = 0;
                    for (int b = 0; b < nb; ++b)
                        for (int64_t j = term_off_u[D[b0 + b]]; j < term_off_u[D[b0 + b] + 1]; ++j)
                            if (t_sweep[j] >= 0) { slots_tab.push_back(j); ++count; }
                    if (count) sched.push_back({L_FINAL_PAULI, 0, off, count, 0, nullptr, 0, 0, 0});
                }
                if (dist || probs) {
                    const size_t off = slots_tab.size();
                    for (int b = 0; b < nb; ++b) { slots_tab.push_back(D[b0 + b]); slots_tab.push_back(b); }
                    sched.push_back({L_FINAL_DIST, 0, off, nb, 0, nullptr, 0, 0, 0});
                    if (probs)
                        for (int b = 0; b < nb; ++b) sched.push_back({L_FULL, 0, 0, 1, 0, work(b), D[b0 + b], 0, 0});
                } else {
                    for (int b = 0; b < nb; ++b) {
                        const int64_t u = D[b0 + b];
                        for (int64_t j = term_off_u[u]; j < term_off_u[u + 1]; ++j)
                            if (!fused_pauli || t_sweep[j] < 0) sched.push_back({L_PAULI, 0, 0, 1, 0, work(b), u, j, 0});
                    }
                }
            }
        };

        std::vector<int64_t> alive(U);
        for (int64_t u = 0; u < U; ++u) alive[u] = u;
        for (int p = 0; p < P && !alive.empty(); ++p) {
            // the largest class of alive states sharing pass p stays on the trunk
            std::vector<std::vector<int64_t>> classes;
            std::unordered_map<uint64_t, std::vector<size_t>> by_sig;
            for (int64_t u : alive) {
                auto& cand = by_sig[sig[u][p]];
                bool placed = false;
                for (size_t ci : cand)
                    if (same_pass(classes[ci][0], u, p)) { classes[ci].push_back(u); placed = true; break; }
                if (!placed) { cand.push_back(classes.size()); classes.push_back({u}); }
            }
            size_t best = 0;
            for (size_t i = 1; i < classes.size(); ++i)
                if (classes[i].size() > classes[best].size()) best = i;
            if (classes[best].size() <= 1 || !need_trunk) {
                run_chains(alive, p);
                alive.clear();
                break;
            }
            std::vector<int64_t> stay = classes[best], D;
            std::vector<char> in_stay(U, 0);
            for (int64_t u : stay) in_stay[u] = 1;
            for (int64_t u : alive)
                if (!in_stay[u]) D.push_back(u);
            if (!D.empty()) run_chains(D, p);
            alive.swap(stay);
            const size_t off = ents.size();
            ents.push_back({p == 0 ? nullptr : (const void*)trunk, (void*)trunk, d_mats + (size_t)alive[0] * slots8, alive[0], 0, 0});
            sched.push_back({L_PASS, p, off, 1, F_STORE, nullptr, 0, 0,
                             (double)state_bytes * (double)rtiles[p] / (double)ntiles * ((p == 0 ? 0 : 1) + 1)});
        }
        if (!alive.empty()) throw std::runtime_error("scheduler left states unfinished");

        // ---- upload tables once, then issue every launch -----------------
        LaunchEntry* dent = E.d_entries.get(ents.size());
        h2d(E, dent, ents.data(), ents.size() * sizeof(LaunchEntry));
        int64_t* dslots = E.d_slots.get(std::max<size_t>(2, slots_tab.size()));
        if (!slots_tab.empty())
            h2d(E, dslots, slots_tab.data(), slots_tab.size() * 8);
        for (const L& l : sched) {
            if (l.kind == L_PASS) {
                EpiArgs e2 = ep;
                e2.flags = l.flags;
                e2.partial = partial;
                e2.sweep = (int)l.j;
                if (!(l.flags & F_SUPPORT)) e2.sup_off = nullptr;
                launch_pass<T>(E, rpd[l.pass], cp.d_groups.p, dent + l.off, l.count, rtiles[l.pass], e2, l.pass == 0,
                               l.pass < P ? &plan.tma[l.pass] : nullptr, &arena, l.bytes);
                if (l.pass >= P) E.stats[13] += l.count;   // read-only Pauli sweeps of whole states
                E.stats[1] += l.count;
            } else if (l.kind == L_FINAL_DIST) {
                finalize_dist_kernel<<<l.count, 1024, 0, E.stream>>>(dslots + l.off, rtiles[P - 1], partial, ep.sup_out,
                                                                     ep.S, ep.target, ep.js_out, R->kind == QV_OUT_JS && !rows,
                                                                     unit_norm);
                CK(cudaGetLastError());
                E.stats[0] += 1;
            } else if (l.kind == L_FINAL_PAULI) {
                finalize_pauli_mt_kernel<<<l.count, 256, 0, E.stream>>>(dslots + l.off, ntiles, ep.pauli_partial,
                                                                       ep.t_flip, ep.t_phase, ep.pauli_out);
                CK(cudaGetLastError());
                E.stats[0] += 1;
            } else if (l.kind == L_FULL) {
                full_probs_kernel<T><<<1184, 256, 0, E.stream>>>(l.state, 1ll << n, ep.sup_out + l.u * (ep.S + 1) + ep.S,
                                                                 ep.full_out + ((size_t)l.u << n));
                CK(cudaGetLastError());
                E.stats[0] += 1;
            } else {
                const int64_t t = uterm_src[l.j];
                const uint64_t F = R->xmask[t] | R->ymask[t], PH = R->ymask[t] | R->zmask[t];
                const int64_t count = F ? (1ll << (n - 1)) : (1ll << n);
                const int64_t per_block = std::min<int64_t>(count, 8192);
                const int64_t nblk = count / per_block;
                double2* p2 = E.d_partial2.get(std::max<int64_t>(nblk, 1 << 20));
                pauli_sweep_kernel<T><<<(unsigned)nblk, 256, 0, E.stream>>>(l.state, n, F, PH, per_block, p2);
                CK(cudaGetLastError());
                finalize_pauli_kernel<<<1, 1024, 0, E.stream>>>(p2, nblk, __builtin_popcountll(R->ymask[t]), ep.pauli_out + l.j);
                CK(cudaGetLastError());
                E.stats[0] += 2;
                E.stats[13] += 1;
            }
        }
        if (!alive.empty()) throw std::runtime_error("scheduler left states unfinished");
        E.stats[2] += (double)C * P;
    }
    // counts mode: CDF rows (sequential cumsum, numpy order), then per circuit
    // PCG64 draws -> integer histogram -> ascending (index, count) pairs
    double* d_counts = nullptr;
    const int64_t row_len = R->kind == QV_OUT_COUNTS ? 2 * R->shots + 1 : 0;
    if (R->kind == QV_OUT_COUNTS) {
        const int64_t dim = 1ll << n;
        cumsum_kernel<<<(unsigned)((U + 127) / 128), 128, 0, E.stream>>>(ep.full_out, dim, U);
        CK(cudaGetLastError());
        std::vector<int64_t> erow(C);
        std::vector<uint64_t> rng((size_t)C * 4);
        for (int64_t i = 0; i < C; ++i) {
            erow[i] = uniq_of[i];
            std::memcpy(rng.data() + 4 * i, R->rng_state + 4 * circuits[i], 4 * sizeof(uint64_t));
        }
        int64_t* d_erow = E.d_slots.get(std::max<int64_t>(2, C));
        h2d(E, d_erow, erow.data(), C * 8);
        uint64_t* d_rng = E.d_support.get(4 * C);
        h2d(E, d_rng, rng.data(), rng.size() * 8);
        d_counts = E.d_pauli_out.get((size_t)C * row_len);
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(C, (int64_t)(1ll << 30) / (dim * 4)));
        unsigned* hist = reinterpret_cast<unsigned*>(E.d_partial2.get((size_t)(chunk * dim * 4 + 15) / 16));
        for (int64_t c0 = 0; c0 < C; c0 += chunk) {
            const int64_t cc = std::min(chunk, C - c0);
            CK(cudaMemsetAsync(hist, 0, (size_t)cc * dim * 4, E.stream));
            sample_kernel<<<(unsigned)cc, 256, 0, E.stream>>>(ep.full_out, d_erow, d_rng, R->shots, dim, hist, c0);
            CK(cudaGetLastError());
            compact_counts_kernel<<<(unsigned)cc, 1024, 0, E.stream>>>(hist, dim, d_counts, row_len, c0);
            CK(cudaGetLastError());
            E.stats[0] += 2;
        }
    }
    double* d_jsrows = nullptr;
    if (rows && ep.S > 0) {
        d_jsrows = ep.js_out;
        js_rows_kernel<<<(unsigned)C, 1024, 0, E.stream>>>(ep.sup_out, d_urow, d_trows, ep.S, d_jsrows);
        CK(cudaGetLastError());
        E.stats[0] += 1;
    }
    cudaEvent_t call1 = E.next_event();
    CK(cudaEventRecord(call1, E.stream));

    // 5. results back to the caller, circuit by circuit
    CK(cudaStreamSynchronize(E.stream));
    float call_ms = 0.f;
    CK(cudaEventElapsedTime(&call_ms, call0, call1));
    E.stats[8] += call_ms;
    if (R->kind == QV_OUT_PAULI) {
        std::vector<double> vals(uterm_src.size());
        if (!vals.empty()) d2h(E, vals.data(), ep.pauli_out, vals.size() * 8);
        for (size_t j = 0; j < uterm_src.size(); ++j) out[uterm_src[j]] = vals[j];
    } else if (R->kind == QV_OUT_SUPPORT) {
        const size_t row = (size_t)ep.S + 1;
        std::vector<double> vals((size_t)U * row);
        d2h(E, vals.data(), ep.sup_out, vals.size() * 8);
        for (int64_t i = 0; i < C; ++i)
            std::memcpy(out + (size_t)circuits[i] * row, vals.data() + (size_t)uniq_of[i] * row, row * 8);
    } else if (R->kind == QV_OUT_JS && rows) {
        // an empty support leaves only the remainder term: (1 - 0)/2 ln 2
        std::vector<double> vals(C, 0.5 * 0.69314718055994530942);
        if (ep.S > 0) d2h(E, vals.data(), d_jsrows, C * 8);
        for (int64_t i = 0; i < C; ++i) out[circuits[i]] = vals[i];
    } else if (R->kind == QV_OUT_JS) {
        std::vector<double> vals(U);
        d2h(E, vals.data(), ep.js_out, U * 8);
        for (int64_t i = 0; i < C; ++i) out[circuits[i]] = vals[uniq_of[i]];
    } else if (R->kind == QV_OUT_COUNTS) {
        std::vector<double> vals((size_t)C * row_len);
        d2h(E, vals.data(), d_counts, vals.size() * 8);
        for (int64_t i = 0; i < C; ++i)
            std::memcpy(out + (size_t)circuits[i] * row_len, vals.data() + (size_t)i * row_len, row_len * 8);
    } else {
        const size_t row = (size_t)1 << n;
        std::vector<double> vals((size_t)U * row);
        d2h(E, vals.data(), ep.full_out, vals.size() * 8);
        for (int64_t i = 0; i < C; ++i)
            std::memcpy(out + (size_t)circuits[i] * row, vals.data() + (size_t)uniq_of[i] * row, row * 8);
    }
    E.stats[6] = P;
    E.stats[7] = plan.k;
}

CachedPlan& get_plan(Engine& E, Topology&& topo) {
    const std::string key = topo.key();
    auto it = E.plans.find(key);
    if (it != E.plans.end()) return *it->second;
    auto cp = std::make_unique<CachedPlan>();
    cp->plan = build_plan(topo, E.precision);
    cp->topo = std::move(topo);
    GroupDesc* d = cp->d_groups.get(std::max<size_t>(1, cp->plan.groups.size()));
    if (!cp->plan.groups.empty())
        CK(cudaMemcpy(d, cp->plan.groups.data(), cp->plan.groups.size() * sizeof(GroupDesc), cudaMemcpyHostToDevice));
    CachedPlan& ref = *cp;
    E.plans.emplace(key, std::move(cp));
    return ref;
}

void execute(Engine& E, const qv_circuits* c, const qv_results* r, double* out, int64_t out_len) {
    Request q{c, r, c ? c->n_qubits : 0, c ? c->n_circuits : 0};
    if (!c || !r || !out) throw ArgError("null argument");
    validate(q);
    const int64_t need = output_size(c, r);
    if (need < 0 || out_len < need) throw ArgError("output buffer too small: need " + std::to_string(need));
    if ((r->kind == QV_OUT_SUPPORT || r->kind == QV_OUT_JS) && r->support_count == 0) {
        // An empty support: a JS loss is the remainder term alone, (1 - 0)/2 ln 2
        // (ddcl.py:37-61 with no target entries); SUPPORT rows hold only the
        // norm, taken from a run on the one-index support {0}.
        if (r->kind == QV_OUT_JS) {
            std::memset(E.stats, 0, sizeof(E.stats));
            for (int64_t i = 0; i < c->n_circuits; ++i) out[i] = 0.5 * 0.69314718055994530942;
            return;
        }
        const uint64_t zero = 0;
        qv_results r1 = *r;
        r1.support_count = 1;
        r1.support = &zero;
        std::vector<double> tmp((size_t)c->n_circuits * 2);
        execute(E, c, &r1, tmp.data(), (int64_t)tmp.size());
        for (int64_t i = 0; i < c->n_circuits; ++i) out[i] = tmp[2 * i + 1];
        return;
    }
    CK(cudaSetDevice(E.device));
    std::memset(E.stats, 0, sizeof(E.stats));
    E.t_entry = std::chrono::steady_clock::now();
    E.events_used = 0;
    CK(cudaStreamSynchronize(E.stream));   // an earlier failed call may have copies in flight
    E.pinned_used = 0;
    E.timed.clear();
    const int n = c->n_qubits;

    auto topo_of = [&](int64_t ci) {
        Topology t;
        t.n = n;
        const int64_t g0 = c->uniform ? 0 : c->gate_offsets[ci];
        const int64_t g1 = c->uniform ? c->n_gates : c->gate_offsets[ci + 1];
        t.kind.assign(c->kinds + g0, c->kinds + g1);
        t.q0.assign(c->q0 + g0, c->q0 + g1);
        t.q1.assign(c->q1 + g0, c->q1 + g1);
        for (size_t g = 0; g < t.kind.size(); ++g)
            if (!is_two_qubit(t.kind[g])) t.q1[g] = -1;
        return t;
    };
    // group circuits by topology (a uniform batch is one group)
    std::vector<std::pair<CachedPlan*, std::vector<int64_t>>> groups;
    if (c->uniform) {
        std::vector<int64_t> all(c->n_circuits);
        for (int64_t i = 0; i < c->n_circuits; ++i) all[i] = i;
        groups.push_back({&get_plan(E, topo_of(0)), std::move(all)});
    } else {
        std::unordered_map<std::string, size_t> index;
        for (int64_t ci = 0; ci < c->n_circuits; ++ci) {
            Topology t = topo_of(ci);
            const std::string key = t.key();
            auto it = index.find(key);
            if (it == index.end()) {
                index.emplace(key, groups.size());
                groups.push_back({&get_plan(E, std::move(t)), {ci}});
            } else {
                groups[it->second].second.push_back(ci);
            }
        }
    }
    for (auto& g : groups) {
        GroupRun run{E, q, *g.first, g.second, {}, out};
        run.angle_rows.resize(g.second.size());
        for (size_t i = 0; i < g.second.size(); ++i) {
            const int64_t ci = g.second[i];
            run.angle_rows[i] = c->uniform ? c->angles + ci * c->n_gates : c->angles + c->gate_offsets[ci];
        }
        if (E.precision == 0) run.run<double>();
        else run.run<float>();
    }
    // device time of pass kernels (event pairs recorded by launch_pass; the
    // stream was synchronised when the results were copied back)
    double ms = 0, tma_ms = 0;
    for (auto& t : E.timed) {
        float x = 0.f;
        CK(cudaEventElapsedTime(&x, t.start, t.stop));
        ms += x;
        if (t.tma) tma_ms += x;
    }
    E.stats[5] = ms;
    E.stats[14] = tma_ms;
    log_launches(E);
}

// ---------------------------------------------------------------------------
// Shift pairs (qv_shift_js): Psi0 once, then one Xi_j per shifted gate, each
// branching off the unshifted trunk at the pass holding its gate and reduced
// against Psi0 in its last pass.
template <typename T>
void run_shift_pairs(Engine& E, CachedPlan& cp, const double* angles, int64_t nshift, const int64_t* gates,
                     const qv_results* R, double* out) {
    typedef typename Cx<T>::V V;
    const Plan& plan = cp.plan;
    const Topology& topo = cp.topo;
    const int n = plan.n, P = (int)plan.pdesc.size();
    if (plan.single_tile) throw ArgError("shift pairs need a register wider than one tile; use qv_execute");
    const int slots = plan.n_slots();
    const size_t slots8 = (size_t)slots * 8;
    const std::vector<int> slot_of = slot_of_gates(plan, topo);
    // pass of each slot
    std::vector<int> pass_of_slot(slots, 0);
    for (int p = 0; p < P; ++p)
        for (int s = plan.pdesc[p].m0; s < plan.pdesc[p].m0 + plan.pdesc[p].nm; ++s) pass_of_slot[s] = p;

    // matrix tables: the base circuit's slots, then per shifted gate j only
    // the matrices of the pass holding it (its chain's first pass), with the
    // Pauli inserted; every later pass of a chain reads the base table
    std::vector<double> base(slots8);
    circuit_matrices(plan, topo, angles, base.data());
    std::vector<double> theta(slots);   // removed global phase per base slot
    for (int sl = 0; sl < slots; ++sl) theta[sl] = normalise_phase(base.data() + (size_t)sl * 8);
    std::vector<double> delta(nshift);   // Xi_j's extra phase relative to Psi0 (see finalize_pair_kernel)
    std::vector<int> start_pass(nshift);
    std::vector<size_t> mod_off(nshift);
    size_t mod_len = 0;
    for (int64_t j = 0; j < nshift; ++j) {
        const int64_t g = gates[j];
        if (g < 0 || g >= (int64_t)topo.kind.size() || !is_rotation(topo.kind[g]) || slot_of[g] < 0)
            throw ArgError("gate_index " + std::to_string(g) + " is not a rotation gate of the circuit");
        start_pass[j] = pass_of_slot[slot_of[g]];
        mod_off[j] = mod_len;
        mod_len += (size_t)plan.pdesc[start_pass[j]].nm * 8;
    }
    std::vector<T> rows(slots8 + mod_len);
    for (size_t q = 0; q < slots8; ++q) rows[q] = (T)base[q];
    for (int64_t j = 0; j < nshift; ++j) {
        const int64_t g = gates[j];
        const PassDesc& pd = plan.pdesc[start_pass[j]];
        T* blk = rows.data() + slots8 + mod_off[j];
        for (size_t q = 0; q < (size_t)pd.nm * 8; ++q) blk[q] = (T)base[(size_t)pd.m0 * 8 + q];
        double m8[8];
        slot_matrix_with_pauli(plan, topo, angles, slot_of[g], (int32_t)g, m8);
        delta[j] = normalise_phase(m8) - theta[slot_of[g]];   // Psi0 conj(Xi) = z e^{-i delta}
        for (int q = 0; q < 8; ++q) blk[(size_t)(slot_of[g] - pd.m0) * 8 + q] = (T)m8[q];
    }
    T* d_mats = reinterpret_cast<T*>(E.d_mats.get(rows.size() * sizeof(T)));
    h2d(E, d_mats, rows.data(), rows.size() * sizeof(T));
    auto mats_base = [&]() { return (const void*)d_mats; };
    // kernels index matrices from the pass's first slot (e.mats + m0): point
    // the chain's first-pass entry m0 slots before its block (inside d_mats)
    auto mats_shift = [&](int64_t j) {
        return (const void*)(d_mats + slots8 + mod_off[j] - (size_t)plan.pdesc[start_pass[j]].m0 * 8);
    };

    EpiArgs ep;
    std::memset(&ep, 0, sizeof(ep));
    ep.n = n;
    ep.S = R->support_count;
    const int64_t ntiles = 1ll << (n - plan.k);
    // every pass on the support's light cone (see light_cone); the norms
    // of Psi0 and Xi are then 1 and Im<Psi0|Xi> = 0 exactly (psi+- = (Psi0 -+
    // i Xi)/sqrt2 are both unit vectors), instead of being swept
    std::vector<PassDesc> rpd(P);
    std::vector<int64_t> rtiles(P);
    const LightCone lc = light_cone(plan, R->support, ep.S);
    for (int p = 0; p < P; ++p) {
        rpd[p] = restrict_pass(plan.pdesc[p], lc.outer_free[p], lc.fresh[p]);
        rtiles[p] = 1ll << rpd[p].n_outer;
    }
    const bool unit_norm = rtiles[P - 1] < ntiles;
    ep.ntiles = rtiles[P - 1];
    uint64_t* dsu = E.d_support.get(std::max<int64_t>(1, ep.S));
    double* dta = E.d_target.get(std::max<int64_t>(1, ep.S));
    if (ep.S > 0) {
        h2d(E, dsu, R->support, ep.S * 8);
        h2d(E, dta, R->target, ep.S * 8);
        upload_support_csr(E, rpd[P - 1], R->support, ep, lc.reach);
    } else {
        std::vector<int32_t> zeros(ep.ntiles + 1, 0);
        int32_t* doff = E.d_sup_off.get(ep.ntiles + 1);
        h2d(E, doff, zeros.data(), zeros.size() * 4);
        ep.sup_off = doff;
    }
    ep.support = dsu;
    ep.target = dta;
    ep.pair_sup = E.d_pauli_out.get((size_t)std::max<int64_t>(1, nshift * ep.S * 4));
    // rows of support indices outside the reach are never written (their amplitude is 0)
    CK(cudaMemsetAsync(ep.pair_sup, 0, (size_t)std::max<int64_t>(1, nshift * ep.S * 4) * sizeof(double), E.stream));
    double* d_out = E.d_js_out.get((size_t)2 * nshift);
    double* d_delta = E.d_delta.get((size_t)nshift);
    h2d(E, d_delta, delta.data(), (size_t)nshift * sizeof(double));

    // memory: Psi0 + trunk + W work states
    const size_t state_bytes = sizeof(V) << n;
    const uint64_t avail = E.state_budget() / state_bytes;
    if (avail < 3) throw ArgError("shift pairs need three " + std::to_string(n) + "-qubit states in the memory budget");
    const int64_t W = std::max<int64_t>(1, std::min<int64_t>({(int64_t)avail - 2, (int64_t)64, nshift}));
    unsigned char* base_ptr = E.d_states.get((size_t)(W + 2) * state_bytes);
    V* psi0 = reinterpret_cast<V*>(base_ptr);
    V* trunk = reinterpret_cast<V*>(base_ptr + state_bytes);
    auto work = [&](int64_t b) { return reinterpret_cast<V*>(base_ptr + (size_t)(2 + b) * state_bytes); };
    double* partial = E.d_partial.get((size_t)W * ntiles * 4);
    StateArena arena{base_ptr, state_bytes, W + 2};

    // ---- schedule ----------------------------------------------------------
    struct L { bool pass; int p; size_t off; int count; int flags; double bytes; };
    auto frac = [&](int p) { return (double)state_bytes * (double)rtiles[p] / (double)ntiles; };   // bytes per sweep
    std::vector<L> sched;
    std::vector<LaunchEntry> ents;
    std::vector<int64_t> slots_tab;
    for (int p = 0; p < P; ++p) {   // phase 1: Psi0
        ents.push_back({p == 0 ? nullptr : (const void*)psi0, (void*)psi0, mats_base(), 0, 0, nullptr});
        sched.push_back({true, p, ents.size() - 1, 1, F_STORE, frac(p) * ((p ? 1 : 0) + 1)});
    }
    std::vector<std::vector<int64_t>> by_pass(P);
    for (int64_t j = 0; j < nshift; ++j) by_pass[start_pass[j]].push_back(j);
    int last_needed = -1;
    for (int p = 0; p < P; ++p)
        if (!by_pass[p].empty()) last_needed = p;
    for (int p = 0; p <= last_needed; ++p) {   // phase 2: branches off the trunk
        const auto& D = by_pass[p];
        for (size_t b0 = 0; b0 < D.size(); b0 += (size_t)W) {
            const int nb = (int)std::min<size_t>((size_t)W, D.size() - b0);
            for (int pp = p; pp < P; ++pp) {
                const bool lastp = pp == P - 1;
                const size_t off = ents.size();
                for (int b = 0; b < nb; ++b) {
                    const void* in = pp == p ? (p == 0 ? nullptr : (const void*)trunk) : (const void*)work(b);
                    ents.push_back({in, lastp ? nullptr : (void*)work(b), pp == p ? mats_shift(D[b0 + b]) : mats_base(),
                                    D[b0 + b], b, (const void*)psi0});
                }
                // a chain's first pass reads the shared trunk once for all nb
                // states; the pair epilogue reads Xi and Psi0 and stores nothing
                const double rd = (pp == p && p == 0) ? 0.0 : (pp == p ? 1.0 / nb : 1.0);
                sched.push_back({true, pp, off, nb, lastp ? F_PAIR : F_STORE, nb * frac(pp) * (lastp ? 2.0 : rd + 1.0)});
            }
            const size_t off = slots_tab.size();
            for (int b = 0; b < nb; ++b) { slots_tab.push_back(D[b0 + b]); slots_tab.push_back(b); }
            sched.push_back({false, 0, off, nb, 0, 0});
        }
        if (p < last_needed) {   // advance the trunk by pass p
            ents.push_back({p == 0 ? nullptr : (const void*)trunk, (void*)trunk, mats_base(), 0, 0, nullptr});
            sched.push_back({true, p, ents.size() - 1, 1, F_STORE, frac(p) * ((p ? 1 : 0) + 1)});
        }
    }
    LaunchEntry* dent = E.d_entries.get(ents.size());
    h2d(E, dent, ents.data(), ents.size() * sizeof(LaunchEntry));
    int64_t* dslots = E.d_slots.get(std::max<size_t>(2, slots_tab.size()));
    if (!slots_tab.empty()) h2d(E, dslots, slots_tab.data(), slots_tab.size() * 8);
    cudaEvent_t call0 = E.next_event();
    CK(cudaEventRecord(call0, E.stream));
    if (E.stats[17] == 0.0) E.stats[17] = E.host_ms();
    for (const L& l : sched) {
        if (l.pass) {
            EpiArgs e2 = ep;
            e2.flags = l.flags;
            e2.partial = partial;
            launch_pass<T>(E, rpd[l.p], cp.d_groups.p, dent + l.off, l.count, rtiles[l.p], e2, l.p == 0,
                           &plan.tma[l.p], &arena, l.bytes);
            E.stats[1] += l.count;
        } else {
            finalize_pair_kernel<<<l.count, 1024, 0, E.stream>>>(dslots + l.off, rtiles[P - 1], partial, ep.pair_sup,
                                                                 ep.S, ep.target, d_out, unit_norm, d_delta);
            CK(cudaGetLastError());
            E.stats[0] += 1;
        }
    }
    cudaEvent_t call1 = E.next_event();
    CK(cudaEventRecord(call1, E.stream));
    d2h(E, out, d_out, (size_t)2 * nshift * 8);
    float call_ms = 0.f;
    CK(cudaEventElapsedTime(&call_ms, call0, call1));
    E.stats[8] += call_ms;
    E.stats[2] += (double)2 * nshift * P;   // sweeps of direct, unshared simulation of the 2n circuits
    E.stats[3] += (double)nshift + 1;
    E.stats[6] = P;
    E.stats[7] = plan.k;
}

void shift_js(Engine& E, const qv_circuits* c, int64_t nshift, const int64_t* gates, const qv_results* r, double* out) {
    if (!c || !gates || !r || !out) throw ArgError("null argument");
    if (c->n_circuits != 1) throw ArgError("shift pairs take exactly one base circuit");
    if (r->kind != QV_OUT_JS) throw ArgError("shift pairs return JS losses (results->kind = QV_OUT_JS)");
    if (r->flags) throw ArgError("shift pairs take one target (no result flags)");
    if (nshift < 1) throw ArgError("no gates to shift");
    Request q{c, r, c->n_qubits, 1};
    validate(q);
    if (r->support_count == 0) {
        // an empty support: run on {0} with target 0 -- each loss is then the
        // remainder term (1 - 0)/2 ln 2 up to rounding, and the shifted gates
        // are still checked
        const uint64_t zero = 0;
        const double p0 = 0.0;
        qv_results r1 = *r;
        r1.support_count = 1;
        r1.support = &zero;
        r1.target = &p0;
        shift_js(E, c, nshift, gates, &r1, out);
        return;
    }
    CK(cudaSetDevice(E.device));
    std::memset(E.stats, 0, sizeof(E.stats));
    E.t_entry = std::chrono::steady_clock::now();
    E.events_used = 0;
    CK(cudaStreamSynchronize(E.stream));   // an earlier failed call may have copies in flight
    E.pinned_used = 0;
    E.timed.clear();
    Topology t;
    t.n = c->n_qubits;
    const int64_t g0 = c->uniform ? 0 : c->gate_offsets[0];
    const int64_t g1 = c->uniform ? c->n_gates : c->gate_offsets[1];
    t.kind.assign(c->kinds + g0, c->kinds + g1);
    t.q0.assign(c->q0 + g0, c->q0 + g1);
    t.q1.assign(c->q1 + g0, c->q1 + g1);
    for (size_t g = 0; g < t.kind.size(); ++g)
        if (!is_two_qubit(t.kind[g])) t.q1[g] = -1;
    CachedPlan& cp = get_plan(E, std::move(t));
    if (E.precision == 0) run_shift_pairs<double>(E, cp, c->angles + g0, nshift, gates, r, out);
    else run_shift_pairs<float>(E, cp, c->angles + g0, nshift, gates, r, out);
    double ms = 0, tma_ms = 0;
    for (auto& t : E.timed) {
        float x = 0.f;
        CK(cudaEventElapsedTime(&x, t.start, t.stop));
        ms += x;
        if (t.tma) tma_ms += x;
    }
    E.stats[5] = ms;
    E.stats[14] = tma_ms;
    log_launches(E);
}

}  // namespace qvb

// ---------------------------------------------------------------------------
using namespace qvb;

extern "C" {

const char* qv_version(void) { return "qvb200 0.1 sm_100a"; }

int qv_device_count(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) return 0;
    return count;
}

int64_t qv_output_size(const qv_circuits* circuits, const qv_results* results) {
    if (!circuits || !results) return -1;
    return output_size(circuits, results);
}

int qv_create(int device, int precision, uint64_t memory_budget_bytes, qv_handle* out) {
    if (!out) return QV_ERR_ARGUMENT;
    *out = nullptr;
    if (precision != QV_COMPLEX128 && precision != QV_COMPLEX64) return QV_ERR_ARGUMENT;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return QV_ERR_CUDA;
    if (device < 0 || device >= count) return QV_ERR_ARGUMENT;
    try {
        auto E = new Engine();
        E->device = device;
        E->precision = precision;
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&E->stream, cudaStreamNonBlocking));
        E->budget = memory_budget_bytes;
        set_kernel_attributes<double>();
        set_kernel_attributes<float>();
        *out = reinterpret_cast<qv_handle>(E);
        return QV_OK;
    } catch (const std::exception&) {
        return QV_ERR_CUDA;
    }
}

int qv_destroy(qv_handle h) {
    if (!h) return QV_ERR_ARGUMENT;
    Engine* E = reinterpret_cast<Engine*>(h);
    {
        std::lock_guard<std::mutex> lk(E->mu);
        cudaSetDevice(E->device);
        if (E->stream) cudaStreamSynchronize(E->stream);
        E->d_states.release(); E->d_mats.release(); E->d_entries.release(); E->d_partial.release();
        E->d_partial2.release(); E->d_sup_out.release(); E->d_js_out.release(); E->d_full_out.release();
        E->d_pauli_out.release(); E->d_target.release(); E->d_cstage.release(); E->d_support.release(); E->d_tflip.release();
        E->d_tphase.release(); E->d_term_off.release(); E->d_slots.release(); E->d_sup_off.release();
        E->d_delta.release();
        E->d_sup_local.release(); E->d_sup_pos.release(); E->d_tsweep.release(); E->d_tfslot.release();
        E->d_tphloc.release(); E->d_tphout.release();
        if (E->pinned) cudaFreeHost(E->pinned);
        E->pinned = nullptr;
        for (auto& kv : E->plans) kv.second->d_groups.release();
        for (auto e : E->events) cudaEventDestroy(e);
        if (E->stream) cudaStreamDestroy(E->stream);
    }
    delete E;
    return QV_OK;
}

int qv_execute(qv_handle h, const qv_circuits* circuits, const qv_results* results, double* out, int64_t out_len) {
    if (!h) return QV_ERR_ARGUMENT;
    Engine* E = reinterpret_cast<Engine*>(h);
    std::lock_guard<std::mutex> lk(E->mu);
    E->err.clear();
    E->err_circuit = -1;
    try {
        execute(*E, circuits, results, out, out_len);
        E->stats[16] = E->host_ms();
        return QV_OK;
    } catch (const CircuitError& e) {
        E->err = e.what();
        E->err_circuit = e.index;
        return QV_ERR_CIRCUIT;
    } catch (const ArgError& e) {
        E->err = e.what();
        return QV_ERR_ARGUMENT;
    } catch (const CudaError& e) {
        E->err = e.what();
        return QV_ERR_CUDA;
    } catch (const std::exception& e) {
        E->err = e.what();
        return QV_ERR_INTERNAL;
    }
}

int qv_shift_js(qv_handle h, const qv_circuits* base, int64_t n_shift, const int64_t* gate_index,
                const qv_results* results, double* out) {
    if (!h) return QV_ERR_ARGUMENT;
    Engine* E = reinterpret_cast<Engine*>(h);
    std::lock_guard<std::mutex> lk(E->mu);
    E->err.clear();
    E->err_circuit = -1;
    try {
        shift_js(*E, base, n_shift, gate_index, results, out);
        E->stats[16] = E->host_ms();
        return QV_OK;
    } catch (const CircuitError& e) {
        E->err = e.what();
        E->err_circuit = e.index;
        return QV_ERR_CIRCUIT;
    } catch (const ArgError& e) {
        E->err = e.what();
        return QV_ERR_ARGUMENT;
    } catch (const CudaError& e) {
        E->err = e.what();
        return QV_ERR_CUDA;
    } catch (const std::exception& e) {
        E->err = e.what();
        return QV_ERR_INTERNAL;
    }
}

// The getters read under the handle's lock (no torn reads while another
// thread's call rewrites them).  The error text stays valid until the next
// call on the handle; callers that share a handle between threads serialise
// call + getters themselves (native.py holds one lock across both).
const char* qv_last_error(qv_handle h) {
    if (!h) return "null handle";
    Engine* E = reinterpret_cast<Engine*>(h);
    std::lock_guard<std::mutex> lk(E->mu);
    return E->err.c_str();
}

int64_t qv_last_error_circuit(qv_handle h) {
    if (!h) return -1;
    Engine* E = reinterpret_cast<Engine*>(h);
    std::lock_guard<std::mutex> lk(E->mu);
    return E->err_circuit;
}

int qv_last_stats(qv_handle h, double* stats, int32_t n_stats) {
    if (!h || !stats) return QV_ERR_ARGUMENT;
    Engine* E = reinterpret_cast<Engine*>(h);
    std::lock_guard<std::mutex> lk(E->mu);
    for (int i = 0; i < n_stats && i < 18; ++i) stats[i] = E->stats[i];
    return QV_OK;
}

}  // extern "C"
