// plancheck.cpp — TEST-ONLY library (libqvb200_plan.so).
//
// Interprets a plan exactly as pass_kernel does (tile staging through the
// swizzled slot maps, register groups, CNOTs folded into the slot maps) but on
// the host with std::complex<double>, so CPU tests can check the planner's
// GF(2) bookkeeping against the oracle without a GPU.  The product library
// (libqvb200.so) does not contain this code and never calls it.
#include <algorithm>
#include <complex>
#include <cstring>
#include <exception>
#include <limits>
#include <vector>

#include "plan.hpp"

using namespace qvb;
using cd = std::complex<double>;

namespace {
Topology make_topo(int n, int64_t ng, const uint8_t* kinds, const int32_t* q0, const int32_t* q1) {
    Topology t;
    t.n = n;
    t.kind.assign(kinds, kinds + ng);
    t.q0.assign(q0, q0 + ng);
    t.q1.assign(q1, q1 + ng);
    for (int64_t g = 0; g < ng; ++g)
        if (!is_two_qubit(t.kind[g])) t.q1[g] = -1;
    return t;
}
}  // namespace

// Shared-memory slot (in amplitudes) of global index g inside the TMA box of a
// pass, computed from the layout's tensor dimensions exactly as the TMA unit
// places a box (dimension 0 fastest, each dimension's box bits packed above
// the previous ones) followed by the 128-byte swizzle of the byte address
// (16-byte chunk ^= 128-byte row mod 8).  Independent of the planner's slot
// columns, so the interpreter checks them against the hardware's layout.
static uint32_t tma_slot(const TmaLayout& tl, int precision, uint64_t g) {
    uint32_t e = 0;
    int at = 0;
    for (int d = 0; d < tl.ndim; ++d) {
        e |= (uint32_t)((g >> tl.lo[d]) & ((1ull << tl.box[d]) - 1)) << at;
        at += tl.box[d];
    }
    const int shift = precision == 0 ? 4 : 3;
    uint32_t byte = e << shift;
    byte ^= ((byte >> 7) & 7u) << 4;
    return byte >> shift;
}

// Outer offset reassembled from the tensor coordinates of a tile (what the
// TMA producer computes); must equal the tile's outer offset.
static uint64_t tma_outer(const TmaLayout& tl, uint64_t outer) {
    uint64_t r = 0;
    for (int d = 0; d < tl.ndim; ++d) {
        const uint64_t coord = (outer >> tl.lo[d]) & ((1ull << tl.span[d]) - 1);
        r |= coord << tl.lo[d];
    }
    return r;
}

// Final state of one circuit after running its plan; out = 2 * 2^n doubles.
// tma = 1 interprets every pass with a TMA layout as tma_pass_kernel does
// (load and store through the TMA box layout, the last register group
// writing in that layout); tma = 2 the same load, the last group storing
// straight to the state; tma = 0 as pass_kernel does.
// Returns the number of passes, -1 on error, -2 on a warp-locality
// violation, -3 on a TMA layout inconsistency.
static int simulate_impl(int n, int64_t n_gates, const uint8_t* kinds, const int32_t* q0, const int32_t* q1,
                         const double* angles, int precision, int max_tile_bits, double* out, int tma) {
    try {
        const Topology topo = make_topo(n, n_gates, kinds, q0, q1);
        const Plan plan = build_plan(topo, precision, max_tile_bits);
        std::vector<double> mats((size_t)plan.n_slots() * 8);
        circuit_matrices(plan, topo, angles, mats.data());
        const int R = reg_bits(precision), NA = 1 << R;
        const int k = plan.k, tb = k - R, nt = 1 << tb;
        const size_t dim = (size_t)1 << std::max(n, k);
        std::vector<cd> st(dim, cd(0, 0)), tile((size_t)1 << k);
        st[0] = 1.0;
        for (size_t p = 0; p < plan.pdesc.size(); ++p) {
            const PassDesc& pd = plan.pdesc[p];
            const TmaLayout& tl = plan.tma[p];
            const bool use_tma = tma && tl.ok;
            const int64_t ntiles = plan.single_tile ? 1 : (1ll << pd.n_outer);
            for (int64_t x = 0; x < ntiles; ++x) {
                uint64_t outer = 0;
                for (int j = 0; j < pd.n_outer; ++j)
                    if ((x >> j) & 1) outer |= 1ull << pd.obits[j];
                if (use_tma && tma_outer(tl, outer) != outer) return -3;
                for (int tid = 0; tid < nt; ++tid) {
                    uint32_t ts = 0;
                    uint64_t tg = 0;
                    for (int j = 0; j < tb; ++j)
                        if ((tid >> j) & 1) { ts ^= pd.swz[j]; tg |= 1ull << pd.sbits[j]; }
                    for (int it = 0; it < NA; ++it) {
                        const uint64_t g = outer | tg | pd.g_hi[it];
                        if (use_tma && tma_slot(tl, precision, g) != (ts ^ pd.swz_hi[it])) return -3;
                        tile[ts ^ pd.swz_hi[it]] = st[g];
                    }
                }
                const int sh = precision == 0 ? 4 : 3;   // descriptors hold byte offsets
                // warp-local segments: without a CTA barrier, every warp must touch
                // exactly the slots it touched in the previous group
                std::vector<std::vector<uint32_t>> prev_sets;
                std::vector<std::vector<cd>> groups_out(nt);
                for (int g = pd.g0; g < pd.g0 + pd.ng; ++g) {
                    const GroupDesc& G = plan.groups[g];
                    const int nwarps = (nt + 31) / 32;
                    std::vector<std::vector<uint32_t>> sets(nwarps);
                    for (int tid = 0; tid < nt; ++tid) {
                        uint32_t base = 0;
                        for (int m = 0; m < tb; ++m)
                            if ((tid >> m) & 1) base ^= G.tcol[m];
                        for (int j = 0; j < NA; ++j) sets[tid / 32].push_back(base ^ G.combo[j]);
                    }
                    for (auto& s : sets) std::sort(s.begin(), s.end());
                    if (g > pd.g0 && !G.cta_sync && sets != prev_sets) return -2;
                    prev_sets = sets;
                    for (int tid = 0; tid < nt; ++tid) {
                        uint32_t base = 0;
                        for (int m = 0; m < tb; ++m)
                            if ((tid >> m) & 1) base ^= G.tcol[m];
                        cd a[16];
                        for (int j = 0; j < NA; ++j) a[j] = tile[(base ^ G.combo[j]) >> sh];
                        for (int r = 0; r < R; ++r) {
                            if (G.mat[r] < 0) continue;
                            const double* M = mats.data() + (size_t)(pd.m0 + G.mat[r]) * 8;
                            const cd m00(M[0], M[1]), m01(M[2], M[3]), m10(M[4], M[5]), m11(M[6], M[7]);
                            for (int j = 0; j < NA; ++j) {
                                if ((j >> r) & 1) continue;
                                const cd u = a[j], v = a[j | (1 << r)];
                                a[j] = m00 * u + m01 * v;
                                a[j | (1 << r)] = m10 * u + m11 * v;
                            }
                        }
                        groups_out[tid].assign(a, a + NA);
                    }
                    // every thread has read its registers before any writes (the
                    // TMA kernel's last group writes after a compute barrier)
                    const bool last_tma = use_tma && g == pd.g0 + pd.ng - 1;
                    for (int tid = 0; tid < nt; ++tid) {
                        uint32_t base = 0, wbase = 0;
                        uint64_t gbase = 0;
                        for (int m = 0; m < tb; ++m)
                            if ((tid >> m) & 1) { base ^= G.tcol[m]; wbase ^= tl.wtcol[m]; gbase ^= tl.gwtcol[m]; }
                        for (int j = 0; j < NA; ++j) {
                            if (last_tma && tma == 2) {   // straight from registers to the state
                                st[outer | (gbase ^ tl.gwcombo[j])] = groups_out[tid][j];
                                continue;
                            }
                            const uint32_t at = last_tma ? (wbase ^ tl.wcombo[j]) : (base ^ G.combo[j]);
                            tile[at >> sh] = groups_out[tid][j];
                        }
                    }
                }
                if (use_tma && tma == 2) continue;   // the last group stored the tile
                for (int tid = 0; tid < nt; ++tid) {
                    uint32_t fs = 0;
                    uint64_t tg = 0;
                    for (int j = 0; j < tb; ++j)
                        if ((tid >> j) & 1) { fs ^= pd.fin[j]; tg |= 1ull << pd.sbits[j]; }
                    for (int it = 0; it < NA; ++it) {
                        const uint64_t g = outer | tg | pd.g_hi[it];
                        st[g] = use_tma ? tile[tma_slot(tl, precision, g)] : tile[fs ^ pd.fin_hi[it]];
                    }
                }
            }
        }
        for (size_t i = 0; i < ((size_t)1 << n); ++i) { out[2 * i] = st[i].real(); out[2 * i + 1] = st[i].imag(); }
        return (int)plan.pdesc.size();
    } catch (const std::exception&) {
        return -1;
    }
}

extern "C" {

int qvp_simulate(int n, int64_t n_gates, const uint8_t* kinds, const int32_t* q0, const int32_t* q1,
                 const double* angles, int precision, int max_tile_bits, double* out) {
    return simulate_impl(n, n_gates, kinds, q0, q1, angles, precision, max_tile_bits, out, 0);
}

int qvp_simulate_tma(int n, int64_t n_gates, const uint8_t* kinds, const int32_t* q0, const int32_t* q1,
                     const double* angles, int precision, int max_tile_bits, double* out) {
    return simulate_impl(n, n_gates, kinds, q0, q1, angles, precision, max_tile_bits, out, 1);
}

// As qvp_simulate_tma, but the last register group of a TMA pass stores its
// registers straight to the state (gwcombo / gwtcol), as tma_pass_kernel's
// default mode does.
int qvp_simulate_tma_direct(int n, int64_t n_gates, const uint8_t* kinds, const int32_t* q0, const int32_t* q1,
                            const double* angles, int precision, int max_tile_bits, double* out) {
    return simulate_impl(n, n_gates, kinds, q0, q1, angles, precision, max_tile_bits, out, 2);
}

// TMA layout of every pass: per pass 4 int64 (ok, ndim, wavefronts, ng);
// returns the pass count or -1.
int qvp_plan_tma(int n, int64_t n_gates, const uint8_t* kinds, const int32_t* q0, const int32_t* q1, int precision,
                 int max_tile_bits, int64_t* out, int32_t cap) {
    try {
        const Topology topo = make_topo(n, n_gates, kinds, q0, q1);
        const Plan plan = build_plan(topo, precision, max_tile_bits);
        for (size_t p = 0; p < plan.pdesc.size() && (int32_t)p < cap; ++p) {
            out[4 * p] = plan.tma[p].ok;
            out[4 * p + 1] = plan.tma[p].ndim;
            out[4 * p + 2] = plan.tma[p].wavefronts;
            out[4 * p + 3] = plan.pdesc[p].ng;
        }
        return (int)plan.pdesc.size();
    } catch (const std::exception&) {
        return -1;
    }
}

// Support probabilities |<s|psi>|^2 of one circuit computed on the support's
// light cone only, as the product does (light_cone / restrict_pass): pass 0
// generates |0...0> in tile 0, later passes visit only their restricted tiles
// and zero-fill their fresh slots.  Every amplitude starts as NaN, so any
// read of data the restricted passes never wrote poisons the result.
// out_probs[s] for each support index; returns the pass count or -1.
int qvp_simulate_cone(int n, int64_t n_gates, const uint8_t* kinds, const int32_t* q0, const int32_t* q1,
                      const double* angles, int precision, int max_tile_bits, const uint64_t* support,
                      int64_t S, double* out_probs, int64_t* tiles_visited) {
    try {
        const Topology topo = make_topo(n, n_gates, kinds, q0, q1);
        const Plan plan = build_plan(topo, precision, max_tile_bits);
        if (plan.single_tile) return -1;
        std::vector<double> mats((size_t)plan.n_slots() * 8);
        circuit_matrices(plan, topo, angles, mats.data());
        const LightCone lc = light_cone(plan, support, S);
        const int R = reg_bits(precision), NA = 1 << R;
        const int k = plan.k, tb = k - R, nt = 1 << tb;
        const double nan = std::numeric_limits<double>::quiet_NaN();
        std::vector<cd> st((size_t)1 << n, cd(nan, nan)), tile((size_t)1 << k);
        const int sh = precision == 0 ? 4 : 3;
        int64_t visited = 0;
        for (size_t p = 0; p < plan.pdesc.size(); ++p) {
            const PassDesc pd = restrict_pass(plan.pdesc[p], lc.outer_free[p], lc.fresh[p]);
            const int64_t ntiles = 1ll << pd.n_outer;
            visited += ntiles;
            for (int64_t x = 0; x < ntiles; ++x) {
                uint64_t outer = 0;
                for (int j = 0; j < pd.n_outer; ++j)
                    if ((x >> j) & 1) outer |= 1ull << pd.obits[j];
                for (int tid = 0; tid < nt; ++tid) {
                    uint32_t ts = 0;
                    uint64_t tg = 0;
                    for (int j = 0; j < tb; ++j)
                        if ((tid >> j) & 1) { ts ^= pd.swz[j]; tg |= 1ull << pd.sbits[j]; }
                    for (int it = 0; it < NA; ++it) {
                        const uint32_t local = (uint32_t)tid | ((uint32_t)it << tb);
                        cd v;
                        if (p == 0) v = (x == 0 && local == 0) ? cd(1, 0) : cd(0, 0);   // generated |0...0>
                        else if (local & pd.fresh) v = cd(0, 0);
                        else v = st[outer | tg | pd.g_hi[it]];
                        tile[ts ^ pd.swz_hi[it]] = v;
                    }
                }
                for (int g = pd.g0; g < pd.g0 + pd.ng; ++g) {
                    const GroupDesc& G = plan.groups[g];
                    for (int tid = 0; tid < nt; ++tid) {
                        uint32_t base = 0;
                        for (int m = 0; m < tb; ++m)
                            if ((tid >> m) & 1) base ^= G.tcol[m];
                        cd a[16];
                        for (int j = 0; j < NA; ++j) a[j] = tile[(base ^ G.combo[j]) >> sh];
                        for (int r = 0; r < R; ++r) {
                            if (G.mat[r] < 0) continue;
                            const double* M = mats.data() + (size_t)(pd.m0 + G.mat[r]) * 8;
                            const cd m00(M[0], M[1]), m01(M[2], M[3]), m10(M[4], M[5]), m11(M[6], M[7]);
                            for (int j = 0; j < NA; ++j) {
                                if ((j >> r) & 1) continue;
                                const cd u = a[j], v = a[j | (1 << r)];
                                a[j] = m00 * u + m01 * v;
                                a[j | (1 << r)] = m10 * u + m11 * v;
                            }
                        }
                        for (int j = 0; j < NA; ++j) tile[(base ^ G.combo[j]) >> sh] = a[j];
                    }
                }
                for (int tid = 0; tid < nt; ++tid) {
                    uint32_t fs = 0;
                    uint64_t tg = 0;
                    for (int j = 0; j < tb; ++j)
                        if ((tid >> j) & 1) { fs ^= pd.fin[j]; tg |= 1ull << pd.sbits[j]; }
                    for (int it = 0; it < NA; ++it) st[outer | tg | pd.g_hi[it]] = tile[fs ^ pd.fin_hi[it]];
                }
            }
        }
        for (int64_t s = 0; s < S; ++s)
            out_probs[s] = (support[s] & ~lc.reach) ? 0.0 : std::norm(st[support[s]]);
        if (tiles_visited) *tiles_visited = visited;
        return (int)plan.pdesc.size();
    } catch (const std::exception&) {
        return -1;
    }
}

int qvp_simulate_cone_tma(int n, int64_t n_gates, const uint8_t* kinds, const int32_t* q0, const int32_t* q1,
                      const double* angles, int precision, int max_tile_bits, const uint64_t* support,
                      int64_t S, double* out_probs, int64_t* tiles_visited) {
    try {
        const Topology topo = make_topo(n, n_gates, kinds, q0, q1);
        const Plan plan = build_plan(topo, precision, max_tile_bits);
        if (plan.single_tile) return -1;
        std::vector<double> mats((size_t)plan.n_slots() * 8);
        circuit_matrices(plan, topo, angles, mats.data());
        const LightCone lc = light_cone(plan, support, S);
        const int R = reg_bits(precision), NA = 1 << R;
        const int k = plan.k, tb = k - R, nt = 1 << tb;
        const double nan = std::numeric_limits<double>::quiet_NaN();
        std::vector<cd> st((size_t)1 << n, cd(nan, nan)), tile((size_t)1 << k);
        const int sh = precision == 0 ? 4 : 3;
        int64_t visited = 0;
        for (size_t p = 0; p < plan.pdesc.size(); ++p) {
            const PassDesc pd = restrict_pass(plan.pdesc[p], lc.outer_free[p], lc.fresh[p]);
            const TmaLayout& tl = plan.tma[p];
            const bool use_tma = p > 0 && tl.ok;
            const int64_t ntiles = 1ll << pd.n_outer;
            visited += ntiles;
            for (int64_t x = 0; x < ntiles; ++x) {
                uint64_t outer = 0;
                for (int j = 0; j < pd.n_outer; ++j)
                    if ((x >> j) & 1) outer |= 1ull << pd.obits[j];
                for (int tid = 0; tid < nt; ++tid) {
                    uint32_t ts = 0;
                    uint64_t tg = 0;
                    for (int j = 0; j < tb; ++j)
                        if ((tid >> j) & 1) { ts ^= pd.swz[j]; tg |= 1ull << pd.sbits[j]; }
                    for (int it = 0; it < NA; ++it) {
                        const uint32_t local = (uint32_t)tid | ((uint32_t)it << tb);
                        cd v;
                        if (p == 0) v = (x == 0 && local == 0) ? cd(1, 0) : cd(0, 0);   // generated |0...0>
                        else if ((local & pd.fresh) && !use_tma) v = cd(0, 0);
                        else v = st[outer | tg | pd.g_hi[it]];   // TMA: fresh slots load whatever is there
                        tile[ts ^ pd.swz_hi[it]] = v;
                    }
                }
                for (int g = pd.g0; g < pd.g0 + pd.ng; ++g) {
                    const GroupDesc& G = plan.groups[g];
                    for (int tid = 0; tid < nt; ++tid) {
                        uint32_t base = 0;
                        for (int m = 0; m < tb; ++m)
                            if ((tid >> m) & 1) base ^= G.tcol[m];
                        cd a[16];
                        for (int j = 0; j < NA; ++j) a[j] = tile[(base ^ G.combo[j]) >> sh];
                        if (use_tma && pd.fresh && g == pd.g0) {   // zero-fill fresh registers as read
                            uint32_t lt = 0;
                            for (int m = 0; m < tb; ++m)
                                if ((tid >> m) & 1) lt ^= tl.flam[m];
                            for (int j = 0; j < NA; ++j) {
                                uint32_t l = lt;
                                for (int r = 0; r < R; ++r)
                                    if ((j >> r) & 1) l ^= tl.fmu[r];
                                if (l & pd.fresh) a[j] = cd(0, 0);
                            }
                        }
                        for (int r = 0; r < R; ++r) {
                            if (G.mat[r] < 0) continue;
                            const double* M = mats.data() + (size_t)(pd.m0 + G.mat[r]) * 8;
                            const cd m00(M[0], M[1]), m01(M[2], M[3]), m10(M[4], M[5]), m11(M[6], M[7]);
                            for (int j = 0; j < NA; ++j) {
                                if ((j >> r) & 1) continue;
                                const cd u = a[j], v = a[j | (1 << r)];
                                a[j] = m00 * u + m01 * v;
                                a[j | (1 << r)] = m10 * u + m11 * v;
                            }
                        }
                        for (int j = 0; j < NA; ++j) tile[(base ^ G.combo[j]) >> sh] = a[j];
                    }
                }
                for (int tid = 0; tid < nt; ++tid) {
                    uint32_t fs = 0;
                    uint64_t tg = 0;
                    for (int j = 0; j < tb; ++j)
                        if ((tid >> j) & 1) { fs ^= pd.fin[j]; tg |= 1ull << pd.sbits[j]; }
                    for (int it = 0; it < NA; ++it) st[outer | tg | pd.g_hi[it]] = tile[fs ^ pd.fin_hi[it]];
                }
            }
        }
        for (int64_t s = 0; s < S; ++s)
            out_probs[s] = (support[s] & ~lc.reach) ? 0.0 : std::norm(st[support[s]]);
        if (tiles_visited) *tiles_visited = visited;
        return (int)plan.pdesc.size();
    } catch (const std::exception&) {
        return -1;
    }
}

// Plan shape: stats[0] passes, [1] groups, [2] matrix slots, [3] fused ops,
// [4] tile bits, [5] single tile, [6] groups needing a CTA barrier;
// per-pass matrices in pass_mats (if non-null, <= cap).
int qvp_plan_stats(int n, int64_t n_gates, const uint8_t* kinds, const int32_t* q0, const int32_t* q1, int precision,
                   int max_tile_bits, int64_t* stats, int32_t* pass_mats, int32_t cap) {
    try {
        const Topology topo = make_topo(n, n_gates, kinds, q0, q1);
        const Plan plan = build_plan(topo, precision, max_tile_bits);
        stats[0] = (int64_t)plan.pdesc.size();
        stats[1] = (int64_t)plan.groups.size();
        stats[2] = plan.n_slots();
        stats[3] = (int64_t)plan.ops.size();
        stats[4] = plan.k;
        stats[5] = plan.single_tile ? 1 : 0;
        int64_t syncs = 0;
        for (const GroupDesc& g : plan.groups) syncs += g.cta_sync;
        stats[6] = syncs;
        if (pass_mats)
            for (size_t p = 0; p < plan.pdesc.size() && (int32_t)p < cap; ++p) pass_mats[p] = plan.pdesc[p].nm;
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// Raw device descriptors of a plan: groups (128 B each) and passes
// (sizeof(PassDesc) each).  Returns the group count; *n_passes gets the pass count.
int qvp_plan_descriptors(int n, int64_t n_gates, const uint8_t* kinds, const int32_t* q0, const int32_t* q1,
                         int precision, int max_tile_bits, void* groups, int32_t group_cap, void* passes,
                         int32_t pass_cap, int32_t* n_passes) {
    try {
        const Topology topo = make_topo(n, n_gates, kinds, q0, q1);
        const Plan plan = build_plan(topo, precision, max_tile_bits);
        if ((int32_t)plan.groups.size() <= group_cap)
            std::memcpy(groups, plan.groups.data(), plan.groups.size() * sizeof(GroupDesc));
        if ((int32_t)plan.pdesc.size() <= pass_cap)
            std::memcpy(passes, plan.pdesc.data(), plan.pdesc.size() * sizeof(PassDesc));
        *n_passes = (int32_t)plan.pdesc.size();
        return (int)plan.groups.size();
    } catch (const std::exception&) {
        return -1;
    }
}

// Tile bit set of every pass as a bit mask (global index bits).
int qvp_plan_pass_masks(int n, int64_t n_gates, const uint8_t* kinds, const int32_t* q0, const int32_t* q1,
                        int precision, int max_tile_bits, uint64_t* masks, int32_t cap) {
    try {
        const Topology topo = make_topo(n, n_gates, kinds, q0, q1);
        const Plan plan = build_plan(topo, precision, max_tile_bits);
        for (size_t p = 0; p < plan.passes.size() && (int32_t)p < cap; ++p) {
            uint64_t m = 0;
            for (int b : plan.passes[p].S) m |= 1ull << b;
            masks[p] = m;
        }
        return (int)plan.passes.size();
    } catch (const std::exception&) {
        return -1;
    }
}

}  // extern "C"
