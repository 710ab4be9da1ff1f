// plan.cpp — see plan.hpp.
//
// Gate semantics restated from the reference kernels (pkg/src/qvirt/kernels.py):
//   H  :18-27   (a0+a1, a0-a1) * 1/sqrt(2)
//   X  :30-37   swap
//   RY :40-50   [[c,-s],[s,c]], c = cos(theta/2), s = sin(theta/2)
//   RZ :53-59   diag(exp(-i theta/2), exp(+i theta/2))
//   CNOT :62-70 swap a[i], a[i|t] where the control bit is set
// RX / CZ are extensions (not in the reference gate set, circuits.py:27-33):
//   RX = [[c,-is],[-is,c]];  CZ(a,b) = H_b CNOT(a,b) H_b.
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <string>
#include <functional>
#include <stdexcept>
#include <unordered_map>

namespace qvb {

namespace {

using cd = std::complex<double>;

inline int popcount64(uint64_t v) { return __builtin_popcountll(v); }

uint64_t op_mask(const FusedOp& op) {
    uint64_t m = 1ull << op.b0;
    if (op.cnot) m |= 1ull << op.b1;
    return m;
}

int coalesce_bits(int precision) { return precision == 0 ? 3 : 4; }  // 2^c amps = 128 B
int bank_bits(int precision) { return precision == 0 ? 3 : 4; }      // 16 B / 8 B words per 128 B row

std::vector<FusedOp> fuse(const Topology& t) {
    std::vector<FusedOp> ops;
    std::vector<int> open(kMaxQubits + 1, -1);
    const int n = t.n;
    auto add_1q = [&](int b, int32_t ref) {
        if (open[b] >= 0) {
            ops[open[b]].gates.push_back(ref);
        } else {
            open[b] = (int)ops.size();
            FusedOp op;
            op.b0 = b;
            op.gates.push_back(ref);
            ops.push_back(std::move(op));
        }
    };
    auto add_cnot = [&](int c, int tb) {
        open[c] = -1;
        open[tb] = -1;
        FusedOp op;
        op.cnot = true;
        op.b0 = c;
        op.b1 = tb;
        ops.push_back(std::move(op));
    };
    for (size_t g = 0; g < t.kind.size(); ++g) {
        const uint8_t k = t.kind[g];
        if (k == G_MEASURE) continue;
        if (k == G_CNOT) {
            add_cnot(n - 1 - t.q0[g], n - 1 - t.q1[g]);
        } else if (k == G_CZ) {
            const int a = n - 1 - t.q0[g], b = n - 1 - t.q1[g];
            add_1q(b, -1);
            add_cnot(a, b);
            add_1q(b, -1);
        } else {
            add_1q(n - 1 - t.q0[g], (int32_t)g);
        }
    }
    return ops;
}

// Greedy pass selection.  Each pass owns k index bits (always including the
// low `c` bits so every tile row is a contiguous 128 B run); it applies, in
// program order, every op whose bits lie in the pass and that does not depend
// on an op left for a later pass.  Two-qubit ops claim bits first (they are
// what forces new passes), one-qubit ops fill the remaining capacity.
std::vector<PassPlan> select_passes(int n, int k, int c, const std::vector<FusedOp>& ops) {
    std::vector<PassPlan> passes;
    std::vector<int> rem(ops.size());
    for (size_t i = 0; i < ops.size(); ++i) rem[i] = (int)i;
    const uint64_t low = (1ull << c) - 1;
    while (!rem.empty()) {
        uint64_t S = low;
        uint64_t blocked = 0;
        for (int i : rem) {
            const uint64_t bits = op_mask(ops[i]);
            if (bits & blocked) { blocked |= bits; continue; }
            if (!ops[i].cnot || !(bits & ~S)) continue;
            if (popcount64(S | bits) <= k) S |= bits;
            else blocked |= bits;
        }
        blocked = 0;
        for (int i : rem) {
            const uint64_t bits = op_mask(ops[i]);
            if (bits & blocked) { blocked |= bits; continue; }
            if (!(bits & ~S)) continue;
            if (!ops[i].cnot && popcount64(S | bits) <= k) { S |= bits; continue; }
            blocked |= bits;
        }
        for (int b = 0; b < n && popcount64(S) < k; ++b) S |= 1ull << b;
        PassPlan pp;
        std::vector<int> left;
        blocked = 0;
        for (int i : rem) {
            const uint64_t bits = op_mask(ops[i]);
            if ((bits & blocked) || (bits & ~S)) { blocked |= bits; left.push_back(i); continue; }
            pp.ops.push_back(i);
        }
        if (pp.ops.empty()) throw std::runtime_error("pass planner made no progress");
        for (int b = 0; b < n; ++b)
            if ((S >> b) & 1) pp.S.push_back(b);
        passes.push_back(std::move(pp));
        rem.swap(left);
    }
    if (passes.empty()) {  // empty circuit: one pass that applies nothing
        PassPlan pp;
        for (int b = 0; b < k; ++b) pp.S.push_back(b);
        passes.push_back(pp);
    }
    return passes;
}

// Builds the register groups of one pass.  Groups are first recorded with the
// slot map Q in force when they are applied; `emit` then splits them into
// warp-local segments and writes the device descriptors.
struct GroupBuilder {
    int k, beta;
    int rbits;             // register bits per group (reg_bits(precision))
    int amp_shift;         // log2(bytes per amplitude): 4 complex128, 3 complex64
    bool tma = false;      // TMA 128-byte swizzle instead of the full bank fold
    uint16_t col[16];      // logical-bit -> slot column (before swizzle): the map Q
    std::vector<std::pair<int, int>> open;  // (logical bit, pass-local matrix index)

    struct Pending {
        std::vector<std::pair<int, int>> ops;  // (bit, matrix)
        uint16_t col[16];                      // Q when the group is applied
        uint32_t targets_after = 0;            // CNOT targets applied before the next group
    };
    std::vector<Pending> pending;

    uint16_t swz(uint32_t v) const {   // bank swizzle, GF(2)-linear
        if (tma) {
            // TMA SWIZZLE_128B: the 16-byte chunk (byte-address bits 4-6) is
            // XORed with the 128-byte row index mod 8 (bits 7-9)
            const int chunk = 4 - amp_shift, row = 7 - amp_shift;
            return (uint16_t)(v ^ (((v >> row) & 7u) << chunk));
        }
        uint32_t r = v;   // every bit above the bank bits folds into them
        for (int j = beta; j < k; ++j)
            if ((v >> j) & 1u) r ^= 1u << (j % beta);
        return (uint16_t)r;
    }
    uint16_t phys(int b) const { return swz(col[b]); }

    void close() {
        if (open.empty()) return;
        Pending p;
        p.ops = open;
        std::memcpy(p.col, col, sizeof(col));
        pending.push_back(p);
        open.clear();
    }

    void cnot(int c, int t) {
        col[c] ^= col[t];   // Q <- Q o CNOT
        if (!pending.empty()) pending.back().targets_after |= 1u << t;
    }

    // Shared-memory bank column (16-byte chunk of a 128-byte row for
    // complex128, 8-byte word for complex64) of pre-swizzle slot column v.
    uint32_t bank(uint32_t v) const { return swz(v) & ((1u << beta) - 1); }
    static int rank_gf2(const uint32_t* v, int m) {
        uint32_t basis[16] = {0};
        int r = 0;
        for (int i = 0; i < m; ++i) {
            uint32_t x = v[i];
            for (int j = 0; j < r && x; ++j)
                if ((x ^ basis[j]) < x) x ^= basis[j];
            if (x) {
                basis[r++] = x;
                std::sort(basis, basis + r, [](uint32_t a, uint32_t b) { return a > b; });
            }
        }
        return r;
    }

    // TMA layout of the pass (init columns) and, at emit time, the inverse of
    // the final slot map Q: physical pre-swizzle column -> final logical index.
    uint16_t init[16];
    std::vector<uint32_t> qinv;

    // Best first-`beta` lanes of a group: lanes 0..beta-1 form one shared-
    // memory wavefront phase, so their bank columns should be independent;
    // for the last group of a TMA pass the same must hold for the writes in
    // the TMA layout.  Returns (score, chosen subset bitmask over `lanes`).
    // For the last group of a TMA pass the first lanes should also write one
    // contiguous 128-byte row of the output (its amplitudes go straight to
    // HBM): their final logical positions are the tile's low bits 0..c-1.
    int coalesce_bits_ = 3;
    std::pair<int, uint32_t> lane_choice(const std::vector<int>& lanes, const uint16_t* cols, bool last_tma) const {
        const int m = (int)lanes.size(), want = std::min(beta, m);
        std::pair<int, uint32_t> best{-1, 0};
        for (uint32_t sub = 0; sub < (1u << m); ++sub) {
            if (__builtin_popcount(sub) != want) continue;
            uint32_t rv[16];
            int c = 0, row = 0;
            uint32_t seen = 0;
            for (int i = 0; i < m; ++i)
                if ((sub >> i) & 1u) {
                    rv[c++] = bank(cols[lanes[i]]);
                    if (last_tma) {
                        const uint32_t l = qinv[cols[lanes[i]]];
                        if (l && !(l & (l - 1)) && l < (1u << coalesce_bits_) && !(seen & l)) { seen |= l; ++row; }
                    }
                }
            // the read banks first, then the write row
            const int score = 8 * rank_gf2(rv, c) + row;
            if (score > best.first) best = {score, sub};
        }
        return best;
    }

    // Register bits of a group (its matrices' bits, padded with bits outside
    // the warp index) and its lanes, padding chosen for the best lane score.
    struct Layout { std::vector<int> reg, lanes; uint32_t sub = 0; int score = -1; };
    Layout group_layout(const Pending& p, uint32_t wmask, bool last_tma) const {
        uint32_t used = 0;
        std::vector<int> reg;
        for (auto& pr : p.ops) { reg.push_back(pr.first); used |= 1u << pr.first; }
        std::vector<int> cand;
        for (int b = k - 1; b >= 0; --b)
            if (!((used >> b) & 1u) && !((wmask >> b) & 1u)) cand.push_back(b);
        const int need = rbits - (int)reg.size();
        Layout best;
        const int m = (int)cand.size();
        for (uint32_t sub = 0; sub < (1u << m); ++sub) {   // cand is highest-first: ties keep high pads
            if (__builtin_popcount(sub) != need) continue;
            Layout l;
            l.reg = reg;
            for (int i = 0; i < m; ++i)
                if ((sub >> i) & 1u) l.reg.push_back(cand[i]);
            uint32_t u = used;
            for (int b : l.reg) u |= 1u << b;
            for (int b = 0; b < k; ++b)
                if (!((u >> b) & 1u) && !((wmask >> b) & 1u)) l.lanes.push_back(b);
            auto lc = lane_choice(l.lanes, p.col, last_tma);
            l.score = lc.first;
            l.sub = lc.second;
            if (l.score > best.score) best = l;
            if (need == 0) break;
        }
        return best;
    }

    // false: keep segments maximal (fewer CTA barriers) and only choose their
    // warp bits for the banks -- QVB200_PLAN_SEGMENTS=max, an A/B knob
    bool split_on_bank_loss = !(getenv("QVB200_PLAN_SEGMENTS") && std::string(getenv("QVB200_PLAN_SEGMENTS")) == "max");

    void emit(std::vector<GroupDesc>& out) {
        const int tb = k - rbits;
        const int nwb = tb > 5 ? tb - 5 : 0;           // warp-index bits
        const uint32_t all = (1u << k) - 1;
        if (tma) {   // inverse of the final slot map Q (col holds it after the last CNOT)
            qinv.assign((size_t)1 << k, 0);
            for (uint32_t l = 0; l < (1u << k); ++l) {
                uint32_t v = 0;
                for (int j = 0; j < k; ++j)
                    if ((l >> j) & 1u) v ^= col[j];
                qinv[v] = l;
            }
        }
        const size_t G = pending.size();
        std::unordered_map<uint64_t, Layout> memo;   // (group, warp mask) -> layout
        auto layout_of = [&](size_t g, uint32_t w) -> const Layout& {
            const uint64_t key = ((uint64_t)g << 32) | w;
            auto it = memo.find(key);
            if (it == memo.end()) it = memo.emplace(key, group_layout(pending[g], w, tma && g + 1 == G)).first;
            return it->second;
        };
        // segments: runs of groups that leave >= nwb bits untouched (no
        // matrix, no CNOT target in between); nwb of those bits index the
        // warp, so consecutive groups only need __syncwarp.  A segment is
        // extended only while sharing the warp bits costs no bank conflicts
        // (a CTA barrier is cheaper than a 2-way conflicted group).
        auto best_w = [&](size_t s0, size_t e0, uint32_t free_bits) {
            std::vector<int> fb;
            for (int b = k - 1; b >= 0; --b)
                if ((free_bits >> b) & 1u) fb.push_back(b);
            std::pair<int, uint32_t> best{-1, 0};
            const int m = (int)fb.size();
            for (uint32_t sub = 0; sub < (1u << m); ++sub) {   // fb is highest-first: ties keep high bits
                if (__builtin_popcount(sub) != nwb) continue;
                uint32_t w = 0;
                for (int i = 0; i < m; ++i)
                    if ((sub >> i) & 1u) w |= 1u << fb[i];
                int score = 0;
                for (size_t g = s0; g < e0; ++g) score += layout_of(g, w).score;
                if (score > best.first) best = {score, w};
            }
            return best;
        };
        auto solo_free = [&](size_t g) {
            uint32_t f = all;
            for (auto& pr : pending[g].ops) f &= ~(1u << pr.first);
            return f;
        };
        std::vector<uint32_t> wmask(G, 0);
        std::vector<int> seg_start(G, 0);
        size_t s = 0;
        while (s < G) {
            uint32_t free_bits = solo_free(s);
            auto cur = best_w(s, s + 1, free_bits);
            size_t e = s + 1;
            while (e < G) {
                uint32_t f = free_bits & ~pending[e - 1].targets_after;
                for (auto& pr : pending[e].ops) f &= ~(1u << pr.first);
                if (__builtin_popcount(f) < nwb) break;
                const auto ext = best_w(s, e + 1, f);
                const auto solo = best_w(e, e + 1, solo_free(e));
                if (split_on_bank_loss && ext.first < cur.first + solo.first) break;
                free_bits = f;
                cur = ext;
                ++e;
            }
            for (size_t g = s; g < e; ++g) { wmask[g] = cur.second; seg_start[g] = g == s; }
            s = e;
        }
        for (size_t gi = 0; gi < G; ++gi) {
            const Pending& p = pending[gi];
            GroupDesc g;
            std::memset(&g, 0, sizeof(g));
            const Layout l = layout_of(gi, wmask[gi]);
            for (int r = 0; r < kRegBits; ++r) g.mat[r] = -1;
            for (size_t r = 0; r < p.ops.size(); ++r) g.mat[r] = p.ops[r].second;
            std::vector<int> order, rest;
            for (size_t i = 0; i < l.lanes.size(); ++i) ((l.sub >> i) & 1u ? order : rest).push_back(l.lanes[i]);
            order.insert(order.end(), rest.begin(), rest.end());
            for (int b = 0; b < k; ++b)
                if ((wmask[gi] >> b) & 1u) order.push_back(b);
            for (int j = 0; j < (1 << rbits); ++j) {
                uint32_t sl = 0;
                for (int r = 0; r < rbits; ++r)
                    if ((j >> r) & 1) sl ^= swz(p.col[l.reg[r]]);
                g.combo[j] = sl << amp_shift;
            }
            for (size_t m = 0; m < order.size(); ++m) g.tcol[m] = (uint32_t)swz(p.col[order[m]]) << amp_shift;
            g.cta_sync = (gi == 0 || seg_start[gi]) ? 1 : 0;
            out.push_back(g);
        }
        pending.clear();
    }
};

}  // namespace

std::string Topology::key() const {
    std::string s;
    s.reserve(8 + kind.size() * 9);
    s.append(reinterpret_cast<const char*>(&n), sizeof(n));
    for (size_t g = 0; g < kind.size(); ++g) {
        s.push_back((char)kind[g]);
        s.append(reinterpret_cast<const char*>(&q0[g]), sizeof(int32_t));
        const int32_t b = is_two_qubit(kind[g]) ? q1[g] : -1;
        s.append(reinterpret_cast<const char*>(&b), sizeof(int32_t));
    }
    return s;
}

int tile_bits_for(int n, int precision) {
    const int kmax = max_tile_bits(precision);
    if (n <= kmax) return std::max(n, reg_bits(precision));
    return kmax;
}

Plan build_plan(const Topology& topo, int precision, int max_tile_bits) {
    Plan plan;
    plan.n = topo.n;
    plan.precision = precision;
    plan.k = tile_bits_for(topo.n, precision);
    if (max_tile_bits > 0) {
        if (max_tile_bits < coalesce_bits(precision) + 2 || max_tile_bits > kMaxTileBits)
            throw std::runtime_error("tile bits out of range");
        plan.k = topo.n <= max_tile_bits ? std::max(topo.n, reg_bits(precision)) : max_tile_bits;
    }
    plan.single_tile = topo.n <= plan.k;
    plan.ops = fuse(topo);
    const int n = topo.n, k = plan.k;
    const int beta = bank_bits(precision);
    if (plan.single_tile) {
        PassPlan pp;
        for (int b = 0; b < k; ++b) pp.S.push_back(b);
        for (size_t i = 0; i < plan.ops.size(); ++i) pp.ops.push_back((int)i);
        plan.passes.push_back(std::move(pp));
    } else {
        plan.passes = select_passes(n, k, coalesce_bits(precision), plan.ops);
    }
    // Bank model of one warp's accesses (warp 0; the other warps differ by a
    // constant XOR): wavefronts of one register set, 128-bit (complex128) or
    // 64-bit (complex64) accesses.
    const int sh = precision == 0 ? 4 : 3, rows = precision == 0 ? 8 : 16;
    const int R = reg_bits(precision), tbits = k - R;
    auto access_wf = [&](const uint32_t* combo, const uint32_t* tcol) {
        int64_t wf = 0;
        for (int j = 0; j < (1 << R); ++j) {
            int count[16] = {0};
            for (int lane = 0; lane < 32; ++lane) {
                uint32_t base = 0;
                for (int m = 0; m < 5 && m < tbits; ++m)
                    if ((lane >> m) & 1) base ^= tcol[m];
                ++count[((base ^ combo[j]) >> sh) & (rows - 1)];
            }
            wf += *std::max_element(count, count + rows);
        }
        return wf;
    };
    const int c = coalesce_bits(precision);
    for (auto& pp : plan.passes) {
        auto build_pass = [&](const uint16_t* init_cols, bool tma) {
            PassDesc d;
            std::memset(&d, 0, sizeof(d));
            d.k = k;
            d.n_outer = plan.single_tile ? 0 : n - k;
            int logical_of[64];
            for (int b = 0; b < 64; ++b) logical_of[b] = -1;
            for (int j = 0; j < k; ++j) { d.sbits[j] = (uint8_t)pp.S[j]; logical_of[pp.S[j]] = j; }
            if (!plan.single_tile) {
                int o = 0;
                for (int b = 0; b < n; ++b)
                    if (logical_of[b] < 0) d.obits[o++] = (uint8_t)b;
            }
            GroupBuilder gb;
            gb.k = k;
            gb.beta = beta;
            gb.rbits = R;
            gb.amp_shift = precision == 0 ? 4 : 3;
            gb.tma = tma;
            gb.coalesce_bits_ = coalesce_bits(precision);
            for (int j = 0; j < 16; ++j) gb.col[j] = gb.init[j] = init_cols[j];
            for (int j = 0; j < k; ++j) d.swz[j] = gb.phys(j);
            d.g0 = (int)plan.groups.size();
            d.m0 = (int)plan.mat_op.size();
            int local_mats = 0;
            // List scheduling of the pass's op DAG (edges: program order on shared
            // bits).  Ready CNOTs are folded into Q immediately (free); register
            // groups are filled with up to R ready MAT1s, longest remaining
            // dependency chain first, so groups are full and few.
            const int m = (int)pp.ops.size();
            std::vector<std::vector<int>> preds(m), succs(m);
            {
                std::vector<int> last(64, -1);
                for (int i = 0; i < m; ++i) {
                    const FusedOp& op = plan.ops[pp.ops[i]];
                    const int bits[2] = {op.b0, op.cnot ? op.b1 : -1};
                    for (int b : bits) {
                        if (b < 0) continue;
                        if (last[b] >= 0) { preds[i].push_back(last[b]); succs[last[b]].push_back(i); }
                        last[b] = i;
                    }
                }
            }
            std::vector<int> height(m, 0);
            for (int i = m - 1; i >= 0; --i)
                for (int s : succs[i]) height[i] = std::max(height[i], height[s] + 1);
            std::vector<char> applied(m, 0), in_group(m, 0);
            std::vector<int> open_ops;
            int done = 0;
            auto ready = [&](int i) {
                for (int p : preds[i])
                    if (!applied[p]) return false;
                return true;
            };
            auto close_group = [&]() {
                gb.close();
                for (int i : open_ops) { applied[i] = 1; ++done; }
                open_ops.clear();
            };
            while (done < m) {
                bool progress = true;
                while (progress) {   // fold every ready CNOT into the slot map
                    progress = false;
                    for (int i = 0; i < m; ++i) {
                        const FusedOp& op = plan.ops[pp.ops[i]];
                        if (!op.cnot || applied[i] || !ready(i)) continue;
                        gb.cnot(logical_of[op.b0], logical_of[op.b1]);
                        applied[i] = 1;
                        ++done;
                        progress = true;
                    }
                }
                if (done == m) break;
                int best = -1;
                for (int i = 0; i < m; ++i) {
                    if (plan.ops[pp.ops[i]].cnot || applied[i] || in_group[i] || !ready(i)) continue;
                    if (best < 0 || height[i] > height[best]) best = i;
                }
                if (best < 0) {
                    if (open_ops.empty()) throw std::runtime_error("group scheduler stalled");
                    close_group();
                    continue;
                }
                in_group[best] = 1;
                open_ops.push_back(best);
                gb.open.push_back({logical_of[plan.ops[pp.ops[best]].b0], local_mats++});
                plan.mat_op.push_back(pp.ops[best]);
                if ((int)open_ops.size() == R) close_group();
            }
            close_group();
            gb.emit(plan.groups);
            d.ng = (int)plan.groups.size() - d.g0;
            d.nm = local_mats;
            for (int j = 0; j < k; ++j) d.fin[j] = gb.phys(j);
            for (int it = 0; it < (1 << R); ++it) {   // a thread's amplitudes: tid | it << (k - R)
                const uint32_t idx = (uint32_t)it << (k - R);
                d.swz_hi[it] = (uint16_t)apply_cols(d.swz, k, idx);
                d.fin_hi[it] = (uint16_t)apply_cols(d.fin, k, idx);
                uint64_t g = 0;
                for (int i = 0; i < R; ++i)
                    if ((it >> i) & 1) g |= 1ull << d.sbits[k - R + i];
                d.g_hi[it] = g;
            }
            pp.n_groups = d.ng;
            pp.n_mats = d.nm;
            plan.pdesc.push_back(d);
        };
        // Store map of the last group (TMA layout) and the bank cost of a pass
        // built on a TMA layout; tl.ok = 0 if it has no register group.
        auto finish_tma = [&](TmaLayout& tl) {
            const PassDesc& d = plan.pdesc.back();
            int64_t wf = 0;
            for (int g = d.g0; g < d.g0 + d.ng; ++g) {
                wf += access_wf(plan.groups[g].combo, plan.groups[g].tcol);
                if (g + 1 < d.g0 + d.ng) wf += access_wf(plan.groups[g].combo, plan.groups[g].tcol);
            }
            tl.ok = d.ng > 0 ? 1 : 0;
            if (d.ng > 0) {
                // physical slot p holds, at the end of the pass, logical fin^-1(p);
                // the last group writes it to the TMA slot of that logical index
                const int shift = precision == 0 ? 4 : 3;
                std::vector<uint32_t> inv((size_t)1 << k);
                for (uint32_t l = 0; l < (1u << k); ++l) inv[apply_cols(d.fin, k, l)] = l;
                const GroupDesc& G = plan.groups[d.g0 + d.ng - 1];
                for (int j = 0; j < (1 << R); ++j)
                    tl.wcombo[j] = (uint32_t)apply_cols(d.swz, k, inv[G.combo[j] >> shift]) << shift;
                for (int mm = 0; mm < tbits && mm < 11; ++mm)
                    tl.wtcol[mm] = (uint32_t)apply_cols(d.swz, k, inv[G.tcol[mm] >> shift]) << shift;
                // global amplitude offsets of the same final positions
                auto global_of = [&](uint32_t l) {
                    uint64_t g = 0;
                    for (int j = 0; j < k; ++j)
                        if ((l >> j) & 1u) g |= 1ull << d.sbits[j];
                    return g;
                };
                for (int j = 0; j < (1 << R); ++j) tl.gwcombo[j] = global_of(inv[G.combo[j] >> shift]);
                for (int mm = 0; mm < tbits && mm < 11; ++mm) tl.gwtcol[mm] = global_of(inv[G.tcol[mm] >> shift]);
                uint32_t row = 0;
                for (int mm = 0; mm < c && mm < tbits; ++mm) row |= inv[G.tcol[mm] >> shift];
                tl.coalesced = row == (1u << c) - 1 ? 1 : 0;
                // first group: physical slot -> initial logical index (the
                // load layout swz is a permutation under the TMA swizzle)
                std::vector<uint32_t> inv0((size_t)1 << k);
                for (uint32_t l = 0; l < (1u << k); ++l) inv0[apply_cols(d.swz, k, l)] = l;
                const GroupDesc& F = plan.groups[d.g0];
                for (int mm = 0; mm < tbits && mm < 11; ++mm) tl.flam[mm] = inv0[F.tcol[mm] >> shift];
                for (int r = 0; r < R; ++r) tl.fmu[r] = inv0[F.combo[1 << r] >> shift];
            }
            tl.wavefronts = wf;
        };
        uint16_t ident[16];
        for (int j = 0; j < 16; ++j) ident[j] = (uint16_t)(j < k ? 1u << j : 0);
        if (plan.single_tile) {
            build_pass(ident, false);
            plan.tma.push_back(TmaLayout{});
            continue;
        }
        // Candidate TMA layouts: the tile bits above the low `c` split into <= 3
        // pieces of <= 8 consecutive global bits, in any order.  Only the bits
        // that land in the swizzled row positions c..c+2 matter for the banks,
        // so one candidate (the fewest pieces) is built per choice of them.
        struct Piece { int lo, len; };
        std::vector<Piece> runs;
        for (int b : pp.S) {
            if (b < c) continue;
            if (!runs.empty() && runs.back().lo + runs.back().len == b) ++runs.back().len;
            else runs.push_back({b, 1});
        }
        std::vector<std::vector<Piece>> cands;
        std::vector<uint64_t> keys;
        std::vector<Piece> acc;
        std::function<void(size_t)> per_run;
        std::function<void(size_t, int, int)> split = [&](size_t r, int start, int end) {
            if (start == end) { per_run(r + 1); return; }
            for (int len = 1; len <= 8 && start + len <= end; ++len) {
                acc.push_back({start, len});
                if (acc.size() <= 3) split(r, start + len, end);
                acc.pop_back();
            }
        };
        per_run = [&](size_t r) {
            if (r < runs.size()) { split(r, runs[r].lo, runs[r].lo + runs[r].len); return; }
            std::vector<int> idx(acc.size());
            for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int)i;
            do {
                std::vector<Piece> order;
                uint64_t key = 0;
                int placed = 0;
                for (int i : idx) {
                    order.push_back(acc[i]);
                    for (int b = acc[i].lo; b < acc[i].lo + acc[i].len && placed < 3; ++b, ++placed)
                        key = (key << 8) | (uint64_t)(b + 1);
                }
                auto it = std::find(keys.begin(), keys.end(), key);
                if (it == keys.end()) { keys.push_back(key); cands.push_back(order); }
                else if (cands[it - keys.begin()].size() > order.size()) cands[it - keys.begin()] = order;
            } while (std::next_permutation(idx.begin(), idx.end()));
        };
        const bool low_ok = k > c && [&]() {
            for (int b = 0; b < c; ++b)
                if (std::find(pp.S.begin(), pp.S.end(), b) == pp.S.end()) return false;
            return true;
        }();
        if (low_ok) per_run(0);
        auto layout_of = [&](const std::vector<Piece>& order, uint16_t* cols, TmaLayout& tl) {
            std::vector<int> pos_of_bit(64, -1);
            int pos = 0;
            for (int b = 0; b < c; ++b) pos_of_bit[b] = pos++;
            for (const Piece& pc : order)
                for (int b = pc.lo; b < pc.lo + pc.len; ++b) pos_of_bit[b] = pos++;
            for (int j = 0; j < 16; ++j) cols[j] = j < k ? (uint16_t)(1u << pos_of_bit[pp.S[j]]) : 0;
            std::vector<char> local(64, 0);
            for (int b : pp.S) local[b] = 1;
            auto span_of = [&](int lo, int len) {   // the piece + outer bits up to the next tile bit
                int e = lo + len;
                while (e < n && !local[e]) ++e;
                return e - lo;
            };
            tl.ndim = 1 + (int)order.size();
            tl.lo[0] = 0;
            tl.box[0] = c;
            tl.span[0] = span_of(0, c);
            for (size_t i = 0; i < order.size(); ++i) {
                tl.lo[i + 1] = order[i].lo;
                tl.box[i + 1] = order[i].len;
                tl.span[i + 1] = span_of(order[i].lo, order[i].len);
            }
        };
        TmaLayout best_tl;
        uint16_t best_cols[16];
        int ngroups_of_last = 0;
        int64_t best_wf = -1;
        for (const auto& cand : cands) {
            uint16_t cols[16];
            TmaLayout tl;
            layout_of(cand, cols, tl);
            const size_t g0 = plan.groups.size(), m0 = plan.mat_op.size(), p0 = plan.pdesc.size();
            build_pass(cols, true);
            finish_tma(tl);
            ngroups_of_last = plan.pdesc.back().ng;
            plan.groups.resize(g0);
            plan.mat_op.resize(m0);
            plan.pdesc.resize(p0);
            if (tl.ok && (best_wf < 0 || tl.wavefronts < best_wf)) {
                best_wf = tl.wavefronts;
                best_tl = tl;
                std::memcpy(best_cols, cols, sizeof(best_cols));
            }
            // conflict-free (every access set at 32 lanes / bank columns
            // wavefronts per register): no candidate can do better
            // (every group's load and store, the last group storing to HBM)
            if (best_wf >= 0 && best_wf <= (int64_t)(2 * ngroups_of_last - 1) * (1 << R) * (32 / rows)) break;
        }
        if (best_wf >= 0) {
            build_pass(best_cols, true);
            finish_tma(best_tl);
            plan.tma.push_back(best_tl);
        } else {
            build_pass(ident, false);
            plan.tma.push_back(TmaLayout{});
        }
    }
    return plan;
}

namespace {
struct M2 { cd a, b, c, d; };  // [[a,b],[c,d]]
M2 mul(const M2& x, const M2& y) {  // x * y
    return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c, x.c * y.b + x.d * y.d};
}
M2 gate_matrix(const Topology& t, int32_t ref, const double* angles) {
    const double inv = 1.0 / std::sqrt(2.0);
    if (ref < 0) return {cd(inv, 0), cd(inv, 0), cd(inv, 0), cd(-inv, 0)};
    const uint8_t k = t.kind[ref];
    switch (k) {
        case G_H: return {cd(inv, 0), cd(inv, 0), cd(inv, 0), cd(-inv, 0)};
        case G_X: return {cd(0, 0), cd(1, 0), cd(1, 0), cd(0, 0)};
        case G_RY: {
            const double c = std::cos(angles[ref] / 2.0), s = std::sin(angles[ref] / 2.0);
            return {cd(c, 0), cd(-s, 0), cd(s, 0), cd(c, 0)};
        }
        case G_RZ: {
            const double c = std::cos(angles[ref] / 2.0), s = std::sin(angles[ref] / 2.0);
            return {cd(c, -s), cd(0, 0), cd(0, 0), cd(c, s)};
        }
        case G_RX: {
            const double c = std::cos(angles[ref] / 2.0), s = std::sin(angles[ref] / 2.0);
            return {cd(c, 0), cd(0, -s), cd(0, -s), cd(c, 0)};
        }
        default: throw std::runtime_error("not a one-qubit gate");
    }
}
}  // namespace

namespace {
// Ordered product of a slot's gates; with pauli_gate >= 0 the generator of
// that rotation (X for RX, Y for RY, Z for RZ) is applied just before it.
void slot_product(const Plan& plan, const Topology& topo, const double* angles, int s, int32_t pauli_gate,
                  double* o) {
    const FusedOp& op = plan.ops[plan.mat_op[s]];
    M2 m{cd(1, 0), cd(0, 0), cd(0, 0), cd(1, 0)};
    bool first = true;
    for (int32_t ref : op.gates) {
        if (ref >= 0 && ref == pauli_gate) {
            M2 p;
            switch (topo.kind[ref]) {
                case G_RX: p = {cd(0, 0), cd(1, 0), cd(1, 0), cd(0, 0)}; break;
                case G_RY: p = {cd(0, 0), cd(0, -1), cd(0, 1), cd(0, 0)}; break;
                case G_RZ: p = {cd(1, 0), cd(0, 0), cd(0, 0), cd(-1, 0)}; break;
                default: throw std::runtime_error("shifted gate is not a rotation");
            }
            m = first ? p : mul(p, m);
            first = false;
        }
        const M2 g = gate_matrix(topo, ref, angles);
        m = first ? g : mul(g, m);
        first = false;
    }
    o[0] = m.a.real(); o[1] = m.a.imag();
    o[2] = m.b.real(); o[3] = m.b.imag();
    o[4] = m.c.real(); o[5] = m.c.imag();
    o[6] = m.d.real(); o[7] = m.d.imag();
}
}  // namespace

void circuit_matrices(const Plan& plan, const Topology& topo, const double* angles, double* out) {
    for (int s = 0; s < plan.n_slots(); ++s) slot_product(plan, topo, angles, s, -1, out + (size_t)s * 8);
}

void slot_matrix_with_pauli(const Plan& plan, const Topology& topo, const double* angles, int slot,
                            int32_t pauli_gate, double* out8) {
    slot_product(plan, topo, angles, slot, pauli_gate, out8);
}

std::vector<int> slot_of_gates(const Plan& plan, const Topology& topo) {
    std::vector<int> slot(topo.kind.size(), -1);
    for (int s = 0; s < plan.n_slots(); ++s)
        for (int32_t ref : plan.ops[plan.mat_op[s]].gates)
            if (ref >= 0) slot[ref] = s;
    return slot;
}

// Light cone of a support-restricted output (SUPPORT / JS results, shift
// pairs).  Backward: a bit that is zero in every support index and that no
// pass from p on touches is a spectator -- the final amplitudes on the support
// only depend on the inputs of pass p whose spectator bits are zero, so
// cone[p] = support bits | tile bits of passes p..P-1.  Forward: every state
// starts as |0...0>, so before pass p only the bits some earlier pass touched
// (seen[p]) can be nonzero.  Pass p then runs on the tiles whose outer bits
// outside cone[p] & seen[p] are zero, and zero-fills the local slots of bits
// it is the first to touch (`fresh`) instead of loading them.  For the QCL
// benchmarks the first two passes touch 1 and 256 tiles and the last three 1,
// 4 and 1024 tiles of 2^16.  Support indices with a bit no pass touches have
// probability exactly 0 (`reach` excludes them).
LightCone light_cone(const Plan& plan, const uint64_t* support, int64_t S) {
    const size_t P = plan.passes.size();
    LightCone lc;
    lc.outer_free.resize(P);
    lc.fresh.resize(P);
    uint64_t acc = 0;
    for (int64_t s = 0; s < S; ++s) acc |= support[s];
    std::vector<uint64_t> cone(P);
    for (size_t p = P; p-- > 0;) {
        for (int b : plan.passes[p].S) acc |= 1ull << b;
        cone[p] = acc;
    }
    uint64_t seen = 0;
    for (size_t p = 0; p < P; ++p) {
        lc.outer_free[p] = cone[p] & seen;
        uint32_t fresh = 0;
        for (size_t j = 0; j < plan.passes[p].S.size(); ++j)
            if (!((seen >> plan.passes[p].S[j]) & 1)) fresh |= 1u << j;
        lc.fresh[p] = fresh;
        for (int b : plan.passes[p].S) seen |= 1ull << b;
    }
    lc.reach = seen;
    return lc;
}

// The pass restricted to the tiles whose outer bits outside `free` are zero.
PassDesc restrict_pass(const PassDesc& pd, uint64_t free, uint32_t fresh) {
    PassDesc r = pd;
    int m = 0;
    for (int j = 0; j < pd.n_outer; ++j)
        if ((free >> pd.obits[j]) & 1) r.obits[m++] = pd.obits[j];
    for (int j = m; j < (int)sizeof(r.obits); ++j) r.obits[j] = 0;
    r.n_outer = m;
    r.fresh = fresh;
    return r;
}

int tile_low_bits(int precision) { return coalesce_bits(precision); }

PassDesc readonly_pass(const Plan& plan, uint64_t S) {
    PassDesc d;
    std::memset(&d, 0, sizeof(d));
    const int k = plan.k, n = plan.n, R = reg_bits(plan.precision);
    d.k = k;
    d.n_outer = n - k;
    int j = 0, o = 0;
    for (int b = 0; b < n; ++b) {
        if ((S >> b) & 1) d.sbits[j++] = (uint8_t)b;
        else d.obits[o++] = (uint8_t)b;
    }
    if (j != k) throw std::runtime_error("read-only pass needs exactly k tile bits");
    for (int i = 0; i < k; ++i) d.swz[i] = d.fin[i] = (uint16_t)(1u << i);
    for (int it = 0; it < (1 << R); ++it) {
        const uint32_t idx = (uint32_t)it << (k - R);
        d.swz_hi[it] = d.fin_hi[it] = (uint16_t)idx;
        uint64_t g = 0;
        for (int i = 0; i < R; ++i)
            if ((it >> i) & 1) g |= 1ull << d.sbits[k - R + i];
        d.g_hi[it] = g;
    }
    return d;
}

}  // namespace qvb
