// Pass planner (host). See planner.hpp and DESIGN.md §3.
//
// The reference applies every layer of every C_j / C_j^dagger as its own
// full-state sweep (proj/src/statevector.cpp:339-381, one sweep per H gate).
// Here a step's gates are list-scheduled into tile passes: a pass may run
// any ops whose "need" qubits (H targets, CNOT targets) lie in its <= k
// local qubits, in any order consistent with the gates' commutation
// relations; diagonal ops (phase layers, exp(-i dt Lambda)) need nothing and
// ride along for free.
#include "planner.hpp"

#include <algorithm>
#include <cstdlib>
#include <bit>
#include <sstream>
#include <stdexcept>

namespace sdb {

namespace {

inline uint64_t bitq(int q) { return 1ull << q; }

}  // namespace

int fixed_bits_for(int k) {
    static const int want = [] {
        const char* e = std::getenv("SDB_FIXED_BITS");
        return e ? std::atoi(e) : 3;
    }();
    return std::max(0, std::min(want, k - 1));
}

namespace {

bool is_diag(const Op& o) { return o.kind == Op::PH || o.kind == Op::DG; }

bool commute(const Op& a, const Op& b) {
    if (is_diag(a) && is_diag(b)) return true;
    if (a.kind == Op::H && b.kind == Op::H) return a.q != b.q;
    if (a.kind == Op::H) return (bitq(a.q) & b.support) == 0;
    if (b.kind == Op::H) return (bitq(b.q) & a.support) == 0;
    if (a.kind == Op::CX && b.kind == Op::CX) {
        return (bitq(a.q) & b.targets) == 0 && (bitq(b.q) & a.targets) == 0;
    }
    const Op& cx = a.kind == Op::CX ? a : b;
    const Op& dg = a.kind == Op::CX ? b : a;
    return (cx.targets & dg.support) == 0;
}

// ---- CNOT network resynthesis -------------------------------------------
// A group's CNOT list is a GF(2)-linear index map M (CX(c,t): x_t ^= x_c, a
// row operation "row t += row c" on M). A tile pass can apply any CNOTs whose
// targets are local, so M is re-expressed as rounds of CNOTs whose targets lie
// in a set T of <= cap qubits: each round turns the rows of T into unit rows
// using every other row (possible iff M restricted to the complement is
// invertible), so ceil(#non-unit rows / cap) rounds suffice when the sets can
// be chosen. The result is the same linear map (checked), hence the same
// amplitude permutation, bit for bit.
namespace {

using Rows = std::vector<uint64_t>;  // row i: bit j set <=> M[i][j]

bool invertible_on(const Rows& M, uint64_t cols_mask, const std::vector<int>& rows) {
    // rank of the submatrix (rows x cols_mask) == |rows|
    std::vector<uint64_t> r;
    for (int i : rows) r.push_back(M[i] & cols_mask);
    size_t rank = 0;
    for (int c = 0; c < 64 && rank < r.size(); ++c) {
        if (!((cols_mask >> c) & 1)) continue;
        size_t piv = rank;
        while (piv < r.size() && !((r[piv] >> c) & 1)) ++piv;
        if (piv == r.size()) continue;
        std::swap(r[piv], r[rank]);
        for (size_t k = 0; k < r.size(); ++k)
            if (k != rank && ((r[k] >> c) & 1)) r[k] ^= r[rank];
        ++rank;
    }
    return rank == r.size();
}

// rows T of M^{-1} (M invertible, m x m)
Rows inverse_rows(const Rows& M, int m) {
    Rows a = M, inv(m);
    for (int i = 0; i < m; ++i) inv[i] = 1ull << i;
    for (int c = 0; c < m; ++c) {
        int piv = c;
        while (piv < m && !((a[piv] >> c) & 1)) ++piv;
        if (piv == m) throw std::logic_error("resynth: singular CNOT map");
        std::swap(a[piv], a[c]);
        std::swap(inv[piv], inv[c]);
        for (int k = 0; k < m; ++k) {
            if (k != c && ((a[k] >> c) & 1)) {
                a[k] ^= a[c];
                inv[k] ^= inv[c];
            }
        }
    }
    return inv;
}

std::vector<std::pair<int, int>> resynth_cnots(const std::vector<std::pair<int, int>>& cnots, int cap) {
    if (cnots.size() < 2 || cap < 1) return cnots;
    std::vector<int> qs;
    for (auto [c, t] : cnots) qs.insert(qs.end(), {c, t});
    std::sort(qs.begin(), qs.end());
    qs.erase(std::unique(qs.begin(), qs.end()), qs.end());
    const int m = static_cast<int>(qs.size());
    if (m > 64) return cnots;
    auto idx = [&](int q) { return static_cast<int>(std::lower_bound(qs.begin(), qs.end(), q) - qs.begin()); };
    Rows M(m);
    for (int i = 0; i < m; ++i) M[i] = 1ull << i;
    for (auto [c, t] : cnots) M[idx(t)] ^= M[idx(c)];
    const Rows target = M;
    std::vector<std::pair<int, int>> red;  // reduction ops (dense indices), applied in order
    auto apply = [&](int c, int t) {
        M[t] ^= M[c];
        red.emplace_back(c, t);
    };
    std::vector<int> original_rounds;
    for (int guard = 0; guard < 4 * m; ++guard) {
        std::vector<int> nonunit;
        for (int i = 0; i < m; ++i)
            if (M[i] != (1ull << i)) nonunit.push_back(i);
        if (nonunit.empty()) break;
        std::vector<int> T;
        const uint64_t all = m >= 64 ? ~0ull : ((1ull << m) - 1);
        auto complement_ok = [&](const std::vector<int>& t) {
            uint64_t tm = 0;
            for (int i : t) tm |= 1ull << i;
            std::vector<int> o;
            for (int i = 0; i < m; ++i)
                if (!((tm >> i) & 1)) o.push_back(i);
            return invertible_on(M, all & ~tm, o);
        };
        if (static_cast<int>(nonunit.size()) <= cap) {
            T = nonunit;
        } else {
            // first cap non-unit rows, then deterministic rotations of the candidate list
            bool found = false;
            for (size_t rot = 0; rot < nonunit.size() && !found; ++rot) {
                std::vector<int> t;
                for (int j = 0; j < cap; ++j) t.push_back(nonunit[(rot + j) % nonunit.size()]);
                if (complement_ok(t)) {
                    T = t;
                    found = true;
                }
            }
            if (!found) return cnots;  // keep the synthesis as given
        }
        uint64_t tm = 0;
        for (int i : T) tm |= 1ull << i;
        const Rows inv = inverse_rows(M, m);
        // rows T <- A_TT rows_T + A_TO rows_O with A = (M^{-1})[T, :]
        // (a) A_TT as row-add ops within T: Gauss-Jordan of A_TT (no swaps)
        const int nt = static_cast<int>(T.size());
        std::vector<uint32_t> att(nt);  // att[r] bit s: A[T_r][T_s]
        for (int r = 0; r < nt; ++r)
            for (int s2 = 0; s2 < nt; ++s2)
                if ((inv[T[r]] >> T[s2]) & 1) att[r] |= 1u << s2;
        std::vector<std::pair<int, int>> ops;  // (src, dst) in T-local indices reducing att to I
        for (int c = 0; c < nt; ++c) {
            if (!((att[c] >> c) & 1)) {
                int piv = -1;
                // rows above c are already unit in columns < c; an invertible
                // block always has a pivot below
                for (int r = c + 1; r < nt; ++r)
                    if ((att[r] >> c) & 1) {
                        piv = r;
                        break;
                    }
                if (piv < 0) return cnots;
                att[c] ^= att[piv];
                ops.emplace_back(piv, c);
            }
            for (int r = 0; r < nt; ++r) {
                if (r != c && ((att[r] >> c) & 1)) {
                    att[r] ^= att[c];
                    ops.emplace_back(c, r);
                }
            }
        }
        // ops reduce A_TT to I: A_TT = product in reverse; applying A_TT to the
        // rows of T = applying the ops in reverse order
        for (auto it = ops.rbegin(); it != ops.rend(); ++it) apply(T[it->first], T[it->second]);
        // (b) adds from outside T
        for (int r = 0; r < nt; ++r) {
            const uint64_t ao = inv[T[r]] & ~tm;
            for (uint64_t b = ao; b; b &= b - 1) apply(std::countr_zero(b), T[r]);
        }
        for (int i : T) {
            if (M[i] != (1ull << i)) return cnots;  // should not happen; keep the given synthesis
        }
    }
    for (int i = 0; i < m; ++i)
        if (M[i] != (1ull << i)) return cnots;
    // forward circuit: the reduction reversed (every CNOT is an involution)
    std::vector<std::pair<int, int>> out;
    for (auto it = red.rbegin(); it != red.rend(); ++it) out.emplace_back(qs[it->first], qs[it->second]);
    // check: same map
    Rows chk(m);
    for (int i = 0; i < m; ++i) chk[i] = 1ull << i;
    for (auto [c, t] : out) chk[idx(t)] ^= chk[idx(c)];
    if (chk != target) return cnots;
    // Use it only if it needs fewer target rounds than the given list (proxy:
    // consecutive windows with at most cap distinct targets).
    auto windows = [cap](const std::vector<std::pair<int, int>>& l) {
        int w = 0;
        std::vector<int> tg;
        for (auto [c, t] : l) {
            (void)c;
            if (std::find(tg.begin(), tg.end(), t) != tg.end()) continue;
            if (tg.empty() || static_cast<int>(tg.size()) == cap) {
                ++w;
                tg.clear();
            }
            tg.push_back(t);
        }
        return w;
    };
    return windows(out) < windows(cnots) ? out : cnots;
}

}  // namespace

// Emits group applications in order. CNOT networks are kept pending so that
// C_g^dagger's inverse network and C_{g+1}'s network, adjacent whenever no
// h_pre layer separates them, become ONE linear map that is re-synthesised as
// a whole (CX(c,t) is an involution, so the inverse network is the list
// reversed; statevector.cpp:341-349 applies runs in list order).
class GroupEmitter {
public:
    GroupEmitter(std::vector<Op>& out, int max_targets, int resynth_cap, bool split_diag, bool cz_to_cx)
        : out_(out), max_targets_(max_targets), cap_(resynth_cap), split_(split_diag), cz_cx_(cz_to_cx) {}

    void group(const GroupSpec& g_in, int gi, double dt_scale) {
        // H_b CZ(a_1,b)..CZ(a_r,b) H_b = CX(a_1->b)..CX(a_r->b): a qubit b in
        // both h_pre and h_post whose only gates between the two layers are CZs
        // (no CNOT, no S) loses both Hadamards, and its CZs become CNOTs with b
        // as target -- the same unitary C_j, with two Hadamard levels fewer
        // (config 4: the Bell-pair groups' odd/even qubits). At most one end of
        // a CZ may be converted (H_a H_b CZ H_a H_b is no CNOT), so the
        // candidates are taken greedily in qubit order.
        const uint64_t conv = cz_cx_ ? convertible(g_in) : 0;
        const GroupSpec* gp = &g_in;
        GroupSpec gc;
        std::vector<std::pair<int, int>> conv_cx;  // (control, target)
        if (conv) {
            gc = g_in;
            gc.h_pre.clear();
            gc.h_post.clear();
            gc.czs.clear();
            for (int q : g_in.h_pre)
                if (!(conv & bitq(q))) gc.h_pre.push_back(q);
            for (int q : g_in.h_post)
                if (!(conv & bitq(q))) gc.h_post.push_back(q);
            for (auto [a, b] : g_in.czs) {
                if (conv & bitq(b)) conv_cx.emplace_back(a, b);
                else if (conv & bitq(a)) conv_cx.emplace_back(b, a);
                else gc.czs.push_back({a, b});
            }
            gp = &gc;
        }
        const GroupSpec& g = *gp;
        if (!g.h_pre.empty()) {
            flush();
            for (int q : g.h_pre) h(q);
        }
        pending_.insert(pending_.end(), g.cnots.begin(), g.cnots.end());
        flush();
        const bool has_phase = !g.czs.empty() || !g.s_layer.empty();
        if (has_phase) ph(g, false);
        for (auto [c, t] : conv_cx) cx(c, bitq(t));
        for (int q : g.h_post) h(q);
        if (split_) {
            for (size_t t = 0; t < g.z_masks.size(); ++t) {
                Op o;
                o.kind = Op::DG;
                o.group = gi;
                o.t0 = static_cast<int>(t);
                o.t1 = static_cast<int>(t + 1);
                o.dt_scale = dt_scale;
                o.support = g.z_masks[t];
                out_.push_back(std::move(o));
            }
        } else {
            Op o;
            o.kind = Op::DG;
            o.group = gi;
            o.dt_scale = dt_scale;
            for (uint64_t m : g.z_masks) o.support |= m;
            out_.push_back(std::move(o));
        }
        for (int q : g.h_post) h(q);
        for (auto [c, t] : conv_cx) cx(c, bitq(t));
        if (has_phase) ph(g, true);
        pending_.assign(g.cnots.rbegin(), g.cnots.rend());
        if (!g.h_pre.empty()) {
            flush();
            for (int q : g.h_pre) h(q);
        }
    }

    void flush() {
        const std::vector<std::pair<int, int>> cn = cap_ > 0 ? resynth_cnots(pending_, cap_) : pending_;
        pending_.clear();
        for (size_t k = 0; k < cn.size();) {
            const int c = cn[k].first;
            uint64_t t = 0;
            while (k < cn.size() && cn[k].first == c) t ^= bitq(cn[k++].second);  // CX(c,t)^2 = 1
            // Same-control CNOTs commute, so a run wider than a tile can hold
            // is split into sub-runs of at most max_targets targets.
            while (std::popcount(t) > max_targets_) {
                uint64_t part = 0;
                for (int j = 0; j < max_targets_; ++j) {
                    const uint64_t lo = t & (~t + 1);
                    part |= lo;
                    t ^= lo;
                }
                cx(c, part);
            }
            if (t) cx(c, t);
        }
    }

private:
    static uint64_t convertible(const GroupSpec& g) {
        uint64_t pre = 0, post = 0, blocked = 0;
        for (int q : g.h_pre) pre |= bitq(q);
        for (int q : g.h_post) post |= bitq(q);
        for (int q : g.s_layer) blocked |= bitq(q);
        for (auto [c, t] : g.cnots) blocked |= bitq(c) | bitq(t);
        uint64_t cand = pre & post & ~blocked, conv = 0;
        for (uint64_t m = cand; m; m &= m - 1) {
            const int b = std::countr_zero(m);
            bool ok = true;
            for (auto [x, y] : g.czs) {
                if ((x == b && (conv & bitq(y))) || (y == b && (conv & bitq(x))) || (x == b && y == b)) ok = false;
            }
            if (ok) conv |= bitq(b);
        }
        return conv;
    }
    void h(int q) {
        Op o;
        o.kind = Op::H;
        o.q = q;
        o.support = o.need = bitq(q);
        out_.push_back(std::move(o));
    }
    void cx(int c, uint64_t t) {
        Op o;
        o.kind = Op::CX;
        o.q = c;
        o.targets = t;
        o.support = t | bitq(c);
        o.need = t;
        out_.push_back(std::move(o));
    }
    void ph(const GroupSpec& g, bool dagger) {
        if (split_) {
            for (int q : g.s_layer) {
                Op o;
                o.kind = Op::PH;
                o.dagger = dagger;
                o.s_mask = o.support = bitq(q);
                out_.push_back(std::move(o));
            }
            for (auto cz : g.czs) {
                Op o;
                o.kind = Op::PH;
                o.dagger = dagger;
                o.czs = {cz};
                o.support = bitq(cz.first) | bitq(cz.second);
                out_.push_back(std::move(o));
            }
            return;
        }
        Op o;
        o.kind = Op::PH;
        o.dagger = dagger;
        for (int q : g.s_layer) o.s_mask |= bitq(q);
        o.czs = g.czs;
        o.support = o.s_mask;
        for (auto [a, b] : g.czs) o.support |= bitq(a) | bitq(b);
        out_.push_back(std::move(o));
    }

    std::vector<Op>& out_;
    int max_targets_, cap_;
    bool split_, cz_cx_;
    std::vector<std::pair<int, int>> pending_;
};

uint64_t to_phys(uint64_t logical, const std::vector<int>& phys_of) {
    uint64_t p = 0;
    while (logical) {
        const int q = std::countr_zero(logical);
        logical &= logical - 1;
        p |= bitq(phys_of[q]);
    }
    return p;
}

}  // namespace

std::vector<Op> step_ops(const std::vector<GroupSpec>& groups, int /*n_qubits*/, int order, int max_targets,
                         int resynth_cap, bool split_diag, bool cz_to_cx) {
    std::vector<Op> ops;
    const int G = static_cast<int>(groups.size());
    GroupEmitter em(ops, max_targets, resynth_cap, split_diag, cz_to_cx);
    if (order == 1 || G <= 1) {
        for (int g = 0; g < G; ++g) em.group(groups[g], g, 1.0);
    } else if (order == 2) {
        // Symmetric Suzuki S2 with the middle group merged.
        for (int g = 0; g < G - 1; ++g) em.group(groups[g], g, 0.5);
        em.group(groups[G - 1], G - 1, 1.0);
        for (int g = G - 2; g >= 0; --g) em.group(groups[g], g, 0.5);
    } else {
        throw std::invalid_argument("trotter order must be 1 or 2");
    }
    em.flush();
    return ops;
}

double reference_sweeps(const std::vector<GroupSpec>& groups, int order) {
    // KernelStats sweeps of one reference group application
    // (statevector.cpp:156-286): H = 1, batched CNOT = 1/2, phase layer = 1,
    // diagonal = 1.
    double per_step = 0.0;
    for (const GroupSpec& g : groups) {
        int runs = 0;
        for (size_t k = 0; k < g.cnots.size(); ++k) {
            if (k == 0 || g.cnots[k].first != g.cnots[k - 1].first) ++runs;
        }
        const bool ph = !g.czs.empty() || !g.s_layer.empty();
        per_step += 2.0 * (double(g.h_pre.size() + g.h_post.size()) + 0.5 * runs + (ph ? 1 : 0)) + 1.0;
    }
    return order == 2 ? 2.0 * per_step : per_step;
}

void finalize_scales(std::vector<PassPlan*>& passes) {
    int cum = 0;
    for (PassPlan* pp : passes) cum += pp->butterflies;
    if (cum & 1) throw std::logic_error("plan_step: odd number of Hadamards in a step");
    // Deferred exact normalisation: butterflies are unnormalised, and
    // multiplying by 2^-e is exact in floating point, so the pending factor
    // is applied only in passes that already multiply every amplitude by a
    // phase (free), when it exceeds 2^48, or at the end of the step.
    int pending = 0;
    for (size_t p = 0; p < passes.size(); ++p) {
        PassPlan& pp = *passes[p];
        pending += pp.butterflies;
        bool has_phase = false;
        for (const PassStage& st : pp.stages) {
            if (st.kind == PassStage::POINT && !pp.points[st.point].terms.empty()) has_phase = true;
        }
        const bool last = p + 1 == passes.size();
        if (last || has_phase || pending >= 96) {
            pp.scale_exp = pending / 2;
            pending -= 2 * pp.scale_exp;
        } else {
            pp.scale_exp = 0;
        }
    }
    if (pending != 0) throw std::logic_error("plan_step: normalisation did not close");
}

namespace {

constexpr size_t kMaxDiagPerPass = 16384;

thread_local const PlannerKnobs* g_knobs = nullptr;

// WHT levels per pass (0 = unlimited): the plan's knob, else SDB_MAX_HDEPTH
int max_hadamard_depth() {
    if (g_knobs && g_knobs->max_hdepth >= 0) return g_knobs->max_hdepth;
    const char* e = std::getenv("SDB_MAX_HDEPTH");
    return e ? std::atoi(e) : 0;
}

bool defer_fixed_hadamards() {
    const char* e = std::getenv("SDB_DEFER_FIXED_H");
    return e && std::atoi(e) != 0;
}

// SDB_DRAM_PATTERN: 0 off, 1 prefer physical bits 3/5 (default), 2 also bits
// 4, 6..10 (measured: config 4 unchanged, config 3 +8 passes and 2% slower)
int dram_pattern_heuristic() {
    const char* e = std::getenv("SDB_DRAM_PATTERN");
    return e ? std::atoi(e) : 1;
}

// SDB_LOOKAHEAD: grow a pass's local set by the op whose closure schedules
// the most gates (1) instead of the first ready op in list order (0)
bool lookahead_growth() {
    if (g_knobs && g_knobs->lookahead >= 0) return g_knobs->lookahead != 0;
    const char* e = std::getenv("SDB_LOOKAHEAD");
    return e && std::atoi(e) != 0;
}

bool consolidate_enabled() {
    const char* e = std::getenv("SDB_CONSOLIDATE");
    return !e || std::atoi(e) != 0;
}

// Orders a pass's ops (valid in the given order) into few stages: all ready
// Hadamards form one WHT stage, then ready CNOTs, and diagonal ops only when
// no gate is ready, so each POINT stage collects every term it can.
std::vector<int> stage_order(const std::vector<Op>& ops, std::vector<int> sched) {
    std::sort(sched.begin(), sched.end());  // program order is a valid order
    const size_t m = sched.size();
    std::vector<std::vector<int>> preds(m);
    bool any_diag = false;
    for (size_t j = 0; j < m; ++j) {
        any_diag |= is_diag(ops[sched[j]]);
        for (size_t i = 0; i < j; ++i)
            if (!commute(ops[sched[i]], ops[sched[j]])) preds[j].push_back(static_cast<int>(i));
    }
    if (!any_diag) return sched;
    std::vector<char> taken(m, 0);
    std::vector<int> out;
    // SDB_CX_BATCH (default 1): every ready CNOT joins one CX run before the
    // next Hadamards (CNOT maps compose, and a WHT stage behind a pending map
    // costs a transpose: config 4's CZ -> CNOT passes went from c B c B c B ...
    // to one c); 0: one CNOT, then look for Hadamards again
    static const bool batch_cx = [] {
        const char* e = std::getenv("SDB_CX_BATCH");
        return !e || std::atoi(e) != 0;
    }();
    auto ready = [&](size_t j) {
        if (taken[j]) return false;
        for (int i : preds[j])
            if (!taken[i]) return false;
        return true;
    };
    while (out.size() < m) {
        bool progress = false;
        for (int cls = 0; cls < 3 && !progress; ++cls) {
            for (bool again = true; again;) {
                again = false;
                for (size_t j = 0; j < m; ++j) {
                    const Op& o = ops[sched[j]];
                    const int c = o.kind == Op::H ? 0 : o.kind == Op::CX ? 1 : 2;
                    if (c != cls || !ready(j)) continue;
                    taken[j] = 1;
                    out.push_back(sched[j]);
                    again = progress = true;
                    if (cls == 1 && !batch_cx) break;  // one CNOT, then look for Hadamards again
                }
                if (cls == 1 && progress) break;
            }
        }
        if (!progress) throw std::logic_error("stage_order: cyclic dependencies");
    }
    return out;
}

// Diagonal ops need no tile-local qubit, so each may sit anywhere between the
// last gate before it and the first gate after it that it does not commute
// with. Given the gate order the scheduler chose, every diagonal op therefore
// has an interval of gaps; stabbing all intervals with the fewest gaps
// (greedy by right end, optimal for intervals) merges them into the fewest
// POINT stages. Passes left without gates are dropped.
void consolidate_diagonals(const std::vector<Op>& ops, std::vector<std::vector<int>>& pass_ops,
                           std::vector<uint64_t>& pass_local) {
    std::vector<int> seq, pass_of;
    std::vector<int> diag;
    for (size_t p = 0; p < pass_ops.size(); ++p) {
        for (int id : pass_ops[p]) {
            if (is_diag(ops[id])) {
                diag.push_back(id);
            } else {
                seq.push_back(id);
                pass_of.push_back(static_cast<int>(p));
            }
        }
    }
    if (seq.empty() || diag.empty()) return;
    // gates per qubit they do not commute with a diagonal on (H: its qubit; CX: targets)
    std::vector<std::vector<int>> on(64);
    for (size_t i = 0; i < seq.size(); ++i) {
        const Op& g = ops[seq[i]];
        uint64_t m = g.kind == Op::H ? bitq(g.q) : g.targets;
        for (; m; m &= m - 1) on[std::countr_zero(m)].push_back(static_cast<int>(i));
    }
    struct Iv {
        int a, b, id;
    };
    std::vector<Iv> iv;
    iv.reserve(diag.size());
    for (int d : diag) {
        int a = 0, b = static_cast<int>(seq.size());
        for (uint64_t m = ops[d].support; m; m &= m - 1) {
            for (int i : on[std::countr_zero(m)]) {
                if (seq[i] < d) a = std::max(a, i + 1);
                else b = std::min(b, i);
            }
        }
        if (a > b) throw std::logic_error("consolidate_diagonals: schedule violates a dependency");
        iv.push_back({a, b, d});
    }
    std::sort(iv.begin(), iv.end(), [](const Iv& x, const Iv& y) { return x.b != y.b ? x.b < y.b : x.a < y.a; });
    std::vector<std::vector<int>> at(seq.size() + 1);
    int stab = -1;
    for (const Iv& v : iv) {
        if (stab < v.a) stab = v.b;
        at[stab].push_back(v.id);
    }
    std::vector<std::vector<int>> out(pass_ops.size());
    for (size_t g = 0; g <= seq.size(); ++g) {
        const int p = g < seq.size() ? pass_of[g] : pass_of.back();
        std::vector<int>& d = at[g];
        std::sort(d.begin(), d.end());
        out[p].insert(out[p].end(), d.begin(), d.end());
        if (g < seq.size()) out[p].push_back(seq[g]);
    }
    std::vector<std::vector<int>> kept;
    std::vector<uint64_t> kept_local;
    for (size_t p = 0; p < out.size(); ++p) {
        bool gate = false;
        for (int id : out[p]) gate |= !is_diag(ops[id]);
        if (!gate) continue;
        kept.push_back(std::move(out[p]));
        kept_local.push_back(pass_local[p]);
    }
    pass_ops = std::move(kept);
    pass_local = std::move(kept_local);
}

}  // namespace

StepPlan plan_step(const std::vector<Op>& ops, const std::vector<GroupSpec>& groups, int n_local,
                   int k, int n_fixed, const std::vector<int>& phys_of, bool finalize) {
    if (k > n_local) k = n_local;
    if (n_fixed > k) n_fixed = k;
    StepPlan plan;
    plan.tile_qubits = k;
    const size_t N = ops.size();
    const int n_logical = static_cast<int>(phys_of.size());

    // logical qubits currently stored at physical positions 0..n_fixed-1
    uint64_t fixed_logical = 0;
    std::vector<int> logical_of(64, -1);
    for (int q = 0; q < n_logical; ++q) logical_of[phys_of[q]] = q;
    for (int p = 0; p < n_fixed; ++p) {
        if (logical_of[p] >= 0) fixed_logical |= bitq(logical_of[p]);
    }
    // Qubits stored on other ranks (physical >= n_local) can never be local.
    uint64_t global_logical = 0;
    for (int q = 0; q < n_logical; ++q) {
        if (phys_of[q] >= n_local) global_logical |= bitq(q);
    }
    for (const Op& o : ops) {
        if (o.need & global_logical) {
            throw std::logic_error("plan_step: op needs a rank-global qubit (remap required)");
        }
    }

    // --- list scheduling with a sliding window and blocker counts
    constexpr size_t W = 768;
    std::vector<char> done(N, 0);
    std::vector<int> blockers(N, 0);
    size_t first = 0, hi = 0;
    auto extend = [&]() {
        const size_t want = std::min(N, first + W);
        for (; hi < want; ++hi) {
            int b = 0;
            for (size_t i = first; i < hi; ++i) {
                if (!done[i] && !commute(ops[i], ops[hi])) ++b;
            }
            blockers[hi] = b;
        }
    };
    std::vector<std::vector<int>> pass_ops;
    std::vector<uint64_t> pass_local;
    std::vector<int> hq(64, 0), dq(64, 0);
    uint64_t good_logical = 0, medium_logical = 0;
    if (dram_pattern_heuristic()) {
        for (int q = 0; q < n_logical; ++q)
            if ((phys_of[q] == 3 || phys_of[q] == 5) && phys_of[q] >= n_fixed && phys_of[q] < n_local) good_logical |= bitq(q);
        for (int q = 0; q < n_logical && dram_pattern_heuristic() >= 2; ++q)
            if ((phys_of[q] == 4 || (phys_of[q] >= 6 && phys_of[q] <= 10)) && phys_of[q] >= n_fixed && phys_of[q] < n_local)
                medium_logical |= bitq(q);
    }
    constexpr size_t kGoodLookahead = 64;
    const int max_depth = max_hadamard_depth();
    const bool defer_fixed = defer_fixed_hadamards();
    const bool gain_mode = lookahead_growth();
    constexpr size_t kGainCandidates = 48;
    while (first < N) {
        uint64_t L = fixed_logical;
        std::vector<int> sched;
        extend();
        int n_gates = 0;
        // Hadamard depth inside the pass: every further WHT level costs about
        // two shared-memory transposes per tile, so a pass stops at max_depth
        // levels (hq: depth of the last gate on a qubit, dq: of the last
        // diagonal containing it; diagonals depend only on gates).
        std::fill(hq.begin(), hq.end(), 0);
        std::fill(dq.begin(), dq.end(), 0);
        auto depth_of = [&](const Op& o) {
            int d = 0;
            for (uint64_t m = o.support; m; m &= m - 1) {
                const int q = std::countr_zero(m);
                d = std::max(d, is_diag(o) ? hq[q] : std::max(hq[q], dq[q]));
            }
            return d + (o.kind == Op::H ? 1 : 0);
        };
        auto depth_ok = [&](const Op& o) {
            if (max_depth > 0 && depth_of(o) > max_depth) return false;
            // Hadamards on the always-local qubits are deferred out of a second
            // WHT level: the next pass has them local anyway, and here they
            // would cost two extra transposes (in and out of registers)
            if ((defer_fixed || o.defer_deep) && o.kind == Op::H && (bitq(o.q) & fixed_logical) && depth_of(o) > 1)
                return false;
            return true;
        };
        for (;;) {
            if (n_gates >= kMaxOpsPerPass || sched.size() >= kMaxDiagPerPass) break;
            long pick = -1;
            for (size_t j = first; j < hi; ++j) {
                if (!done[j] && blockers[j] == 0 && (ops[j].need & ~L) == 0 && depth_ok(ops[j])) {
                    pick = static_cast<long>(j);
                    break;
                }
            }
            if (pick < 0 && gain_mode) {
                // Look-ahead growth: each distinct set of new qubits a ready op
                // would add is tried on a copy of the scheduler state, and the
                // one whose closure schedules the most gates per added qubit
                // wins (keeps the local set spatially coherent on chains, where
                // first-in-list growth takes every other qubit of a Bell-pair
                // group); ties keep list order.
                std::vector<uint64_t> tried;
                double best_gain = -1.0;
                for (size_t j = first; j < hi; ++j) {
                    if (done[j] || blockers[j] != 0 || std::popcount(L | ops[j].need) > k || !depth_ok(ops[j])) continue;
                    const uint64_t add = ops[j].need & ~L;
                    if (std::find(tried.begin(), tried.end(), add) != tried.end()) continue;
                    tried.push_back(add);
                    if (tried.size() > kGainCandidates) break;
                    const uint64_t L2 = L | add;
                    std::vector<char> d2(done.begin() + first, done.begin() + hi);
                    std::vector<int> b2(blockers.begin() + first, blockers.begin() + hi);
                    std::vector<int> hq2 = hq, dq2 = dq;
                    int gates = 0;
                    for (bool any = true; any;) {
                        any = false;
                        for (size_t i = first; i < hi; ++i) {
                            const size_t r = i - first;
                            if (d2[r] || b2[r] != 0 || (ops[i].need & ~L2)) continue;
                            const Op& o = ops[i];
                            int d = 0;
                            for (uint64_t m = o.support; m; m &= m - 1) {
                                const int q = std::countr_zero(m);
                                d = std::max(d, is_diag(o) ? hq2[q] : std::max(hq2[q], dq2[q]));
                            }
                            d += o.kind == Op::H ? 1 : 0;
                            if (max_depth > 0 && d > max_depth) continue;
                            for (uint64_t m = o.support; m; m &= m - 1) {
                                const int q = std::countr_zero(m);
                                if (is_diag(o)) dq2[q] = std::max(dq2[q], d);
                                else hq2[q] = std::max(hq2[q], d);
                            }
                            d2[r] = 1;
                            if (!is_diag(o)) ++gates;
                            for (size_t j2 = i + 1; j2 < hi; ++j2)
                                if (!d2[j2 - first] && !commute(o, ops[j2])) --b2[j2 - first];
                            any = true;
                        }
                    }
                    const double gain = double(gates) / double(std::max(1, std::popcount(add)));
                    if (gain > best_gain) {
                        best_gain = gain;
                        pick = static_cast<long>(j);
                    }
                }
                if (pick >= 0) L |= ops[pick].need;
            }
            if (pick < 0) {
                // HBM pattern: a tile with a local bit at physical 3 or 5 spreads
                // over twice the channels (tools/membench3: 8.3 -> 6.0 ms at
                // n=30 for otherwise high local bits), so a pass without one
                // takes such an op first, and a pass with one leaves the others
                // to later passes when it can.
                // Second tier: bits 4, 6..10 (7.1-7.4 ms) when no 3/5 is left.
                auto tier = [&](uint64_t m) { return (m & good_logical) ? 2 : (m & medium_logical) ? 1 : 0; };
                const int have = tier(L);
                long fallback = -1, best_up = -1;
                int best_up_tier = have;
                for (size_t j = first; j < hi; ++j) {
                    if (!done[j] && blockers[j] == 0 && std::popcount(L | ops[j].need) <= k && depth_ok(ops[j])) {
                        const int t = tier(ops[j].need & ~L);
                        if (!(good_logical | medium_logical)) {
                            pick = static_cast<long>(j);
                            break;
                        }
                        if (have == 2) {
                            if (t == 0) {
                                pick = static_cast<long>(j);
                                break;
                            }
                        } else if (t == 2) {
                            pick = static_cast<long>(j);
                            break;
                        } else if (t > best_up_tier) {
                            best_up_tier = t;
                            best_up = static_cast<long>(j);
                        }
                        if (fallback < 0) fallback = static_cast<long>(j);
                        if (have < 2 && j > first + kGoodLookahead) break;
                    }
                }
                if (pick < 0) pick = best_up >= 0 ? best_up : fallback;
                if (pick < 0) break;
                L |= ops[pick].need;
            }
            {
                const Op& o = ops[pick];
                const int d = depth_of(o);
                for (uint64_t m = o.support; m; m &= m - 1) {
                    const int q = std::countr_zero(m);
                    if (is_diag(o)) dq[q] = std::max(dq[q], d);
                    else hq[q] = std::max(hq[q], d);
                }
            }
            done[pick] = 1;
            sched.push_back(static_cast<int>(pick));
            if (!is_diag(ops[pick])) ++n_gates;
            for (size_t j = pick + 1; j < hi; ++j) {
                if (!done[j] && !commute(ops[pick], ops[j])) --blockers[j];
            }
            while (first < N && done[first]) ++first;
            extend();
        }
        if (sched.empty()) throw std::logic_error("plan_step: no schedulable op (tile too small?)");
        pass_ops.push_back(stage_order(ops, std::move(sched)));
        pass_local.push_back(L);
    }

    if (consolidate_enabled()) consolidate_diagonals(ops, pass_ops, pass_local);

    // --- lower each pass to physical stages
    int cum = 0;
    for (size_t p = 0; p < pass_ops.size(); ++p) {
        PassPlan pp;
        uint64_t Lphys = to_phys(pass_local[p], phys_of);
        // pad with the lowest free physical bits (keeps accesses contiguous)
        for (int b = 0; b < n_local && std::popcount(Lphys) < k; ++b) Lphys |= bitq(b);
        for (int b = 0; b < n_local; ++b) {
            if (Lphys & bitq(b)) pp.lpos.push_back(b);
        }
        std::vector<int> coord(64, -1);
        for (size_t j = 0; j < pp.lpos.size(); ++j) coord[pp.lpos[j]] = static_cast<int>(j);
        auto local_mask = [&](uint64_t logical) {
            uint32_t m = 0;
            while (logical) {
                const int q = std::countr_zero(logical);
                logical &= logical - 1;
                const int c = coord[phys_of[q]];
                if (c < 0) throw std::logic_error("plan_step: needed qubit not local");
                m |= 1u << c;
            }
            return m;
        };
        std::vector<int> s_count(64, 0);
        auto flush_point = [&]() {
            if (pp.stages.empty() || pp.stages.back().kind != PassStage::POINT) return;
            PointSpec& ps = pp.points[pp.stages.back().point];
            for (int b = 0; b < 64; ++b) {
                const int c = s_count[b] & 3;
                if (c & 1) ps.s1 |= bitq(b);
                if (c & 2) ps.s2 |= bitq(b);
                s_count[b] = 0;
            }
        };
        for (int id : pass_ops[p]) {
            const Op& o = ops[id];
            pp.op_ids.push_back(id);
            if (o.kind == Op::H) {
                flush_point();
                const uint32_t m = local_mask(bitq(o.q));
                if (!pp.stages.empty() && pp.stages.back().kind == PassStage::WHT) {
                    pp.stages.back().mask ^= m;
                } else {
                    PassStage st{PassStage::WHT};
                    st.mask = m;
                    pp.stages.push_back(st);
                }
            } else if (o.kind == Op::CX) {
                flush_point();
                PassStage st{PassStage::CX};
                st.mask = local_mask(o.targets);
                const int pc = phys_of[o.q];
                if (coord[pc] >= 0) st.ctrl_local = coord[pc];
                else st.ctrl_phys = pc;
                pp.stages.push_back(st);
            } else {
                if (pp.stages.empty() || pp.stages.back().kind != PassStage::POINT) {
                    PassStage st{PassStage::POINT};
                    st.point = static_cast<int>(pp.points.size());
                    pp.points.emplace_back();
                    pp.stages.push_back(st);
                }
                PointSpec& ps = pp.points[pp.stages.back().point];
                if (o.kind == Op::PH) {
                    uint64_t s = o.s_mask;
                    while (s) {
                        const int q = std::countr_zero(s);
                        s &= s - 1;
                        s_count[phys_of[q]] += o.dagger ? 3 : 1;
                    }
                    for (auto [a, b] : o.czs) ps.cz_masks.push_back(bitq(phys_of[a]) | bitq(phys_of[b]));
                } else {
                    const GroupSpec& g = groups[o.group];
                    const size_t t1 = o.t1 < 0 ? g.z_masks.size() : static_cast<size_t>(o.t1);
                    for (size_t t = static_cast<size_t>(o.t0); t < t1; ++t) {
                        ps.terms.push_back({to_phys(g.z_masks[t], phys_of), g.coeffs[t], o.dt_scale});
                    }
                }
            }
        }
        flush_point();
        // drop WHT stages that cancelled to nothing
        std::vector<PassStage> kept;
        for (const PassStage& st : pp.stages) {
            if (st.kind == PassStage::WHT && st.mask == 0) continue;
            kept.push_back(st);
        }
        pp.stages = std::move(kept);
        int levels = 0;
        for (const PassStage& st : pp.stages) {
            if (st.kind == PassStage::WHT) levels += std::popcount(st.mask);
        }
        pp.butterflies = levels;
        cum += levels;
        plan.passes.push_back(std::move(pp));
    }
    (void)cum;
    if (finalize) {
        std::vector<PassPlan*> ptrs;
        for (PassPlan& pp : plan.passes) ptrs.push_back(&pp);
        finalize_scales(ptrs);
    }
    plan.ref_sweeps = 0.0;
    return plan;
}

ShardedStep plan_sharded_step(const std::vector<Op>& ops, const std::vector<GroupSpec>& groups, int n_local,
                              int k, int n_fixed, const std::vector<int>& phys_in) {
    ShardedStep out;
    out.phys_in = phys_in;
    const int n = static_cast<int>(phys_in.size());
    const int g = n - n_local;
    std::vector<int> L = phys_in;
    auto global_set = [&]() {
        uint64_t G = 0;
        for (int q = 0; q < n; ++q) {
            if (L[q] >= n_local) G |= bitq(q);
        }
        return G;
    };
    std::vector<int> rem(ops.size());
    for (size_t i = 0; i < rem.size(); ++i) rem[i] = static_cast<int>(i);
    constexpr size_t W = 1024;

    // Chooses and applies one exchange bringing the global qubits that
    // `upcoming` (op indices into `stream`) needs first.
    auto make_exchange = [&](const std::vector<const Op*>& upcoming) {
        const uint64_t G = global_set();
        // the first op that needs a global qubit sets the mandatory part; later
        // ops' global needs are added while enough local qubits that the first
        // op does not need can be evicted for them
        uint64_t incoming = 0, protect = 0;
        int evictable = 0;
        for (const Op* o : upcoming) {
            const uint64_t want = o->need & G;
            if (!want) continue;
            if (!incoming) {
                incoming = want;
                protect = o->need & ~G;
                for (int q = 0; q < n; ++q) {
                    if (L[q] >= n_fixed && L[q] < n_local && !((protect >> q) & 1)) ++evictable;
                }
                if (std::popcount(incoming) > evictable) {
                    throw std::logic_error("plan_sharded_step: tile too small for the shard (op needs more local qubits)");
                }
                continue;
            }
            if (std::popcount(incoming | want) > std::min(g, evictable)) break;
            incoming |= want;
        }
        if (!incoming) throw std::logic_error("plan_sharded_step: exchange without a global need");
        const int gp = std::popcount(incoming);
        // next use of every qubit in the upcoming stream
        std::vector<size_t> next_use(n, SIZE_MAX);
        uint64_t seen = 0;
        for (size_t i = 0; i < upcoming.size() && seen != (n >= 64 ? ~0ull : ((1ull << n) - 1)); ++i) {
            uint64_t m = upcoming[i]->need & ~seen;
            seen |= upcoming[i]->need;
            while (m) {
                const int q = std::countr_zero(m);
                m &= m - 1;
                next_use[q] = i;
            }
        }
        // candidates: local qubits outside the always-local low bits
        std::vector<int> cand;
        for (int q = 0; q < n; ++q) {
            if (L[q] >= n_fixed && L[q] < n_local) cand.push_back(q);
        }
        const int t0 = n_local - gp;
        std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) {
            if (next_use[a] != next_use[b]) return next_use[a] > next_use[b];
            return L[a] > L[b];  // prefer qubits already high (fewer sigma moves)
        });
        if (static_cast<int>(cand.size()) < gp) throw std::logic_error("plan_sharded_step: no qubit to evict");
        std::vector<int> evict(cand.begin(), cand.begin() + gp);
        ExchangeSpec ex;
        ex.sigma.resize(n_local);
        for (int b = 0; b < n_local; ++b) ex.sigma[b] = b;
        // place evicted qubits on T = t0..n_local-1 (keep those already there)
        std::vector<int> tslot_owner(gp, -1);
        std::vector<int> pending;
        for (int e : evict) {
            if (L[e] >= t0) tslot_owner[L[e] - t0] = e;
            else pending.push_back(e);
        }
        std::vector<int> logical_at(n_local, -1);
        for (int q = 0; q < n; ++q) {
            if (L[q] < n_local) logical_at[L[q]] = q;
        }
        for (int e : pending) {
            int slot = 0;
            while (tslot_owner[slot] >= 0) ++slot;
            const int pe = L[e], pt = t0 + slot;
            std::swap(ex.sigma[pe], ex.sigma[pt]);
            const int other = logical_at[pt];
            if (other >= 0) L[other] = pe;
            L[e] = pt;
            logical_at[pe] = other;
            logical_at[pt] = e;
            tslot_owner[slot] = e;
        }
        // pair incoming global qubits (ascending global position) with T slots
        std::vector<int> inc;
        for (uint64_t m = incoming; m; m &= m - 1) inc.push_back(std::countr_zero(m));
        std::sort(inc.begin(), inc.end(), [&](int a, int b) { return L[a] < L[b]; });
        for (int i = 0; i < gp; ++i) {
            const int qi = inc[i], qe = tslot_owner[i];
            ex.swaps.emplace_back(L[qi], t0 + i);
            L[qe] = L[qi];
            L[qi] = t0 + i;
        }
        return ex;
    };

    while (true) {
        const uint64_t G = global_set();
        // dependency-closed set of remaining ops that need no global qubit
        std::vector<int> take, rest;
        {
            // an op is taken if it needs no global qubit and commutes with every
            // op held back before it; once many ops are held back the rest of
            // the step simply waits for the next segment
            constexpr size_t kMaxBlocked = 512;
            std::vector<int> blocked;
            for (size_t j = 0; j < rem.size(); ++j) {
                const Op& o = ops[rem[j]];
                bool ok = blocked.size() < kMaxBlocked && (o.need & G) == 0;
                if (ok) {
                    for (int b : blocked) {
                        if (!commute(ops[b], o)) {
                            ok = false;
                            break;
                        }
                    }
                }
                if (ok) {
                    take.push_back(rem[j]);
                } else {
                    rest.push_back(rem[j]);
                    if (blocked.size() < kMaxBlocked) blocked.push_back(rem[j]);
                }
            }
        }
        Segment seg;
        seg.phys_of = L;
        if (!take.empty()) {
            std::vector<Op> seg_ops;
            for (int i : take) seg_ops.push_back(ops[i]);
            seg.plan = plan_step(seg_ops, groups, n_local, k, n_fixed, L, false);
        }
        if (rest.empty()) {
            // lookahead into the next step: remap now if its first op needs a global qubit
            if (g > 0 && !ops.empty() && (ops[0].need & global_set())) {
                std::vector<const Op*> up;
                for (size_t i = 0; i < ops.size() && i < W; ++i) up.push_back(&ops[i]);
                seg.exchange_after = true;
                seg.ex = make_exchange(up);
            }
            out.segs.push_back(std::move(seg));
            break;
        }
        if (take.empty() && !out.segs.empty() && out.segs.back().plan.passes.empty()) {
            std::ostringstream os;
            os << "plan_sharded_step: no progress at op " << rem.front() << " (kind " << ops[rem.front()].kind
               << ", need 0x" << std::hex << ops[rem.front()].need << ", globals 0x" << G << ")";
            throw std::logic_error(os.str());
        }
        std::vector<const Op*> up;
        for (size_t i = 0; i < rest.size() && up.size() < W; ++i) up.push_back(&ops[rest[i]]);
        for (size_t i = 0; i < ops.size() && up.size() < W; ++i) up.push_back(&ops[i]);
        seg.exchange_after = true;
        seg.ex = make_exchange(up);
        out.segs.push_back(std::move(seg));
        rem = std::move(rest);
    }
    out.phys_out = L;
    // A segment that ends in an exchange stores its last pass out of place
    // through sigma; a segment without passes gets a permute-only pass.
    std::vector<PassPlan*> all;
    for (Segment& sg : out.segs) {
        if (sg.exchange_after) {
            if (sg.plan.passes.empty()) {
                PassPlan pp;
                const int kk = std::min(k, n_local);
                for (int b = 0; b < kk; ++b) pp.lpos.push_back(b);
                sg.plan.passes.push_back(std::move(pp));
            }
            sg.plan.passes.back().store_sigma = sg.ex.sigma;
            sg.plan.passes.back().xswaps = sg.ex.swaps;
        }
        for (PassPlan& pp : sg.plan.passes) all.push_back(&pp);
        out.n_exchanges += sg.exchange_after ? 1 : 0;
    }
    out.n_passes = static_cast<int>(all.size());
    finalize_scales(all);
    return out;
}

std::string describe_sharded_json(const ShardedStep& s) {
    std::ostringstream os;
    os << "{\"phys_in\":[";
    for (size_t i = 0; i < s.phys_in.size(); ++i) os << (i ? "," : "") << s.phys_in[i];
    os << "],\"phys_out\":[";
    for (size_t i = 0; i < s.phys_out.size(); ++i) os << (i ? "," : "") << s.phys_out[i];
    os << "],\"segments\":[";
    for (size_t i = 0; i < s.segs.size(); ++i) {
        const Segment& sg = s.segs[i];
        os << (i ? "," : "") << "{\"plan\":" << describe_json(sg.plan) << ",\"exchange\":";
        if (!sg.exchange_after) {
            os << "null";
        } else {
            os << "{\"sigma\":[";
            for (size_t b = 0; b < sg.ex.sigma.size(); ++b) os << (b ? "," : "") << sg.ex.sigma[b];
            os << "],\"swaps\":[";
            for (size_t b = 0; b < sg.ex.swaps.size(); ++b)
                os << (b ? "," : "") << "[" << sg.ex.swaps[b].first << "," << sg.ex.swaps[b].second << "]";
            os << "]}";
        }
        os << "}";
    }
    os << "]}";
    return os.str();
}

std::string describe(const StepPlan& p) {
    std::ostringstream os;
    os << "tile_qubits=" << p.tile_qubits << " passes=" << p.passes.size()
       << " ref_sweeps=" << p.ref_sweeps << "\n";
    for (size_t i = 0; i < p.passes.size(); ++i) {
        const PassPlan& pp = p.passes[i];
        os << "pass " << i << " local{";
        for (size_t j = 0; j < pp.lpos.size(); ++j) os << (j ? "," : "") << pp.lpos[j];
        os << "} ops=" << pp.op_ids.size() << " scale=2^-" << pp.scale_exp << " :";
        for (const PassStage& st : pp.stages) {
            if (st.kind == PassStage::WHT) os << " H[" << std::popcount(st.mask) << "]";
            else if (st.kind == PassStage::CX) os << " CX";
            else {
                const PointSpec& ps = pp.points[st.point];
                os << " P[cz" << ps.cz_masks.size() << ",t" << ps.terms.size() << "]";
            }
        }
        os << "\n";
    }
    return os.str();
}

std::string describe_json(const StepPlan& p) {
    std::ostringstream os;
    os.precision(17);
    os << "{\"tile_qubits\":" << p.tile_qubits << ",\"passes\":[";
    for (size_t i = 0; i < p.passes.size(); ++i) {
        const PassPlan& pp = p.passes[i];
        os << (i ? "," : "") << "{\"lpos\":[";
        for (size_t j = 0; j < pp.lpos.size(); ++j) os << (j ? "," : "") << pp.lpos[j];
        os << "],\"scale_exp\":" << pp.scale_exp << ",\"stages\":[";
        for (size_t j = 0; j < pp.stages.size(); ++j) {
            const PassStage& st = pp.stages[j];
            os << (j ? "," : "");
            if (st.kind == PassStage::WHT) {
                os << "{\"kind\":\"wht\",\"mask\":" << st.mask << "}";
            } else if (st.kind == PassStage::CX) {
                os << "{\"kind\":\"cx\",\"mask\":" << st.mask << ",\"ctrl_local\":" << st.ctrl_local
                   << ",\"ctrl_phys\":" << st.ctrl_phys << "}";
            } else {
                const PointSpec& ps = pp.points[st.point];
                os << "{\"kind\":\"point\",\"s1\":" << ps.s1 << ",\"s2\":" << ps.s2 << ",\"cz\":[";
                for (size_t k = 0; k < ps.cz_masks.size(); ++k) os << (k ? "," : "") << ps.cz_masks[k];
                os << "],\"terms\":[";
                for (size_t k = 0; k < ps.terms.size(); ++k) {
                    os << (k ? "," : "") << "[" << ps.terms[k].mask << "," << ps.terms[k].coeff << ","
                       << ps.terms[k].dt_scale << "]";
                }
                os << "]}";
            }
        }
        os << "]}";
    }
    os << "]}";
    return os.str();
}

KnobScope::KnobScope(const PlannerKnobs* k) : prev_(g_knobs) { g_knobs = k; }
KnobScope::~KnobScope() { g_knobs = prev_; }

}  // namespace sdb
