// Pass -> micro-program lowering (host). See internal.hpp for the device
// semantics of LOAD / CFG / BFLY / POINT / STORE.
//
// Register configs: each thread holds R = min(4, k) local coordinates in
// registers. The tile is loaded straight into registers, so the LOAD config
// (and the config the STORE runs from) keeps local coordinates 0..2 on the
// thread lanes 0..2: every 8 lanes then cover one 128-byte line. A WHT
// stage's coordinates are covered in chunks of R; the chunk holding
// coordinates 0..2 is scheduled in the middle of the pass so the first and
// last configs stay coalesced. Coordinates already in the current config are
// done in place. CNOT runs become a pending affine index map that the next
// transpose applies on its write side (no extra shared-memory traffic).
#include "lower.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdlib>
#include <sstream>
#include <stdexcept>

namespace sdb {

namespace {

// Affine GF(2) map on local coordinates: x -> A x ^ sum_{outer ctrl set} flip.
struct Affine {
    std::vector<uint32_t> col;  // image of e_j
    std::vector<std::pair<int, uint32_t>> outer;
    bool identity = true;

    explicit Affine(int k) : col(k) {
        for (int j = 0; j < k; ++j) col[j] = 1u << j;
    }
    static uint32_t apply_cx(uint32_t v, int c, uint32_t T) { return ((v >> c) & 1u) ? v ^ T : v; }
    void compose_local(int c, uint32_t T) {
        for (uint32_t& v : col) v = apply_cx(v, c, T);
        for (auto& o : outer) o.second = apply_cx(o.second, c, T);
        identity = false;
    }
    void compose_outer(int phys, uint32_t T) {
        identity = false;
        for (auto& o : outer) {
            if (o.first == phys) {  // flips of one control bit add up (the map is affine)
                o.second ^= T;
                return;
            }
        }
        outer.emplace_back(phys, T);
    }
};

uint32_t lowest_bits(uint32_t m, int count) {
    uint32_t out = 0;
    for (int i = 0; i < count && m; ++i) {
        const uint32_t lo = m & (~m + 1u);
        out |= lo;
        m ^= lo;
    }
    return out;
}

uint32_t pext_host(uint32_t v, uint32_t mask) {
    uint32_t out = 0, bit = 1;
    for (uint32_t m = mask; m; m &= m - 1, bit <<= 1) {
        if (v & m & (~m + 1u)) out |= bit;
    }
    return out;
}

// Thread-coordinate order of a config: tid bit b <-> order[b]. Lanes 0..2
// take coordinates 0..2 when they are thread coordinates (coalescing);
// otherwise three coordinates with distinct residues mod 3 (conflict-free
// 128-bit shared-memory access, see swz in internal.hpp); the rest ascend.
std::vector<int> thread_order(uint32_t others, uint32_t prefer34 = 0, uint32_t prefer34b = 0) {
    std::vector<int> order;
    uint32_t rest = others;
    if ((others & 7u) == 7u) {
        order = {0, 1, 2};
        rest &= ~7u;
    } else {
        bool used[3] = {false, false, false};
        for (uint32_t m = others; m && order.size() < 3; m &= m - 1) {
            const int c = std::countr_zero(m);
            if (!used[c % 3]) {
                used[c % 3] = true;
                order.push_back(c);
                rest &= ~(1u << c);
            }
        }
    }
    // lanes 3 and 4 take preferred coordinates (bits a lane swap can reach)
    for (uint32_t pref : {prefer34, prefer34b}) {
        for (uint32_t m = rest & pref; m && order.size() < 5; m &= m - 1) {
            order.push_back(std::countr_zero(m));
            rest &= ~(m & (~m + 1u));
        }
    }
    for (uint32_t m = rest; m; m &= m - 1) order.push_back(std::countr_zero(m));
    return order;
}

// SDB_LANE_SWAPS bit 0: emit lane swaps, bit 1: steer coordinates onto lanes 3/4
int lane_swap_mode() {
    static const int m = [] {
        const char* e = std::getenv("SDB_LANE_SWAPS");
        return e ? std::atoi(e) : 3;
    }();
    return m;
}
bool lane_swaps_enabled() { return (lane_swap_mode() & 3) != 0; }
// POINT mode 5's sign-pattern table size (pass_device.cuh kPatTerms)
constexpr int kPatTermsHost = 6;

// SDB_SPLIT_POINTS: most pattern-table points a non-table POINT may be cut
// into (default 4, i.e. <= 24 terms; 1 or 0: never cut)
int point_split_max() {
    static const int v = [] {
        const char* e = std::getenv("SDB_SPLIT_POINTS");
        return e ? std::atoi(e) : 4;
    }();
    return v;
}

// SDB_CX_FOLD=0: trailing CNOT stages keep their own transpose
bool cx_fold_enabled() {
    const char* e = std::getenv("SDB_CX_FOLD");
    return !e || std::atoi(e) != 0;
}
// SDB_LANE_BFLY=0: lane swaps only (no in-place cross-lane butterflies)
// SDB_LANE_BFLY=2: also for coordinates a later stage needs (it fetches them
// with its own transpose)
int lane_bfly_mode() {
    const char* e = std::getenv("SDB_LANE_BFLY");  // read per plan (experiments switch it)
    return e ? std::atoi(e) : 1;
}
bool lane_bfly_enabled() { return lane_bfly_mode() != 0; }

// Factor cover of a table point: split the coordinates its terms touch into
// at most three disjoint sets of <= kMaxFacBits coordinates such that no
// term's local part spans two sets (connected components of the "appear in
// one term" relation, first-fit-decreasing into bins). Empty result: no such
// cover, use the full angle table with a sincos per amplitude.
constexpr int kMaxFacBits = 8;
// big_ok: a single factor may span up to kMaxBigFacBits coordinates (its
// table is then rebuilt only when the tile's sign pattern changes, so the
// caller allows it only when that happens a few times per CTA).
constexpr int kMaxBigFacBits = 11;
// Factors may share coordinates: each term only has to lie inside one of
// them (the phase is the product of the factors' tables, every term counted in
// the first factor that contains it). Greedy set growth over a few orders of
// the term supports; empty result: no cover with <= 3 factors of <= 8 bits.
std::vector<uint32_t> overlapping_cover(const std::vector<uint32_t>& us_in) {
    std::vector<uint32_t> us;
    for (uint32_t u : us_in)
        if (u) us.push_back(u);
    std::sort(us.begin(), us.end());
    us.erase(std::unique(us.begin(), us.end()), us.end());
    if (us.empty()) return {};
    uint64_t rng = 0x9e3779b97f4a7c15ull;
    for (int attempt = 0; attempt < 64; ++attempt) {
        std::vector<uint32_t> ord = us;
        if (attempt == 0) {
            std::stable_sort(ord.begin(), ord.end(),
                             [](uint32_t a, uint32_t b) { return std::popcount(a) > std::popcount(b); });
        } else {
            for (size_t i = ord.size(); i > 1; --i) {
                rng ^= rng << 13;
                rng ^= rng >> 7;
                rng ^= rng << 17;
                std::swap(ord[i - 1], ord[rng % i]);
            }
        }
        std::vector<uint32_t> sets;
        bool ok = true;
        for (uint32_t u : ord) {
            int best = -1, grow = 99;
            for (size_t f = 0; f < sets.size(); ++f) {
                const int g = std::popcount(u & ~sets[f]);
                if (std::popcount(sets[f] | u) <= kMaxFacBits && g < grow) {
                    grow = g;
                    best = static_cast<int>(f);
                }
            }
            if (best >= 0 && (grow == 0 || sets.size() == 3)) {
                sets[best] |= u;
            } else if (sets.size() < 3) {
                sets.push_back(u);
            } else if (best >= 0) {
                sets[best] |= u;
            } else {
                ok = false;
                break;
            }
        }
        if (ok) return sets;
    }
    return {};
}

std::vector<uint32_t> factor_cover(const std::vector<uint32_t>& us, uint32_t tm, bool big_ok) {
    if (big_ok && std::popcount(tm) <= kMaxBigFacBits && std::popcount(tm) > kMaxFacBits) return {tm};
    std::vector<int> parent(32);
    for (int i = 0; i < 32; ++i) parent[i] = i;
    auto find = [&](int x) {
        while (parent[x] != x) x = parent[x] = parent[parent[x]];
        return x;
    };
    for (uint32_t u : us) {
        if (!u) continue;
        const int a = std::countr_zero(u);
        for (uint32_t m = u & (u - 1); m; m &= m - 1) parent[find(std::countr_zero(m))] = find(a);
    }
    std::vector<uint32_t> comps;
    for (uint32_t m = tm; m; m &= m - 1) {
        const int c = std::countr_zero(m);
        if (find(c) != c) continue;
        uint32_t comp = 0;
        for (uint32_t q = tm; q; q &= q - 1) {
            if (find(std::countr_zero(q)) == c) comp |= q & (~q + 1u);
        }
        comps.push_back(comp);
    }
    std::stable_sort(comps.begin(), comps.end(),
                     [](uint32_t a, uint32_t b) { return std::popcount(a) > std::popcount(b); });
    // fewest bins first, then the most balanced (smallest total table size)
    for (int nb = 1; nb <= 3; ++nb) {
        const int cap = std::min(kMaxFacBits, (std::popcount(tm) + nb - 1) / nb + 2);
        std::vector<uint32_t> bins(nb, 0);
        bool ok = true;
        for (uint32_t c : comps) {
            int best = -1;
            for (int b = 0; b < nb; ++b) {
                if (std::popcount(bins[b] | c) > cap) continue;
                if (best < 0 || std::popcount(bins[b]) < std::popcount(bins[best])) best = b;
            }
            if (best < 0) {
                ok = false;
                break;
            }
            bins[best] |= c;
        }
        if (!ok) continue;
        std::vector<uint32_t> out;
        for (uint32_t b : bins) {
            if (b) out.push_back(b);
        }
        if (out.empty()) out.push_back(0);
        return out;
    }
    return overlapping_cover(us);
}

}  // namespace

HostPlanArrays lower_plan(const StepPlan& sp, int n_local, int table_threshold, int rbits) {
    HostPlanArrays A;
    for (const PassPlan& pp : sp.passes) {
        const int K = static_cast<int>(pp.lpos.size());
        const int R = std::min(rbits, K);
        const uint32_t all = K >= 32 ? ~0u : ((1u << K) - 1u);
        const bool coalesce = K - R >= 3;
        const uint32_t low3 = coalesce ? 7u : 0u;
        PassDev pd{};
        pd.k = K;
        uint64_t Lphys = 0;
        std::vector<int> coord(64, -1);
        for (int j = 0; j < K; ++j) {
            pd.lpos[j] = pp.lpos[j];
            Lphys |= 1ull << pp.lpos[j];
            coord[pp.lpos[j]] = j;
        }
        int no = 0;
        for (int b = 0; b < n_local; ++b) {
            if (!(Lphys & (1ull << b))) pd.opos[no++] = b;
        }
        pd.n_outer = no;
        pd.scale = std::ldexp(1.0, -pp.scale_exp);
        pd.op_off = static_cast<int>(A.ops.size());
        pd.table_point = -1;
        pd.n_cfg = 0;
        pd.cfg_off = static_cast<int>(A.cfg_tb.size());
        pd.rbits = R;
        pd.qt_off = static_cast<int>(A.qt_words.size());
        pd.tab_words = 0;
        pd.table_scale = 1.0;
        auto local_of = [&](uint64_t phys) {
            uint32_t m = 0;
            for (int j = 0; j < K; ++j) {
                if ((phys >> pp.lpos[j]) & 1) m |= 1u << j;
            }
            return m;
        };

        // upcoming WHT coordinates (for filling partial configs)
        std::vector<uint32_t> wht_after(pp.stages.size() + 1, 0);
        for (int i = static_cast<int>(pp.stages.size()) - 1; i >= 0; --i) {
            wht_after[i] = wht_after[i + 1] | (pp.stages[i].kind == PassStage::WHT ? pp.stages[i].mask : 0u);
        }
        // current config: register slot j holds coordinate regc[j], thread
        // bit b holds thr[b] (lanes are thread bits 0..4)
        uint32_t cur = 0;
        int regc[kMaxR] = {0, 0, 0, 0, 0};
        std::vector<int> thr;
        bool loaded = false;
        bool scale_placed = false;
        Affine P(K);
        int transposes = 0;
        bool only_point = true;
        auto fill = [&](uint32_t chunk, uint32_t prefer) {
            // complete `chunk` to R coordinates: preferred (upcoming WHT) coords
            // first, then high coordinates outside 0..2, then anything.
            uint32_t cfg = chunk;
            auto take = [&](uint32_t pool, bool high_first) {
                while (std::popcount(cfg) < R && (pool & ~cfg)) {
                    const uint32_t cand = pool & ~cfg;
                    const uint32_t b = high_first ? (1u << (31 - std::countl_zero(cand))) : (cand & (~cand + 1u));
                    cfg |= b;
                }
            };
            take(prefer & ~low3, false);
            take(all & ~low3, true);
            take(all, true);
            return cfg;
        };
        // the pending CNOT map P as a PermDev (swizzled-slot tables), P reset
        auto make_perm = [&]() {
            PermDev pm{};
            for (int x = 0; x < 64; ++x) {
                uint32_t lo = 0, hi = 0;
                for (int b = 0; b < 6; ++b) {
                    if ((x >> b) & 1) {
                        if (b < K) lo ^= P.col[b];
                        if (b + 6 < K) hi ^= P.col[b + 6];
                    }
                }
                pm.lo[x] = static_cast<uint16_t>(host_swz(lo));
                pm.hi[x] = static_cast<uint16_t>(host_swz(hi));
            }
            if (P.outer.size() > 32) throw std::logic_error("lower_plan: too many outer-controlled CNOT controls");
            pm.n_ctrl = static_cast<int>(P.outer.size());
            for (size_t b = 0; b < P.outer.size(); ++b) {
                pm.ctrl_phys[b] = P.outer[b].first;
                pm.flip[b] = host_swz(P.outer[b].second);
            }
            const int idx = static_cast<int>(A.perms.size());
            A.perms.push_back(pm);
            P = Affine(K);
            return idx;
        };
        // a config given explicitly (register coordinates, thread order)
        auto emit_explicit = [&](int kind, const int (&rc)[kMaxR], const std::vector<int>& order, uint32_t mask) {
            MicroOpDev op{};
            op.kind = kind;
            op.mask = mask;
            op.perm = -1;
            op.arg = pd.n_cfg++;
            const int nt = 1 << (K - R);
            for (int tid = 0; tid < nt; ++tid) {
                uint32_t tb = 0;
                for (size_t b = 0; b < order.size(); ++b) {
                    if ((tid >> b) & 1) tb |= 1u << order[b];
                }
                A.cfg_tb.push_back(tb | (host_swz(tb) << 16));
            }
            cur = 0;
            for (int j = 0; j < R; ++j) {
                const int c = rc[j];
                op.swc[j] = static_cast<uint16_t>(host_swz(1u << c));
                op.cidx |= static_cast<uint64_t>(c) << (8 * j);
                op.c_off[j] = 1ull << pp.lpos[c];
                regc[j] = c;
                cur |= 1u << c;
            }
            if (kind == kOpCfg && !P.identity) {
                op.perm = make_perm();
                only_point = false;
            }
            if (kind == kOpCfg) ++transposes;
            A.ops.push_back(op);
            thr = order;
        };
        // a config by its register set (ascending slots), thread order by rule
        auto emit = [&](int kind, uint32_t cfg, uint32_t prefer34 = 0, uint32_t prefer34b = 0) {
            int rc[kMaxR] = {0, 0, 0, 0, 0};
            int j = 0;
            for (uint32_t m = cfg; m && j < kMaxR; m &= m - 1, ++j) rc[j] = std::countr_zero(m);
            emit_explicit(kind, rc, thread_order(all & ~cfg, prefer34, prefer34b), cfg);
        };
        // register slot j <-> lane bit b through warp shuffles
        auto emit_swap = [&](int j, int b) {
            int rc[kMaxR] = {regc[0], regc[1], regc[2], regc[3], regc[4]};
            std::vector<int> order = thr;
            std::swap(rc[j], order[b]);
            emit_explicit(kOpSwap, rc, order, static_cast<uint32_t>(j | (b << 4)));
        };
        // LOAD (identity positions), then flush a pending CNOT map if any.
        auto load = [&](uint32_t cfg, uint32_t prefer34 = 0) {
            emit(kOpLoad, cfg, prefer34);
            loaded = true;
            if (!P.identity) emit(kOpCfg, cfg);
        };
        // the table goes to the POINT stage with the most real-angle terms
        int table_stage_point = -1;
        {
            size_t best = static_cast<size_t>(table_threshold);
            for (const PassStage& st : pp.stages) {
                if (st.kind != PassStage::POINT) continue;
                const size_t nt = pp.points[st.point].terms.size();
                if (nt > best) {
                    best = nt;
                    table_stage_point = st.point;
                }
            }
        }
        // CNOT stages already folded into an earlier transpose (below)
        std::vector<char> cx_folded(pp.stages.size(), 0);
        for (size_t si = 0; si < pp.stages.size(); ++si) {
            const PassStage& st = pp.stages[si];
            const uint32_t after = wht_after[si + 1];
            if (st.kind == PassStage::WHT) {
                only_point = false;
                uint32_t bits = st.mask;
                // lanes 3 and 4 exist (and keep lanes 0..2 untouched) for >= 32 threads
                const bool swaps = lane_swaps_enabled() && K - R >= 5;
                const bool emit_swaps = swaps && (lane_swap_mode() & 1);
                const bool steer = swaps && (lane_swap_mode() & 2);
                while (bits) {
                    if (loaded && P.identity && (bits & cur)) {
                        const uint32_t doing = bits & cur;
                        MicroOpDev b{};
                        b.kind = kOpBfly;
                        b.mask = 0;
                        for (int j = 0; j < R; ++j)
                            if ((doing >> regc[j]) & 1u) b.mask |= 1u << j;
                        b.perm = -1;
                        A.ops.push_back(b);
                        bits &= ~doing;
                        continue;
                    }
                    if (!loaded) {
                        const uint32_t chunk = lowest_bits(bits & ~low3, R);
                        const uint32_t cfg = fill(chunk, (bits | after) & ~chunk);
                        load(cfg, steer ? (bits & ~cfg) : 0u);
                        continue;
                    }
                    // coordinates left only on lanes 3/4: bring them into registers
                    // with shuffles (a fraction of a transpose's cost) in exchange
                    // for register coordinates this stage is done with
                    if (emit_swaps && P.identity) {
                        const uint32_t lanes34 = (1u << thr[3]) | (1u << thr[4]);
                        if ((bits & ~lanes34) == 0) {
                            for (int b = 3; b <= 4; ++b) {
                                if (!((bits >> thr[b]) & 1u)) continue;
                                if (lane_bfly_enabled() && (lane_bfly_mode() == 2 || !((after >> thr[b]) & 1u))) {
                                    // no later stage of the pass needs the coordinate in a
                                    // register: butterfly it across lanes in place
                                    MicroOpDev y{};
                                    y.kind = kOpLaneBfly;
                                    y.mask = static_cast<uint32_t>(b);
                                    y.perm = -1;
                                    A.ops.push_back(y);
                                    bits &= ~(1u << thr[b]);
                                    continue;
                                }
                                int jbest = -1;
                                for (int j = 0; j < R; ++j) {
                                    if ((bits >> regc[j]) & 1u) continue;
                                    if (jbest < 0 || (((after >> regc[jbest]) & 1u) && !((after >> regc[j]) & 1u))) jbest = j;
                                }
                                emit_swap(jbest, b);
                            }
                            continue;
                        }
                    }
                    uint32_t chunk;
                    if (bits & low3) {
                        chunk = bits & low3;
                        chunk |= lowest_bits(bits & ~low3, R - std::popcount(chunk));
                    } else {
                        chunk = lowest_bits(bits, R);
                    }
                    const uint32_t cfg = fill(chunk, (bits | after) & ~chunk);
                    // The pass's last transpose (it takes every remaining coordinate
                    // of its last WHT stage): CNOT stages right behind this stage
                    // that touch none of those coordinates commute with the
                    // butterflies still to come, so they ride this transpose's
                    // write side instead of costing a transpose of their own
                    // before the store (config 4: 3 -> 2 transposes in such passes).
                    if (cx_fold_enabled() && after == 0 && (chunk & ~bits) == 0 && (bits & ~chunk) == 0) {
                        size_t sj = si + 1;
                        uint32_t sup = 0;
                        for (; sj < pp.stages.size() && pp.stages[sj].kind == PassStage::CX; ++sj)
                            sup |= pp.stages[sj].mask | (pp.stages[sj].ctrl_local >= 0 ? 1u << pp.stages[sj].ctrl_local : 0u);
                        if (sj > si + 1 && (sup & bits) == 0) {
                            for (size_t c = si + 1; c < sj; ++c) {
                                const PassStage& cs = pp.stages[c];
                                if (cs.ctrl_local >= 0) P.compose_local(cs.ctrl_local, cs.mask);
                                else P.compose_outer(cs.ctrl_phys, cs.mask);
                                cx_folded[c] = 1;
                            }
                        }
                    }
                    emit(kOpCfg, cfg, steer ? (bits & ~cfg) : 0u, steer ? (after & ~cfg) : 0u);
                }
            } else if (st.kind == PassStage::CX) {
                only_point = false;
                if (cx_folded[si]) continue;
                if (st.ctrl_local >= 0) P.compose_local(st.ctrl_local, st.mask);
                else P.compose_outer(st.ctrl_phys, st.mask);
            } else {
                if (!loaded) {
                    load(fill(lowest_bits(after & ~low3, R), after));
                } else if (!P.identity) {
                    emit(kOpCfg, fill(lowest_bits(after & ~low3, R), after));
                }
                const PointSpec& ps = pp.points[st.point];
                PointDev pt{};
                pt.s1L = local_of(ps.s1);
                pt.s2L = local_of(ps.s2);
                pt.s1H = ps.s1 & ~Lphys;
                pt.s2H = ps.s2 & ~Lphys;
                pt.qt_word = -1;
                // CZ pairs by locality
                std::vector<std::pair<int, int>> ll;
                pt.lo_off = static_cast<int>(A.lo_pairs.size());
                pt.oo_off = static_cast<int>(A.oo_pairs.size());
                // Pairs with an outer qubit only depend on the tile: grouped by
                // outer bit, a tile needs one test per outer bit instead of one
                // per pair (config 5 groups carry ~180 CZs): local-outer pairs
                // as (local mask << 8) | outer bit, outer-outer pairs as
                // (1 << a) | mask of a's partners above a. CZ^2 = 1, so XOR.
                std::vector<uint32_t> lo_by(64, 0);
                std::vector<uint64_t> oo_by(64, 0);
                for (uint64_t m : ps.cz_masks) {
                    const int a = std::countr_zero(m);
                    const int b = 63 - std::countl_zero(m);
                    const bool la = (Lphys >> a) & 1, lb = (Lphys >> b) & 1;
                    if (la && lb) ll.emplace_back(coord[a], coord[b]);
                    else if (la) lo_by[b] ^= 1u << coord[a];
                    else if (lb) lo_by[a] ^= 1u << coord[b];
                    else oo_by[a] ^= 1ull << b;
                }
                for (int b = 0; b < 64; ++b)
                    if (lo_by[b]) A.lo_pairs.push_back((lo_by[b] << 8) | uint32_t(b));
                for (int a = 0; a < 64; ++a)
                    if (oo_by[a]) A.oo_pairs.push_back((1ull << a) | oo_by[a]);
                pt.n_lo = static_cast<int>(A.lo_pairs.size()) - pt.lo_off;
                pt.n_oo = static_cast<int>(A.oo_pairs.size()) - pt.oo_off;
                if (!ll.empty()) {
                    pt.qt_word = static_cast<int>(A.qt_words.size()) - pd.qt_off;
                    const uint32_t N = 1u << K;
                    std::vector<uint64_t> words((N + 63) / 64, 0);
                    for (uint32_t l = 0; l < N; ++l) {
                        uint32_t par = 0;
                        for (auto [a, b] : ll) par ^= ((l >> a) & (l >> b) & 1u);
                        if (par) words[l >> 6] |= 1ull << (l & 63);
                    }
                    A.qt_words.insert(A.qt_words.end(), words.begin(), words.end());
                }
                pt.term_off = static_cast<int>(A.term_hmask.size());
                pt.n_terms = static_cast<int>(ps.terms.size());
                pt.seg_off = static_cast<int>(A.segs.size());
                if (st.point == table_stage_point) {
                    struct T {
                        uint32_t u;
                        uint64_t zh;
                        double c;
                    };
                    std::vector<T> ts;
                    uint32_t tm = 0;
                    for (const PointTerm& t : ps.terms) {
                        const uint32_t u = local_of(t.mask);
                        tm |= u;
                        ts.push_back({u, t.mask & ~Lphys, t.coeff * t.dt_scale});
                    }
                    std::vector<uint32_t> us;
                    uint64_t pm_mixed = 0;  // outer bits of terms with local support
                    for (const T& t : ts) {
                        us.push_back(t.u);
                        if (t.u) pm_mixed |= t.zh;
                    }
                    // a big single table pays off when each CTA sees ~1-2 sign patterns:
                    // 2^(n_outer - |pm|) tiles per pattern >= tiles per CTA (~2^n_outer / 296)
                    const bool big_ok = std::popcount(pm_mixed) <= 8;
                    const std::vector<uint32_t> facs = factor_cover(us, tm, big_ok);
                    pt.table_mask = tm;
                    pt.table_bits = std::popcount(tm);
                    pt.n_fac = static_cast<int>(facs.size());
                    std::vector<int> fac_of(ts.size(), 0);
                    if (pt.n_fac > 0) {
                        int off = 0;
                        for (int f = 0; f < pt.n_fac; ++f) {
                            pt.fac_mask[f] = facs[f];
                            pt.fac_bits[f] = std::popcount(facs[f]);
                            pt.fac_coff[f] = off;
                            off += 2 * (1 << pt.fac_bits[f]);
                        }
                        pd.tab_words = off;
                        for (size_t i = 0; i < ts.size(); ++i) {
                            int f = 0;
                            while (f + 1 < pt.n_fac && (ts[i].u & ~facs[f])) ++f;
                            fac_of[i] = f;
                            ts[i].u = pext_host(ts[i].u, facs[f]);
                        }
                    } else {
                        pd.tab_words = std::max(2, 1 << pt.table_bits);
                        for (T& t : ts) t.u = pext_host(t.u, tm);
                    }
                    std::vector<size_t> ord(ts.size());
                    for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
                    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
                        return fac_of[a] != fac_of[b] ? fac_of[a] < fac_of[b] : ts[a].u < ts[b].u;
                    });
                    std::vector<T> sorted;
                    std::vector<int> sfac;
                    for (size_t i : ord) {
                        sorted.push_back(ts[i]);
                        sfac.push_back(fac_of[i]);
                    }
                    for (size_t i = 0; i < sorted.size();) {
                        size_t j = i;
                        while (j < sorted.size() && sorted[j].u == sorted[i].u && sfac[j] == sfac[i]) ++j;
                        A.segs.push_back({sorted[i].u, static_cast<int>(i), static_cast<int>(j), sfac[i]});
                        i = j;
                    }
                    pt.n_seg = static_cast<int>(A.segs.size()) - pt.seg_off;
                    for (int f = 0; f < pt.n_fac; ++f) {
                        pt.fac_sbeg[f] = pt.n_seg;
                        pt.fac_send[f] = 0;
                        for (int sg = 0; sg < pt.n_seg; ++sg) {
                            if (A.segs[pt.seg_off + sg].fac != f) continue;
                            pt.fac_sbeg[f] = std::min(pt.fac_sbeg[f], sg);
                            pt.fac_send[f] = std::max(pt.fac_send[f], sg + 1);
                        }
                        if (pt.fac_send[f] == 0) pt.fac_sbeg[f] = 0;
                    }
                    // Terms with no local support (u = 0) give a phase that is
                    // constant over the tile: in factor mode it is precomputed
                    // per tile (tile_phase) instead of entering the tables, so
                    // the tables depend only on the outer bits of mixed terms.
                    pt.c0_seg = -1;
                    if (pt.n_fac > 0 && pt.n_seg > 0 && A.segs[pt.seg_off].fac == 0 && A.segs[pt.seg_off].u == 0) {
                        pt.c0_seg = 0;
                        pt.fac_sbeg[0] = 1;
                        if (pt.fac_send[0] < 1) pt.fac_send[0] = 1;
                    }
                    for (const T& t : sorted) {
                        A.term_hmask.push_back(t.zh);
                        A.term_lmask.push_back(0);
                        A.term_coeffs.push_back(t.c);
                    }
                    pd.flags |= kPassNeedsTable;
                    pd.table_point = static_cast<int>(A.points.size());
                } else {
                    for (const PointTerm& t : ps.terms) {
                        A.term_hmask.push_back(t.mask & ~Lphys);
                        A.term_lmask.push_back(local_of(t.mask));
                        A.term_coeffs.push_back(t.coeff * t.dt_scale);
                    }
                }
                // A point other than the pass's table point with more terms than
                // one sign-pattern table holds (kPatTermsHost) would sum its terms
                // and take a sincos per amplitude (modes 1/2); it is cut into
                // consecutive points of <= kPatTermsHost terms instead, each a
                // per-tile pattern table (mode 5) and one complex multiply per
                // amplitude. The first carries the S/CZ quarter turns; the phases
                // multiply, so only the summation order changes.
                int n_chunks = 1;
                if (pd.table_point != static_cast<int>(A.points.size()) && pt.n_terms > kPatTermsHost) {
                    const int c = (pt.n_terms + kPatTermsHost - 1) / kPatTermsHost;
                    if (c <= point_split_max()) n_chunks = c;
                }
                const int all_terms = pt.n_terms;
                if (n_chunks > 1) pt.n_terms = kPatTermsHost;
                for (int chunk = 0; chunk < n_chunks; ++chunk) {
                    if (chunk > 0) {
                        pt.term_off += kPatTermsHost;
                        pt.n_terms = std::min(kPatTermsHost, all_terms - chunk * kPatTermsHost);
                        pt.s1L = pt.s2L = 0;
                        pt.s1H = pt.s2H = 0;
                        pt.n_lo = pt.n_oo = 0;
                        pt.qt_word = -1;
                    }
                    MicroOpDev po{};
                    po.kind = kOpPoint;
                    po.perm = -1;
                    po.arg = static_cast<int>(A.points.size());
                    // per-config constants of this point: compact table index of each
                    // register coordinate (swc01/swc23) and QT(r_s) for the 2^R
                    // register combinations r_s (pad, bit s)
                    std::vector<uint32_t> cbits;
                    for (int j = 0; j < R; ++j) cbits.push_back(1u << regc[j]);
                    if (pd.table_point == static_cast<int>(A.points.size())) {
                        for (size_t j = 0; j < cbits.size(); ++j)
                            po.swc[j] = static_cast<uint16_t>(pext_host(cbits[j], pt.table_mask));
                        for (int f = 0; f < pt.n_fac; ++f)
                            for (size_t j = 0; j < cbits.size(); ++j)
                                po.fo[f][j] = static_cast<uint16_t>(host_swz(pext_host(cbits[j], pt.fac_mask[f])));
                    }
                    uint32_t qr = 0;
                    if (pt.qt_word >= 0) {
                        const uint64_t* words = A.qt_words.data() + pd.qt_off + pt.qt_word;
                        for (int sidx = 0; sidx < (1 << cbits.size()); ++sidx) {
                            uint32_t r = 0;
                            for (size_t j = 0; j < cbits.size(); ++j) {
                                if ((sidx >> j) & 1) r |= cbits[j];
                            }
                            if ((words[r >> 6] >> (r & 63)) & 1ull) qr |= 1u << sidx;
                        }
                    }
                    po.pad = qr;
                    if (pp.scale_exp > 0 && !scale_placed && pt.n_terms > 0) {
                        po.mask = 1u;
                        scale_placed = true;
                        if (pd.table_point == static_cast<int>(A.points.size()) && pt.n_fac > 0) pd.table_scale = pd.scale;
                    }
                    A.ops.push_back(po);
                    A.points.push_back(pt);
                }
            }
        }
        if (!loaded) {
            load(fill(0, 0));
        }
        // A CNOT map still pending at the end is applied by the store's
        // addressing (no transpose) when the lanes stay coalesced.
        int store_perm_idx = -1;
        // ... only when the map keeps coordinates 0..2 in place and out of every
        // other image (each 8-lane group still writes one 128-byte line);
        // otherwise the stores would scatter 16-byte pieces (config 5: 7.8 ms
        // passes at n=28, 6x the pass roofline) and a transpose is cheaper
        bool lanes_kept = true;
        for (int j = 0; j < K; ++j)
            lanes_kept &= ((low3 >> j) & 1u) ? P.col[j] == (1u << j) : (P.col[j] & low3) == 0u;
        for (const auto& o : P.outer) lanes_kept &= (o.second & low3) == 0u;
        if (loaded && !P.identity && !(cur & low3) && pp.store_sigma.empty() && lanes_kept) {
            store_perm_idx = make_perm();
            only_point = false;
        } else if (!P.identity || (cur & low3)) {
            emit(kOpCfg, fill(0, 0));
        }
        MicroOpDev so{};
        so.kind = kOpStore;
        so.perm = store_perm_idx;
        // An in-place store through a CNOT map writes other warps' positions:
        // without a transpose (block barrier) since the load, warps of a CTA
        // may still be loading them (or be a tile behind), so the store syncs.
        if (store_perm_idx >= 0 && transposes == 0) so.mask |= 4u;
        if (!pp.xswaps.empty()) {
            pd.x_bits = static_cast<int>(pp.xswaps.size());
            pd.x_t0 = n_local - pd.x_bits;
            for (int i = 0; i < pd.x_bits && i < 8; ++i) pd.x_gpos[i] = pp.xswaps[i].first;
        }
        if (!pp.store_sigma.empty()) {
            pd.store_perm = 1;
            for (int j = 0; j < K; ++j) pd.st_lpos[j] = pp.store_sigma[pp.lpos[j]];
            for (int j = 0; j < pd.n_outer; ++j) pd.st_opos[j] = pp.store_sigma[pd.opos[j]];
            for (int j = 0; j < R; ++j) so.c_off[j] = 1ull << pp.store_sigma[pp.lpos[regc[j]]];
        }
        if (pp.scale_exp > 0 && !scale_placed) so.mask |= 2u;
        A.ops.push_back(so);
        pd.n_ops = static_cast<int>(A.ops.size()) - pd.op_off;
        pd.n_qt_words = static_cast<int>(A.qt_words.size()) - pd.qt_off;
        // Per-tile phase tables depend on the tile only through the outer bits
        // of the table terms (PM). Those bits go to the top of the tile index,
        // so a CTA walking t, t + grid, ... keeps the same table for long runs
        // of tiles and rebuilds it only when t >> pat_shift changes.
        pd.pat_shift = 64;
        pd.tphase_off = -1;
        static const bool reorder = [] {
            const char* e = std::getenv("SDB_TABLE_REUSE");
            return !e || std::atoi(e) != 0;
        }();
        if (pd.table_point >= 0 && reorder) {
            const PointDev& tp = A.points[pd.table_point];
            uint64_t pm = 0;
            for (int sg = 0; sg < tp.n_seg; ++sg) {
                if (sg == tp.c0_seg) continue;  // tile-constant terms: tile_phase
                const SegDev& d = A.segs[tp.seg_off + sg];
                for (int q = d.begin; q < d.end; ++q) pm |= A.term_hmask[tp.term_off + q];
            }
            if (tp.c0_seg >= 0) pd.tphase_off = 0;  // assigned by the executor (tile_phase buffer)
            std::vector<int> rest, top;
            for (int j = 0; j < pd.n_outer; ++j) ((pm >> pd.opos[j]) & 1 ? top : rest).push_back(pd.opos[j]);
            int j = 0;
            for (int b : rest) pd.opos[j++] = b;
            for (int b : top) pd.opos[j++] = b;
            pd.pat_shift = static_cast<int>(rest.size());
            static const bool blocked = [] {
                const char* e = std::getenv("SDB_BLOCKED");
                return !e || std::atoi(e) != 0;
            }();
            pd.blocked = blocked ? 1 : 0;
            if (!pp.store_sigma.empty()) {
                for (int q = 0; q < pd.n_outer; ++q) pd.st_opos[q] = pp.store_sigma[pd.opos[q]];
            }
        }
        A.passes.push_back(pd);
        A.pass_class.push_back(only_point ? 1 : 0);
        A.transposes.push_back(transposes);
    }
    return A;
}

void verify_lowering(const HostPlanArrays& A) {
    // Every register config op must place the element with local index l in
    // the thread/register its tables say; only SWAP moves data without going
    // through those tables, so simulate its shuffles and compare.
    for (size_t p = 0; p < A.passes.size(); ++p) {
        const PassDev& pd = A.passes[p];
        const int R = pd.rbits, NT = 1 << (pd.k - R), NR = 1 << R;
        auto label = [&](const MicroOpDev& op, int tid, int s) {
            uint32_t l = A.cfg_tb[pd.cfg_off + static_cast<size_t>(op.arg) * NT + tid] & 0xffffu;
            for (int j = 0; j < R; ++j)
                if ((s >> j) & 1) l |= 1u << ((op.cidx >> (8 * j)) & 255u);
            return l;
        };
        const MicroOpDev* prev = nullptr;
        for (int i = 0; i < pd.n_ops; ++i) {
            const MicroOpDev& op = A.ops[pd.op_off + i];
            if (op.kind == kOpSwap) {
                if (!prev) throw std::logic_error("verify_lowering: swap before load");
                const int J = static_cast<int>(op.mask & 15u), B = static_cast<int>(op.mask >> 4);
                for (int tid = 0; tid < NT; ++tid) {
                    const bool hi = (tid >> B) & 1;
                    const int partner = tid ^ (1 << B);
                    for (int s = 0; s < NR; ++s) {
                        // where register s of thread tid gets its value from (lane_swap)
                        int st = tid, ss = s;
                        const bool sj = (s >> J) & 1;
                        if (hi && !sj) { st = partner; ss = s | (1 << J); }
                        if (!hi && sj) { st = partner; ss = s & ~(1 << J); }
                        if (label(op, tid, s) != label(*prev, st, ss)) {
                            std::ostringstream os;
                            os << "verify_lowering: pass " << p << " op " << i << " swap(" << J << "," << B
                               << ") tid " << tid << " s " << s;
                            throw std::logic_error(os.str());
                        }
                    }
                }
            }
            if (op.kind == kOpLoad || op.kind == kOpCfg || op.kind == kOpSwap) prev = &op;
        }
    }
}

std::string describe_program(const HostPlanArrays& a) {
    std::ostringstream os;
    for (size_t p = 0; p < a.passes.size(); ++p) {
        const PassDev& pd = a.passes[p];
        os << "pass " << p << " k=" << pd.k << " transposes=" << a.transposes[p] << " :";
        for (int i = 0; i < pd.n_ops; ++i) {
            const MicroOpDev& op = a.ops[pd.op_off + i];
            if (op.kind == kOpLoad) os << " LD{" << std::hex << op.mask << std::dec << "}";
            else if (op.kind == kOpCfg) os << " CFG{" << std::hex << op.mask << std::dec << (op.perm >= 0 ? ",perm" : "") << "}";
            else if (op.kind == kOpBfly) os << " B" << std::popcount(op.mask);
            else if (op.kind == kOpSwap) os << " X" << (op.mask & 15u) << ":" << (op.mask >> 4);
            else if (op.kind == kOpLaneBfly) os << " Y" << op.mask;
            else if (op.kind == kOpPoint) {
                const PointDev& pt = a.points[op.arg];
                std::string tdesc;
                if (pt.n_seg && pt.n_fac) {
                    tdesc = "F";
                    for (int f = 0; f < pt.n_fac; ++f) tdesc += (f ? "+" : "") + std::to_string(pt.fac_bits[f]);
                } else if (pt.n_seg) {
                    tdesc = "T" + std::to_string(pt.table_bits);
                }
                os << " P[t" << pt.n_terms << tdesc << ",lo" << pt.n_lo
                   << ",oo" << pt.n_oo << (pt.qt_word >= 0 ? ",qt" : "") << "]";
            } else os << " ST" << ((op.mask & 2u) ? "*s" : "");
        }
        os << "\n";
    }
    return os.str();
}

}  // namespace sdb
