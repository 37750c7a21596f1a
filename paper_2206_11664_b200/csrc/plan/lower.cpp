// Pass -> micro-program lowering (host). See internal.hpp for the device
// semantics of CFG / BFLY / POINT / STORE.
//
// Register configs: each thread holds R = min(4, k) local coordinates in
// registers. A WHT stage's coordinates are covered in ascending chunks of
// R (the lowest coordinates first, so the final config of a pass tends to
// hold high coordinates and the store can go straight from registers to
// HBM with coalesced lanes); coordinates already in the current config are
// done in place. CNOT runs become a pending affine index map that the next
// transpose applies on its write side (no extra shared-memory traffic).
#include "lower.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
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
        outer.emplace_back(phys, T);
        identity = false;
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

uint32_t slot_mask(uint32_t coords, uint32_t cfg) {
    // slot j of a config <-> its j-th lowest coordinate
    uint32_t out = 0;
    int j = 0;
    for (uint32_t m = cfg; m; m &= m - 1, ++j) {
        if (coords & (m & (~m + 1u))) out |= 1u << j;
    }
    return out;
}

}  // namespace

HostPlanArrays lower_plan(const StepPlan& sp, int n_local, int table_threshold, int rbits) {
    HostPlanArrays A;
    for (const PassPlan& pp : sp.passes) {
        const int K = static_cast<int>(pp.lpos.size());
        const int R = std::min(rbits, K);
        const uint32_t all = K >= 32 ? ~0u : ((1u << K) - 1u);
        const uint32_t low3 = 7u & all;
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

        // upcoming WHT coordinates (for filling partial configs)
        std::vector<uint32_t> wht_after(pp.stages.size() + 1, 0);
        for (int i = static_cast<int>(pp.stages.size()) - 1; i >= 0; --i) {
            wht_after[i] = wht_after[i + 1] | (pp.stages[i].kind == PassStage::WHT ? pp.stages[i].mask : 0u);
        }
        uint32_t cur = 0;  // current config (0 = data still in the load buffer)
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
        auto emit_cfg = [&](uint32_t cfg) {
            MicroOpDev op{};
            op.kind = kOpCfg;
            op.mask = cfg;
            op.perm = -1;
            {
                // per-thread base: thread bits scattered into the non-register coordinates
                const int nt = 1 << (K - R);
                const uint32_t others = all & ~cfg;
                op.arg = pd.n_cfg++;
                for (int tid = 0; tid < nt; ++tid) {
                    uint32_t tb = 0, v = static_cast<uint32_t>(tid);
                    for (uint32_t m = others; m; m &= m - 1, v >>= 1) {
                        if (v & 1u) tb |= m & (~m + 1u);
                    }
                    A.cfg_tb.push_back(tb | (host_swz(tb) << 16));
                }
                uint32_t sw[4] = {0, 0, 0, 0};
                int j = 0;
                for (uint32_t m = cfg; m && j < 4; m &= m - 1, ++j) {
                    const int c = std::countr_zero(m);
                    sw[j] = host_swz(1u << c);
                    op.cidx |= static_cast<uint32_t>(c) << (8 * j);
                    op.c_off[j] = 1ull << pp.lpos[c];
                }
                op.swc01 = sw[0] | (sw[1] << 16);
                op.swc23 = sw[2] | (sw[3] << 16);
            }
            if (!P.identity) {
                PermDev pm{};
                for (int x = 0; x < 64; ++x) {
                    uint32_t lo = 0, hi = 0;
                    for (int j = 0; j < 6; ++j) {
                        if ((x >> j) & 1) {
                            if (j < K) lo ^= P.col[j];
                            if (j + 6 < K) hi ^= P.col[j + 6];
                        }
                    }
                    pm.lo[x] = static_cast<uint16_t>(host_swz(lo));
                    pm.hi[x] = static_cast<uint16_t>(host_swz(hi));
                }
                if (P.outer.size() > 16) throw std::logic_error("lower_plan: too many outer-controlled CNOT runs");
                pm.n_ctrl = static_cast<int>(P.outer.size());
                for (size_t j = 0; j < P.outer.size(); ++j) {
                    pm.ctrl_phys[j] = P.outer[j].first;
                    pm.flip[j] = host_swz(P.outer[j].second);
                }
                op.perm = static_cast<int>(A.perms.size());
                A.perms.push_back(pm);
                P = Affine(K);
                only_point = false;
            }
            if (cur != 0) ++transposes;
            A.ops.push_back(op);
            cur = cfg;
        };
        for (size_t si = 0; si < pp.stages.size(); ++si) {
            const PassStage& st = pp.stages[si];
            if (st.kind == PassStage::WHT) {
                only_point = false;
                uint32_t bits = st.mask;
                while (bits) {
                    if (cur != 0 && P.identity && (bits & cur)) {
                        const uint32_t doing = bits & cur;
                        {
                            MicroOpDev b{};
                            b.kind = kOpBfly;
                            b.mask = slot_mask(doing, cur);
                            b.perm = -1;
                            A.ops.push_back(b);
                        }
                        bits &= ~doing;
                        continue;
                    }
                    const uint32_t chunk = lowest_bits(bits, R);
                    emit_cfg(fill(chunk, (bits | wht_after[si + 1]) & ~chunk));
                }
            } else if (st.kind == PassStage::CX) {
                only_point = false;
                if (st.ctrl_local >= 0) P.compose_local(st.ctrl_local, st.mask);
                else P.compose_outer(st.ctrl_phys, st.mask);
            } else {
                if (cur == 0 || !P.identity) {
                    const uint32_t next = wht_after[si + 1];
                    emit_cfg(fill(lowest_bits(next & ~low3, R), next));
                }
                const PointSpec& ps = pp.points[st.point];
                PointDev pt{};
                pt.s1 = ps.s1;
                pt.s2 = ps.s2;
                pt.qt_off = -1;
                // CZ pairs by locality
                std::vector<std::pair<int, int>> ll;
                pt.lo_off = static_cast<int>(A.lo_pairs.size());
                pt.oo_off = static_cast<int>(A.oo_pairs.size());
                for (uint64_t m : ps.cz_masks) {
                    const int a = std::countr_zero(m);
                    const int b = 63 - std::countl_zero(m);
                    const bool la = (Lphys >> a) & 1, lb = (Lphys >> b) & 1;
                    if (la && lb) ll.emplace_back(coord[a], coord[b]);
                    else if (la) A.lo_pairs.push_back((uint32_t(coord[a]) << 8) | uint32_t(b));
                    else if (lb) A.lo_pairs.push_back((uint32_t(coord[b]) << 8) | uint32_t(a));
                    else A.oo_pairs.push_back(m);
                }
                pt.n_lo = static_cast<int>(A.lo_pairs.size()) - pt.lo_off;
                pt.n_oo = static_cast<int>(A.oo_pairs.size()) - pt.oo_off;
                if (!ll.empty()) {
                    pt.qt_off = static_cast<int>(A.qt_words.size());
                    const uint32_t N = 1u << K;
                    std::vector<uint64_t> words((N + 63) / 64, 0);
                    for (uint32_t l = 0; l < N; ++l) {
                        uint32_t par = 0;
                        for (auto [a, b] : ll) par ^= ((l >> a) & (l >> b) & 1u);
                        if (par) words[l >> 6] |= 1ull << (l & 63);
                    }
                    A.qt_words.insert(A.qt_words.end(), words.begin(), words.end());
                }
                pt.term_off = static_cast<int>(A.term_masks.size());
                pt.n_terms = static_cast<int>(ps.terms.size());
                pt.seg_off = static_cast<int>(A.segs.size());
                if (pt.n_terms > table_threshold && pd.table_point < 0) {
                    struct T {
                        uint32_t u;
                        uint64_t zh;
                        double c;
                    };
                    std::vector<T> ts;
                    for (const PointTerm& t : ps.terms) {
                        uint32_t u = 0;
                        for (int j = 0; j < K; ++j) {
                            if ((t.mask >> pp.lpos[j]) & 1) u |= 1u << j;
                        }
                        ts.push_back({u, t.mask & ~Lphys, t.coeff * t.dt_scale});
                    }
                    std::stable_sort(ts.begin(), ts.end(), [](const T& a, const T& b) { return a.u < b.u; });
                    uint32_t tm = 0;
                    for (size_t i = 0; i < ts.size();) {
                        size_t j = i;
                        while (j < ts.size() && ts[j].u == ts[i].u) ++j;
                        A.segs.push_back({ts[i].u, static_cast<int>(i), static_cast<int>(j), 0});
                        tm |= ts[i].u;
                        i = j;
                    }
                    pt.n_seg = static_cast<int>(A.segs.size()) - pt.seg_off;
                    pt.table_mask = tm;
                    for (const T& t : ts) {
                        A.term_masks.push_back(t.zh);
                        A.term_coeffs.push_back(t.c);
                    }
                    pd.flags |= kPassNeedsTable;
                    pd.table_point = static_cast<int>(A.points.size());
                } else {
                    for (const PointTerm& t : ps.terms) {
                        A.term_masks.push_back(t.mask);
                        A.term_coeffs.push_back(t.coeff * t.dt_scale);
                    }
                }
                {
                    MicroOpDev po{};
                    po.kind = kOpPoint;
                    po.perm = -1;
                    po.arg = static_cast<int>(A.points.size());
                    if (pp.scale_exp > 0 && !scale_placed && pt.n_terms > 0) {
                        po.mask = 1u;
                        scale_placed = true;
                    }
                    A.ops.push_back(po);
                }
                A.points.push_back(pt);
            }
        }
        if (cur == 0 || !P.identity) emit_cfg(fill(0, 0));
        // direct store when the register coordinates avoid coordinates 0..2
        MicroOpDev so{};
        so.kind = kOpStore;
        so.mask = (cur & low3) == 0 ? 1u : 0u;
        so.perm = -1;
        if (!(so.mask & 1u)) ++transposes;
        if (pp.scale_exp > 0 && !scale_placed) so.mask |= 2u;
        A.ops.push_back(so);
        pd.n_ops = static_cast<int>(A.ops.size()) - pd.op_off;
        A.passes.push_back(pd);
        A.pass_class.push_back(only_point ? 1 : 0);
        A.transposes.push_back(transposes);
    }
    return A;
}

std::string describe_program(const HostPlanArrays& a) {
    std::ostringstream os;
    for (size_t p = 0; p < a.passes.size(); ++p) {
        const PassDev& pd = a.passes[p];
        os << "pass " << p << " k=" << pd.k << " transposes=" << a.transposes[p] << " :";
        for (int i = 0; i < pd.n_ops; ++i) {
            const MicroOpDev& op = a.ops[pd.op_off + i];
            if (op.kind == kOpCfg) os << " CFG{" << std::hex << op.mask << std::dec << (op.perm >= 0 ? ",perm" : "") << "}";
            else if (op.kind == kOpBfly) os << " B" << std::popcount(op.mask);
            else if (op.kind == kOpPoint) {
                const PointDev& pt = a.points[op.arg];
                os << " P[t" << pt.n_terms << (pt.n_seg ? "T" : "") << ",lo" << pt.n_lo << ",oo" << pt.n_oo
                   << (pt.qt_off >= 0 ? ",qt" : "") << "]";
            } else os << ((op.mask & 1u) ? " ST" : " ST(smem)") << ((op.mask & 2u) ? "*s" : "");
        }
        os << "\n";
    }
    return os.str();
}

}  // namespace sdb
