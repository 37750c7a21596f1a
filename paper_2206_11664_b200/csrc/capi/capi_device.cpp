// extern "C" device entry points: state lifecycle, the reference's
// single-sweep kernels, and the fused Trotter plan (evolve_grouped).
#include <cuda_runtime_api.h>

#include <algorithm>
#include <bit>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>

#include "../plan/lower.hpp"
#include "exchange.hpp"
#include "../cuda/jit.hpp"
#include "../plan/planner.hpp"
#include "guard.hpp"

namespace sdb {
void write_text_out(const std::string& s, char* buf, size_t cap, size_t* len);
}

struct sd_state {
    sdb::StateImpl impl;
};

// One planned Trotter step for a given starting layout (segments, remaps),
// lowered and uploaded. Plans are cached per layout: the layout sequence of a
// sharded evolution cycles after a few steps.
struct StepExec {
    sdb::ShardedStep ss;
    std::vector<sdb::PassDev> host_passes;
    std::vector<int> pass_class;  // 0 fused, 1 diagonal-only
    std::vector<int> seg_first, seg_count;
    std::vector<void*> jit_fn;    // specialised kernel per pass (nullptr = interpreter)
    std::vector<size_t> smem;     // dynamic shared memory per pass
    std::vector<int> threads;     // block size per specialised pass kernel (0: the kernel's default)
    sdb::PlanDev dev{};
    void* dev_block = nullptr;
    double2* tile_phase = nullptr;  // per-tile constant phases (passes with tphase_off >= 0)
    double phase_dt = std::nan("");  // dt the tile phases were computed for
    cudaGraphExec_t graph = nullptr; // one captured step (small, launch-bound states)
    double graph_dt = std::nan("");
    std::string program;
    bool relabel = false;  // unsharded: the last pass stores out of place into the plan's layout
};

struct sd_plan {
    sd_state* state = nullptr;
    std::vector<sdb::GroupSpec> groups;
    sd_plan_options opts{};
    std::vector<sdb::Op> ops;  // one Trotter step (gate level)
    int k = 12;
    std::map<std::vector<int>, std::unique_ptr<StepExec>> steps;
    StepExec* first = nullptr;  // plan of the canonical (identity) layout
    bool profiling = false;
    double ms[4] = {0, 0, 0, 0};
    uint64_t launches[4] = {0, 0, 0, 0};
    double bytes[4] = {0, 0, 0, 0};
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
    std::vector<int> ev_class;
    size_t ev_used = 0;
    int n_ref_sweeps = 0;
    std::vector<int> layout;  // unsharded: physical layout the steps run in (empty: identity)
    // Schedule family: -1 the cost model / SDB_SPLIT_DIAG decide, 0 whole-group
    // diagonal ops, 1 per-term diagonal ops (with knobs.max_hdepth). Set by the
    // plan-time autotuner (sd_plan_create), which times the candidates.
    int split = -1;
    sdb::PlannerKnobs knobs;
    // measured ms/step: whole-group, per-term (<= 2 Hadamard levels per pass),
    // whole-group ring, per-term <= 3 levels, per-term with no cap (0: not timed)
    double tune_ms[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    // Temporal blocking across Trotter steps (order 1): a plan of macro_reps
    // steps (the group list repeated) whose passes let the tail of one step
    // share passes with the head of the next; evolve() runs whole macro steps
    // through it and the remainder through this plan. Kept only when it
    // measures faster per Trotter step (sd_plan_create).
    sd_plan* macro = nullptr;
    int macro_reps = 0;
    double tune_ms_macro = 0.0;  // measured ms per Trotter step of the macro candidate (0: not timed)
    int macro_passes_tried = 0;  // passes per macro step of the candidate (0: none built)
};

namespace {

// Largest CNOT run (same control) kept as one op; same-control CNOTs commute,
// so a run can be cut anywhere. SDB_CX_SPLIT overrides (experiments).
int cx_split(int k) {
    if (const char* e = std::getenv("SDB_CX_SPLIT")) return std::max(1, std::atoi(e));
    (void)k;
    return 1;  // single CNOTs schedule best (config 5: 3471 -> 2003 passes/step)
}

// Capacity of a CNOT resynthesis round: the tile's free coordinates.
// SDB_CX_RESYNTH=0 keeps the synthesised CNOT order.
int resynth_cap(int k) {
    if (const char* e = std::getenv("SDB_CX_RESYNTH"); e && std::atoi(e) == 0) return 0;
    return k - sdb::fixed_bits_for(k);
}

// SDB_SPLIT_DIAG=1 / 0 forces per-term / whole-group diagonal ops; by default
// best_step_ops picks by its cost model.
int split_diag_mode() {
    if (const char* e = std::getenv("SDB_SPLIT_DIAG")) {
        const int v = std::atoi(e);
        return v < 0 ? -1 : (v != 0 ? 1 : 0);
    }
    return -1;
}

// Step ops with or without CNOT resynthesis, whichever schedules into fewer
// passes (an exchange counts as two passes of traffic) from the identity
// layout; resynthesis wins on CNOT-heavy groups (config 5) and can lose a
// pass or two where the given CNOT order commutes better (config 3).
std::vector<sdb::Op> best_step_ops(const std::vector<sdb::GroupSpec>& gs, int n, int order, int k, int n_local,
                                   int split_force = -1) {
    std::vector<int> ident(n);
    std::iota(ident.begin(), ident.end(), 0);
    const bool sharded = n_local < n;
    // Cost in units of a whole-diagonal pass. Per-term-diagonal passes carry
    // more transposes and phase stages (~1.8x a pass of the default plan at
    // n=30, profiles/r1_notes.md); an exchange moves half a shard or more over
    // NVLink (~2 passes). Sharded states take the plan with the fewest
    // exchanges first (the north star's "at most one exchange per group").
    struct Score {
        int exchanges;
        double cost;
    };
    auto score = [&](const std::vector<sdb::Op>& o, bool split) {
        const sdb::ShardedStep ss = sdb::plan_sharded_step(o, gs, n_local, k, sdb::fixed_bits_for(k), ident);
        return Score{ss.n_exchanges, ss.n_passes * (split ? 1.8 : 1.0) + 2.0 * ss.n_exchanges};
    };
    auto better = [&](const Score& a, const Score& b) {
        if (sharded && a.exchanges != b.exchanges) return a.exchanges < b.exchanges;
        return a.cost < b.cost;
    };
    const int cap = resynth_cap(k);
    const int split_env = split_force >= 0 ? split_force : split_diag_mode();
    // SDB_CZ_CX: -1 (default) try CZ -> CNOT conversion both ways, 0 off, 1 forced
    const int czcx_env = [] {
        const char* e = std::getenv("SDB_CZ_CX");
        return e ? std::atoi(e) : -1;
    }();
    std::vector<sdb::Op> best;
    Score best_score{0, 0.0};
    for (int split = 0; split < 2; ++split) {
        if ((split_env == 0 && split) || (split_env == 1 && !split)) continue;
        // one GPU: per-term diagonals never paid off (config 1: 0.081 -> 0.162 ms,
        // config 4: 92 -> 104 ms per step), so only sharded states consider them
        if (split_env < 0 && split && !sharded) continue;
        for (int rs = 0; rs < 2; ++rs) {
            if (rs && cap == 0) continue;
            for (int defer = 1; defer >= 0; --defer)
            for (int czcx = 1; czcx >= 0; --czcx) {
                if ((czcx_env == 0 && czcx) || (czcx_env == 1 && !czcx)) continue;
                auto o = sdb::step_ops(gs, n, order, cx_split(k), rs ? cap : 0, split != 0, czcx != 0);
                // Hadamards on the always-local qubits deferred out of second WHT
                // levels (fewer transposes in phase passes: config 4 97.4 -> 95.3 ms)
                for (sdb::Op& op : o) op.defer_deep = defer != 0;
                const Score sc = score(o, split != 0);
                if (best.empty() || better(sc, best_score)) {
                    best = std::move(o);
                    best_score = sc;
                }
            }
        }
    }
    return best;
}

// best_step_ops under the plan's knobs; when the look-ahead growth of the
// local set (planner.cpp) is not fixed by the plan or SDB_LOOKAHEAD, it is
// kept where it schedules the step into fewer passes from the identity layout
// (config 4 per-term: 9 -> 7; config 5 needs more passes with it). Call with
// a KnobScope on `knobs` alive.
std::vector<sdb::Op> choose_step_ops(const std::vector<sdb::GroupSpec>& gs, int n, int order, int k, int n_local,
                                     int split, sdb::PlannerKnobs& knobs) {
    if (knobs.lookahead >= 0 || std::getenv("SDB_LOOKAHEAD")) return best_step_ops(gs, n, order, k, n_local, split);
    std::vector<int> ident(n);
    std::iota(ident.begin(), ident.end(), 0);
    int best_la = 0, best_passes = 0;
    std::vector<sdb::Op> best_ops;
    for (int la = 0; la < 2; ++la) {
        // the look-ahead's what-if closures cost O(window^2) per growth: plans of
        // hundreds of passes per step (config 5: 1505, 6 s -> 27 s of planning)
        // keep list-order growth
        if (la == 1 && best_passes > 256) break;
        knobs.lookahead = la;
        auto o = best_step_ops(gs, n, order, k, n_local, split);
        const int np_ = sdb::plan_sharded_step(o, gs, n_local, k, sdb::fixed_bits_for(k), ident).n_passes;
        if (la == 0 || np_ < best_passes) {
            best_la = la;
            best_passes = np_;
            best_ops = std::move(o);
        }
    }
    knobs.lookahead = best_la;
    return best_ops;
}

using sdb::guard;
using sdb::require;

sdb::StateImpl& st(sd_state* s) {
    if (!s) throw std::invalid_argument("null state");
    return s->impl;
}

void check_qubit(const sdb::StateImpl& s, int q) {
    if (q < 0 || q >= s.n) throw std::out_of_range("qubit index out of range");
}

void require_unsharded(const sdb::StateImpl& s) {
    if (s.world != 1) throw std::invalid_argument("single-sweep kernels need an unsharded state");
}

void permute_local(sdb::StateImpl& s);
void permute_into_xbuf(sdb::StateImpl& s, const std::vector<int>& new_pos);

// Kernels that address qubits directly need the logical layout: an unsharded
// state evolved under a relabelled layout (plan layout search) is permuted
// back first; a relabelled sharded state must be canonicalised collectively.
void require_identity_layout(sdb::StateImpl& s) {
    bool ident = true;
    for (int q = 0; q < s.n; ++q) ident &= s.phys_of[q] == q;
    if (ident) return;
    if (s.world != 1) throw std::logic_error("state layout is relabelled");
    SDB_CUDA(cudaSetDevice(s.device));
    permute_local(s);
}

void bump(sdb::StateImpl& s, uint64_t reads, uint64_t writes) {
    s.stats.amp_reads += reads;
    s.stats.amp_writes += writes;
    s.stats.kernel_calls += 1;
}

void hadamard(sdb::StateImpl& s, int t) {
    check_qubit(s, t);
    sdb::launch_hadamard(s, t);
    bump(s, s.amps_count(), s.amps_count());
}

void batched_cnot(sdb::StateImpl& s, int c, uint64_t targets) {
    check_qubit(s, c);
    const uint64_t all = s.amps_count() - 1;
    if (targets == 0) throw std::invalid_argument("batched cnot needs at least one target");
    if ((targets & ~all) || (targets & (1ull << c))) {
        throw std::invalid_argument("batched cnot targets overlap control or exceed register");
    }
    sdb::launch_batched_cnot(s, c, targets);
    bump(s, s.amps_count() >> 1, s.amps_count() >> 1);
}

void phase_layer(sdb::StateImpl& s, uint64_t s_mask, const int32_t* pairs, size_t n_pairs, bool dagger) {
    if (s_mask & ~(s.amps_count() - 1)) throw std::invalid_argument("phase layer s_mask exceeds register");
    require(n_pairs == 0 || pairs != nullptr, "null cz pair array");
    std::vector<uint64_t> pm;
    for (size_t k = 0; k < n_pairs; ++k) {
        const int a = pairs[2 * k], b = pairs[2 * k + 1];
        check_qubit(s, a);
        check_qubit(s, b);
        if (a == b) throw std::invalid_argument("cz pair with equal qubits");
        pm.push_back((1ull << a) | (1ull << b));
    }
    sdb::launch_phase_layer(s, s_mask, pm, dagger);
    bump(s, s.amps_count(), s.amps_count());
}

void diag_exp(sdb::StateImpl& s, const uint64_t* masks, const double* coeffs, size_t m, double dt) {
    require(m == 0 || (masks && coeffs), "null diagonal arrays");
    if (!std::isfinite(dt)) throw std::invalid_argument("diagonal exp: non-finite time step");
    const uint64_t all = s.amps_count() - 1;
    for (size_t k = 0; k < m; ++k) {
        if (masks[k] & ~all) throw std::invalid_argument("diagonal exp: mask exceeds register");
    }
    sdb::launch_diag_exp(s, std::vector<uint64_t>(masks, masks + m), std::vector<double>(coeffs, coeffs + m), dt);
    bump(s, s.amps_count(), s.amps_count());
}

sdb::GroupSpec spec_of(const sd_group_desc& d) {
    sdb::GroupSpec g;
    g.h_pre.assign(d.h_pre, d.h_pre + d.n_h_pre);
    g.s_layer.assign(d.s_layer, d.s_layer + d.n_s);
    g.h_post.assign(d.h_post, d.h_post + d.n_h_post);
    for (size_t k = 0; k < d.n_cnots; ++k) g.cnots.emplace_back(d.cnots[2 * k], d.cnots[2 * k + 1]);
    for (size_t k = 0; k < d.n_czs; ++k) g.czs.emplace_back(d.czs[2 * k], d.czs[2 * k + 1]);
    if (d.n_terms) {
        require(d.z_masks && d.signed_coeffs, "group has no diagonal (not synthesised)");
        g.z_masks.assign(d.z_masks, d.z_masks + d.n_terms);
        g.coeffs.assign(d.signed_coeffs, d.signed_coeffs + d.n_terms);
    }
    return g;
}

// Reference apply_clifford / apply_clifford_inverse (statevector.cpp:339-381).
void clifford_unfused(sdb::StateImpl& s, const sdb::GroupSpec& g, bool inverse) {
    std::vector<std::pair<int, uint64_t>> runs;
    for (size_t k = 0; k < g.cnots.size();) {
        const int c = g.cnots[k].first;
        uint64_t t = 0;
        while (k < g.cnots.size() && g.cnots[k].first == c) t |= 1ull << g.cnots[k++].second;
        runs.emplace_back(c, t);
    }
    std::vector<int32_t> pairs;
    for (auto [a, b] : g.czs) pairs.insert(pairs.end(), {a, b});
    uint64_t smask = 0;
    for (int q : g.s_layer) smask |= 1ull << q;
    const bool ph = !g.czs.empty() || !g.s_layer.empty();
    if (!inverse) {
        for (int q : g.h_pre) hadamard(s, q);
        for (auto [c, t] : runs) batched_cnot(s, c, t);
        if (ph) phase_layer(s, smask, pairs.data(), g.czs.size(), false);
        for (int q : g.h_post) hadamard(s, q);
    } else {
        for (int q : g.h_post) hadamard(s, q);
        if (ph) phase_layer(s, smask, pairs.data(), g.czs.size(), true);
        for (auto it = runs.rbegin(); it != runs.rend(); ++it) batched_cnot(s, it->first, it->second);
        for (int q : g.h_pre) hadamard(s, q);
    }
}

// ---------------------------------------------------------------- plan build
// terms per POINT stage above which a per-tile table is used (SDB_TABLE_THRESHOLD: experiments)
const int kTableThreshold = [] {
    const char* e = std::getenv("SDB_TABLE_THRESHOLD");
    return e ? std::atoi(e) : 0;  // 0: the pass's largest phase stage always gets the table
}();

// Register coordinates of specialised kernels; the interpreter kernel always
// runs 4. SDB_RBITS=3..5 forces a value. By default the per-term schedule
// runs 5 (32 amplitudes per thread, 128 threads: its passes carry two
// Hadamard levels, and the fifth register coordinate saves a transpose or a
// lane swap per level -- config 4 72.2 -> 68.4 ms/step) and the whole-group
// schedule 4 (config 2 1.05 vs 1.19 ms, config 3 equal, config 5 at n=28
// 2257 vs 2309 ms with 5).
int jit_rbits(int split = -1) {
    static const int env = [] {
        const char* e = std::getenv("SDB_RBITS");
        return e ? std::clamp(std::atoi(e), 3, sdb::kMaxR) : 0;
    }();
    if (env) return env;
    return split == 1 ? 5 : 4;
}

void upload_step(sd_plan& p, StepExec& E, const sdb::StepPlan& combined) {
    sdb::StateImpl& s = p.state->impl;
    const bool jit = sdb::jit_wanted(s.n_local);
    const int rbits = jit ? jit_rbits(p.split >= 0 ? p.split : split_diag_mode()) : 4;
    sdb::HostPlanArrays A = sdb::lower_plan(combined, s.n_local, kTableThreshold, rbits);
    A.tma = p.knobs.tma;
    A.ring = p.knobs.ring;
    sdb::verify_lowering(A);  // register-config bookkeeping of lane swaps (host check, cheap)
    E.pass_class = A.pass_class;
    E.program = sdb::describe_program(A);
    E.jit_fn.assign(A.passes.size(), nullptr);
    E.smem.resize(A.passes.size());
    for (size_t i = 0; i < A.passes.size(); ++i) E.smem[i] = sdb::tile_pass_smem(A.passes[i]);
    if (jit) {
        E.jit_fn = sdb::jit_pass_kernels(A, s.device);
        E.threads.resize(A.passes.size());
        for (size_t i = 0; i < A.passes.size(); ++i) {
            E.smem[i] += sdb::jit_pass_smem_extra(A, i);
            E.threads[i] = sdb::jit_pass_threads(A, i);
        }
    }
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t sizes[] = {
        al(std::max<size_t>(1, A.passes.size()) * sizeof(sdb::PassDev)),
        al(std::max<size_t>(1, A.ops.size()) * sizeof(sdb::MicroOpDev)),
        al(std::max<size_t>(1, A.perms.size()) * sizeof(sdb::PermDev)),
        al(std::max<size_t>(1, A.points.size()) * sizeof(sdb::PointDev)),
        al(std::max<size_t>(1, A.segs.size()) * sizeof(sdb::SegDev)),
        al(std::max<size_t>(1, A.lo_pairs.size()) * sizeof(uint32_t)),
        al(std::max<size_t>(1, A.oo_pairs.size()) * 8),
        al(std::max<size_t>(1, A.qt_words.size()) * 8),
        al(std::max<size_t>(1, A.cfg_tb.size()) * sizeof(sdb::CfgThreadDev)),
        al(std::max<size_t>(1, A.term_hmask.size()) * 8),
        al(std::max<size_t>(1, A.term_lmask.size()) * 4),
        al(std::max<size_t>(1, A.term_coeffs.size()) * 8),
    };
    size_t total = 0;
    for (size_t v : sizes) total += v;
    SDB_CUDA(cudaSetDevice(s.device));
    SDB_CUDA(cudaMalloc(&E.dev_block, total));
    std::vector<unsigned char> host(total, 0);
    size_t off = 0;
    int slot = 0;
    auto put = [&](const void* src, size_t bytes) {
        if (bytes) std::memcpy(host.data() + off, src, bytes);
        void* dptr = static_cast<unsigned char*>(E.dev_block) + off;
        off += sizes[slot++];
        return dptr;
    };
    E.dev.passes = static_cast<const sdb::PassDev*>(put(A.passes.data(), A.passes.size() * sizeof(sdb::PassDev)));
    E.dev.ops = static_cast<const sdb::MicroOpDev*>(put(A.ops.data(), A.ops.size() * sizeof(sdb::MicroOpDev)));
    E.dev.perms = static_cast<const sdb::PermDev*>(put(A.perms.data(), A.perms.size() * sizeof(sdb::PermDev)));
    E.dev.points = static_cast<const sdb::PointDev*>(put(A.points.data(), A.points.size() * sizeof(sdb::PointDev)));
    E.dev.segs = static_cast<const sdb::SegDev*>(put(A.segs.data(), A.segs.size() * sizeof(sdb::SegDev)));
    E.dev.lo_pairs = static_cast<const uint32_t*>(put(A.lo_pairs.data(), A.lo_pairs.size() * sizeof(uint32_t)));
    E.dev.oo_pairs = static_cast<const uint64_t*>(put(A.oo_pairs.data(), A.oo_pairs.size() * 8));
    E.dev.qt_words = static_cast<const uint64_t*>(put(A.qt_words.data(), A.qt_words.size() * 8));
    E.dev.cfg_tb = static_cast<const sdb::CfgThreadDev*>(put(A.cfg_tb.data(), A.cfg_tb.size() * sizeof(sdb::CfgThreadDev)));
    E.dev.term_hmask = static_cast<const uint64_t*>(put(A.term_hmask.data(), A.term_hmask.size() * 8));
    E.dev.term_lmask = static_cast<const uint32_t*>(put(A.term_lmask.data(), A.term_lmask.size() * 4));
    E.dev.term_coeffs = static_cast<const double*>(put(A.term_coeffs.data(), A.term_coeffs.size() * 8));
    // per-tile constant phase buffers (offsets assigned here, filled per dt)
    size_t n_phase = 0;
    for (sdb::PassDev& pd : A.passes) {
        if (pd.tphase_off >= 0) {
            pd.tphase_off = static_cast<int>(n_phase);
            n_phase += size_t(1) << pd.n_outer;
        }
    }
    if (n_phase) {
        SDB_CUDA(cudaMalloc(reinterpret_cast<void**>(&E.tile_phase), n_phase * sizeof(double2)));
        std::memcpy(host.data(), A.passes.data(), A.passes.size() * sizeof(sdb::PassDev));  // updated offsets
    }
    E.dev.tile_phase = E.tile_phase;
    SDB_CUDA(cudaMemcpy(E.dev_block, host.data(), total, cudaMemcpyHostToDevice));
    E.host_passes = std::move(A.passes);
}

// The step plan starting in `layout`. `end` (unsharded only): the layout the
// step must leave the state in; a different one is reached by storing the
// step's last pass out of place through the relabelling (no extra pass).
StepExec& step_for(sd_plan& p, const std::vector<int>& layout, const std::vector<int>* end = nullptr) {
    sdb::StateImpl& s = p.state->impl;
    const sdb::KnobScope knobs(&p.knobs);
    const bool relabel = end && s.world == 1 && *end != layout;
    std::vector<int> key = layout;
    if (relabel) key.insert(key.end(), end->begin(), end->end());
    auto it = p.steps.find(key);
    if (it != p.steps.end()) return *it->second;
    auto E = std::make_unique<StepExec>();
    E->ss = sdb::plan_sharded_step(p.ops, p.groups, s.n_local, p.k, sdb::fixed_bits_for(p.k), layout);
    if (relabel && !E->ss.segs.empty() && !E->ss.segs.back().plan.passes.empty() &&
        E->ss.segs.back().plan.passes.back().store_sigma.empty()) {
        // physical bit layout[q] -> end[q] in the step's last store
        std::vector<int> sigma(s.n_local);
        for (int q = 0; q < s.n_local; ++q) sigma[layout[q]] = (*end)[q];
        E->ss.segs.back().plan.passes.back().store_sigma = sigma;
        E->ss.phys_out = *end;
        E->relabel = true;
    }
    sdb::StepPlan combined;
    combined.tile_qubits = p.k;
    for (const sdb::Segment& sg : E->ss.segs) {
        E->seg_first.push_back(static_cast<int>(combined.passes.size()));
        E->seg_count.push_back(static_cast<int>(sg.plan.passes.size()));
        for (const sdb::PassPlan& pp : sg.plan.passes) combined.passes.push_back(pp);
    }
    upload_step(p, *E, combined);
    if ((E->ss.n_exchanges > 0 || E->relabel) && !s.xbuf) {
        SDB_CUDA(cudaSetDevice(s.device));
        cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&s.xbuf), 16 * s.amps_count());
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw sdb::OomError("cannot allocate the exchange buffer");
        }
        s.xbuf_amps = s.amps_count();
    }
    StepExec& ref = *E;
    p.steps.emplace(key, std::move(E));
    return ref;
}

// HBM streaming cost of a pass by its local physical bits (tools/membench3,
// profiles/r1_membench3_n30.txt): bit 3 or 5 local ~1.0, else bits 4 or
// 6..10 ~1.25, else ~1.45 (relative to a pass with a good pattern).
double pattern_cost(const std::vector<int>& lpos) {
    bool good = false, medium = false;
    for (int b : lpos) {
        good |= b == 3 || b == 5;
        medium |= b == 4 || (b >= 6 && b <= 10);
    }
    return good ? 1.0 : medium ? 1.25 : 1.45;
}

double layout_cost(const sd_plan& p, const std::vector<int>& layout) {
    const sdb::StateImpl& s = p.state->impl;
    const sdb::ShardedStep ss = sdb::plan_sharded_step(p.ops, p.groups, s.n_local, p.k, sdb::fixed_bits_for(p.k), layout);
    double c = 0.0;
    static const double w2 = [] {
        const char* e = std::getenv("SDB_LAYOUT_W2");
        return e ? std::atof(e) : 1.0;
    }();
    for (const sdb::Segment& sg : ss.segs)
        for (const sdb::PassPlan& pp : sg.plan.passes) {
            int wht = 0;
            for (const sdb::PassStage& st : pp.stages) wht += st.kind == sdb::PassStage::WHT;
            // passes with two Hadamard stages take ~1.35x a single-stage pass
            const double base = wht >= 2 ? 1.35 : 1.0;
            c += base * (1.0 + (wht >= 2 ? w2 : 1.0) * (pattern_cost(pp.lpos) - 1.0));
        }
    return c;
}

// Unsharded states of >= 22 qubits may run their steps in a relabelled qubit
// layout: each evolve call enters it inside its first step and leaves it inside
// its last (the steps' final stores run out of place through the relabelling,
// no extra pass; needs the second buffer), so states stay in logical order
// between calls. Random search (a few transpositions from the best
// so far) with a trial budget set by the plan size, scored by pass count
// weighted with each pass's HBM pattern; kept only if it beats the identity by 2%.
void choose_layout(sd_plan& p) {
    sdb::StateImpl& s = p.state->impl;
    if (const char* e = std::getenv("SDB_LAYOUT_SEARCH"); e && std::atoi(e) == 0) return;
    if (s.world != 1 || s.n_local < 22 || !p.opts.fuse || p.opts.use_graph > 0) return;
    size_t free_b = 0, total_b = 0;
    SDB_CUDA(cudaSetDevice(s.device));
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    if (!s.xbuf && free_b < 16 * s.amps_count() + (size_t(4) << 30)) return;
    const int n = s.n;
    std::vector<int> ident(n);
    std::iota(ident.begin(), ident.end(), 0);
    const double base = layout_cost(p, ident);
    double best = base;
    std::vector<int> best_l;
    uint64_t rng = 0x243f6a8885a308d3ull;
    // deterministic budget by plan size (~1 s of planning for config 4's 13 passes)
    const int trials = std::clamp(5200 / std::max(1, static_cast<int>(base)), 0, 400);
    static const bool fix_line = [] {
        const char* e = std::getenv("SDB_LAYOUT_FIX_LINE");
        return !e || std::atoi(e) != 0;
    }();
    for (int trial = 0; trial < trials; ++trial) {
        std::vector<int> cand = best_l.empty() ? ident : best_l;
        // a few random transpositions away from the best layout so far
        const int moves = 1 + static_cast<int>(rng % 3);
        for (int m = 0; m < moves; ++m) {
            rng ^= rng << 13;
            rng ^= rng >> 7;
            rng ^= rng << 17;
            // the always-local line bits 0..fb-1 keep their qubits, so the
            // relabelling stores entering / leaving the layout move whole
            // 128-byte lines (SDB_LAYOUT_FIX_LINE=0: search them too)
            const int fb = fix_line ? sdb::fixed_bits_for(p.k) : 0;
            const int a = fb + static_cast<int>(rng % (n - fb)), b = fb + static_cast<int>((rng >> 20) % (n - fb));
            std::swap(cand[a], cand[b]);
        }
        const double c = layout_cost(p, cand);
        if (c < best) {
            best = c;
            best_l = cand;
        }
    }
    if (!best_l.empty() && best < 0.98 * base) p.layout = best_l;
}

void plan_build(sd_plan& p) {
    sdb::StateImpl& s = p.state->impl;
    const int order = p.opts.order;
    require(order == 1 || order == 2, "trotter order must be 1 or 2");
    p.n_ref_sweeps = static_cast<int>(std::lround(sdb::reference_sweeps(p.groups, order)));
    if (!p.opts.fuse) return;
    int k = p.opts.tile_qubits > 0 ? p.opts.tile_qubits : 12;
    p.k = std::min({k, sdb::max_tile_qubits(), s.n_local});
    const sdb::KnobScope knobs(&p.knobs);
    p.ops = choose_step_ops(p.groups, s.n, order, p.k, s.n_local, p.split, p.knobs);
    choose_layout(p);
    std::vector<int> ident(s.n);
    std::iota(ident.begin(), ident.end(), 0);
    p.first = &step_for(p, p.layout.empty() ? ident : p.layout);
}

// ---- plan-time autotuning of the schedule family (unsharded states)
//
// Whole-group diagonal ops (the default schedule) and per-term diagonal ops
// with at most two Hadamard levels per pass trade pass count against
// per-pass compute: config 4 runs 13 light passes or 10 heavier ones, and which
// is faster depends on how compute-bound the heavier passes are (config 4:
// 89.7 vs 82.4 ms; config 3: 469 vs 703 ms; config 2: 1.14 vs 2.0 ms). When
// the per-term schedule needs fewer passes, both plans are built and one
// steady-state step of each is timed on the exchange buffer as scratch (the
// state is untouched); the faster plan is kept. SDB_AUTOTUNE=0 disables it,
// and an explicit SDB_SPLIT_DIAG / SDB_MAX_HDEPTH experiment bypasses it.
bool autotune_wanted(const sd_plan& p) {
    const sdb::StateImpl& s = p.state->impl;
    if (const char* e = std::getenv("SDB_AUTOTUNE"); e && std::atoi(e) == 0) return false;
    if (std::getenv("SDB_SPLIT_DIAG") || std::getenv("SDB_MAX_HDEPTH")) return false;
    return s.world == 1 && s.n_local >= 22 && p.opts.fuse && p.opts.use_graph <= 0 && p.opts.order >= 1;
}

// SDB_MACRO: Trotter steps per macro step tried at plan time (default 2;
// 0 or 1: none)
int macro_reps_wanted() {
    const char* e = std::getenv("SDB_MACRO");
    return e ? std::atoi(e) : 2;
}

// SDB_AUTOTUNE_DEEP=0 drops candidate D (per-term, <= 3 Hadamard levels per pass)
bool deep_candidate_wanted() {
    const char* e = std::getenv("SDB_AUTOTUNE_DEEP");
    return !e || std::atoi(e) != 0;
}

bool ensure_scratch(sdb::StateImpl& s) {
    if (s.xbuf) return true;
    size_t free_b = 0, total_b = 0;
    SDB_CUDA(cudaSetDevice(s.device));
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (free_b < 16 * s.amps_count() + (size_t(4) << 30)) return false;
    if (cudaMalloc(reinterpret_cast<void**>(&s.xbuf), 16 * s.amps_count()) != cudaSuccess) {
        cudaGetLastError();
        s.xbuf = nullptr;
        return false;
    }
    s.xbuf_amps = s.amps_count();
    return true;
}

void run_step_fused(sd_plan& p, double dt, const std::vector<int>* end);

// ms per steady-state step of plan P, run on the exchange buffer (zeroed
// scratch); the state's buffer, layout and counters are restored
double time_steady_step(sd_plan& P) {
    sdb::StateImpl& s = P.state->impl;
    std::vector<int> L(s.n);
    std::iota(L.begin(), L.end(), 0);
    if (!P.layout.empty()) L = P.layout;
    const std::vector<int> saved_layout = s.phys_of;
    const sd_kernel_stats saved_stats = s.stats;
    const double dt = 0.01;
    SDB_CUDA(cudaSetDevice(s.device));
    SDB_CUDA(cudaMemsetAsync(s.xbuf, 0, 16 * s.amps_count(), s.stream));
    std::swap(s.amps, s.xbuf);
    cudaEvent_t a = nullptr, b = nullptr;
    double ms = 0.0;
    try {
        s.phys_of = L;
        run_step_fused(P, dt, &L);  // warm-up: builds and uploads the steady-state step
        SDB_CUDA(cudaEventCreate(&a));
        SDB_CUDA(cudaEventCreate(&b));
        SDB_CUDA(cudaEventRecord(a, s.stream));
        constexpr int kSteps = 2;
        for (int i = 0; i < kSteps; ++i) run_step_fused(P, dt, &L);
        SDB_CUDA(cudaEventRecord(b, s.stream));
        SDB_CUDA(cudaEventSynchronize(b));
        float f = 0.0f;
        SDB_CUDA(cudaEventElapsedTime(&f, a, b));
        ms = f / kSteps;
    } catch (...) {
        std::swap(s.amps, s.xbuf);
        s.phys_of = saved_layout;
        s.stats = saved_stats;
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
        throw;
    }
    std::swap(s.amps, s.xbuf);
    s.phys_of = saved_layout;
    s.stats = saved_stats;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

void record_start(sd_plan& p, int cls) {
    if (!p.profiling) return;
    if (p.ev_used == p.ev_pool.size()) {
        cudaEvent_t a, b;
        SDB_CUDA(cudaEventCreate(&a));
        SDB_CUDA(cudaEventCreate(&b));
        p.ev_pool.emplace_back(a, b);
        p.ev_class.push_back(0);
    }
    p.ev_class[p.ev_used] = cls;
    SDB_CUDA(cudaEventRecord(p.ev_pool[p.ev_used].first, p.state->impl.stream));
}

void record_end(sd_plan& p, double bytes) {
    if (!p.profiling) return;
    SDB_CUDA(cudaEventRecord(p.ev_pool[p.ev_used].second, p.state->impl.stream));
    p.bytes[p.ev_class[p.ev_used]] += bytes;
    p.launches[p.ev_class[p.ev_used]] += 1;
    ++p.ev_used;
}

void harvest(sd_plan& p) {
    if (!p.profiling || p.ev_used == 0) return;
    SDB_CUDA(cudaStreamSynchronize(p.state->impl.stream));
    for (size_t i = 0; i < p.ev_used; ++i) {
        float ms = 0.f;
        SDB_CUDA(cudaEventElapsedTime(&ms, p.ev_pool[i].first, p.ev_pool[i].second));
        p.ms[p.ev_class[i]] += ms;
    }
    p.ev_used = 0;
}

// Destination table of a fused exchange store: chunk c of this rank's
// (sigma-stored) shard goes to the current receive buffer of the rank whose
// swapped global bits are c (exchange_routes), itself included.
void set_exchange_destinations(sdb::StateImpl& s, const sdb::ExchangeSpec& ex) {
    if (!s.xdst_dev) SDB_CUDA(cudaMalloc(reinterpret_cast<void**>(&s.xdst_dev), 256 * sizeof(double2*)));
    std::vector<double2*> tab(256, nullptr);
    for (const sdb::Route& rt : sdb::exchange_routes(s.n_local, s.n, s.rank, ex)) {
        const auto& pb = s.peer_buf.at(static_cast<size_t>(rt.peer));
        double* recv = s.parity == 0 ? pb.second : pb.first;
        tab[rt.send_off / rt.count] = reinterpret_cast<double2*>(recv);
    }
    SDB_CUDA(cudaMemcpyAsync(s.xdst_dev, tab.data(), tab.size() * sizeof(double2*), cudaMemcpyHostToDevice, s.stream));
}

// after every rank's fused exchange pass has completed
void finish_p2p_exchange(sdb::StateImpl& s) {
    std::swap(s.amps, s.xbuf);
    s.parity ^= 1;
}

// per-tile constant phases of the step's diagonal passes, once per dt
void ensure_tile_phase(sd_plan& p, StepExec& E, double dt) {
    if (!E.tile_phase || E.phase_dt == dt) return;
    sdb::StateImpl& s = p.state->impl;
    const uint64_t rank_bits = uint64_t(s.rank) << s.n_local;
    for (size_t i = 0; i < E.host_passes.size(); ++i) {
        if (E.host_passes[i].tphase_off >= 0) {
            sdb::launch_tile_phase(s, E.host_passes[i], static_cast<int>(i), E.dev, dt, rank_bits,
                                   E.tile_phase + E.host_passes[i].tphase_off);
        }
    }
    E.phase_dt = dt;
}

void run_segment(sd_plan& p, StepExec& E, size_t seg, double dt) {
    sdb::StateImpl& s = p.state->impl;
    const uint64_t rank_bits = uint64_t(s.rank) << s.n_local;
    ensure_tile_phase(p, E, dt);
    const double bytes = 2.0 * 16.0 * double(s.amps_count());
    const bool exch = E.ss.segs[seg].exchange_after;
    const int first = E.seg_first[seg], count = E.seg_count[seg];
    static const int debug_passes = [] {
        const char* e = std::getenv("SDB_DEBUG_PASSES");  // debugging: run only the first N passes
        return e ? std::atoi(e) : -1;
    }();
    for (int i = first; i < first + count; ++i) {
        if (debug_passes >= 0 && i >= debug_passes) break;
        const bool to_buf = (exch || (E.relabel && seg + 1 == E.ss.segs.size())) && i == first + count - 1;
        // fused exchange: the pass stores straight into the peers' receive buffers
        double2* const* xdst = nullptr;
        if (to_buf && s.p2p) {
            set_exchange_destinations(s, E.ss.segs[seg].ex);
            xdst = s.xdst_dev;
        }
        record_start(p, xdst ? 2 : E.pass_class[i]);
        if (E.jit_fn[i]) {
            sdb::launch_tile_pass_jit(E.jit_fn[i], s, E.host_passes[i], i, E.dev, dt, rank_bits,
                                      to_buf ? s.xbuf : nullptr, E.smem[i], xdst, E.threads[i]);
        } else {
            sdb::launch_tile_pass(s, E.host_passes[i], i, E.dev, dt, rank_bits, to_buf ? s.xbuf : nullptr, xdst);
        }
        record_end(p, bytes);
        bump(s, s.amps_count(), s.amps_count());
        if (p.profiling && p.ev_used >= 4096) harvest(p);
    }
}

void run_step_fused(sd_plan& p, double dt, const std::vector<int>* end = nullptr) {
    sdb::StateImpl& s = p.state->impl;
    StepExec& E = step_for(p, s.phys_of, end);
    for (size_t seg = 0; seg < E.ss.segs.size(); ++seg) {
        run_segment(p, E, seg, dt);
        if (E.ss.segs[seg].exchange_after) {
            if (s.p2p) {
                sdb::nccl_barrier(s);  // every rank's fused store has landed
                finish_p2p_exchange(s);
                continue;
            }
            const double xb = 2.0 * 16.0 * double(s.amps_count()) *
                              (1.0 - std::ldexp(1.0, -static_cast<int>(E.ss.segs[seg].ex.swaps.size())));
            record_start(p, 2);
            sdb::exchange_nccl(s, E.ss.segs[seg].ex);
            record_end(p, xb);
        }
    }
    if (E.relabel) {
        std::swap(s.amps, s.xbuf);
        s.parity ^= 1;
    }
    s.phys_of = E.ss.phys_out;
}

void run_step_unfused(sd_plan& p, double dt) {
    sdb::StateImpl& s = p.state->impl;
    auto apply = [&](const sdb::GroupSpec& g, double f) {
        clifford_unfused(s, g, false);
        diag_exp(s, g.z_masks.data(), g.coeffs.data(), g.z_masks.size(), dt * f);
        clifford_unfused(s, g, true);
    };
    const int G = static_cast<int>(p.groups.size());
    if (p.opts.order == 1 || G <= 1) {
        for (const auto& g : p.groups) apply(g, 1.0);
    } else {
        for (int g = 0; g < G - 1; ++g) apply(p.groups[g], 0.5);
        apply(p.groups[G - 1], 1.0);
        for (int g = G - 2; g >= 0; --g) apply(p.groups[g], 0.5);
    }
}

// Small states are launch-bound (config 1: a 1 MiB state streams in well under
// a microsecond): one step's launches are captured into a CUDA graph per
// (layout, dt) and replayed. Used on one unsharded device when the shard has
// <= 20 qubits (use_graph = 1 forces it, -1 disables it), not while profiling.
bool graph_mode(const sd_plan& p) {
    const sdb::StateImpl& s = p.state->impl;
    if (!p.opts.fuse || s.world != 1 || p.profiling || p.opts.use_graph < 0) return false;
    return p.opts.use_graph > 0 || s.n_local <= 20;
}

void run_step_graph(sd_plan& p, double dt) {
    sdb::StateImpl& s = p.state->impl;
    StepExec& E = step_for(p, s.phys_of);
    if (!E.graph || !(E.graph_dt == dt)) {
        if (E.graph) SDB_CUDA(cudaGraphExecDestroy(E.graph));
        E.graph = nullptr;
        ensure_tile_phase(p, E, dt);  // outside the graph: once per dt
        cudaGraph_t g = nullptr;
        SDB_CUDA(cudaStreamBeginCapture(s.stream, cudaStreamCaptureModeThreadLocal));
        for (size_t seg = 0; seg < E.ss.segs.size(); ++seg) run_segment(p, E, seg, dt);
        SDB_CUDA(cudaStreamEndCapture(s.stream, &g));
        SDB_CUDA(cudaGraphInstantiate(&E.graph, g, 0));
        SDB_CUDA(cudaGraphDestroy(g));
        E.graph_dt = dt;
    } else {
        for (size_t i = 0; i < E.host_passes.size(); ++i) bump(s, s.amps_count(), s.amps_count());
    }
    SDB_CUDA(cudaGraphLaunch(E.graph, s.stream));
    s.phys_of = E.ss.phys_out;
}

void evolve(sd_plan& p, double dt, int n_steps, bool wait) {
    require(std::isfinite(dt), "plan needs finite total_time");
    if (n_steps < 0) throw std::invalid_argument("plan needs n_steps >= 0");
    sdb::StateImpl& s = p.state->impl;
    SDB_CUDA(cudaSetDevice(s.device));
    const bool graphs = graph_mode(p);
    // A relabelled plan layout is entered inside the call's first step and left
    // inside its last one: the state is in logical order between calls.
    const bool relayout = !p.layout.empty() && s.world == 1 && p.opts.fuse && !graphs;
    if (p.macro && n_steps >= p.macro_reps) {
        // each call leaves the state in logical order, so the two plans compose
        const int m = n_steps / p.macro_reps;
        evolve(*p.macro, dt, m, false);
        n_steps -= m * p.macro_reps;
    }
    std::vector<int> ident(s.n);
    std::iota(ident.begin(), ident.end(), 0);
    for (int step = 0; step < n_steps; ++step) {
        if (!p.opts.fuse) run_step_unfused(p, dt);
        else if (graphs) run_step_graph(p, dt);
        else run_step_fused(p, dt, relayout ? (step + 1 == n_steps ? &ident : &p.layout) : nullptr);
    }
    if (wait) SDB_CUDA(cudaStreamSynchronize(s.stream));
    harvest(p);
}

// Exchanges that bring a relabelled sharded layout back to the identity
// (logical qubit q at physical bit q): (1) fix the set of global qubits,
// (2) if the global qubits sit in the wrong order, swap them all out and back
// in order. The remaining local permutation is done by permute_local().
std::vector<sdb::ExchangeSpec> canonical_exchanges(std::vector<int>& L, int n_local) {
    const int n = static_cast<int>(L.size());
    const int g = n - n_local;
    std::vector<sdb::ExchangeSpec> out;
    auto apply = [&](const std::vector<int>& to_top, const std::vector<int>& incoming) {
        // to_top: local qubits that leave (placed on T by sigma); incoming: global qubits, paired in order
        const int gp = static_cast<int>(incoming.size());
        const int t0 = n_local - gp;
        sdb::ExchangeSpec ex;
        ex.sigma.resize(n_local);
        std::iota(ex.sigma.begin(), ex.sigma.end(), 0);
        std::vector<int> at(n_local, -1);
        for (int q = 0; q < n; ++q) {
            if (L[q] < n_local) at[L[q]] = q;
        }
        // target slot of each leaving qubit: t0 + i; move it there by a transposition
        for (int i = 0; i < gp; ++i) {
            const int e = to_top[i];
            const int pe = L[e], pt = t0 + i;
            if (pe == pt) continue;
            const int other = at[pt];
            // compose the transposition (pe pt) into sigma (sigma maps original bit -> new bit)
            for (int b = 0; b < n_local; ++b) {
                if (ex.sigma[b] == pe) ex.sigma[b] = pt;
                else if (ex.sigma[b] == pt) ex.sigma[b] = pe;
            }
            L[e] = pt;
            if (other >= 0) L[other] = pe;
            at[pt] = e;
            at[pe] = other;
        }
        for (int i = 0; i < gp; ++i) {
            const int qi = incoming[i], qe = to_top[i];
            ex.swaps.emplace_back(L[qi], t0 + i);
            L[qe] = L[qi];
            L[qi] = t0 + i;
        }
        out.push_back(std::move(ex));
    };
    std::vector<int> W, V;
    for (int q = 0; q < n; ++q) {
        if (q >= n_local && L[q] < n_local) W.push_back(q);
        if (q < n_local && L[q] >= n_local) V.push_back(q);
    }
    if (!W.empty()) {
        std::sort(V.begin(), V.end(), [&](int a, int b) { return L[a] < L[b]; });
        apply(W, V);
    }
    bool ordered = true;
    for (int q = n_local; q < n; ++q) ordered &= L[q] == q;
    if (!ordered && g > 0) {
        // swap every global bit out (its current holder comes local)...
        std::vector<int> out_q, in_q;
        std::vector<int> at(n, -1);
        for (int q = 0; q < n; ++q) at[L[q]] = q;
        for (int i = 0; i < g; ++i) {
            in_q.push_back(at[n_local + i]);
            out_q.push_back(at[n_local - g + i]);
        }
        apply(out_q, in_q);
        // ...and bring logical n_local+i back to global bit n_local+i
        std::fill(at.begin(), at.end(), -1);
        for (int q = 0; q < n; ++q) at[L[q]] = q;
        out_q.clear();
        in_q.clear();
        for (int i = 0; i < g; ++i) {
            out_q.push_back(n_local + i);
            in_q.push_back(at[n_local + i]);
        }
        apply(out_q, in_q);
    }
    return out;
}

// state <- the state with its local physical bits permuted (new_pos[b]), via xbuf
void permute_into_xbuf(sdb::StateImpl& s, const std::vector<int>& new_pos) {
    if (!s.xbuf) {
        SDB_CUDA(cudaMalloc(reinterpret_cast<void**>(&s.xbuf), 16 * s.amps_count()));
        s.xbuf_amps = s.amps_count();
    }
    sdb::launch_permute_bits(s, s.amps, s.xbuf, new_pos.data(), s.n_local);
}

void permute_local(sdb::StateImpl& s) {
    std::vector<int> new_pos(s.n_local);
    bool ident = true;
    for (int q = 0; q < s.n_local; ++q) {
        if (s.phys_of[q] >= s.n_local) throw std::logic_error("permute_local: global qubits not canonical");
        new_pos[s.phys_of[q]] = q;
        ident &= s.phys_of[q] == q;
    }
    if (ident) return;
    permute_into_xbuf(s, new_pos);
    std::swap(s.amps, s.xbuf);
    s.parity ^= 1;
    for (int q = 0; q < s.n_local; ++q) s.phys_of[q] = q;
}

void canonicalize_nccl(sdb::StateImpl& s) {
    std::vector<int> L = s.phys_of;
    const auto exs = canonical_exchanges(L, s.n_local);
    for (const sdb::ExchangeSpec& ex : exs) {
        permute_into_xbuf(s, ex.sigma);
        sdb::exchange_nccl(s, ex);
    }
    s.phys_of = L;
    permute_local(s);
    SDB_CUDA(cudaStreamSynchronize(s.stream));
}

bool is_identity(const std::vector<int>& L) {
    for (size_t q = 0; q < L.size(); ++q) {
        if (L[q] != static_cast<int>(q)) return false;
    }
    return true;
}

}  // namespace

extern "C" {

sd_status sd_state_create_shard(int n, int rank, int world, int device, sd_state** out) {
    return guard([&] {
        require(out != nullptr, "out is null");
        if (n < 0 || n > 40) throw std::invalid_argument("state vector qubit count out of range");
        require(world >= 1 && (world & (world - 1)) == 0, "world size must be a power of two");
        require(rank >= 0 && rank < world, "rank out of range");
        const int g = std::countr_zero(static_cast<unsigned>(world));
        require(n - g >= 1, "too many ranks for this state");
        auto h = std::make_unique<sd_state>();
        sdb::StateImpl& s = h->impl;
        s.n = n;
        s.n_local = n - g;
        s.rank = rank;
        s.world = world;
        s.device = device;
        s.phys_of.resize(n);
        std::iota(s.phys_of.begin(), s.phys_of.end(), 0);
        SDB_CUDA(cudaSetDevice(device));
        SDB_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
        const size_t bytes = sizeof(double) * 2 * s.amps_count();
        cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&s.amps), bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            cudaStreamDestroy(s.stream);
            throw sdb::OomError("cannot allocate " + std::to_string(bytes) + " bytes of state");
        }
        sdb::launch_set_basis(s, rank == 0 ? 0 : ~0ull);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
        *out = h.release();
    });
}


sd_status sd_state_create(int n, int device, sd_state** out) { return sd_state_create_shard(n, 0, 1, device, out); }

void sd_state_destroy(sd_state* h) {
    if (!h) return;
    sdb::StateImpl& s = h->impl;
    cudaSetDevice(s.device);
    if (s.stream) cudaStreamSynchronize(s.stream);
    try {
        sdb::nccl_detach(s);
    } catch (...) {
    }
    for (void* ptr : s.ipc_opened) cudaIpcCloseMemHandle(ptr);
    if (s.xdst_dev) cudaFree(s.xdst_dev);
    if (s.amps) cudaFree(s.amps);
    if (s.xbuf) cudaFree(s.xbuf);
    if (s.reduce_buf) cudaFree(s.reduce_buf);
    if (s.stream) cudaStreamDestroy(s.stream);
    delete h;
}

sd_status sd_state_info(const sd_state* h, int* n, int* nl, int* rank, int* world) {
    return guard([&] {
        require(h != nullptr, "null state");
        if (n) *n = h->impl.n;
        if (nl) *nl = h->impl.n_local;
        if (rank) *rank = h->impl.rank;
        if (world) *world = h->impl.world;
    });
}

sd_status sd_state_stream(const sd_state* h, void** stream) {
    return guard([&] {
        require(h != nullptr && stream != nullptr, "null argument");
        *stream = h->impl.stream;
    });
}

sd_status sd_state_device_ptr(const sd_state* h, void** ptr) {
    return guard([&] {
        require(h != nullptr && ptr != nullptr, "null argument");
        *ptr = h->impl.amps;
    });
}

sd_status sd_sync(sd_state* h) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        SDB_CUDA(cudaSetDevice(s.device));
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_state_set_basis(sd_state* h, uint64_t index) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        if (s.n < 64 && (index >> s.n) != 0) throw std::out_of_range("basis index out of range");
        SDB_CUDA(cudaSetDevice(s.device));
        std::iota(s.phys_of.begin(), s.phys_of.end(), 0);
        const uint64_t owner = index >> s.n_local;
        sdb::launch_set_basis(s, owner == uint64_t(s.rank) ? (index & (s.amps_count() - 1)) : ~0ull);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_state_set_plus(sd_state* h) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        SDB_CUDA(cudaSetDevice(s.device));
        std::iota(s.phys_of.begin(), s.phys_of.end(), 0);
        // plus_state: 1/sqrt(dim) everywhere (statevector.cpp:74-79)
        const double a = 1.0 / std::sqrt(std::ldexp(1.0, s.n));
        sdb::launch_fill(s, a, 0.0);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_state_set_random(sd_state* h, uint64_t seed) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(s.world == 1, "sharded random_state needs a cross-rank norm; use set_random_unnormalized + norm");
        SDB_CUDA(cudaSetDevice(s.device));
        std::iota(s.phys_of.begin(), s.phys_of.end(), 0);
        sdb::launch_random(s, seed);
        const double nsq = sdb::device_norm_sq(s);
        sdb::launch_scale(s, 1.0 / std::sqrt(nsq));
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_state_upload(sd_state* h, const double* re_im, uint64_t n_amps) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(re_im != nullptr, "null host buffer");
        require(n_amps == s.amps_count(), "upload size does not match the shard");
        SDB_CUDA(cudaSetDevice(s.device));
        std::iota(s.phys_of.begin(), s.phys_of.end(), 0);
        SDB_CUDA(cudaMemcpyAsync(s.amps, re_im, n_amps * 16, cudaMemcpyHostToDevice, s.stream));
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_state_download(sd_state* h, double* re_im, uint64_t n_amps) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(re_im != nullptr, "null host buffer");
        require(n_amps == s.amps_count(), "download size does not match the shard");
        if (!is_identity(s.phys_of)) {
            SDB_CUDA(cudaSetDevice(s.device));
            if (s.world == 1) permute_local(s);
            else if (s.nccl) canonicalize_nccl(s);  // collective: every rank downloads
            else throw std::runtime_error("sharded state is relabelled: call sd_local_canonicalize first");
        }
        SDB_CUDA(cudaSetDevice(s.device));
        SDB_CUDA(cudaMemcpyAsync(re_im, s.amps, n_amps * 16, cudaMemcpyDeviceToHost, s.stream));
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_state_download_range(sd_state* h, uint64_t first, uint64_t count, double* re_im) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(re_im != nullptr || count == 0, "null host buffer");
        if (first > s.amps_count() || count > s.amps_count() - first)
            throw std::out_of_range("download range outside the shard");
        if (!is_identity(s.phys_of)) {
            SDB_CUDA(cudaSetDevice(s.device));
            if (s.world == 1) permute_local(s);
            else if (s.nccl) canonicalize_nccl(s);
            else throw std::runtime_error("sharded state is relabelled: call sd_local_canonicalize first");
        }
        if (count == 0) return;
        SDB_CUDA(cudaSetDevice(s.device));
        SDB_CUDA(cudaMemcpyAsync(re_im, s.amps + 2 * first, count * 16, cudaMemcpyDeviceToHost, s.stream));
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_state_norm_sq(sd_state* h, double* out) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(out != nullptr, "null output");
        SDB_CUDA(cudaSetDevice(s.device));
        *out = sdb::device_norm_sq(s);
    });
}

sd_status sd_state_inner(sd_state* a, sd_state* b, double* re, double* im) {
    return guard([&] {
        sdb::StateImpl& x = st(a);
        sdb::StateImpl& y = st(b);
        require(re != nullptr, "null output");
        if (x.n != y.n || x.n_local != y.n_local) throw std::invalid_argument("fidelity: dimension mismatch");
        require_identity_layout(x);
        require_identity_layout(y);
        SDB_CUDA(cudaSetDevice(x.device));
        SDB_CUDA(cudaStreamSynchronize(y.stream));
        sdb::device_inner(x, y, re, im);
    });
}

sd_status sd_state_copy(sd_state* dst, const sd_state* src) {
    return guard([&] {
        sdb::StateImpl& d = st(dst);
        require(src != nullptr, "null state");
        const sdb::StateImpl& s = src->impl;
        require(d.n == s.n && d.n_local == s.n_local, "state shapes differ");
        SDB_CUDA(cudaSetDevice(d.device));
        SDB_CUDA(cudaStreamSynchronize(s.stream));
        SDB_CUDA(cudaMemcpyAsync(d.amps, s.amps, d.amps_count() * 16, cudaMemcpyDeviceToDevice, d.stream));
        SDB_CUDA(cudaStreamSynchronize(d.stream));
        d.phys_of = s.phys_of;
    });
}

sd_status sd_kernel_stats_get(const sd_state* h, sd_kernel_stats* out) {
    return guard([&] {
        require(h != nullptr && out != nullptr, "null argument");
        *out = h->impl.stats;
    });
}

sd_status sd_kernel_stats_reset(sd_state* h) {
    return guard([&] { st(h).stats = sd_kernel_stats{0, 0, 0}; });
}

sd_status sd_apply_hadamard(sd_state* h, int t) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require_unsharded(s);
        require_identity_layout(s);
        SDB_CUDA(cudaSetDevice(s.device));
        hadamard(s, t);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_apply_batched_cnot(sd_state* h, int c, uint64_t targets) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require_unsharded(s);
        require_identity_layout(s);
        SDB_CUDA(cudaSetDevice(s.device));
        batched_cnot(s, c, targets);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_apply_phase_layer(sd_state* h, uint64_t s_mask, const int32_t* pairs, size_t n_pairs, int dagger) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require_unsharded(s);
        require_identity_layout(s);
        SDB_CUDA(cudaSetDevice(s.device));
        phase_layer(s, s_mask, pairs, n_pairs, dagger != 0);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_apply_diagonal_exp(sd_state* h, const uint64_t* masks, const double* coeffs, size_t m, double dt) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require_unsharded(s);
        require_identity_layout(s);
        SDB_CUDA(cudaSetDevice(s.device));
        diag_exp(s, masks, coeffs, m, dt);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_apply_clifford(sd_state* h, const sd_group_desc* g) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(g != nullptr, "null group");
        require_unsharded(s);
        require_identity_layout(s);
        SDB_CUDA(cudaSetDevice(s.device));
        clifford_unfused(s, spec_of(*g), false);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_apply_clifford_inverse(sd_state* h, const sd_group_desc* g) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(g != nullptr, "null group");
        require_unsharded(s);
        require_identity_layout(s);
        SDB_CUDA(cudaSetDevice(s.device));
        clifford_unfused(s, spec_of(*g), true);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_plan_options_default(sd_plan_options* o) {
    return guard([&] {
        require(o != nullptr, "null options");
        std::memset(o, 0, sizeof(*o));
        o->order = 1;
        o->tile_qubits = 0;
        o->fuse = 1;
        o->use_graph = 0;
        o->relabel = 1;
    });
}

sd_status sd_plan_create(sd_state* h, const sd_group_desc* groups, size_t n_groups, const sd_plan_options* opts,
                         sd_plan** out) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(out != nullptr, "out is null");
        require(n_groups == 0 || groups != nullptr, "null group array");
        auto p = std::make_unique<sd_plan>();
        p->state = h;
        if (opts) p->opts = *opts;
        else sd_plan_options_default(&p->opts);
        for (size_t i = 0; i < n_groups; ++i) {
            sdb::GroupSpec g = spec_of(groups[i]);
            auto chk = [&](int q) { check_qubit(s, q); };
            for (int q : g.h_pre) chk(q);
            for (int q : g.h_post) chk(q);
            for (int q : g.s_layer) chk(q);
            for (auto [a, b] : g.cnots) { chk(a); chk(b); }
            for (auto [a, b] : g.czs) { chk(a); chk(b); }
            for (uint64_t m : g.z_masks) {
                if (s.n < 64 && (m >> s.n)) throw std::invalid_argument("diagonal exp: mask exceeds register");
            }
            p->groups.push_back(std::move(g));
        }
        if (!p->opts.fuse) require_unsharded(s);
        if (autotune_wanted(*p)) {
            // candidate B: per-term diagonal ops, <= 2 Hadamard levels per pass
            auto q = std::make_unique<sd_plan>();
            q->state = h;
            q->opts = p->opts;
            q->groups = p->groups;
            q->split = 1;
            q->knobs.max_hdepth = 2;
            p->split = 0;
            plan_build(*p);
            const bool had_scratch = s.xbuf != nullptr;
            // candidate C: whole-group ops through the ring pipeline (two warp
            // groups, three TMA stages, TMA stores) -- faster for config 3
            // (448 -> 415 ms), slower for configs 2 and 4
            auto r = std::make_unique<sd_plan>();
            r->state = h;
            r->opts = p->opts;
            r->groups = p->groups;
            r->split = 0;
            r->knobs.ring = 1;
            // candidate D: per-term diagonal ops with <= 3 Hadamard levels per pass
            // (config 4: same 7 passes as B, 46.3 vs 47.7 ms; with no cap the
            // step needs 4 passes, but their second and third POINT stages
            // evaluate terms per amplitude: 160 ms), timed when B is and D needs
            // no more passes than B
            auto d = std::make_unique<sd_plan>();
            d->state = h;
            d->opts = p->opts;
            d->groups = p->groups;
            d->split = 1;
            d->knobs.max_hdepth = 3;
            // candidate E: per-term diagonal ops, no cap on Hadamard levels (config 4:
            // 4 heavy passes, 45.9 ms; their extra POINT stages cut into pattern
            // points by the lowering), timed when it needs fewer passes than D
            auto e = std::make_unique<sd_plan>();
            e->state = h;
            e->opts = p->opts;
            e->groups = p->groups;
            e->split = 1;
            e->knobs.max_hdepth = 0;
            try {
                plan_build(*q);
                const bool fewer = q->first && p->first && q->first->ss.n_passes < p->first->ss.n_passes;
                if (ensure_scratch(s)) {
                    double t[5] = {time_steady_step(*p), 0.0, 0.0, 0.0, 0.0};
                    if (fewer) t[1] = time_steady_step(*q);
                    plan_build(*r);
                    t[2] = time_steady_step(*r);
                    if (fewer && deep_candidate_wanted()) {
                        plan_build(*d);
                        if (d->first && d->first->ss.n_passes <= q->first->ss.n_passes) t[3] = time_steady_step(*d);
                        plan_build(*e);
                        if (e->first && d->first && e->first->ss.n_passes < d->first->ss.n_passes) t[4] = time_steady_step(*e);
                    }
                    // E's few heavy passes are issue-bound (11.4 ms each at n=30, 0.46 of
                    // the copy peak) and slow down with the SM clock under sw_power_cap,
                    // where D's near-HBM-bound passes do not: E is kept only when it wins
                    // by 3% (measured: 45.0 vs 45.3 ms, a tie)
                    int best = 0;
                    for (int c = 1; c < 5; ++c)
                        if (t[c] > 0.0 && t[c] < (c == 4 ? 0.97 : 1.0) * t[best]) best = c;
                    for (int c = 0; c < 5; ++c)
                        p->tune_ms[c] = q->tune_ms[c] = r->tune_ms[c] = d->tune_ms[c] = e->tune_ms[c] = t[c];
                    if (best == 1) std::swap(p, q);
                    if (best == 2) std::swap(p, r);
                    if (best == 3) std::swap(p, d);
                    if (best == 4) std::swap(p, e);
                }
            } catch (const sdb::OomError&) {
                // no room for another candidate: keep the whole-group plan
            }
            sd_plan_destroy(q.release());
            sd_plan_destroy(r.release());
            sd_plan_destroy(d.release());
            sd_plan_destroy(e.release());
            // Macro step (order 1 only: repeating an S2 group list is not two S2
            // steps): the kept schedule family planned over macro_reps steps at
            // once, kept when it needs fewer passes per Trotter step and times
            // faster per step (config 4: 7 -> 6 passes per step at 2 steps)
            const int reps = macro_reps_wanted();
            if (p->opts.order == 1 && reps >= 2 && p->first) {
                sd_plan* m = new sd_plan;
                m->state = h;
                m->opts = p->opts;
                for (int rr = 0; rr < reps; ++rr) m->groups.insert(m->groups.end(), p->groups.begin(), p->groups.end());
                m->split = p->split;
                m->knobs = p->knobs;
                m->knobs.lookahead = -1;
                bool keep = false;
                try {
                    plan_build(*m);
                    if (m->first) p->macro_passes_tried = m->first->ss.n_passes;
                    if (m->first && m->first->ss.n_passes < reps * p->first->ss.n_passes && ensure_scratch(s)) {
                        const double tm = time_steady_step(*m) / reps;
                        const double tp = time_steady_step(*p);
                        m->tune_ms[0] = tm;
                        p->tune_ms_macro = tm;
                        keep = (tm > 0.0 && tm < 0.98 * tp) || std::getenv("SDB_MACRO_FORCE");
                    }
                } catch (const sdb::OomError&) {
                    keep = false;
                }
                if (keep) {
                    p->macro = m;
                    p->macro_reps = reps;
                } else {
                    sd_plan_destroy(m);
                }
            }
            // the scratch stays only if a kept plan's layout needs the second buffer
            if (!had_scratch && s.xbuf && p->layout.empty() && (!p->macro || p->macro->layout.empty())) {
                SDB_CUDA(cudaSetDevice(s.device));
                SDB_CUDA(cudaFree(s.xbuf));
                s.xbuf = nullptr;
                s.xbuf_amps = 0;
            }
        } else {
            plan_build(*p);
        }
        *out = p.release();
    });
}

void sd_plan_destroy(sd_plan* p) {
    if (!p) return;
    sd_plan_destroy(p->macro);
    cudaSetDevice(p->state->impl.device);
    for (auto& e : p->ev_pool) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    for (auto& kv : p->steps) {
        if (kv.second->graph) cudaGraphExecDestroy(kv.second->graph);
        if (kv.second->dev_block) cudaFree(kv.second->dev_block);
        if (kv.second->tile_phase) cudaFree(kv.second->tile_phase);
    }
    delete p;
}

sd_status sd_plan_get_info(const sd_plan* p, sd_plan_info* o) {
    return guard([&] {
        require(p != nullptr && o != nullptr, "null argument");
        const sdb::StateImpl& s = p->state->impl;
        std::memset(o, 0, sizeof(*o));
        o->n_ref_sweeps_per_step = p->n_ref_sweeps;
        o->n_group_applications = static_cast<int>(p->opts.order == 2 && p->groups.size() > 1
                                                        ? 2 * p->groups.size() - 1
                                                        : p->groups.size());
        if (p->opts.fuse) {
            // steady state: the plan of the current layout (identity until the first exchange)
            auto it = p->steps.find(s.phys_of);
            const StepExec* E = it != p->steps.end() && p->layout.empty() ? it->second.get() : p->first;
            o->n_passes_per_step = E->ss.n_passes;
            o->n_exchanges_per_step = E->ss.n_exchanges;
            o->tile_qubits = p->k;
            o->n_kernels_per_step = o->n_passes_per_step;
            o->bytes_per_step = 2.0 * 16.0 * double(s.amps_count()) * o->n_passes_per_step;
            o->schedule = p->split == 1 ? 1 : 0;
            o->tune_ms_whole = p->tune_ms[0];
            o->tune_ms_split = p->tune_ms[1];
            o->tune_ms_whole_ring = p->tune_ms[2];
            o->tune_ms_split_deep = p->tune_ms[3];
            o->tune_ms_split_nocap = p->tune_ms[4];
            o->tune_ms_macro = p->tune_ms_macro;
            o->macro_passes = p->macro_passes_tried;
            if (p->macro && p->macro->first) {
                o->macro_steps = p->macro_reps;
                o->macro_passes = p->macro->first->ss.n_passes;
                // steady state runs whole macro steps: bytes per Trotter step
                o->bytes_per_step = 2.0 * 16.0 * double(s.amps_count()) * o->macro_passes / p->macro_reps;
            }
            o->ring = p->knobs.ring;
            o->max_hdepth = p->knobs.max_hdepth;
        } else {
            o->n_passes_per_step = p->n_ref_sweeps;
            o->n_kernels_per_step = 0;
            o->bytes_per_step = 2.0 * 16.0 * double(s.amps_count()) * p->n_ref_sweeps;
        }
    });
}

sd_status sd_plan_describe(const sd_plan* p, char* buf, size_t cap, size_t* len) {
    return guard([&] {
        require(p != nullptr, "null plan");
        std::string txt = "unfused reference schedule\n";
        if (p->opts.fuse) {
            txt.clear();
            const StepExec& E = *p->first;
            for (size_t i = 0; i < E.ss.segs.size(); ++i) {
                txt += "segment " + std::to_string(i) + ": " + sdb::describe(E.ss.segs[i].plan);
                if (E.ss.segs[i].exchange_after) {
                    txt += "  exchange swaps";
                    for (auto [gb, lb] : E.ss.segs[i].ex.swaps) txt += " (" + std::to_string(gb) + "," + std::to_string(lb) + ")";
                    txt += "\n";
                }
            }
            txt += E.program;
        }
        sdb::write_text_out(txt, buf, cap, len);
    });
}

sd_status sd_plan_preview(int n, int world, const sd_group_desc* groups, size_t n_groups, const sd_plan_options* opts,
                          sd_plan_info* info, char* json, size_t cap, size_t* len) {
    return guard([&] {
        require(n_groups == 0 || groups != nullptr, "null group array");
        require(world >= 1 && (world & (world - 1)) == 0, "world size must be a power of two");
        sd_plan_options o{};
        if (opts) o = *opts;
        else sd_plan_options_default(&o);
        require(o.order == 1 || o.order == 2, "trotter order must be 1 or 2");
        const int n_local = n - std::countr_zero(static_cast<unsigned>(world));
        require(n_local >= 1, "too many ranks for this state");
        std::vector<sdb::GroupSpec> gs;
        for (size_t i = 0; i < n_groups; ++i) gs.push_back(spec_of(groups[i]));
        std::vector<int> phys(n);
        std::iota(phys.begin(), phys.end(), 0);
        int k = o.tile_qubits > 0 ? o.tile_qubits : 12;
        k = std::min({k, sdb::max_tile_qubits(), n_local});
        sdb::PlannerKnobs knobs;
        const sdb::KnobScope scope(&knobs);
        const auto ops = choose_step_ops(gs, n, o.order, k, n_local, -1, knobs);
        // steps until the layout repeats (the executor caches one plan per layout)
        std::vector<sdb::ShardedStep> steps;
        std::vector<std::vector<int>> seen;
        int cycle_start = 0;
        for (int it = 0; it < 16; ++it) {
            auto f = std::find(seen.begin(), seen.end(), phys);
            if (f != seen.end()) {
                cycle_start = static_cast<int>(f - seen.begin());
                break;
            }
            seen.push_back(phys);
            steps.push_back(sdb::plan_sharded_step(ops, gs, n_local, k, sdb::fixed_bits_for(k), phys));
            phys = steps.back().phys_out;
        }
        if (info) {
            const sdb::ShardedStep& st = steps[static_cast<size_t>(cycle_start)];
            std::memset(info, 0, sizeof(*info));
            info->n_passes_per_step = st.n_passes;
            info->n_ref_sweeps_per_step = static_cast<int>(std::lround(sdb::reference_sweeps(gs, o.order)));
            info->n_group_applications =
                static_cast<int>(o.order == 2 && gs.size() > 1 ? 2 * gs.size() - 1 : gs.size());
            info->tile_qubits = k;
            info->n_kernels_per_step = st.n_passes;
            info->n_exchanges_per_step = st.n_exchanges;
            info->bytes_per_step = 2.0 * 16.0 * std::ldexp(1.0, n_local) * st.n_passes;
        }
        std::string js = "{\"n_local\":" + std::to_string(n_local) + ",\"cycle_start\":" +
                         std::to_string(cycle_start) + ",\"steps\":[";
        for (size_t i = 0; i < steps.size(); ++i) js += (i ? "," : "") + sdb::describe_sharded_json(steps[i]);
        js += "]}";
        sdb::write_text_out(js, json, cap, len);
    });
}

sd_status sd_evolve(sd_plan* p, double dt, int n_steps) {
    return guard([&] {
        require(p != nullptr, "null plan");
        evolve(*p, dt, n_steps, true);
    });
}

sd_status sd_evolve_async(sd_plan* p, double dt, int n_steps) {
    return guard([&] {
        require(p != nullptr, "null plan");
        evolve(*p, dt, n_steps, false);
    });
}

sd_status sd_plan_set_profiling(sd_plan* p, int enable) {
    return guard([&] {
        require(p != nullptr, "null plan");
        for (sd_plan* q = p; q; q = q->macro) {
            harvest(*q);
            q->profiling = enable != 0;
            for (int c = 0; c < 4; ++c) {
                q->ms[c] = 0.0;
                q->launches[c] = 0;
                q->bytes[c] = 0.0;
            }
        }
    });
}

sd_status sd_plan_kernel_times(sd_plan* p, double* ms, uint64_t* launches, double* bytes, int n_classes) {
    return guard([&] {
        require(p != nullptr, "null plan");
        for (int c = 0; c < n_classes && c < 4; ++c) {
            if (ms) ms[c] = 0.0;
            if (launches) launches[c] = 0;
            if (bytes) bytes[c] = 0.0;
        }
        for (sd_plan* q = p; q; q = q->macro) {
            harvest(*q);
            for (int c = 0; c < n_classes && c < 4; ++c) {
                if (ms) ms[c] += q->ms[c];
                if (launches) launches[c] += q->launches[c];
                if (bytes) bytes[c] += q->bytes[c];
            }
        }
    });
}

sd_status sd_comm_unique_id(unsigned char id[128]) {
    return guard([&] {
        require(id != nullptr, "null id buffer");
        sdb::nccl_unique_id(id);
    });
}

sd_status sd_state_attach_comm(sd_state* h, const unsigned char id[128]) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(id != nullptr, "null id");
        sdb::nccl_attach(s, id);
    });
}

sd_status sd_state_canonicalize(sd_state* h) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        SDB_CUDA(cudaSetDevice(s.device));
        if (is_identity(s.phys_of)) return;
        if (s.world == 1) permute_local(s);
        else canonicalize_nccl(s);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_state_create_local_shards(int n, int world, const int* devices, sd_state** out) {
    return guard([&] {
        require(out != nullptr, "out is null");
        require(world >= 1 && (world & (world - 1)) == 0, "world size must be a power of two");
        for (int r = 0; r < world; ++r) out[r] = nullptr;
        for (int r = 0; r < world; ++r) {
            const sd_status st = sd_state_create_shard(n, r, world, devices ? devices[r] : 0, &out[r]);
            if (st != SD_OK) {
                for (int q = 0; q < r; ++q) sd_state_destroy(out[q]);
                throw std::runtime_error(sd_last_error());
            }
        }
    });
}

sd_status sd_evolve_local(sd_plan* const* plans, int world, double dt, int n_steps) {
    return guard([&] {
        require(plans != nullptr && world >= 1, "null plan array");
        require(std::isfinite(dt), "plan needs finite total_time");
        if (n_steps < 0) throw std::invalid_argument("plan needs n_steps >= 0");
        std::vector<sdb::StateImpl*> shards(world);
        for (int r = 0; r < world; ++r) {
            require(plans[r] != nullptr && plans[r]->opts.fuse, "local evolution needs fused plans");
            shards[r] = &plans[r]->state->impl;
            require(shards[r]->rank == r && shards[r]->world == world, "plans[r] must drive shard r of `world`");
        }
        for (int step = 0; step < n_steps; ++step) {
            std::vector<StepExec*> E(world);
            for (int r = 0; r < world; ++r) {
                require(shards[r]->phys_of == shards[0]->phys_of, "shards disagree on the layout");
                SDB_CUDA(cudaSetDevice(shards[r]->device));
                E[r] = &step_for(*plans[r], shards[r]->phys_of);
            }
            for (size_t seg = 0; seg < E[0]->ss.segs.size(); ++seg) {
                for (int r = 0; r < world; ++r) {
                    SDB_CUDA(cudaSetDevice(shards[r]->device));
                    run_segment(*plans[r], *E[r], seg, dt);
                }
                if (E[0]->ss.segs[seg].exchange_after) {
                    if (shards[0]->p2p) {
                        for (sdb::StateImpl* sh : shards) {
                            SDB_CUDA(cudaSetDevice(sh->device));
                            SDB_CUDA(cudaStreamSynchronize(sh->stream));
                        }
                        for (sdb::StateImpl* sh : shards) finish_p2p_exchange(*sh);
                    } else {
                        sdb::exchange_local(shards, E[0]->ss.segs[seg].ex);
                    }
                }
            }
            for (int r = 0; r < world; ++r) shards[r]->phys_of = E[r]->ss.phys_out;
        }
        for (int r = 0; r < world; ++r) {
            SDB_CUDA(cudaSetDevice(shards[r]->device));
            SDB_CUDA(cudaStreamSynchronize(shards[r]->stream));
            harvest(*plans[r]);
        }
    });
}

sd_status sd_local_canonicalize(sd_state* const* hs, int world) {
    return guard([&] {
        require(hs != nullptr && world >= 1, "null shard array");
        std::vector<sdb::StateImpl*> shards(world);
        for (int r = 0; r < world; ++r) shards[r] = &st(hs[r]);
        std::vector<int> L = shards[0]->phys_of;
        if (is_identity(L)) return;
        const auto exs = canonical_exchanges(L, shards[0]->n_local);
        for (const sdb::ExchangeSpec& ex : exs) {
            for (sdb::StateImpl* s : shards) {
                SDB_CUDA(cudaSetDevice(s->device));
                permute_into_xbuf(*s, ex.sigma);
            }
            sdb::exchange_local(shards, ex);
        }
        for (sdb::StateImpl* s : shards) {
            SDB_CUDA(cudaSetDevice(s->device));
            s->phys_of = L;
            permute_local(*s);
            SDB_CUDA(cudaStreamSynchronize(s->stream));
        }
    });
}

sd_status sd_exchange_routes(int n, int n_local, int rank, const int32_t* swaps, size_t n_swaps, sd_route* out,
                             size_t cap, size_t* n_out) {
    return guard([&] {
        require(n_swaps == 0 || swaps != nullptr, "null swap array");
        require(rank >= 0 && n_local >= 1 && n_local <= n && rank < (1 << (n - n_local)), "rank out of range");
        sdb::ExchangeSpec ex;
        for (size_t i = 0; i < n_swaps; ++i) ex.swaps.emplace_back(swaps[2 * i], swaps[2 * i + 1]);
        const auto routes = sdb::exchange_routes(n_local, n, rank, ex);
        if (n_out) *n_out = routes.size();
        for (size_t i = 0; i < routes.size() && i < cap && out; ++i) {
            out[i] = sd_route{routes[i].peer, routes[i].send_off, routes[i].recv_off, routes[i].count};
        }
    });
}

sd_status sd_jit_compile_preview(int n, int world, const sd_group_desc* groups, size_t n_groups,
                                 const sd_plan_options* opts, size_t* n_programs) {
    return guard([&] {
        require(n_groups == 0 || groups != nullptr, "null group array");
        require(world >= 1 && (world & (world - 1)) == 0, "world size must be a power of two");
        sd_plan_options o{};
        if (opts) o = *opts;
        else sd_plan_options_default(&o);
        const int n_local = n - std::countr_zero(static_cast<unsigned>(world));
        std::vector<sdb::GroupSpec> gs;
        for (size_t i = 0; i < n_groups; ++i) gs.push_back(spec_of(groups[i]));
        std::vector<int> phys(n);
        std::iota(phys.begin(), phys.end(), 0);
        int k = o.tile_qubits > 0 ? o.tile_qubits : 12;
        k = std::min({k, sdb::max_tile_qubits(), n_local});
        sdb::PlannerKnobs knobs;
        const sdb::KnobScope scope(&knobs);
        const auto ops = choose_step_ops(gs, n, o.order, k, n_local, -1, knobs);
        const sdb::ShardedStep ss = sdb::plan_sharded_step(ops, gs, n_local, k, sdb::fixed_bits_for(k), phys);
        sdb::StepPlan combined;
        combined.tile_qubits = k;
        for (const sdb::Segment& sg : ss.segs)
            for (const sdb::PassPlan& pp : sg.plan.passes) combined.passes.push_back(pp);
        const sdb::HostPlanArrays A = sdb::lower_plan(combined, n_local, kTableThreshold, jit_rbits(split_diag_mode()));
        const size_t np = sdb::jit_compile_only(A);
        if (n_programs) *n_programs = np;
    });
}

namespace {
void ensure_xbuf(sdb::StateImpl& s) {
    if (s.xbuf) return;
    SDB_CUDA(cudaSetDevice(s.device));
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&s.xbuf), 16 * s.amps_count());
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw sdb::OomError("cannot allocate the exchange buffer");
    }
    s.xbuf_amps = s.amps_count();
}
}  // namespace

sd_status sd_local_enable_p2p(sd_state* const* hs, int world) {
    return guard([&] {
        require(hs != nullptr && world >= 1, "null shard array");
        std::vector<sdb::StateImpl*> shards(world);
        for (int r = 0; r < world; ++r) {
            shards[r] = &st(hs[r]);
            require(shards[r]->rank == r && shards[r]->world == world, "shards[r] must be rank r of `world`");
            ensure_xbuf(*shards[r]);
        }
        for (sdb::StateImpl* a : shards) {
            SDB_CUDA(cudaSetDevice(a->device));
            for (sdb::StateImpl* b : shards) {
                if (b->device == a->device) continue;
                int ok = 0;
                SDB_CUDA(cudaDeviceCanAccessPeer(&ok, a->device, b->device));
                if (!ok) throw std::runtime_error("devices cannot access each other's memory");
                const cudaError_t e = cudaDeviceEnablePeerAccess(b->device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) SDB_CUDA(e);
                cudaGetLastError();
            }
        }
        for (sdb::StateImpl* a : shards) {
            a->peer_buf.clear();
            for (sdb::StateImpl* b : shards) a->peer_buf.emplace_back(b->amps, b->xbuf);
            a->parity = 0;
            a->p2p = true;
        }
    });
}

sd_status sd_state_ipc_handles(sd_state* h, unsigned char out[128]) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(out != nullptr, "null output");
        ensure_xbuf(s);
        SDB_CUDA(cudaSetDevice(s.device));
        cudaIpcMemHandle_t a, b;
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
        SDB_CUDA(cudaIpcGetMemHandle(&a, s.amps));
        SDB_CUDA(cudaIpcGetMemHandle(&b, s.xbuf));
        std::memcpy(out, &a, 64);
        std::memcpy(out + 64, &b, 64);
    });
}

sd_status sd_state_attach_peers(sd_state* h, const unsigned char* handles) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(handles != nullptr, "null handles");
        require(s.nccl != nullptr, "attach the NCCL communicator first (sd_state_attach_comm)");
        ensure_xbuf(s);
        SDB_CUDA(cudaSetDevice(s.device));
        s.peer_buf.assign(static_cast<size_t>(s.world), {nullptr, nullptr});
        for (int r = 0; r < s.world; ++r) {
            if (r == s.rank) {
                s.peer_buf[r] = {s.amps, s.xbuf};
                continue;
            }
            void* p[2] = {nullptr, nullptr};
            for (int k = 0; k < 2; ++k) {
                cudaIpcMemHandle_t hd;
                std::memcpy(&hd, handles + 128 * r + 64 * k, 64);
                SDB_CUDA(cudaIpcOpenMemHandle(&p[k], hd, cudaIpcMemLazyEnablePeerAccess));
                s.ipc_opened.push_back(p[k]);
            }
            s.peer_buf[r] = {static_cast<double*>(p[0]), static_cast<double*>(p[1])};
        }
        s.parity = 0;
        s.p2p = true;
        sdb::nccl_barrier(s);
    });
}

// save_raw / load_raw (statevector.cpp:383-401): raw little-endian (re, im)
// doubles, index = basis. A shard writes its own index range
// [rank 2^n_local, (rank+1) 2^n_local) after restoring the canonical layout
// (collective for NCCL-attached shards), so the rank files concatenate to the
// reference's file. Streamed through a pinned staging buffer.
namespace {
constexpr size_t kRawChunkAmps = size_t(1) << 22;  // 64 MiB per transfer
}

sd_status sd_state_save_raw(sd_state* h, const char* path) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(path != nullptr, "null path");
        SDB_CUDA(cudaSetDevice(s.device));
        if (!is_identity(s.phys_of)) {
            if (s.world == 1) permute_local(s);
            else if (s.nccl) canonicalize_nccl(s);
            else throw std::runtime_error("sharded state is relabelled: call sd_local_canonicalize first");
        }
        std::FILE* f = std::fopen(path, "wb");
        if (!f) throw std::runtime_error(std::string("save_raw: cannot open ") + path);
        double* stage = nullptr;
        const size_t chunk = std::min<size_t>(kRawChunkAmps, s.amps_count());
        SDB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&stage), 16 * chunk));
        try {
            for (uint64_t off = 0; off < s.amps_count(); off += chunk) {
                const size_t m = std::min<uint64_t>(chunk, s.amps_count() - off);
                SDB_CUDA(cudaMemcpyAsync(stage, s.amps + 2 * off, 16 * m, cudaMemcpyDeviceToHost, s.stream));
                SDB_CUDA(cudaStreamSynchronize(s.stream));
                if (std::fwrite(stage, 16, m, f) != m) throw std::runtime_error("save_raw: write failed");
            }
        } catch (...) {
            cudaFreeHost(stage);
            std::fclose(f);
            throw;
        }
        cudaFreeHost(stage);
        if (std::fclose(f) != 0) throw std::runtime_error("save_raw: close failed");
    });
}

sd_status sd_state_load_raw(sd_state* h, const char* path) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(path != nullptr, "null path");
        std::FILE* f = std::fopen(path, "rb");
        if (!f) throw std::runtime_error(std::string("load_raw: cannot open ") + path);
        std::fseek(f, 0, SEEK_END);
        const long bytes = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        if (bytes < 0 || static_cast<uint64_t>(bytes) != 16 * s.amps_count()) {
            std::fclose(f);
            throw std::invalid_argument("load_raw: file size does not match the state (shard)");
        }
        SDB_CUDA(cudaSetDevice(s.device));
        std::iota(s.phys_of.begin(), s.phys_of.end(), 0);
        double* stage = nullptr;
        const size_t chunk = std::min<size_t>(kRawChunkAmps, s.amps_count());
        SDB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&stage), 16 * chunk));
        try {
            for (uint64_t off = 0; off < s.amps_count(); off += chunk) {
                const size_t m = std::min<uint64_t>(chunk, s.amps_count() - off);
                if (std::fread(stage, 16, m, f) != m) throw std::runtime_error("load_raw: read failed");
                SDB_CUDA(cudaMemcpyAsync(s.amps + 2 * off, stage, 16 * m, cudaMemcpyHostToDevice, s.stream));
                SDB_CUDA(cudaStreamSynchronize(s.stream));
            }
        } catch (...) {
            cudaFreeHost(stage);
            std::fclose(f);
            throw;
        }
        cudaFreeHost(stage);
        std::fclose(f);
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Observables and the per-term baseline on (sharded) states: expectation
// (evolve.cpp:99-135), norm / fidelity (statevector.cpp:403-418),
// apply_pauli_rotation (statevector.cpp:288-337), evolve_baseline
// (evolve.cpp:21-45), and the generic gates apply_single_qubit /
// apply_two_qubit (statevector.cpp:101-154).
//
// Masks are mapped through the state's logical -> physical layout, so a
// relabelled state needs no canonicalisation. A term whose X part touches a
// global (rank) bit pairs amplitudes across shards: every shard first takes a
// copy of its partner shard (rank ^ x_hi) into its exchange buffer -- NCCL
// send/recv for one process per GPU, device copies for in-process shards --
// and terms are visited grouped by x_hi so each partner is copied once.
// Partial sums are per shard in a fixed block order, combined over shards in
// rank order (all-gather, not a reduction), so results are deterministic.
namespace {

uint64_t phys_mask(const sdb::StateImpl& s, uint64_t logical) {
    uint64_t out = 0;
    for (uint64_t m = logical; m; m &= m - 1) out |= 1ull << s.phys_of[std::countr_zero(m)];
    return out;
}

// The shards one call drives: all of them (in-process), or this rank's one
// (NCCL: the call is collective over the communicator).
struct ShardSet {
    std::vector<sdb::StateImpl*> sh;
    bool nccl = false;
    int n = 0, n_local = 0;
};

ShardSet one_shard(sd_state* h) {
    ShardSet S;
    sdb::StateImpl& s = st(h);
    S.sh = {&s};
    S.n = s.n;
    S.n_local = s.n_local;
    if (s.world > 1) {
        if (!s.nccl)
            throw std::invalid_argument("sharded state without a communicator: attach one (sd_state_attach_comm) "
                                        "or use the sd_local_* entry points for in-process shards");
        S.nccl = true;
    }
    return S;
}

ShardSet local_set(sd_state* const* hs, int world) {
    require(hs != nullptr && world >= 1, "null shard array");
    ShardSet S;
    for (int r = 0; r < world; ++r) {
        sdb::StateImpl& s = st(hs[r]);
        require(s.rank == r && s.world == world, "shards[r] must be rank r of `world`");
        require(r == 0 || s.phys_of == S.sh[0]->phys_of, "shards disagree on the layout");
        S.sh.push_back(&s);
    }
    S.n = S.sh[0]->n;
    S.n_local = S.sh[0]->n_local;
    return S;
}

void sync_all(const ShardSet& S) {
    for (sdb::StateImpl* s : S.sh) {
        SDB_CUDA(cudaSetDevice(s->device));
        SDB_CUDA(cudaStreamSynchronize(s->stream));
    }
}

// every shard's exchange buffer <- a copy of shard rank ^ x_hi
void fetch_partners(ShardSet& S, uint64_t x_hi) {
    for (sdb::StateImpl* s : S.sh) ensure_xbuf(*s);
    if (S.nccl) {
        sdb::StateImpl& s = *S.sh[0];
        SDB_CUDA(cudaSetDevice(s.device));
        sdb::nccl_copy_partner(s, s.rank ^ static_cast<int>(x_hi));
        SDB_CUDA(cudaStreamSynchronize(s.stream));
        return;
    }
    sync_all(S);
    for (sdb::StateImpl* s : S.sh) {
        const sdb::StateImpl& p = *S.sh[s->rank ^ static_cast<int>(x_hi)];
        SDB_CUDA(cudaSetDevice(s->device));
        SDB_CUDA(cudaMemcpyPeerAsync(s->xbuf, s->device, p.amps, p.device, 16 * s->amps_count(), s->stream));
    }
    sync_all(S);
}

// per-rank values (rank order) of `local` vectors computed per shard
std::vector<double> gather_ranks(ShardSet& S, const std::vector<std::vector<double>>& local) {
    if (S.nccl) return sdb::nccl_gather(*S.sh[0], local[0]);
    std::vector<double> out;
    for (const auto& v : local) out.insert(out.end(), v.begin(), v.end());
    return out;
}

int world_of(const ShardSet& S) { return S.sh[0]->world; }

void check_term_masks(const ShardSet& S, const uint64_t* x, const uint64_t* z, size_t m, const char* what) {
    const uint64_t all = S.n >= 64 ? ~0ull : ((1ull << S.n) - 1);
    for (size_t k = 0; k < m; ++k) {
        if ((x[k] | z[k]) & ~all) throw std::invalid_argument(what);
    }
}

void expectation_set(ShardSet& S, const uint64_t* x, const uint64_t* z, const double* coeffs, size_t m, double* re,
                     double* imag_residue) {
    require(re != nullptr, "null output");
    require(m == 0 || (x && z && coeffs), "null term arrays");
    check_term_masks(S, x, z, m, "hamiltonian/state qubit counts differ");
    const sdb::StateImpl& s0 = *S.sh[0];
    std::vector<uint64_t> xp(m), zp(m);
    for (size_t k = 0; k < m; ++k) {
        xp[k] = phys_mask(s0, x[k]);
        zp[k] = phys_mask(s0, z[k]);
    }
    // visit terms grouped by the global part of X (one partner copy per group)
    std::vector<size_t> order(m);
    std::iota(order.begin(), order.end(), size_t(0));
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t a, size_t b) { return (xp[a] >> S.n_local) < (xp[b] >> S.n_local); });
    std::vector<std::vector<double>> part(S.sh.size(), std::vector<double>(2 * m, 0.0));
    uint64_t have = ~0ull;
    for (size_t k : order) {
        const uint64_t x_hi = xp[k] >> S.n_local;
        if (x_hi != 0 && x_hi != have) {
            fetch_partners(S, x_hi);
            have = x_hi;
        }
        for (size_t i = 0; i < S.sh.size(); ++i) {
            sdb::StateImpl& s = *S.sh[i];
            SDB_CUDA(cudaSetDevice(s.device));
            sdb::device_expectation_term(s, xp[k], zp[k], s.xbuf, &part[i][2 * k], &part[i][2 * k + 1]);
        }
    }
    const std::vector<double> all = gather_ranks(S, part);
    const int W = world_of(S);
    double tr = 0.0, ti = 0.0;
    for (size_t k = 0; k < m; ++k) {
        double sr = 0.0, si = 0.0;
        for (int r = 0; r < W; ++r) {
            sr += all[2 * m * r + 2 * k];
            si += all[2 * m * r + 2 * k + 1];
        }
        tr += coeffs[k] * sr;
        ti += coeffs[k] * si;
    }
    *re = tr;
    if (imag_residue) *imag_residue = std::abs(ti);
}

void rotation_set(ShardSet& S, uint64_t x, uint64_t z, double coeff, double dt) {
    const sdb::StateImpl& s0 = *S.sh[0];
    const uint64_t xp = phys_mask(s0, x), zp = phys_mask(s0, z);
    const uint64_t x_hi = xp >> S.n_local;
    if (x_hi) fetch_partners(S, x_hi);
    for (sdb::StateImpl* s : S.sh) {
        SDB_CUDA(cudaSetDevice(s->device));
        sdb::launch_pauli_rotation(*s, xp, zp, coeff, dt, x_hi ? s->xbuf : nullptr);
        bump(*s, s->amps_count(), s->amps_count());
    }
    if (x_hi) sync_all(S);  // the partner copies are reused by the next term
}

double norm_set(ShardSet& S) {
    std::vector<std::vector<double>> part(S.sh.size(), std::vector<double>(1, 0.0));
    for (size_t i = 0; i < S.sh.size(); ++i) {
        SDB_CUDA(cudaSetDevice(S.sh[i]->device));
        part[i][0] = sdb::device_norm_sq(*S.sh[i]);
    }
    const std::vector<double> all = gather_ranks(S, part);
    double v = 0.0;
    for (double p : all) v += p;
    return std::sqrt(v);
}

void canonical_set(ShardSet& S, sd_state* const* hs) {
    if (is_identity(S.sh[0]->phys_of)) return;
    if (S.nccl || world_of(S) == 1) {
        SDB_CUDA(cudaSetDevice(S.sh[0]->device));
        if (world_of(S) == 1) permute_local(*S.sh[0]);
        else canonicalize_nccl(*S.sh[0]);
        SDB_CUDA(cudaStreamSynchronize(S.sh[0]->stream));
        return;
    }
    if (sd_local_canonicalize(hs, world_of(S)) != SD_OK) throw std::runtime_error(sd_last_error());
}

double fidelity_set(ShardSet& A, ShardSet& B, sd_state* const* ha, sd_state* const* hb) {
    require(A.n == B.n && A.n_local == B.n_local && A.sh.size() == B.sh.size(), "fidelity: dimension mismatch");
    canonical_set(A, ha);
    canonical_set(B, hb);
    std::vector<std::vector<double>> part(A.sh.size(), std::vector<double>(2, 0.0));
    for (size_t i = 0; i < A.sh.size(); ++i) {
        SDB_CUDA(cudaSetDevice(B.sh[i]->device));
        SDB_CUDA(cudaStreamSynchronize(B.sh[i]->stream));
        SDB_CUDA(cudaSetDevice(A.sh[i]->device));
        sdb::device_inner(*A.sh[i], *B.sh[i], &part[i][0], &part[i][1]);
    }
    const std::vector<double> all = gather_ranks(A, part);
    double re = 0.0, im = 0.0;
    for (size_t r = 0; 2 * r < all.size(); ++r) {
        re += all[2 * r];
        im += all[2 * r + 1];
    }
    return std::hypot(re, im);
}

bool approx_unitary(const double* u, int d) {
    // U U^dagger == I within 1e-10 (statevector.cpp:29-50)
    for (int r = 0; r < d; ++r) {
        for (int c = 0; c < d; ++c) {
            std::complex<double> e = 0.0;
            for (int k = 0; k < d; ++k)
                e += std::complex<double>(u[2 * (r * d + k)], u[2 * (r * d + k) + 1]) *
                     std::conj(std::complex<double>(u[2 * (c * d + k)], u[2 * (c * d + k) + 1]));
            if (std::abs(e - (r == c ? 1.0 : 0.0)) > 1e-10) return false;
        }
    }
    return true;
}

}  // namespace

extern "C" {

sd_status sd_apply_pauli_rotation(sd_state* h, uint64_t x_mask, uint64_t z_mask, double coeff, double dt) {
    return guard([&] {
        ShardSet S = one_shard(h);
        check_term_masks(S, &x_mask, &z_mask, 1, "pauli rotation: qubit count mismatch");
        rotation_set(S, x_mask, z_mask, coeff, dt);
        sync_all(S);
    });
}

sd_status sd_local_apply_pauli_rotation(sd_state* const* hs, int world, uint64_t x_mask, uint64_t z_mask,
                                        double coeff, double dt) {
    return guard([&] {
        ShardSet S = local_set(hs, world);
        check_term_masks(S, &x_mask, &z_mask, 1, "pauli rotation: qubit count mismatch");
        rotation_set(S, x_mask, z_mask, coeff, dt);
        sync_all(S);
    });
}

static void baseline_set(ShardSet& S, const uint64_t* x, const uint64_t* z, const double* coeffs, size_t n_terms,
                         double dt, int n_steps) {
    require(n_terms == 0 || (x && z && coeffs), "null term arrays");
    if (n_steps < 0) throw std::invalid_argument("plan needs n_steps >= 0");
    if (!std::isfinite(dt)) throw std::invalid_argument("plan needs finite total_time");
    check_term_masks(S, x, z, n_terms, "hamiltonian/state qubit counts differ");
    for (int step = 0; step < n_steps; ++step)
        for (size_t k = 0; k < n_terms; ++k) rotation_set(S, x[k], z[k], coeffs[k], dt);
    sync_all(S);
}

sd_status sd_evolve_baseline(sd_state* h, const uint64_t* x, const uint64_t* z, const double* coeffs, size_t n_terms,
                             double dt, int n_steps) {
    return guard([&] {
        ShardSet S = one_shard(h);
        baseline_set(S, x, z, coeffs, n_terms, dt, n_steps);
    });
}

sd_status sd_local_evolve_baseline(sd_state* const* hs, int world, const uint64_t* x, const uint64_t* z,
                                   const double* coeffs, size_t n_terms, double dt, int n_steps) {
    return guard([&] {
        ShardSet S = local_set(hs, world);
        baseline_set(S, x, z, coeffs, n_terms, dt, n_steps);
    });
}

sd_status sd_expectation(sd_state* h, const uint64_t* x, const uint64_t* z, const double* coeffs, size_t n_terms,
                         double* re, double* imag_residue) {
    return guard([&] {
        ShardSet S = one_shard(h);
        expectation_set(S, x, z, coeffs, n_terms, re, imag_residue);
    });
}

sd_status sd_local_expectation(sd_state* const* hs, int world, const uint64_t* x, const uint64_t* z,
                               const double* coeffs, size_t n_terms, double* re, double* imag_residue) {
    return guard([&] {
        ShardSet S = local_set(hs, world);
        expectation_set(S, x, z, coeffs, n_terms, re, imag_residue);
    });
}

sd_status sd_state_norm(sd_state* h, double* out) {
    return guard([&] {
        require(out != nullptr, "null output");
        ShardSet S = one_shard(h);
        *out = norm_set(S);
    });
}

sd_status sd_local_norm(sd_state* const* hs, int world, double* out) {
    return guard([&] {
        require(out != nullptr, "null output");
        ShardSet S = local_set(hs, world);
        *out = norm_set(S);
    });
}

sd_status sd_state_fidelity(sd_state* a, sd_state* b, double* out) {
    return guard([&] {
        require(out != nullptr, "null output");
        ShardSet A = one_shard(a), B = one_shard(b);
        *out = fidelity_set(A, B, &a, &b);
    });
}

sd_status sd_local_fidelity(sd_state* const* a, sd_state* const* b, int world, double* out) {
    return guard([&] {
        require(out != nullptr, "null output");
        ShardSet A = local_set(a, world), B = local_set(b, world);
        *out = fidelity_set(A, B, a, b);
    });
}

sd_status sd_apply_single_qubit(sd_state* h, const double* u, int target) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(u != nullptr, "null matrix");
        require_unsharded(s);
        check_qubit(s, target);
        if (!approx_unitary(u, 2)) throw std::invalid_argument("single-qubit matrix is not unitary");
        SDB_CUDA(cudaSetDevice(s.device));
        sdb::launch_single_qubit(s, u, s.phys_of[target]);
        bump(s, s.amps_count(), s.amps_count());
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_apply_two_qubit(sd_state* h, const double* u, int q1, int q2) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require(u != nullptr, "null matrix");
        require_unsharded(s);
        check_qubit(s, q1);
        check_qubit(s, q2);
        if (q1 == q2) throw std::invalid_argument("two-qubit gate requires distinct qubits");
        if (!approx_unitary(u, 4)) throw std::invalid_argument("two-qubit matrix is not unitary");
        SDB_CUDA(cudaSetDevice(s.device));
        sdb::launch_two_qubit(s, u, s.phys_of[q1], s.phys_of[q2]);
        bump(s, s.amps_count(), s.amps_count());
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

sd_status sd_exact_evolve(sd_state* h, const uint64_t* x, const uint64_t* z, const double* coeffs, size_t n_terms,
                          double t) {
    return guard([&] {
        sdb::StateImpl& s = st(h);
        require_unsharded(s);
        if (s.n > 12) throw std::invalid_argument("exact_evolve limited to n <= 12 qubits");
        require(n_terms == 0 || (x && z && coeffs), "null term arrays");
        if (!std::isfinite(t)) throw std::invalid_argument("exact_evolve: non-finite time");
        check_term_masks(one_shard(h), x, z, n_terms, "hamiltonian/state qubit counts differ");
        require_identity_layout(s);
        SDB_CUDA(cudaSetDevice(s.device));
        sdb::launch_exact_evolve(s, x, z, coeffs, n_terms, t);
        SDB_CUDA(cudaStreamSynchronize(s.stream));
    });
}

}  // extern "C"

