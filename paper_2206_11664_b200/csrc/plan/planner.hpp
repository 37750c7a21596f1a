// Pass planner: turns one Trotter step (a sequence of C_j, D_j, C_j^dagger
// sandwiches, reference proj/src/evolve.cpp:47-58) into a short list of
// shared-memory tile passes over the state.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace sdb {

// Gate ops per pass (planner cap): every gate op lowers to <= 2 micro-ops, so
// a pass's program staged in shared memory stays <= ~13 KiB.
constexpr int kMaxOpsPerPass = 96;

// Physical bits kept local in every pass (0..2: 8 lanes x 16 B = one 128-byte
// line); tiles of <= 3 qubits keep at least one free coordinate.
int fixed_bits_for(int k);

// Per-plan planner settings (override the SDB_* environment knobs) for the
// planning calls made while a KnobScope is alive on this thread.
struct PlannerKnobs {
    int max_hdepth = -1;  // WHT levels per pass, -1: SDB_MAX_HDEPTH / unlimited
    int tma = -1;         // specialised kernels stage tile loads through TMA (-1: default on / SDB_TMA)
    int ring = -1;        // ring pipeline (-1: default for R = 5 programs / SDB_RING; 0 off, 1 on)
    int lookahead = -1;   // look-ahead growth of a pass's local set (-1: SDB_LOOKAHEAD, default off)
};
class KnobScope {
  public:
    explicit KnobScope(const PlannerKnobs* k);
    ~KnobScope();
    KnobScope(const KnobScope&) = delete;
    KnobScope& operator=(const KnobScope&) = delete;

  private:
    const PlannerKnobs* prev_;
};

// One group as the planner sees it (a flattened DiagonalGroup).
struct GroupSpec {
    std::vector<int> h_pre, s_layer, h_post;
    std::vector<std::pair<int, int>> cnots, czs;
    std::vector<uint64_t> z_masks;
    std::vector<double> coeffs;
};

// Gate-level operation in logical qubits.
struct Op {
    enum Kind { H, CX, PH, DG } kind = H;
    int q = -1;              // H target, CX control
    uint64_t targets = 0;    // CX target mask
    uint64_t s_mask = 0;     // PH
    bool dagger = false;     // PH
    std::vector<std::pair<int, int>> czs;  // PH
    int group = -1;          // DG: index into groups
    int t0 = 0, t1 = -1;     // DG: term range [t0, t1) of the group (t1 < 0: all terms)
    double dt_scale = 1.0;   // DG: multiplier of dt
    bool defer_deep = false; // H on an always-local qubit: leave for the next pass rather than a 2nd WHT level
    uint64_t support = 0;    // qubits acted on (commutation checks)
    uint64_t need = 0;       // qubits that must be tile-local
};

// Builds the op sequence of one Trotter step (order 1 or 2).
// CNOT runs wider than max_targets are split (same-control CNOTs commute).
// resynth_cap > 0: re-synthesise each group's CNOT network into rounds whose
// targets fit resynth_cap tile-local qubits (same linear map, fewer passes).
// split_diag: every diagonal term (Pauli-Z string, S, CZ) becomes its own op
// with its own support, so Hadamards of later layers can run ahead in the
// same pass wherever a qubit's terms are done (temporal blocking).
// cz_to_cx: a qubit whose h_pre and h_post Hadamards enclose only CZs drops
// both, its CZs becoming CNOTs onto it (H_b CZ(a,b) H_b = CX(a->b)).
std::vector<Op> step_ops(const std::vector<GroupSpec>& groups, int n_qubits, int order, int max_targets,
                         int resynth_cap = 0, bool split_diag = false, bool cz_to_cx = false);

// A pass in physical bit positions.
struct PassStage {
    enum Kind { WHT, CX, POINT } kind;
    uint32_t mask = 0;       // WHT local mask / CX local target mask
    int ctrl_local = -1;     // CX
    int ctrl_phys = -1;      // CX (outer control)
    int point = -1;          // POINT: index into PassPlan::points
};

struct PointTerm {
    uint64_t mask;   // physical
    double coeff;    // signed coefficient c
    double dt_scale; // weight = -dt * dt_scale * coeff
};

struct PointSpec {
    uint64_t s1 = 0, s2 = 0;  // physical: quarter += popc(i&s1) + 2 popc(i&s2)
    std::vector<uint64_t> cz_masks;        // physical, 2 bits each (one per pair)
    std::vector<PointTerm> terms;
};

struct PassPlan {
    std::vector<int> lpos;      // physical positions of local coordinates (ascending)
    std::vector<PassStage> stages;
    std::vector<PointSpec> points;
    int butterflies = 0;        // WHT levels applied in this pass
    int scale_exp = 0;          // store scale = 2^-scale_exp
    std::vector<int> op_ids;    // ops scheduled here (debug)
    std::vector<int> store_sigma;  // non-empty: store out of place through this local bit permutation
    std::vector<std::pair<int, int>> xswaps;  // the exchange that follows (global bit, top local bit)
};

struct StepPlan {
    std::vector<PassPlan> passes;
    int tile_qubits = 0;
    double ref_sweeps = 0.0;     // reference KernelStats sweeps per step
    int group_applications = 0;
};

// Greedy list scheduling of `ops` into tile passes of <= k local qubits, of
// which the lowest `n_fixed` physical bits are always local (coalescing).
// phys_of maps logical qubit -> physical bit (identity for one device).
// finalize_scales = false leaves scale_exp at 0 (the sharded planner places
// the exact normalisation over all segments of a step, finalize_scales()).
StepPlan plan_step(const std::vector<Op>& ops, const std::vector<GroupSpec>& groups, int n_local,
                   int k, int n_fixed, const std::vector<int>& phys_of, bool finalize = true);

// Deferred exact normalisation over a pass sequence (see planner.cpp).
void finalize_scales(std::vector<PassPlan*>& passes);

double reference_sweeps(const std::vector<GroupSpec>& groups, int order);

// ------------------------------------------------------- sharded steps
// A state sharded over P = 2^g ranks keeps physical bits >= n_local on the
// rank index. A Hadamard or CNOT target on such a "global" bit needs a qubit
// remap: the step is cut into segments whose needed qubits are all local,
// and between segments an exchange swaps g' <= g global bits with the top
// g' local bits T_i = n_local - g' + i. Before the swap a local bit
// permutation sigma moves the evicted qubits onto T (folded into the last
// pass of the segment, which stores out of place). Rank r then sends local
// chunk c (top g' bits = c) to the rank whose swapped global bits equal c
// and receives into chunk [sender's swapped global bits].
struct ExchangeSpec {
    std::vector<int> sigma;                  // new physical position of local bit b (size n_local)
    std::vector<std::pair<int, int>> swaps;  // (global physical bit, local physical bit T_i)
};

struct Segment {
    StepPlan plan;                // passes in the segment's starting layout
    std::vector<int> phys_of;     // layout the passes run in
    bool exchange_after = false;
    ExchangeSpec ex;
};

struct ShardedStep {
    std::vector<int> phys_in, phys_out;
    std::vector<Segment> segs;
    int n_exchanges = 0;
    int n_passes = 0;   // including permute-only passes in front of exchanges
};

// Plans one Trotter step starting from layout phys_in. Exchanges are chosen
// Belady-style (evict the local qubits whose next use is furthest, looking
// into the next step); when the next step's first op would need a global
// qubit the remap is scheduled at the end of this step, so every exchange
// follows a pass of the same step except possibly the very first.
ShardedStep plan_sharded_step(const std::vector<Op>& ops, const std::vector<GroupSpec>& groups, int n_local,
                              int k, int n_fixed, const std::vector<int>& phys_in);

std::string describe_sharded_json(const ShardedStep& s);

std::string describe(const StepPlan& p);
// Machine-readable schedule (tests emulate it on the CPU).
std::string describe_json(const StepPlan& p);

}  // namespace sdb
