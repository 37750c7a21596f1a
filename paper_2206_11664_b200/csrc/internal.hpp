// Internal types shared by the C ABI, the planner and the CUDA launchers.
// Not part of the public boundary (include/simdiag_c.h is).
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "simdiag_c.h"

namespace sdb {

// ---------------------------------------------------------------- errors
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct OomError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);
#define SDB_CUDA(call) ::sdb::cuda_check((call), #call)

// ------------------------------------------------------- device-side plan
// A tile pass: every CTA loads 2^k amplitudes whose index bits outside
// `lpos` are fixed (the tile's outer bits), runs the stage list on them in
// shared memory and stores them back in place. One pass = one full-state
// HBM read + write.
enum StageKind : int {
    kStageWht = 0,    // unnormalised butterflies on local coords in `mask`
    kStageCx = 1,     // l -> l ^ targets when the control bit is set
    kStagePoint = 2,  // pointwise i^q(i) * exp(i*phi(i)), see PointDev
};

struct StageDev {
    int kind;
    uint32_t mask;    // WHT: local coordinate mask; CX: local target mask
    int ctrl_local;   // CX: local coordinate of the control, or -1
    int ctrl_phys;    // CX: physical bit of an outer control, or -1
    int point;        // POINT: index into PointDev array
    int pad;
};

// Pointwise factor on physical index i (of the whole state: the shard's rank
// bits are OR-ed in by the kernel):
//   q(i)   = popc(i & s1) + 2*popc(i & s2) + 2*parity(#CZ pairs fully set in i)
//   phi(i) = -dt * sum_t  c_t * (-1)^{popc(i & zmask_t)}
//   a     <- a * i^q * exp(i*phi)
// Direct mode (n_seg == 0): loop over the terms' full masks.
// Table mode  (n_seg > 0): terms are grouped by their local part u (a mask
// over tile coordinates); per tile the kernel forms
//   A[u] = sum_{t in seg(u)} c_t (-1)^{popc(outer_bits & zh_t)}
// and a Walsh-Hadamard transform over `table_mask` turns A into phi/(-dt)
// for all 2^k amplitudes of the tile (SURVEY §7 "Diagonal").
struct PointDev {
    uint64_t s1;
    uint64_t s2;
    int n_cz;
    int cz_off;    // into cz pair masks (uint64 with 2 bits set)
    int n_terms;
    int term_off;  // into term masks / coefficients
    int n_seg;
    int seg_off;   // into SegDev
    uint32_t table_mask;
    int pad;
};

struct SegDev {
    uint32_t u;    // local part of the terms' masks (tile coordinates)
    int begin;     // terms [begin, end) relative to PointDev::term_off
    int end;
    int pad;
};

struct PassDev {
    int k;                 // local qubit count (tile = 2^k amplitudes)
    int n_outer;           // outer bit count (= n_local - k)
    int n_stages;
    int stage_off;
    int lpos[16];          // physical bit position of local coordinate j
    int opos[64];          // physical bit position of outer coordinate j
    double scale;          // applied on store (exact power of two)
    int flags;             // kPassNeedsTable: some POINT stage uses the angle table
    int pad;
};
constexpr int kPassNeedsTable = 1;

// --------------------------------------------------------------- handles
struct StateImpl {
    int n = 0;        // logical qubits (whole state)
    int n_local = 0;  // qubits stored here: 2^n_local amplitudes
    int rank = 0, world = 1;
    int device = 0;
    double* amps = nullptr;  // interleaved (re, im)
    cudaStream_t stream = nullptr;
    sd_kernel_stats stats{0, 0, 0};
    // Physical layout: phys_of[q] = physical index bit holding logical q.
    // Bits >= n_local select the rank. Identity unless a plan relabelled.
    std::vector<int> phys_of;
    void* nccl = nullptr;        // ncclComm_t when attached
    double* xbuf = nullptr;      // exchange receive buffer (lazily allocated)
    uint64_t xbuf_amps = 0;
    double* reduce_buf = nullptr;
    uint64_t amps_count() const { return uint64_t(1) << n_local; }
};

// Unfused primitive launchers (kernels_basic.cu).
void launch_set_basis(StateImpl& s, uint64_t local_index_or_max);
void launch_fill(StateImpl& s, double re, double im);
void launch_random(StateImpl& s, uint64_t seed);
void launch_scale(StateImpl& s, double f);
double device_norm_sq(StateImpl& s);
void device_inner(StateImpl& a, StateImpl& b, double* re, double* im);
void launch_hadamard(StateImpl& s, int target_phys);
void launch_batched_cnot(StateImpl& s, int control_phys, uint64_t targets_phys);
void launch_phase_layer(StateImpl& s, uint64_t s_mask, const std::vector<uint64_t>& pair_masks,
                        bool dagger);
void launch_diag_exp(StateImpl& s, const std::vector<uint64_t>& masks,
                     const std::vector<double>& coeffs, double dt);
void launch_permute_bits(StateImpl& s, const double* src, double* dst, const int* new_pos,
                         int n_bits);

// Fused pass launcher (pass_kernel.cu). `dev_*` are device arrays owned by
// the plan; `pass_host` is the host copy of the descriptor (for k).
struct PlanDev {
    const PassDev* passes;
    const StageDev* stages;
    const PointDev* points;
    const SegDev* segs;
    const uint64_t* cz_masks;
    const uint64_t* term_masks;
    const double* term_coeffs;  // c_t * dt_scale; the kernel multiplies by -dt
};
void launch_tile_pass(StateImpl& s, const PassDev& pass_host, int pass_index, const PlanDev& plan,
                      double dt, uint64_t rank_bits);
int max_tile_qubits();

}  // namespace sdb
