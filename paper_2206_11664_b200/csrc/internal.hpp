// Internal types shared by the C ABI, the planner and the CUDA launchers.
// Not part of the public boundary (include/simdiag_c.h is).
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "plan_dev.h"
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
// (the POD structures live in plan_dev.h; see there for the semantics)
inline uint32_t host_swz(uint32_t l) { return l ^ ((l >> 3) & 7u) ^ ((l >> 6) & 7u) ^ ((l >> 9) & 7u); }

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
    void* nccl = nullptr;    // ncclComm_t when attached
    double* xbuf = nullptr;  // exchange receive buffer (lazily allocated)
    uint64_t xbuf_amps = 0;
    // Fused exchange over peer memory (sd_state_attach_peers /
    // sd_local_enable_p2p): peer_buf[r] = rank r's two state buffers as they
    // were when peers were attached; amps/xbuf swap roles at every exchange and
    // `parity` tracks which of the two is a rank's current receive buffer.
    bool p2p = false;
    int parity = 0;
    std::vector<std::pair<double*, double*>> peer_buf;
    std::vector<void*> ipc_opened;       // peer mappings to close on destroy
    double2** xdst_dev = nullptr;        // device table: destination per chunk
    double* reduce_buf = nullptr;
    int sm_count = 0;
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
// apply_pauli_rotation (statevector.cpp:288-337) and one term of expectation
// (evolve.cpp:99-135): <psi| i^{phase} X^x Z^z |psi>. x and z are PHYSICAL
// masks including the global (rank) bits; when x has global bits, `partner`
// is a copy of shard rank ^ (x >> n_local) taken before the update.
void launch_pauli_rotation(StateImpl& s, uint64_t x, uint64_t z, double coeff, double dt,
                           const double* partner = nullptr);
void device_expectation_term(StateImpl& s, uint64_t x, uint64_t z, const double* partner, double* re, double* im);
// apply_single_qubit / apply_two_qubit (statevector.cpp:101-154); u holds
// row-major complex entries as (re, im) pairs; physical qubit positions.
void launch_single_qubit(StateImpl& s, const double* u, int target);
void launch_two_qubit(StateImpl& s, const double* u, int q1, int q2);
// exact_evolve (evolve.cpp:60-97): psi <- exp(-i H t) psi, H = sum_k c_k P_k
void launch_exact_evolve(StateImpl& s, const uint64_t* x, const uint64_t* z, const double* c, size_t m, double t);

// Fused pass launcher (pass_kernel.cu).
// out: destination buffer (nullptr = in place on s.amps); xdst: device table of
// per-chunk destination buffers for a fused exchange store (nullptr: none).
void launch_tile_pass(StateImpl& s, const PassDev& pass_host, int pass_index, const PlanDev& plan,
                      double dt, uint64_t rank_bits, double* out, double2* const* xdst = nullptr);
int max_tile_qubits();
// per-tile constant phases of a pass's table point (PassDev::tphase_off)
void launch_tile_phase(StateImpl& s, const PassDev& pass_host, int pass_index, const PlanDev& plan, double dt,
                       uint64_t rank_bits, double2* out);

}  // namespace sdb
