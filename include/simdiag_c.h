/*
 * simdiag_c.h -- C ABI of the B200 Trotter hot path (libsimdiag_b200.so).
 *
 * The reference (arXiv 2206.11664 `simdiag`) exposes only a C++ API; this
 * header is the thin extern "C" layer SURVEY.md §8(b) specifies under it.
 * Every entry point names the reference interface it replaces
 * (paths relative to the reference root). Conventions:
 *   - every call returns sd_status; on failure sd_last_error() holds a
 *     thread-local message. Status codes map 1:1 onto the reference's
 *     exception types (invalid_argument / out_of_range / runtime_error);
 *   - host arrays are copied at call time, never retained;
 *   - handles own their device memory; one handle is used by one host
 *     thread at a time;
 *   - device calls are stream-ordered on the state's stream and return
 *     after completion unless documented otherwise (sd_evolve_async);
 *   - amplitudes are interleaved (re, im) doubles, index bit q = qubit q.
 * No torch types cross this boundary.
 */
#ifndef SIMDIAG_C_H
#define SIMDIAG_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sd_status {
    SD_OK = 0,
    SD_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    SD_OUT_OF_RANGE = 2,     /* std::out_of_range */
    SD_RUNTIME_ERROR = 3,    /* std::runtime_error */
    SD_CUDA_ERROR = 4,
    SD_NCCL_ERROR = 5,
    SD_OOM = 6
} sd_status;

const char* sd_last_error(void);
const char* sd_version(void);

/* ------------------------------------------------------------------ */
/* Host side: Hamiltonian, grouping, synthesis (bit-exact)             */
/* ------------------------------------------------------------------ */

typedef struct sd_hamiltonian sd_hamiltonian;

/* Hamiltonian::from_terms  (proj/include/simdiag/hamiltonian.hpp:25-28,
 * proj/src/hamiltonian.cpp:36-69). merged may be NULL. */
sd_status sd_hamiltonian_from_terms(int n_qubits, const uint64_t* x_masks, const uint64_t* z_masks,
                                    const double* coeffs, size_t n_terms, double drop_tolerance,
                                    size_t* merged, sd_hamiltonian** out);
/* gen_tfim / gen_syk (proj/include/simdiag/models.hpp:13-34,
 * proj/src/models.cpp:17-92): the paper's benchmark models, identical to the
 * reference's (same counter-RNG draws and term order). The SYK counts may be
 * NULL. */
sd_status sd_gen_tfim(int n_qubits, uint64_t seed, sd_hamiltonian** out);
sd_status sd_gen_syk(int n_qubits, uint64_t seed, size_t* candidate_quadruples, size_t* merge_collisions,
                     sd_hamiltonian** out);
/* Hamiltonian::load (hamiltonian.hpp:33, hamiltonian.cpp:71-118) on an
 * in-memory text buffer. */
sd_status sd_hamiltonian_load_text(const char* text, size_t len, double drop_tolerance,
                                   sd_hamiltonian** out);
/* Hamiltonian::load_file (hamiltonian.hpp:34-35, hamiltonian.cpp:120-126). */
sd_status sd_hamiltonian_load_file(const char* path, double drop_tolerance, sd_hamiltonian** out);
/* Hamiltonian::save (hamiltonian.cpp:128-133). Writes up to cap bytes
 * (NUL-terminated when room) and the full length to *len. */
sd_status sd_hamiltonian_save_text(const sd_hamiltonian* h, char* buf, size_t cap, size_t* len);
sd_status sd_hamiltonian_info(const sd_hamiltonian* h, int* n_qubits, size_t* n_terms);
/* Hamiltonian::terms() copied out; any pointer may be NULL. */
sd_status sd_hamiltonian_terms(const sd_hamiltonian* h, uint64_t* x_masks, uint64_t* z_masks,
                               double* coeffs);
void sd_hamiltonian_destroy(sd_hamiltonian* h);

/* Result of greedy_partition + diagonalize_group over every group. */
typedef struct sd_groups sd_groups;

/* greedy_partition (hamiltonian.hpp:59, hamiltonian.cpp:135-158) followed
 * by diagonalize_group per group (diagonalize.hpp:61, diagonalize.cpp:188-212). */
sd_status sd_partition(const sd_hamiltonian* h, sd_groups** out);
/* greedy_partition only; circuits are left empty and sd_group_get reports
 * n_terms with z_masks/coeffs NULL. */
sd_status sd_partition_only(const sd_hamiltonian* h, sd_groups** out);
/* diagonalize_group on one explicit group (for synthesis KATs). */
sd_status sd_diagonalize_terms(int n_qubits, const uint64_t* x_masks, const uint64_t* z_masks,
                               const double* coeffs, size_t n_terms, sd_groups** out);
sd_status sd_groups_count(const sd_groups* g, size_t* n_groups);
void sd_groups_destroy(sd_groups* g);

/* Flattened DiagonalGroup (proj/include/simdiag/clifford_circuit.hpp:14-53)
 * plus the source CommutingGroup terms. Pointers borrow from the owner. */
typedef struct sd_group_desc {
    int group_index;
    int n_qubits;
    size_t n_h_pre;
    const int32_t* h_pre;
    size_t n_cnots;
    const int32_t* cnots; /* 2*n_cnots: (control, target) in application order */
    size_t n_czs;
    const int32_t* czs;   /* 2*n_czs: (low, high) */
    size_t n_s;
    const int32_t* s_layer;
    size_t n_h_post;
    const int32_t* h_post;
    size_t n_terms;
    const uint64_t* z_masks;     /* diagonalised masks   (DiagonalGroup::z_masks) */
    const double* signed_coeffs; /* (DiagonalGroup::signed_coeffs) */
    const uint64_t* src_x;       /* source terms (CommutingGroup::terms) */
    const uint64_t* src_z;
    const double* src_coeffs;
} sd_group_desc;

sd_status sd_group_get(const sd_groups* g, size_t index, sd_group_desc* out);

/* diag_document (proj/src/serialize.cpp:46-66, serialize.hpp:21): the `diag`
 * JSON of a synthesised partition -- circuits, hex z-masks, signed
 * coefficients -- the bit-exact grouping/circuit diff format. Same cap/len
 * protocol as sd_hamiltonian_save_text. */
sd_status sd_groups_diag_json(const sd_groups* g, int n_qubits, char* buf, size_t cap, size_t* len);

/* ------------------------------------------------------------------ */
/* Device state (replaces StateVector, statevector.hpp:34-97)          */
/* ------------------------------------------------------------------ */

typedef struct sd_state sd_state;

/* KernelStats (statevector.hpp:23-27): amplitude loads/stores per sweep. */
typedef struct sd_kernel_stats {
    uint64_t amp_reads;
    uint64_t amp_writes;
    uint64_t kernel_calls;
} sd_kernel_stats;

/* StateVector(n) = |0..0> on one device. Unlike the reference (n <= 30,
 * statevector.cpp:63-65) the cap is device memory. */
sd_status sd_state_create(int n_qubits, int device, sd_state** out);
/* One shard of a 2^n state split over `world` ranks on the top log2(world)
 * qubits; this rank holds indices [rank*2^(n-g), (rank+1)*2^(n-g)). */
sd_status sd_state_create_shard(int n_qubits, int rank, int world, int device, sd_state** out);
void sd_state_destroy(sd_state* s);
sd_status sd_state_info(const sd_state* s, int* n_qubits, int* n_local_qubits, int* rank,
                        int* world);
/* cudaStream_t of the state, for event timing by the caller. */
sd_status sd_state_stream(const sd_state* s, void** stream);
/* Raw device pointer to this shard's 2^n_local amplitudes (interleaved
 * re/im doubles, physical layout). */
sd_status sd_state_device_ptr(const sd_state* s, void** ptr);
sd_status sd_sync(sd_state* s);

/* zero_state / basis |index>, plus_state, random_state(n, seed)
 * (statevector.cpp:59-93; same counter-based RNG, generated on device). */
sd_status sd_state_set_basis(sd_state* s, uint64_t index);
sd_status sd_state_set_plus(sd_state* s);
sd_status sd_state_set_random(sd_state* s, uint64_t seed);
/* Host <-> device copies of this shard, logical index order. n_amps must
 * equal the shard size. */
sd_status sd_state_upload(sd_state* s, const double* re_im, uint64_t n_amps);
sd_status sd_state_download(sd_state* s, double* re_im, uint64_t n_amps);
/* Amplitudes [first, first + count) of this shard in logical order (the
 * reference's StateVector::operator[] over a range, statevector.hpp:48-50) --
 * partial readout of states larger than host memory allows at once. */
sd_status sd_state_download_range(sd_state* s, uint64_t first, uint64_t count, double* re_im);
/* save_raw / load_raw (statevector.cpp:383-401): raw little-endian (re, im)
 * doubles of this shard's index range in logical order (a relabelled layout is
 * canonicalised first, collectively for NCCL-attached shards); the rank files
 * concatenate to the reference's file. */
sd_status sd_state_save_raw(sd_state* s, const char* path);
sd_status sd_state_load_raw(sd_state* s, const char* path);
/* Sum |a|^2 over this shard (pairwise tree on device) -> sqrt is the
 * caller's once shards are combined; norm() of statevector.cpp:403-407 is
 * sqrt(sd_state_norm_sq) for world == 1. */
sd_status sd_state_norm_sq(sd_state* s, double* out);
/* <a|b> over this shard (fidelity(), statevector.cpp:409-418, is |.| of
 * the sum over shards). */
sd_status sd_state_inner(sd_state* a, sd_state* b, double* re, double* im);
sd_status sd_state_copy(sd_state* dst, const sd_state* src);
sd_status sd_kernel_stats_get(const sd_state* s, sd_kernel_stats* out);
sd_status sd_kernel_stats_reset(sd_state* s);

/* ---- single-sweep kernels (StateVector methods, statevector.hpp:53-82) */
/* apply_hadamard (statevector.cpp:156-174) */
sd_status sd_apply_hadamard(sd_state* s, int target);
/* apply_batched_cnot (statevector.cpp:176-203) */
sd_status sd_apply_batched_cnot(sd_state* s, int control, uint64_t targets);
/* apply_phase_layer (statevector.cpp:205-245); pairs = 2*n_pairs ints */
sd_status sd_apply_phase_layer(sd_state* s, uint64_t s_mask, const int32_t* pairs, size_t n_pairs,
                               int dagger);
/* apply_diagonal_exp (statevector.cpp:247-286) */
sd_status sd_apply_diagonal_exp(sd_state* s, const uint64_t* z_masks, const double* coeffs,
                                size_t n_terms, double dt);
/* apply_clifford / apply_clifford_inverse (statevector.cpp:339-381):
 * the reference's unfused layer-by-layer sweep sequence. */
sd_status sd_apply_clifford(sd_state* s, const sd_group_desc* g);
sd_status sd_apply_clifford_inverse(sd_state* s, const sd_group_desc* g);

/* ---- the paper's comparison method and observables */
/* apply_pauli_rotation (statevector.cpp:288-337): exp(-i coeff dt P), P the
 * Hermitian Pauli with symplectic masks (x, z) (pauli.hpp:23-61). */
sd_status sd_apply_pauli_rotation(sd_state* s, uint64_t x_mask, uint64_t z_mask, double coeff, double dt);
/* evolve_baseline (evolve.cpp:21-45): n_steps x one rotation sweep per term
 * in the given order (Hamiltonian order, or groups flattened = group-major). */
sd_status sd_evolve_baseline(sd_state* s, const uint64_t* x_masks, const uint64_t* z_masks, const double* coeffs,
                             size_t n_terms, double dt, int n_steps);
/* expectation (evolve.cpp:99-135): sum_k coeffs[k] <psi|P_k|psi>; real part
 * in *re, |imaginary residue| in *imag_residue (may be NULL). Device
 * reductions in a fixed order (bit-identical for any launch).
 *
 * Sharded states (one process per GPU, communicator attached): these calls,
 * sd_apply_pauli_rotation, sd_evolve_baseline, sd_state_norm and
 * sd_state_fidelity are COLLECTIVE -- every rank calls them with the same
 * arguments. A term whose X part flips a global (rank) qubit pairs
 * amplitudes across shards: each rank copies its partner shard (rank ^ the
 * global X bits) into its exchange buffer over NCCL first. Per-shard partials
 * are all-gathered and summed in rank order, so the result is identical on
 * every rank. Masks address LOGICAL qubits; a relabelled state is handled by
 * mapping them to physical bits (no canonicalisation). */
sd_status sd_expectation(sd_state* s, const uint64_t* x_masks, const uint64_t* z_masks, const double* coeffs,
                         size_t n_terms, double* re, double* imag_residue);
/* norm() (statevector.cpp:403-407) of the whole (sharded) state. */
sd_status sd_state_norm(sd_state* s, double* out);
/* fidelity() = |<a|b>| (statevector.cpp:409-418) of two whole (sharded)
 * states with the same shape (relabelled layouts are canonicalised first). */
sd_status sd_state_fidelity(sd_state* a, sd_state* b, double* out);
/* The same operations on `world` in-process shards (sd_state_create_local_shards). */
sd_status sd_local_expectation(sd_state* const* shards, int world, const uint64_t* x_masks,
                               const uint64_t* z_masks, const double* coeffs, size_t n_terms, double* re,
                               double* imag_residue);
sd_status sd_local_apply_pauli_rotation(sd_state* const* shards, int world, uint64_t x_mask, uint64_t z_mask,
                                        double coeff, double dt);
sd_status sd_local_evolve_baseline(sd_state* const* shards, int world, const uint64_t* x_masks,
                                   const uint64_t* z_masks, const double* coeffs, size_t n_terms, double dt,
                                   int n_steps);
sd_status sd_local_norm(sd_state* const* shards, int world, double* out);
sd_status sd_local_fidelity(sd_state* const* a, sd_state* const* b, int world, double* out);

/* apply_single_qubit / apply_two_qubit (statevector.hpp:53-55,
 * statevector.cpp:101-154): u = row-major 2x2 (8 doubles) / 4x4 (32 doubles)
 * complex matrix as (re, im) pairs, unitary within 1e-10 (else
 * SD_INVALID_ARGUMENT, "... matrix is not unitary"); the two-qubit local
 * index is 2*bit(q1) + bit(q2). Unsharded states. */
sd_status sd_apply_single_qubit(sd_state* s, const double* u, int target);
sd_status sd_apply_two_qubit(sd_state* s, const double* u, int q1, int q2);
/* exact_evolve (evolve.hpp:38-42, evolve.cpp:60-97): psi <- exp(-i H t) psi
 * for n <= 12 (the reference's dense test oracle; here a time-sliced Taylor
 * series on the device). */
sd_status sd_exact_evolve(sd_state* s, const uint64_t* x_masks, const uint64_t* z_masks, const double* coeffs,
                          size_t n_terms, double t);

/* ------------------------------------------------------------------ */
/* Fused Trotter plan (replaces evolve_grouped, evolve.cpp:47-58)       */
/* ------------------------------------------------------------------ */

typedef struct sd_plan sd_plan;

typedef struct sd_plan_options {
    int order;        /* 1 = first-order Lie-Trotter (evolve_grouped), 2 = Suzuki S2 */
    int tile_qubits;  /* k: qubits per shared-memory tile; 0 = auto */
    int fuse;         /* 1 = fused tile passes (default); 0 = reference sweep sequence */
    int use_graph;    /* 0 = auto (replay each step as a CUDA graph for unsharded states of
                         <= 20 qubits, which are launch-bound), 1 = always, -1 = never */
    int relabel;      /* 1 = allow qubit relabelling between passes (default) */
    int reserved[7];
} sd_plan_options;

sd_status sd_plan_options_default(sd_plan_options* o);
/* groups: DiagonalGroups in evolution order (as passed to evolve_grouped).
 * Host data is copied. For unsharded states of >= 22 qubits the plan is
 * autotuned: when per-term diagonal ops schedule into fewer passes, both
 * schedules are built and one step of each is timed on the state's second
 * buffer (the state itself is untouched); the faster one is kept
 * (sd_plan_info::schedule). SDB_AUTOTUNE=0 disables it. */
sd_status sd_plan_create(sd_state* s, const sd_group_desc* groups, size_t n_groups,
                         const sd_plan_options* opts, sd_plan** out);
void sd_plan_destroy(sd_plan* p);

typedef struct sd_plan_info {
    int n_passes_per_step;      /* P_sched: full-state sweeps per step */
    int n_ref_sweeps_per_step;  /* P_ref: the reference's sweeps per step (KernelStats) */
    int n_group_applications;   /* P_floor */
    int n_exchanges_per_step;   /* qubit remaps that cross ranks */
    int tile_qubits;
    int n_kernels_per_step;     /* kernel launches per step */
    double bytes_per_step;      /* algorithmic HBM bytes per step, this shard */
    int schedule;               /* 0: whole-group diagonal ops, 1: per-term diagonal ops */
    double tune_ms_whole;       /* plan-time autotune: ms per step of each schedule (0: not timed) */
    double tune_ms_split;
    double tune_ms_whole_ring;  /* ... whole-group schedule through the ring pipeline */
    int ring;                   /* ring pipeline: -1 default (per-term plans), 0 off, 1 on */
    double tune_ms_split_deep;  /* ... per-term schedule with <= 3 Hadamard levels per pass */
    int max_hdepth;             /* Hadamard levels per pass of the kept plan (0: no cap, -1: default) */
    int macro_steps;            /* > 0: whole groups of this many Trotter steps run as one planned macro step */
    int macro_passes;           /* passes per macro step of the kept (or, macro_steps = 0, the tried) macro plan */
    double tune_ms_macro;       /* plan-time autotune: ms per Trotter step of the macro plan (0: not timed) */
    double tune_ms_split_nocap; /* ... per-term schedule with no cap on Hadamard levels per pass */
} sd_plan_info;

sd_status sd_plan_get_info(const sd_plan* p, sd_plan_info* out);
/* Human-readable schedule dump (for DESIGN/debug); same cap/len protocol as
 * sd_hamiltonian_save_text. */
sd_status sd_plan_describe(const sd_plan* p, char* buf, size_t cap, size_t* len);

/* Host-only: run the planner for a (sharded) state shape without touching a
 * device; fills *info (may be NULL) and writes the schedule as JSON
 * (passes -> local bit positions, stages, exact scale exponents). */
sd_status sd_plan_preview(int n_qubits, int world, const sd_group_desc* groups, size_t n_groups,
                          const sd_plan_options* opts, sd_plan_info* info, char* json, size_t cap,
                          size_t* len);

/* EvolutionPlan{total_time = dt*n_steps, n_steps} then evolve_grouped:
 * n_steps Trotter steps of size dt. n_steps == 0 is a no-op (evolve.cpp:13).
 * Blocks until complete. */
sd_status sd_evolve(sd_plan* p, double dt, int n_steps);
/* Same but returns after enqueueing on the state's stream. */
sd_status sd_evolve_async(sd_plan* p, double dt, int n_steps);

/* Per-kernel-class device time (CUDA events around every launch while
 * enabled). classes: 0 = fused tile pass, 1 = diagonal-only pass,
 * 2 = exchange, 3 = other. */
sd_status sd_plan_set_profiling(sd_plan* p, int enable);
sd_status sd_plan_kernel_times(sd_plan* p, double* ms_by_class, uint64_t* launches_by_class,
                               double* bytes_by_class, int n_classes);

/* Plans for large shards (default n_local >= 22; SDB_JIT=0/1 overrides) run
 * each pass as a kernel specialised for its micro-program, generated and
 * compiled for sm_100a with NVRTC at plan time. Host-only check: plan the
 * first step for an n-qubit state over `world` ranks and compile every
 * distinct pass program (no device needed). */
sd_status sd_jit_compile_preview(int n_qubits, int world, const sd_group_desc* groups, size_t n_groups,
                                 const sd_plan_options* opts, size_t* n_programs);

/* ------------------------------------------------------------------ */
/* Multi-rank exchange (NCCL over NVLink; one process per GPU)          */
/* ------------------------------------------------------------------ */

/* The state shards on the top log2(world) qubits (sd_state_create_shard).
 * Diagonals, S/CZ layers and CNOTs with a global control run without
 * communication; a Hadamard or CNOT target on a global qubit is handled by a
 * qubit remap that the planner inserts between pass segments: the pass in
 * front of it stores out of place through a local bit permutation, then the
 * ranks swap chunks (no reference counterpart -- the reference has
 * no distributed state). */

/* 128-byte ncclUniqueId, produced on rank 0 and broadcast by the caller. */
sd_status sd_comm_unique_id(unsigned char id[128]);
/* Bind a shard state to an NCCL communicator over all `world` ranks
 * (libnccl.so.2 is resolved at run time). sd_evolve then performs the remaps
 * with grouped ncclSend/ncclRecv on the state's stream. */
sd_status sd_state_attach_comm(sd_state* s, const unsigned char id[128]);
/* Restore the canonical layout (logical qubit q at physical bit q) of a
 * relabelled state; collective over the communicator for sharded states.
 * sd_state_download does this implicitly. */
sd_status sd_state_canonicalize(sd_state* s);

/* Several shards driven by ONE process (devices[r] may repeat, e.g. virtual
 * shards on one GPU): remaps are device copies between the shards' buffers,
 * with exactly the NCCL path's routing. plans[r] must be created on shard r. */
sd_status sd_state_create_local_shards(int n_qubits, int world, const int* devices, sd_state** out);
sd_status sd_evolve_local(sd_plan* const* plans, int world, double dt, int n_steps);
sd_status sd_local_canonicalize(sd_state* const* shards, int world);

/* Fused exchange over peer memory: the pass in front of a remap stores every
 * amplitude straight into the receiving rank's buffer (NVLink stores, one
 * kernel for compute + exchange; no separate collective), followed by one
 * barrier; state and receive buffers then swap roles. Multi-process:
 * sd_state_ipc_handles gives this shard's two 64-byte cudaIpcMemHandles (state,
 * receive buffer); the caller all-gathers them (world x 128 bytes in rank
 * order) and passes them to sd_state_attach_peers on every rank (after
 * sd_state_attach_comm, which supplies the barrier). In-process shards:
 * sd_local_enable_p2p. */
sd_status sd_state_ipc_handles(sd_state* s, unsigned char out[128]);
sd_status sd_state_attach_peers(sd_state* s, const unsigned char* handles);
sd_status sd_local_enable_p2p(sd_state* const* shards, int world);

/* Chunk routing of one remap exchange for `rank` (host-only; the routing both
 * transports execute, exported for multi-process tests). swaps = 2*n_swaps
 * ints (global bit, local bit) as in sd_plan_preview's JSON. Offsets and
 * counts are in amplitudes of the rank's shard: send B[send_offset, +count)
 * to peer, receive into A[recv_offset, +count); peer == rank is a local copy. */
typedef struct sd_route {
    int peer;
    uint64_t send_offset;
    uint64_t recv_offset;
    uint64_t count;
} sd_route;
sd_status sd_exchange_routes(int n_qubits, int n_local, int rank, const int32_t* swaps, size_t n_swaps,
                             sd_route* out, size_t cap, size_t* n_out);

#ifdef __cplusplus
}
#endif

#endif /* SIMDIAG_C_H */
