"""ctypes declarations for libsimdiag_b200.so (include/simdiag_c.h).

The shared library is the product: host grouping/synthesis in C++ and the
sm_100a kernels. There is no fallback: if the library is missing, importing
this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libsimdiag_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(no CPU fallback exists by design)"
    )

# RTLD_LOCAL: the library exports the reference's C++ names (simdiag::...), which
# must not interpose on the reference compiled into oracle/_ref by the tests.
lib = C.CDLL(LIB_PATH, mode=C.RTLD_LOCAL)

u64 = C.c_uint64
i32 = C.c_int32
P = C.c_void_p
sz = C.c_size_t
dbl = C.c_double


class GroupDesc(C.Structure):
    _fields_ = [
        ("group_index", C.c_int),
        ("n_qubits", C.c_int),
        ("n_h_pre", sz), ("h_pre", C.POINTER(i32)),
        ("n_cnots", sz), ("cnots", C.POINTER(i32)),
        ("n_czs", sz), ("czs", C.POINTER(i32)),
        ("n_s", sz), ("s_layer", C.POINTER(i32)),
        ("n_h_post", sz), ("h_post", C.POINTER(i32)),
        ("n_terms", sz),
        ("z_masks", C.POINTER(u64)),
        ("signed_coeffs", C.POINTER(dbl)),
        ("src_x", C.POINTER(u64)),
        ("src_z", C.POINTER(u64)),
        ("src_coeffs", C.POINTER(dbl)),
    ]


class KernelStats(C.Structure):
    _fields_ = [("amp_reads", u64), ("amp_writes", u64), ("kernel_calls", u64)]


class PlanOptions(C.Structure):
    _fields_ = [
        ("order", C.c_int),
        ("tile_qubits", C.c_int),
        ("fuse", C.c_int),
        ("use_graph", C.c_int),
        ("relabel", C.c_int),
        ("reserved", C.c_int * 7),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("n_passes_per_step", C.c_int),
        ("n_ref_sweeps_per_step", C.c_int),
        ("n_group_applications", C.c_int),
        ("n_exchanges_per_step", C.c_int),
        ("tile_qubits", C.c_int),
        ("n_kernels_per_step", C.c_int),
        ("bytes_per_step", dbl),
        ("schedule", C.c_int),
        ("tune_ms_whole", dbl),
        ("tune_ms_split", dbl),
        ("tune_ms_whole_ring", dbl),
        ("ring", C.c_int),
        ("tune_ms_split_deep", dbl),
        ("max_hdepth", C.c_int),
        ("macro_steps", C.c_int),
        ("macro_passes", C.c_int),
        ("tune_ms_macro", dbl),
        ("tune_ms_split_nocap", dbl),
    ]


def _sig(name, argtypes, restype=C.c_int):
    f = getattr(lib, name)
    f.argtypes = argtypes
    f.restype = restype
    return f


PP = C.POINTER(P)
sd_last_error = _sig("sd_last_error", [], C.c_char_p)
sd_version = _sig("sd_version", [], C.c_char_p)
sd_hamiltonian_from_terms = _sig(
    "sd_hamiltonian_from_terms",
    [C.c_int, C.POINTER(u64), C.POINTER(u64), C.POINTER(dbl), sz, dbl, C.POINTER(sz), PP],
)
sd_gen_tfim = _sig("sd_gen_tfim", [C.c_int, u64, PP])
sd_gen_syk = _sig("sd_gen_syk", [C.c_int, u64, C.POINTER(sz), C.POINTER(sz), PP])
sd_hamiltonian_load_text = _sig("sd_hamiltonian_load_text", [C.c_char_p, sz, dbl, PP])
sd_hamiltonian_load_file = _sig("sd_hamiltonian_load_file", [C.c_char_p, dbl, PP])
sd_hamiltonian_save_text = _sig("sd_hamiltonian_save_text", [P, C.c_char_p, sz, C.POINTER(sz)])
sd_hamiltonian_info = _sig("sd_hamiltonian_info", [P, C.POINTER(C.c_int), C.POINTER(sz)])
sd_hamiltonian_terms = _sig("sd_hamiltonian_terms", [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(dbl)])
sd_hamiltonian_destroy = _sig("sd_hamiltonian_destroy", [P], None)
sd_partition = _sig("sd_partition", [P, PP])
sd_partition_only = _sig("sd_partition_only", [P, PP])
sd_diagonalize_terms = _sig(
    "sd_diagonalize_terms", [C.c_int, C.POINTER(u64), C.POINTER(u64), C.POINTER(dbl), sz, PP]
)
sd_groups_count = _sig("sd_groups_count", [P, C.POINTER(sz)])
sd_groups_destroy = _sig("sd_groups_destroy", [P], None)
sd_group_get = _sig("sd_group_get", [P, sz, C.POINTER(GroupDesc)])

sd_state_create = _sig("sd_state_create", [C.c_int, C.c_int, PP])
sd_state_create_shard = _sig("sd_state_create_shard", [C.c_int, C.c_int, C.c_int, C.c_int, PP])
sd_state_destroy = _sig("sd_state_destroy", [P], None)
sd_state_info = _sig("sd_state_info", [P] + [C.POINTER(C.c_int)] * 4)
sd_state_stream = _sig("sd_state_stream", [P, PP])
sd_state_device_ptr = _sig("sd_state_device_ptr", [P, PP])
sd_sync = _sig("sd_sync", [P])
sd_state_set_basis = _sig("sd_state_set_basis", [P, u64])
sd_state_set_plus = _sig("sd_state_set_plus", [P])
sd_state_set_random = _sig("sd_state_set_random", [P, u64])
sd_state_upload = _sig("sd_state_upload", [P, P, u64])
sd_state_download = _sig("sd_state_download", [P, P, u64])
sd_state_download_range = _sig("sd_state_download_range", [P, u64, u64, P])
sd_state_norm_sq = _sig("sd_state_norm_sq", [P, C.POINTER(dbl)])
sd_state_inner = _sig("sd_state_inner", [P, P, C.POINTER(dbl), C.POINTER(dbl)])
sd_state_copy = _sig("sd_state_copy", [P, P])
sd_kernel_stats_get = _sig("sd_kernel_stats_get", [P, C.POINTER(KernelStats)])
sd_kernel_stats_reset = _sig("sd_kernel_stats_reset", [P])
sd_apply_hadamard = _sig("sd_apply_hadamard", [P, C.c_int])
sd_apply_batched_cnot = _sig("sd_apply_batched_cnot", [P, C.c_int, u64])
sd_apply_phase_layer = _sig("sd_apply_phase_layer", [P, u64, C.POINTER(i32), sz, C.c_int])
sd_apply_diagonal_exp = _sig("sd_apply_diagonal_exp", [P, C.POINTER(u64), C.POINTER(dbl), sz, dbl])
sd_apply_clifford = _sig("sd_apply_clifford", [P, C.POINTER(GroupDesc)])
sd_apply_clifford_inverse = _sig("sd_apply_clifford_inverse", [P, C.POINTER(GroupDesc)])

sd_plan_options_default = _sig("sd_plan_options_default", [C.POINTER(PlanOptions)])
sd_plan_create = _sig("sd_plan_create", [P, C.POINTER(GroupDesc), sz, C.POINTER(PlanOptions), PP])
sd_plan_destroy = _sig("sd_plan_destroy", [P], None)
sd_plan_get_info = _sig("sd_plan_get_info", [P, C.POINTER(PlanInfo)])
sd_plan_describe = _sig("sd_plan_describe", [P, C.c_char_p, sz, C.POINTER(sz)])
sd_plan_preview = _sig(
    "sd_plan_preview",
    [C.c_int, C.c_int, C.POINTER(GroupDesc), sz, C.POINTER(PlanOptions), C.POINTER(PlanInfo), C.c_char_p, sz,
     C.POINTER(sz)],
)
sd_evolve = _sig("sd_evolve", [P, dbl, C.c_int])
sd_evolve_async = _sig("sd_evolve_async", [P, dbl, C.c_int])
sd_plan_set_profiling = _sig("sd_plan_set_profiling", [P, C.c_int])
sd_plan_kernel_times = _sig(
    "sd_plan_kernel_times", [P, C.POINTER(dbl), C.POINTER(u64), C.POINTER(dbl), C.c_int]
)
sd_comm_unique_id = _sig("sd_comm_unique_id", [C.c_char_p])
sd_state_attach_comm = _sig("sd_state_attach_comm", [P, C.c_char_p])
sd_state_canonicalize = _sig("sd_state_canonicalize", [P])
sd_groups_diag_json = _sig("sd_groups_diag_json", [P, C.c_int, C.c_char_p, sz, C.POINTER(sz)])
sd_state_save_raw = _sig("sd_state_save_raw", [P, C.c_char_p])
sd_state_load_raw = _sig("sd_state_load_raw", [P, C.c_char_p])
sd_apply_pauli_rotation = _sig("sd_apply_pauli_rotation", [P, u64, u64, dbl, dbl])
sd_evolve_baseline = _sig("sd_evolve_baseline", [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(dbl), sz, dbl, C.c_int])
sd_expectation = _sig("sd_expectation", [P, C.POINTER(u64), C.POINTER(u64), C.POINTER(dbl), sz, C.POINTER(dbl),
                                         C.POINTER(dbl)])
PU, PD = C.POINTER(u64), C.POINTER(dbl)
sd_state_norm = _sig("sd_state_norm", [P, PD])
sd_state_fidelity = _sig("sd_state_fidelity", [P, P, PD])
sd_local_expectation = _sig("sd_local_expectation", [C.POINTER(P), C.c_int, PU, PU, PD, sz, PD, PD])
sd_local_apply_pauli_rotation = _sig("sd_local_apply_pauli_rotation", [C.POINTER(P), C.c_int, u64, u64, dbl, dbl])
sd_local_evolve_baseline = _sig("sd_local_evolve_baseline", [C.POINTER(P), C.c_int, PU, PU, PD, sz, dbl, C.c_int])
sd_local_norm = _sig("sd_local_norm", [C.POINTER(P), C.c_int, PD])
sd_local_fidelity = _sig("sd_local_fidelity", [C.POINTER(P), C.POINTER(P), C.c_int, PD])
sd_apply_single_qubit = _sig("sd_apply_single_qubit", [P, PD, C.c_int])
sd_apply_two_qubit = _sig("sd_apply_two_qubit", [P, PD, C.c_int, C.c_int])
sd_exact_evolve = _sig("sd_exact_evolve", [P, PU, PU, PD, sz, dbl])
sd_jit_compile_preview = _sig("sd_jit_compile_preview", [C.c_int, C.c_int, C.POINTER(GroupDesc), sz,
                                                         C.POINTER(PlanOptions), C.POINTER(sz)])
sd_state_create_local_shards = _sig("sd_state_create_local_shards", [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(P)])
sd_evolve_local = _sig("sd_evolve_local", [C.POINTER(P), C.c_int, dbl, C.c_int])
sd_local_canonicalize = _sig("sd_local_canonicalize", [C.POINTER(P), C.c_int])
sd_local_enable_p2p = _sig("sd_local_enable_p2p", [C.POINTER(P), C.c_int])
sd_state_ipc_handles = _sig("sd_state_ipc_handles", [P, C.c_char_p])
sd_state_attach_peers = _sig("sd_state_attach_peers", [P, C.c_char_p])


class Route(C.Structure):
    _fields_ = [("peer", C.c_int), ("send_offset", u64), ("recv_offset", u64), ("count", u64)]


sd_exchange_routes = _sig("sd_exchange_routes", [C.c_int, C.c_int, C.c_int, C.POINTER(i32), sz, C.POINTER(Route), sz,
                                                 C.POINTER(sz)])

EXPORTED = [
    "sd_last_error", "sd_version",
    "sd_hamiltonian_from_terms", "sd_hamiltonian_load_text", "sd_hamiltonian_load_file",
    "sd_hamiltonian_save_text", "sd_hamiltonian_info", "sd_hamiltonian_terms",
    "sd_hamiltonian_destroy", "sd_partition", "sd_partition_only", "sd_diagonalize_terms",
    "sd_groups_count", "sd_groups_destroy", "sd_group_get",
    "sd_state_create", "sd_state_create_shard", "sd_state_destroy", "sd_state_info",
    "sd_state_stream", "sd_state_device_ptr", "sd_sync", "sd_state_set_basis", "sd_state_set_plus",
    "sd_state_set_random", "sd_state_upload", "sd_state_download", "sd_state_download_range", "sd_state_norm_sq",
    "sd_state_inner", "sd_state_copy", "sd_kernel_stats_get", "sd_kernel_stats_reset",
    "sd_apply_hadamard", "sd_apply_batched_cnot", "sd_apply_phase_layer", "sd_apply_diagonal_exp",
    "sd_apply_clifford", "sd_apply_clifford_inverse",
    "sd_plan_options_default", "sd_plan_create", "sd_plan_destroy", "sd_plan_get_info",
    "sd_plan_describe", "sd_plan_preview", "sd_evolve", "sd_evolve_async", "sd_plan_set_profiling",
    "sd_plan_kernel_times", "sd_comm_unique_id", "sd_state_attach_comm", "sd_state_canonicalize",
    "sd_state_create_local_shards", "sd_evolve_local", "sd_local_canonicalize", "sd_exchange_routes",
    "sd_jit_compile_preview", "sd_apply_pauli_rotation", "sd_evolve_baseline", "sd_expectation",
    "sd_local_enable_p2p", "sd_state_ipc_handles", "sd_state_attach_peers", "sd_groups_diag_json",
    "sd_state_save_raw", "sd_state_load_raw",
    "sd_state_norm", "sd_state_fidelity", "sd_local_expectation", "sd_local_apply_pauli_rotation",
    "sd_local_evolve_baseline", "sd_local_norm", "sd_local_fidelity", "sd_apply_single_qubit",
    "sd_apply_two_qubit", "sd_exact_evolve", "sd_gen_tfim", "sd_gen_syk",
]


class SimdiagError(RuntimeError):
    pass


class CudaError(SimdiagError):
    pass


class NcclError(SimdiagError):
    pass


class OutOfMemory(SimdiagError, MemoryError):
    pass


def check(status: int) -> None:
    """Map sd_status onto the reference's exception types
    (invalid_argument -> ValueError, out_of_range -> IndexError,
    runtime_error -> RuntimeError)."""
    if status == 0:
        return
    msg = (sd_last_error() or b"").decode(errors="replace")
    if status == 1:
        raise ValueError(msg)
    if status == 2:
        raise IndexError(msg)
    if status == 3:
        raise RuntimeError(msg)
    if status == 4:
        raise CudaError(msg)
    if status == 5:
        raise NcclError(msg)
    if status == 6:
        raise OutOfMemory(msg)
    raise SimdiagError(f"status {status}: {msg}")
