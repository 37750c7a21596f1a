"""Python mirror of the reference's public API (proj/include/simdiag/*.hpp)
over the C ABI of libsimdiag_b200.so.

Names, argument meaning and error behaviour follow the reference:
  PauliString             pauli.hpp:23-61
  Hamiltonian             hamiltonian.hpp:19-45 (from_terms / load / save)
  greedy_partition        hamiltonian.hpp:59
  diagonalize_group       diagonalize.hpp:61
  CliffordCircuit, DiagonalGroup   clifford_circuit.hpp:14-53
  StateVector             statevector.hpp:34-97 (device-resident here)
  EvolutionPlan, evolve_grouped    evolve.hpp:15-35
Exceptions: std::invalid_argument -> ValueError, std::out_of_range ->
IndexError, std::runtime_error -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as A
from ._capi import check

K_MAX_QUBITS = 64
K_DROP_TOLERANCE = 1e-12


def _u64arr(vals) -> "C.Array":
    vals = list(vals)
    return (C.c_uint64 * max(1, len(vals)))(*vals)


def _dblarr(vals) -> "C.Array":
    vals = list(vals)
    return (C.c_double * max(1, len(vals)))(*vals)


def _i32arr(vals) -> "C.Array":
    vals = list(vals)
    return (C.c_int32 * max(1, len(vals)))(*vals)


# --------------------------------------------------------------------- Pauli


@dataclasses.dataclass(frozen=True)
class PauliString:
    """Symplectic Pauli string; qubit 0 is the leftmost character and owns
    bit 0 of both masks (pauli.hpp:15-17)."""

    n_qubits: int
    x_mask: int
    z_mask: int

    @staticmethod
    def parse(text: str, n_qubits: Optional[int] = None) -> "PauliString":
        n = len(text) if n_qubits is None else n_qubits
        if n < 0 or n > K_MAX_QUBITS:
            raise ValueError(f"qubit count must be in [0, 64], got {n}")
        if len(text) != n:
            raise ValueError(f"pauli string length {len(text)} does not match qubit count {n}")
        x = z = 0
        for q, ch in enumerate(text):
            if ch not in "IXYZ":
                raise ValueError(f"invalid pauli character '{ch}' at position {q + 1}")
            if ch in "XY":
                x |= 1 << q
            if ch in "ZY":
                z |= 1 << q
        return PauliString(n, x, z)

    @staticmethod
    def from_masks(n_qubits: int, x: int, z: int) -> "PauliString":
        if n_qubits < 0 or n_qubits > K_MAX_QUBITS:
            raise ValueError(f"qubit count must be in [0, 64], got {n_qubits}")
        if (x | z) >> n_qubits:
            raise ValueError("mask has bits beyond qubit count")
        return PauliString(n_qubits, x, z)

    def str(self) -> str:  # noqa: A003 - mirrors PauliString::str()
        return "".join("IXZY"[((self.x_mask >> q) & 1) | (((self.z_mask >> q) & 1) << 1)] for q in range(self.n_qubits))

    def phase_exp(self) -> int:
        return bin(self.x_mask & self.z_mask).count("1") & 3


def commutes(a: PauliString, b: PauliString) -> bool:
    if a.n_qubits != b.n_qubits:
        raise ValueError("commutes: qubit counts differ")
    return ((bin(a.x_mask & b.z_mask).count("1") + bin(a.z_mask & b.x_mask).count("1")) & 1) == 0


@dataclasses.dataclass
class WeightedTerm:
    coeff: float
    pauli: PauliString


# --------------------------------------------------------------- Hamiltonian


class Hamiltonian:
    """Handle over the C++ Hamiltonian (merge + drop on construction)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None):
            A.sd_hamiltonian_destroy(self._h)
            self._h = None

    @staticmethod
    def from_terms(n_qubits: int, terms: Sequence, drop_tolerance: float = K_DROP_TOLERANCE,
                   return_merged: bool = False):
        xs, zs, cs = [], [], []
        for t in terms:
            if isinstance(t, WeightedTerm):
                c, p = t.coeff, t.pauli
            else:
                c, p = t
            if isinstance(p, str):
                p = PauliString.parse(p, n_qubits)
            if p.n_qubits != n_qubits:
                raise ValueError("term qubit count does not match hamiltonian")
            xs.append(p.x_mask)
            zs.append(p.z_mask)
            cs.append(float(c))
        merged = C.c_size_t(0)
        out = C.c_void_p()
        check(A.sd_hamiltonian_from_terms(n_qubits, _u64arr(xs), _u64arr(zs), _dblarr(cs), len(cs),
                                          drop_tolerance, C.byref(merged), C.byref(out)))
        h = Hamiltonian(out.value)
        return (h, merged.value) if return_merged else h

    @staticmethod
    def load(text: str, drop_tolerance: float = K_DROP_TOLERANCE) -> "Hamiltonian":
        b = text.encode()
        out = C.c_void_p()
        check(A.sd_hamiltonian_load_text(b, len(b), drop_tolerance, C.byref(out)))
        return Hamiltonian(out.value)

    @staticmethod
    def load_file(path: str, drop_tolerance: float = K_DROP_TOLERANCE) -> "Hamiltonian":
        out = C.c_void_p()
        check(A.sd_hamiltonian_load_file(path.encode(), drop_tolerance, C.byref(out)))
        return Hamiltonian(out.value)

    def save(self) -> str:
        n = C.c_size_t(0)
        check(A.sd_hamiltonian_save_text(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(A.sd_hamiltonian_save_text(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    @property
    def n_qubits(self) -> int:
        n = C.c_int(0)
        check(A.sd_hamiltonian_info(self._h, C.byref(n), None))
        return n.value

    def term_count(self) -> int:
        m = C.c_size_t(0)
        check(A.sd_hamiltonian_info(self._h, None, C.byref(m)))
        return m.value

    def term_arrays(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        m = self.term_count()
        x = np.zeros(max(1, m), np.uint64)
        z = np.zeros(max(1, m), np.uint64)
        c = np.zeros(max(1, m), np.float64)
        check(A.sd_hamiltonian_terms(self._h, x.ctypes.data_as(C.POINTER(C.c_uint64)),
                                     z.ctypes.data_as(C.POINTER(C.c_uint64)),
                                     c.ctypes.data_as(C.POINTER(C.c_double))))
        return x[:m], z[:m], c[:m]

    def terms(self) -> List[WeightedTerm]:
        n = self.n_qubits
        x, z, c = self.term_arrays()
        return [WeightedTerm(float(ci), PauliString(n, int(xi), int(zi))) for xi, zi, ci in zip(x, z, c)]


def gen_tfim(n_qubits: int, seed: int) -> Hamiltonian:
    """Fully connected TFIM (models.hpp:13, models.cpp:17-35)."""
    out = C.c_void_p()
    check(A.sd_gen_tfim(n_qubits, seed, C.byref(out)))
    return Hamiltonian(out.value)


def gen_syk(n_qubits: int, seed: int, with_info: bool = False):
    """SYK quartic Majorana model over 2n modes (models.hpp:29-34,
    models.cpp:48-90); with_info adds (candidate_quadruples, merge_collisions)."""
    out = C.c_void_p()
    q, col = C.c_size_t(0), C.c_size_t(0)
    check(A.sd_gen_syk(n_qubits, seed, C.byref(q), C.byref(col), C.byref(out)))
    h = Hamiltonian(out.value)
    return (h, (q.value, col.value)) if with_info else h


# ----------------------------------------------------------------- circuits


@dataclasses.dataclass
class CliffordCircuit:
    n_qubits: int = 0
    h_pre: List[int] = dataclasses.field(default_factory=list)
    cnots: List[Tuple[int, int]] = dataclasses.field(default_factory=list)
    czs: List[Tuple[int, int]] = dataclasses.field(default_factory=list)
    s_layer: List[int] = dataclasses.field(default_factory=list)
    h_post: List[int] = dataclasses.field(default_factory=list)

    def empty(self) -> bool:
        return self.gate_count() == 0

    def gate_count(self) -> int:
        return len(self.h_pre) + len(self.cnots) + len(self.czs) + len(self.s_layer) + len(self.h_post)


@dataclasses.dataclass
class CommutingGroup:
    group_index: int
    terms: List[WeightedTerm]


@dataclasses.dataclass
class DiagonalGroup:
    group_index: int
    circuit: CliffordCircuit
    z_masks: List[int]
    signed_coeffs: List[float]
    terms: List[WeightedTerm] = dataclasses.field(default_factory=list)

    def _desc(self):
        """Flatten into sd_group_desc; returns (desc, keepalive)."""
        c = self.circuit
        keep = [
            _i32arr(c.h_pre), _i32arr([q for p in c.cnots for q in p]), _i32arr([q for p in c.czs for q in p]),
            _i32arr(c.s_layer), _i32arr(c.h_post), _u64arr(self.z_masks), _dblarr(self.signed_coeffs),
        ]
        d = A.GroupDesc()
        d.group_index = self.group_index
        d.n_qubits = c.n_qubits
        d.n_h_pre, d.h_pre = len(c.h_pre), keep[0]
        d.n_cnots, d.cnots = len(c.cnots), keep[1]
        d.n_czs, d.czs = len(c.czs), keep[2]
        d.n_s, d.s_layer = len(c.s_layer), keep[3]
        d.n_h_post, d.h_post = len(c.h_post), keep[4]
        d.n_terms = len(self.z_masks)
        d.z_masks, d.signed_coeffs = keep[5], keep[6]
        return d, keep


def _groups_from_handle(handle, n_qubits: int, synthesized: bool):
    cnt = C.c_size_t(0)
    check(A.sd_groups_count(handle, C.byref(cnt)))
    out = []
    for g in range(cnt.value):
        d = A.GroupDesc()
        check(A.sd_group_get(handle, g, C.byref(d)))
        circ = CliffordCircuit(
            n_qubits=n_qubits,
            h_pre=[d.h_pre[i] for i in range(d.n_h_pre)],
            cnots=[(d.cnots[2 * i], d.cnots[2 * i + 1]) for i in range(d.n_cnots)],
            czs=[(d.czs[2 * i], d.czs[2 * i + 1]) for i in range(d.n_czs)],
            s_layer=[d.s_layer[i] for i in range(d.n_s)],
            h_post=[d.h_post[i] for i in range(d.n_h_post)],
        )
        terms = [WeightedTerm(d.src_coeffs[i], PauliString(n_qubits, d.src_x[i], d.src_z[i])) for i in range(d.n_terms)]
        if synthesized:
            zm = [d.z_masks[i] for i in range(d.n_terms)]
            cf = [d.signed_coeffs[i] for i in range(d.n_terms)]
            out.append(DiagonalGroup(d.group_index, circ, zm, cf, terms))
        else:
            out.append(CommutingGroup(d.group_index, terms))
    A.sd_groups_destroy(handle)
    return out


def greedy_partition(h: Hamiltonian) -> List[CommutingGroup]:
    out = C.c_void_p()
    check(A.sd_partition_only(h._h, C.byref(out)))
    return _groups_from_handle(out, h.n_qubits, synthesized=False)


def partition_and_diagonalize(h: Hamiltonian) -> List[DiagonalGroup]:
    """greedy_partition followed by diagonalize_group on every group."""
    out = C.c_void_p()
    check(A.sd_partition(h._h, C.byref(out)))
    return _groups_from_handle(out, h.n_qubits, synthesized=True)


def diagonalize_group(group) -> DiagonalGroup:
    terms = group.terms if isinstance(group, CommutingGroup) else list(group)
    if not terms:
        raise ValueError("cannot diagonalize an empty group")
    n = terms[0].pauli.n_qubits
    out = C.c_void_p()
    check(A.sd_diagonalize_terms(n, _u64arr(t.pauli.x_mask for t in terms), _u64arr(t.pauli.z_mask for t in terms),
                                 _dblarr(t.coeff for t in terms), len(terms), C.byref(out)))
    d = _groups_from_handle(out, n, synthesized=True)[0]
    d.group_index = group.group_index if isinstance(group, CommutingGroup) else 0
    return d


# --------------------------------------------------------------------- state


class StateVector:
    """Device-resident 2^n complex128 state (StateVector, statevector.hpp).

    Mutating methods run the reference's single-sweep semantics on the GPU;
    `amplitudes()` downloads to host. With world > 1 this object is one
    shard on the top log2(world) qubits.
    """

    def __init__(self, n_qubits: int, device: int = 0, rank: int = 0, world: int = 1, _handle=None):
        if _handle is None:
            h = C.c_void_p()
            check(A.sd_state_create_shard(n_qubits, rank, world, device, C.byref(h)))
        else:
            h = C.c_void_p(_handle)
        self._s = h
        nl = C.c_int(0)
        check(A.sd_state_info(self._s, None, C.byref(nl), None, None))
        self.n = n_qubits
        self.n_local = nl.value
        self.rank, self.world, self.device = rank, world, device

    def __del__(self):
        if getattr(self, "_s", None):
            A.sd_state_destroy(self._s)
            self._s = None

    # constructors (statevector.hpp:37-45)
    @staticmethod
    def zero_state(n_qubits: int, device: int = 0) -> "StateVector":
        return StateVector(n_qubits, device)

    @staticmethod
    def plus_state(n_qubits: int, device: int = 0) -> "StateVector":
        s = StateVector(n_qubits, device)
        check(A.sd_state_set_plus(s._s))
        return s

    @staticmethod
    def random_state(n_qubits: int, seed: int, device: int = 0) -> "StateVector":
        s = StateVector(n_qubits, device)
        check(A.sd_state_set_random(s._s, seed))
        return s

    @staticmethod
    def basis_state(n_qubits: int, index: int, device: int = 0) -> "StateVector":
        s = StateVector(n_qubits, device)
        check(A.sd_state_set_basis(s._s, index))
        return s

    def n_qubits(self) -> int:
        return self.n

    def dim(self) -> int:
        return 1 << self.n

    def set_basis(self, index: int) -> None:
        check(A.sd_state_set_basis(self._s, index))

    def upload(self, amps: np.ndarray) -> None:
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        check(A.sd_state_upload(self._s, a.ctypes.data, a.size))

    def upload_ptr(self, host_ptr: int, n_amps: int) -> None:
        check(A.sd_state_upload(self._s, host_ptr, n_amps))

    def download_ptr(self, host_ptr: int, n_amps: int) -> None:
        check(A.sd_state_download(self._s, host_ptr, n_amps))

    def amplitudes(self, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        """This shard's amplitudes in logical order; `first`/`count` read a
        range (operator[] over a slice) without staging the whole shard."""
        if first == 0 and count is None:
            out = np.empty(1 << self.n_local, np.complex128)
            check(A.sd_state_download(self._s, out.ctypes.data, out.size))
            return out
        count = (1 << self.n_local) - first if count is None else count
        out = np.empty(count, np.complex128)
        check(A.sd_state_download_range(self._s, first, count, out.ctypes.data))
        return out

    def norm_sq_local(self) -> float:
        v = C.c_double()
        check(A.sd_state_norm_sq(self._s, C.byref(v)))
        return v.value

    def norm(self) -> float:
        """norm() of the whole state (statevector.cpp:403-407); for a shard of
        a multi-process state this is collective over the communicator."""
        if self.world == 1:
            return math.sqrt(self.norm_sq_local())
        v = C.c_double()
        check(A.sd_state_norm(self._s, C.byref(v)))
        return v.value

    def stats(self) -> dict:
        k = A.KernelStats()
        check(A.sd_kernel_stats_get(self._s, C.byref(k)))
        return {"amp_reads": k.amp_reads, "amp_writes": k.amp_writes, "kernel_calls": k.kernel_calls}

    def reset_stats(self) -> None:
        check(A.sd_kernel_stats_reset(self._s))

    def stream(self) -> int:
        p = C.c_void_p()
        check(A.sd_state_stream(self._s, C.byref(p)))
        return p.value or 0

    def device_ptr(self) -> int:
        p = C.c_void_p()
        check(A.sd_state_device_ptr(self._s, C.byref(p)))
        return p.value or 0

    def attach_comm(self, unique_id: bytes) -> None:
        """Bind this shard to an NCCL communicator (sd_state_attach_comm);
        every rank passes the same 128-byte id from comm_unique_id()."""
        check(A.sd_state_attach_comm(self._s, C.create_string_buffer(bytes(unique_id), 128)))

    def save_raw(self, path: str) -> None:
        """statevector.cpp:383-387: raw (re, im) doubles of this shard, logical order."""
        check(A.sd_state_save_raw(self._s, str(path).encode()))

    def load_raw(self, path: str) -> None:
        """statevector.cpp:389-401 into this (existing) shard."""
        check(A.sd_state_load_raw(self._s, str(path).encode()))

    def ipc_handles(self) -> bytes:
        """This shard's two cudaIpcMemHandles (state, receive buffer), 128 bytes."""
        buf = C.create_string_buffer(128)
        check(A.sd_state_ipc_handles(self._s, buf))
        return buf.raw

    def attach_peers(self, all_handles: Sequence[bytes]) -> None:
        """Fused exchange over peer memory: every rank's ipc_handles(), in rank
        order (sd_state_attach_peers; needs attach_comm first)."""
        blob = b"".join(bytes(h) for h in all_handles)
        check(A.sd_state_attach_peers(self._s, C.create_string_buffer(blob, len(blob))))

    def canonicalize(self) -> None:
        """Undo qubit relabelling (collective for NCCL-attached shards)."""
        check(A.sd_state_canonicalize(self._s))

    def sync(self) -> None:
        check(A.sd_sync(self._s))

    # single-sweep kernels (statevector.hpp:53-82)
    def apply_hadamard(self, target: int) -> None:
        check(A.sd_apply_hadamard(self._s, target))

    def apply_batched_cnot(self, control: int, targets: int) -> None:
        check(A.sd_apply_batched_cnot(self._s, control, targets))

    def apply_phase_layer(self, s_mask: int, cz_pairs: Sequence[Tuple[int, int]], dagger: bool = False) -> None:
        flat = [q for p in cz_pairs for q in p]
        check(A.sd_apply_phase_layer(self._s, s_mask, _i32arr(flat), len(cz_pairs), 1 if dagger else 0))

    def apply_diagonal_exp(self, z_masks, coeffs=None, dt: float = 0.0) -> None:
        if isinstance(z_masks, DiagonalGroup):
            g, dt = z_masks, (coeffs if coeffs is not None else dt)
            z_masks, coeffs = g.z_masks, g.signed_coeffs
        if len(z_masks) != len(coeffs):
            raise ValueError("diagonal exp: mask/coefficient count mismatch")
        check(A.sd_apply_diagonal_exp(self._s, _u64arr(z_masks), _dblarr(coeffs), len(z_masks), dt))

    def apply_clifford(self, g: DiagonalGroup) -> None:
        d, keep = g._desc()
        check(A.sd_apply_clifford(self._s, C.byref(d)))

    def apply_clifford_inverse(self, g: DiagonalGroup) -> None:
        d, keep = g._desc()
        check(A.sd_apply_clifford_inverse(self._s, C.byref(d)))

    def apply_pauli_rotation(self, term: WeightedTerm, dt: float) -> None:
        """exp(-i coeff dt P) (statevector.cpp:288-337); collective for a
        shard of a multi-process state."""
        check(A.sd_apply_pauli_rotation(self._s, term.pauli.x_mask, term.pauli.z_mask, term.coeff, dt))

    def apply_single_qubit(self, u, target: int) -> None:
        """Generic 2x2 unitary (statevector.cpp:101-122), row-major."""
        m = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(4))
        check(A.sd_apply_single_qubit(self._s, m.ctypes.data_as(C.POINTER(C.c_double)), target))

    def apply_two_qubit(self, u, q1: int, q2: int) -> None:
        """Generic 4x4 unitary (statevector.cpp:124-154); local index
        2*bit(q1) + bit(q2)."""
        m = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(16))
        check(A.sd_apply_two_qubit(self._s, m.ctypes.data_as(C.POINTER(C.c_double)), q1, q2))


def norm(psi: StateVector) -> float:
    return psi.norm()


def fidelity(a, b) -> float:
    """|<a|b>| (statevector.cpp:409-418) of whole states: StateVectors
    (collective for multi-process shards) or LocalShards."""
    v = C.c_double()
    if isinstance(a, LocalShards):
        check(A.sd_local_fidelity(a._arr(), b._arr(), a.world, C.byref(v)))
    else:
        check(A.sd_state_fidelity(a._s, b._s, C.byref(v)))
    return v.value


# ----------------------------------------------------------------- evolution


@dataclasses.dataclass
class EvolutionPlan:
    """evolve.hpp:15-23; `order` (1 or 2) is this framework's extension."""

    total_time: float = 0.0
    n_steps: int = 1
    order: int = 1

    def dt(self) -> float:
        return self.total_time / self.n_steps

    def validate(self) -> None:
        if self.n_steps < 0:
            raise ValueError("plan needs n_steps >= 0")
        if not math.isfinite(self.total_time):
            raise ValueError("plan needs finite total_time")


class TrotterPlan:
    """A compiled schedule (sd_plan): fused tile passes for one Trotter step
    over `groups`, bound to `psi`. Reusable across evolve() calls."""

    def __init__(self, psi: StateVector, groups: Sequence[DiagonalGroup], order: int = 1,
                 tile_qubits: int = 0, fuse: bool = True, use_graph: Optional[bool] = None):
        self.psi = psi
        opts = A.PlanOptions()
        check(A.sd_plan_options_default(C.byref(opts)))
        opts.order = order
        opts.tile_qubits = tile_qubits
        opts.fuse = 1 if fuse else 0
        opts.use_graph = 0 if use_graph is None else (1 if use_graph else -1)  # None: auto (small states)
        descs = (A.GroupDesc * max(1, len(groups)))()
        self._keep = []
        for i, g in enumerate(groups):
            d, k = g._desc()
            descs[i] = d
            self._keep.append(k)
        h = C.c_void_p()
        check(A.sd_plan_create(psi._s, descs, len(groups), C.byref(opts), C.byref(h)))
        self._p = h

    def __del__(self):
        if getattr(self, "_p", None):
            A.sd_plan_destroy(self._p)
            self._p = None

    def info(self) -> dict:
        i = A.PlanInfo()
        check(A.sd_plan_get_info(self._p, C.byref(i)))
        return {f: getattr(i, f) for f, _ in A.PlanInfo._fields_}

    def describe(self) -> str:
        n = C.c_size_t(0)
        check(A.sd_plan_describe(self._p, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(A.sd_plan_describe(self._p, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def evolve(self, dt: float, n_steps: int, wait: bool = True) -> None:
        check((A.sd_evolve if wait else A.sd_evolve_async)(self._p, dt, n_steps))

    def set_profiling(self, on: bool) -> None:
        check(A.sd_plan_set_profiling(self._p, 1 if on else 0))

    def kernel_times(self) -> dict:
        ms = (C.c_double * 4)()
        ln = (C.c_uint64 * 4)()
        by = (C.c_double * 4)()
        check(A.sd_plan_kernel_times(self._p, ms, ln, by, 4))
        names = ["tile_pass", "diag_pass", "exchange", "other"]
        return {names[c]: {"ms": ms[c], "launches": ln[c], "bytes": by[c]} for c in range(4)}


def plan_preview(n_qubits: int, groups: Sequence[DiagonalGroup], order: int = 1, tile_qubits: int = 0,
                 world: int = 1) -> Tuple[dict, dict]:
    """Host-only planner run: (info, schedule-as-dict). No device needed."""
    import json

    opts = A.PlanOptions()
    check(A.sd_plan_options_default(C.byref(opts)))
    opts.order = order
    opts.tile_qubits = tile_qubits
    descs = (A.GroupDesc * max(1, len(groups)))()
    keep = []
    for i, g in enumerate(groups):
        d, k = g._desc()
        descs[i] = d
        keep.append(k)
    info = A.PlanInfo()
    n = C.c_size_t(0)
    check(A.sd_plan_preview(n_qubits, world, descs, len(groups), C.byref(opts), C.byref(info), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(A.sd_plan_preview(n_qubits, world, descs, len(groups), C.byref(opts), None, buf, n.value + 1, C.byref(n)))
    return {f: getattr(info, f) for f, _ in A.PlanInfo._fields_}, json.loads(buf.value.decode())


def evolve_grouped(groups: Sequence[DiagonalGroup], psi: StateVector, plan: EvolutionPlan, **options) -> None:
    """evolve_grouped (evolve.cpp:47-58): per step and group, C_j, exp(-i dt
    Lambda_j), C_j^dagger -- executed as fused tile passes on the GPU."""
    plan.validate()
    dt = plan.dt() if plan.n_steps > 0 else 0.0
    if plan.n_steps == 0:
        return
    TrotterPlan(psi, groups, order=plan.order, **options).evolve(dt, plan.n_steps)


def _term_arrays(terms):
    xs = _u64arr([t.pauli.x_mask for t in terms])
    zs = _u64arr([t.pauli.z_mask for t in terms])
    cs = _dblarr([t.coeff for t in terms])
    return xs, zs, cs


def evolve_baseline(h, psi, plan: EvolutionPlan) -> None:
    """The paper's per-term baseline (evolve.cpp:21-45): n_steps x one rotation
    sweep per term; `h` is a Hamiltonian (input order) or a list of
    CommutingGroup/DiagonalGroup (group-major order). `psi` is a StateVector
    (collective for a multi-process shard) or LocalShards."""
    plan.validate()
    if isinstance(h, Hamiltonian):
        if h.n_qubits != psi.n:
            raise ValueError("hamiltonian/state qubit counts differ")
        terms = h.terms()
    else:
        terms = [t for g in h for t in g.terms]
    dt = plan.dt() if plan.n_steps > 0 else 0.0
    xs, zs, cs = _term_arrays(terms)
    if isinstance(psi, LocalShards):
        check(A.sd_local_evolve_baseline(psi._arr(), psi.world, xs, zs, cs, len(terms), dt, plan.n_steps))
    else:
        check(A.sd_evolve_baseline(psi._s, xs, zs, cs, len(terms), dt, plan.n_steps))


def expectation(h: "Hamiltonian", psi, with_residue: bool = False):
    """<psi|H|psi> (evolve.cpp:99-135) as device reductions; returns the real
    part (and the |imaginary residue| when with_residue). `psi` is a
    StateVector (collective for a multi-process shard) or LocalShards."""
    if h.n_qubits != psi.n:
        raise ValueError("hamiltonian/state qubit counts differ")
    terms = h.terms()
    xs, zs, cs = _term_arrays(terms)
    re, im = C.c_double(), C.c_double()
    if isinstance(psi, LocalShards):
        check(A.sd_local_expectation(psi._arr(), psi.world, xs, zs, cs, len(terms), C.byref(re), C.byref(im)))
    else:
        check(A.sd_expectation(psi._s, xs, zs, cs, len(terms), C.byref(re), C.byref(im)))
    return (re.value, im.value) if with_residue else re.value


K_EXACT_EVOLVE_MAX_QUBITS = 12


def exact_evolve(h: "Hamiltonian", psi: StateVector, t: float) -> StateVector:
    """exp(-i H t) psi for n <= 12 (evolve.cpp:60-97, the reference's dense
    test oracle) as a new state; computed on the device."""
    if h.n_qubits != psi.n:
        raise ValueError("hamiltonian/state qubit counts differ")
    out = StateVector(psi.n, device=psi.device)
    check(A.sd_state_copy(out._s, psi._s))
    xs, zs, cs = _term_arrays(h.terms())
    check(A.sd_exact_evolve(out._s, xs, zs, cs, h.term_count(), t))
    return out


def comm_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; broadcast it with torch.distributed)."""
    buf = C.create_string_buffer(128)
    check(A.sd_comm_unique_id(buf))
    return buf.raw


class LocalShards:
    """`world` shards of one 2^n state driven by this process (devices may
    repeat: virtual shards on one GPU). Exchanges are device copies with the
    same routing as the NCCL path (sd_state_create_local_shards)."""

    def __init__(self, n_qubits: int, world: int, devices: Optional[Sequence[int]] = None):
        arr = (C.c_void_p * world)()
        devs = (C.c_int * world)(*(devices if devices is not None else [0] * world))
        check(A.sd_state_create_local_shards(n_qubits, world, devs, arr))
        self.shards = [StateVector(n_qubits, devs[r], r, world, _handle=arr[r]) for r in range(world)]
        self.n, self.world = n_qubits, world
        self.n_local = self.shards[0].n_local
        self.plans: List["TrotterPlan"] = []

    def upload(self, amps: np.ndarray) -> None:
        a = np.ascontiguousarray(amps, dtype=np.complex128).reshape(self.world, 1 << self.n_local)
        for r, s in enumerate(self.shards):
            s.upload(a[r])

    def set_basis(self, index: int) -> None:
        for s in self.shards:
            s.set_basis(index)

    def enable_p2p(self) -> None:
        """Fused exchanges: each remap's last pass stores straight into the
        receiving shard's buffer (sd_local_enable_p2p)."""
        arr = (C.c_void_p * self.world)(*[s._s.value for s in self.shards])
        check(A.sd_local_enable_p2p(arr, self.world))

    def plan(self, groups: Sequence[DiagonalGroup], order: int = 1, tile_qubits: int = 0) -> None:
        self.plans = [TrotterPlan(s, groups, order=order, tile_qubits=tile_qubits) for s in self.shards]

    def evolve(self, dt: float, n_steps: int) -> None:
        arr = (C.c_void_p * self.world)(*[p._p.value for p in self.plans])
        check(A.sd_evolve_local(arr, self.world, dt, n_steps))

    def _arr(self):
        return (C.c_void_p * self.world)(*[s._s.value for s in self.shards])

    def amplitudes(self) -> np.ndarray:
        check(A.sd_local_canonicalize(self._arr(), self.world))
        return np.concatenate([s.amplitudes() for s in self.shards])

    def norm(self) -> float:
        v = C.c_double()
        check(A.sd_local_norm(self._arr(), self.world, C.byref(v)))
        return v.value

    def apply_pauli_rotation(self, term: WeightedTerm, dt: float) -> None:
        check(A.sd_local_apply_pauli_rotation(self._arr(), self.world, term.pauli.x_mask, term.pauli.z_mask,
                                              term.coeff, dt))


def exchange_routes(n_qubits: int, n_local: int, rank: int, swaps) -> List[Tuple[int, int, int, int]]:
    """(peer, send_offset, recv_offset, count) of one remap for `rank`
    (sd_exchange_routes; host-only)."""
    flat = [int(v) for p in swaps for v in p]
    arr = (C.c_int32 * max(1, len(flat)))(*flat)
    cnt = C.c_size_t(0)
    check(A.sd_exchange_routes(n_qubits, n_local, rank, arr, len(swaps), None, 0, C.byref(cnt)))
    out = (A.Route * max(1, cnt.value))()
    check(A.sd_exchange_routes(n_qubits, n_local, rank, arr, len(swaps), out, cnt.value, C.byref(cnt)))
    return [(r.peer, r.send_offset, r.recv_offset, r.count) for r in out[:cnt.value]]


def jit_compile_preview(n_qubits: int, groups: Sequence[DiagonalGroup], order: int = 1, tile_qubits: int = 0,
                        world: int = 1) -> int:
    """Host-only: NVRTC-compile the specialised kernels of the first step's
    passes (sd_jit_compile_preview); returns the number of distinct programs."""
    opts = A.PlanOptions()
    check(A.sd_plan_options_default(C.byref(opts)))
    opts.order = order
    opts.tile_qubits = tile_qubits
    descs = (A.GroupDesc * max(1, len(groups)))()
    keep = []
    for i, g in enumerate(groups):
        d, k = g._desc()
        descs[i] = d
        keep.append(k)
    n = C.c_size_t(0)
    check(A.sd_jit_compile_preview(n_qubits, world, descs, len(groups), C.byref(opts), C.byref(n)))
    return n.value


def diag_document(h: "Hamiltonian") -> str:
    """The reference's `diag` JSON document (serialize.cpp:46-66) of
    greedy_partition + diagonalize_group: circuits, hex z-masks, signed
    coefficients (sd_groups_diag_json)."""
    g = C.c_void_p()
    check(A.sd_partition(h._h, C.byref(g)))
    try:
        n = C.c_size_t(0)
        check(A.sd_groups_diag_json(g, h.n_qubits, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(A.sd_groups_diag_json(g, h.n_qubits, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()
    finally:
        A.sd_groups_destroy(g)
