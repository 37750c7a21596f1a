"""CPU oracle loaders -- TEST INFRASTRUCTURE ONLY.

Two checkers, both CPU, neither ever used by the product:
  port : oracle/build/liboracle.so, the plain-C restatement
         (oracle/simdiag_oracle.c, cites the reference per function);
  ref  : oracle/_ref/libsimdiag_ref.so, the reference's own sources
         (/root/reference/proj/src/*.cpp) compiled by oracle/Makefile with
         the shim oracle/ref_harness.cpp.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import List, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "build", "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libsimdiag_ref.so")

u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
dblp = C.POINTER(C.c_double)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@dataclasses.dataclass
class Group:
    """A synthesised group in plain arrays (DiagonalGroup + source terms)."""
    h_pre: List[int]
    cnots: List[Tuple[int, int]]
    czs: List[Tuple[int, int]]
    s_layer: List[int]
    h_post: List[int]
    src_x: List[int]
    src_z: List[int]
    src_c: List[float]
    z_masks: List[int]
    coeffs: List[float]


def parse_text(text: str):
    """Hamiltonian::load line format -> (n, x, z, c) before merging
    (proj/src/hamiltonian.cpp:71-118, without its error reporting)."""
    n = None
    xs, zs, cs = [], [], []
    for line in text.splitlines():
        line = line.split("#", 1)[0].split()
        if not line:
            continue
        c, p = float(line[0]), line[1]
        if n is None:
            n = len(p)
        x = z = 0
        for q, ch in enumerate(p):
            if ch in "XY":
                x |= 1 << q
            if ch in "ZY":
                z |= 1 << q
        xs.append(x)
        zs.append(z)
        cs.append(c)
    return n, xs, zs, cs


class Port:
    def __init__(self, path: str = PORT_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.or_from_terms.argtypes = [u64p, u64p, dblp, C.c_int64, C.c_double, u64p, u64p, dblp]
        L.or_from_terms.restype = C.c_int64
        L.or_greedy_partition.argtypes = [u64p, u64p, C.c_int64, i64p]
        L.or_greedy_partition.restype = C.c_int64
        L.or_independent_subset.argtypes = [u64p, u64p, C.c_int64, C.c_int, i64p]
        L.or_independent_subset.restype = C.c_int64
        L.or_diagonalize.argtypes = [C.c_int, u64p, u64p, dblp, C.c_int64, i32p, i32p, i32p, i32p, i32p, i64p,
                                     u64p, dblp]
        L.or_diagonalize.restype = C.c_int
        for name in ("sv_hadamard",):
            getattr(L, name).argtypes = [dblp, C.c_int, C.c_int]
        L.sv_batched_cnot.argtypes = [dblp, C.c_int, C.c_int, C.c_uint64]
        L.sv_phase_layer.argtypes = [dblp, C.c_int, C.c_uint64, i32p, C.c_int64, C.c_int]
        L.sv_diagonal_exp.argtypes = [dblp, C.c_int, u64p, dblp, C.c_int64, C.c_double]
        L.or_evolve_grouped.argtypes = [dblp, C.c_int, C.c_void_p, C.c_int64, C.c_double, C.c_int64, C.c_int]
        L.or_random_state.argtypes = [dblp, C.c_int, C.c_uint64]
        L.or_norm.argtypes = [dblp, C.c_int]
        L.or_norm.restype = C.c_double
        L.or_threads.restype = C.c_int
        L.or_group_size.restype = C.c_size_t

    def threads(self) -> int:
        return self.lib.or_threads()

    def from_terms(self, xs, zs, cs, tol=1e-12):
        m = len(cs)
        x = np.array(xs, np.uint64)
        z = np.array(zs, np.uint64)
        c = np.array(cs, np.float64)
        ox, oz, oc = np.zeros(max(m, 1), np.uint64), np.zeros(max(m, 1), np.uint64), np.zeros(max(m, 1))
        k = self.lib.or_from_terms(_p(x, u64p), _p(z, u64p), _p(c, dblp), m, tol, _p(ox, u64p), _p(oz, u64p),
                                   _p(oc, dblp))
        return [int(v) for v in ox[:k]], [int(v) for v in oz[:k]], [float(v) for v in oc[:k]]

    def load(self, text: str):
        n, xs, zs, cs = parse_text(text)
        x, z, c = self.from_terms(xs, zs, cs)
        return n, x, z, c

    def greedy_partition(self, xs, zs) -> List[int]:
        m = len(xs)
        x = np.array(xs, np.uint64)
        z = np.array(zs, np.uint64)
        g = np.zeros(max(m, 1), np.int64)
        self.lib.or_greedy_partition(_p(x, u64p), _p(z, u64p), m, _p(g, i64p))
        return [int(v) for v in g[:m]]

    def independent_subset(self, n, xs, zs) -> List[int]:
        m = len(xs)
        x = np.array(xs, np.uint64)
        z = np.array(zs, np.uint64)
        idx = np.zeros(max(m, 1), np.int64)
        k = self.lib.or_independent_subset(_p(x, u64p), _p(z, u64p), m, n, _p(idx, i64p))
        return [int(v) for v in idx[:k]]

    def diagonalize(self, n, xs, zs, cs) -> Group:
        m = len(xs)
        x = np.array(xs, np.uint64)
        z = np.array(zs, np.uint64)
        c = np.array(cs, np.float64)
        cap = 2 * n * n + 4
        bufs = [np.zeros(cap, np.int32) for _ in range(5)]
        counts = np.zeros(5, np.int64)
        zo = np.zeros(max(m, 1), np.uint64)
        co = np.zeros(max(m, 1))
        rc = self.lib.or_diagonalize(n, _p(x, u64p), _p(z, u64p), _p(c, dblp), m, *[_p(b, i32p) for b in bufs],
                                     _p(counts, i64p), _p(zo, u64p), _p(co, dblp))
        if rc == 1:
            raise ValueError("oracle: invalid group")
        if rc == 2:
            raise RuntimeError("oracle: group not simultaneously diagonalized")
        h_pre, cx, cz, s, hp = bufs
        nh, ncx, ncz, ns, nhp = [int(v) for v in counts]
        return Group(
            [int(v) for v in h_pre[:nh]], [(int(cx[2 * i]), int(cx[2 * i + 1])) for i in range(ncx)],
            [(int(cz[2 * i]), int(cz[2 * i + 1])) for i in range(ncz)], [int(v) for v in s[:ns]],
            [int(v) for v in hp[:nhp]], list(xs), list(zs), list(cs),
            [int(v) for v in zo[:m]], [float(v) for v in co[:m]])

    def partition_and_diagonalize(self, text: str) -> Tuple[int, List[Group]]:
        n, x, z, c = self.load(text)
        gid = self.greedy_partition(x, z)
        groups = []
        for g in range(max(gid) + 1 if gid else 0):
            ks = [k for k, v in enumerate(gid) if v == g]
            groups.append(self.diagonalize(n, [x[k] for k in ks], [z[k] for k in ks], [c[k] for k in ks]))
        return n, groups

    def _pack(self, groups: Sequence[Group]):
        """Build the or_group array (see simdiag_oracle.c)."""
        class OrGroup(C.Structure):
            _fields_ = [("counts", C.c_int64 * 5), ("h_pre", i32p), ("cnots", i32p), ("czs", i32p),
                        ("s_layer", i32p), ("h_post", i32p), ("m", C.c_int64), ("zm", u64p), ("cf", dblp)]
        assert C.sizeof(OrGroup) == self.lib.or_group_size()
        arr = (OrGroup * max(1, len(groups)))()
        keep = []
        for i, g in enumerate(groups):
            parts = [np.array(g.h_pre or [0], np.int32), np.array([q for p in g.cnots for q in p] or [0], np.int32),
                     np.array([q for p in g.czs for q in p] or [0], np.int32), np.array(g.s_layer or [0], np.int32),
                     np.array(g.h_post or [0], np.int32), np.array(g.z_masks or [0], np.uint64),
                     np.array(g.coeffs or [0.0], np.float64)]
            keep.append(parts)
            arr[i].counts[:] = [len(g.h_pre), len(g.cnots), len(g.czs), len(g.s_layer), len(g.h_post)]
            arr[i].h_pre, arr[i].cnots, arr[i].czs, arr[i].s_layer, arr[i].h_post = [_p(a, i32p) for a in parts[:5]]
            arr[i].m = len(g.z_masks)
            arr[i].zm = _p(parts[5], u64p)
            arr[i].cf = _p(parts[6], dblp)
        return arr, keep

    def evolve_grouped(self, psi: np.ndarray, n: int, groups: Sequence[Group], dt: float, steps: int,
                       order: int = 1) -> np.ndarray:
        a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        arr, keep = self._pack(groups)
        self.lib.or_evolve_grouped(a.ctypes.data_as(dblp), n, C.cast(arr, C.c_void_p), len(groups), dt, steps,
                                   order)
        return a

    def random_state(self, n: int, seed: int) -> np.ndarray:
        a = np.zeros(1 << n, np.complex128)
        self.lib.or_random_state(a.ctypes.data_as(dblp), n, seed)
        return a

    def hadamard(self, psi, n, t):
        a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        self.lib.sv_hadamard(a.ctypes.data_as(dblp), n, t)
        return a

    def batched_cnot(self, psi, n, c, targets):
        a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        self.lib.sv_batched_cnot(a.ctypes.data_as(dblp), n, c, targets)
        return a

    def phase_layer(self, psi, n, s_mask, pairs, dagger):
        a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        pr = np.array([q for p in pairs for q in p] or [0], np.int32)
        self.lib.sv_phase_layer(a.ctypes.data_as(dblp), n, s_mask, _p(pr, i32p), len(pairs), 1 if dagger else 0)
        return a

    def diagonal_exp(self, psi, n, masks, coeffs, dt):
        a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        zm = np.array(masks or [0], np.uint64)
        cf = np.array(coeffs or [0.0], np.float64)
        self.lib.sv_diagonal_exp(a.ctypes.data_as(dblp), n, _p(zm, u64p), _p(cf, dblp), len(masks), dt)
        return a


class Ref:
    """The reference compiled from its own sources (oracle/_ref)."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_partition_text.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_diagonalize_terms.argtypes = [C.c_int, u64p, u64p, dblp, C.c_size_t, C.POINTER(C.c_void_p)]
        L.ref_load_save.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_groups_free.argtypes = [C.c_void_p]
        L.ref_groups_count.argtypes = [C.c_void_p]
        L.ref_groups_nqubits.argtypes = [C.c_void_p]
        L.ref_group_sizes.argtypes = [C.c_void_p, C.c_int, i64p]
        L.ref_group_data.argtypes = [C.c_void_p, C.c_int, i32p, i32p, i32p, i32p, i32p, u64p, u64p, dblp, u64p, dblp]
        L.ref_evolve_grouped.argtypes = [C.c_void_p, dblp, C.c_int, C.c_double, C.c_int, C.c_int, u64p]
        L.ref_random_state.argtypes = [C.c_int, C.c_uint64, dblp]
        L.ref_plus_state.argtypes = [C.c_int, dblp]
        L.ref_kernel.argtypes = [C.c_int, dblp, C.c_int, C.c_int, C.c_uint64, i32p, C.c_size_t, u64p, dblp,
                                 C.c_size_t, C.c_double]
        L.ref_pauli_rotation.argtypes = [dblp, C.c_int, C.c_uint64, C.c_uint64, C.c_double, C.c_double]
        L.ref_evolve_baseline_text.argtypes = [C.c_char_p, C.c_size_t, dblp, C.c_int, C.c_double, C.c_int]
        L.ref_expectation_text.argtypes = [C.c_char_p, C.c_size_t, dblp, C.c_int, dblp, dblp]
        L.ref_diag_json.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
        L.ref_norm.argtypes = [dblp, C.c_int]
        L.ref_norm.restype = C.c_double

        L.ref_gen_save_text.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t),
                                        u64p]
        L.ref_partition_timed.argtypes = [C.c_char_p, C.c_size_t, dblp, C.POINTER(C.c_size_t)]
        L.ref_generic_gate.argtypes = [dblp, C.c_int, dblp, C.c_int, C.c_int]
        L.ref_evolve_baseline_groups.argtypes = [C.c_void_p, dblp, C.c_int, C.c_double, C.c_int]
        L.ref_sv_create.argtypes = [C.c_int]
        L.ref_sv_create.restype = C.c_void_p
        L.ref_sv_free.argtypes = [C.c_void_p]
        L.ref_sv_set_basis.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_sv_write.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, dblp]
        L.ref_sv_read.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, dblp]
        L.ref_sv_evolve.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_int]
        L.ref_sv_norm.argtypes = [C.c_void_p]
        L.ref_sv_norm.restype = C.c_double
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_get_threads.restype = C.c_int

    def _err(self, rc):
        if rc == 0:
            return
        msg = self.lib.ref_last_error().decode()
        raise {1: ValueError, 2: IndexError}.get(rc, RuntimeError)(msg)

    def _groups(self, h) -> List[Group]:
        out = []
        for g in range(self.lib.ref_groups_count(h)):
            sz = np.zeros(6, np.int64)
            self.lib.ref_group_sizes(h, g, _p(sz, i64p))
            nh, ncx, ncz, ns, nhp, m = [int(v) for v in sz]
            b = [np.zeros(max(1, k), np.int32) for k in (nh, 2 * ncx, 2 * ncz, ns, nhp)]
            sx, sz_, zm = (np.zeros(max(1, m), np.uint64) for _ in range(3))
            sc, cf = np.zeros(max(1, m)), np.zeros(max(1, m))
            self.lib.ref_group_data(h, g, *[_p(a, i32p) for a in b], _p(sx, u64p), _p(sz_, u64p), _p(sc, dblp),
                                    _p(zm, u64p), _p(cf, dblp))
            out.append(Group([int(v) for v in b[0][:nh]],
                             [(int(b[1][2 * i]), int(b[1][2 * i + 1])) for i in range(ncx)],
                             [(int(b[2][2 * i]), int(b[2][2 * i + 1])) for i in range(ncz)],
                             [int(v) for v in b[3][:ns]], [int(v) for v in b[4][:nhp]],
                             [int(v) for v in sx[:m]], [int(v) for v in sz_[:m]], [float(v) for v in sc[:m]],
                             [int(v) for v in zm[:m]], [float(v) for v in cf[:m]]))
        return out

    def partition_text(self, text: str, synthesize: bool = True):
        """Returns (handle, n, groups); free the handle with free()."""
        h = C.c_void_p()
        b = text.encode()
        self._err(self.lib.ref_partition_text(b, len(b), 1 if synthesize else 0, C.byref(h)))
        return h, self.lib.ref_groups_nqubits(h), self._groups(h)

    def free(self, h):
        self.lib.ref_groups_free(h)

    def load_save(self, text: str) -> str:
        b = text.encode()
        n = C.c_size_t(0)
        self._err(self.lib.ref_load_save(b, len(b), None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self._err(self.lib.ref_load_save(b, len(b), buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def diagonalize(self, n, xs, zs, cs) -> Group:
        x, z, c = np.array(xs, np.uint64), np.array(zs, np.uint64), np.array(cs, np.float64)
        h = C.c_void_p()
        self._err(self.lib.ref_diagonalize_terms(n, _p(x, u64p), _p(z, u64p), _p(c, dblp), len(cs), C.byref(h)))
        try:
            return self._groups(h)[0]
        finally:
            self.free(h)

    def evolve_grouped(self, h, psi: np.ndarray, n: int, dt: float, steps: int, order: int = 1):
        a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        st = np.zeros(3, np.uint64)
        self._err(self.lib.ref_evolve_grouped(h, a.ctypes.data_as(dblp), n, dt, steps, order, _p(st, u64p)))
        return a, {"amp_reads": int(st[0]), "amp_writes": int(st[1]), "kernel_calls": int(st[2])}

    def random_state(self, n: int, seed: int) -> np.ndarray:
        a = np.zeros(1 << n, np.complex128)
        self._err(self.lib.ref_random_state(n, seed, a.ctypes.data_as(dblp)))
        return a

    def kernel(self, which: int, psi, n, a=0, mask=0, pairs=(), masks=(), coeffs=(), dt=0.0):
        st = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        pr = np.array([q for p in pairs for q in p] or [0], np.int32)
        zm = np.array(list(masks) or [0], np.uint64)
        cf = np.array(list(coeffs) or [0.0], np.float64)
        self._err(self.lib.ref_kernel(which, st.ctypes.data_as(dblp), n, a, mask, _p(pr, i32p), len(pairs),
                                      _p(zm, u64p), _p(cf, dblp), len(masks), dt))
        return st

    def norm(self, psi, n) -> float:
        a = np.ascontiguousarray(psi, dtype=np.complex128)
        return self.lib.ref_norm(a.ctypes.data_as(dblp), n)

    def diag_json(self, h) -> str:
        """diag_document(...).dump() (serialize.cpp:46-66) of a partition_text handle."""
        n = C.c_size_t(0)
        self._err(self.lib.ref_diag_json(h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self._err(self.lib.ref_diag_json(h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def pauli_rotation(self, psi, n, x, z, coeff, dt):
        """StateVector::apply_pauli_rotation (statevector.cpp:288-337)."""
        a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        self._err(self.lib.ref_pauli_rotation(a.ctypes.data_as(dblp), n, x, z, coeff, dt))
        return a

    def gen_text(self, model: str, n: int, seed: int):
        """gen_tfim / gen_syk (models.cpp:17-92) saved as text, + SYK counts."""
        which = {"tfim": 0, "syk": 1}[model]
        ln = C.c_size_t(0)
        info = np.zeros(2, np.uint64)
        self._err(self.lib.ref_gen_save_text(which, n, seed, None, 0, C.byref(ln), _p(info, u64p)))
        buf = C.create_string_buffer(ln.value + 1)
        self._err(self.lib.ref_gen_save_text(which, n, seed, buf, ln.value + 1, C.byref(ln), _p(info, u64p)))
        return buf.value.decode(), (int(info[0]), int(info[1]))

    def partition_timed(self, text: str):
        """(seconds, n_groups) of greedy_partition alone on a loaded Hamiltonian."""
        b = text.encode()
        secs, ng = C.c_double(0), C.c_size_t(0)
        self._err(self.lib.ref_partition_timed(b, len(b), C.byref(secs), C.byref(ng)))
        return secs.value, ng.value

    def generic_gate(self, psi, n, u, q1, q2=-1):
        """apply_single_qubit (q2 < 0) / apply_two_qubit (statevector.cpp:101-154)."""
        a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        m = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(-1))
        self._err(self.lib.ref_generic_gate(a.ctypes.data_as(dblp), n, m.ctypes.data_as(dblp), q1, q2))
        return a

    def evolve_baseline_groups(self, h, psi, n, dt, steps):
        """evolve_baseline(span<const CommutingGroup>) (evolve.cpp:34-45), restated loop."""
        a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        self._err(self.lib.ref_evolve_baseline_groups(h, a.ctypes.data_as(dblp), n, dt, steps))
        return a

    def evolve_baseline(self, text: str, psi, n, dt, steps):
        """evolve_baseline(Hamiltonian, ...) (evolve.cpp:21-32), restated loop."""
        a = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        b = text.encode()
        self._err(self.lib.ref_evolve_baseline_text(b, len(b), a.ctypes.data_as(dblp), n, dt, steps))
        return a

    def expectation(self, text: str, psi, n):
        """expectation (evolve.cpp:99-135), restated loop: (re, |imag residue|)."""
        a = np.ascontiguousarray(psi, dtype=np.complex128)
        b = text.encode()
        re, im = C.c_double(), C.c_double()
        self._err(self.lib.ref_expectation_text(b, len(b), a.ctypes.data_as(dblp), n, C.byref(re), C.byref(im)))
        return re.value, im.value


class RefState:
    """A persistent reference StateVector (oracle/_ref): evolve_grouped's loop
    runs on it in place, so timings exclude host copies."""

    def __init__(self, ref: Ref, n: int):
        self.ref, self.n = ref, n
        self.h = ref.lib.ref_sv_create(n)
        if not self.h:
            ref._err(3)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_sv_free(self.h)
            self.h = None

    def set_basis(self, index: int) -> None:
        self.ref._err(self.ref.lib.ref_sv_set_basis(self.h, index))

    def write(self, first: int, a: np.ndarray) -> None:
        a = np.ascontiguousarray(a, dtype=np.complex128)
        self.ref._err(self.ref.lib.ref_sv_write(self.h, first, a.size, a.ctypes.data_as(dblp)))

    def read(self, first: int, count: int) -> np.ndarray:
        out = np.empty(count, np.complex128)
        self.ref._err(self.ref.lib.ref_sv_read(self.h, first, count, out.ctypes.data_as(dblp)))
        return out

    def evolve(self, groups_handle, dt: float, steps: int, order: int = 1) -> None:
        self.ref._err(self.ref.lib.ref_sv_evolve(self.h, groups_handle, dt, steps, order))

    def norm(self) -> float:
        return self.ref.lib.ref_sv_norm(self.h)


def port() -> Port:
    return Port()


def ref() -> Ref:
    return Ref()
