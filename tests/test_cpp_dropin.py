"""The reference's C++ API (include/simdiag/*.hpp) as a drop-in: a C++
program written against it (tests/cpp/test_dropin.cpp -- Hamiltonian::load,
greedy_partition, diagonalize_group, StateVector, evolve_grouped, save_raw)
compiles and links against libsimdiag_b200.so on CPU, and on the GPU its
evolved state matches the reference compiled from its own sources."""
import os
import subprocess

import numpy as np
import pytest

from paper_2206_11664_b200 import models as M

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2206_11664_b200", "lib")


def build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-L" + LIB, "-lsimdiag_b200",
                    "-Wl,-rpath," + LIB], check=True)
    return exe


def test_cpp_dropin_compiles_against_reference_api(tmp_path):
    assert os.path.exists(build(tmp_path))


def _gates_reference(ref, port, text, n):
    """The .gates sequence of test_dropin.cpp through the reference."""
    c, s_ = np.cos(0.3), np.sin(0.3)
    ry = np.array([[c, -s_], [s_, c]], np.complex128)
    ph = np.array([[1, 0], [0, np.exp(0.7j)]], np.complex128)
    u = np.zeros(16, np.complex128)
    u[0] = u[5] = u[14] = 1.0
    u[11] = np.exp(0.4j)
    a = np.zeros(1 << n, np.complex128)
    a[0] = 1.0
    for q in range(n):
        a = ref.generic_gate(a, n, ry if q % 2 else ph, q)
    for q in range(n):
        a = ref.generic_gate(a, n, ry, q)
    for q in range(0, n - 1, 2):
        a = ref.generic_gate(a, n, u, q, q + 1)
    a = ref.generic_gate(a, n, u, n - 1, 0)
    _, xs, zs, cs = port.load(text)
    for x, z, cf in zip(xs, zs, cs):
        a = ref.pauli_rotation(a, n, x, z, cf, 0.37)
    return a


def _dense_expm(port, text, n, psi0, t):
    from scipy.linalg import expm

    _, xs, zs, cs = port.load(text)
    dim = 1 << n
    H = np.zeros((dim, dim), np.complex128)
    b = np.arange(dim)
    for x, z, cf in zip(xs, zs, cs):
        base = cf * (1j ** (bin(x & z).count("1") & 3))
        par = np.array([bin(v & z).count("1") & 1 for v in range(dim)])
        H[b ^ x, b] += np.where(par == 1, -base, base)
    return expm(-1j * t * H) @ psi0


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,steps", [(4, 12, 60), (1, 10, 100)])
def test_cpp_dropin_evolution_matches_reference(cfg, n, steps, tmp_path, ref, port):
    exe = build(tmp_path)
    text = M.config_text(cfg, n=n)
    hpath = tmp_path / "h.txt"
    hpath.write_text(text)
    out = tmp_path / "psi.raw"
    dt = M.CONFIGS[cfg]["dt"]
    r = subprocess.run([exe, str(hpath), "neel", repr(dt), str(steps), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rd = lambda suffix: np.fromfile(str(out) + suffix, dtype=np.complex128)  # noqa: E731
    psi0 = np.zeros(1 << n, np.complex128)
    psi0[M.neel_index(n)] = 1
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, steps, 1)
    assert np.max(np.abs(rd("") - want)) < 1e-10
    # evolve_grouped in a step-and-measure loop (cached plan): same state
    assert np.max(np.abs(rd(".loop") - want)) < 1e-10
    # evolve_baseline, Hamiltonian order and group-major order
    assert np.max(np.abs(rd(".baseline") - ref.evolve_baseline(text, psi0, n, dt, steps))) < 1e-10
    assert np.max(np.abs(rd(".gbase") - ref.evolve_baseline_groups(h, psi0, n, dt, steps))) < 1e-10
    ref.free(h)
    # generic gates + pauli rotations
    assert np.max(np.abs(rd(".gates") - _gates_reference(ref, port, text, n))) < 1e-12
    # expectation on the evolved state
    e, im = [float(v) for v in open(str(out) + ".expect").read().split()]
    e_ref, im_ref = ref.expectation(text, want, n)
    assert abs(e - e_ref) < 1e-12 * max(1.0, abs(e_ref))
    assert abs(im) < 1e-12
    # exact_evolve against a dense matrix exponential
    assert np.max(np.abs(rd(".exact") - _dense_expm(port, text, n, psi0, dt * steps))) < 1e-10
