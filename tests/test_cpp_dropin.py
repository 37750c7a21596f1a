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


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,steps", [(4, 12, 60), (1, 10, 100)])
def test_cpp_dropin_evolution_matches_reference(cfg, n, steps, tmp_path, ref):
    exe = build(tmp_path)
    text = M.config_text(cfg, n=n)
    hpath = tmp_path / "h.txt"
    hpath.write_text(text)
    out = tmp_path / "psi.raw"
    dt = M.CONFIGS[cfg]["dt"]
    r = subprocess.run([exe, str(hpath), "neel", repr(dt), str(steps), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = np.fromfile(out, dtype=np.complex128)
    psi0 = np.zeros(1 << n, np.complex128)
    psi0[M.neel_index(n)] = 1
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, steps, 1)
    ref.free(h)
    assert np.max(np.abs(got - want)) < 1e-10
