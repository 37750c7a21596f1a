"""Run-time specialised tile-pass kernels (csrc/cuda/jit.cpp): the NVRTC
sources generated for a plan compile for sm_100a on CPU, and on the GPU the
specialised kernels (used for shards >= 22 qubits, i.e. by the benchmark)
reproduce the reference exactly like the interpreter kernel does."""
import os

import numpy as np
import pytest

from paper_2206_11664_b200 import models as M


def test_jit_sources_compile_for_sm100a(sd):
    for cfg, n in ((4, 16), (2, 12)):
        groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(M.config_text(cfg, n=n)))
        assert sd.simdiag.jit_compile_preview(n, groups, order=M.CONFIGS[cfg]["order"]) >= 1


@pytest.fixture
def force_jit():
    old = os.environ.get("SDB_JIT")
    os.environ["SDB_JIT"] = "1"
    yield
    if old is None:
        del os.environ["SDB_JIT"]
    else:
        os.environ["SDB_JIT"] = old


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,k", [(4, 16, 12), (2, 12, 12), (3, 13, 12), (5, 13, 10)])
def test_jit_evolution_matches_reference(cfg, n, k, sd, ref, port, force_jit):
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order, dt, steps = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"] * 5, 3
    init = M.CONFIGS[cfg]["init"]
    if init[0] == "plus":
        psi0 = np.full(1 << n, 1 / np.sqrt(1 << n), np.complex128)
    elif init[0] == "random":
        psi0 = port.random_state(n, init[1])
    else:
        psi0 = np.zeros(1 << n, np.complex128)
        psi0[M.initial_index(cfg, n)] = 1
    s = sd.StateVector(n)
    s.upload(psi0)
    sd.TrotterPlan(s, groups, order=order, tile_qubits=k).evolve(dt, steps)
    got = s.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, steps, order)
    ref.free(h)
    assert np.max(np.abs(got - want)) < 1e-10
    assert abs(np.linalg.norm(got) - 1) < 1e-12


@pytest.mark.gpu
def test_jit_sharded_local_shards(sd, ref, force_jit):
    cfg, n, world = 4, 14, 4
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    psi0 = np.zeros(1 << n, np.complex128)
    psi0[M.neel_index(n)] = 1
    sh = sd.LocalShards(n, world)
    sh.upload(psi0)
    sh.plan(groups, tile_qubits=10)
    sh.evolve(0.05, 3)
    got = sh.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, 0.05, 3, 1)
    ref.free(h)
    assert np.max(np.abs(got - want)) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,mode", [(4, 16, "two_ctas"), (3, 14, "two_ctas"),
                                        (4, 16, "ring"), (3, 14, "ring"), (2, 14, "ring"),
                                        (4, 16, "ring_register_stores")])
def test_jit_per_term_five_register_coordinates(cfg, n, mode, sd, ref, port, force_jit, monkeypatch):
    """Per-term diagonal schedule (the one the autotuner keeps for config 4):
    its specialised kernels run 32 amplitudes per thread (R = 5) through the
    ring pipeline (two warp groups, three TMA stages, TMA stores; the default),
    the ring with register stores, or two CTAs per SM -- against the
    reference, with few CTAs so each walks many tiles."""
    monkeypatch.setenv("SDB_SPLIT_DIAG", "1")
    monkeypatch.setenv("SDB_MAX_HDEPTH", "2")
    monkeypatch.setenv("SDB_MAX_CTAS", "5")
    monkeypatch.setenv("SDB_RING", "0" if mode == "two_ctas" else "1")
    monkeypatch.setenv("SDB_TMA_STORE", "0" if mode == "ring_register_stores" else "1")
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order, dt, steps = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"] * 5, 3
    init = M.CONFIGS[cfg]["init"]
    if init[0] == "plus":
        psi0 = np.full(1 << n, 1 / np.sqrt(1 << n), np.complex128)
    elif init[0] == "random":
        psi0 = port.random_state(n, init[1])
    else:
        psi0 = np.zeros(1 << n, np.complex128)
        psi0[M.initial_index(cfg, n)] = 1
    s = sd.StateVector(n)
    s.upload(psi0)
    plan = sd.TrotterPlan(s, groups, order=order, tile_qubits=12)
    plan.evolve(dt, steps)
    got = s.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, steps, order)
    ref.free(h)
    assert np.max(np.abs(got - want)) < 1e-10
    assert abs(np.linalg.norm(got) - 1) < 1e-12


@pytest.mark.parametrize("ring", ["0", "1"])
def test_jit_per_term_sources_compile_r5(sd, monkeypatch, ring):
    """Host-only: per-term plans lower to 5 register coordinates (32 amplitudes
    per thread), pass the lowering's own check, and their NVRTC programs --
    ring-pipeline variant included -- compile for sm_100a."""
    monkeypatch.setenv("SDB_SPLIT_DIAG", "1")
    monkeypatch.setenv("SDB_MAX_HDEPTH", "2")
    monkeypatch.setenv("SDB_RING", ring)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(M.config_text(4, n=16)))
    assert sd.simdiag.jit_compile_preview(16, groups, order=1) >= 1


@pytest.mark.gpu
@pytest.mark.parametrize("max_ctas", [None, "3"])
def test_jit_ring_edge_grids_and_shards(max_ctas, sd, ref, force_jit, monkeypatch):
    """Ring pipeline (R = 5 per-term plans) at grid extremes -- one tile per CTA
    (the second warp group idle) and three CTAs walking every tile -- and on
    four in-process shards, where the passes in front of a remap store into
    the exchange buffers (register stores inside the ring)."""
    monkeypatch.setenv("SDB_SPLIT_DIAG", "1")
    monkeypatch.setenv("SDB_MAX_HDEPTH", "2")
    if max_ctas:
        monkeypatch.setenv("SDB_MAX_CTAS", max_ctas)
    cfg, n = 4, 16
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    psi0 = np.zeros(1 << n, np.complex128)
    psi0[M.neel_index(n)] = 1
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, 0.05, 3, 1)
    ref.free(h)
    s = sd.StateVector(n)
    s.upload(psi0)
    sd.TrotterPlan(s, groups, order=1, tile_qubits=12).evolve(0.05, 3)
    assert np.max(np.abs(s.amplitudes() - want)) < 1e-10
    sh = sd.LocalShards(n, 4)
    sh.upload(psi0)
    sh.plan(groups, tile_qubits=12)
    sh.evolve(0.05, 3)
    assert np.max(np.abs(sh.amplitudes() - want)) < 1e-10


def test_jit_deep_per_term_split_points_compile(sd, monkeypatch):
    """Host-only: per-term plans with no cap on Hadamard levels (config 4 at
    n=30: 4 passes) carry POINT stages of up to 12 terms besides the table
    point; those are cut into <= 6-term sign-pattern points (lower.cpp), and
    the programs compile for sm_100a."""
    monkeypatch.setenv("SDB_SPLIT_DIAG", "1")
    monkeypatch.setenv("SDB_MAX_HDEPTH", "0")
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(M.config_text(4, n=30)))
    assert sd.simdiag.jit_compile_preview(30, groups, order=1) == 4


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,split_points", [(4, 22, "1"), (4, 22, "4"), (3, 22, "4")])
def test_jit_deep_per_term_matches_reference(cfg, n, split_points, sd, ref, port, force_jit, monkeypatch):
    """Per-term plans with no cap on Hadamard levels per pass, with the
    non-table POINT stages summed per amplitude (SDB_SPLIT_POINTS=1) or cut
    into sign-pattern points (4, the default), through the specialised kernels."""
    monkeypatch.setenv("SDB_SPLIT_DIAG", "1")
    monkeypatch.setenv("SDB_MAX_HDEPTH", "0")
    monkeypatch.setenv("SDB_SPLIT_POINTS", split_points)
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order, dt = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"] * 5
    psi0 = port.random_state(n, 11)
    s = sd.StateVector(n)
    s.upload(psi0)
    sd.TrotterPlan(s, groups, order=order).evolve(dt, 2)
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, 2, order)
    ref.free(h)
    got = s.amplitudes()
    assert np.max(np.abs(got - want)) < 1e-10
    assert abs(np.linalg.norm(got) - 1) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n,hdepth,fold", [(4, 16, "3", "0"), (4, 16, "3", "2"), (4, 16, "0", "2"), (3, 14, "2", "2"),
                                               (5, 14, "2", "1")])
def test_jit_cnot_maps_folded_into_the_stage(cfg, n, hdepth, fold, sd, ref, port, force_jit, monkeypatch):
    """A CNOT-map transpose right behind the TMA LOAD is read off the staged
    tile through the inverse map, one in front of a plain TMA STORE is written
    into the stage through the map (jit.cpp load_fold / store_fold): off,
    conflict-limited (default) and always, against the reference. Config 5
    (outer-controlled CNOT flips, R = 5 ring kernels) runs the default."""
    monkeypatch.setenv("SDB_SPLIT_DIAG", "1")
    monkeypatch.setenv("SDB_MAX_HDEPTH", hdepth)
    monkeypatch.setenv("SDB_MAX_CTAS", "5")
    monkeypatch.setenv("SDB_RING", "1")
    monkeypatch.setenv("SDB_LOAD_FOLD", fold)
    monkeypatch.setenv("SDB_STORE_FOLD", fold)
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order, dt, steps = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"] * 5, 3
    init = M.CONFIGS[cfg]["init"]
    if init[0] == "random":
        psi0 = port.random_state(n, init[1])
    else:
        psi0 = port.random_state(n, 7)  # a dense state: every slot of every tile is checked
    s = sd.StateVector(n)
    s.upload(psi0)
    plan = sd.TrotterPlan(s, groups, order=order, tile_qubits=12)
    plan.evolve(dt, steps)
    got = s.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, steps, order)
    ref.free(h)
    assert np.max(np.abs(got - want)) < 1e-10
    assert abs(np.linalg.norm(got) - 1) < 1e-12


@pytest.mark.parametrize("cfg,n,hdepth", [(4, 30, "3"), (4, 30, "0"), (5, 16, "0")])
def test_jit_folded_sources_compile(sd, monkeypatch, cfg, n, hdepth):
    """Host-only: programs with the LOAD / STORE folds forced compile for sm_100a."""
    monkeypatch.setenv("SDB_SPLIT_DIAG", "1")
    monkeypatch.setenv("SDB_MAX_HDEPTH", hdepth)
    monkeypatch.setenv("SDB_RING", "1")
    monkeypatch.setenv("SDB_LOAD_FOLD", "2")
    monkeypatch.setenv("SDB_STORE_FOLD", "2")
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(M.config_text(cfg, n=n)))
    assert sd.simdiag.jit_compile_preview(n, groups, order=1) >= 1
