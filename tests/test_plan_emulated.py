"""Planner correctness without a GPU: the fused schedule (as exported by
sd_plan_preview) is emulated in numpy and compared with the oracle's
evolve_grouped (proj/src/evolve.cpp:47-58) -- this checks the list
scheduler's commutation-based reordering, CNOT-run splitting, the phase /
diagonal fusion and the exact power-of-two normalisation."""
import numpy as np
import pytest

from paper_2206_11664_b200 import models as M
from tests.plan_emulator import run_schedule


def initial(port, cfg, n):
    init = M.CONFIGS[cfg]["init"]
    if init[0] == "plus":
        return np.full(1 << n, 1 / np.sqrt(1 << n), np.complex128)
    if init[0] == "random":
        return port.random_state(n, init[1])
    a = np.zeros(1 << n, np.complex128)
    a[M.initial_index(cfg, n)] = 1
    return a


CASES = [(1, 8, 4), (1, 10, 6), (2, 9, 5), (3, 9, 5), (3, 10, 7), (4, 10, 5), (4, 11, 6), (5, 10, 6), (5, 11, 8)]


@pytest.mark.parametrize("cfg,n,k", CASES)
def test_schedule_matches_oracle(cfg, n, k, sd, port):
    text = M.config_text(cfg, n=n)
    _, og = port.partition_and_diagonalize(text)
    sg = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order = M.CONFIGS[cfg]["order"]
    info, sched = sd.plan_preview(n, sg, order=order, tile_qubits=k)
    passes = sched["steps"][0]["segments"][0]["plan"]["passes"]
    assert len(sched["steps"]) == 1 and len(sched["steps"][0]["segments"]) == 1
    assert info["n_passes_per_step"] == len(passes)
    assert all(len(p["lpos"]) == min(k, n) for p in passes)
    psi0 = initial(port, cfg, n)
    dt = M.CONFIGS[cfg]["dt"] * 7  # larger angles make ordering bugs visible
    want = port.evolve_grouped(psi0, n, og, dt, 2, order)
    got = run_schedule(psi0, n, sched, dt, steps=2)
    assert np.max(np.abs(got - want)) < 1e-11
    assert abs(np.linalg.norm(got) - 1) < 1e-13


def test_fused_pass_count_beats_reference_sweeps(sd):
    for cfg in (1, 2, 3, 4):
        text = M.config_text(cfg)
        g = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
        info, _ = sd.plan_preview(M.CONFIGS[cfg]["n"], g, order=M.CONFIGS[cfg]["order"], tile_qubits=12)
        assert info["n_passes_per_step"] * 8 < info["n_ref_sweeps_per_step"]


def test_cnot_resynthesis_cuts_passes(sd, monkeypatch):
    """Config 5 (Jordan-Wigner, CNOT-heavy groups): re-synthesising each CNOT
    network into rounds of tile-local targets needs fewer passes than running
    the synthesised CNOT list as given."""
    text = M.config_text(5)
    g = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    info, _ = sd.plan_preview(33, g, order=1, tile_qubits=12)
    monkeypatch.setenv("SDB_CX_RESYNTH", "0")
    info0, _ = sd.plan_preview(33, g, order=1, tile_qubits=12)
    assert info["n_passes_per_step"] < 0.9 * info0["n_passes_per_step"]
    assert info["n_passes_per_step"] * 8 < info["n_ref_sweeps_per_step"]


SHARDED = [(3, 10, 6, 4), (1, 10, 6, 2), (2, 9, 5, 4), (3, 10, 6, 2), (3, 10, 6, 8), (4, 11, 6, 2), (4, 11, 7, 4), (4, 12, 8, 8),
           (5, 10, 6, 4), (5, 11, 7, 2)]


@pytest.mark.parametrize("cfg,n,k,world", SHARDED)
def test_sharded_schedule_matches_oracle(cfg, n, k, world, sd, port):
    """The sharded planner (segments + qubit-remap exchanges over `world`
    ranks) emulated on the full state reproduces the oracle."""
    text = M.config_text(cfg, n=n)
    _, og = port.partition_and_diagonalize(text)
    sg = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order = M.CONFIGS[cfg]["order"]
    info, sched = sd.plan_preview(n, sg, order=order, tile_qubits=k, world=world)
    n_local = sched["n_local"]
    for st in sched["steps"]:
        for seg in st["segments"]:
            for p in seg["plan"]["passes"]:
                assert max(p["lpos"]) < n_local  # passes only touch local bits
    psi0 = initial(port, cfg, n)
    dt = M.CONFIGS[cfg]["dt"] * 7
    steps = 3
    want = port.evolve_grouped(psi0, n, og, dt, steps, order)
    got = run_schedule(psi0, n, sched, dt, steps=steps)
    assert np.max(np.abs(got - want)) < 1e-11
    assert abs(np.linalg.norm(got) - 1) < 1e-13
    if cfg == 4:
        # every qubit needs four Hadamard layers per step, so the global ones
        # must come local at least once per step
        assert info["n_exchanges_per_step"] >= 1


PLANNER_MODES = [
    # per-term diagonal ops (temporal blocking of Hadamard layers), diagonal
    # consolidation, Hadamard-depth cap, no HBM-pattern heuristic
    {"SDB_SPLIT_DIAG": "1", "SDB_MAX_HDEPTH": "0"},
    {"SDB_SPLIT_DIAG": "1", "SDB_MAX_HDEPTH": "2"},
    {"SDB_SPLIT_DIAG": "1", "SDB_CONSOLIDATE": "0"},
    {"SDB_DRAM_PATTERN": "0", "SDB_CX_RESYNTH": "0"},
    {"SDB_DEFER_FIXED_H": "1", "SDB_SPLIT_DIAG": "0"},
    {"SDB_DRAM_PATTERN": "2"},
]


@pytest.mark.parametrize("mode", range(len(PLANNER_MODES)))
@pytest.mark.parametrize("cfg,n,k,world", [(1, 10, 6, 1), (3, 10, 6, 2), (4, 11, 6, 2), (5, 10, 6, 1), (2, 9, 5, 1)])
def test_planner_modes_match_oracle(mode, cfg, n, k, world, sd, port, monkeypatch):
    """The planner variants selectable through the environment all produce
    schedules equivalent to the reference evolution."""
    for key, val in PLANNER_MODES[mode].items():
        monkeypatch.setenv(key, val)
    text = M.config_text(cfg, n=n)
    _, og = port.partition_and_diagonalize(text)
    sg = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order = M.CONFIGS[cfg]["order"]
    info, sched = sd.plan_preview(n, sg, order=order, tile_qubits=k, world=world)
    psi0 = initial(port, cfg, n)
    dt = M.CONFIGS[cfg]["dt"] * 7
    want = port.evolve_grouped(psi0, n, og, dt, 3, order)
    got = run_schedule(psi0, n, sched, dt, steps=3)
    assert np.max(np.abs(got - want)) < 1e-11
    assert abs(np.linalg.norm(got) - 1) < 1e-13
