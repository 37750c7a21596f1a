"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU
oracle -- the reference compiled from its sources (ref) and the C
restatement (port). Tolerances from the north star: max per-amplitude
|dpsi| <= 1e-10 and |1-||psi||| <= 1e-12 after all steps."""
import numpy as np
import pytest

from paper_2206_11664_b200 import models as M

pytestmark = pytest.mark.gpu

TOL_AMP = 1e-10
TOL_NORM = 1e-12


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return a / np.linalg.norm(a)


def initial(port, cfg, n):
    init = M.CONFIGS[cfg]["init"]
    if init[0] == "plus":
        return np.full(1 << n, 1 / np.sqrt(1 << n), np.complex128)
    if init[0] == "random":
        return port.random_state(n, init[1])
    a = np.zeros(1 << n, np.complex128)
    a[M.initial_index(cfg, n)] = 1
    return a


# ------------------------------------------------------ single kernels

def test_single_sweep_kernels_match_reference(sd, ref):
    n = 11
    for seed in range(4):
        psi0 = rand_state(n, seed)
        s = sd.StateVector(n)
        s.upload(psi0)
        rng = np.random.default_rng(100 + seed)
        t = int(rng.integers(n))
        s.apply_hadamard(t)
        want = ref.kernel(0, psi0, n, a=t)
        assert np.max(np.abs(s.amplitudes() - want)) < 1e-15
        c = int(rng.integers(n))
        T = 0
        for q in rng.choice([q for q in range(n) if q != c], size=3, replace=False):
            T |= 1 << int(q)
        s.apply_batched_cnot(c, T)
        want = ref.kernel(1, want, n, a=c, mask=T)
        assert np.array_equal(s.amplitudes(), want)
        pairs = [(0, 3), (2, 5), (4, 9)]
        smask = 0b10010011
        for dag in (False, True):
            s.apply_phase_layer(smask, pairs, dag)
            want = ref.kernel(2, want, n, a=int(dag), mask=smask, pairs=pairs)
            assert np.array_equal(s.amplitudes(), want)
        masks = [int(x) for x in rng.integers(0, 1 << n, size=37)]
        coeffs = [float(x) for x in rng.normal(size=37)]
        s.apply_diagonal_exp(masks, coeffs, 0.013)
        want = ref.kernel(3, want, n, masks=masks, coeffs=coeffs, dt=0.013)
        assert np.max(np.abs(s.amplitudes() - want)) < 1e-13
        st = s.stats()
        assert st["kernel_calls"] == 5  # H, CNOT batch, 2 phase layers, diagonal
        assert st["amp_reads"] == (1 << n) * 4 + (1 << n) // 2


def test_kernel_argument_errors_match_reference(sd):
    s = sd.StateVector(6)
    with pytest.raises(IndexError):
        s.apply_hadamard(6)
    with pytest.raises(ValueError):
        s.apply_batched_cnot(1, 0)
    with pytest.raises(ValueError):
        s.apply_batched_cnot(1, 0b10)
    with pytest.raises(ValueError):
        s.apply_phase_layer(1 << 7, [])
    with pytest.raises(ValueError):
        s.apply_phase_layer(0, [(2, 2)])
    with pytest.raises(ValueError):
        s.apply_diagonal_exp([1 << 9], [1.0], 0.1)
    with pytest.raises(ValueError):
        s.apply_diagonal_exp([1], [1.0], float("nan"))


def test_random_state_matches_reference(sd, ref):
    for n, seed in ((10, 2), (14, 7)):
        got = sd.StateVector.random_state(n, seed).amplitudes()
        want = ref.random_state(n, seed)
        assert np.max(np.abs(got - want)) < 1e-14


# ----------------------------------------------------- fused evolution

@pytest.mark.parametrize("cfg,n,k", [(1, 12, 8), (2, 12, 7), (3, 12, 9), (4, 13, 8), (5, 12, 10),
                                     (1, 14, 12), (3, 14, 12), (4, 15, 13), (5, 14, 11)])
def test_fused_evolve_matches_reference(cfg, n, k, sd, ref, port):
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order, dt = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"] * 5
    psi0 = initial(port, cfg, n)
    s = sd.StateVector(n)
    s.upload(psi0)
    plan = sd.TrotterPlan(s, groups, order=order, tile_qubits=k)
    plan.evolve(dt, 4)
    got = s.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, 4, order)
    ref.free(h)
    assert np.max(np.abs(got - want)) < TOL_AMP
    assert abs(np.linalg.norm(got) - 1) < TOL_NORM
    st = s.stats()
    assert st["kernel_calls"] == 4 * plan.info()["n_passes_per_step"]


@pytest.mark.parametrize("env", [{"SDB_SPLIT_DIAG": "1"}, {"SDB_SPLIT_DIAG": "1", "SDB_MAX_HDEPTH": "2"},
                                 {"SDB_DRAM_PATTERN": "0", "SDB_CX_RESYNTH": "0"}])
@pytest.mark.parametrize("jit", ["0", "1"])
@pytest.mark.parametrize("cfg,n,k", [(4, 14, 12), (3, 13, 10), (5, 13, 12)])
def test_planner_modes_on_device(cfg, n, k, jit, env, sd, ref, port, monkeypatch):
    """Planner variants (per-term diagonals, Hadamard-depth cap, no HBM-pattern
    heuristic / CNOT resynthesis) through both the interpreter and the
    NVRTC-specialised kernels (lane swaps, several POINT stages per pass)."""
    if cfg == 5 and jit == "1":
        # ~800 distinct programs per planner mode (minutes of NVRTC on a fresh box);
        # config 5's specialised kernels are covered by test_jit and test_many_tiles_per_cta
        pytest.skip("config 5 runs its planner modes through the interpreter kernel")
    monkeypatch.setenv("SDB_JIT", jit)
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order, dt = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"] * 5
    psi0 = initial(port, cfg, n)
    s = sd.StateVector(n)
    s.upload(psi0)
    plan = sd.TrotterPlan(s, groups, order=order, tile_qubits=k)
    plan.evolve(dt, 3)
    got = s.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, 3, order)
    ref.free(h)
    assert np.max(np.abs(got - want)) < TOL_AMP
    assert abs(np.linalg.norm(got) - 1) < TOL_NORM


@pytest.mark.parametrize("split", ["0", "1"])
@pytest.mark.parametrize("czcx", ["0", "1"])
@pytest.mark.parametrize("cfg,n,k", [(4, 16, 12), (1, 14, 12), (3, 13, 10)])
def test_cz_to_cnot_conversion_on_device(cfg, n, k, czcx, split, sd, ref, port, monkeypatch):
    """Groups whose h_pre qubits see only CZs before h_post (config 4's
    Bell-pair groups, config 1) with the Hadamard pairs dropped and the CZs
    run as CNOTs onto those qubits (SDB_CZ_CX=1) and without (0), through the
    NVRTC-specialised kernels, both diagonal-op families."""
    monkeypatch.setenv("SDB_JIT", "1")
    monkeypatch.setenv("SDB_CZ_CX", czcx)
    monkeypatch.setenv("SDB_SPLIT_DIAG", split)
    if split == "1":
        monkeypatch.setenv("SDB_MAX_HDEPTH", "2")
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order, dt = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"] * 5
    psi0 = rand_state(n, 5)
    s = sd.StateVector(n)
    s.upload(psi0)
    plan = sd.TrotterPlan(s, groups, order=order, tile_qubits=k)
    plan.evolve(dt, 3)
    got = s.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, 3, order)
    ref.free(h)
    assert np.max(np.abs(got - want)) < TOL_AMP
    assert abs(np.linalg.norm(got) - 1) < TOL_NORM


@pytest.mark.parametrize("jit", ["0", "1"])
@pytest.mark.parametrize("cfg,n", [(3, 16), (5, 16), (4, 17)])
def test_many_tiles_per_cta(cfg, n, jit, sd, ref, port, monkeypatch):
    """Few CTAs walking many tiles: warps of a CTA drift apart in programs
    without a block barrier (lane swaps, CNOT-only passes), which in-place
    stores through a CNOT map and table rebuilds must tolerate."""
    monkeypatch.setenv("SDB_JIT", jit)
    monkeypatch.setenv("SDB_MAX_CTAS", "2")
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order, dt = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"] * 5
    psi0 = rand_state(n, 3)
    s = sd.StateVector(n)
    s.upload(psi0)
    sd.TrotterPlan(s, groups, order=order, use_graph=False).evolve(dt, 2)
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, 2, order)
    ref.free(h)
    assert np.max(np.abs(s.amplitudes() - want)) < TOL_AMP


def test_unfused_reference_schedule_matches(sd, ref, port):
    n, cfg = 11, 3
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    psi0 = initial(port, cfg, n)
    s = sd.StateVector(n)
    s.upload(psi0)
    plan = sd.TrotterPlan(s, groups, order=1, fuse=False)
    plan.evolve(0.03, 2)
    h, _, _ = ref.partition_text(text)
    want, stats = ref.evolve_grouped(h, psi0, n, 0.03, 2, 1)
    ref.free(h)
    assert np.max(np.abs(s.amplitudes() - want)) < 1e-12
    assert s.stats()["amp_reads"] == stats["amp_reads"]  # identical KernelStats traffic


def test_config1_full_run_matches_reference(sd, ref):
    """Config 1 exactly as BASELINE states it: n=16, Neel, dt=0.01, 100 steps."""
    cfg = 1
    n = 16
    text = M.config_text(cfg)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    s = sd.StateVector(n)
    s.set_basis(M.neel_index(n))
    sd.evolve_grouped(groups, s, sd.EvolutionPlan(total_time=1.0, n_steps=100))
    got = s.amplitudes()
    psi0 = np.zeros(1 << n, np.complex128)
    psi0[M.neel_index(n)] = 1
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, 0.01, 100, 1)
    ref.free(h)
    assert np.max(np.abs(got - want)) < TOL_AMP
    assert abs(np.linalg.norm(got) - 1) < TOL_NORM


def test_tile_width_invariance(sd, port):
    """Every tile width produces the same state (different pass schedules)."""
    n, cfg = 13, 5
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    psi0 = initial(port, cfg, n)
    outs = []
    for k in (5, 7, 9, 11, 13):
        s = sd.StateVector(n)
        s.upload(psi0)
        sd.TrotterPlan(s, groups, tile_qubits=k).evolve(0.02, 3)
        outs.append(s.amplitudes())
    for o in outs[1:]:
        assert np.max(np.abs(o - outs[0])) < 1e-12


def test_zero_steps_and_empty_plan_are_noops(sd):
    n = 8
    s = sd.StateVector(n)
    s.set_basis(5)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(M.config_text(4, n=n)))
    sd.evolve_grouped(groups, s, sd.EvolutionPlan(total_time=0.0, n_steps=0))
    a = s.amplitudes()
    assert a[5] == 1 and np.count_nonzero(a) == 1
    with pytest.raises(ValueError):
        sd.evolve_grouped(groups, s, sd.EvolutionPlan(total_time=1.0, n_steps=-1))
