"""Edge cases of the fused device path against the reference compiled from
its sources: the smallest registers (n = 1..4, tile wider than the state),
identity and constant terms, single-term and diagonal-only groups, terms on
the top qubit, duplicate terms merged by from_terms, an empty Hamiltonian,
order-2 steps, and n_steps = 0."""
import os

import numpy as np
import pytest

from paper_2206_11664_b200 import models as M

pytestmark = pytest.mark.gpu


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return a / np.linalg.norm(a)


def run_both(sd, ref, text, n, dt=0.11, steps=3, order=1, k=0):
    psi0 = rand_state(n, n + steps)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    s = sd.StateVector(n)
    s.upload(psi0)
    sd.TrotterPlan(s, groups, order=order, tile_qubits=k).evolve(dt, steps)
    got = s.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, steps, order)
    ref.free(h)
    return got, want


@pytest.mark.parametrize("text,n", [
    ("0.7 X\n-0.3 Z\n0.2 Y\n", 1),
    ("1.0 XX\n0.5 YY\n-0.25 ZZ\n0.4 ZI\n", 2),
    ("0.9 XYZ\n-0.4 ZZZ\n0.3 IXI\n0.8 YIY\n", 3),
    ("1.0 XZYX\n1.0 ZXXY\n-0.5 IIIZ\n0.3 YYYY\n0.2 ZIZI\n", 4),
])
@pytest.mark.parametrize("order", [1, 2])
def test_tiny_registers(text, n, order, sd, ref):
    got, want = run_both(sd, ref, text, n, order=order)
    assert np.max(np.abs(got - want)) < 1e-12
    assert abs(np.linalg.norm(got) - 1) < 1e-12


def test_identity_and_duplicate_terms(sd, ref):
    # identity term (global phase), duplicates merged in first-seen order, a
    # term cancelling to zero (dropped), a term on the top qubit
    text = "0.5 IIIIIIII\n0.3 XXIIIIII\n0.2 XXIIIIII\n0.4 ZIIIIIIZ\n-0.4 ZIIIIIIZ\n0.6 IIIIIIIY\n0.1 YZIIIIIX\n"
    got, want = run_both(sd, ref, text, 8)
    assert np.max(np.abs(got - want)) < 1e-12


def test_diagonal_only_and_single_term_groups(sd, ref):
    text = "0.3 ZZIIIIIIII\n-0.7 IZZIIIIIII\n0.2 IIIIIIIIIZ\n0.9 XIIIIIIIIX\n"
    got, want = run_both(sd, ref, text, 10, k=6)
    assert np.max(np.abs(got - want)) < 1e-12


def test_every_tile_width(sd, ref):
    text = "0.4 XZYIXZ\n0.3 ZZZZZZ\n-0.2 YIYIYI\n0.5 IXIXIX\n0.1 XXXXXX\n"
    outs = []
    for k in range(1, 7):
        got, want = run_both(sd, ref, text, 6, k=k)
        assert np.max(np.abs(got - want)) < 1e-12, k
        outs.append(got)


def test_empty_hamiltonian_and_zero_steps(sd):
    n = 5
    psi0 = rand_state(n, 1)
    s = sd.StateVector(n)
    s.upload(psi0)
    sd.TrotterPlan(s, [], order=1).evolve(0.1, 4)
    assert np.max(np.abs(s.amplitudes() - psi0)) == 0.0
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load("1.0 XIIII\n"))
    sd.TrotterPlan(s, groups).evolve(0.1, 0)
    assert np.max(np.abs(s.amplitudes() - psi0)) == 0.0


def test_download_range_matches_full_download(sd):
    n = 12
    rng = np.random.default_rng(5)
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    s = sd.StateVector(n)
    s.upload(a / np.linalg.norm(a))
    full = s.amplitudes()
    for first, count in ((0, 1), (17, 100), (4000, 96), (0, 1 << n), (1 << n, 0)):
        assert np.array_equal(s.amplitudes(first, count), full[first:first + count])
    with pytest.raises(IndexError):
        s.amplitudes(4000, 97)


def test_relabelled_layout_is_transparent(sd, ref):
    """States of >= 22 qubits may run their steps in a relabelled layout (plan
    layout search); readout, direct kernels and a second plan must not see it."""
    from paper_2206_11664_b200 import models as M
    n, cfg = 22, 4
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    rng = np.random.default_rng(11)
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    a /= np.linalg.norm(a)
    s = sd.StateVector(n)
    s.upload(a)
    dt = 0.02
    sd.TrotterPlan(s, groups, order=1).evolve(dt, 2)
    s.apply_hadamard(3)                                        # direct kernel after a relabelled step
    sd.TrotterPlan(s, list(reversed(groups)), order=1).evolve(dt, 1)
    got = s.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, a, n, dt, 2, 1)
    want = ref.kernel(0, want, n, a=3)
    ref.free(h)
    # the reversed-order plan: groups applied in reverse order
    g2 = list(reversed(groups))
    s2 = sd.StateVector(n)
    s2.upload(want)
    sd.TrotterPlan(s2, g2, order=1, use_graph=False).evolve(dt, 1)
    assert np.max(np.abs(got - s2.amplitudes())) < 1e-12
    assert abs(np.linalg.norm(got) - 1) < 1e-12


def test_autotune_keeps_state_and_reports_both_schedules(sd, port):
    """Plan-time autotuning (sd_plan_create, unsharded >= 22 qubits) times both
    schedule families on the scratch buffer: the state is untouched, both times
    are reported and the kept schedule is the faster one."""
    import os

    from paper_2206_11664_b200 import models as M

    if os.environ.get("SDB_AUTOTUNE") == "0":
        pytest.skip("autotune disabled")
    n = 22
    text = M.config_text(4, n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    a0 = port.random_state(n, 5)
    psi = sd.StateVector(n)
    psi.upload(a0)
    plan = sd.TrotterPlan(psi, groups, order=1)
    info = plan.info()
    assert np.array_equal(psi.amplitudes(), a0)
    if info["tune_ms_whole"] > 0:
        assert info["tune_ms_split"] > 0
        faster = 1 if info["tune_ms_split"] < info["tune_ms_whole"] else 0
        assert info["schedule"] == faster
    plan.evolve(0.01, 2)
    _, og = port.partition_and_diagonalize(text)
    want = port.evolve_grouped(a0, n, og, 0.01, 2, 1)
    assert np.max(np.abs(psi.amplitudes() - want)) < 1e-10


@pytest.mark.parametrize("steps", [1, 4, 5])
def test_macro_step_plan_matches_reference(steps, sd, ref, port, monkeypatch):
    """Two Trotter steps planned as one macro step (order 1, group list
    repeated; SDB_MACRO_FORCE keeps it regardless of the timing), whole macro
    steps plus an odd remainder step through the base plan, against the
    reference's evolve_grouped loop."""
    if os.environ.get("SDB_AUTOTUNE") == "0":
        pytest.skip("autotune disabled")
    monkeypatch.setenv("SDB_MACRO_FORCE", "1")
    n = 22
    text = M.config_text(4, n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    a0 = port.random_state(n, 7)
    psi = sd.StateVector(n)
    psi.upload(a0)
    plan = sd.TrotterPlan(psi, groups, order=1)
    info = plan.info()
    assert np.array_equal(psi.amplitudes(), a0)
    if info["macro_steps"] == 0:
        pytest.skip("macro plan needs no fewer passes per step at this size")
    assert info["macro_steps"] == 2 and info["macro_passes"] < 2 * info["n_passes_per_step"]
    dt = 0.05
    plan.evolve(dt, steps)
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, a0, n, dt, steps, 1)
    ref.free(h)
    got = psi.amplitudes()
    assert np.max(np.abs(got - want)) < 1e-10
    assert abs(np.linalg.norm(got) - 1) < 1e-12
