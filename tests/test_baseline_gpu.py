"""The paper's comparison method and observables on the device (SURVEY 8f
rows 1-2): apply_pauli_rotation / evolve_baseline (statevector.cpp:288-337,
evolve.cpp:21-45) and expectation (evolve.cpp:99-135) against the reference
compiled from its sources, plus SPEC.md:634's property that grouped evolution
equals the group-major per-term baseline (terms of a group commute)."""
import numpy as np
import pytest

from paper_2206_11664_b200 import models as M

pytestmark = pytest.mark.gpu


def rand_state(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return a / np.linalg.norm(a)


def test_pauli_rotation_matches_reference(sd, ref):
    n = 9
    rng = np.random.default_rng(5)
    psi0 = rand_state(n, 3)
    s = sd.StateVector(n)
    s.upload(psi0)
    want = psi0
    for k in range(24):
        x = 0 if k % 5 == 0 else int(rng.integers(1, 1 << n))
        z = int(rng.integers(0, 1 << n))
        c, dt = float(rng.normal()), 0.07
        s.apply_pauli_rotation(sd.WeightedTerm(c, sd.PauliString.from_masks(n, x, z)), dt)
        want = ref.pauli_rotation(want, n, x, z, c, dt)
    assert np.max(np.abs(s.amplitudes() - want)) < 1e-13
    assert s.stats()["kernel_calls"] == 24


@pytest.mark.parametrize("cfg,n,steps", [(4, 10, 5), (3, 9, 3), (5, 9, 2)])
def test_evolve_baseline_matches_reference(cfg, n, steps, sd, ref, port):
    text = M.config_text(cfg, n=n)
    H = sd.Hamiltonian.load(text)
    psi0 = rand_state(n, cfg)
    s = sd.StateVector(n)
    s.upload(psi0)
    dt = M.CONFIGS[cfg]["dt"] * 5
    sd.evolve_baseline(H, s, sd.EvolutionPlan(total_time=dt * steps, n_steps=steps))
    want = ref.evolve_baseline(text, psi0, n, dt, steps)
    assert np.max(np.abs(s.amplitudes() - want)) < 1e-12


@pytest.mark.parametrize("cfg,n", [(4, 10), (3, 10), (5, 9), (2, 9)])
def test_expectation_matches_reference(cfg, n, sd, ref):
    text = M.config_text(cfg, n=n)
    H = sd.Hamiltonian.load(text)
    psi0 = rand_state(n, 7 + cfg)
    s = sd.StateVector(n)
    s.upload(psi0)
    got, res = sd.expectation(H, s, with_residue=True)
    want, wres = ref.expectation(text, psi0, n)
    assert abs(got - want) < 1e-12 * max(1.0, abs(want))
    assert res < 1e-12


@pytest.mark.parametrize("cfg,n", [(4, 11), (3, 10), (5, 10)])
def test_grouped_equals_group_major_baseline(cfg, n, sd):
    """terms of a commuting group commute, so C D C^dagger per
    group equals the per-term rotations of that group in any order."""
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    psi0 = rand_state(n, 11)
    a = sd.StateVector(n)
    a.upload(psi0)
    b = sd.StateVector(n)
    b.upload(psi0)
    plan = sd.EvolutionPlan(total_time=0.3, n_steps=3)
    sd.evolve_grouped(groups, a, plan)
    sd.evolve_baseline(groups, b, plan)
    assert np.max(np.abs(a.amplitudes() - b.amplitudes())) < 1e-10
