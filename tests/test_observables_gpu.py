"""Observables and the per-term baseline on sharded states (SURVEY §8f rows
1-2): expectation (proj/src/evolve.cpp:99-135), norm / fidelity
(proj/src/statevector.cpp:403-418), apply_pauli_rotation
(statevector.cpp:288-337), evolve_baseline (evolve.cpp:21-45), plus the
generic gates (statevector.cpp:101-154) and exact_evolve (evolve.cpp:60-97).

Sharded states are in-process shards on one GPU (the same code path as one
process per GPU except for the transport of the partner shard: device copies
here, NCCL send/recv there). States are evolved first, so the shards sit in a
relabelled qubit layout and terms whose X part flips a global qubit pair
amplitudes across shards.
"""
import numpy as np
import pytest

from paper_2206_11664_b200 import models as M

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _sharded_state(sd, port, cfg, n, world, steps):
    """(shards, reference state) after `steps` fused Trotter steps from a
    random state (shards relabelled by the remaps)."""
    text = M.config_text(cfg, n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    a0 = port.random_state(n, 11)
    sh = sd.LocalShards(n, world)
    sh.upload(a0)
    sh.plan(groups, order=1)
    dt = M.CONFIGS[cfg]["dt"]
    sh.evolve(dt, steps)
    _, og = port.partition_and_diagonalize(text)
    want = port.evolve_grouped(a0, n, og, dt, steps, 1)
    return text, sh, want


@pytest.mark.parametrize("cfg,n,world", [(4, 12, 4), (3, 12, 8), (5, 13, 2), (4, 14, 1)])
def test_sharded_expectation_matches_reference(cfg, n, world, sd, port, ref):
    text, sh, want = _sharded_state(sd, port, cfg, n, world, 3)
    H = sd.Hamiltonian.load(text)
    e, im = sd.expectation(H, sh, with_residue=True)
    e_ref, im_ref = ref.expectation(text, want, n)
    assert abs(e - e_ref) <= TOL * max(1.0, abs(e_ref)), (e, e_ref)
    assert im < 1e-12
    assert abs(sh.norm() - 1.0) < 1e-12
    assert abs(sd.fidelity(sh, sh) - 1.0) < 1e-12


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_fidelity_between_states(world, sd, port):
    n = 11
    a = port.random_state(n, 3)
    b = port.random_state(n, 4)
    sa, sb = sd.LocalShards(n, world), sd.LocalShards(n, world)
    sa.upload(a)
    sb.upload(b)
    assert abs(sd.fidelity(sa, sb) - abs(np.vdot(a, b))) < 1e-13


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_pauli_rotations_match_reference(world, sd, port, ref):
    """Every X/Y pattern, including X on the global (top) qubits."""
    n = 11
    a0 = port.random_state(n, 5)
    sh = sd.LocalShards(n, world)
    sh.upload(a0)
    want = a0.copy()
    rng = np.random.default_rng(7)
    for k in range(24):
        x = int(rng.integers(0, 1 << n)) if k % 3 else (1 << (n - 1)) | (1 << 2)
        z = int(rng.integers(0, 1 << n))
        c = float(rng.normal())
        term = sd.WeightedTerm(c, sd.PauliString(n, x, z))
        sh.apply_pauli_rotation(term, 0.13)
        want = ref.pauli_rotation(want, n, x, z, c, 0.13)
    assert np.max(np.abs(sh.amplitudes() - want)) < TOL


def test_sharded_evolve_baseline_matches_reference(sd, port, ref):
    cfg, n, world, steps = 5, 12, 4, 2
    text = M.config_text(cfg, n)
    H = sd.Hamiltonian.load(text)
    psi0 = np.zeros(1 << n, np.complex128)
    psi0[M.initial_index(cfg, n)] = 1
    sh = sd.LocalShards(n, world)
    sh.upload(psi0)
    dt = M.CONFIGS[cfg]["dt"]
    sd.evolve_baseline(H, sh, sd.EvolutionPlan(total_time=dt * steps, n_steps=steps))
    want = ref.evolve_baseline(text, psi0, n, dt, steps)
    assert np.max(np.abs(sh.amplitudes() - want)) < 1e-10


def test_generic_gates_match_reference(sd, port, ref):
    n = 9
    a0 = port.random_state(n, 9)
    psi = sd.StateVector(n)
    psi.upload(a0)
    want = a0.copy()
    rng = np.random.default_rng(3)
    for k in range(12):
        m = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
        q, _ = np.linalg.qr(m)
        if k % 2:
            q1, q2 = [int(v) for v in rng.choice(n, 2, replace=False)]
            psi.apply_two_qubit(q, q1, q2)
            want = ref.generic_gate(want, n, q, q1, q2)
        else:
            t = int(rng.integers(0, n))
            u2 = np.linalg.qr(m[:2, :2])[0]
            psi.apply_single_qubit(u2, t)
            want = ref.generic_gate(want, n, u2, t)
    assert np.max(np.abs(psi.amplitudes() - want)) < TOL
    with pytest.raises(ValueError, match="not unitary"):
        psi.apply_single_qubit(np.array([[1, 1], [0, 1]]), 0)
    with pytest.raises(ValueError, match="distinct"):
        psi.apply_two_qubit(np.eye(4), 2, 2)
    with pytest.raises(IndexError):
        psi.apply_single_qubit(np.eye(2), n)


def test_exact_evolve_matches_dense_expm(sd, port):
    from scipy.linalg import expm

    n, t = 8, 0.7
    text = M.config_text(3, n)
    H = sd.Hamiltonian.load(text)
    a0 = port.random_state(n, 1)
    psi = sd.StateVector(n)
    psi.upload(a0)
    out = sd.exact_evolve(H, psi, t)
    _, xs, zs, cs = port.load(text)
    dim = 1 << n
    Hd = np.zeros((dim, dim), np.complex128)
    b = np.arange(dim)
    for x, z, c in zip(xs, zs, cs):
        base = c * (1j ** (bin(x & z).count("1") & 3))
        par = np.array([bin(v & z).count("1") & 1 for v in range(dim)])
        Hd[b ^ x, b] += np.where(par == 1, -base, base)
    want = expm(-1j * t * Hd) @ a0
    assert np.max(np.abs(out.amplitudes() - want)) < 1e-11
    assert np.max(np.abs(psi.amplitudes() - a0)) == 0.0  # input untouched
    with pytest.raises(ValueError, match="n <= 12"):
        sd.exact_evolve(sd.Hamiltonian.load(M.config_text(4, 14)), sd.StateVector(14), 0.1)
