"""Full BASELINE step counts at reduced n (SURVEY 8c oracle plan): every config's
own generator and initial state, all of its Trotter steps, against the
reference compiled from its sources -- the accumulated error of hundreds of
fused steps, through the sharded path where the config is a multi-GPU one.
Tolerances from the north star: max per-amplitude |dpsi| <= 1e-10 and
|1-||psi||| <= 1e-12 (the reference's own norm drifts by ~1e-11 over these
runs; the GPU state is normalised exactly)."""
import numpy as np
import pytest

from paper_2206_11664_b200 import models as M

pytestmark = pytest.mark.gpu

TOL_AMP = 1e-10
TOL_NORM = 1e-12


def _initial(port, cfg, n):
    init = M.CONFIGS[cfg]["init"]
    if init[0] == "plus":
        return np.full(1 << n, 1 / np.sqrt(1 << n), np.complex128)
    if init[0] == "random":
        return port.random_state(n, init[1])
    a = np.zeros(1 << n, np.complex128)
    a[M.initial_index(cfg, n)] = 1
    return a


@pytest.mark.parametrize("cfg,n,world", [(2, 16, 1), (3, 16, 1), (4, 20, 2), (4, 20, 1), (5, 16, 8)])
def test_full_step_count_matches_reference(cfg, n, world, sd, ref, port):
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order, dt, steps = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"], M.CONFIGS[cfg]["steps"]
    psi0 = _initial(port, cfg, n)
    if world == 1:
        s = sd.StateVector(n)
        s.upload(psi0)
        sd.TrotterPlan(s, groups, order=order).evolve(dt, steps)
        got = s.amplitudes()
    else:
        sh = sd.LocalShards(n, world)
        sh.enable_p2p()
        sh.upload(psi0)
        sh.plan(groups, order=order)
        sh.evolve(dt, steps)
        got = sh.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, steps, order)
    ref.free(h)
    assert np.max(np.abs(got - want)) < TOL_AMP
    assert abs(np.linalg.norm(got) - 1) < TOL_NORM
