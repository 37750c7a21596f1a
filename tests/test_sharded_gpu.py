"""Sharded execution on one GPU: `world` virtual shards of one state driven
by this process (sd_state_create_local_shards / sd_evolve_local). The plan,
the sigma-permuting store of the pass in front of each remap and the chunk
routing are exactly those of the NCCL path (only the transport differs:
device copies instead of ncclSend/ncclRecv), so these tests pin the sharded
data path against the reference CPU oracle."""
import numpy as np
import pytest

from paper_2206_11664_b200 import models as M

pytestmark = pytest.mark.gpu

TOL_AMP = 1e-10
TOL_NORM = 1e-12


def initial(port, cfg, n):
    init = M.CONFIGS[cfg]["init"]
    if init[0] == "plus":
        return np.full(1 << n, 1 / np.sqrt(1 << n), np.complex128)
    if init[0] == "random":
        return port.random_state(n, init[1])
    a = np.zeros(1 << n, np.complex128)
    a[M.initial_index(cfg, n)] = 1
    return a


@pytest.mark.parametrize("fused", [False, True], ids=["copy-exchange", "fused-p2p"])
@pytest.mark.parametrize("cfg,n,world,k", [(1, 12, 2, 8), (2, 12, 4, 8), (3, 12, 2, 9), (4, 13, 2, 9),
                                           (4, 13, 8, 8), (4, 15, 4, 12), (5, 12, 4, 8), (5, 13, 8, 9)])
def test_local_shards_match_reference(cfg, n, world, k, fused, sd, ref, port):
    text = M.config_text(cfg, n=n)
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    order, dt, steps = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"] * 5, 3
    psi0 = initial(port, cfg, n)
    sh = sd.LocalShards(n, world)
    if fused:
        sh.enable_p2p()
    sh.upload(psi0)
    sh.plan(groups, order=order, tile_qubits=k)
    sh.evolve(dt, steps)
    info = sh.plans[0].info()  # steady-state layout
    got = sh.amplitudes()
    h, _, _ = ref.partition_text(text)
    want, _ = ref.evolve_grouped(h, psi0, n, dt, steps, order)
    ref.free(h)
    assert np.max(np.abs(got - want)) < TOL_AMP
    assert abs(np.linalg.norm(got) - 1) < TOL_NORM
    if cfg == 4:
        assert info["n_exchanges_per_step"] >= 1  # four Hadamard layers per step reach every qubit


def test_local_shards_agree_across_world_sizes(sd, port):
    """Config-5 generator: P = 1, 2, 4, 8 give the same state (the indirect
    n=33 parity argument of SURVEY 8c, exercised at n=13)."""
    cfg, n = 5, 13
    groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(M.config_text(cfg, n=n)))
    psi0 = initial(port, cfg, n)
    outs = []
    for world in (1, 2, 4, 8):
        sh = sd.LocalShards(n, world)
        sh.upload(psi0)
        sh.plan(groups, tile_qubits=9)
        sh.evolve(0.02, 4)
        outs.append(sh.amplitudes())
    for o in outs[1:]:
        assert np.max(np.abs(o - outs[0])) < 1e-12
