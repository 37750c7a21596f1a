"""Multi-rank host logic on CPU (gloo, world_size 2 and 4, one process per
rank): every rank plans the sharded schedule itself (sd_plan_preview, host
C++), the plans must agree, and the ranks then run it on their own shards --
passes emulated in numpy on the shard's global indices, every qubit remap
executed with the chunk routing the C++ exchange uses
(sd_exchange_routes, the same function exchange_nccl() loops over) over
torch.distributed point-to-point. The gathered final state must match the
reference CPU oracle. The NCCL transport itself needs >1 GPU; see
tests/test_sharded_gpu.py for the same routing on device."""
import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, n, k, steps, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2206_11664_b200 as sd
        from paper_2206_11664_b200 import models as M
        from oracle import oracle as O
        from tests.plan_emulator import permute_bits, run_passes, step_at

        text = M.config_text(cfg, n=n)
        groups = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
        order, dt = M.CONFIGS[cfg]["order"], M.CONFIGS[cfg]["dt"] * 7
        _, sched = sd.plan_preview(n, groups, order=order, tile_qubits=k, world=world)
        # every rank must have planned the identical schedule
        mine = json.dumps(sched, sort_keys=True)
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        assert all(p == mine for p in allp)
        n_local = sched["n_local"]
        port_ = O.port()
        init = M.CONFIGS[cfg]["init"]
        if init[0] == "random":
            psi0 = port_.random_state(n, init[1])
        elif init[0] == "plus":
            psi0 = np.full(1 << n, 1 / np.sqrt(1 << n), np.complex128)
        else:
            psi0 = np.zeros(1 << n, np.complex128)
            psi0[M.initial_index(cfg, n)] = 1
        sz = 1 << n_local
        a = psi0[rank * sz:(rank + 1) * sz].copy()
        idx = np.arange(sz, dtype=np.uint64) + np.uint64(rank * sz)
        layout = list(range(n))
        n_ex = 0
        for i in range(steps):
            st = step_at(sched, i)
            assert st["phys_in"] == layout
            for seg in st["segments"]:
                a = run_passes(a, n, seg["plan"]["passes"], dt, idx)
                ex = seg["exchange"]
                if ex is None:
                    continue
                n_ex += 1
                B = permute_bits(a, n_local, ex["sigma"])  # the pass's sigma store
                A = np.empty_like(a)
                reqs = []
                bufs = []
                for peer, so, ro, cnt in sd.exchange_routes(n, n_local, rank, ex["swaps"]):
                    if peer == rank:
                        A[ro:ro + cnt] = B[so:so + cnt]
                        continue
                    sbuf = torch.from_numpy(B[so:so + cnt].view(np.float64).copy())
                    rbuf = torch.empty(2 * cnt, dtype=torch.float64)
                    reqs.append(dist.isend(sbuf, peer))
                    reqs.append(dist.irecv(rbuf, peer))
                    bufs.append((ro, cnt, rbuf, sbuf))
                for r in reqs:
                    r.wait()
                for ro, cnt, rbuf, _ in bufs:
                    A[ro:ro + cnt] = rbuf.numpy().view(np.complex128)
                a = A
            layout = st["phys_out"]
        full = [None] * world
        dist.all_gather_object(full, a)
        if rank == 0:
            phys = np.concatenate(full)
            inv = [0] * n
            for qq, p in enumerate(layout):
                inv[p] = qq
            got = permute_bits(phys, n, inv)
            _, og = port_.partition_and_diagonalize(text)
            want = port_.evolve_grouped(psi0, n, og, dt, steps, order)
            q.put((float(np.max(np.abs(got - want))), abs(float(np.linalg.norm(got)) - 1.0), n_ex))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,n,k,world", [(4, 11, 7, 2), (5, 10, 6, 2), (3, 10, 6, 4), (2, 9, 6, 4)])
def test_multirank_gloo_schedule_matches_oracle(cfg, n, k, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, n, k, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    err, nerr, n_ex = q.get(timeout=10)
    assert err < 1e-11 and nerr < 1e-13
    assert n_ex >= 1  # the run really exercised remaps


def test_bench_launcher_starts_one_process_per_gpu():
    """`bench.py --gpus N` without WORLD_SIZE re-launches itself under
    torch.distributed.run: every rank joins one gloo group and sees world == N."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launch-check", "--n", "12"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["launch_check"] and d["world"] == 2 and d["ranks"] == [0, 1]
