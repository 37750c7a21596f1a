"""Probe: Trotter steps planned together (order-1 group list repeated r
times = r steps per plan step). Prints ms per Trotter step and passes.
    python tools/macro_probe.py [cfg] [reps...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_11664_b200 as S  # noqa: E402
from paper_2206_11664_b200 import models as M  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = [int(r) for r in sys.argv[2:]] or [1, 2, 3]
n = M.CONFIGS[cfg]["n"]
g = S.partition_and_diagonalize(S.Hamiltonian.load(M.config_text(cfg)))
psi = S.StateVector(n)
psi.set_basis(M.initial_index(cfg, n))
dt = M.CONFIGS[cfg]["dt"]
for r in reps:
    plan = S.TrotterPlan(psi, list(g) * r, order=1)
    info = plan.info()
    plan.evolve(dt, 2)
    steps = max(2, 12 // r)
    t = time.perf_counter()
    plan.evolve(dt, steps)
    ms = (time.perf_counter() - t) * 1e3 / (steps * r)
    print(f"reps {r}: {ms:.2f} ms per Trotter step, passes/plan-step {info['n_passes_per_step']}, "
          f"tune {info.get('tune_ms_whole')} / {info.get('tune_ms_split')}", flush=True)
    del plan
