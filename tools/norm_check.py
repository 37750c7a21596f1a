"""Norm after a few steps of a BASELINE config (debugging aid).
usage: python tools/norm_check.py cfg n steps"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_11664_b200 as S  # noqa: E402
from paper_2206_11664_b200 import models as M  # noqa: E402
from oracle import oracle as O  # noqa: E402

cfg, n, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
text = M.config_text(cfg, None if n == M.CONFIGS[cfg]["n"] else n)
groups = S.partition_and_diagonalize(S.Hamiltonian.load(text))
psi = S.StateVector(n)
init = M.CONFIGS[cfg]["init"]
if init[0] == "basis":
    psi.set_basis(M.initial_index(cfg, n))
elif init[0] == "random":
    psi.upload(O.port().random_state(n, init[1]))
plan = S.TrotterPlan(psi, groups, order=M.CONFIGS[cfg]["order"])
plan.evolve(M.CONFIGS[cfg]["dt"], steps)
print(f"cfg {cfg} n {n} steps {steps} env {[k + '=' + v for k, v in os.environ.items() if k.startswith('SDB_')]} "
      f"passes {plan.info()['n_passes_per_step']} norm-1 {psi.norm() - 1:.3e}", flush=True)
