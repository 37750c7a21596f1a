"""Runs a few Trotter steps of a BASELINE config for ncu captures.
usage: python tools/profile_pass.py [cfg] [n] [steps] [tile]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_11664_b200 as S  # noqa: E402
from paper_2206_11664_b200 import models as M  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 28
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
tile = int(sys.argv[4]) if len(sys.argv) > 4 else 0
text = M.config_text(cfg, None if n == M.CONFIGS[cfg]["n"] else n)
groups = S.partition_and_diagonalize(S.Hamiltonian.load(text))
psi = S.StateVector(n)
if M.CONFIGS[cfg]["init"][0] == "basis":
    psi.set_basis(M.initial_index(cfg, n))
plan = S.TrotterPlan(psi, groups, order=M.CONFIGS[cfg]["order"], tile_qubits=tile)
print(plan.describe())
plan.evolve(M.CONFIGS[cfg]["dt"], steps)
print("norm", psi.norm())
