"""Writes the state after the first SDB_DEBUG_PASSES passes of one step of a
config (debugging aid): python tools/pass_diff.py cfg n out.npy"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_11664_b200 as S  # noqa: E402
from paper_2206_11664_b200 import models as M  # noqa: E402
from oracle import oracle as O  # noqa: E402

cfg, n, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
groups = S.partition_and_diagonalize(S.Hamiltonian.load(M.config_text(cfg, n)))
psi = S.StateVector(n)
psi.upload(O.port().random_state(n, 7))
plan = S.TrotterPlan(psi, groups, order=M.CONFIGS[cfg]["order"], use_graph=False)
plan.evolve(M.CONFIGS[cfg]["dt"], 1)
np.save(out, psi.amplitudes())
