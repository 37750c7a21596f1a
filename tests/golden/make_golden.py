"""Generates tests/golden/ from the REFERENCE ITSELF (oracle/_ref, compiled
from /root/reference/proj/src by oracle/Makefile). TEST INFRASTRUCTURE ONLY.

Run in the container that has /root/reference (the GPU box does not):
    make -C oracle && python tests/golden/make_golden.py

Writes:
  groups_cfg{1..5}.json.gz  greedy_partition + diagonalize_group of each
                            BASELINE config at its full size: source terms,
                            circuits, z-masks, signed coefficients (doubles as
                            float.hex, masks as hex) -- the bit-exact contract.
  states.npz                reference evolve_grouped outputs on small seeded
                            cases of every config generator (+ config 1 at its
                            full BASELINE size) and random_state vectors.
  cases.json                the parameters of every state case.
"""
import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2206_11664_b200 import models as M  # noqa: E402

# (name, cfg, n, steps): reduced-n runs of each generator at the config's own
# dt/order/initial state; config 1 runs at its full BASELINE size.
STATE_CASES = [
    ("cfg1_full", 1, 16, 100),
    ("cfg2_n9", 2, 9, 40),
    ("cfg3_n10", 3, 10, 20),
    ("cfg4_n12", 4, 12, 200),
    ("cfg5_n10", 5, 10, 10),
]
RANDOM_STATES = [(12, 2), (10, 7)]


def group_doc(g):
    return {
        "h_pre": g.h_pre, "cnots": [list(p) for p in g.cnots], "czs": [list(p) for p in g.czs],
        "s_layer": g.s_layer, "h_post": g.h_post,
        "src_x": [hex(v) for v in g.src_x], "src_z": [hex(v) for v in g.src_z],
        "src_c": [float(v).hex() for v in g.src_c],
        "z_masks": [hex(v) for v in g.z_masks], "coeffs": [float(v).hex() for v in g.coeffs],
    }


def initial(ref, cfg, n):
    init = M.CONFIGS[cfg]["init"]
    if init[0] == "plus":
        return np.full(1 << n, 1 / np.sqrt(1 << n), np.complex128)
    if init[0] == "random":
        return ref.random_state(n, init[1])
    a = np.zeros(1 << n, np.complex128)
    a[M.initial_index(cfg, n)] = 1
    return a


def main():
    ref = O.ref()
    for cfg in (1, 2, 3, 4, 5):
        text = M.config_text(cfg)
        h, n, groups = ref.partition_text(text)
        ref.free(h)
        doc = {"config": cfg, "n": n, "groups": [group_doc(g) for g in groups]}
        with gzip.open(os.path.join(HERE, f"groups_cfg{cfg}.json.gz"), "wt") as f:
            json.dump(doc, f, separators=(",", ":"))
        print(f"cfg{cfg}: n={n} groups={len(groups)}")
    arrays, cases = {}, []
    for name, cfg, n, steps in STATE_CASES:
        text = M.config_text(cfg, None if n == M.CONFIGS[cfg]["n"] else n)
        h, nn, _ = ref.partition_text(text)
        psi0 = initial(ref, cfg, n)
        out, stats = ref.evolve_grouped(h, psi0, n, M.CONFIGS[cfg]["dt"], steps, M.CONFIGS[cfg]["order"])
        ref.free(h)
        arrays[name] = out
        cases.append({"name": name, "config": cfg, "n": n, "steps": steps, "dt": M.CONFIGS[cfg]["dt"],
                      "order": M.CONFIGS[cfg]["order"], "init": list(M.CONFIGS[cfg]["init"]),
                      "ref_norm": ref.norm(out, n), "ref_kernel_stats": stats})
        print(f"{name}: |psi|-1 = {ref.norm(out, n) - 1:.3e}")
    for n, seed in RANDOM_STATES:
        arrays[f"random_{n}_{seed}"] = ref.random_state(n, seed)
    np.savez_compressed(os.path.join(HERE, "states.npz"), **arrays)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump({"state_cases": cases, "random_states": RANDOM_STATES}, f, indent=1)


if __name__ == "__main__":
    main()
