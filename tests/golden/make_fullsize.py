"""Full-size parity fixtures from the REFERENCE ITSELF (oracle/_ref) --
TEST INFRASTRUCTURE ONLY.

Runs the reference's evolve_grouped (proj/src/evolve.cpp:47-58, compiled from
/root/reference/proj/src by oracle/Makefile; S2 is the SURVEY §8a D1
composition in oracle/ref_harness.cpp) at the BASELINE sizes of configs 2, 3
and 4, and stores a fingerprint of each state (tests/fingerprint.py) after
the listed step counts:

    config 2  n=25 TFIM 5x5, |+>^25, S2 dt=0.02      after 20 and 500 steps
    config 3  n=28 random 4-local M=2000, random_state(28, 2), dt=0.005   1 step
    config 4  n=30 XXZ chain, Neel, dt=0.01          after 1 and 3 steps
    config 5  its generator at n=26 (the reference caps n <= 30; n=33 has no CPU
              oracle), |1^16 0^10>, dt=0.01              after 1 step

Run where /root/reference exists (needs ~34 GiB host RAM for n=30):
    make -C oracle && python tests/golden/make_fullsize.py [case ...]
Writes tests/golden/fullsize_<case>.npz (a few hundred KB each).
"""
import ctypes as C
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from fingerprint import fingerprint  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2206_11664_b200 import models as M  # noqa: E402

CASES = {
    "cfg4_n30": (4, [1, 3]),
    "cfg3_n28": (3, [1]),
    "cfg2_n25": (2, [20, 500]),
    "cfg5_n26": (5, [1], 26),
}


def run_case(name: str, ref: O.Ref) -> None:
    cfg, checkpoints = CASES[name][:2]
    n = CASES[name][2] if len(CASES[name]) > 2 else M.CONFIGS[cfg]["n"]
    dt, order = M.CONFIGS[cfg]["dt"], M.CONFIGS[cfg]["order"]
    h, nn, _ = ref.partition_text(M.config_text(cfg, None if n == M.CONFIGS[cfg]["n"] else n), synthesize=True)
    assert nn == n
    init = M.CONFIGS[cfg]["init"]
    if init[0] == "basis":
        a = np.zeros(1 << n, np.complex128)
        a[M.initial_index(cfg, n)] = 1.0
    elif init[0] == "plus":
        a = np.full(1 << n, 1.0 / np.sqrt(float(1 << n)), np.complex128)
    else:
        a = ref.random_state(n, init[1])
    st = np.zeros(3, np.uint64)
    done = 0
    for k in checkpoints:
        t0 = time.perf_counter()
        ref._err(ref.lib.ref_evolve_grouped(h, a.ctypes.data_as(C.POINTER(C.c_double)), n, dt, k - done, order,
                                            st.ctypes.data_as(C.POINTER(C.c_uint64))))
        secs = time.perf_counter() - t0
        per = secs / (k - done)
        done = k
        fp = fingerprint(a, n)
        out = os.path.join(HERE, f"fullsize_{name}_s{k}.npz")
        np.savez_compressed(out, cfg=cfg, n=n, steps=k, dt=dt, order=order, ref_s_per_step=per,
                            ref_threads=ref_threads(), **fp)
        print(f"{name}: {k} steps, {per:.1f} s/step ({ref_threads()} threads), norm {float(fp['norm']):.17g}"
              f" -> {os.path.basename(out)}", flush=True)
    ref.free(h)
    del a


def ref_threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def main(argv):
    ref = O.ref()
    for name in (argv or list(CASES)):
        run_case(name, ref)


if __name__ == "__main__":
    main(sys.argv[1:])
