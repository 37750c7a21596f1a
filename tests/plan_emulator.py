"""Numpy emulation of a fused schedule (sd_plan_preview JSON) -- test only.

Applies each pass's stages to the whole state exactly as the sm_100a tile
kernel applies them per tile (every stage is tile-local, so applying it
globally is equivalent). Used to check the planner's reordering and
lowering against the oracle without a GPU.
"""
from __future__ import annotations

import numpy as np


def _popcount(a: np.ndarray) -> np.ndarray:
    a = a.copy()
    c = np.zeros_like(a)
    while np.any(a):
        c += a & np.uint64(1)
        a >>= np.uint64(1)
    return c


def permute_bits(a: np.ndarray, n: int, new_pos) -> np.ndarray:
    """psi'[f(i)] = psi[i] where f moves bit b of i to bit new_pos[b]."""
    idx = np.arange(1 << n, dtype=np.uint64)
    f = np.zeros_like(idx)
    for b, p in enumerate(new_pos):
        f |= ((idx >> np.uint64(b)) & np.uint64(1)) << np.uint64(p)
    out = np.empty_like(a)
    out[f] = a
    return out


def exchange_map(n: int, n_local: int, ex: dict):
    """Physical bit map of one exchange: sigma on the local bits, then each
    (global bit, local bit) pair swapped."""
    pos = list(ex["sigma"]) + list(range(n_local, n))
    for gb, lb in ex["swaps"]:
        pos = [lb if p == gb else (gb if p == lb else p) for p in pos]
    return pos


def run_passes(a: np.ndarray, n: int, passes, dt: float, idx=None) -> np.ndarray:
    """Apply passes to `a`, whose entry j has global index idx[j] (default:
    the whole state). Every stage only pairs entries that differ in local
    bits, so a rank's shard can be emulated on its own."""
    if idx is None:
        idx = np.arange(1 << n, dtype=np.uint64)
    base = idx[0] if len(idx) else np.uint64(0)
    for p in passes:
        lpos = p["lpos"]
        for st in p["stages"]:
            if st["kind"] == "wht":
                for j in range(len(lpos)):
                    if (st["mask"] >> j) & 1:
                        b = 1 << lpos[j]
                        lo = (idx & np.uint64(b)) == 0
                        i0 = (idx[lo] - base).astype(np.int64)
                        i1 = i0 + b
                        x, y = a[i0].copy(), a[i1].copy()
                        a[i0], a[i1] = x + y, x - y
            elif st["kind"] == "cx":
                T = 0
                for j in range(len(lpos)):
                    if (st["mask"] >> j) & 1:
                        T |= 1 << lpos[j]
                cb = lpos[st["ctrl_local"]] if st["ctrl_local"] >= 0 else st["ctrl_phys"]
                on = ((idx >> np.uint64(cb)) & np.uint64(1)) == 1
                src = np.where(on, idx ^ np.uint64(T), idx) - base
                a = a[src.astype(np.int64)]
            else:
                q = _popcount(idx & np.uint64(st["s1"])) + 2 * _popcount(idx & np.uint64(st["s2"]))
                cz = np.zeros_like(idx)
                for m in st["cz"]:
                    cz ^= ((idx & np.uint64(m)) == np.uint64(m)).astype(np.uint64)
                q = (q + 2 * cz) & np.uint64(3)
                a = a * (1j ** q.astype(np.int64))
                if st["terms"]:
                    ang = np.zeros(len(idx))
                    for mask, c, s in st["terms"]:
                        par = _popcount(idx & np.uint64(mask)) & np.uint64(1)
                        ang += np.where(par == 1, -c * s, c * s)
                    a = a * np.exp(1j * (-dt) * ang)
        a = a * (2.0 ** -p["scale_exp"])
    return a


def step_at(sched: dict, i: int) -> dict:
    steps, c0 = sched["steps"], sched["cycle_start"]
    if i < len(steps):
        return steps[i]
    return steps[c0 + (i - c0) % (len(steps) - c0)]


def run_schedule(psi: np.ndarray, n: int, sched: dict, dt: float, steps: int = 1) -> np.ndarray:
    """Full-state emulation of a (possibly sharded) schedule from
    sd_plan_preview: passes in the physical layout, exchanges as physical
    bit permutations; returns the state in logical qubit order."""
    a = np.array(psi, dtype=np.complex128, copy=True)
    n_local = sched["n_local"]
    layout = list(range(n))
    for i in range(steps):
        st = step_at(sched, i)
        assert st["phys_in"] == layout
        for seg in st["segments"]:
            a = run_passes(a, n, seg["plan"]["passes"], dt)
            if seg["exchange"] is not None:
                a = permute_bits(a, n, exchange_map(n, n_local, seg["exchange"]))
        layout = st["phys_out"]
    # physical -> logical: logical qubit q lives at physical bit layout[q]
    inv = [0] * n
    for q, p in enumerate(layout):
        inv[p] = q
    return permute_bits(a, n, inv)
