"""Full-size state fingerprints -- TEST INFRASTRUCTURE ONLY.

A 2^30-amplitude reference state (16 GiB) cannot be committed, and the
reference needs minutes per Trotter step at BASELINE sizes, so the full-size
parity fixtures (tests/golden/fullsize_*.npz, made by
tests/golden/make_fullsize.py from oracle/_ref, the reference compiled from
its own sources) hold a fingerprint of the reference's state instead:

* ``idx``/``val``: the amplitudes at 2^14 pseudo-random indices plus the
  2^12 largest-magnitude amplitudes (where an error of fixed relative size is
  largest in absolute terms), compared per amplitude (max |dpsi| <= 1e-10);
* ``bsum``: per block of 2^(n-12) consecutive amplitudes, the weighted sum
  sum_i w(i) psi_i with unit weights w(i) = exp(2 pi i frac(i phi)) -- a linear
  sketch that covers EVERY amplitude: an error delta at index j moves its
  block's sum by |delta| (unless it cancels against another error with the
  matching pseudo-random phase), while agreement to 1e-15 per amplitude
  keeps the sums within ~1e-13;
* ``bnrm``: per block, sum_i |psi_i|^2 (phase-blind mass distribution);
* ``norm``: the reference's ||psi||.

The same functions run on the GPU box over the downloaded product state.
"""
from __future__ import annotations

import numpy as np

PHI = 0.6180339887498949  # frac of the golden ratio
N_RANDOM = 1 << 14
N_TOP = 1 << 12
BLOCK_BITS = 12  # 2^12 blocks per state


def sample_indices(n: int, seed: int = 0x5EED) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed + n))
    return np.unique(rng.integers(0, 1 << n, size=min(N_RANDOM, 1 << n), dtype=np.int64))


def _chunks(n: int):
    step = 1 << min(n, 24)
    for first in range(0, 1 << n, step):
        yield first, min(step, (1 << n) - first)


def block_sketch(get_chunk, n: int):
    """(bsum, bnrm) over 2^BLOCK_BITS blocks; get_chunk(first, count) returns
    psi[first:first+count] (a host array or a device download)."""
    nb = 1 << min(BLOCK_BITS, n)
    blk = (1 << n) // nb
    bsum = np.zeros(nb, np.complex128)
    bnrm = np.zeros(nb, np.float64)
    for first, cnt in _chunks(n):
        a = np.asarray(get_chunk(first, cnt), dtype=np.complex128)
        i = np.arange(first, first + cnt, dtype=np.float64)
        ph = 2.0 * np.pi * np.mod(i * PHI, 1.0)
        w = np.cos(ph) + 1j * np.sin(ph)
        b0 = first // blk
        nbl = max(1, cnt // blk)
        if cnt >= blk:
            bsum[b0:b0 + nbl] += (w * a).reshape(nbl, blk).sum(axis=1)
            bnrm[b0:b0 + nbl] += (a.real ** 2 + a.imag ** 2).reshape(nbl, blk).sum(axis=1)
        else:
            bsum[b0] += (w * a).sum()
            bnrm[b0] += float((a.real ** 2 + a.imag ** 2).sum())
    return bsum, bnrm


def top_indices(get_chunk, n: int, k: int = N_TOP) -> np.ndarray:
    best_i = np.zeros(0, np.int64)
    best_v = np.zeros(0, np.float64)
    for first, cnt in _chunks(n):
        m = np.abs(np.asarray(get_chunk(first, cnt)))
        kk = min(k, cnt)
        sel = np.argpartition(m, cnt - kk)[cnt - kk:]
        best_i = np.concatenate([best_i, sel.astype(np.int64) + first])
        best_v = np.concatenate([best_v, m[sel]])
        if best_i.size > k:
            keep = np.argpartition(best_v, best_v.size - k)[best_v.size - k:]
            best_i, best_v = best_i[keep], best_v[keep]
    return np.sort(best_i)


def fingerprint(psi: np.ndarray, n: int) -> dict:
    get = lambda f, c: psi[f:f + c]  # noqa: E731
    idx = np.union1d(sample_indices(n), top_indices(get, n))
    bsum, bnrm = block_sketch(get, n)
    nrm = float(np.sqrt(bnrm.sum()))
    return {"idx": idx, "val": psi[idx].copy(), "bsum": bsum, "bnrm": bnrm, "norm": np.float64(nrm)}


def compare(fp: dict, get_chunk, n: int) -> dict:
    """Deviations of a product state from a reference fingerprint, streamed
    chunk by chunk (get_chunk(first, count) -> psi[first:first+count])."""
    idx = fp["idx"]
    got = np.zeros(idx.size, np.complex128)

    def fetch(first, cnt):
        a = np.asarray(get_chunk(first, cnt), dtype=np.complex128)
        lo, hi = np.searchsorted(idx, [first, first + cnt])
        got[lo:hi] = a[idx[lo:hi] - first]
        return a

    bsum, bnrm = block_sketch(fetch, n)
    return {
        "max_abs_dpsi_sampled": float(np.max(np.abs(got - fp["val"]))),
        "n_sampled": int(idx.size),
        "max_abs_dblock_sketch": float(np.max(np.abs(bsum - fp["bsum"]))),
        "max_abs_dblock_mass": float(np.max(np.abs(bnrm - fp["bnrm"]))),
        "norm_err": abs(float(np.sqrt(bnrm.sum())) - 1.0),
        "ref_norm_err": abs(float(fp["norm"]) - 1.0),
    }
