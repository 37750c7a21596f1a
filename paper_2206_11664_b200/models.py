"""Seeded generators for the BASELINE.json workloads.

Each generator returns (n_qubits, terms) with terms = [(coeff, pauli_text)]
in a pinned order (greedy_partition is order-dependent) and
can render the reference text format (`Hamiltonian::save`, 17 significant
digits, proj/src/hamiltonian.cpp:128-133), so the reference CPU path and
this framework load bit-identical inputs. Randomness is the reference's
counter RNG (proj/include/simdiag/rng.hpp:15-49), restated here with
documented tags; draws are pure functions of (seed, tag, indices).
The paper's own benchmark models (gen_tfim/gen_syk, proj/src/models.cpp)
are not the BASELINE configs.
"""
from __future__ import annotations

import math
from typing import List, Tuple

M64 = (1 << 64) - 1

# RNG tags (ASCII-ish constants, documented in DESIGN.md §6)
TAG_FIELD = 0x6669656C64      # "field": h_i ~ U[-1, 1]
TAG_KW = 0x6B77               # random k-local: weight
TAG_KQ = 0x6B71               # random k-local: qubit draw
TAG_KP = 0x6B70               # random k-local: Pauli letter
TAG_KC = 0x6B63               # random k-local: coefficient
TAG_JW_Z = 0x6A7A             # JW: Z_p coefficients
TAG_JW_ZZ = 0x6A7A7A          # JW: Z_p Z_q coefficients
TAG_JW_HOP = 0x6A68           # JW: hopping endpoints/type
TAG_JW_HOPC = 0x6A6863        # JW: hopping coefficients
TAG_JW_DBL = 0x6A64           # JW: double-excitation qubits/letters
TAG_JW_DBLC = 0x6A6463        # JW: double-excitation coefficients


def splitmix64(v: int) -> int:
    v = (v + 0x9E3779B97F4A7C15) & M64
    v = ((v ^ (v >> 30)) * 0xBF58476D1CE4E5B9) & M64
    v = ((v ^ (v >> 27)) * 0x94D049BB133111EB) & M64
    return v ^ (v >> 31)


def rng_hash(seed: int, tag: int, a: int = 0, b: int = 0, c: int = 0, d: int = 0) -> int:
    h = splitmix64((seed ^ 0x243F6A8885A308D3) & M64)
    for w in (tag, a, b, c, d):
        h = splitmix64(h ^ (w & M64))
    return h


def uniform01(word: int) -> float:
    return float(word >> 11) * (2.0 ** -53)


def uniform_pm1(word: int) -> float:
    return 2.0 * uniform01(word) - 1.0


def gaussian(word: int) -> float:
    u1 = uniform01(splitmix64(word ^ 0x5BF0A8DC))
    u2 = uniform01(splitmix64(word ^ 0x94D0CA12))
    return math.sqrt(-2.0 * math.log1p(-u1)) * math.cos(2.0 * math.pi * u2)


def _pauli(n: int, letters: dict) -> str:
    s = ["I"] * n
    for q, ch in letters.items():
        s[q] = ch
    return "".join(s)


Terms = List[Tuple[float, str]]


def heisenberg_chain(n: int, jxy: float, jz: float, seed: int, periodic: bool = True) -> Terms:
    """J_xy (X_i X_{i+1} + Y_i Y_{i+1}) + J_z Z_i Z_{i+1} bond-major, then
    h_i Z_i with h_i ~ U[-1,1] (configs 1 and 4)."""
    terms: Terms = []
    nb = n if periodic else n - 1
    for i in range(nb):
        j = (i + 1) % n
        terms.append((jxy, _pauli(n, {i: "X", j: "X"})))
        terms.append((jxy, _pauli(n, {i: "Y", j: "Y"})))
        terms.append((jz, _pauli(n, {i: "Z", j: "Z"})))
    for i in range(n):
        terms.append((uniform_pm1(rng_hash(seed, TAG_FIELD, i)), _pauli(n, {i: "Z"})))
    return terms


def tfim_2d(rows: int, cols: int, j: float, g: float) -> Terms:
    """-J Z_i Z_j on nearest neighbours of an open rows x cols lattice
    (row-major sites, each site's right bond then down bond), then -g X_i
    (config 2)."""
    n = rows * cols
    terms: Terms = []
    for r in range(rows):
        for c in range(cols):
            q = r * cols + c
            if c + 1 < cols:
                terms.append((-j, _pauli(n, {q: "Z", q + 1: "Z"})))
            if r + 1 < rows:
                terms.append((-j, _pauli(n, {q: "Z", q + cols: "Z"})))
    for q in range(n):
        terms.append((-g, _pauli(n, {q: "X"})))
    return terms


def random_k_local(n: int, m: int, seed: int, kmax: int = 4) -> Terms:
    """m distinct strings: weight w ~ U{1..kmax}, w qubits without
    replacement (partial Fisher-Yates), letters uniform over {X,Y,Z},
    c ~ N(0,1); draws that repeat an earlier string are skipped (config 3)."""
    seen = set()
    terms: Terms = []
    d = 0
    while len(terms) < m:
        w = 1 + rng_hash(seed, TAG_KW, d) % kmax
        pool = list(range(n))
        letters = {}
        for k in range(w):
            r = k + rng_hash(seed, TAG_KQ, d, k) % (n - k)
            pool[k], pool[r] = pool[r], pool[k]
            letters[pool[k]] = "XYZ"[rng_hash(seed, TAG_KP, d, k) % 3]
        s = _pauli(n, letters)
        if s not in seen:
            seen.add(s)
            terms.append((gaussian(rng_hash(seed, TAG_KC, d)), s))
        d += 1
    return terms


def _two_distinct(n: int, seed: int, tag: int, d: int) -> Tuple[int, int]:
    a = rng_hash(seed, tag, d, 0) % n
    b = rng_hash(seed, tag, d, 1) % (n - 1)
    if b >= a:
        b += 1
    return (a, b) if a < b else (b, a)


def jordan_wigner(n: int, n_hop: int, n_double: int, sigma: float, seed: int) -> Terms:
    """Synthetic JW-style fermionic Hamiltonian (config 5): n Z_p, all
    Z_p Z_q (p<q), n_hop hopping strings X_p Z..Z X_q or Y_p Z..Z Y_q over
    random p<q, n_double weight-4 double excitations on 4 random qubits
    a<b<c<d with letters uniform over {X,Y} and Z-chains strictly inside
    (a,b) and (c,d). Coefficients ~ N(0, sigma) (sigma is the std dev).
    Duplicates merge in Hamiltonian::from_terms."""
    terms: Terms = []
    for p in range(n):
        terms.append((sigma * gaussian(rng_hash(seed, TAG_JW_Z, p)), _pauli(n, {p: "Z"})))
    for p in range(n):
        for q in range(p + 1, n):
            terms.append((sigma * gaussian(rng_hash(seed, TAG_JW_ZZ, p, q)), _pauli(n, {p: "Z", q: "Z"})))
    for d in range(n_hop):
        p, q = _two_distinct(n, seed, TAG_JW_HOP, d)
        ch = "XY"[rng_hash(seed, TAG_JW_HOP, d, 2) & 1]
        letters = {k: "Z" for k in range(p + 1, q)}
        letters[p] = ch
        letters[q] = ch
        terms.append((sigma * gaussian(rng_hash(seed, TAG_JW_HOPC, d)), _pauli(n, letters)))
    for d in range(n_double):
        pool = list(range(n))
        for k in range(4):
            r = k + rng_hash(seed, TAG_JW_DBL, d, k) % (n - k)
            pool[k], pool[r] = pool[r], pool[k]
        a, b, c, e = sorted(pool[:4])
        letters = {k: "Z" for k in list(range(a + 1, b)) + list(range(c + 1, e))}
        for k, q in enumerate((a, b, c, e)):
            letters[q] = "XY"[rng_hash(seed, TAG_JW_DBL, d, 4 + k) & 1]
        terms.append((sigma * gaussian(rng_hash(seed, TAG_JW_DBLC, d)), _pauli(n, letters)))
    return terms


def to_text(terms: Terms) -> str:
    """Hamiltonian::save format: `%.17g <pauli>` per line."""
    return "".join(f"{c:.17g} {p}\n" for c, p in terms)


# --------------------------------------------------------------- configs

def neel_index(n: int) -> int:
    """|0101...> with qubit 0 leftmost: odd qubits set."""
    return sum(1 << q for q in range(1, n, 2))


CONFIGS = {
    1: dict(name="heisenberg_xxx_n16", n=16, order=1, dt=0.01, steps=100, init=("basis", "neel")),
    2: dict(name="tfim2d_5x5", n=25, order=2, dt=0.02, steps=500, init=("plus",)),
    3: dict(name="random_klocal_n28_m2000", n=28, order=1, dt=0.005, steps=200, init=("random", 2)),
    4: dict(name="heisenberg_xxz_n30", n=30, order=1, dt=0.01, steps=1000, init=("basis", "neel")),
    5: dict(name="jordan_wigner_n33", n=33, order=1, dt=0.01, steps=50, init=("basis", 0xFFFF)),
}


def config_terms(cfg: int, n: int = None) -> Terms:
    """Terms of BASELINE config `cfg`; `n` overrides the qubit count for
    reduced-size parity runs of the same generator."""
    nn = n if n is not None else CONFIGS[cfg]["n"]
    if cfg == 1:
        return heisenberg_chain(nn, 1.0, 1.0, seed=0)
    if cfg == 2:
        if n is None:
            return tfim_2d(5, 5, 1.0, 1.5)
        rows = max(1, int(round(math.sqrt(nn))))
        return tfim_2d(rows, nn // rows, 1.0, 1.5)
    if cfg == 3:
        return random_k_local(nn, 2000 if n is None else min(2000, 40 * nn), seed=1)
    if cfg == 4:
        return heisenberg_chain(nn, 1.0, 0.5, seed=3)
    if cfg == 5:
        return jordan_wigner(nn, 4000, 4000, 0.1, seed=4)
    raise ValueError(f"unknown config {cfg}")


def config_text(cfg: int, n: int = None) -> str:
    return to_text(config_terms(cfg, n))


def initial_index(cfg: int, n: int) -> int:
    init = CONFIGS[cfg]["init"]
    if init[0] != "basis":
        raise ValueError("config does not start from a basis state")
    if init[1] == "neel":
        return neel_index(n)
    return init[1] & ((1 << n) - 1)
