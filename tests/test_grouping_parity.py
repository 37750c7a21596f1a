"""Bit-exact grouping + Clifford synthesis parity (north star: "grouping and
Clifford circuits must be bit-identical") on every BASELINE config and on
seeded random Hamiltonians: product C++ vs the compiled reference vs the C
restatement."""
import random

import pytest

from paper_2206_11664_b200 import models as M


def as_tuple_prod(g):
    c = g.circuit
    return (c.h_pre, c.cnots, c.czs, c.s_layer, c.h_post, g.z_masks, g.signed_coeffs,
            [(t.pauli.x_mask, t.pauli.z_mask, t.coeff) for t in g.terms])


def as_tuple_or(g):
    return (g.h_pre, g.cnots, g.czs, g.s_layer, g.h_post, g.z_masks, g.coeffs,
            list(zip(g.src_x, g.src_z, g.src_c)))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_configs_bit_identical(cfg, sd, port, ref):
    text = M.config_text(cfg)
    h, n, rg = ref.partition_text(text)
    ref.free(h)
    _, pg = port.partition_and_diagonalize(text)
    sg = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
    R = [as_tuple_or(g) for g in rg]
    assert [as_tuple_or(g) for g in pg] == R
    assert [as_tuple_prod(g) for g in sg] == R


def random_text(rng, n, m):
    lines = []
    for _ in range(m):
        w = rng.randint(1, min(n, 5))
        qs = rng.sample(range(n), w)
        s = ["I"] * n
        for q in qs:
            s[q] = rng.choice("XYZ")
        c = rng.choice([1.0, -1.0, 0.5]) if rng.random() < 0.2 else rng.uniform(-1, 1)
        lines.append(f"{c!r} {''.join(s)}")
    return "\n".join(lines) + "\n"


def test_random_hamiltonians_bit_identical(sd, port, ref):
    rng = random.Random(2206)
    for trial in range(150):
        n = rng.randint(1, 12)
        m = rng.randint(1, 80)
        text = random_text(rng, n, m)
        h, _, rg = ref.partition_text(text)
        ref.free(h)
        _, pg = port.partition_and_diagonalize(text)
        sg = sd.partition_and_diagonalize(sd.Hamiltonian.load(text))
        R = [as_tuple_or(g) for g in rg]
        assert [as_tuple_or(g) for g in pg] == R, trial
        assert [as_tuple_prod(g) for g in sg] == R, trial


def test_random_commuting_groups_bit_identical(sd, port, ref):
    """Random commuting groups built as diagonal strings conjugated through a
    random Clifford word (as proj/tests/oracle.cpp:164-218 does)."""
    rng = random.Random(41)

    def conj(rows, kind, a, b):
        out = []
        for x, z, s in rows:
            bx = lambda w, q: (w >> q) & 1
            if kind == "H":
                s ^= bx(x, a) & bx(z, a)
                xa, za = bx(x, a), bx(z, a)
                x = (x & ~(1 << a)) | (za << a)
                z = (z & ~(1 << a)) | (xa << a)
            elif kind == "S":
                s ^= bx(x, a) & bx(z, a)
                z ^= bx(x, a) << a
            elif kind == "C":
                s ^= bx(x, a) & bx(z, b) & (1 if bx(x, b) == bx(z, a) else 0)
                x ^= bx(x, a) << b
                z ^= bx(z, b) << a
            else:
                s ^= bx(x, a) & bx(x, b) & (bx(z, a) ^ bx(z, b))
                xa, xb = bx(x, a), bx(x, b)
                z ^= xa << b
                z ^= xb << a
            out.append((x, z, s))
        return out

    for trial in range(200):
        n = rng.randint(2, 8)
        m = rng.randint(1, min(10, 1 << n))
        zs = rng.sample(range(1, 1 << n), min(m, (1 << n) - 1))
        rows = [(0, z, 0) for z in zs]
        for _ in range(3 * n):
            kind = rng.choice("HSCZ")
            a = rng.randrange(n)
            b = rng.randrange(n)
            while b == a:
                b = rng.randrange(n)
            rows = conj(rows, kind, a, b)
        cs = [(-1.0 if s else 1.0) * rng.uniform(-1, 1) for _, _, s in rows]
        xs = [x for x, _, _ in rows]
        zz = [z for _, z, _ in rows]
        r = ref.diagonalize(n, xs, zz, cs)
        p = port.diagonalize(n, xs, zz, cs)
        terms = [sd.WeightedTerm(c, sd.PauliString(n, x, z)) for x, z, c in zip(xs, zz, cs)]
        s = sd.diagonalize_group(terms)
        assert as_tuple_or(p) == as_tuple_or(r), trial
        assert as_tuple_prod(s)[:7] == as_tuple_or(r)[:7], trial
