"""Known-answer tests restated from the reference's own test suite, run
against all three implementations of the host path:
  product : paper_2206_11664_b200 (C++ host library over the C ABI)
  port    : oracle/simdiag_oracle.c (the CPU restatement -- pinning it)
  ref     : the reference compiled from its sources (oracle/_ref)
Sources: proj/tests/test_diagonalize.cpp:28-109,243-248,
proj/tests/test_tableau.cpp:164-183, proj/tests/test_hamiltonian.cpp:14-99,149-164.
"""
import pytest

from paper_2206_11664_b200 import models as M

WORKED = ["YIXI", "IXIY", "XZYZ", "YZXZ", "XIYI", "IYIX", "ZXZY", "ZYZX"]


def masks(texts):
    xs, zs = [], []
    for t in texts:
        x = z = 0
        for q, ch in enumerate(t):
            if ch in "XY":
                x |= 1 << q
            if ch in "ZY":
                z |= 1 << q
        xs.append(x)
        zs.append(z)
    return xs, zs


def diag_with(impl, sd, port, ref, texts, coeff=1.0):
    n = len(texts[0])
    xs, zs = masks(texts)
    cs = [coeff] * len(texts)
    if impl == "product":
        terms = [sd.WeightedTerm(c, sd.PauliString(n, x, z)) for x, z, c in zip(xs, zs, cs)]
        d = sd.diagonalize_group(terms)
        c = d.circuit
        return dict(h_pre=c.h_pre, cnots=c.cnots, czs=c.czs, s=c.s_layer, h_post=c.h_post, z=d.z_masks,
                    c=d.signed_coeffs)
    o = (port if impl == "port" else ref).diagonalize(n, xs, zs, cs)
    return dict(h_pre=o.h_pre, cnots=o.cnots, czs=o.czs, s=o.s_layer, h_post=o.h_post, z=o.z_masks, c=o.coeffs)


IMPLS = ["product", "port", "ref"]


@pytest.mark.parametrize("impl", IMPLS)
def test_worked_example_circuit_and_signed_diagonal(impl, sd, port, request):
    ref = request.getfixturevalue("ref") if impl == "ref" else None
    d = diag_with(impl, sd, port, ref, WORKED)
    assert d["h_pre"] == [2, 3]
    assert d["cnots"] == [(1, 3), (2, 3)]
    assert d["czs"] == [(0, 2), (1, 2), (1, 3)]
    assert d["s"] == [0, 1]
    assert d["h_post"] == [0, 1, 2, 3]
    assert d["z"] == [0b0001, 0b0010, 0b0101, 0b1001, 0b1101, 0b1010, 0b1110, 0b0110]
    assert d["c"] == [-1, 1, -1, -1, -1, 1, 1, 1]


@pytest.mark.parametrize("impl", IMPLS)
def test_identity_and_x_only_groups(impl, sd, port, request):
    ref = request.getfixturevalue("ref") if impl == "ref" else None
    d = diag_with(impl, sd, port, ref, ["ZZII", "IZZI", "ZIIZ", "IIZZ"], 0.5)
    assert d["h_pre"] == d["cnots"] == d["czs"] == d["s"] == d["h_post"] == []
    assert d["z"] == masks(["ZZII", "IZZI", "ZIIZ", "IIZZ"])[1]
    assert d["c"] == [0.5] * 4
    d = diag_with(impl, sd, port, ref, ["XIII", "IXII", "IIXI", "IIIX"])
    assert d["h_post"] == [0, 1, 2, 3] and d["h_pre"] == [] and d["cnots"] == []
    d = diag_with(impl, sd, port, ref, ["X"], 0.7)
    assert d["h_post"] == [0] and d["z"] == [1] and d["c"] == [0.7]


@pytest.mark.parametrize("impl", IMPLS)
def test_non_commuting_group_raises_runtime_error(impl, sd, port, request):
    ref = request.getfixturevalue("ref") if impl == "ref" else None
    with pytest.raises(RuntimeError):
        diag_with(impl, sd, port, ref, ["XX", "ZI"])


def test_appendix_independent_subset_port(port):
    terms = ["ZYXI", "ZXYI", "IYXZ", "IXYZ", "YIZX", "YZIX", "XIZY", "XZIY"]
    xs, zs = masks(terms)
    idx = port.independent_subset(4, xs, zs)
    assert [terms[i] for i in idx] == ["YIZX", "ZXYI", "IYXZ", "IXYZ"]
    assert port.independent_subset(2, *masks(["ZZ", "ZZ"])) == [0]
    assert port.independent_subset(2, *masks(["ZI", "IZ", "ZZ"])) == [0, 1]
    assert port.independent_subset(4, *masks(WORKED)) == [0, 1, 2, 3]


def gen_tfim(n, seed):
    """Restatement of gen_tfim (proj/src/models.cpp:17-35) for the TFIM KATs."""
    terms = []
    for i in range(n):
        for j in range(i + 1, n):
            terms.append((M.uniform_pm1(M.rng_hash(seed, 0x7A7A, i, j)), "".join("Z" if q in (i, j) else "I" for q in range(n))))
    for i in range(n):
        terms.append((M.uniform_pm1(M.rng_hash(seed, 0x7878, i)), "".join("X" if q == i else "I" for q in range(n))))
    return terms


def test_tfim_partition_kats_product(sd):
    h = sd.Hamiltonian.from_terms(8, gen_tfim(8, 42))
    g = sd.greedy_partition(h)
    assert [len(x.terms) for x in g] == [28, 8]
    h = sd.Hamiltonian.from_terms(30, gen_tfim(30, 1))
    assert h.term_count() == 465
    g = sd.greedy_partition(h)
    assert len(g) == 2 and max(len(x.terms) for x in g) == 435


def test_tfim_partition_kats_port(port):
    for n, seed, sizes in ((8, 42, [28, 8]), (30, 1, [435, 30])):
        t = gen_tfim(n, seed)
        x, z, c = port.from_terms(*masks([p for _, p in t]), [c for c, _ in t])
        gid = port.greedy_partition(x, z)
        assert [gid.count(k) for k in range(max(gid) + 1)] == sizes


def test_worked_group_stays_whole(sd, port):
    text = "".join(f"1 {t}\n" for t in WORKED)
    assert [len(g.terms) for g in sd.greedy_partition(sd.Hamiltonian.load(text))] == [8]
    n, x, z, c = port.load(text)
    assert port.greedy_partition(x, z) == [0] * 8


def test_load_merges_drops_and_keeps_first_seen_order(sd, port):
    h = sd.Hamiltonian.load("1.0 XX\n2.0 ZZ\n0.25 XX\n-1.0 YY\n")
    t = h.terms()
    assert [p.pauli.str() for p in t] == ["XX", "ZZ", "YY"] and t[0].coeff == 1.25
    h = sd.Hamiltonian.load("1.0 ZI\n0.5 ZI\n0.0 XX\n")
    assert h.term_count() == 1 and h.terms()[0].coeff == 1.5
    n, x, z, c = port.load("1.0 XX\n2.0 ZZ\n0.25 XX\n-1.0 YY\n")
    assert c == [1.25, 2.0, -1.0]


def test_load_errors_name_the_line(sd):
    with pytest.raises(ValueError, match="line 2"):
        sd.Hamiltonian.load("0.5 ZZ\nnope ZZ\n")
    with pytest.raises(ValueError, match="line 2"):
        sd.Hamiltonian.load("0.5 ZZ\n0.5 ZZZ\n")
    with pytest.raises(ValueError):
        sd.Hamiltonian.load("0.5 ZA\n")
    with pytest.raises(ValueError, match="no terms"):
        sd.Hamiltonian.load("# empty\n")
    with pytest.raises(ValueError, match="position 2"):
        sd.PauliString.parse("XQZ")


def test_save_load_round_trip(sd):
    text = M.config_text(3, n=10)
    h = sd.Hamiltonian.load(text)
    h2 = sd.Hamiltonian.load(h.save())
    assert [(t.coeff, t.pauli) for t in h.terms()] == [(t.coeff, t.pauli) for t in h2.terms()]


def test_save_matches_reference_save(sd, ref):
    for cfg in (1, 3, 5):
        text = M.config_text(cfg)
        assert sd.Hamiltonian.load(text).save() == ref.load_save(text)
