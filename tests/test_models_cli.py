"""the paper's benchmark models (gen_tfim / gen_syk,
proj/src/models.cpp:17-92), first-fit grouping at SYK scale
(proj/src/hamiltonian.cpp:135-158) and the SPEC command line
(SPEC.md `cli`; the reference ships only a placeholder, proj/tools/main.cpp).

Every host-side result is compared with the reference compiled from its own
sources (oracle/_ref): generated Hamiltonians byte-for-byte through
Hamiltonian::save, groupings term-for-term, the diag document value-for-value.
"""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2206_11664_b200", "lib", "simdiag")


@pytest.mark.parametrize("model,n,seed", [("tfim", 2, 0), ("tfim", 11, 3), ("tfim", 30, 7), ("syk", 2, 1),
                                          ("syk", 7, 9), ("syk", 12, 5)])
def test_generators_match_reference(model, n, seed, sd, ref):
    text, info = ref.gen_text(model, n, seed)
    if model == "tfim":
        h = sd.gen_tfim(n, seed)
    else:
        h, mine = sd.gen_syk(n, seed, with_info=True)
        assert mine == info
    assert h.save() == text


def test_generator_errors(sd):
    with pytest.raises(ValueError, match="tfim requires"):
        sd.gen_tfim(1, 0)
    with pytest.raises(ValueError, match="syk requires"):
        sd.gen_syk(65, 0)


def _ref_groups(ref, text):
    h, _, groups = ref.partition_text(text, synthesize=False)
    ref.free(h)
    return [(g.src_x, g.src_z) for g in groups]


def _our_groups(sd, text):
    return [([t.pauli.x_mask for t in g.terms], [t.pauli.z_mask for t in g.terms])
            for g in sd.greedy_partition(sd.Hamiltonian.load(text))]


@pytest.mark.parametrize("n,seed", [(6, 0), (10, 2), (14, 5), (20, 5)])
def test_syk_grouping_matches_reference(n, seed, sd, ref):
    text, _ = ref.gen_text("syk", n, seed)
    assert _our_groups(sd, text) == _ref_groups(ref, text)


def test_tfim_grouping_kat(sd):
    """proj/tests/test_hamiltonian.cpp:149-164: TFIM at n=30 gives 2 groups, 465 terms."""
    groups = sd.greedy_partition(sd.gen_tfim(30, 1))
    assert len(groups) == 2
    assert sum(len(g.terms) for g in groups) == 465
    assert [len(g.terms) for g in groups] == [435, 30]


def test_grouping_matches_reference_on_dense_random_hamiltonians(sd, ref):
    """Random Paulis with many identity/commuting collisions: groups whose
    spans saturate, identity terms, repeated basis vectors."""
    rng = np.random.default_rng(11)
    for trial in range(20):
        n = int(rng.integers(2, 9))
        m = int(rng.integers(1, 120))
        letters = "IXYZ" if trial % 2 else "IIIZZX"
        lines = []
        for _ in range(m):
            p = "".join(letters[int(v)] for v in rng.integers(0, len(letters), n))
            lines.append(f"{rng.normal():.17g} {p}\n")
        text = "".join(lines)
        assert _our_groups(sd, text) == _ref_groups(ref, text), trial


def _run(*args, check=True):
    r = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stderr
    return r


def test_cli_gen_partition_diag_match_reference(tmp_path, sd, ref):
    for model, n, seed in [("tfim", 9, 4), ("syk", 6, 2)]:
        f = tmp_path / f"{model}.txt"
        _run("gen", "--model", model, "--qubits", str(n), "--seed", str(seed), "--out", str(f))
        text, _ = ref.gen_text(model, n, seed)
        assert f.read_text() == text
        out = _run("partition", str(f), "--out", str(tmp_path / "assign.txt")).stdout
        want = _ref_groups(ref, text)
        assert f"n_g={len(want)}" in out
        assign = [int(line.split()[1]) for line in (tmp_path / "assign.txt").read_text().splitlines()]
        xz = sd.Hamiltonian.load(text).term_arrays()
        for k, g in enumerate(assign):
            assert int(xz[0][k]) in want[g][0]
        js = _run("diag", str(f)).stdout.strip()
        h, _, _ = ref.partition_text(text)
        # value-identical (every double parses to the same bits); nlohmann's
        # Grisu2 does not always print the shortest round-trip form
        assert json.loads(js) == json.loads(ref.diag_json(h))
        ref.free(h)


def test_cli_exit_codes(tmp_path):
    assert _run("partition", str(tmp_path / "missing.txt"), check=False).returncode == 2
    empty = tmp_path / "empty.txt"
    empty.write_text("")
    assert _run("partition", str(empty), check=False).returncode == 2
    bad = tmp_path / "bad.txt"
    bad.write_text("1.0 XQ\n")
    r = _run("diag", str(bad), check=False)
    assert r.returncode == 2 and "line 1" in r.stderr
    assert _run("gen", "--model", "nope", "--qubits", "3", check=False).returncode == 2
    assert _run("frobnicate", check=False).returncode == 2


@pytest.mark.gpu
def test_cli_run_verify_bench(tmp_path):
    f = tmp_path / "syk.txt"
    _run("gen", "--model", "syk", "--qubits", "8", "--seed", "3", "--out", str(f))
    csv = tmp_path / "trace.csv"
    r = _run("run", str(f), "--t", "0.2", "--steps", "20", "--init", "random:4", "--csv", str(csv), "--verify")
    assert "fidelity deficit" in r.stderr
    rows = csv.read_text().splitlines()
    assert rows[0] == "step,time,energy" and len(rows) == 22
    e = [float(x.split(",")[2]) for x in rows[1:]]
    assert max(e) - min(e) < 1e-3  # energy is conserved up to Trotter error
    r = _run("verify", str(f), "--t", "0.1", "--steps", "5")
    assert "exact_evolve" in r.stdout
    r = _run("bench", "--model", "tfim", "--qubits", "10:11", "--repeats", "3")
    lines = r.stdout.strip().splitlines()
    assert lines[0].startswith("model,n_qubits,m,n_g,method")
    assert len(lines) == 5 and all(float(x.split(",")[6]) > 0 for x in lines[1:])
