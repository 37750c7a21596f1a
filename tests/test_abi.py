"""The C ABI boundary (include/simdiag_c.h) -- CPU only, no compute calls.

Every function the header declares must be exported by the product library
and bound by the Python mirror (paper_2206_11664_b200/_capi.py)."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "simdiag_c.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:sd_status|void|const char\*)\s+(sd_\w+)\s*\(", text, flags=re.M)
    assert len(names) > 60
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    import paper_2206_11664_b200._capi as A
    out = subprocess.run(["nm", "-D", "--defined-only", A.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_python_mirror_binds_every_declared_symbol():
    import paper_2206_11664_b200._capi as A
    missing = [n for n in declared() if n not in A.EXPORTED or not hasattr(A, n)]
    assert not missing, missing


def test_errors_map_to_reference_exceptions():
    """Status codes -> the reference's exception types, without a GPU."""
    import pytest

    import paper_2206_11664_b200 as S
    with pytest.raises(ValueError, match="invalid pauli character"):
        S.Hamiltonian.load("1.0 XQ\n")
    with pytest.raises(ValueError):
        S.PauliString.parse("XYZ", 2)
