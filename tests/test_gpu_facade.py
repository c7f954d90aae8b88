"""GPU: the reference's own operators vs the C++ drop-in layer (integration/), one process.

integration/_build/vsr_b200_parity links the UNMODIFIED reference objects (oracle/_ref) and
vsr::b200 (libfvsr_b200.so) and checks plan bit-exactness, exec tolerance, the row-range
contract, the sparsity report and the exception taxonomy (see integration/parity_main.cpp).
It is built in the build container (needs the reference headers) and travels with the repo.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "integration", "_build", "vsr_b200_parity")


def test_reference_vs_dropin():
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/vsr_b200_parity not built (needs the reference tree at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK: 0 failure(s)" in r.stdout
