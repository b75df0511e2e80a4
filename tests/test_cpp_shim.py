"""The C++ cgv:: shim (the reference's API re-declared over the C ABI) passes
reference-style tests compiled against it (paper_1905_01549_b200/cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "paper_1905_01549_b200", "cpp", "cgv_shim_tests")


def test_shim_builds():
    assert os.path.exists(BIN), "run __graft_entry__.build()"


@pytest.mark.gpu
def test_shim_reference_tests_pass():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stderr
    assert "0 failures" in out.stdout


def test_shim_host_helpers():
    """csr_from_triplets / dot / norm2 of the shim (host code, no device call)."""
    if not os.path.exists(BIN):
        pytest.skip("run __graft_entry__.build()")
    out = subprocess.run([BIN, "--host"], capture_output=True, text=True, timeout=60)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stderr
    assert "0 failures" in out.stdout
