"""The C++ drop-in shims (paper_1112_5717_b200/shim/*.cpp) rethrow every C-ABI
status as the reference's own exception subclass (errors.hpp:9-66):
DimensionMismatch, OverlapError, SingularDiagonal with the index the
reference's recursion reports (local to its base block, kernels.cpp:87-90),
SingularMatrix.  These checks run before any device work, so they need no GPU
(oracle/shim_check.cpp `errors` mode, linked like the relinked acceptance suite)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_check")


@pytest.mark.skipif(not os.path.exists(BIN), reason="shim_check not built (needs /root/reference)")
def test_shim_error_mapping():
    out = subprocess.run([BIN, "errors"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "errors: 0 failures" in out.stdout
