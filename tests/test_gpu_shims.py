"""ranklab::mm and ranklab::trsm -- the reference's declared substitution seam
(kernels.hpp:13-38) -- on the GPU through the C++ shim
(paper_1112_5717_b200/shim/ranklab_kernels_gpu.cpp): bodies and exact OpCounter
charges equal the reference's own kernels (compiled from kernels.cpp with the
definitions renamed) for mm with every alpha/beta kind and all 8 trsm variants
at several thresholds, on strided views (oracle/shim_check.cpp `parity`)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_check")


@pytest.mark.skipif(not os.path.exists(BIN), reason="shim_check not built (needs /root/reference)")
def test_mm_trsm_shims_equal_reference_kernels():
    out = subprocess.run([BIN, "parity"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "parity: 0 failures" in out.stdout
