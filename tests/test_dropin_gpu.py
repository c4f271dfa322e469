"""GPU: the C++ drop-in path. oracle/_ref/dropin_test is tests/cxx/dropin_test.cpp compiled HERE against the
unmodified reference headers + include/tla/device.hpp + libtlb.so (oracle/Makefile `dropin`); it travels to the GPU
box as a prebuilt binary. It runs the reference's own copy / gemm / eval checks (test_tensor.cpp:86-203) with the
reference computing the expected cells on the host and libtlb computing them on the device."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "dropin_test"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not BIN.exists(), reason="oracle/_ref/dropin_test was not built (no /root/reference at build time)")
def test_reference_api_runs_on_device_and_matches_the_reference():
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
