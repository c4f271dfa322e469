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


def test_cli_runs_the_hot_path_on_device(capsys):
    """python -m paper_2603_02298_b200 copy / gemm / eval: one JSON line each, plans as the parity tests see them."""
    import json
    from paper_2603_02298_b200.__main__ import main
    assert main(["copy", "(512,256):(256,1)", "(512,256):(1,512)", "--elem-bytes", "4", "--steps", "2"]) == 0
    assert json.loads(capsys.readouterr().out)["plan"] == "tiled"
    assert main(["gemm", "(512,256):(256,1)", "(256,256):(256,1)", "(512,256):(256,1)", "--steps", "2"]) == 0
    assert json.loads(capsys.readouterr().out)["plan"] == "umma_2sm"
    assert main(["eval", "(4,8):(1,4)", "--count", "32", "--steps", "1"]) == 0
    assert json.loads(capsys.readouterr().out)["first"] == [0, 1, 2, 3, 4, 5, 6, 7]
