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


def test_calls_are_capturable_in_a_cuda_graph():
    """The launch path does no allocation or synchronisation (tensor maps travel as kernel parameters), so a stream of
    copy / eval / GEMM calls can be captured once and replayed: same results as eager, replay after replay."""
    import numpy as np
    import torch
    from paper_2603_02298_b200 import host
    M = 1024
    i = torch.arange(M, device="cuda").view(M, 1)
    p = torch.arange(M, device="cuda").view(1, M)
    a = ((i * 7 + p * 3 + 1) % 11).to(torch.bfloat16).contiguous()
    b = ((i * 5 + p * 2 + 2) % 13).to(torch.bfloat16).contiguous()
    at = torch.empty(M * M, dtype=torch.int16, device="cuda")             # A transposed by tlb_copy inside the graph
    c = torch.zeros(M, M, dtype=torch.float32, device="cuda")
    idx = torch.empty(M * M, dtype=torch.int64, device="cuda")
    ta = host.tensor_of(f"({M},{M}):({M},1)", a.view(-1).view(torch.int16), ranked=True)
    tb = host.tensor_of(f"({M},{M}):({M},1)", b.view(-1).view(torch.int16), ranked=True)
    tat = host.tensor_of(f"({M},{M}):(1,{M})", at, ranked=True)           # same logical A, M-major storage
    tc = host.tensor_of(f"({M},{M}):({M},1)", c.view(-1), ranked=True)
    ca, cat = host.tensor_of(f"({M},{M}):({M},1)", a.view(-1).view(torch.int16)), host.tensor_of(f"({M},{M}):(1,{M})", at)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):                                               # warm up outside the capture (attribute set-up)
            host.copy(ca, cat)
            host.gemm_bf16(tat, tb, tc)
            host.eval_range(f"({M},{M}):({M},1)", 0, M * M, idx)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    c.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        host.copy(ca, cat)                                               # A -> M-major copy (tiled plan)
        host.gemm_bf16(tat, tb, tc)                                      # NT-style operand on tcgen05, C += A B^T
        host.eval_range(f"({M},{M}):({M},1)", 0, M * M, idx)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ref = a.double() @ b.double().t()
    assert torch.equal(c.double(), 3 * ref)                              # three replays accumulated into C, exactly
    assert torch.equal(at.view(M, M), a.view(torch.int16).t().contiguous())
    ii = torch.arange(M * M, device="cuda")
    assert torch.equal(idx, (ii % M) * M + ii // M)                      # L(i) of (M,M):(M,1) over the colex index
