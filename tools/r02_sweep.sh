#!/bin/bash
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_dropin_gpu.py -m gpu -q -x 2>&1 | tail -12
python - <<'PY'
# NT (MN-major operands) at a short k-loop: 256 x 256 plan vs the wide plan
import sys, os, torch
sys.path.insert(0, '.')
from paper_2603_02298_b200 import abi, host
lib = abi.load()
M = N = 4096
for K in (2048, 4096):
    for wide in ("0", "1"):
        host.config("GEMM_WIDE", wide)
        sets = []
        for s in range(3):
            a = torch.empty(M * K, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
            b = torch.empty(N * K, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
            c = torch.zeros(M * N, dtype=torch.float32, device="cuda")
            sets.append((host.tensor_of(f"({M},{K}):(1,{M})", a.view(torch.int16), ranked=True),
                         host.tensor_of(f"({N},{K}):(1,{N})", b.view(torch.int16), ranked=True),
                         host.tensor_of(f"({M},{N}):({N},1)", c, ranked=True)))
        for i in range(3): host.gemm_bf16(*sets[i % 3])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(50): host.gemm_bf16(*sets[i % 3])
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        print(f"NT {M}x{N}x{K} GEMM_WIDE={wide} plan {lib.tlb_last_plan().decode()}: {ms*1e3:.1f} us {2*M*N*K/ms/1e9:.1f} TFLOP/s")
PY
