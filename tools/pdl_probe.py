"""Scratch: cost of programmatic dependent launch when the GEMM follows other kinds of stream work."""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_02298_b200 import abi, host
M = 4096
a = torch.empty(M * M, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
b = torch.empty(M * M, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
c = torch.zeros(M * M, dtype=torch.float32, device="cuda")
ta = host.tensor_of(f"({M},{M}):({M},1)", a.view(torch.int16), ranked=True)
tb = host.tensor_of(f"({M},{M}):({M},1)", b.view(torch.int16), ranked=True)
tc = host.tensor_of(f"({M},{M}):(1,{M})", c, ranked=True)
x = torch.zeros(1 << 20, device="cuda")
y = torch.zeros(1 << 26, dtype=torch.uint8, device="cuda")
z = torch.zeros(1 << 26, dtype=torch.uint8, device="cuda")
hp = torch.zeros(1 << 26, dtype=torch.uint8).pin_memory()
def run(name, pre):
    for _ in range(3):
        pre(); host.gemm_bf16(ta, tb, tc)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        pre(); host.gemm_bf16(ta, tb, tc)
    torch.cuda.synchronize()
    print(f"{name:32s}: {(time.perf_counter()-t0)/20*1e3:.3f} ms per (pre + gemm)")
run("gemm only", lambda: None)
run("small torch kernel + gemm", lambda: x.add_(1))
run("D2D memcpy 64 MiB + gemm", lambda: z.copy_(y))
run("H2D memcpy 64 MiB + gemm", lambda: y.copy_(hp, non_blocking=True))
