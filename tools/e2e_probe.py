"""Scratch: PCIe bandwidth seen by torch for pinned buffers and the time of tlb_gemm_bf16_host on the C2 shape."""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_02298_b200 import abi, host
lib = abi.load()
M = 4096
h = torch.empty(64 * 2**20, dtype=torch.uint8).pin_memory()
d = torch.empty(64 * 2**20, dtype=torch.uint8, device="cuda")
for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"torch pinned {name} 64 MiB: {dt*1e3:.2f} ms  {64*2**20/dt/1e9:.1f} GB/s")
ha = (torch.rand(M * M) * 2 - 1).to(torch.bfloat16).view(torch.int16).pin_memory()
hb = (torch.rand(M * M) * 2 - 1).to(torch.bfloat16).view(torch.int16).pin_memory()
hc = torch.zeros(M * M, dtype=torch.float32).pin_memory()
ta = host.tensor_of(f"({M},{M}):({M},1)", ha, ranked=True)
tb = host.tensor_of(f"({M},{M}):({M},1)", hb, ranked=True)
tc = host.tensor_of(f"({M},{M}):(1,{M})", hc, ranked=True)
for i in range(8):
    t0 = time.perf_counter()
    host.gemm_bf16_host(ta, tb, tc)
    print(f"tlb_gemm_bf16_host call {i}: {(time.perf_counter()-t0)*1e3:.2f} ms")
