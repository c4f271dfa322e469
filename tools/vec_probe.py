"""Scratch: times the `vec` copy plan (one mode contiguous on both sides) against torch copy_."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_02298_b200 import abi, host
lib = abi.load()
def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e-3
n = 2 ** 30
src = torch.arange(n, dtype=torch.int32, device="cuda")
dst = torch.empty(n, dtype=torch.int32, device="cuda")
s = t(lambda: dst.copy_(src))
print(f"torch copy_ 4 GiB: {2*n*4/s/1e9:.0f} GB/s")
cases = [(f"{n}:1", f"{n}:1", "contiguous"),
         (f"(1024,1024,1024):(1,1024,1048576)", f"(1024,1024,1024):(1,1048576,1024)", "swap of the two outer modes (4 KiB rows)"),
         (f"(64,4096,4096):(1,64,262144)", f"(64,4096,4096):(1,262144,64)", "swap of the two outer modes (256 B rows)")]
for sl, dl, name in cases:
    a = host.tensor_of(sl, src)
    b = host.tensor_of(dl, dst)
    s = t(lambda: host.copy(a, b))
    print(f"{name:48s} plan {lib.tlb_last_plan().decode():6s}: {s*1e6:8.1f} us  {2*n*4/s/1e9:.0f} GB/s")
