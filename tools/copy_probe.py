"""Scratch: times tlb_copy on the C1 (8192^2 fp32 transpose) and C3 (4 GiB hierarchical permute) layouts."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_02298_b200 import abi, host
lib = abi.load()

def t(fn, n):
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

which = sys.argv[1:] or ["c1", "c3"]
if "c1" in which:
    n = 8192
    src = torch.arange(n * n, dtype=torch.int32, device="cuda")
    dst = torch.empty(n * n, dtype=torch.int32, device="cuda")
    a = host.tensor_of(f"({n},{n}):({n},1)", src)
    b = host.tensor_of(f"({n},{n}):(1,{n})", dst)
    s = t(lambda: host.copy(a, b), 50)
    ok = torch.equal(dst.view(n, n), src.view(n, n).t())
    print(f"C1 plan {lib.tlb_last_plan().decode()}: {s*1e6:.1f} us  {2*n*n*4/s/1e9:.0f} GB/s  correct={ok}")
    del src, dst
if "c3" in which:
    T = 4096
    sl = f"((8,128),(4,64),{T}):((1,2048),(8,32),262144)"
    dl = f"((8,128),(4,64),{T}):((128,1),(65536,1024),262144)"
    src = torch.arange(262144 * T, dtype=torch.int32, device="cuda")
    dst = torch.empty(262144 * T, dtype=torch.int32, device="cuda")
    a = host.tensor_of(sl, src)
    b = host.tensor_of(dl, dst)
    s = t(lambda: host.copy(a, b), 10)
    print(f"C3 plan {lib.tlb_last_plan().decode()}: {s*1e6:.1f} us  {2*262144*T*4/s/1e9:.0f} GB/s")
