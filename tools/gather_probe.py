"""Scratch: old two-evaluation gather (forced, path 1) vs the joint gather fallback on layouts with no vec / tiled plan."""
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
cases = [("(4096,4096):(4097,1)", "(4096,4096):(1,4096)", 2), ("(4096,4096):(4097,1)", "(4096,4096):(1,4096)", 1),
         ("((4,16),(32,4),4096):((1,512),(4,128),2048)", "((4,16),(32,4),4096):((2048,1),(16,512),8192)", 4)]
for sl, dl, eb in cases:
    ls, ld = host.L(sl), host.L(dl)
    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[eb]
    src = torch.zeros(ls.cosize, dtype=dt, device="cuda")
    dst = torch.zeros(ld.cosize, dtype=dt, device="cuda")
    a, b = host.tensor_of(ls, src), host.tensor_of(ld, dst)
    for path in (1, 0):
        lib.tlb_copy_set_path(path)
        s = t(lambda: host.copy(a, b))
        lib.tlb_copy_set_path(0)
        print(f"eb={eb} path={path} plan={lib.tlb_last_plan().decode():7s} {2*ls.size*eb/s/1e9:8.0f} GB/s   {sl[:40]}")
