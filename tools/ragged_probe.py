"""Scratch: transposes / permutes with ragged extents: the gather plan (COPY_RAGGED=0) against the whole-tile body + edge strips."""
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


cases = [("(8000,6000):(6000,1)", "(8000,6000):(1,8000)", 4, torch.int32), ("(8001,6001):(6001,1)", "(8001,6001):(1,8001)", 4, torch.int32),
         ("(8000,6000):(6000,1)", "(8000,6000):(1,8000)", 2, torch.int16), ("(1000,1000):(1000,1)", "(1000,1000):(1,1000)", 4, torch.int32),
         ("(300,300,300):(1,300,90000)", "(300,300,300):(90000,300,1)", 4, torch.int32)]
for sl, dl, eb, dt in cases:
    n = host.L(sl).size
    src = torch.arange(n, dtype=dt, device="cuda")
    dst = torch.zeros(n, dtype=dt, device="cuda")
    a, b = host.tensor_of(sl, src), host.tensor_of(dl, dst)
    out = []
    for r in ("0", "22"):
        host.config("COPY_RAGGED", r)
        sec = t(lambda: host.copy(a, b))
        out.append(f"{lib.tlb_last_plan().decode()} {2 * n * eb / sec / 1e9:.0f} GB/s ({sec * 1e6:.0f} us)")
    host.config("COPY_RAGGED", None)
    print(f"eb={eb} {sl} -> {dl}: " + " | ".join(out))
