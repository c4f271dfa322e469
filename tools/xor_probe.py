"""Scratch: gather over swizzled (Xor) destinations: 16-byte vectors per evaluation (COPY_GATHER_RUN=0) against 32 / 64-byte
runs with 256-bit accesses, on the bench's Cx_xor_dst layouts (2^26 cells) for several cell sizes."""
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


flat, sw = "(128,8,65536):(1,128,1024)", "(128,8,65536):(f1,f144,f1024)"
for eb, dt in ((2, torch.int16), (4, torch.int32), (8, torch.int64)):
    n = host.L(flat).size
    src = torch.arange(n, dtype=dt, device="cuda")
    dst = torch.zeros(n, dtype=dt, device="cuda")
    for s_, d_ in ((flat, sw), (sw, flat), (sw, sw)):
        a, b = host.tensor_of(s_, src), host.tensor_of(d_, dst)
        out = []
        for run in ("0", "1"):
            host.config("COPY_GATHER_RUN", run)
            sec = t(lambda: host.copy(a, b))
            out.append(f"{lib.tlb_last_plan().decode()} {2 * n * eb / sec / 1e9:.0f} GB/s")
        host.config("COPY_GATHER_RUN", None)
        print(f"eb={eb} {'flat' if s_ == flat else 'xor'} -> {'flat' if d_ == flat else 'xor'}: " + " | ".join(out))
