"""Scratch: transposes whose destination-contiguous run is short (32 or 64 rows per tile): the staged plan with 4-8 KiB tiles."""
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


M = 2 ** 22
dts = {2: torch.int16, 4: torch.int32, 8: torch.int64}
for nn, eb in ((32, 4), (64, 4), (96, 4), (64, 2), (128, 2), (48, 4), (16, 8)):
    for rev in (False, True):
        sl, dl = f"({M},{nn}):({nn},1)", f"({M},{nn}):(1,{M})"
        if rev:
            sl, dl = dl, sl
        n = M * nn
        src = torch.arange(n, dtype=torch.int64, device="cuda").to(dts[eb])
        dst = torch.zeros_like(src)
        a, b = host.tensor_of(sl, src), host.tensor_of(dl, dst)
        sec = t(lambda: host.copy(a, b))
        print(f"{M} x {nn} eb={eb} {'planar -> interleaved' if rev else 'interleaved -> planar'}: {lib.tlb_last_plan().decode()} {2 * n * eb / sec / 1e9:.0f} GB/s")
        del src, dst
