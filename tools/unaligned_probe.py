"""Scratch: transposes whose bases / leading dimensions are not multiples of 16 bytes (tiled_u): vector-shaped lanes with cell-sized
accesses (COPY_CELL_TILES=0) against consecutive lanes on consecutive cells."""
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


cases = [("(8192,8192):(8193,1)", "(8192,8192):(1,8192)", 4), ("(8192,8192):(8193,1)", "(8192,8192):(1,8193)", 2), ("(8192,8192):(8193,1)", "(8192,8192):(1,8193)", 8),
         ("(8001,6001):(6001,1)", "(8001,6001):(1,8001)", 4), ("(8001,6001):(6001,1)", "(8001,6001):(1,8001)", 2)]
dts = {2: torch.int16, 4: torch.int32, 8: torch.int64}
for sl, dl, eb in cases:
    n = host.L(sl).size
    src = torch.arange(host.L(sl).cosize, dtype=torch.int64, device="cuda").to(dts[eb])
    dst = torch.zeros(host.L(dl).cosize, dtype=dts[eb], device="cuda")
    a, b = host.tensor_of(sl, src), host.tensor_of(dl, dst)
    out = []
    for k in ("0", "1"):
        host.config("COPY_CELL_TILES", k)
        sec = t(lambda: host.copy(a, b))
        out.append(f"{lib.tlb_last_plan().decode()} {2 * n * eb / sec / 1e9:.0f} GB/s")
    host.config("COPY_CELL_TILES", None)
    print(f"eb={eb} {sl} -> {dl}: " + " | ".join(out))
