"""Scratch: interleave / de-interleave copies (AoS <-> SoA, CHW <-> HWC) and an odd-length contiguous byte copy: which plan, what rate."""
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


J = 2 ** 24
cases = [(f"(4,{J}):(1,4)", f"(4,{J}):({J},1)", 4, "AoS4 -> SoA"), (f"(4,{J}):({J},1)", f"(4,{J}):(1,4)", 4, "SoA -> AoS4"),
         (f"(3,{J}):(1,3)", f"(3,{J}):({J},1)", 4, "AoS3 -> SoA"), (f"(2,{J}):(1,2)", f"(2,{J}):({J},1)", 2, "complex bf16 split"),
         ("(224,224,3,256):(1,224,50176,150528)", "(224,224,3,256):(3,672,1,150528)", 4, "CHW -> HWC x256"),
         ("(5001,5003):(1,5001)", "(5001,5003):(1,5001)", 1, "odd contiguous bytes")]
dts = {1: torch.uint8, 2: torch.int16, 4: torch.int32}
for sl, dl, eb, what in cases:
    n = host.L(sl).size
    src = torch.arange(n, dtype=torch.int64, device="cuda").to(dts[eb])
    dst = torch.zeros(n, dtype=dts[eb], device="cuda")
    a, b = host.tensor_of(sl, src), host.tensor_of(dl, dst)
    sec = t(lambda: host.copy(a, b))
    print(f"{what}: {lib.tlb_last_plan().decode()} {2 * n * eb / sec / 1e9:.0f} GB/s ({sec * 1e6:.0f} us)")
M = 2 ** 22
for nn, eb in ((16, 4), (12, 4), (6, 4), (16, 2), (5, 8)):
    sl, dl = f"({M},{nn}):({nn},1)", f"({M},{nn}):(1,{M})"
    n = M * nn
    src = torch.arange(n, dtype=torch.int64, device="cuda").to({2: torch.int16, 4: torch.int32, 8: torch.int64}[eb])
    dst = torch.zeros_like(src)
    a, b = host.tensor_of(sl, src), host.tensor_of(dl, dst)
    sec = t(lambda: host.copy(a, b))
    ok = torch.equal(dst.view(nn, M), src.view(M, nn).t())
    print(f"tall-skinny transpose {M} x {nn} eb={eb}: {lib.tlb_last_plan().decode()} {2 * n * eb / sec / 1e9:.0f} GB/s ({sec * 1e6:.0f} us) correct={ok}")
for nn, eb in ((24, 4), (9, 4), (32, 2), (100, 1), (24, 2)):
    for rev in (False, True):
        sl, dl = f"({M},{nn}):({nn},1)", f"({M},{nn}):(1,{M})"
        if rev:
            sl, dl = dl, sl
        n = M * nn
        src = torch.arange(n, dtype=torch.int64, device="cuda").to({1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[eb])
        dst = torch.zeros_like(src)
        a, b = host.tensor_of(sl, src), host.tensor_of(dl, dst)
        out = []
        for kk in ("0", "1"):
            host.config("COPY_CELL_TILES", kk)
            sec = t(lambda: host.copy(a, b))
            out.append(f"{lib.tlb_last_plan().decode()} {2 * n * eb / sec / 1e9:.0f} GB/s")
        host.config("COPY_CELL_TILES", None)
        print(f"{M} x {nn} eb={eb} {'planar -> interleaved' if rev else 'interleaved -> planar'}: " + " | ".join(out))
