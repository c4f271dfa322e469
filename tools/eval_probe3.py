"""Scratch: tlb_eval_range on layouts whose extents are not powers of two (64-bit multiply-shift division in the peel) and with an Xor leaf."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_02298_b200 import abi, host
lib = abi.load()
chunk = 2 ** 27
buf = torch.empty(chunk, dtype=torch.int64, device="cuda")
for name, Lt, i_max in (("pow2 (C5)", "((128,64),(512,1024)):((65536,1),(8388608,64))", 2 ** 32), ("1000^3 reversed", "(1000,1000,1000):(1000000,1000,1)", 10 ** 9),
                        ("(96,17,3,2^20)", "(96,17,3,1048576):(1,96,1632,4896)", 96 * 17 * 3 * 2 ** 20), ("1000^3 beyond 2^32 offsets", "(1000,1000,1000):(7000000,7000,7)", 10 ** 9),
                        ("swizzled rows", "(128,8,1048576):(f1,f144,f1024)", 2 ** 30), ("leaf 0 = 3 cells", "(3,1048576,64):(1,3,3145728)", 3 * 2 ** 26)):
    nchunks = max(1, min(8, i_max // chunk))
    for i in range(2):
        host.eval_range(Lt, i % nchunks * chunk, chunk, buf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(8):
        host.eval_range(Lt, (i % nchunks) * chunk, chunk, buf)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) / 8 * 1e-3
    print(f"{name}: plan {lib.tlb_last_plan().decode()} {chunk * 8 / s / 1e9:.0f} GB/s")
