"""Scratch: throughput of the thread-value partitioned copy (tlb_copy_tv with the library-derived TV layout) against tlb_copy on
the same layouts: a contiguous 1 GiB fp32 copy (V = 4), the C1 transpose (V = 1) and a row-padded copy."""
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


cases = [("contiguous 2^28 fp32", "(16384,16384):(1,16384)", "(16384,16384):(1,16384)", 2 ** 28),
         ("C1 transpose", "(8192,8192):(8192,1)", "(8192,8192):(1,8192)", 2 ** 26),
         ("padded rows", "(4096,16384):(1,4100)", "(4096,16384):(1,4096)", 4100 * 16384)]
for name, sl, dl, cap in cases:
    src = torch.arange(cap, dtype=torch.int32, device="cuda")
    dst = torch.zeros(cap, dtype=torch.int32, device="cuda")
    a, b = host.tensor_of(sl, src), host.tensor_of(dl, dst)
    n = host.L(sl).size
    s0 = t(lambda: host.copy(a, b), 10)
    p0 = lib.tlb_last_plan().decode()
    ref = dst.clone()
    for threads in (256, 1024, 65536):
        tv = host.copy_tv_auto(sl, dl, 4, threads)
        dst.zero_()
        s1 = t(lambda: host.copy_tv(a, b, tv), 10)
        print(f"{name}: tlb_copy {p0} {2*n*4/s0/1e9:.0f} GB/s | tv {tv} plan {lib.tlb_last_plan().decode()} {2*n*4/s1/1e9:.0f} GB/s equal={torch.equal(dst, ref)}")
    del src, dst, ref
