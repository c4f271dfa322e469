"""Scratch: host-side time of one tlb_copy / tlb_gemm_bf16 / tlb_eval_range call (planning + launch, the stream never blocks the host):
a tiny problem so that the GPU is always ahead, 2000 calls."""
import sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_02298_b200 import abi, host
lib = abi.load()


def per_call(fn, n=2000):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = time.perf_counter() - t0
    torch.cuda.synchronize()
    return dt / n * 1e6


cases = [("vec 4096", "4096:1", "4096:1", 4), ("tiled 256x128", "(256,128):(128,1)", "(256,128):(1,256)", 4),
         ("C3 tile", "((8,128),(4,64),2):((1,2048),(8,32),262144)", "((8,128),(4,64),2):((128,1),(65536,1024),262144)", 4),
         ("gather 8x3", "(8,3):(1,8)", "(8,3):(3,1)", 8), ("interleave", "(4,4096):(1,4)", "(4,4096):(4096,1)", 4),
         ("xor run", "(128,8,4):(1,128,1024)", "(128,8,4):(f1,f144,f1024)", 4)]
for name, sl, dl, eb in cases:
    n = max(host.L(sl).cosize if "f" not in sl else 4096, 4096)
    src = torch.zeros(2 * n, dtype=torch.int64, device="cuda")
    dst = torch.zeros(2 * n, dtype=torch.int64, device="cuda")
    a = host.make_tensor(host.L(sl).lower(), src.data_ptr(), 2 * n * 8 // eb, eb)
    b = host.make_tensor(host.L(dl).lower(), dst.data_ptr(), 2 * n * 8 // eb, eb)
    us = per_call(lambda: host.copy((a, None), (b, None)))
    print(f"tlb_copy {name}: plan {lib.tlb_last_plan().decode()} {us:.1f} us per call on the host")
M = 256
ta = host.tensor_of(f"({M},{M}):({M},1)", torch.zeros(M * M, dtype=torch.int16, device="cuda"), ranked=True)
tb = host.tensor_of(f"({M},{M}):({M},1)", torch.zeros(M * M, dtype=torch.int16, device="cuda"), ranked=True)
tc = host.tensor_of(f"({M},{M}):(1,{M})", torch.zeros(M * M, dtype=torch.float32, device="cuda"), ranked=True)
print(f"tlb_gemm_bf16 256^3: {per_call(lambda: host.gemm_bf16(ta, tb, tc)):.1f} us per call (plan {lib.tlb_last_plan().decode()})")
out = torch.empty(4096, dtype=torch.int64, device="cuda")
print(f"tlb_eval_range 4096: {per_call(lambda: host.eval_range('((128,64),(512,1024)):((65536,1),(8388608,64))', 0, 4096, out)):.1f} us per call")
x = torch.zeros(4096, device="cuda"); y = torch.zeros(4096, device="cuda")
print(f"torch copy_ 4096 (for scale): {per_call(lambda: y.copy_(x)):.1f} us per call")
