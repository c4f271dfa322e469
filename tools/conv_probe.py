"""Scratch: the CONV line's GEMM (M 32768, N 1024, K 1152, row-major fp32 C) with A as the im2col LAYOUT of the NHWC input (rank-5
tensor map) against the same GEMM on a materialised A, and with the C orientation of tools/gemm_probe.py."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_02298_b200 import abi, host
lib = abi.load()


def t(fn, n=20):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e-3


M, N, K = 32768, 1024, 1152
fl = 2.0 * M * N * K
cases = [("im2col layout, C row-major", "((32,32,32),(128,3,3)):((128,4352,147968),(1,128,4352))", "(1024,1152):(1152,1)", "(32768,1024):(1024,1)"),
         ("materialised A, C row-major", "(32768,1152):(1152,1)", "(1024,1152):(1152,1)", "(32768,1024):(1024,1)"),
         ("materialised A, C column-major", "(32768,1152):(1152,1)", "(1024,1152):(1152,1)", "(32768,1024):(1,32768)")]
for name, la, lb, lc in cases:
    sets = []
    for _ in range(2):
        a = torch.empty(host.L(la).lower().max_offset + 1, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
        b = torch.empty(host.L(lb).lower().max_offset + 1, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
        c = torch.zeros(host.L(lc).lower().max_offset + 1, dtype=torch.float32, device="cuda")
        sets.append((host.tensor_of(la, a.view(torch.int16), ranked=True), host.tensor_of(lb, b.view(torch.int16), ranked=True), host.tensor_of(lc, c, ranked=True)))
    for knobs in ({}, {"GEMM_GROUP_M": "4"}, {"GEMM_GROUP_M": "16"}, {"GEMM_GROUP_M": "32"}):
        for k, v in knobs.items():
            host.config(k, v)
        sec = t(lambda i: host.gemm_bf16(*sets[i % 2]))
        for k in knobs:
            host.config(k, None)
        print(f"{name} {knobs}: plan {lib.tlb_last_plan().decode()} {sec * 1e6:.1f} us {fl / sec / 1e12:.0f} TFLOP/s")
    del sets
