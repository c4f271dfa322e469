"""Scratch: throughput of the other bulk-evaluation entry points on the C5 layouts (2^26-element windows)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_02298_b200 import abi, host
Lt = "((128,64),(512,1024)):((65536,1),(8388608,64))"
Rt = "(64,1024,128,512):(128,4194304,1,8192)"
n = 2 ** 26
def t(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3
out = torch.empty(n, dtype=torch.int64, device="cuda")
crd = torch.empty(n, 4, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
s = t(lambda: host.eval_range(Rt, 2**31, n, out)); print(f"eval_range R      : {n/s/1e9:7.1f} G evals/s  {n*8/s/1e9:7.0f} GB/s written")
s = t(lambda: host.idx2crd_range(Lt, 2**31, n, crd)); print(f"idx2crd           : {n/s/1e9:7.1f} G elems/s  {n*32/s/1e9:7.0f} GB/s written")
s = t(lambda: host.crd2idx_range(Lt, crd, n, out)); print(f"crd2idx           : {n/s/1e9:7.1f} G elems/s  {n*40/s/1e9:7.0f} GB/s moved")
s = t(lambda: host.rinv_check_range(Lt, Rt, 2**31, n, cnt)); print(f"rinv check L(R(k)): {n/s/1e9:7.1f} G checks/s (no memory traffic)")
s = t(lambda: host.compose_check_range("(8192,8192):(1,8192)", "(8192,8192):(8192,1)", "(8192,8192):(8192,1)", 0, n, cnt)); print(f"compose check     : {n/s/1e9:7.1f} G checks/s")
ax = torch.empty(n, 2, dtype=torch.int64, device="cuda")
s = t(lambda: host.eval_axes_range("((128,64),(512,1024)):((e0,e1),(128*e0,64*e1))", 2, 2**31, n, ax)); print(f"eval_axes (2 axes) : {n/s/1e9:7.1f} G elems/s  {n*16/s/1e9:7.0f} GB/s written")
