"""Command line over the C ABI, in the style of the reference's `tla` tool (cli.hpp:23-46: one subcommand, layouts as
text), for the calls the reference CLI does not have:

    python -m paper_2603_02298_b200 plan  "(8192,8192):(8192,1)" "(8192,8192):(1,8192)" --elem-bytes 4
    python -m paper_2603_02298_b200 copy  "(8192,8192):(8192,1)" "(8192,8192):(1,8192)" --elem-bytes 4 [--steps 20]
    python -m paper_2603_02298_b200 gemm  "(4096,4096):(4096,1)" "(4096,4096):(4096,1)" "(4096,4096):(1,4096)"
    python -m paper_2603_02298_b200 eval  "((128,64),(512,1024)):((65536,1),(8388608,64))" --begin 0 --count 1048576

`plan` runs on the host only (contract checks + planner, no device). The others allocate synthetic device buffers,
run the call through libtlb.so and print one JSON line with the plan and the device-timed throughput. Exit codes follow
the reference (cli.hpp:215-221): 0 ok, 1 a tla-style error (contract, bounds, ...), 2 a usage / parse error.
"""
from __future__ import annotations

import argparse
import json
import sys

from . import abi, host


def _timed(torch, fn, steps, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e-3


def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        raise abi.TlbError(abi.TLB_ERR_CUDA, "no CUDA device: libtlb has no CPU fallback")
    return torch


def cmd_plan(a):
    print(json.dumps({"plan": host.copy_plan(a.src, a.dst, a.elem_bytes, a.begin, a.end)}))


def cmd_copy(a):
    torch = _need_cuda()
    ls, ld = host.L(a.src), host.L(a.dst)
    dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[a.elem_bytes]
    src = torch.arange(ls.cosize, device="cuda").to(dt)
    dst = torch.zeros(ld.cosize, dtype=dt, device="cuda")
    s, d = host.tensor_of(ls, src), host.tensor_of(ld, dst)
    sec = _timed(torch, lambda: host.copy(s, d), a.steps)
    n = ls.size
    print(json.dumps({"plan": abi.load().tlb_last_plan().decode(), "elements": n, "us": sec * 1e6,
                      "GB/s": 2 * n * a.elem_bytes / sec / 1e9}))


def cmd_gemm(a):
    torch = _need_cuda()
    la, lb, lc = host.L(a.a), host.L(a.b), host.L(a.c)
    ta_ = torch.empty(la.cosize, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    tb_ = torch.empty(lb.cosize, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    tc_ = torch.zeros(lc.cosize, dtype=torch.float32, device="cuda")
    ta = host.tensor_of(la, ta_.view(torch.int16), ranked=True)
    tb = host.tensor_of(lb, tb_.view(torch.int16), ranked=True)
    tc = host.tensor_of(lc, tc_, ranked=True)
    sec = _timed(torch, lambda: host.gemm_bf16(ta, tb, tc), a.steps)
    m, k = la.top_sizes()
    n = lb.top_sizes()[0]
    print(json.dumps({"plan": abi.load().tlb_last_plan().decode(), "M": m, "N": n, "K": k, "us": sec * 1e6,
                      "TFLOP/s": 2.0 * m * n * k / sec / 1e12}))


def cmd_eval(a):
    torch = _need_cuda()
    out = torch.empty(a.count, dtype=torch.int64, device="cuda")
    sec = _timed(torch, lambda: host.eval_range(a.layout, a.begin, a.count, out), a.steps)
    head = out[: min(8, a.count)].cpu().tolist()
    print(json.dumps({"count": a.count, "us": sec * 1e6, "GB/s": a.count * 8 / sec / 1e9, "first": head}))


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2603_02298_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("plan", help="the copy plan tlb_copy would choose (host only)")
    p.add_argument("src"), p.add_argument("dst")
    p.add_argument("--elem-bytes", type=int, default=4, choices=[1, 2, 4, 8, 16])
    p.add_argument("--begin", type=int, default=0), p.add_argument("--end", type=int, default=2**64 - 1)
    p.set_defaults(fn=cmd_plan)
    p = sub.add_parser("copy", help="dst(i) = src(i) on device, timed")
    p.add_argument("src"), p.add_argument("dst")
    p.add_argument("--elem-bytes", type=int, default=4, choices=[1, 2, 4, 8])
    p.add_argument("--steps", type=int, default=10)
    p.set_defaults(fn=cmd_copy)
    p = sub.add_parser("gemm", help="C(m,n) += A(m,k) B(n,k), bf16 operands, fp32 C, timed")
    p.add_argument("a"), p.add_argument("b"), p.add_argument("c")
    p.add_argument("--steps", type=int, default=10)
    p.set_defaults(fn=cmd_gemm)
    p = sub.add_parser("eval", help="index map L(i) over [begin, begin + count) into device memory, timed")
    p.add_argument("layout")
    p.add_argument("--begin", type=int, default=0), p.add_argument("--count", type=int, default=1 << 20)
    p.add_argument("--steps", type=int, default=10)
    p.set_defaults(fn=cmd_eval)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code not in (0, None) else 0
    try:
        a.fn(a)
    except (ValueError, IndexError) as e:   # layout text that does not parse
        print(f"parse error: {e}", file=sys.stderr)
        return 2
    except abi.TlbError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
