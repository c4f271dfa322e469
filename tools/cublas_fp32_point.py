"""Scratch measurement (NOT part of the product or the bench): cuBLAS bf16 x bf16 GEMMs with an fp32 output through torch
(out_dtype=float32) on M N K: bf16 out, fp32 out (beta = 0) and fp32 C accumulated in place (beta = 1, the reference's
contract C += A B^T), with the bench's recipe (3 rotating operand sets, CUDA events)."""
import sys
import torch

M, N, K = (int(x) for x in sys.argv[1:4])
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 30
sets = [((torch.rand(M, K, device="cuda") * 2 - 1).to(torch.bfloat16), (torch.rand(N, K, device="cuda") * 2 - 1).to(torch.bfloat16),
         torch.zeros(M, N, dtype=torch.float32, device="cuda")) for _ in range(3)]


def timed(fn):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


fl = 2.0 * M * N * K
for name, fn in (("bf16 out", lambda i: torch.matmul(sets[i % 3][0], sets[i % 3][1].t())),
                 ("fp32 out, beta 0", lambda i: torch.mm(sets[i % 3][0], sets[i % 3][1].t(), out_dtype=torch.float32, out=sets[i % 3][2])),
                 ("fp32 C += (beta 1)", lambda i: torch.addmm(sets[i % 3][2], sets[i % 3][0], sets[i % 3][1].t(), out_dtype=torch.float32,
                                                              out=sets[i % 3][2]))):
    ms = timed(fn)
    print(f"cuBLAS {M}x{N}x{K} {name}: {ms * 1e3:.1f} us  {fl / ms / 1e9:.1f} TFLOP/s")
