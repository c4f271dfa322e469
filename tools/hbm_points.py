"""Scratch measurement (NOT part of the product or the bench): what plain library kernels reach on this box for
write-only, read+write and transpose traffic, with the bench's timing recipe."""
import torch


def t(fn, n=20):
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


x = torch.empty(2**28, dtype=torch.int64, device="cuda")
y = torch.empty(2**28, dtype=torch.int64, device="cuda")
s = t(lambda: x.fill_(7))
print(f"fill_ 2 GiB (write only): {2**31 / s / 1e9:.0f} GB/s")
s = t(lambda: y.copy_(x))
print(f"copy_ 2 GiB (read + write): {2 * 2**31 / s / 1e9:.0f} GB/s")
a = torch.empty(8192, 8192, dtype=torch.float32, device="cuda")
b = torch.empty(8192, 8192, dtype=torch.float32, device="cuda")
s = t(lambda: b.copy_(a.t()))
print(f"torch transpose copy 8192^2 fp32: {2 * 8192 * 8192 * 4 / s / 1e9:.0f} GB/s")
s = t(lambda: b.copy_(a))
print(f"torch plain copy 8192^2 fp32 (512 MiB): {2 * 8192 * 8192 * 4 / s / 1e9:.0f} GB/s")
s = t(lambda: torch.arange(2**28, out=x))
print(f"torch.arange int64 2 GiB (index map, write only): {2**31 / s / 1e9:.0f} GB/s")
