"""Scratch: times tlb_eval_range on the C5 layout (2^28-element chunks of the 2^32-element index map)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_02298_b200 import abi, host
Lt = "((128,64),(512,1024)):((65536,1),(8388608,64))"
chunk = 2 ** 28
buf = torch.empty(chunk, dtype=torch.int64, device="cuda")
for i in range(3):
    host.eval_range(Lt, i * chunk, chunk, buf)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(16):
    host.eval_range(Lt, (i % 16) * chunk, chunk, buf)
e1.record()
torch.cuda.synchronize()
s = e0.elapsed_time(e1) / 16 * 1e-3
print(f"C5 chunk: {s*1e6:.1f} us  {chunk*8/s/1e9:.0f} GB/s")
