"""Scratch measurement (NOT part of the product or the bench): torch.bmm (cuBLAS) on the C4 shape."""
import subprocess, sys, threading, time
import torch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
M = 8192
a = torch.empty(B, M, M, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
b = torch.empty(B, M, M, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
c = torch.empty(B, M, M, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    torch.bmm(a, b.transpose(1, 2), out=c)
torch.cuda.synchronize()
rows = []
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu", "--format=csv,noheader,nounits", "-lms", "50"],
                     stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [rows.append(l.strip()) for l in p.stdout], daemon=True).start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    torch.bmm(a, b.transpose(1, 2), out=c)
e1.record()
torch.cuda.synchronize()
time.sleep(0.1)
p.terminate()
ms = e0.elapsed_time(e1) / steps
print(f"torch.bmm bf16 {B} x 8192^3 (bf16 out): {ms:.2f} ms/step  {2 * M**3 * B / ms / 1e9:.1f} TFLOP/s  clocks: {rows[-6:]}")
