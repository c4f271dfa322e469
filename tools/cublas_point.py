"""Scratch measurement (NOT part of the product or the bench): cuBLAS bf16 via torch.matmul on the bench's
C2 shape and timing recipe, to know what the vendor library reaches on the same box / same clocks."""
import subprocess, sys, threading, time
import torch

M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sets = []
for s in range(3):
    a = (torch.rand(M, K, device="cuda") * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(N, K, device="cuda") * 2 - 1).to(torch.bfloat16)
    sets.append((a, b))
for i in range(5):
    torch.matmul(sets[i % 3][0], sets[i % 3][1].t())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
rows = []
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "20"],
                     stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [rows.append(l.strip()) for l in p.stdout], daemon=True).start()
time.sleep(0.2)
e0.record()
for i in range(steps):
    torch.matmul(sets[i % 3][0], sets[i % 3][1].t())
e1.record()
torch.cuda.synchronize()
time.sleep(0.1)
p.terminate()
ms = e0.elapsed_time(e1) / steps
print(f"torch.matmul bf16 {M}^3 x{steps}: {ms*1e3:.1f} us/step  {2*M*N*K/ms/1e9:.1f} TFLOP/s   clocks/power samples: {rows[-8:]}")
