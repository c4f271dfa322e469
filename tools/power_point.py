"""Scratch: sustained loop of our GEMM or torch.matmul with nvidia-smi power / clock samples taken during the loop."""
import subprocess, sys, threading, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
which, S, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
a = torch.empty(S * S, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
b = torch.empty(S * S, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
if which == "ours":
    from paper_2603_02298_b200 import abi, host
    c = torch.zeros(S * S, dtype=torch.float32, device="cuda")
    ta = host.tensor_of(f"({S},{S}):({S},1)", a.view(torch.int16), ranked=True)
    tb = host.tensor_of(f"({S},{S}):({S},1)", b.view(torch.int16), ranked=True)
    tc = host.tensor_of(f"({S},{S}):(1,{S})", c, ranked=True)
    step = lambda: host.gemm_bf16(ta, tb, tc)
else:
    A, B = a.view(S, S), b.view(S, S)
    step = lambda: torch.matmul(A, B.t())
for _ in range(3):
    step()
torch.cuda.synchronize()
rows = []
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw.instant,clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "20"],
                     stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [rows.append(l.strip()) for l in p.stdout], daemon=True).start()
time.sleep(0.3)
n0 = len(rows)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    step()
e1.record()
torch.cuda.synchronize()
n1 = len(rows)
p.terminate()
ms = e0.elapsed_time(e1) / steps
mid = rows[n0 + 2:n1] or rows[-3:]
print(f"{which} {S}^3 x{steps}: {ms*1e3:.1f} us/step {2*S**3/ms/1e9:.1f} TFLOP/s; samples during loop ({len(mid)}): first {mid[:3]} ... last {mid[-3:]}")
