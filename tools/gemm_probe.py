"""Times tlb_gemm_bf16 on one TN problem (M N K [steps] [batch]) with the bench's recipe; with TLB_GEMM_TRACE set, the
library also dumps the per-CTA timeline of the last launch."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_02298_b200 import abi, host

M, N, K = (int(x) for x in sys.argv[1:4])
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
batch = int(sys.argv[5]) if len(sys.argv) > 5 else 1
import os
lib = abi.load()
sets = []
nsets = int(os.environ.get('PROBE_SETS', 3 if batch == 1 else 1))
LD = int(os.environ.get('PROBE_LD', K))  # leading dimension of A and B (elements); > K pads the rows
for s in range(nsets):
    a = torch.empty(batch * M * LD, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    b = torch.empty(batch * N * LD, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    c = torch.zeros(batch * M * N, dtype=torch.bfloat16 if os.environ.get('PROBE_C16') else torch.float32, device="cuda")
    sets.append((host.tensor_of(f"({M},{K}):({LD},1)", a.view(torch.int16), ranked=True),
                 host.tensor_of(f"({N},{K}):({LD},1)", b.view(torch.int16), ranked=True),
                 host.tensor_of(f"({M},{N}):(1,{M})", c.view(torch.int16) if c.dtype == torch.bfloat16 else c, ranked=True)))


def step(i):
    ta, tb, tc = sets[i % nsets]
    if batch == 1:
        host.gemm_bf16(ta, tb, tc)
    else:
        host.gemm_bf16_batched(ta, tb, tc, M * LD, N * LD, M * N, 0, batch)


import subprocess, threading, time
rows = []
for i in range(3):
    step(i)
torch.cuda.synchronize()
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu", "--format=csv,noheader,nounits", "-lms", "50"],
                     stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [rows.append(l.strip()) for l in p.stdout], daemon=True).start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h0 = time.perf_counter()
for i in range(steps):
    step(i)
h1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
time.sleep(0.1)
p.terminate()
print("clocks/power/temp:", rows[-6:])
print(f"host launch loop: {(h1 - h0) / steps * 1e6:.1f} us/call")
print(f"{M}x{N}x{K} batch {batch} plan {lib.tlb_last_plan().decode()}: {ms * 1e3:.1f} us/step  {2 * M * N * K * batch / ms / 1e9:.1f} TFLOP/s")
