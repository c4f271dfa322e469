#!/bin/bash
# Scratch: sustained-throughput sweep of the tcgen05 GEMM knobs (power-capped regime).
run() { echo -n "$1 :: "; env $1 python tools/power_point.py ours $2 $3 2>&1 | tail -1 | cut -c1-60; }
for S in 4096 8192; do
  if [ $S = 8192 ]; then N=400; else N=2500; fi
  for v in "$@"; do run "$v" $S $N; done
done
