#!/bin/bash
for s in "4096 4096 2048" "4096 4096 3072" "4096 4096 4096" "4096 4096 5120" "8192 8192 2048" "8192 8192 3072" "8192 8192 4096" "8192 4096 4096" "2048 2048 8192" "3072 3072 8192"; do
  set -- $s
  echo "== $s"
  TLB_GEMM_WIDE=1 timeout 120 python tools/gemm_probe.py $1 $2 $3 50 2>&1 | tail -1
  TLB_GEMM_WIDE=0 timeout 120 python tools/gemm_probe.py $1 $2 $3 50 2>&1 | tail -1
done
