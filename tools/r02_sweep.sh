#!/bin/bash
for rep in 1 2; do
for o in 0 1; do
  echo "== SK_ORDER=$o"
  TLB_GEMM_SK_ORDER=$o timeout 120 python tools/gemm_probe.py 4096 4096 4096 50 2>&1 | tail -1
  TLB_GEMM_SK_ORDER=$o timeout 120 python tools/gemm_probe.py 8192 8192 8192 20 2>&1 | tail -1
  TLB_GEMM_SK_ORDER=$o timeout 120 python tools/gemm_probe.py 4096 4096 4096 3000 2>&1 | tail -1
done
done
TLB_GEMM_SK_ORDER=1 timeout 600 python -m pytest tests/test_gemm_gpu.py -m gpu -q -x -k "wide_plan_kat or c2 or chunked or fuzz" 2>&1 | tail -3
