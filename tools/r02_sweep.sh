#!/bin/bash
for er in 1 0 1 0; do
echo "== EARLY_RELEASE=$er"
TLB_GEMM_EARLY_RELEASE=$er timeout 300 python tools/gemm_probe.py 8192 8192 8192 6 64 2>&1 | tail -1
TLB_GEMM_EARLY_RELEASE=$er timeout 120 python tools/gemm_probe.py 4096 4096 4096 3000 2>&1 | tail -1
done
