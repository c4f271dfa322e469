#!/bin/bash
# Round-2 final GEMM capture: C2 (4 launches) then the first per-batch launches of C4 after launch chunking
ncu --set full --clock-control none -k regex:umma_wide -c 8 -f -o gpurun_out/r02b_gemm \
    python bench.py --steps 1 --warmup 3 --no-cpu --quick --only C4 > /dev/null 2> gpurun_out/r02b_gemm.err
ls -la gpurun_out/r02b_gemm.ncu-rep
timeout 600 python -m pytest tests/test_copy_gpu.py -m gpu -q -x 2>&1 | tail -3
