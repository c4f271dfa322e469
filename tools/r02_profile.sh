#!/bin/bash
# Round-2 ncu captures (run under gpurun; summaries are made afterwards with tools/ncu_summary.py).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --quick > gpurun_out/r02_launches_bench.json 2> gpurun_out/r02_launches.err
ncu --set full --clock-control none -k regex:umma_wide -c 12 -f -o gpurun_out/r02_gemm \
    python bench.py --steps 1 --warmup 3 --no-cpu --quick --only C2_bf16_c,C4 > /dev/null 2> gpurun_out/r02_gemm.err
ncu --set full --clock-control none --import-source on -k regex:"tiled_kernel|eval_warp" -c 12 -f -o gpurun_out/r02_copy \
    python bench.py --steps 1 --warmup 3 --no-cpu --quick --only C1,C3,C5 > /dev/null 2> gpurun_out/r02_copy.err
ls -la gpurun_out/*.ncu-rep
