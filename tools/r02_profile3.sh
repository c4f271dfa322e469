#!/bin/bash
# Round-2 FINAL ncu captures (the kernels as committed at the end of the round). The .ncu-rep files stay on the GPU box
# (together they exceed gpurun's 64 MiB return limit); tools/ncu_summary.py turns them into the summaries kept in profiles/r02c_*.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r02c_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --quick > gpurun_out/r02c_launches_bench.json 2> gpurun_out/r02c_launches.err
ncu --set full --clock-control none -k regex:umma_wide -c 12 -f -o /tmp/r02c_gemm \
    python bench.py --steps 1 --warmup 3 --no-cpu --quick --only C2_bf16_c,C4 > /dev/null 2> gpurun_out/r02c_gemm.err
ncu --set full --clock-control none --import-source on -k regex:"tiled_kernel|eval_warp|interleave_kernel|gather_run_kernel" -c 24 -f -o /tmp/r02c_copy \
    python bench.py --steps 1 --warmup 3 --no-cpu --quick --only C1,C3,C5,Cx > /dev/null 2> gpurun_out/r02c_copy.err
python tools/ncu_summary.py /tmp/r02c_gemm.ncu-rep gpurun_out/r02c_gemm_ncu
python tools/ncu_summary.py /tmp/r02c_copy.ncu-rep gpurun_out/r02c_copy_eval_ncu
ls -la /tmp/r02c_*.ncu-rep gpurun_out/r02c_*
