#!/bin/bash
# Round-2 final captures, second part: the warp evaluator (C5) and the interleave kernel
ncu --set full --clock-control none --import-source on -k regex:"eval_warp|interleave_kernel" -c 12 -f -o /tmp/r02c_eval \
    python bench.py --steps 1 --warmup 3 --no-cpu --quick --only C5,Cx > /dev/null 2> gpurun_out/r02c_eval.err
python tools/ncu_summary.py /tmp/r02c_eval.ncu-rep gpurun_out/r02c_eval_interleave_ncu
