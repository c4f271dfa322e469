#!/bin/bash
# Round-2 compute-sanitizer passes over the kernels added / changed this round (summaries go to profiles/r02_sanitizer.txt)
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
run() { # name tool pytest-args...
  local name=$1 tool=$2; shift 2
  timeout 1200 $S --tool $tool --print-limit 5 python -m pytest "$@" -x -q -m gpu > gpurun_out/san_$name.log 2>&1
  echo "== $name ($tool): $(grep -E 'passed|failed' gpurun_out/san_$name.log | tail -1) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$name.log | tail -1)"
}
run copy_mem memcheck tests/test_copy_gpu.py -k "not c1 and not c3 and not full and not 4096"
run eval_mem memcheck tests/test_eval_gpu.py -k "not 2_32 and not full and not c5"
run gemm_mem memcheck tests/test_gemm_gpu.py -k "multicast_plan_matches or packed_plan_runs or conv_im2col or gett_folded_modes_on_tensor or chunked"
run copy_race racecheck tests/test_copy_gpu.py -k "tiled or strided_runs or xor_layouts_vectorised or last_writer or ragged or compositions or narrow or interleave"
run gemm_mem2 memcheck tests/test_gemm_gpu.py -k "mn_major_operands_on_tensor_cores or c_in_the_operand_type or degenerate or simt_fallback"
run gemm_sync synccheck tests/test_gemm_gpu.py -k "multicast_plan_matches or umma_kat_exact or mn_major_operands_on_tensor_cores"
