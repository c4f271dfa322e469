#!/bin/bash
# Scratch: DRAM / L2 traffic of the wide GEMM at 8192^3 against cuBLAS, for padded leading dimensions and rasterisation groups.
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
show() { echo "$1: $(grep -E 'dram__bytes_read|dram__bytes_write|gpu__time|hit_rate|tensor' $2 | awk -F'","' '{printf "%s=%s%s ", $(NF-2), $NF, $(NF-1)}' | tr -d '"\n')"; }
ncu --metrics $M --clock-control none -k regex:'gemm|nvjet|cutlass|sm100' -s 3 -c 1 --csv --log-file gpurun_out/nt_cublas.csv python tools/cublas_point.py 8192 3 > /dev/null 2>&1
show cublas gpurun_out/nt_cublas.csv
for ld in 8192 8256 8320; do
  PROBE_LD=$ld ncu --metrics $M --clock-control none -k regex:umma_ -s 3 -c 1 --csv --log-file gpurun_out/nt_ld$ld.csv python tools/gemm_probe.py 8192 8192 8192 3 > /dev/null 2>&1
  show "ours ld=$ld" gpurun_out/nt_ld$ld.csv
done
for g in 2 4 16 32; do
  TLB_GEMM_GROUP_M=$g ncu --metrics $M --clock-control none -k regex:umma_ -s 3 -c 1 --csv --log-file gpurun_out/nt_g$g.csv python tools/gemm_probe.py 8192 8192 8192 3 > /dev/null 2>&1
  show "ours group_m=$g" gpurun_out/nt_g$g.csv
done
for ld in 8192 8256; do
echo "timing ld=$ld:"; PROBE_LD=$ld python tools/gemm_probe.py 8192 8192 8192 20 2>&1 | tail -1
echo "sustained ld=$ld:"; PROBE_LD=$ld python tools/gemm_probe.py 8192 8192 8192 20 8 2>&1 | tail -1
done
