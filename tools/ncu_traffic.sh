#!/bin/bash
# Scratch: DRAM traffic per batch of the batched wide GEMM as the launch gets longer (worker drift?), and throughput at equal total work.
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct"
show() { echo "$1: $(grep -E 'dram__bytes_read|dram__bytes_write|gpu__time|hit_rate|tensor' $2 | awk -F'","' '{printf "%s=%s%s ", $(NF-2), $NF, $(NF-1)}' | tr -d '"\n')"; }
for b in 1 2 4 8 16 64; do
  ncu --metrics $M --clock-control none -k regex:umma_ -s 3 -c 1 --csv --log-file gpurun_out/nt_b$b.csv python tools/gemm_probe.py 8192 8192 8192 2 $b > /dev/null 2>&1
  show "batch=$b" gpurun_out/nt_b$b.csv
done
for rep in 1 2; do
python tools/gemm_probe.py 8192 8192 8192 6 64 2>&1 | tail -1
python tools/gemm_probe.py 8192 8192 8192 48 8 2>&1 | tail -1
python tools/gemm_probe.py 8192 8192 8192 384 1 2>&1 | tail -1
done
python tools/cublas_point.py 8192 384 2>&1 | tail -1
