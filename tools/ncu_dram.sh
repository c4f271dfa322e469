#!/bin/bash
# Scratch: DRAM / L2 traffic of the GEMM kernel at 8192^3 for a few rasterisation groups.
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex.sum"
for g in "$@"; do
  TLB_GEMM_GROUP_M=$g ncu --metrics $M --clock-control none -k regex:umma_ -s 3 -c 1 --csv --log-file gpurun_out/ncu_g$g.csv python tools/gemm_probe.py 8192 8192 8192 3 > /dev/null 2>&1
  echo "group_m=$g: $(grep -E 'dram__bytes_read|dram__bytes_write|gpu__time|hit_rate' gpurun_out/ncu_g$g.csv | awk -F'","' '{printf "%s=%s ", $(NF-2), $NF}' | tr -d '"\n')"
done
