#!/bin/bash
# Scratch: traffic counters of our tcgen05 GEMM and of cuBLAS (torch.matmul) on the same shape, for the energy comparison.
S=${1:-8192}
TAG=${2:-ours}
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_red.sum,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,sm__inst_executed.sum,smsp__cycles_active.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__cluster_dim_x,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcnode_gpc.sum,lts__ltcfabric2lts_cycles_active.sum,lts__d_sectors.sum,lts__d_sectors_fill_device.sum,lts__t_requests_op_read.sum,lts__t_requests_srcnode_gpc.sum,lts__t_sectors.sum,lts__t_sectors_lookup_miss.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_sectors_srcunit_ltcfabric_lookup_miss.sum"
if [ "$TAG" = cublas ]; then
ncu --metrics $M --clock-control none -k regex:'gemm|nvjet|cutlass|sm100' -s 3 -c 1 --csv --log-file gpurun_out/ncu_cublas_$S.csv python tools/cublas_point.py $S 3 > /dev/null 2>&1
else
ncu --metrics $M --clock-control none -k regex:umma_ -s 3 -c 1 --csv --log-file gpurun_out/ncu_${TAG}_$S.csv python tools/gemm_probe.py $S $S $S 3 > /dev/null 2>&1
fi
