#!/bin/bash
python -m pytest tests/test_gemm_gpu.py -x -q -m gpu -k "chunked or c4_batched or batched" 2>&1 | tail -3
for rep in 1 2; do
python tools/gemm_probe.py 8192 8192 8192 6 64 2>&1 | tail -1
TLB_GEMM_CHUNK_WAVES=0 python tools/gemm_probe.py 8192 8192 8192 6 64 2>&1 | tail -1
TLB_GEMM_CHUNK_WAVES=4 python tools/gemm_probe.py 8192 8192 8192 6 64 2>&1 | tail -1
TLB_GEMM_CHUNK_WAVES=16 python tools/gemm_probe.py 8192 8192 8192 6 64 2>&1 | tail -1
done
python tools/gemm_probe.py 16384 16384 16384 6 1 2>&1 | tail -1
TLB_GEMM_CHUNK_WAVES=0 python tools/gemm_probe.py 16384 16384 16384 6 1 2>&1 | tail -1
python tools/cublas_point.py 16384 6 2>&1 | tail -1
python bench.py --only C4 --no-cpu --steps 20 > gpurun_out/b_c4.json 2>gpurun_out/b_c4.err; python -c "
import json
d=json.load(open('gpurun_out/b_c4.json'))
print('C2', d['value'], d['clocks'])
for e in d['other_configs']: print(e['name'], round(e['value'],1), e['ms_per_step'], e['config'].get('plan'), e['roofline']['frac'])
"
