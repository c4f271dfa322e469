#!/bin/bash
timeout 600 python -m pytest tests/test_copy_gpu.py -x -q -m gpu 2>&1 | tail -12
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q -m gpu -k "packed" 2>&1 | tail -3
python bench.py --only Cg --no-cpu --quick --steps 20 > gpurun_out/b_cx.json 2>gpurun_out/b_cx.err; python -c "
import json
d=json.load(open('gpurun_out/b_cx.json'))
for e in d['other_configs']: print(e['name'], round(e['value'],1), e['ms_per_step'], e['config'].get('plan'))
"
