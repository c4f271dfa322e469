#!/bin/bash
for rep in 1 2 3; do
for dbg in 0 64; do
TLB_GEMM_DEBUG=$dbg python bench.py --only Cg --no-cpu --quick --steps 30 > gpurun_out/b_cg.json 2>/dev/null; python -c "
import json
d=json.load(open('gpurun_out/b_cg.json'))
print('debug=$dbg', 'C2', round(d['value'],1), [(e['name'], round(e['value'],1)) for e in d['other_configs']])
"
done
done
