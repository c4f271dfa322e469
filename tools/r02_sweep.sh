#!/bin/bash
# Scratch: TMA-fed persistent copy sweep + new GEMM tests
echo "== LDG tiled"; python tools/copy_probe.py c1 c3 2>&1 | tail -2
for st in 2 3 4 6; do for ct in 1 2 3 4; do
  echo "== TMA stages=$st ctas=$ct"; TLB_COPY_TMA=1 TLB_COPY_TMA_STAGES=$st TLB_COPY_TMA_CTAS=$ct python tools/copy_probe.py c1 c3 2>&1 | tail -2
done; done
echo "== LB128"; TLB_COPY_LB256=0 TLB_COPY_TMA=1 TLB_COPY_TMA_STAGES=4 TLB_COPY_TMA_CTAS=3 python tools/copy_probe.py c1 c3 2>&1 | tail -2
TLB_COPY_LB256=0 TLB_COPY_TMA=1 TLB_COPY_TMA_STAGES=6 TLB_COPY_TMA_CTAS=2 python tools/copy_probe.py c1 c3 2>&1 | tail -2
python -m pytest tests/test_gemm_gpu.py -x -q -m gpu -k "packed or conv or gett" 2>&1 | tail -5
python bench.py --only Cg --no-cpu --steps 20 --gemm-only > gpurun_out/b_cg.json 2>gpurun_out/b_cg.err; python - <<'PY'
import json
d=json.load(open('gpurun_out/b_cg.json'))
for e in d['other_configs']: print(e['name'], e['value'], e['config'].get('plan'))
PY
