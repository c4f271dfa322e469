#!/bin/bash
# Full GPU suite + full bench + reference arm (what the driver runs at round end)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_pytest.log; tail -4 gpurun_out/r02_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/r02_smoke.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_ref.err; echo "ref exit $?"
timeout 900 python bench.py > gpurun_out/r02_bench_final.json 2> gpurun_out/r02_bench.err; echo "bench exit $?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/r02_bench_final.json'))
o=d.pop('other_configs')
print('C2', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks'].get('sm_mhz_in_kernel'), (d['clocks'].get('sustained_probe') or {}).get('tflops'), d['library_same_box'])
for e in o:
    r=e.get('roofline') or {}
    print(e['name'], round(e['value'],1), e['unit'], 'ms', round(e.get('ms_per_step',0),3), 'frac', r.get('frac') and round(r['frac'],3), e['config'].get('plan'))
PY
