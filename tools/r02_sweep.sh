#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q --durations=25 2>&1 | tail -45
echo "== bench --gpus 2 on a 1-GPU box must fail loudly"
timeout 300 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --quick > gpurun_out/b_2gpu.json 2> gpurun_out/b_2gpu.err; echo "exit $?"; tail -3 gpurun_out/b_2gpu.err
echo "== bench --gpus 2 --share-gpu (functional)"
timeout 600 python bench.py --gpus 2 --share-gpu --steps 3 --warmup 3 --no-cpu --quick --only C1,C5 > gpurun_out/b_2share.json 2> gpurun_out/b_2share.err; echo "exit $?"; python -c "
import json
d=json.load(open('gpurun_out/b_2share.json'))
print(d['n_gpus'], d['verify'], [ (e['name'], e['n_gpus'], round(e['value'],1)) for e in d['other_configs']])
"
