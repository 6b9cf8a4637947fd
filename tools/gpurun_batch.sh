#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_variants_gpu.py -q -x -k "gram" 2>&1 | tail -3
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 12 > gpurun_out/kn.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/kn.json')); print(round(d['value']), round(d['ms_per_step'],2))"; done
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/kn.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/kn.json')); print('c4', d['value'], round(d['ms_per_step'],2))"
