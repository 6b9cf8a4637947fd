#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_device_pipeline_gpu.py tests/test_fx_gpu.py tests/test_modes_gpu.py -q -x 2>&1 | tail -3
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/kn.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/kn.json')); print(round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), d['self_check']['bitwise_equal'])"; done
python tools/e2e_prof.py --reps 2 2>&1 | sed -n 1,12p
