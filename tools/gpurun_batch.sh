#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_device_pipeline_gpu.py tests/test_multirank_gpu.py -q -x 2>&1 | tail -4
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_jd.json 2> gpurun_out/bench_c2_jd.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c2_jd.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['self_check'], d['gpu_launches']); print(d['roofline']['tiers'])"
HX_JOINT_DEDUP=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_jd0.json 2> gpurun_out/bench_c2_jd0.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c2_jd0.json')); print(d['value'], d['ms_per_step'])"
timeout 900 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1_jd.json 2> gpurun_out/bench_c1_jd.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c1_jd.json')); print('c1', d['value'], d['ms_per_step'], d['e2e']['value'])"
