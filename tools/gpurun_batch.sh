#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_variants_gpu.py -q -x -k "small_gram or shared_memory_tiers or register_golub" > gpurun_out/gputest_sg.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_sg.log
tail -25 gpurun_out/gputest_sg.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_sg.json 2> gpurun_out/bench_c2_sg.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c2_sg.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['self_check'])"
HX_SMALL_GRAM=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_sg0.json 2> gpurun_out/bench_c2_sg0.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c2_sg0.json')); print(d['value'], d['ms_per_step'])"
