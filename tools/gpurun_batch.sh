#!/bin/bash
# scratch batch for one gpurun call (edited per call)
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_variants_gpu.py -q -x -k "gram" > gpurun_out/gputest_gram.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_gram.log
tail -5 gpurun_out/gputest_gram.log
HX_GRAM=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gram1.csv python tools/profile_run.py --config c2 > /dev/null 2>&1
HX_GRAM=1 timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_gram1.json 2> gpurun_out/bench_gram1.err
HX_GRAM=0 timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_gram0.json 2> gpurun_out/bench_gram0.err
