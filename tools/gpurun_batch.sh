#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_variants_gpu.py tests/test_large_gpu.py -q -x -k "gram or large" > gpurun_out/gputest_gram.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_gram.log
timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_rel.json 2> gpurun_out/bench_c4_rel.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:sym_chase --log-file gpurun_out/launches_c4_rel.csv python tools/profile_run.py --config c4 > /dev/null 2>&1
