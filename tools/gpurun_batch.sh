#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_variants_gpu.py tests/test_large_gpu.py tests/test_device_pipeline_gpu.py -q -x -k "gram or large or independent" > gpurun_out/gputest_gram.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_gram.log
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_half.json 2> gpurun_out/bench_half.err
timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_half.json 2> gpurun_out/bench_c4_half.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:sym_chase --log-file gpurun_out/launches_half.csv python tools/profile_run.py --config c2 > /dev/null 2>&1
