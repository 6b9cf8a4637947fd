#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_device_pipeline_gpu.py tests/test_multirank_gpu.py -q -x > gpurun_out/gputest_dp.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_dp.log
python tools/timeline.py --config c2 > gpurun_out/timeline_c2_il.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_il.json 2> gpurun_out/bench_il.err
