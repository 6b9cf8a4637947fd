#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_device_pipeline_gpu.py tests/test_variants_gpu.py -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py --config c2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:small_bidiag -c 2 -o gpurun_out/bidiag python tools/profile_run.py --config c2 --levels 2 --parent-only > gpurun_out/ncu_bidiag.log 2>&1
