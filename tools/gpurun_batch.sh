#!/bin/bash
set -x
timeout 1200 python -m pytest tests/test_variants_gpu.py tests/test_device_pipeline_gpu.py tests/test_large_gpu.py tests/test_parity_gpu.py -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> /dev/null
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/c5_2048.csv python tools/c5_sample.py --n 2048 --batch 1341 > /dev/null 2>&1
