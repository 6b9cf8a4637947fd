#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_device_pipeline_gpu.py tests/test_fx_gpu.py tests/test_modes_gpu.py tests/test_parity_gpu.py -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
timeout 300 python tools/e2e_prof.py --config c2 --reps 5 > gpurun_out/e2e_c2.txt 2>&1
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
