#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_variants_gpu.py -q -x -k "gram" > gpurun_out/gramtest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gramtest.log
timeout 900 python -m pytest tests/test_eigvalsh_gpu.py tests/test_variants_gpu.py tests/test_device_pipeline_gpu.py tests/test_parity_gpu.py -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
for gm in 1 0; do
  HX_GRAM=$gm timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_gram$gm.json 2> gpurun_out/bench_gram$gm.err
done
HX_GRAM=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gram.csv python tools/profile_run.py --config c2 > /dev/null 2>&1
