#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_variants_gpu.py -q -x -k "register_golub or shared_memory_tiers" > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bidiag --csv --log-file gpurun_out/bidiag_reg1.csv python tools/profile_run.py --config c2 > /dev/null 2>&1
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_reg1.json 2> /dev/null
