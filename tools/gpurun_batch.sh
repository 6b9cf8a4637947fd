#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_device_pipeline_gpu.py -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
timeout 300 python bench.py --config c1 --steps 2000 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for r in device host; do
timeout 300 python tools/e2e_prof.py --config c1 --reps 30 --rng $r > gpurun_out/e2e_c1_$r.txt 2>&1
timeout 300 python tools/e2e_prof.py --config c2 --reps 5 --rng $r > gpurun_out/e2e_c2_$r.txt 2>&1
done
