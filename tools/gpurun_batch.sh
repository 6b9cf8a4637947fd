#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_variants_gpu.py tests/test_modes_gpu.py -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
for sp in 20 0 100; do
  HX_CHASE_SPIN_NS=$sp timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_spin$sp.json 2> /dev/null
done
for o in big-then-small big-first; do
  HX_E2E_ORDER=$o timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_order_$o.json 2> /dev/null
done
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py --config c2 > /dev/null 2>&1
