#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_variants_gpu.py -q -x -k "rank_update" > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
for t in 1 0; do
  HX_RU_TMA=$t timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_tma$t.json 2> gpurun_out/bench_tma$t.err
  HX_RU_TMA=$t timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_tma$t.csv python tools/profile_run.py --config c2 --levels 4 --parent-only > /dev/null 2>&1
done
