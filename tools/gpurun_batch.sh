#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_variants_gpu.py tests/test_parity_gpu.py tests/test_large_gpu.py -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
for b in 1 0; do
  HX_RU_BULK=$b timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_bulk$b.json 2> gpurun_out/bench_bulk$b.err
  HX_RU_BULK=$b timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bulk$b.csv python tools/profile_run.py --config c2 --levels 4 --parent-only > /dev/null 2>&1
done
HX_RU_BULK=1 timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/bench_c4_bulk1.json 2>&1
HX_RU_BULK=0 timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline --steps 3 > gpurun_out/bench_c4_bulk0.json 2>&1
