#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_variants_gpu.py -q -x -k "gram" > gpurun_out/gputest_gram.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_gram.log
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_wfix.json 2> gpurun_out/bench_wfix.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic_L4.csv python tools/profile_run.py --config c2 --levels 4 --parent-only > /dev/null 2>&1
