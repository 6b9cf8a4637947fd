#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config c3 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/bench_c3_L3.json 2> gpurun_out/bench_c3_L3.err
HX_LANES=0 timeout 600 python bench.py --config c3 --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/bench_c3_L0.json 2> gpurun_out/bench_c3_L0.err
timeout 600 python bench.py > gpurun_out/bench_c2_L3.json 2> gpurun_out/bench_c2_L3.err
