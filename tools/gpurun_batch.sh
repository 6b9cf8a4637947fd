#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
for r in 1 2; do
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_capd$r.json 2> gpurun_out/bench_capd$r.err
HX_SYM_CAP=5 timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_cap5$r.json 2> gpurun_out/bench_cap5$r.err
done
