#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
for W in 0 3 4 5; do
HX_E2E_WORKERS=$W timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_e2eW$W.json 2> gpurun_out/bench_e2eW$W.err
done
HX_E2E_WORKERS=3 HX_E2E_ORDER=big-first timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_e2eW3b.json 2> gpurun_out/bench_e2eW3b.err
