#!/bin/bash
# scratch batch for one gpurun call (edited per call)
set -x
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_full.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_full.log
tail -5 gpurun_out/gputest_full.log
bash tools/fp64_profile.sh gpurun_out
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_poly.json 2> gpurun_out/bench_poly.err
