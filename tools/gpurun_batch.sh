#!/bin/bash
# scratch batch for one gpurun call (edited per call)
set -x
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_full.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_full.log
tail -30 gpurun_out/gputest_full.log
timeout 400 python bench.py > gpurun_out/bench_c2_gram.json 2> gpurun_out/bench_c2_gram.err
timeout 600 python bench.py --config c4 --no-cpu-baseline > gpurun_out/bench_c4_gram.json 2> gpurun_out/bench_c4_gram.err
