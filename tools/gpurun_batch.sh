#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_variants_gpu.py -q -x -k "complex_gram" > gpurun_out/gputest_cg.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_cg.log
tail -25 gpurun_out/gputest_cg.log
timeout 900 python bench.py --config c5 --no-cpu-baseline > gpurun_out/bench_c5_cg.json 2> gpurun_out/bench_c5_cg.err
