#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_variants_gpu.py tests/test_large_gpu.py -q -x -k "gram or large or nu64 or 64" > gpurun_out/gputest_gram.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_gram.log
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_tri.json 2> gpurun_out/bench_tri.err
timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_tri.json 2> gpurun_out/bench_c4_tri.err
HX_GRAM_TRI=0 timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_tri0.json 2> gpurun_out/bench_c4_tri0.err
