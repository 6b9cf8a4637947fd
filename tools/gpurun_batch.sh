#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_variants_gpu.py -q -x -k "hermitian_chase" > gpurun_out/gputest_h.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_h.log
tail -5 gpurun_out/gputest_h.log
bash tools/fp64_profile.sh gpurun_out
for c in c3 c4 c1 c5; do
timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
