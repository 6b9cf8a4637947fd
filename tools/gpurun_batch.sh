#!/bin/bash
# Round-end check on the GPU box: smoke, the GPU test suite, the default bench line and the reference arm.
#   gpurun --timeout 3600 -- 'bash tools/gpurun_batch.sh'
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_all.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_all.log
tail -4 gpurun_out/gputest_all.log
timeout 900 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref_c2.json 2> gpurun_out/r02_bench_ref_c2.err
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_c2.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['cpu_baseline']['value'], d['self_check'], d['gpu_launches'], d['clocks'])
r=json.load(open('gpurun_out/r02_bench_ref_c2.json')); print('ref', r['value'], r['cpu_baseline']['cores'])"
