#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_all.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_all.log
tail -6 gpurun_out/gputest_all.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_nw.json 2> gpurun_out/bench_c2_nw.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c2_nw.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['self_check'])"
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_nw.json 2> gpurun_out/bench_c4_nw.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c4_nw.json')); print('c4', d['value'], d['ms_per_step'])"
timeout 900 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_nw.json 2> gpurun_out/bench_c3_nw.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c3_nw.json')); print('c3', d['value'], d['ms_per_step'])"
MM=gpu__time_duration.sum,sm__warps_active.avg.per_cycle_active,smsp__inst_executed.sum
timeout 600 ncu --metrics $MM --clock-control none --kernel-name regex:"zone_" -c 10 --csv --log-file gpurun_out/zone_n.csv python tools/profile_run.py --config c2 --levels 4 --parent-only > /dev/null 2>&1
grep zone_ gpurun_out/zone_n.csv | cut -d, -f5,8,9,13- | head
