#!/bin/bash
set -x
for v in "HX_CHASE_RCL=0" "HX_CHASE_RCL=2 HX_CHASE_CLNW=8" "HX_CHASE_RCL=2 HX_CHASE_CLNW=8 HX_CHASE_REG=1" "HX_CHASE_REG=1"; do
  tag=$(echo $v | tr ' =' '_-')
  env $v timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_$tag.json 2> /dev/null
  env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chase --csv --log-file gpurun_out/chase_$tag.csv python tools/profile_run.py --config c2 --levels 4 --parent-only > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bd_chase -c 1 -o gpurun_out/chase_nw16 python tools/profile_run.py --config c2 --levels 4 --parent-only > gpurun_out/ncu_chase16.log 2>&1
HX_CHASE_REG=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:bd_chase -c 1 -o gpurun_out/chase_nw16_reg python tools/profile_run.py --config c2 --levels 4 --parent-only > gpurun_out/ncu_chase16r.log 2>&1
