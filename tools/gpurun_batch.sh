#!/bin/bash
set -x
for nw in 2 8 4; do
  HX_CHASE_RNW=$nw timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/bench_rnw$nw.json 2> /dev/null
done
HX_CHASE_RNW=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chase --csv --log-file gpurun_out/chase_rnw2.csv python tools/profile_run.py --config c2 --levels 3 --parent-only > /dev/null 2>&1
HX_CHASE_RNW=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chase --csv --log-file gpurun_out/chase_rnw4.csv python tools/profile_run.py --config c2 --levels 3 --parent-only > /dev/null 2>&1
