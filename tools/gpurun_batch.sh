#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.per_cycle_active --clock-control none --kernel-name regex:"zone_" -c 40 --csv --log-file gpurun_out/zone_l.csv python tools/profile_run.py --config c2 --levels 2,3 > /dev/null 2>&1
HX_ZONE_FUSE=0 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.per_cycle_active --clock-control none --kernel-name regex:"zone_" -c 40 --csv --log-file gpurun_out/zone_l0.csv python tools/profile_run.py --config c2 --levels 2,3 > /dev/null 2>&1
