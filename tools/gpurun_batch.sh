#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/inst_c2.csv python tools/profile_run.py --config c2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/inst_c2.csv | head -32
