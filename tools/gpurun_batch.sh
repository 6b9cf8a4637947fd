#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
i=0
for M in 0,1,2,1,2,0,0 0,1,2,0,1,2,0 0,1,2,0,1,2,1 0,1,2,1,2,0,1 0,1,2,3,3,0,1 0,1,2,0,1,0,1; do
i=$((i+1))
HX_LANE_MAP=$M python tools/timeline.py --config c2 > gpurun_out/timeline_c2_M$i.txt 2>&1
echo $M >> gpurun_out/timeline_c2_M$i.txt
done
