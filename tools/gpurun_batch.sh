#!/bin/bash
cd $GRAFT_REPO_ROOT
for m in "" "0,1,2,0,1,2,1" "0,1,2,0,0,1,2" "0,1,2,1,2,0,0" "0,1,1,2,2,2,2" "0,1,2,3,3,1,2" "0,1,2,2,1,1,2"; do
  HX_LANE_MAP=$m timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 12 > gpurun_out/lm.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/lm.json')); print('map [$m]', round(d['value']), round(d['ms_per_step'],2))"
done
