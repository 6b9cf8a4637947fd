#!/bin/bash
cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 12 > gpurun_out/kn.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/kn.json')); print('$*', round(d['value']), round(d['ms_per_step'],2))"; }
run A=1
run HX_CHASE_SPIN_NS=0
run HX_CHASE_SPIN_NS=50
run HX_CHASE_SPIN_NS=100
run HX_CHASE_SPIN_NS=200
run A=2
