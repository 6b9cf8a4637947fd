#!/bin/bash
cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/kn.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/kn.json')); print('$*', round(d['value']), 'e2e', round(d['e2e']['value']))"; }
run A=1
run HX_E2E_ORDER=big2-then-small
run HX_E2E_ORDER=big2-then-small HX_E2E_WORKERS=5
run A=2
HX_E2E_ORDER=big2-then-small python tools/e2e_prof.py --reps 2 2>&1 | sed -n 24,48p
