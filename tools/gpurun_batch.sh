#!/bin/bash
set -x
timeout 300 python tools/e2e_prof.py --config c1 --reps 20 > gpurun_out/e2e_c1.txt 2>&1
