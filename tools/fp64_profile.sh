#!/bin/bash
# Executed-FP64 profiles of the current build (ncu instruction counts per kernel): c2 pass, c2 N = 2048 tier, c4.
# Run on the GPU box: bash tools/fp64_profile.sh  ->  profiles/r02_fp64_executed_{c2,c2_L4_parent,c4}.{json,txt}
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum
OUT=${1:-gpurun_out}
run() {  # name label args...
  local name=$1 label=$2; shift 2
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $OUT/fp64_$name.csv python tools/profile_run.py "$@" > /dev/null 2>&1
  python tools/ncu_flops.py $OUT/fp64_$name.csv --json $OUT/r02_fp64_executed_$name.json --label "$label" > $OUT/r02_fp64_executed_$name.txt
}
run c2 "c2 one level set as the bench step submits it (tools/profile_run.py --config c2 --concurrent: run_levels, same-cell small tiers deduplicated together), serialised under ncu" --config c2 --concurrent
run c2_L4_parent "c2 level 4 parent tier (N = 2048, 64 matrices at Gamma), tools/profile_run.py --config c2 --levels 4 --parent-only" --config c2 --levels 4 --parent-only
run c4 "c4 one pass (tools/profile_run.py --config c4), serialised under ncu" --config c4
run c3 "c3 one pass (tools/profile_run.py --config c3), serialised under ncu" --config c3
