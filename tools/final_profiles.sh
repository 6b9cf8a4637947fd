#!/bin/bash
# Regenerates the measured artefacts of the current build on the GPU box (-> gpurun_out/, copied to profiles/):
# executed-FP64 profiles (c2 pass, c2 N = 2048 tier, c5 per matrix size), bench lines of every config, the
# reference arm, and the ncu launch list of the bench command.   bash tools/final_profiles.sh [quick]
cd $GRAFT_REPO_ROOT
OUT=gpurun_out
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum
run() {  # name label args...
  local name=$1 label=$2; shift 2
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $OUT/fp64_$name.csv python tools/profile_run.py "$@" > /dev/null 2>&1
  python tools/ncu_flops.py $OUT/fp64_$name.csv --json $OUT/r02_fp64_executed_$name.json --label "$label" > $OUT/r02_fp64_executed_$name.txt
}
run c2 "c2 one level set as the bench step submits it (tools/profile_run.py --config c2 --concurrent: run_levels, same-cell small tiers deduplicated together), serialised under ncu" --config c2 --concurrent
run c2_L4_parent "c2 level 4 parent tier (N = 2048, 64 matrices at Gamma), tools/profile_run.py --config c2 --levels 4 --parent-only" --config c2 --levels 4 --parent-only
ARGS=""
for nb in 32:20000 64:5000 128:2000 256:500 512:200 1024:50 2048:16; do
  n=${nb%%:*}; b=${nb##*:}
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file $OUT/fp64_c5_n$n.csv python tools/c5_sample.py --n $n --batch $b > /dev/null 2>&1
  python tools/ncu_flops.py $OUT/fp64_c5_n$n.csv --json $OUT/c5_n$n.json --label "c5 n=$n batch=$b (tools/c5_sample.py), serialised under ncu" > $OUT/r02_fp64_executed_c5_n$n.txt
  ARGS="$ARGS $n:$b:$OUT/c5_n$n.json"
done
python tools/c5_exec_json.py $OUT/r02_fp64_executed_c5.json $ARGS
# the bench reads profiles/: refresh them before the bench lines
cp $OUT/r02_fp64_executed_c2.json $OUT/r02_fp64_executed_c2_L4_parent.json $OUT/r02_fp64_executed_c5.json profiles/
timeout 900 python bench.py > $OUT/r02_bench_c2.json 2> $OUT/r02_bench_c2.err
timeout 900 python bench.py --impl reference > $OUT/r02_bench_ref_c2.json 2> $OUT/r02_bench_ref_c2.err
for c in c1 c3 c4 c5; do
  timeout 1500 python bench.py --config $c > $OUT/r02_bench_$c.json 2> $OUT/r02_bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file $OUT/launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_bench_c2.log 2>&1
python tools/ncu_summary.py $OUT/launches_bench_c2.csv > $OUT/r02_launches_bench_c2.txt 2>&1
for c in c1 c2 c3 c4 c5; do python -c "
import json,sys
d=json.load(open('$OUT/r02_bench_$c.json')); print('$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d.get('cpu_baseline',{}).get('value'))"; done
cat $OUT/r02_bench_ref_c2.json | head -c 600
