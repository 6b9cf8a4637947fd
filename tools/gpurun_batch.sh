#!/bin/bash
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum
for c in c2; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/fp64_$c.csv python tools/profile_run.py --config $c > /dev/null 2>&1
  python tools/ncu_flops.py gpurun_out/fp64_$c.csv 25 --json gpurun_out/r02_fp64_executed_$c.json --label "$c one pass (tools/profile_run.py --config $c), serialised under ncu" > gpurun_out/r02_fp64_executed_$c.txt 2>&1
done
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/fp64_c2_L4.csv python tools/profile_run.py --config c2 --levels 4 --parent-only > /dev/null 2>&1
python tools/ncu_flops.py gpurun_out/fp64_c2_L4.csv 25 --json gpurun_out/r02_fp64_executed_c2_L4_parent.json --label "c2 level-4 parent tier (N=2048, 64 masks at Gamma), one hx_eval_idos_batch_device" > gpurun_out/r02_fp64_executed_c2_L4_parent.txt 2>&1
args=""
for nb in 32:20000 64:5000 128:2000 256:500 512:200 1024:50 2048:16; do
  n=${nb%%:*}; b=${nb##*:}
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/fp64_c5_$n.csv python tools/c5_sample.py --n $n --batch $b > /dev/null 2>&1
  python tools/ncu_flops.py gpurun_out/fp64_c5_$n.csv 10 --json gpurun_out/fp64_c5_$n.json > gpurun_out/r02_fp64_executed_c5_n$n.txt
  args="$args $n:$b:gpurun_out/fp64_c5_$n.json"
done
python tools/c5_exec_json.py gpurun_out/r02_fp64_executed_c5.json $args > gpurun_out/c5_exec.log 2>&1
rm -f gpurun_out/fp64_*.csv
