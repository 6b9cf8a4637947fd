#!/bin/bash
set -x
timeout 900 python -m pytest tests/test_multirank_gpu.py -q -x > gpurun_out/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest.log
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum
args=""
for nb in 32:20000 64:5000 128:2000 256:500 512:200 1024:50 2048:16; do
  n=${nb%%:*}; b=${nb##*:}
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/fp64_c5_$n.csv python tools/c5_sample.py --n $n --batch $b > /dev/null 2>&1
  python tools/ncu_flops.py gpurun_out/fp64_c5_$n.csv 10 --json gpurun_out/fp64_c5_$n.json > gpurun_out/fp64_c5_$n.txt
  args="$args $n:$b:gpurun_out/fp64_c5_$n.json"
done
python tools/c5_exec_json.py gpurun_out/r02_fp64_executed_c5.json $args > gpurun_out/c5_exec.log 2>&1
cp gpurun_out/r02_fp64_executed_c5.json profiles/
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config c1 --steps 2000 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
