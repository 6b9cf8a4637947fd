set -x
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum
timeout 300 python -m pytest tests/test_device_pipeline_gpu.py -x -q > gpurun_out/devpipe.log 2>&1; echo "exit $?" >> gpurun_out/devpipe.log
for c in c2 c1 c3 c4; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/fp64_$c.csv python tools/profile_run.py --config $c > gpurun_out/fp64_$c.log 2>&1
  python tools/ncu_flops.py gpurun_out/fp64_$c.csv 25 --json gpurun_out/r02_fp64_executed_$c.json --label "$c one pass (tools/profile_run.py --config $c), serialised under ncu" > gpurun_out/r02_fp64_executed_$c.txt 2>&1
done
timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/fp64_c2_L4.csv python tools/profile_run.py --config c2 --levels 4 --parent-only > gpurun_out/fp64_c2_L4.log 2>&1
python tools/ncu_flops.py gpurun_out/fp64_c2_L4.csv 25 --json gpurun_out/r02_fp64_executed_c2_L4_parent.json --label "c2 level-4 parent tier (N=2048, 64 masks at Gamma), one hx_eval_idos_batch_device" > gpurun_out/r02_fp64_executed_c2_L4_parent.txt 2>&1
cp gpurun_out/r02_fp64_executed_*.json profiles/
timeout 400 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches.log 2>&1
