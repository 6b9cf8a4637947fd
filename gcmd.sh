set -x
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gpu_all.log
timeout 300 python tools/profile_run.py --config c2 --warm 1 --passes 2 > gpurun_out/prof0.log 2>&1; echo rc=$?
HX_PANEL_CLUSTER=1 timeout 300 python tools/profile_run.py --config c2 --warm 1 --passes 2 > gpurun_out/prof1.log 2>&1; echo rc=$?
tail -12 gpurun_out/prof0.log gpurun_out/prof1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_p0.csv python tools/profile_run.py --config c2 > /dev/null 2>&1; echo ncu0=$?
HX_PANEL_CLUSTER=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_p1.csv python tools/profile_run.py --config c2 > /dev/null 2>&1; echo ncu1=$?
