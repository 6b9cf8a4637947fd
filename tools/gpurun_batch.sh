#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_variants_gpu.py -q -x -k "small_gram" > gpurun_out/gputest_sg.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_sg.log
tail -4 gpurun_out/gputest_sg.log
python scratch_sg.py
