#!/bin/bash
set -x
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_full.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_full.log
tail -5 gpurun_out/gputest_full.log
