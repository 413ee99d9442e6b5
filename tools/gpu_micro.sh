#!/bin/bash
mkdir -p gpurun_out
timeout 200 python tools/dbg_pgs.py > gpurun_out/dbg.log 2>&1
timeout 300 python -m pytest tests/test_gpu_pgs_pipe.py -x -q > gpurun_out/pytest_pgs.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pgs.log
CNB_PGS_PROFILE=1 timeout 300 python tools/pgs_profile.py --groups 7500 --sweeps 30 > gpurun_out/pgs_profile_pipe.log 2>&1
timeout 300 python tools/pgs_profile.py --groups 2000 7500 --sweeps 30 > gpurun_out/pgs_time_pipe.log 2>&1
