#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pgs_pipe_kernel -s 1 -c 1 -o gpurun_out/pgs_pipe python tools/pgs_profile.py --groups 7500 --sweeps 30 --reps 1 > gpurun_out/ncu_pgs.log 2>&1; echo "exit $?" >> gpurun_out/ncu_pgs.log
