#!/bin/bash
# PGS kernels: parity tests, phase profiles of both grid kernels, block-solve microbenchmark.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pgs_pipe.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_pgs.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pgs.log
for k in pipe grid; do
  CNB_PGS_KERNEL=$k CNB_PGS_PROFILE=1 timeout 300 python tools/pgs_profile.py --groups 2000 7500 --sweeps 30 > gpurun_out/pgs_profile_$k.log 2>&1
  CNB_PGS_KERNEL=$k timeout 300 python tools/pgs_profile.py --groups 2000 7500 --sweeps 30 > gpurun_out/pgs_time_$k.log 2>&1
done
timeout 120 python tools/block_solve_bench.py > gpurun_out/block_solve.log 2>&1
