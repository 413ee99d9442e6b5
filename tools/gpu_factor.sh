#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/factor_profile.py > gpurun_out/factor.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/factor_launches.csv python tools/factor_profile.py --reps 1 > gpurun_out/factor_ncu.log 2>&1
