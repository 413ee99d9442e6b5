#!/bin/bash
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv python tools/profile_step.py 1 > gpurun_out/step_ncu.log 2>&1; echo "exit $?" >> gpurun_out/step_ncu.log
