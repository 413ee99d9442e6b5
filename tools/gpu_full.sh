#!/bin/bash
# full GPU validation: all gpu tests, default bench, PGS profile
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
CNB_PGS_PROFILE=1 timeout 300 python tools/pgs_profile.py --groups 7500 --sweeps 30 > gpurun_out/pgs_profile_pipe.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 900 python bench.py --workload cfg4 --steps 10 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench cfg4 exit $?" >> gpurun_out/bench_cfg4.err
