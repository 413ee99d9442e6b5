mkdir -p gpurun_out
timeout 900 ncu --kernel-name regex:potrf_kernel --launch-skip 600 --launch-count 3 --set full --clock-control none --import-source on -o gpurun_out/potrf_full -f python tools/factor_profile.py --reps 1 > gpurun_out/ncu_potrf.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_potrf.log
