mkdir -p gpurun_out
timeout 900 ncu --kernel-name regex:syrk_kernel --launch-skip 300 --launch-count 12 --set full --clock-control none --import-source on -o gpurun_out/syrk_full -f python tools/factor_profile.py --reps 1 > gpurun_out/ncu_syrk.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_syrk.log
