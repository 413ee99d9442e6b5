# cfg4 evidence: launch list of one bench run (timed region inclusive) and a full
# capture of one batched PGS launch (a late Newton iteration)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/cfg4_launches.csv python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4_ncu_bench.log 2>&1
echo "launches exit $?" >> gpurun_out/cfg4_ncu_bench.log
timeout 900 ncu --kernel-name regex:pgs_copy_kernel --launch-skip 34 --launch-count 1 --set full --clock-control none \
  --import-source on -o gpurun_out/cfg4_pgs_copy_full -f python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4_ncu_full.log 2>&1
echo "full exit $?" >> gpurun_out/cfg4_ncu_full.log
