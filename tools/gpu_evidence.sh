#!/bin/bash
# ncu evidence for one cfg3 step (run under gpurun; one GPU):
#   1. launch list of the bench command itself (gpu__time_duration.sum per launch)
#   2. --set full captures of the largest launch of each DMMA kernel and of the
#      pipelined PGS kernel, picked from a launch list of tools/profile_step.py
set -u
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-cfg1-pair > gpurun_out/ev_plain.json 2> gpurun_out/ev_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_bench_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-cfg1-pair > gpurun_out/ev_bench_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_step_launches.csv \
  python tools/profile_step.py 1 > gpurun_out/ev_step_ncu.log 2>&1
for k in syrk_kernel panel_mma_kernel gram_kernel pgs_pipe_kernel; do
  idx=$(python - "$k" <<'PY'
import csv, sys
name = sys.argv[1]
rows = list(csv.reader(open("gpurun_out/ev_step_launches.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
t = [float(r[vi].replace(",", "")) for r in rows[h + 1:] if len(r) > vi and r[ki].split("(")[0].replace("void ", "").endswith(name)]
print(max(range(len(t)), key=t.__getitem__) if t else 0)
PY
)
  echo "$k largest launch index $idx" >> gpurun_out/ev_pick.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s "$idx" -c 1 -f \
    -o gpurun_out/ev_$k python tools/profile_step.py 1 > gpurun_out/ev_$k.log 2>&1
done
echo done >> gpurun_out/ev_pick.log
