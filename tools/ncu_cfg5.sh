#!/bin/bash
# Config-5 ncu evidence on the GPU box (run from the repo root under gpurun):
# 1. launch list (gpu__time_duration.sum, one metric, no replay);
# 2. --set full of one run's 13 level kernels by application replay (a
#    config-5 kernel can touch ~130 GB of device memory, too much for kernel
#    replay's save/restore), exported to CSV on the box; the .ncu-rep is kept
#    only when it is small enough to travel back.
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/r02_cfg5_launches.csv" \
  python tools/profile_cfg.py 5 > "$OUT/r02_ncu_l.log" 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on --replay-mode application \
  --kernel-name regex:level_kernel --launch-count 13 -o /tmp/r02_cfg5_full \
  python tools/profile_cfg.py 5 --once > "$OUT/r02_ncu_f.log" 2>&1
echo "full capture rc=$?"
ncu -i /tmp/r02_cfg5_full.ncu-rep --page raw --csv > "$OUT/r02_cfg5_full_raw.csv" 2>&1
ncu -i /tmp/r02_cfg5_full.ncu-rep --page details --csv > "$OUT/r02_cfg5_full_details.csv" 2>&1
ls -la /tmp/r02_cfg5_full.ncu-rep
sz=$(stat -c %s /tmp/r02_cfg5_full.ncu-rep)
if [ "$sz" -lt 40000000 ]; then cp /tmp/r02_cfg5_full.ncu-rep "$OUT/"; fi
ncu -i /tmp/r02_cfg5_full.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > "$OUT/r02_cfg5_source_sass.csv.gz"
ls -la "$OUT"
