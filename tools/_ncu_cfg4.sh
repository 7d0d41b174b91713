set -u
OUT=gpurun_out
ncu --set full --clock-control none --import-source on --kernel-name regex:level_kernel --launch-skip 21 --launch-count 3 -o /tmp/r02_cfg4_top python tools/profile_cfg.py 4 > $OUT/r02_cfg4_ncu.log 2>&1
echo rc=$?
ncu -i /tmp/r02_cfg4_top.ncu-rep --page raw --csv > $OUT/r02_cfg4_top_raw.csv 2>&1
ncu -i /tmp/r02_cfg4_top.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $OUT/r02_cfg4_top_source_sass.csv.gz
ls -la /tmp/r02_cfg4_top.ncu-rep $OUT
