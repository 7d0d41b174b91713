python tools/quick_bench.py 4 3 > gpurun_out/fs_base.log 2>&1
for s in 0 1 3 4 7 8 9; do BCSS_FORCE_SHAPE=$s python tools/quick_bench.py 4 3 > gpurun_out/fs_$s.log 2>&1; done
