run() { timeout 600 "$@" 2>&1 | grep '^{' ; }
for rep in 1 2; do
echo "## oldcost_$rep"; run python tools/variant.py oldcost tools/quick_bench.py 2 3 4
echo "## newcost_$rep"; run python tools/quick_bench.py 2 3 4
for mb in 16 32 64; do echo "## newcost_slice${mb}_$rep"; BCSS_SLICE_MB=$mb run python tools/quick_bench.py 3 4; done
echo "## oldcost_slice32_$rep"; BCSS_SLICE_MB=32 run python tools/variant.py oldcost tools/quick_bench.py 3 4
done
echo "## oldcost_cfg5"; run python tools/variant.py oldcost tools/quick_bench.py 5
echo "## newcost_cfg5"; run python tools/quick_bench.py 5
echo "## newcost_slice32_cfg5"; BCSS_SLICE_MB=32 run python tools/quick_bench.py 5
