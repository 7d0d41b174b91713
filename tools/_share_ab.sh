run() { timeout 300 "$@" 2>&1 | grep '^{' ; }
for rep in 1 2; do
echo "## base_$rep"; run python tools/quick_bench.py 3 4
for f in 0.6 0.75 0.85 0.95 1.0; do echo "## share_${f}_$rep"; BCSS_SHARE=$f run python tools/quick_bench.py 3 4; done
done
