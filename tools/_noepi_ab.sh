run() { timeout 300 "$@" 2>&1 | grep '^{' ; }
for rep in 1 2; do
echo "## base_$rep"; run python tools/quick_bench.py 3 4
echo "## noepi_$rep"; run python tools/variant.py noepi tools/quick_bench.py 3 4
done
