set -u
O=gpurun_out
(time python -m pytest tests -m gpu -x -q 2>&1 | tail -6) > $O/f_pytest.log 2>&1
python bench.py --steps 20 --warmup 5 > $O/f_bench5.json 2> $O/f_bench5.err
for c in 2 3 4; do python bench.py --config $c --steps 20 --warmup 5 > $O/f_bench$c.json 2> $O/f_bench$c.err; done
python bench.py --impl reference --steps 20 --warmup 5 > $O/f_ref5.json 2> $O/f_ref5.err
bash tools/ncu_cfg5.sh $O > $O/f_ncu5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/f_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/f_ncu_bench.log 2>&1
tail -3 $O/f_pytest.log; for f in $O/f_bench?.json $O/f_ref5.json; do tail -c 300 $f; echo; done
