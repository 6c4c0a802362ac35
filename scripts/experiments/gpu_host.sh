O=gpurun_out/host; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "pipeline or fullsize or score_compact" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
for w in C2 C3; do timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; echo $w rc=$?; done
timeout 600 python bench.py --workload C2 --graphs --no-cpu-baseline > $O/bench_C2g.json 2> $O/bench_C2g.err
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err; echo C4 rc=$?
