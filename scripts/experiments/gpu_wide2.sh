O=gpurun_out/wide2; mkdir -p $O
timeout 600 python scripts/phase_timing.py run > $O/phase.txt 2>&1; echo phase rc=$?
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "score" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
for w in C2 C3 C5; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/bench_$w.json 2> $O/bench_$w.err; echo $w rc=$?; done
timeout 600 python bench.py --workload C2 --graphs --no-cpu-baseline --no-e2e > $O/bench_C2g.json 2> $O/bench_C2g.err
timeout 600 python bench.py --workload C2 --no-fused --no-cpu-baseline --no-e2e > $O/bench_C2nf.json 2> $O/bench_C2nf.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_C4.json 2> $O/bench_C4.err; echo C4 rc=$?
timeout 600 python bench.py --no-fused --no-cpu-baseline --no-e2e > $O/bench_C4nf.json 2> $O/bench_C4nf.err; echo C4nf rc=$?
