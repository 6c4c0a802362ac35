O=gpurun_out/wide; mkdir -p $O
timeout 600 python scripts/phase_timing.py run > $O/phase.txt 2>&1; echo phase rc=$?
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "score_compact or fullsize or smoke" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/pytest.log
for w in C2 C3; do timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/bench_$w.json 2> $O/bench_$w.err; echo $w rc=$?; done
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_C4.json 2> $O/bench_C4.err; echo C4 rc=$?
