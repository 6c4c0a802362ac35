O=gpurun_out/r02h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pdl" > $O/pytest_pdl.log 2>&1; echo pytest_pdl rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "(compact or pipeline or fullsize or rasterize or cdf) and not pdl" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -2 $O/pytest.log
run() { n=$1; shift; timeout 600 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err; echo "bench $n rc=$?"; }
run c4 --no-cpu-baseline --no-e2e
run c2 --workload C2 --no-cpu-baseline --no-e2e
run c2_pdl --workload C2 --pdl --no-cpu-baseline --no-e2e
run c5 --workload C5 --steps 20 --no-cpu-baseline --no-e2e
run c3 --workload C3 --no-cpu-baseline --no-e2e
for f in c4 c2 c2_pdl c5 c3; do python - $f <<'PY'
import json, sys
d=json.loads([l for l in open(f"gpurun_out/r02h/bench_{sys.argv[1]}.json") if l.startswith("{")][-1])
print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],4), d["per_kernel_ms"], "roof", round(d["roofline"]["frac"],3), "sec", round(d["secondary_roofline"]["frac"],3), d["compact_by_layout"])
PY
done
