O=gpurun_out/r02d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pdl or nv12 or rasterize or cdf or score_compact" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest.log
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err; echo "bench $n rc=$?"; }
run c2 --workload C2 --no-cpu-baseline
run c2_pdl --workload C2 --pdl --no-cpu-baseline
run cdf --workload cdf --steps 20 --no-cpu-baseline
for f in c2 c2_pdl cdf; do python - $f <<'PY'
import json, sys
d=json.loads([l for l in open(f"gpurun_out/r02d/bench_{sys.argv[1]}.json") if l.startswith("{")][-1])
print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],4), d["per_kernel_ms"], round(d["roofline"]["frac"],3), "e2e", round(d.get("e2e",{}).get("value",0)))
PY
done
