O=gpurun_out/r02f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 180 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "pdl" > $O/pytest_pdl.log 2>&1; echo pytest_pdl rc=$?
tail -3 $O/pytest_pdl.log
timeout 120 python scripts/pdl_timing.py > $O/pdl_timing.txt 2>&1; echo timing rc=$?; cat $O/pdl_timing.txt
run() { n=$1; shift; timeout 300 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err; echo "bench $n rc=$?"; }
run c2 --workload C2 --no-cpu-baseline
run c2_pdl --workload C2 --pdl --no-cpu-baseline

for f in c2 c2_pdl; do python - $f <<'PY'
import json, sys
d=json.loads([l for l in open(f"gpurun_out/r02f/bench_{sys.argv[1]}.json") if l.startswith("{")][-1])
print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],4), d["per_kernel_ms"], "roof", round(d["roofline"]["frac"],3), "sec", round(d["secondary_roofline"]["frac"],3), "e2e", round(d.get("e2e",{}).get("value",0)))
PY
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "pipeline or score_compact" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest.log
