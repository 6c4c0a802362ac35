O=gpurun_out/r02g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "compact and not tp and not nv12 or rasterize or cdf" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head -10
run() { n=$1; shift; timeout 600 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err; echo "bench $n rc=$?"; }
run c4_planar --frame-layout planar --no-fused --no-cpu-baseline --no-e2e
run cdf --workload cdf --steps 20 --no-cpu-baseline
for f in c4_planar cdf; do python - $f <<'PY'
import json, sys
d=json.loads([l for l in open(f"gpurun_out/r02g/bench_{sys.argv[1]}.json") if l.startswith("{")][-1])
print(sys.argv[1], round(d["value"]), round(d["ms_per_step"],4), d["per_kernel_ms"], "roof", round(d["roofline"]["frac"],3))
if "compact_by_layout" in d: print(d["compact_by_layout"], d["secondary_roofline"]["frac"])
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'compact_' --csv --log-file $O/ncu_planar.csv python bench.py --frame-layout planar --no-fused --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet > /dev/null 2>$O/ncu.err; echo ncu rc=$?
