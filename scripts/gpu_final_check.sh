# Final-tree check: build, smoke(), pytest -m gpu, default bench line (outputs in gpurun_out/fin/)
O=gpurun_out/fin; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -1 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
python - $O/bench.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
print("bench", round(d["value"]), "frames/s", "%.4f ms" % d["ms_per_step"], "kv %.3f" % d["roofline"]["frac"], "step %.3f" % d["step_roofline"]["frac"], "e2e", round(d["e2e"]["value"]), d["clocks"])
PY
