O=gpurun_out/nv12; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "nv12" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -1 $O/pytest.log
timeout 1200 python bench.py --frames nv12 --no-cpu-baseline --no-e2e --steps 20 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/nv12/bench.json") if l.startswith("{")][-1])
print("compact ms", d["per_kernel_ms"]["compact"], "alone", d["compact_by_layout"]["nv12_fused"]["ms"], "frac", d["secondary_roofline"]["frac"], "step", d["ms_per_step"])
PY
