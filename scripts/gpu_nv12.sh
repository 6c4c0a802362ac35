# NV12 fused-preprocessing check: build, the NV12 parity tests, the C4 NV12 bench line, one full ncu capture of the
# staged kernel.  Outputs in gpurun_out/${NV_OUT:-nv}/.
O=gpurun_out/${NV_OUT:-nv}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "nv12" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -1 $O/pytest.log
timeout 600 python bench.py --frames nv12 --no-cpu-baseline > $O/bench_nv12.json 2>$O/nv12.err; echo bench rc=$?
python - $O/bench_nv12.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
print("ms/step %.3f" % d["ms_per_step"], "nv12", d["compact_by_layout"], "frac %.3f" % d["secondary_roofline"]["frac"])
PY
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:compact_nv12_staged -s 3 -c 1 -o $O/prof \
  python bench.py --frames nv12 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet > $O/ncu.log 2>&1; echo ncu rc=$?
fi
