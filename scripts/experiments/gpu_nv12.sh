timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "nv12" > gpurun_out/pytest_nv12.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_nv12.log
timeout 600 python bench.py --frames nv12 --no-cpu-baseline --steps 20 > gpurun_out/bench_nv12.json 2> gpurun_out/bench_nv12.err; echo bench rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_nv12.json").read().strip().splitlines()[-1])
print(round(d["value"]), d["ms_per_step"], d["per_kernel_ms"], d["compact_by_layout"])
PY
