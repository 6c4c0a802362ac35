timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "compact_tp or temporal" > gpurun_out/pytest_tp.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_tp.log
timeout 600 python bench.py --temporal-patch 2 --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/bench_tp2.json 2> gpurun_out/bench_tp2.err; echo bench tp2 rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_tp2.json").read().strip().splitlines()[-1])
print(round(d["value"]), d["ms_per_step"], d["per_kernel_ms"], d["compact_by_layout"])
PY
