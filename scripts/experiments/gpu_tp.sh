# full GPU tests + the default bench + the temporal-patch bench (1 GPU)
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
timeout 600 python bench.py --temporal-patch 2 --no-cpu-baseline > gpurun_out/bench_tp2.json 2> gpurun_out/bench_tp2.err; echo bench tp2 rc=$?
tail -2 gpurun_out/bench_tp2.err
python - <<'PY'
import json
for f in ["bench_default", "bench_tp2"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["value"]), d["ms_per_step"], d["per_kernel_ms"], d["roofline"]["frac"], d["compact_by_layout"], d.get("e2e", {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
