timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "compact or pipeline or nv12 or temporal or smoke" > gpurun_out/pytest_scan.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_scan.log
for args in "--no-fused" "--workload C2 --no-fused" "--temporal-patch 2" "--frames nv12"; do
  timeout 900 python bench.py $args --no-cpu-baseline --steps 20 > gpurun_out/sc.json 2> gpurun_out/sc.err
  python - "$args" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/sc.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]), round(d["ms_per_step"], 4), {k: round(x, 4) for k, x in d["per_kernel_ms"].items()}, {k: (round(v["ms"], 4), round(v["gbs"])) for k, v in d["compact_by_layout"].items()})
PY
done
