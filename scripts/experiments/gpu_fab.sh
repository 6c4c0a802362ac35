for args in "--workload C4" "--workload C5" "--workload C3" "--workload C2"; do
  timeout 900 python bench.py $args --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/fab.json 2> gpurun_out/fab.err
  python - "$args" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/fab.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]), round(d["ms_per_step"], 4), {k: round(x, 4) for k, x in d["per_kernel_ms"].items()})
PY
done
