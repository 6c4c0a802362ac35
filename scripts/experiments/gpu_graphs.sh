for args in "--workload C2" "--workload C2 --graphs" "--workload C4 --graphs" "--workload C3 --graphs"; do
  n=$(echo $args | tr -d ' -')
  timeout 900 python bench.py $args --no-cpu-baseline --steps 30 > gpurun_out/g_$n.json 2> gpurun_out/g_$n.err; echo "$args rc=$?"
  tail -2 gpurun_out/g_$n.err | grep -v "^\[rank"
  python - $n <<'PY'
import json, sys
f = sys.argv[1]
d = json.loads(open(f"gpurun_out/g_{f}.json").read().strip().splitlines()[-1])
print(f, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x, 4) for k, x in d["per_kernel_ms"].items()}, round(d["e2e"]["value"]), d["warmup"], d["status"])
PY
done
