for args in "--workload C5" "--workload C5 --no-fused" "--workload C3" "--workload C3 --no-fused"; do
  n=$(echo $args | tr -d ' -')
  timeout 900 python bench.py $args --no-cpu-baseline --steps 10 > gpurun_out/b_$n.json 2> gpurun_out/b_$n.err; echo "$args rc=$?"
  python - $n <<'PY'
import json, sys
f = sys.argv[1]
d = json.loads(open(f"gpurun_out/b_{f}.json").read().strip().splitlines()[-1])
print(f, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x, 4) for k, x in d["per_kernel_ms"].items()}, {k: round(x) for k, x in d["per_kernel_gbs"].items()}, round(d["e2e"]["value"]), d["roofline"]["frac"])
PY
done
