for d in 2 3 4 5; do timeout 300 python bench.py --workload C2 --pdl --chain-depth $d --no-cpu-baseline --no-e2e > gpurun_out/d$d.json 2>/dev/null; python - $d <<'PY'
import json, sys
d=json.loads([l for l in open(f"gpurun_out/d{sys.argv[1]}.json") if l.startswith("{")][-1])
print("depth", sys.argv[1], round(d["value"]), round(d["ms_per_step"]*1000,1), "us", round(d["roofline"]["frac"],3))
PY
done
