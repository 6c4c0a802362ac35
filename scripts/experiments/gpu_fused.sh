# fused score+compact vs separate: C4 (default) and C2
for wl in C4 C2; do
  for f in "" "--fused"; do
    timeout 600 python bench.py --workload $wl $f --no-cpu-baseline --steps 30 > gpurun_out/b_${wl}${f}.json 2> gpurun_out/b_${wl}${f}.err; echo "$wl $f rc=$?"
    python - "$wl$f" <<'PY'
import json, sys
f = sys.argv[1]
d = json.loads(open(f"gpurun_out/b_{f}.json").read().strip().splitlines()[-1])
print(f, round(d["value"]), round(d["ms_per_step"], 4), {k: round(v, 4) for k, v in d["per_kernel_ms"].items()},
      {k: round(v) for k, v in d["per_kernel_gbs"].items()}, round(d["e2e"]["value"]))
PY
  done
done
