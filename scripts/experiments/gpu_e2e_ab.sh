for rep in 1 2; do
for f in "--fused" "--no-fused"; do
  timeout 900 python bench.py $f --no-cpu-baseline --steps 30 > gpurun_out/e2e_ab.json 2> gpurun_out/e2e_ab.err
  python - "$f" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/e2e_ab.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]), round(d["e2e"]["value"]), round(d["e2e"]["wall_clock_value"]), round(d["ms_per_step"], 4))
PY
done
done
