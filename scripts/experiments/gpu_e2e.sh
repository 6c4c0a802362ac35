for args in "--workload C3" "--workload C4" "--workload C2" "--workload C2 --graphs"; do
  timeout 900 python bench.py $args --no-cpu-baseline --steps 30 > gpurun_out/e2e.json 2> gpurun_out/e2e.err
  python - "$args" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/e2e.json").read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]), round(d["e2e"]["value"]), round(d["e2e"]["wall_clock_value"]), d["e2e"]["h2d_bytes_per_step"])
PY
done
