timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "kv or paged or mrope or pipeline or temporal or fullsize" > gpurun_out/pytest_mr.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_mr.log
for args in "--rope mrope" "--rope mrope --kv-mode copy" "--rope mrope --workload C5"; do
  n=$(echo $args | tr -d ' -')
  timeout 900 python bench.py $args --no-cpu-baseline --steps 10 > gpurun_out/b_$n.json 2> gpurun_out/b_$n.err; echo "$args rc=$?"
  python - $n <<'PY'
import json, sys
f = sys.argv[1]
d = json.loads(open(f"gpurun_out/b_{f}.json").read().strip().splitlines()[-1])
print(f, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x, 4) for k, x in d["per_kernel_ms"].items()}, {k: round(x) for k, x in d["per_kernel_gbs"].items()}, round(d["e2e"]["value"]), round(d["roofline"]["frac"], 3))
PY
done
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet --rope mrope --streams 64"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'kv_gather' --csv --log-file gpurun_out/ncu_mrope.csv $B > /dev/null 2>gpurun_out/ncu_mrope.err; echo ncu rc=$?
grep kv_gather gpurun_out/ncu_mrope.csv | tail -6
