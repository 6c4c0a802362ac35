timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "compact or pipeline" > gpurun_out/pytest_ctma.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_ctma.log
for v in 1 0; do
CS_COMPACT_TMA=$v timeout 600 python bench.py --no-fused --no-cpu-baseline --steps 20 > gpurun_out/bench_ctma$v.json 2> gpurun_out/bench_ctma$v.err; echo bench rc=$?
CS_COMPACT_TMA=$v timeout 600 python bench.py --no-fused --workload C2 --no-cpu-baseline --steps 30 > gpurun_out/bench_ctma_c2_$v.json 2> gpurun_out/bench_ctma_c2_$v.err; echo bench rc=$?
python - $v <<'PY'
import json, sys
v = sys.argv[1]
for f in [f"bench_ctma{v}", f"bench_ctma_c2_{v}"]:
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, round(d["value"]), round(d["ms_per_step"], 4), {k: round(x, 4) for k, x in d["per_kernel_ms"].items()}, {k: round(x) for k, x in d["per_kernel_gbs"].items()}, {k: (round(x["ms"], 4), round(x["gbs"])) for k, x in d["compact_by_layout"].items()})
PY
done
