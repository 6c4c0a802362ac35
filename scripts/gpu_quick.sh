# Quick GPU check of the current tree: build, smoke, GPU tests, the default bench lines and the multi-rank (shared
# GPU, gloo) strong-scaling path.  Outputs in gpurun_out/quick/.
O=gpurun_out/quick; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest_gpu.log
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err; echo "bench $n rc=$?"; }
run c4
run c5 --workload C5 --steps 20 --no-cpu-baseline
run c3 --workload C3 --no-cpu-baseline
run c2 --workload C2 --no-cpu-baseline
export CS_BENCH_SHARED_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/mr_c4_strong.json 2> $O/mr_c4_strong.err; echo mr rc=$?
unset CS_BENCH_SHARED_GPU
for f in $O/bench_*.json $O/mr_c4_strong.json; do echo $f; python - "$f" <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
except Exception as e:
    print("  no line", e); sys.exit()
print("  value %.0f ms/step %.3f scaling %s streams %s kept %.3f frac %.3f step_frac %.3f" % (d["value"], d["ms_per_step"], d["scaling"], d["config"]["streams_total"], d["kept_fraction"], d["roofline"]["frac"], d["step_roofline"]["frac"]))
print("  by scene", {k: round(v, 3) for k, v in d.get("kept_fraction_by_scene", {}).items()}, "per_rank", [round(r["ms_per_step"], 3) for r in d.get("per_rank", [])])
PY
done
