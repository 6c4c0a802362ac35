# Default bench lines after a change of defaults: C4, C5, C3, C2, NV12, the 2-rank shared-GPU strong-scaling path
# and the pipeline GPU tests.  Outputs in gpurun_out/def/.
O=gpurun_out/def; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "pipeline" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest.log
run() { n=$1; shift; timeout 900 python bench.py --no-cpu-baseline "$@" > $O/$n.json 2> $O/$n.err; echo "$n rc=$?"; }
run c4; run c5 --workload C5 --steps 20; run c3 --workload C3; run c2 --workload C2; run nv12 --frames nv12; run c4_seq --no-overlap
export CS_BENCH_SHARED_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/mr.json 2> $O/mr.err; echo mr rc=$?
unset CS_BENCH_SHARED_GPU
for f in $O/*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
    print("%-22s %10.0f frames/s  ms %.4f  overlap %s  e2e %.0f  frac %.3f step %.3f per_rank %s" % (sys.argv[1].split("/")[-1], d["value"], d["ms_per_step"], d["config"].get("overlap"), d["e2e"]["value"], d["roofline"]["frac"], d["step_roofline"]["frac"], [round(r["ms_per_step"], 3) for r in d["per_rank"]]))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
