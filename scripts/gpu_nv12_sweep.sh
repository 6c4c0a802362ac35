# NV12 fused-preprocessing kernel variants (compile-time macros), C4 NV12 bench, compact time in and out of the step
O=gpurun_out/nv12sweep; mkdir -p $O
SRCS=$(ls paper_2604_06036_b200/csrc/*.cu)
for v in "0 4" "1 2" "1 3" "0 3"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include \
    -DCS_NV12_PIPE=$1 -DCS_NV12_CTAS=$2 -o paper_2604_06036_b200/libcodecsight.so $SRCS > $O/build_$1_$2.log 2>&1
  timeout 600 python bench.py --frames nv12 --no-cpu-baseline --no-e2e --steps 20 > $O/bench_$1_$2.json 2> $O/bench_$1_$2.err
  python - $1 $2 <<'PY'
import json, sys
d=json.loads([l for l in open(f"gpurun_out/nv12sweep/bench_{sys.argv[1]}_{sys.argv[2]}.json") if l.startswith("{")][-1])
print("pipe", sys.argv[1], "ctas", sys.argv[2], "compact ms", round(d["per_kernel_ms"]["compact"],4), "alone", round(d["compact_by_layout"]["nv12_fused"]["ms"],4), "frac", round(d["secondary_roofline"]["frac"],3), "step", round(d["ms_per_step"],3))
PY
done
python -c "import __graft_entry__ as g; g.build()" > $O/build_default.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "nv12" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest.log
