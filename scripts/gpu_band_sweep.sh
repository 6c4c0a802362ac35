# planar band gather geometry sweep (compile-time macros): C4 planar compaction time
O=gpurun_out/band; mkdir -p $O
SRCS=$(ls paper_2604_06036_b200/csrc/*.cu)
for v in "3 7 2" "5 5 2" "7 4 2" "3 6 3"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include \
    -DCS_BAND_RUN=$1 -DCS_BAND_WARPS=$2 -DCS_BAND_STAGES=$3 -o paper_2604_06036_b200/libcodecsight.so $SRCS > $O/build_$1_$2_$3.log 2>&1 || { echo "build $v failed"; continue; }
  timeout 600 python bench.py --frame-layout planar --no-fused --no-cpu-baseline --no-e2e --steps 20 > $O/b_$1_$2_$3.json 2> $O/b_$1_$2_$3.err
  python - $1 $2 $3 <<'PY'
import json, sys
a = "_".join(sys.argv[1:4])
d=json.loads([l for l in open(f"gpurun_out/band/b_{a}.json") if l.startswith("{")][-1])
print("run/warps/stages", a, "compact ms", round(d["per_kernel_ms"]["compact"],4), "alone planar", round(d["compact_by_layout"]["planar"]["ms"],4), round(d["compact_by_layout"]["planar"]["gbs"]), "GB/s frac", round(d["secondary_roofline"]["frac"],3))
PY
done
python -c "import __graft_entry__ as g; g.build()" > $O/build_default.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "compact and not tp and not nv12" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest.log
