# staged NV12 preprocessing geometry sweep (rows per part, warps per CTA): C4 NV12 compaction time
O=gpurun_out/nvs; mkdir -p $O
SRCS=$(ls paper_2604_06036_b200/csrc/*.cu)
for v in "4 16" "14 8" "4 8" "2 16"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include \
    -DCS_NVS_ROWS=$1 -DCS_NVS_WARPS=$2 -o paper_2604_06036_b200/libcodecsight.so $SRCS > $O/build_$1_$2.log 2>&1 || { echo "build $v failed"; continue; }
  timeout 600 python bench.py --frames nv12 --no-cpu-baseline --no-e2e --steps 20 > $O/b_$1_$2.json 2> $O/b_$1_$2.err
  python - $1 $2 <<'PY'
import json, sys
a = "_".join(sys.argv[1:3])
try:
    d=json.loads([l for l in open(f"gpurun_out/nvs/b_{a}.json") if l.startswith("{")][-1])
    print("rows/warps", a, "compact ms", round(d["per_kernel_ms"]["compact"],4), "alone", round(d["compact_by_layout"]["nv12_fused"]["ms"],4), "frac", round(d["secondary_roofline"]["frac"],3))
except Exception as e:
    print("rows/warps", a, "failed", e)
PY
done
python -c "import __graft_entry__ as g; g.build()" > $O/build_default.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "nv12" > $O/pytest.log 2>&1; echo pytest rc=$?; tail -1 $O/pytest.log
