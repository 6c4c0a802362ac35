# Build libcodecsight.so variants (extra nvcc -D flags) and time the C4 NV12 bench with each.
# usage: VARIANTS="name1:-DA=1 -DB=2;name2:-DA=2" [BASE_ARGS="--frames nv12"] [ARGS=...] [PYTEST=0] bash scripts/gpu_variants.sh
# (outputs in gpurun_out/var/)
O=gpurun_out/var; mkdir -p $O
LIB=paper_2604_06036_b200/libcodecsight.so
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
cp $LIB $O/base.so
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name=${v%%:*}; flags=${v#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $flags \
    -I include -o $O/$name.so paper_2604_06036_b200/csrc/*.cu > $O/$name.build 2>&1 || { echo "$name build failed"; continue; }
  cp $O/$name.so $LIB; touch $LIB
  pr=skip; if [ "${PYTEST:-1}" = 1 ]; then timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "nv12" > $O/$name.pytest 2>&1; pr=$?; fi
  timeout 600 python bench.py ${BASE_ARGS---frames nv12} --no-cpu-baseline --steps 10 $ARGS > $O/$name.json 2>$O/$name.err
  python - $O/$name.json "$name" $pr <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
    print(sys.argv[2], "pytest rc", sys.argv[3], "ms/step %.3f" % d["ms_per_step"], "nv12 %.4f ms" % d["compact_by_layout"].get("nv12_fused", {}).get("ms", 0), "kv %.3f GB/s" % d["kv_refresh_gbs"], "value %.0f" % d["value"])
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
cp $O/base.so $LIB; touch $LIB
