# C2 chained (PDL) fused kernel: shared-memory budget per CTA (CS_FUSED_SMEM_KB) x chain depth sweep, A/B on one box.
# usage: bash scripts/gpu_c2_budget.sh   (outputs in gpurun_out/c2b/)
O=gpurun_out/c2b; mkdir -p $O
LIB=paper_2604_06036_b200/libcodecsight.so
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
cp $LIB $O/base.so
for kb in ${KBS:-56 68 84 100}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DCS_FUSED_SMEM_KB=${kb}u \
    -I include -o $O/b$kb.so paper_2604_06036_b200/csrc/*.cu > $O/b$kb.build 2>&1 || { echo "b$kb build failed"; continue; }
done
for rnd in 1 2; do
  for kb in ${KBS:-56 68 84 100}; do
    cp $O/b$kb.so $LIB; touch $LIB
    for dep in ${DEPS:-3 4}; do
      timeout 300 python bench.py --workload C2 --chain-depth $dep --no-cpu-baseline --no-e2e --steps 50 > $O/b$kb.d$dep.$rnd.json 2>/dev/null
      python - $O/b$kb.d$dep.$rnd.json $kb $dep <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
print("kb", sys.argv[2], "depth", sys.argv[3], "us %.1f" % (d["ms_per_step"] * 1e3), "frac %.3f" % d["roofline"]["frac"])
PY
    done
  done
done
cp $O/base.so $LIB; touch $LIB
