# L2 fetch granularity x workload (outputs in gpurun_out/l2f/)
O=gpurun_out/l2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for rnd in 1 2; do for b in 0 32 64 128; do for w in "mrope:--rope mrope" "c4:"; do
  n=${w%%:*}; a=${w#*:}
  timeout 600 python scripts/l2_fetch_exp.py $b $a --no-cpu-baseline --no-e2e --steps 20 > $O/$n.$b.$rnd.json 2> $O/$n.$b.$rnd.err
  python - $O/$n.$b.$rnd.json $n $b <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
print(sys.argv[2], "l2fetch", sys.argv[3], "ms %.4f" % d["ms_per_step"], "kv frac %.3f" % d["roofline"]["frac"], "fused %.3f" % (d.get("secondary_roofline") or {}).get("frac", 0))
PY
  grep l2_fetch $O/$n.$b.$rnd.err | head -1
done; done; done
