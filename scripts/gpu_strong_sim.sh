# Per-rank work of strong-scaled C4 on one GPU: 256/N streams (N = 1, 2, 4, 8) with the default path, CUDA graphs
# and the overlap mode; ideal per-rank step = (N=1 step) / N.  Outputs in gpurun_out/strong/.
O=gpurun_out/strong; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for S in 256 128 64 32; do
  for v in "base:" "graphs:--graphs" "ovl:--overlap"; do
    n=${v%%:*}; a=${v#*:}
    timeout 600 python bench.py --streams $S --no-cpu-baseline --steps 20 $a > $O/s${S}_$n.json 2>$O/s${S}_$n.err
    python - $O/s${S}_$n.json $S $n <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
    print("streams %s %-7s ms/step %.4f frames/s %.0f e2e %.0f host_enqueue_ms %.3f" % (sys.argv[2], sys.argv[3], d["ms_per_step"], d["value"], d["e2e"]["value"], d.get("host_enqueue_ms_per_step") or 0))
except Exception as e:
    print(sys.argv[2], sys.argv[3], "failed", e)
PY
  done
done
