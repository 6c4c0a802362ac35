O=gpurun_out/nv12; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "nv12" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -1 $O/pytest.log; grep -E "^E  |FAILED" $O/pytest.log | head -8
timeout 600 python bench.py --frames nv12 --no-cpu-baseline --no-e2e --steps 20 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads([l for l in open("gpurun_out/nv12/bench.json") if l.startswith("{")][-1])
print("compact ms", d["per_kernel_ms"]["compact"], "alone", d["compact_by_layout"]["nv12_fused"]["ms"], "frac", d["secondary_roofline"]["frac"], "step", d["ms_per_step"])
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'compact_nv12' --csv --log-file $O/ncu.csv python bench.py --frames nv12 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet > /dev/null 2>$O/ncu.err; echo ncu rc=$?
python scripts/ncu_summary.py launches $O/ncu.csv | head -8
