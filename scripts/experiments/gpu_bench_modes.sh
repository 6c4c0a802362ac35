# bench the C4 workload in both KV modes and C5 (paged), plus C3
set -x
timeout 900 python bench.py --kv-mode paged --cpu-seconds 5 > gpurun_out/bench_c4_paged.json 2> gpurun_out/bench_c4_paged.err; echo rc=$?
timeout 900 python bench.py --kv-mode copy --no-cpu-baseline > gpurun_out/bench_c4_copy.json 2> gpurun_out/bench_c4_copy.err; echo rc=$?
timeout 1200 python bench.py --workload C5 --kv-mode paged --steps 20 --cpu-seconds 10 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo rc=$?
timeout 900 python bench.py --workload C3 --kv-mode paged --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo rc=$?
for f in gpurun_out/bench_c4_paged gpurun_out/bench_c4_copy gpurun_out/bench_c5 gpurun_out/bench_c3; do tail -2 $f.err; python -c "
import json,sys
d=json.load(open('$f.json'))
print('$f', 'value', round(d['value']), 'ms/step', round(d['ms_per_step'],3), 'kv', d['per_kernel_ms'], 'roof', round(d['roofline']['frac'],3), round(d['roofline']['achieved']), 'e2e', round(d.get('e2e',{}).get('value',0)), 'status', d['status'], 'clk', d['clocks'])
"; done
