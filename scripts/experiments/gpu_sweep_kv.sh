# sweep of the TMA ring geometry (warps per CTA, stage KB, stages) on the C4 bench, both KV modes
for cfg in "8,8,3" "8,6,4" "8,4,6" "4,16,3" "4,12,4" "4,8,6" "6,8,4" "2,16,6"; do
  for m in paged copy; do
    CS_KV_TMA=$cfg timeout 300 python bench.py --kv-mode $m --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/s.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/s.json')); print('$cfg', '$m', round(d['per_kernel_ms']['kv_refresh'],3), round(d['roofline']['frac'],4))"
  done
done
