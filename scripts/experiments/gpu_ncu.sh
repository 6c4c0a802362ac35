# ncu evidence for the bench workload (run under gpurun, 1 GPU).  Outputs land in gpurun_out/.
set -x
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --quiet"
# 1) launch list of the step (cold-cache, serialised; compare SHARES)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'score_kernel|compact_|kv_' --csv --log-file gpurun_out/ncu_launches.csv $B > /dev/null 2>gpurun_out/ncu_launches.err
echo launches rc=$?
# 2) full capture of the top kernels on a 16-stream shard (same kernels, smaller footprint for replay)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'kv_gather|compact_gather|score_kernel' \
  -s 3 -c 3 -o gpurun_out/prof_full $B --streams 16 > /dev/null 2>gpurun_out/ncu_full.err
echo full rc=$?
ls -la gpurun_out/
