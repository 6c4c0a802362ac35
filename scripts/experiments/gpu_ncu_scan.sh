B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet --no-fused"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'compact_scan' -s 3 -c 1 -o gpurun_out/prof_scan $B > /dev/null 2>gpurun_out/ncu_scan.err
echo rc=$?
