set -x
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --quiet"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kv_gather_tma' -s 1 -c 1 -o gpurun_out/prof_kvtma $B --streams 64 > /dev/null 2>gpurun_out/ncu_kv.err
echo kv rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel|compact_' -s 3 -c 3 -o gpurun_out/prof_sc $B --streams 256 > /dev/null 2>gpurun_out/ncu_sc.err
echo sc rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
