set -x
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --quiet"
python scripts/copy_ref.py 2 > gpurun_out/copy_ref.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kv_gather' -s 1 -c 1 -o gpurun_out/prof_kv64 $B --streams 64 > /dev/null 2>gpurun_out/ncu_kv.err
echo kv rc=$?
timeout 600 ncu --set full --clock-control none -k regex:'copy|elementwise' -s 3 -c 1 -o gpurun_out/prof_copy python scripts/copy_ref.py 2 > /dev/null 2>gpurun_out/ncu_copy.err
echo copy rc=$?
cat gpurun_out/copy_ref.txt
