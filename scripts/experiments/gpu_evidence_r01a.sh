# Round evidence: smoke, all GPU tests, every bench line, ncu launch list + full captures.  Outputs in gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > gpurun_out/gpu_info.txt
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4 rc=$?
timeout 900 python bench.py --kv-mode copy --no-cpu-baseline > gpurun_out/bench_c4_copy.json 2> gpurun_out/bench_c4_copy.err
timeout 900 python bench.py --rope mrope --no-cpu-baseline > gpurun_out/bench_c4_mrope.json 2> gpurun_out/bench_c4_mrope.err
timeout 900 python bench.py --frames nv12 --no-cpu-baseline > gpurun_out/bench_c4_nv12.json 2> gpurun_out/bench_c4_nv12.err
timeout 1200 python bench.py --workload C5 --steps 20 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5 rc=$?
timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --cpu-seconds 6 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --quiet"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'score_kernel|compact_|kv_' --csv --log-file gpurun_out/ncu_launches.csv $B > /dev/null 2>gpurun_out/ncu_launches.err
echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kv_gather_tma' -s 1 -c 1 -o gpurun_out/prof_kv $B --streams 64 > /dev/null 2>gpurun_out/ncu_kv.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel|compact_' -s 3 -c 3 -o gpurun_out/prof_sc $B > /dev/null 2>gpurun_out/ncu_sc.err
echo full rc=$?
