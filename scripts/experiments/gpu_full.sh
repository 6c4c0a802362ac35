# full round check: smoke, all GPU tests, benches (C4 default, C5, C3, C2), ncu launch list + full capture
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4 rc=$?
timeout 1200 python bench.py --workload C5 --steps 20 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5 rc=$?
timeout 900 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3 rc=$?
timeout 900 python bench.py --workload C2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2 rc=$?
timeout 900 python bench.py --kv-mode copy --no-cpu-baseline > gpurun_out/bench_c4_copy.json 2> gpurun_out/bench_c4_copy.err; echo c4copy rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --cpu-seconds 6 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --quiet"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'score_kernel|compact_|kv_' --csv --log-file gpurun_out/ncu_launches.csv $B > /dev/null 2>gpurun_out/ncu_launches.err
echo launches rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'kv_gather|compact_gather|score_kernel|kv_plan' \
  -s 5 -c 4 -o gpurun_out/prof_full $B --streams 32 > /dev/null 2>gpurun_out/ncu_full.err
echo full rc=$?
