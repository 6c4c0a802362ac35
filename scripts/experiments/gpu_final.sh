# Round evidence for the current code: smoke, all GPU tests, every bench line, ncu launch list of the default bench
# command and full captures of its kernels.  Outputs in gpurun_out/final/.
mkdir -p gpurun_out/final
O=gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 $O/pytest_gpu.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $O/gpu_info.txt
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err; echo "bench $n rc=$?"; }
run c4 
run c4_nofused --no-fused --no-cpu-baseline
run c4_copy --kv-mode copy --no-cpu-baseline
run c4_mrope --rope mrope --no-cpu-baseline
run c4_nv12 --frames nv12 --no-cpu-baseline
run c4_tp2 --temporal-patch 2 --no-cpu-baseline
run c5 --workload C5 --steps 20
run c3 --workload C3 --no-cpu-baseline
run c2 --workload C2 --no-cpu-baseline
run c2_graphs --workload C2 --graphs --no-cpu-baseline
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --cpu-seconds 6 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref rc=$?
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'score_kernel|compact_|kv_' --csv --log-file $O/ncu_launches.csv $B > /dev/null 2>$O/ncu_launches.err
echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kv_gather_tma' -s 1 -c 1 -o $O/prof_kv $B > /dev/null 2>$O/ncu_kv.err
echo kv full rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 3 -c 1 -o $O/prof_fused $B > /dev/null 2>$O/ncu_fused.err
echo fused full rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kv_plan_paged|kv_prefix' -s 2 -c 2 -o $O/prof_plan $B > /dev/null 2>$O/ncu_plan.err
echo plan full rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'compact_gather' -s 3 -c 1 -o $O/prof_compact $B --no-fused > /dev/null 2>$O/ncu_compact.err
echo compact full rc=$?
ls -la $O
