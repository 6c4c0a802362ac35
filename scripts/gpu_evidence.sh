# Final round-1 evidence for the current code: smoke, all GPU tests, every bench line, ncu launch lists (C4, C5, C2,
# C3) and full captures of the hot kernels.  Outputs in gpurun_out/evidence/.
O=gpurun_out/evidence; mkdir -p $O
nproc > $O/host.txt; grep -m1 "model name" /proc/cpuinfo >> $O/host.txt
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
run c4_graphs --graphs --no-cpu-baseline
run c5 --workload C5 --steps 20
run c3 --workload C3 --no-cpu-baseline
run c2 --workload C2 --no-cpu-baseline
run c2_graphs --workload C2 --graphs --no-cpu-baseline
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --cpu-seconds 6 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref rc=$?
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'score_kernel|compact_|kv_' --csv --log-file $O/ncu_launches_c4.csv $B > /dev/null 2>$O/l4.err; echo l4 rc=$?
for w in C5 C3 C2; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'score_kernel|compact_|kv_' --csv --log-file $O/ncu_launches_$w.csv $B --workload $w > /dev/null 2>$O/l_$w.err; echo l $w rc=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kv_gather_tma' -s 3 -c 1 -o $O/prof_kv_c4 $B > /dev/null 2>$O/f1.err; echo kv4 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 3 -c 1 -o $O/prof_fused_c4 $B > /dev/null 2>$O/f2.err; echo fused4 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 3 -c 1 -o $O/prof_fused_c2 $B --workload C2 > /dev/null 2>$O/f3.err; echo fused2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kv_gather_tma|score_kernel' -s 6 -c 2 -o $O/prof_c3 $B --workload C3 > /dev/null 2>$O/f4.err; echo c3 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kv_plan_paged|kv_prefix' -s 2 -c 2 -o $O/prof_plan_c4 $B > /dev/null 2>$O/f5.err; echo plan rc=$?
timeout 600 python scripts/phase_timing.py run > $O/phase.txt 2>&1; echo phase rc=$?
ls $O | wc -l
