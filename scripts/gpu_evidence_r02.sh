# Round-2 evidence for the current code: smoke, all GPU tests, every bench line, ncu launch lists and full captures
# of the hot kernels, the multi-rank (shared GPU, gloo) strong-scaling path.  Outputs in gpurun_out/ev2/.
O=${EV_OUT:-gpurun_out/ev5}; mkdir -p $O
nproc > $O/host.txt; grep -m1 "model name" /proc/cpuinfo >> $O/host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $O/gpu_info.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -k pdl > $O/pytest_pdl.log 2>&1; echo pytest_pdl rc=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not pdl" > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 $O/pytest_gpu.log
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err; echo "bench $n rc=$?"; }
run c4
run c5 --workload C5 --steps 20
run c3 --workload C3 --no-cpu-baseline
run c2 --workload C2 --no-cpu-baseline
run c2_nopdl --workload C2 --no-pdl --no-cpu-baseline
run c4_seq --no-overlap --no-cpu-baseline
run c5_seq --workload C5 --steps 20 --no-overlap --no-cpu-baseline
run c4_nv12 --frames nv12 --no-cpu-baseline
run c4_tp2 --temporal-patch 2 --no-cpu-baseline
run c4_mrope --rope mrope --no-cpu-baseline
run c4_copy --kv-mode copy --no-cpu-baseline
run c4_planar --frame-layout planar --no-fused --no-cpu-baseline
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"compact_" --csv --log-file $O/ncu_launches_C4planar.csv python bench.py --frame-layout planar --no-fused --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet > /dev/null 2>$O/l_planar.err; echo l planar rc=$?
run c4_graphs --graphs --no-cpu-baseline
run cdf --workload cdf --steps 20
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --cpu-seconds 6 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref rc=$?
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:'score_kernel|compact_|kv_' --csv --log-file $O/ncu_launches_C4.csv $B > /dev/null 2>$O/l4.err; echo l4 rc=$?
for w in C5 C3; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:'score_kernel|compact_|kv_' --csv --log-file $O/ncu_launches_$w.csv $B --workload $w > /dev/null 2>$O/l_$w.err; echo l $w rc=$?
done
timeout 900 ncu --metrics $M --clock-control none -k regex:'score_kernel|compact_|kv_' --csv --log-file $O/ncu_launches_C2.csv $B --workload C2 --no-pdl > /dev/null 2>$O/l_C2.err; echo l C2 rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:'score_kernel' --csv --log-file $O/ncu_launches_C2pdl.csv $B --workload C2 --pdl > /dev/null 2>$O/l_c2pdl.err; echo l c2pdl rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:'compact_|score_kernel|kv_' --csv --log-file $O/ncu_launches_C4nv12.csv $B --frames nv12 > /dev/null 2>$O/l_nv12.err; echo l nv12 rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:'mv_rasterize|score_kernel|similar_hist' --csv --log-file $O/ncu_launches_cdf.csv $B --workload cdf > /dev/null 2>$O/l_cdf.err; echo l cdf rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kv_gather_tma' -s 3 -c 1 -o $O/prof_kv_c4 $B > /dev/null 2>$O/f1.err; echo kv4 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 3 -c 1 -o $O/prof_fused_c4 $B > /dev/null 2>$O/f2.err; echo fused4 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 3 -c 1 -o $O/prof_fused_c2 $B --workload C2 --no-pdl > /dev/null 2>$O/f3.err; echo fused2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'compact_nv12_staged' -s 3 -c 1 -o $O/prof_nv12 $B --frames nv12 > /dev/null 2>$O/f4.err; echo nv12 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'mv_rasterize' -s 3 -c 1 -o $O/prof_rast $B --workload cdf > /dev/null 2>$O/f5.err; echo rast rc=$?
python scripts/sass_summary.py > $O/sass.txt 2>&1
export CS_BENCH_SHARED_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/mr_c4_strong.json 2> $O/mr_c4_strong.err; echo mr rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --cpu-seconds 2 > $O/mr_ref.json 2> $O/mr_ref.err; echo mr_ref rc=$?
ls $O | wc -l
