# Evidence pass 2: default bench with the all-cores oracle baseline, reference arm, multi-rank path on one GPU,
# C5 (largest config) ncu launch list and full captures of its two hot kernels.  Outputs in gpurun_out/ev2/.
O=gpurun_out/ev2; mkdir -p $O
nproc > $O/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> $O/nproc.txt; grep MemAvailable /proc/meminfo >> $O/nproc.txt
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; echo c4 rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 --cpu-seconds 6 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref rc=$?
export CS_BENCH_SHARED_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --streams 64 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_shared2.json 2> $O/bench_shared2.err; echo shared2 rc=$?
unset CS_BENCH_SHARED_GPU
B="python bench.py --workload C5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'score_kernel|compact_|kv_' --csv --log-file $O/c5_launches.csv $B > /dev/null 2>$O/c5_l.err; echo c5 launches rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'kv_gather_tma' -s 2 -c 1 -o $O/c5_prof_kv $B > /dev/null 2>$O/c5_kv.err; echo c5 kv full rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 3 -c 1 -o $O/c5_prof_fused $B > /dev/null 2>$O/c5_f.err; echo c5 fused full rc=$?
ls -la $O
