# C2 (32 x 1080p streams, prune + compact only): where the fused kernel's time goes
O=gpurun_out/c2; mkdir -p $O
timeout 600 python bench.py --workload C2 --no-fused --no-cpu-baseline > $O/bench_c2_nofused.json 2> $O/b1.err; echo nofused rc=$?
timeout 600 python bench.py --workload C2 --no-cpu-baseline > $O/bench_c2.json 2> $O/b2.err; echo fused rc=$?
B="python bench.py --workload C2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches.csv $B > /dev/null 2>$O/l.err; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 3 -c 1 -o $O/prof_fused $B > /dev/null 2>$O/f.err; echo fused full rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel|compact_gather' -s 3 -c 2 -o $O/prof_two $B --no-fused > /dev/null 2>$O/t.err; echo two full rc=$?
