# ncu full capture of the fused score+compact kernel at C4 (256 streams) and C2
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet --fused"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 1 -c 1 \
  -o gpurun_out/prof_fused_c4 $B --workload C4 > gpurun_out/ncu_fused_c4.out 2>gpurun_out/ncu_fused_c4.err; echo c4 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 1 -c 1 \
  -o gpurun_out/prof_fused_c2 $B --workload C2 > gpurun_out/ncu_fused_c2.out 2>gpurun_out/ncu_fused_c2.err; echo c2 rc=$?
tail -3 gpurun_out/ncu_fused_c4.err
ls -la gpurun_out/*.ncu-rep
