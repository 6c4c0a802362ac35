# Copy a scripts/gpu_evidence_r02.sh output directory into profiles/ under the round-2 names, with the ncu
# summaries (launch lists, full captures) and profiles/ncu_summary.json rebuilt from it.
# usage: bash scripts/collect_evidence_r02.sh gpurun_out/ev6
set -e
E=${1:?evidence directory}
P=profiles
for n in c4 c4_seq c4_copy c4_mrope c4_nv12 c4_tp2 c4_graphs c4_planar c5 c5_seq c3 c2 c2_nopdl cdf ref; do
  [ -s $E/bench_$n.json ] && cp $E/bench_$n.json $P/r02_bench_$n.json
done
for w in C4 C5 C3 C2 C2pdl C4nv12 C4planar cdf; do
  if [ -s $E/ncu_launches_$w.csv ]; then
    cp $E/ncu_launches_$w.csv $P/r02_ncu_launches_$w.csv
    python scripts/ncu_summary.py launches $E/ncu_launches_$w.csv > $P/r02_ncu_launches_$w.txt
  fi
done
python scripts/ncu_traffic.py $E > $P/ncu_summary.json
for r in kv_c4 fused_c4 fused_c2 nv12 rast; do
  [ -s $E/prof_$r.ncu-rep ] && python scripts/ncu_summary.py report $E/prof_$r.ncu-rep > $P/r02_ncu_full_$r.txt
done
cp $E/sass.txt $P/r02_sass_gpu_box.txt
cp $E/mr_c4_strong.json $P/r02_multirank_snake_shared_gpu.json
cp $E/mr_ref.json $P/r02_multirank_ref.json
(echo "# pytest -m gpu -k pdl"; cat $E/pytest_pdl.log; echo "# pytest -m gpu -k 'not pdl'"; cat $E/pytest_gpu.log) \
  > $P/r02_pytest_gpu.txt
cp $E/smoke.log $P/r02_smoke.txt
cp $E/gpu_info.txt $P/r02_gpu_info.txt
cp $E/host.txt $P/r02_host_cpu.txt
