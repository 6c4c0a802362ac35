O=gpurun_out/sp; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 3 -c 1 -o $O/prof_sp_cdf $B --workload cdf > /dev/null 2>$O/f1.err; echo sp rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'score_kernel' -s 3 -c 1 -o $O/prof_sp_nv12 $B --frames nv12 > /dev/null 2>$O/f2.err; echo sp2 rc=$?
