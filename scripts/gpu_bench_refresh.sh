# Re-run the bench lines a bench.py change affects (outputs in gpurun_out/br/; copy into profiles/r02_bench_*.json)
O=gpurun_out/br; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err; echo "bench $n rc=$?"; }
run c2_nopdl --workload C2 --no-pdl --no-cpu-baseline
run c4_seq --no-overlap --no-cpu-baseline
run c5_seq --workload C5 --steps 20 --no-overlap --no-cpu-baseline
run c4_tp2 --temporal-patch 2 --no-cpu-baseline
