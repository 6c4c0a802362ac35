# Re-run the pipelined (overlap-mode) bench lines: C4 (with the CPU baselines), C5, C3 and the C4 variants that
# pipeline.  Outputs in gpurun_out/bl/.
O=gpurun_out/bl; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err; echo "bench $n rc=$?"; }
run c4
run c5 --workload C5 --steps 20
run c3 --workload C3 --no-cpu-baseline
run c4_nv12 --frames nv12 --no-cpu-baseline
run c4_mrope --rope mrope --no-cpu-baseline
run c4_copy --kv-mode copy --no-cpu-baseline
run c4_planar --frame-layout planar --no-fused --no-cpu-baseline
