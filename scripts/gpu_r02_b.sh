O=gpurun_out/r02b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "nv12 or cdf or misaligned or wide or rne" > $O/pytest.log 2>&1; echo pytest rc=$?
tail -3 $O/pytest.log
run() { n=$1; shift; timeout 1200 python bench.py "$@" > $O/bench_$n.json 2> $O/bench_$n.err; echo "bench $n rc=$?"; }
run c4_nv12 --frames nv12 --no-cpu-baseline
run cdf --workload cdf --steps 20
export CS_BENCH_SHARED_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/mr_c4_strong.json 2> $O/mr_c4_strong.err; echo mr rc=$?
unset CS_BENCH_SHARED_GPU
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'compact_gather' -s 3 -c 1 -o $O/prof_nv12 python bench.py --frames nv12 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --quiet > /dev/null 2>$O/ncu.err; echo ncu rc=$?
