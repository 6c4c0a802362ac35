# multi-rank bench path on one GPU (gloo, all ranks on GPU 0): sharding, barriers, max-over-ranks, counter reduce
export CS_BENCH_SHARED_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --workload C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mr_ours.json 2> gpurun_out/mr_ours.err; echo ours rc=$?
tail -c 600 gpurun_out/mr_ours.json; echo
tail -3 gpurun_out/mr_ours.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --impl reference --gpus 2 --workload C2 --steps 2 --warmup 1 --cpu-seconds 2 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo ref rc=$?
wc -l gpurun_out/mr_ref.json; tail -c 300 gpurun_out/mr_ref.json
