"""N>1 path on CPU: two gloo ranks shard streams round-robin, run the (oracle) path on their shard, and reduce
counters (SUM) and times (MAX); the result must equal one process running every stream."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_2604_06036_b200 import shard

N_STREAMS = 6
N_FRAMES = 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_counters(ids):
    import oracle.ref as ref
    cfg = synth.CONFIGS["C1"]
    g = synth.make_grid(448, 448)
    tot = np.zeros(16, np.uint64)
    for sid in ids:
        mb = synth.stream_metadata(448, 448, synth.scene_of(cfg, sid), synth.stream_seed(cfg, sid), N_FRAMES)
        types = synth.frame_types(N_FRAMES, 4)
        out = ref.score_patches(g, mb[None], types[None], np.zeros((1, 33), np.uint32))
        tot += out["counters"]
    return tot


def _worker(rank, world, port, q, scaling="weak"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = (shard.stream_ids(rank, world, N_STREAMS // world) if scaling == "weak" else
           shard.shard_ids(rank, world, N_STREAMS, "strong"))
    assert all(shard.owner(i, world) == rank for i in ids)
    c = torch.from_numpy(_shard_counters(ids).astype(np.int64))
    tot = shard.reduce_counters(c)
    t = shard.reduce_max(torch.tensor([float(rank + 1)], dtype=torch.float64))
    per = shard.gather_per_rank(torch.tensor([10.0 * rank, float(len(ids))], dtype=torch.float64))
    if rank == 0:
        owned = [(shard.stream_ids(r, world, N_STREAMS // world) if scaling == "weak" else
                  shard.shard_ids(r, world, N_STREAMS, "strong")) for r in range(world)]
        q.put((tot.numpy().tolist(), float(t[0]), sorted(sum(owned, [])), per))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,scaling", [(2, "weak"), (3, "weak"), (2, "strong"), (4, "strong")])
def test_sharded_counters_equal_single_process(world, scaling):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, scaling)) for r in range(world)]
    for p in procs:
        p.start()
    tot, tmax, all_ids, per = q.get(timeout=300)
    # per-rank vectors gathered in rank order (the bench's per-rank times / shard sizes)
    assert [r[0] for r in per] == [10.0 * r for r in range(world)]
    if scaling == "strong":
        assert [int(r[1]) for r in per] == [len(shard.partition(r, world, N_STREAMS)) for r in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all_ids == list(range(N_STREAMS))            # every stream owned exactly once
    assert tmax == float(world)                          # MAX over ranks
    ref_tot = _shard_counters(range(N_STREAMS))
    assert tot == ref_tot.astype(np.int64).tolist()      # SUM of shards == whole job


@pytest.mark.parametrize("n_total,per_rank", [(256, None), (None, 128)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_bench_shards_partition_the_configs(world, n_total, per_rank):
    """C4 (strong: the same 256 streams at every N) and C5 (weak: 128 per GPU, 1,024 at N = 8): every global stream
    id owned by exactly one rank, equal shard sizes, and C4's alternating static / high-motion streams split evenly
    (each rank holds as many of one as of the other)."""
    if n_total is not None:
        shards = [shard.shard_ids(r, world, n_total, "strong") for r in range(world)]
        expect = n_total
    else:
        shards = [shard.shard_ids(r, world, per_rank, "weak") for r in range(world)]
        expect = per_rank * world
    ids = sorted(sum(shards, []))
    assert ids == list(range(expect))
    assert len({len(x) for x in shards}) == 1
    for r, x in enumerate(shards):
        assert all(shard.owner(i, world) == r for i in x)
    if n_total is None and world == 8:
        assert expect == 1024
    if n_total is not None and world > 1:
        cfg = synth.CONFIGS["C4"]
        for x in shards:
            kinds = [synth.scene_of(cfg, i) for i in x]
            assert kinds.count("static") == kinds.count("high") == len(x) // 2
    with pytest.raises(ValueError):
        shard.shard_ids(0, world, 8, "bogus")


def test_bench_scaling_defaults():
    import bench
    ns = type("A", (), {"scaling": None, "tau": 0.25, "alpha": 0.0, "group_size": 2})()
    assert bench.workload("C4", None, "paged", ns)["scaling"] == "strong"
    assert bench.workload("C4", None, "paged", ns)["streams"] == 256
    c5 = bench.workload("C5", None, "paged", ns)
    assert c5["scaling"] == "weak" and c5["streams"] == 128
    ns.scaling = "weak"
    assert bench.workload("C4", None, "paged", ns)["scaling"] == "weak"
