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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = shard.stream_ids(rank, world, N_STREAMS // world)
    assert all(shard.owner(i, world) == rank for i in ids)
    c = torch.from_numpy(_shard_counters(ids).astype(np.int64))
    tot = shard.reduce_counters(c)
    t = shard.reduce_max(torch.tensor([float(rank + 1)], dtype=torch.float64))
    if rank == 0:
        q.put((tot.numpy().tolist(), float(t[0]), sorted(sum((shard.stream_ids(r, world, N_STREAMS // world)
                                                              for r in range(world)), []))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_counters_equal_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    tot, tmax, all_ids = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all_ids == list(range(N_STREAMS))            # every stream owned exactly once
    assert tmax == float(world)                          # MAX over ranks
    ref_tot = _shard_counters(range(N_STREAMS))
    assert tot == ref_tot.astype(np.int64).tolist()      # SUM of shards == whole job
