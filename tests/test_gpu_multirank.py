"""The N > 1 path with the product kernels, on the one GPU a test box has: two processes over gloo,
both on cuda:0, each running the bench's Pipeline (fused score+compact, paged KV refresh, pipelined steps) on its
snake-order shard of the streams, then reducing the u64 counters (SUM) exactly as bench.py does.  The ranks' kernels
never wait on each other (no data-path collective), so sharing one GPU changes nothing but the timing, which is not
checked here.  The reduced counters and each stream's keep masks and KV slot maps must equal one process running every
stream."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_STREAMS, W, S, GOP, STEPS = 6, 8, 2, 4, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(ids, overlap):
    """Run the Pipeline over global stream ids; return (counters, {sid: (mask_ring, slot_map)})."""
    import synth
    from paper_2604_06036_b200 import _abi as abi
    from paper_2604_06036_b200.pipeline import Pipeline
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS["C1"]
    g = synth.make_grid(448, 448)
    kv = dict(synth.TOY_KV)
    n = len(ids)
    pipe = Pipeline(g, n, W, S, GOP, kv, n_prompt=4, device=dev, frame_layout=abi.CS_LAYOUT_GROUPED,
                    kv_mode="paged", compact_chunk=S, fused=True, overlap=overlap)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    pipe.init_cache_fill(gen)
    meta = {sid: synth.stream_metadata(448, 448, synth.scene_of(cfg, sid), synth.stream_seed(cfg, sid),
                                       W + S * STEPS) for sid in ids}
    frame = torch.zeros(3 * 448 * 448, dtype=torch.bfloat16, device=dev)
    for k in range(STEPS):
        f0, nf = pipe.new_frames(k)
        mb = np.stack([meta[sid][f0:f0 + nf] for sid in ids])
        types = np.stack([synth.frame_types(nf, GOP, f0)] * n)
        ptrs = abi.ptr_array([frame] * (n * nf), dev)
        fidx = np.tile(np.arange(f0, f0 + nf, dtype=np.int32), n)
        pipe.step(k, torch.from_numpy(mb.view(np.uint8)).to(dev), ptrs, torch.from_numpy(fidx).to(dev),
                  torch.from_numpy(types).to(dev))
    pipe.join()
    torch.cuda.synchronize()
    assert int(pipe.status.item()) == 0
    masks = pipe.mask_ring.cpu().numpy()
    slots = pipe.slots[pipe.cur].cpu().numpy()
    per = {sid: (masks[i].copy(), slots[i].copy()) for i, sid in enumerate(ids)}
    return pipe.counters.cpu().numpy().astype(np.int64), per


def _worker(rank, world, port, q, overlap):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_06036_b200 import shard
    ids = shard.shard_ids(rank, world, N_STREAMS, "strong")
    cnt, per = _run(ids, overlap)
    tot = shard.reduce_counters(torch.from_numpy(cnt))  # (gloo on CPU tensors; NCCL on a multi-GPU box)
    q.put((rank, ids, tot.numpy().tolist(), {sid: (m.tolist(), s.tolist()) for sid, (m, s) in per.items()}))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,overlap", [(2, True), (3, False)])
def test_multirank_product_path_equals_single_process(world, overlap):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, overlap)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref_cnt, ref_per = _run(list(range(N_STREAMS)), overlap)
    owned = sorted(sum((ids for _, ids, _, _ in res), []))
    assert owned == list(range(N_STREAMS))              # the shards partition the streams
    for _, _, tot, per in res:
        assert tot == ref_cnt.tolist()                   # every rank holds the same reduced counters
        for sid, (m, s) in per.items():
            assert np.array_equal(np.array(m, np.int64), ref_per[sid][0].astype(np.int64))
            assert np.array_equal(np.array(s), ref_per[sid][1])
