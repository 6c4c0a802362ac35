"""Full-size parity in the bench's own launch configuration (BASELINE configs C3, C4 and C5 shapes).

The GPU runs the whole batch of streams exactly as bench.py does (Pipeline, paged KV, grouped frames); the oracle,
which is per-stream independent, re-runs a deterministic sample of streams from the same inputs and every output of
those streams is compared (masks, GOP state, compaction rows of their frames, dispositions, p_old, slot maps and the
pool rows).  Sizes: C4 = 256 1080p streams (w=16, s=4, 28-layer Qwen2-VL-7B KV); C3 = 64 1080p streams (w=32, s=4); C5 = 128 4K
streams (w=64, s=8); fused = the bench's default one-launch score+compact.
"""
import numpy as np
import pytest
import torch

import synth
from synth import make_grid

import kvcheck

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _host(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16) if t.dtype == torch.bfloat16 else t.cpu().numpy()


def to_grouped(frame, g):
    p, G = g["patch"], g["group"]
    ngr, ngc = g["grid_h"] // G, g["grid_w"] // G
    x = frame.reshape(3, ngr, G, p, ngc, G, p)
    return np.ascontiguousarray(x.transpose(1, 4, 2, 5, 0, 3, 6)).reshape(-1)


@pytest.mark.parametrize("cfg_name,S,steps,sample,fused,rope,overlap", [
    ("C4", 256, 3, [0, 1, 254, 255], False, "1d", False),
    ("C4", 256, 3, [0, 1, 254, 255], True, "1d", False),
    ("C4", 256, 4, [0, 1, 254, 255], True, "1d", True),     # the bench's default: pipelined steps (overlap mode)
    ("C4", 256, 3, [0, 255], True, "mrope", False),
    ("C3", 64, 3, [0, 63], True, "1d", True),
    ("C5", 128, 2, [0, 127], False, "1d", False),
    ("C5", 128, 2, [0, 127], True, "1d", True)])
def test_fullsize_sampled_streams(ref, cfg_name, S, steps, sample, fused, rope, overlap):
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    from paper_2604_06036_b200 import _abi as abi
    from paper_2604_06036_b200.pipeline import Pipeline
    cfg = synth.CONFIGS[cfg_name]
    sw, sh = cfg["src"]
    g = make_grid(sw, sh)
    w, s, gop = cfg["window"], cfg["stride"], cfg["gop"]
    kvb = cfg["kv"] if rope == "1d" else synth.QWEN_MROPE_KV   # M-RoPE: the bench's --rope mrope cache (NEXT-3)
    pipe = Pipeline(g, S, w, s, gop, kvb, n_prompt=cfg["n_prompt"], device=DEV,
                    frame_layout=abi.CS_LAYOUT_GROUPED, kv_mode="paged", compact_chunk=s, fused=fused,
                    overlap=overlap)
    ring = pipe.ring  # (w + s; w + 2s in overlap mode)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(11)
    pipe.init_cache_fill(gen)
    gens = [synth.StreamGen(sw, sh, synth.scene_of(cfg, i), synth.stream_seed(cfg, i)) for i in range(S)]
    rng = np.random.default_rng(3)
    # distinct frames for the sampled streams, one shared frame for the others (their pixels are not checked)
    planar = {si: synth.random_frames(w, 448, 448, rng) for si in sample}
    shared = torch.from_numpy(to_grouped(synth.random_frames(1, 448, 448, rng)[0], g).view(np.int16)).to(DEV)
    dev_frames = {si: [torch.from_numpy(to_grouped(f, g).view(np.int16)).to(DEV) for f in planar[si]]
                  for si in sample}
    nw = 32
    st_h = {si: dict(gop=np.zeros((1, nw + 1), np.uint32), mring=np.zeros((1, ring, nw), np.uint32),
                     tring=np.zeros((1, ring), np.uint8), slot=None) for si in sample}
    L = kvb["layers"]
    stats = {}
    for k in range(steps):
        f0, n = pipe.new_frames(k)
        mb = np.stack([np.stack([gn.next_frame() for _ in range(n)]) for gn in gens])
        types = np.stack([synth.frame_types(n, gop, f0)] * S)
        ptr_list = []
        for si in range(S):
            for j in range(n):
                ptr_list.append(dev_frames[si][j % w] if si in sample else shared)
        fptr = abi.ptr_array(ptr_list, DEV)
        fidx = np.tile(np.arange(f0, f0 + n, dtype=np.int32), S)
        pool_before = {si: _host(pipe.caches[0][si]).copy() for si in sample}
        refr = {si: _host(pipe.refreshed[si]) for si in sample}
        pipe.step(k, torch.from_numpy(mb.view(np.uint8)).to(DEV), fptr, torch.from_numpy(fidx).to(DEV),
                  torch.from_numpy(types).to(DEV))
        pipe.join()
        torch.cuda.synchronize()
        assert int(pipe.status.item()) == 0
        off = f0 % ring
        mring_d = pipe.mask_ring.cpu().numpy().view(np.uint32)
        gop_d = pipe.gop_state.cpu().numpy().view(np.uint32)
        slot_d = pipe.slots[pipe.cur].cpu().numpy()          # after the swap: window k
        disp_d, pold_d, nt_d = pipe.disposition.cpu().numpy(), pipe.p_old.cpu().numpy(), pipe.n_tokens.cpu().numpy()
        for si in sample:
            h = st_h[si]
            h["tring"][0, off:off + n] = types[si]
            so = ref.score_patches(g, mb[si:si + 1], np.ascontiguousarray(h["tring"][:, off:]), h["gop"],
                                   frame_stride=ring - off, want_score=False)
            h["mring"][0, off:off + n] = so["keep_mask"][0, :n]
            assert (mring_d[si] == h["mring"][0]).all()
            assert (gop_d[si] == h["gop"][0]).all()
            # kv refresh of this stream (paged), pool rows compared in full
            kv = pipe.kv
            win = dict(window=w, stride=s, step=k, ring_frames=ring)
            pool = pool_before[si]
            pre = pool.copy()
            ko = ref.kv_refresh_paged(g, kv, win, h["mring"], h["tring"], [pool], h["slot"], pipe.token_cap,
                                      [refr[si]] if k >= 1 else None, pipe.token_cap)
            ntok = int(ko["n_tokens"][0, 0]) + cfg["n_prompt"]
            assert (nt_d[si] == ko["n_tokens"][0]).all()
            assert (disp_d[si, :ntok] == ko["disposition"][0, :ntok]).all()
            assert (pold_d[si, :ntok] == ko["p_old"][0, :ntok]).all()
            assert (slot_d[si, :ntok] == ko["slot_new"][0, :ntok]).all()
            # the whole pool: refreshed rows and untouched rows bit-identical, rotated keys within the bf16 bound
            kvcheck.check_pool_step(_host(pipe.caches[0][si]), pre, pool, ko["disposition"][0], ko["slot_new"][0],
                                    ntok, kv, refr=refr[si] if k >= 1 else None, stats=stats,
                                    tag=f"{cfg_name} step {k} stream {si}")
            h["slot"] = ko["slot_new"]
        # compaction of the last chunk (the packed buffer holds the last s frames of the step)
        last0 = 0 if fused else n - min(n, s)   # fused: one compaction of all the step's frames
        nl = n - last0
        offs = pipe.frame_offsets[:S * nl + 1].cpu().numpy()
        src_d = pipe.src_index.cpu().numpy()
        pos_d = pipe.pos_ids.cpu().numpy()
        packed_d = pipe.packed.view(torch.int16).cpu().numpy().view(np.uint16)
        for si in sample:
            mask = st_h[si]["mring"][:, off + last0:off + n]
            fr = [to_grouped(planar[si][(last0 + j) % w], g) for j in range(nl)]
            co = ref.compact(g, mask.copy(), np.arange(f0 + last0, f0 + n, dtype=np.int32), fr, nl * 1024, 1, nl,
                             frame_layout=1)
            a, b = int(offs[si * nl]), int(offs[si * nl + nl])
            cnt = int(co["frame_offsets"][-1])
            assert b - a == cnt
            assert (packed_d[a:b] == co["packed"][:cnt]).all()
            assert (pos_d[a:b] == co["pos_ids"][:cnt]).all()
            assert (src_d[a:b] - si * nl * 1024 == co["src_index"][:cnt]).all()
    kvcheck.assert_rotation_bits(stats)


@pytest.mark.parametrize("overlap", [False, True])
def test_fullsize_nv12_sampled_streams(ref, overlap):
    """C4 from NV12 decoder frames (the bench's --frames nv12): 256 1080p streams, the staged fused preprocessing in
    the bench's launch configuration (Pipeline, chunks of s frames, paged KV refresh, pipelined steps when overlap);
    every packed row of the sampled streams' frames bit-exact vs the oracle (codecsight_ref_compact_nv12 on their
    own masks and planes), the counters' source-sector bytes included in the per-call totals."""
    import gc
    gc.collect()
    torch.cuda.empty_cache()
    from paper_2604_06036_b200 import _abi as abi
    from paper_2604_06036_b200.pipeline import Pipeline
    cfg = synth.CONFIGS["C4"]
    sw, sh = cfg["src"]
    g = make_grid(sw, sh)
    w, s, gop = cfg["window"], cfg["stride"], cfg["gop"]
    S, sample, steps = 256, [0, 1, 254, 255], 3
    pre = dict(src_w=sw, src_h=sh, y_pitch=sw, uv_pitch=sw)
    pipe = Pipeline(g, S, w, s, gop, cfg["kv"], n_prompt=cfg["n_prompt"], device=DEV,
                    frame_layout=abi.CS_LAYOUT_GROUPED, kv_mode="paged", compact_chunk=s, preprocess=pre,
                    overlap=overlap)
    ring = pipe.ring
    gen = torch.Generator(device=DEV)
    gen.manual_seed(5)
    pipe.init_cache_fill(gen)
    gens = [synth.StreamGen(sw, sh, synth.scene_of(cfg, i), synth.stream_seed(cfg, i)) for i in range(S)]
    rng = np.random.default_rng(8)
    planes = {si: [(rng.integers(16, 236, size=(sh, sw), dtype=np.uint8),
                    rng.integers(16, 241, size=(sh // 2, sw), dtype=np.uint8)) for _ in range(w)] for si in sample}
    shared_y = torch.from_numpy(rng.integers(16, 236, size=(sh, sw), dtype=np.uint8)).to(DEV)
    shared_uv = torch.from_numpy(rng.integers(16, 241, size=(sh // 2, sw), dtype=np.uint8)).to(DEV)
    dev_planes = {si: [(torch.from_numpy(y).to(DEV), torch.from_numpy(uv).to(DEV)) for y, uv in planes[si]]
                  for si in sample}
    nw = 32
    st_h = {si: dict(gop=np.zeros((1, nw + 1), np.uint32), mring=np.zeros((1, ring, nw), np.uint32),
                     tring=np.zeros((1, ring), np.uint8)) for si in sample}
    pre_h = ref.make_pre(sw, sh, sw, sw)
    for k in range(steps):
        f0, n = pipe.new_frames(k)
        mb = np.stack([np.stack([gn.next_frame() for _ in range(n)]) for gn in gens])
        types = np.stack([synth.frame_types(n, gop, f0)] * S)
        ys, uvs = [], []
        for si in range(S):
            for j in range(n):
                y, uv = dev_planes[si][j % w] if si in sample else (shared_y, shared_uv)
                ys.append(y)
                uvs.append(uv)
        fptr = (abi.ptr_array(ys, DEV), abi.ptr_array(uvs, DEV))
        fidx = np.tile(np.arange(f0, f0 + n, dtype=np.int32), S)
        pipe.step(k, torch.from_numpy(mb.view(np.uint8)).to(DEV), fptr, torch.from_numpy(fidx).to(DEV),
                  torch.from_numpy(types).to(DEV))
        pipe.join()
        torch.cuda.synchronize()
        assert int(pipe.status.item()) == 0
        off = f0 % ring
        mring_d = pipe.mask_ring.cpu().numpy().view(np.uint32)
        for si in sample:
            h = st_h[si]
            h["tring"][0, off:off + n] = types[si]
            so = ref.score_patches(g, mb[si:si + 1], np.ascontiguousarray(h["tring"][:, off:]), h["gop"],
                                   frame_stride=ring - off, want_score=False)
            h["mring"][0, off:off + n] = so["keep_mask"][0, :n]
            assert (mring_d[si] == h["mring"][0]).all()
        # the packed buffer holds the step's last chunk of s frames
        last0 = n - min(n, s)
        nl = n - last0
        offs = pipe.frame_offsets[:S * nl + 1].cpu().numpy()
        src_d, pos_d = pipe.src_index.cpu().numpy(), pipe.pos_ids.cpu().numpy()
        packed_d = pipe.packed.view(torch.int16).cpu().numpy().view(np.uint16)
        for si in sample:
            mask = np.ascontiguousarray(st_h[si]["mring"][:, off + last0:off + n])
            ysi = [planes[si][(last0 + j) % w][0] for j in range(nl)]
            uvsi = [planes[si][(last0 + j) % w][1] for j in range(nl)]
            co = ref.compact_nv12(g, pre_h, mask, np.arange(f0 + last0, f0 + n, dtype=np.int32), ysi, uvsi,
                                  nl * 1024, 1, nl)
            a, b = int(offs[si * nl]), int(offs[si * nl + nl])
            cnt = int(co["frame_offsets"][-1])
            assert b - a == cnt
            assert (packed_d[a:b] == co["packed"][:cnt]).all(), int((packed_d[a:b] != co["packed"][:cnt]).sum())
            assert (pos_d[a:b] == co["pos_ids"][:cnt]).all()
            assert (src_d[a:b] - si * nl * 1024 == co["src_index"][:cnt]).all()
