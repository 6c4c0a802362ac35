#!/usr/bin/env python3
"""Experiment: what a small torch op enqueued right before the fused score+compact call costs (the bench's steps copy
the step's frame types into the ring just before it).  C3 and C2 shapes, one B200:
  (a) 20 fused calls back to back, (b) each preceded by a 1-element fill, (c) by a 1 KB device copy, (d) by the
  step's real frame-type ring copy; per-call average from CUDA events around the 20."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2604_06036_b200 import _abi as abi  # noqa: E402

dev = torch.device("cuda:0")
for name, S in (("C2", 32), ("C3", 64)):
    cfg = synth.CONFIGS[name]
    sw, sh = cfg["src"]
    g = synth.make_grid(sw, sh)
    n = cfg["stride"]
    gens = [synth.StreamGen(sw, sh, synth.scene_of(cfg, s), synth.stream_seed(cfg, s)) for s in range(S)]
    mb = np.stack([np.stack([gn.next_frame() for _ in range(n)]) for gn in gens])
    mb_d = torch.from_numpy(np.ascontiguousarray(mb).view(np.uint8).copy()).to(dev)
    types_src = torch.from_numpy(np.stack([synth.frame_types(n, cfg["gop"], 4)] * S)).to(dev)
    types = torch.empty_like(types_src)
    types.copy_(types_src)
    nw = abi.grid_words(g)
    frames = [torch.randn(3 * 448 * 448, device=dev).to(torch.bfloat16) for _ in range(S * n)]
    fptr = abi.ptr_array(frames, dev)
    fidx = torch.arange(S * n, dtype=torch.int32, device=dev)
    cap = S * n * 1024
    packed = torch.empty(cap, 588, dtype=torch.bfloat16, device=dev)
    pos = torch.empty(cap, 3, dtype=torch.int32, device=dev)
    src = torch.empty(cap, dtype=torch.int32, device=dev)
    offs = torch.empty(S * n + 1, dtype=torch.int32, device=dev)
    ws = torch.zeros(abi.score_compact_workspace_size(S), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(abi.NCOUNTERS, dtype=torch.int64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    km = torch.zeros(S, n, nw, dtype=torch.int32, device=dev)
    kc = torch.zeros(S, n, dtype=torch.int32, device=dev)
    gs = torch.zeros(S, nw + 1, dtype=torch.int32, device=dev)
    gs[:, nw] = 1
    one = torch.zeros(1, device=dev)
    a1k, b1k = torch.zeros(1024, dtype=torch.uint8, device=dev), torch.ones(1024, dtype=torch.uint8, device=dev)

    def call():
        abi.codecsight_score_compact(g, S, n, mb_d, types, km, n, gs, None, kc, fidx, fptr, cap, packed, pos, src,
                                     offs, ws, cnt, st, frame_layout=abi.CS_LAYOUT_GROUPED)

    pre = {"none": None, "fill": lambda: one.fill_(1.0), "copy1k": lambda: a1k.copy_(b1k),
           "types": lambda: types.copy_(types_src)}
    for rep in range(3):
        for k, fn in pre.items():
            call()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                if fn:
                    fn()
                call()
            e1.record()
            torch.cuda.synchronize()
            if rep == 2:
                print(f"{name}: preceded by {k:7s} {e0.elapsed_time(e1) / 20 * 1e3:7.1f} us per call")
