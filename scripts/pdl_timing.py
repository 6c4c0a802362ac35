#!/usr/bin/env python3
"""Experiment: does the programmatic dependent launch of the fused score+compact kernel (CS_LAUNCH_PDL) overlap?
Back-to-back C2-shaped launches (32 1080p streams x 4 frames, two alternating workspaces) on the phase-timing build
(scripts/libcodecsight_phase.so, score.cu with -DCS_PHASE_TIMING); prints, for the last two launches A and B, the
per-CTA %globaltimer stamps relative to A's first CTA start: CTA start, scoring done (before the PDL wait), past
the wait, CTA end.

    python scripts/phase_timing.py build && python scripts/pdl_timing.py     # (GPU box)
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "scripts", "libcodecsight_phase.so")


def main():
    import torch
    import synth
    from paper_2604_06036_b200 import _abi as abi
    abi.LIB_PATH = LIB
    L = abi.lib()
    L.codecsight_debug_phase_slot.restype = C.c_int
    L.codecsight_debug_phase_slot.argtypes = [C.c_void_p, C.c_int, C.c_int]
    dev = torch.device("cuda:0")
    S, n = 32, 4
    cfg = synth.CONFIGS["C2"]
    g = synth.make_grid(1920, 1080)
    gens = [synth.StreamGen(1920, 1080, synth.scene_of(cfg, s), synth.stream_seed(cfg, s)) for s in range(S)]
    mbs = [torch.from_numpy(np.stack([np.stack([gn.next_frame() for _ in range(n)]) for gn in gens]).view(np.uint8)
                            .copy()).to(dev) for _ in range(2)]
    types = torch.from_numpy(np.stack([synth.frame_types(n, 16, 5)] * S)).to(dev)
    nw = abi.grid_words(g)
    frames = [torch.randn(3 * 448 * 448, device=dev).to(torch.bfloat16) for _ in range(S * n)]
    fptr = abi.ptr_array(frames, dev)
    fidx = torch.arange(S * n, dtype=torch.int32, device=dev)
    cap = S * n * 1024
    packed = torch.empty(cap, 588, dtype=torch.bfloat16, device=dev)
    pos = torch.empty(cap, 3, dtype=torch.int32, device=dev)
    src = torch.empty(cap, dtype=torch.int32, device=dev)
    offs = torch.empty(S * n + 1, dtype=torch.int32, device=dev)
    ws = [torch.zeros(abi.score_compact_workspace_size(S), dtype=torch.uint8, device=dev) for _ in range(4)]
    cnt = torch.zeros(abi.NCOUNTERS, dtype=torch.int64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    km = torch.zeros(S, n, nw, dtype=torch.int32, device=dev)
    kc = torch.zeros(S, n, dtype=torch.int32, device=dev)
    gs = torch.zeros(S, nw + 1, dtype=torch.int32, device=dev)
    gs[:, nw] = 1
    nct = S * n
    D = 3  # chain depth (output buffer sets); D + 1 workspaces
    outs = [(torch.empty_like(packed), torch.empty_like(pos), torch.empty_like(src), torch.empty_like(offs),
             torch.empty_like(kc)) for _ in range(D)]
    for flags in (0, abi.CS_LAUNCH_PDL):
        chain_t = (torch.zeros(S, dtype=torch.int32, device=dev), torch.zeros(D, dtype=torch.int32, device=dev))
        torch.cuda.synchronize()
        N = 8
        for i in range(N):
            pk, ps, sr, of, kk = outs[i % D]
            abi.codecsight_score_compact_ex(g, S, n, mbs[i & 1], types, n, km, n, gs, None, kk, fidx, fptr, cap,
                                            pk, ps, sr, of, ws[i % 4], cnt, st, flags=flags,
                                            chain=(chain_t[0], chain_t[1], i) if flags else None,
                                            frame_layout=abi.CS_LAYOUT_GROUPED)
        torch.cuda.synchronize()
        ph = []
        for slot in ((N - 2) & 1, (N - 1) & 1):
            h = np.zeros((nct, 12), np.uint64)
            assert L.codecsight_debug_phase_slot(h.ctypes.data, nct, slot) == 0
            ph.append(h.astype(np.int64))
        t0 = ph[0][:, 0].min()
        print(f"flags={flags}")
        for name, h in (("A", ph[0]), ("B", ph[1])):
            rel = (h - t0) / 1000.0
            print(f"  {name}: start {rel[:, 0].min():7.1f}..{rel[:, 0].max():7.1f} us  scored(pre-wait) "
                  f"{rel[:, 11].min():7.1f}..{rel[:, 11].max():7.1f}  post-wait {rel[:, 4].min():7.1f}.."
                  f"{rel[:, 4].max():7.1f}  offsets {rel[:, 6].min():7.1f}..{rel[:, 6].max():7.1f}  compacted "
                  f"{rel[:, 7].min():7.1f}..{rel[:, 7].max():7.1f}  end {rel[:, 8].min():7.1f}..{rel[:, 8].max():7.1f}")


if __name__ == "__main__":
    main()
