#!/usr/bin/env python3
"""Experiment: per-CTA phase timestamps of the fused score+compact kernel (score.cu built with -DCS_PHASE_TIMING
into scripts/libcodecsight_phase.so).  Prints, per workload shape, the distribution over CTAs of the time from the
grid's first CTA start to: CTA start, stream ticket, prologue done, first / last MB chunk landed, pass 2 start,
scoring done, keep masks written, offset resolved (look-back), compaction done, CTA end; and per-CTA phase lengths.

    python scripts/phase_timing.py build      # here (nvcc)
    python scripts/phase_timing.py run        # on the GPU box
"""
import ctypes as C
import glob
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "scripts", "libcodecsight_phase.so")


def build():
    import __graft_entry__ as ge
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2604_06036_b200", "csrc", "*.cu")))
    subprocess.check_call([ge._nvcc()] + ge.NVCC_FLAGS + ["-DCS_PHASE_TIMING", "-I", os.path.join(ROOT, "include"),
                                                           "-o", LIB] + srcs)


def run():
    import torch
    import synth
    from paper_2604_06036_b200 import _abi as abi
    abi.LIB_PATH = LIB
    L = abi.lib()
    L.codecsight_debug_phase.restype = C.c_int
    L.codecsight_debug_phase.argtypes = [C.c_void_p, C.c_int]
    L.codecsight_debug_smid.restype = C.c_int
    L.codecsight_debug_smid.argtypes = [C.c_void_p, C.c_int]
    dev = torch.device("cuda:0")
    for name, S in (("C2", 32), ("C3", 64), ("C4", 256)):
        cfg = synth.CONFIGS[name]
        sw, sh = cfg["src"]
        g = synth.make_grid(sw, sh)
        n = cfg["stride"]
        gens = [synth.StreamGen(sw, sh, synth.scene_of(cfg, s), synth.stream_seed(cfg, s)) for s in range(S)]
        for _ in range(4):
            for gn in gens:
                gn.next_frame()
        mb = np.stack([np.stack([gn.next_frame() for _ in range(n)]) for gn in gens])
        mb_d = torch.from_numpy(np.ascontiguousarray(mb).view(np.uint8).copy()).to(dev)
        types = torch.from_numpy(np.stack([synth.frame_types(n, cfg["gop"], 4)] * S)).to(dev)
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
        cluster = min(n, 8)
        nct = S * cluster
        res = []
        for rep in range(6):
            gs = torch.zeros(S, nw + 1, dtype=torch.int32, device=dev)
            gs[:, nw] = 1
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            abi.codecsight_score_compact(g, S, n, mb_d, types, km, n, gs, None, kc, fidx, fptr, cap, packed, pos, src,
                                         offs, ws, cnt, st, frame_layout=abi.CS_LAYOUT_GROUPED)
            e1.record()
            torch.cuda.synchronize()
            ev_ms = e0.elapsed_time(e1)
            h = np.zeros((nct, 12), np.uint64)
            assert L.codecsight_debug_phase(h.ctypes.data, nct) == 0
            smid = np.zeros(nct, np.uint32)
            assert L.codecsight_debug_smid(smid.ctypes.data, nct) == 0
            if rep >= 2:
                res.append(h.astype(np.int64) - int(h[:, 0].min()))
        gs = torch.zeros(S, nw + 1, dtype=torch.int32, device=dev)
        gs[:, nw] = 1
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            abi.codecsight_score_compact(g, S, n, mb_d, types, km, n, gs, None, kc, fidx, fptr, cap, packed, pos, src,
                                         offs, ws, cnt, st, frame_layout=abi.CS_LAYOUT_GROUPED)
        e1.record()
        torch.cuda.synchronize()
        print(f"   20 back-to-back calls: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per call")
        kept = float(kc.sum().item()) / (S * n * 1024)
        print(f"== {name}: {S} streams x {n} frames, {nct} CTAs, kept {kept:.2f}")
        labels = ["start", "ticket", "prologue", "1st chunk", "scored", "masks", "offset", "compacted", "end"]
        print(f"   CUDA-event time of the call: {ev_ms * 1e3:.1f} us (launch + CTA span + drain)")
        # compaction end by the number of this grid's CTAs sharing the CTA's SM (balanced shares are equal per warp)
        r = res[-1]
        per_sm = np.bincount(smid, minlength=int(smid.max()) + 1)
        share = per_sm[smid]
        for c in sorted(set(share.tolist())):
            v = r[share == c, 7] / 1e3
            print(f"   CTAs on SMs holding {c} of the grid's CTAs: {v.size:4d}, compacted med {np.median(v):7.1f} us"
                  f"  max {v.max():7.1f}")
        for r in res[-1:]:
            for k, lab in enumerate(labels):
                v = r[:, k] / 1e3
                print(f"   {lab:10s} min {v.min():7.1f} us  med {np.median(v):7.1f}  max {v.max():7.1f}")
            labels += ["pass2", "last chunk"]
            for a, b in ((0, 1), (1, 2), (2, 3), (3, 10), (10, 9), (9, 4), (4, 5), (5, 6), (6, 7), (7, 8)):
                d = (r[:, b] - r[:, a]) / 1e3
                print(f"   {labels[a]:>10s} -> {labels[b]:10s} per CTA: med {np.median(d):6.1f} us  max {d.max():6.1f}")


def run_score():
    """The non-fused scoring kernel (codecsight_score_patches) at the NEXT-4 cdf shape (64 1080p streams x 16
    frames: clusters of 8 CTAs x 2 frames) and the NV12-C4 shape (256 streams x 4 frames)."""
    import torch
    import synth
    from paper_2604_06036_b200 import _abi as abi
    abi.LIB_PATH = LIB
    L = abi.lib()
    L.codecsight_debug_phase.restype = C.c_int
    L.codecsight_debug_phase.argtypes = [C.c_void_p, C.c_int]
    L.codecsight_debug_smid.restype = C.c_int
    L.codecsight_debug_smid.argtypes = [C.c_void_p, C.c_int]
    dev = torch.device("cuda:0")
    for name, cname, S, n in (("cdf", "C4", 64, 16), ("C4", "C4", 256, 4)):
        cfg = synth.CONFIGS[cname]
        sw, sh = cfg["src"]
        g = synth.make_grid(sw, sh)
        gens = [synth.StreamGen(sw, sh, synth.scene_of(cfg, s), synth.stream_seed(cfg, s)) for s in range(S)]
        mb = np.stack([np.stack([gn.next_frame() for _ in range(n)]) for gn in gens])
        mb_d = torch.from_numpy(np.ascontiguousarray(mb).view(np.uint8).copy()).to(dev)
        types = torch.from_numpy(np.stack([synth.frame_types(n, cfg["gop"], 1)] * S)).to(dev)
        nw = abi.grid_words(g)
        cnt = torch.zeros(abi.NCOUNTERS, dtype=torch.int64, device=dev)
        st = torch.zeros(1, dtype=torch.int32, device=dev)
        km = torch.zeros(S, n, nw, dtype=torch.int32, device=dev)
        kc = torch.zeros(S, n, dtype=torch.int32, device=dev)
        sc = torch.zeros(S, n, g["grid_w"] * g["grid_h"], dtype=torch.float32, device=dev)
        cluster = min(n, 8)
        fpc = (n + cluster - 1) // cluster
        nct = S * ((n + fpc - 1) // fpc)
        res = []
        for rep in range(6):
            gs = torch.zeros(S, nw + 1, dtype=torch.int32, device=dev)
            gs[:, nw] = 1
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            abi.codecsight_score_patches(g, S, n, mb_d, types, km, n, gs, sc, kc, cnt, st)
            e1.record()
            torch.cuda.synchronize()
            ev_ms = e0.elapsed_time(e1)
            h = np.zeros((nct, 12), np.uint64)
            assert L.codecsight_debug_phase(h.ctypes.data, nct) == 0
            smid = np.zeros(nct, np.uint32)
            assert L.codecsight_debug_smid(smid.ctypes.data, nct) == 0
            if rep >= 2:
                res.append(h.astype(np.int64) - int(h[:, 0].min()))
        print(f"== score_patches {name}: {S} streams x {n} frames, {nct} CTAs ({fpc} frames each)")
        print(f"   CUDA-event time of the call: {ev_ms * 1e3:.1f} us")
        r = res[-1]
        per_sm = np.bincount(smid, minlength=int(smid.max()) + 1)
        share = per_sm[smid]
        for c in sorted(set(share.tolist())):
            v = r[share == c, 8] / 1e3
            print(f"   CTAs on SMs holding {c}: {v.size:4d}, end med {np.median(v):7.1f} us  max {v.max():7.1f}")
        labels = {0: "start", 2: "prologue", 3: "1st chunk", 10: "last chunk", 9: "pass2", 4: "scored", 5: "masks",
                  8: "end"}
        for k, lab in labels.items():
            v = r[:, k] / 1e3
            print(f"   {lab:10s} min {v.min():7.1f} us  med {np.median(v):7.1f}  max {v.max():7.1f}")
        ks = list(labels)
        for a, b in zip(ks[:-1], ks[1:]):
            d = (r[:, b] - r[:, a]) / 1e3
            print(f"   {labels[a]:>10s} -> {labels[b]:10s} per CTA: med {np.median(d):6.1f} us  max {d.max():6.1f}")


if __name__ == "__main__":
    {"build": build, "run": run, "score": run_score}[sys.argv[1]]()
