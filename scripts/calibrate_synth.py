#!/usr/bin/env python3
"""Kept fraction of each synthetic scene kind, measured with the oracle (test/bench infrastructure).

PAPER.md:563 (§6 motion levels): codec-guided pruning removes 50 %, 27 % and 13 % of the visual tokens of low-,
medium- and high-motion videos (UCF-Crime).  The generator's scene kinds are calibrated against those numbers: for
each kind, `streams` seeded streams run `frames` consumed frames through the oracle's score_patches (Eq. 1-4, GOP
accumulation, group expansion; 1080p, GOP 16, tau 0.25, alpha 0) and the kept fraction = kept patches / patches
over every frame after the first GOP (I-frames included, as a window of w = 16 frames contains one).

    python scripts/calibrate_synth.py [--frames 64] [--streams 8] [--scenes low,medium,high,traffic,static]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

# calibration targets: kept fraction = 1 - pruned fraction; traffic = "medium-high"
TARGETS = {"low": 0.50, "medium": 0.73, "high": 0.87, "traffic": 0.80, "static": 1.0 / 16}


def kept_fraction(scene: str, streams: int = 8, frames: int = 64, gop: int = 16, src=None, seed0: int = 0,
                  per_stream: bool = False):
    import oracle.ref as ref
    sw, sh = src if src is not None else ((3840, 2160) if scene == "traffic" else (1920, 1080))
    g = synth.make_grid(sw, sh)
    nw = 32
    fr = []
    for si in range(streams):
        mb = synth.stream_metadata(sw, sh, scene, 100003 * (seed0 + 1) + si, frames)
        types = synth.frame_types(frames, gop)
        out = ref.score_patches(g, mb[None], types[None], np.zeros((1, nw + 1), np.uint32), want_score=False)
        kc = out["kept_count"][0, gop:].astype(np.float64)        # steady state: after the first GOP
        fr.append(kc.sum() / (kc.size * 1024))
    return (float(np.mean(fr)), fr) if per_stream else float(np.mean(fr))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--streams", type=int, default=8)
    ap.add_argument("--scenes", default="static,low,medium,high,traffic")
    a = ap.parse_args()
    for sc in a.scenes.split(","):
        m, fr = kept_fraction(sc, a.streams, a.frames, per_stream=True)
        print(f"{sc:8s} kept {m:.3f} (target {TARGETS.get(sc, float('nan')):.3f})  per stream "
              f"{' '.join(f'{x:.2f}' for x in fr)}")


if __name__ == "__main__":
    main()
