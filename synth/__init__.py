"""Seeded synthetic inputs shared by the tests, the bench and the smoke check.

This module holds NO arithmetic of the method (no scoring, thresholding, accumulation, compaction or
indexing).  It only draws inputs: H.264-style per-macroblock metadata (quarter-pel motion vectors, MB type,
SAD residual energy), I/P frame types, model-input frames and KV-cache contents, with the shapes and value
distributions of the paper's surveillance / traffic workloads (recipe in DESIGN.md "Input recipe").

Configs C1..C5 are BASELINE.json ``configs[0..4]`` with the concrete readings of SURVEY.md §8(d) / Q28-Q31.
"""
from __future__ import annotations

import math

import numpy as np

MB_DTYPE = np.dtype([("mvx", "<i2"), ("mvy", "<i2"), ("sad", "<u2"), ("type", "u1"), ("rsv", "u1")])
FRAME_I, FRAME_P = 0, 1
MB_INTER, MB_SKIP, MB_INTRA = 0, 1, 2


def make_grid(src_w: int, src_h: int, tau: float = 0.25, alpha: float = 0.0, mb_size: int = 16, patch: int = 14,
              grid_w: int = 32, grid_h: int = 32, group: int = 2) -> dict:
    """Geometry dict accepted by both the oracle binding and the CUDA binding."""
    return dict(src_w=src_w, src_h=src_h, mb_size=mb_size, mb_cols=-(-src_w // mb_size),
                mb_rows=-(-src_h // mb_size), patch=patch, grid_w=grid_w, grid_h=grid_h, group=group,
                tau=float(tau), alpha=float(alpha))


QWEN_KV = dict(layers=28, kv_heads=4, head_dim=128, dtype=0, rope_base=1e6)  # Qwen2-VL-7B shape, bf16
TOY_KV = dict(layers=2, kv_heads=2, head_dim=16, dtype=1, rope_base=1e4)     # SPEC toy scale, fp32
# Qwen2-VL multimodal RoPE: 64 frequency pairs split t/h/w = 16/24/24, one temporal position per frame (NEXT-3)
QWEN_MROPE_KV = dict(QWEN_KV, rope_mode=1, mrope_section=(16, 24, 24), t_per_frame=1)

# BASELINE.json configs with SURVEY §8(d) readings.  "scenes" is either a list cycled over stream ids or
# the string "mixed" (even ids static, odd ids high-motion: C4).
CONFIGS = {
    "C1": dict(name="C1-oracle", src=(448, 448), streams=1, window=8, stride=2, gop=4, frames=64,
               scenes=["static", "translating_object", "multi_object", "noise", "scene_cut"], kv=TOY_KV,
               n_prompt=32, config_id=1),
    "C2": dict(name="C2-prune-compact-1080p", src=(1920, 1080), streams=32, window=16, stride=4, gop=16,
               frames=512, scenes=["low", "medium"], kv=None, n_prompt=0, config_id=2),
    "C3": dict(name="C3-kv-refresh-qwen2vl7b", src=(1920, 1080), streams=64, window=32, stride=4, gop=16,
               frames=None, scenes=["low", "medium"], kv=QWEN_KV, n_prompt=32, config_id=3),
    "C4": dict(name="C4-full-1080p-mixed", src=(1920, 1080), streams=256, window=16, stride=4, gop=16,
               frames=None, scenes="mixed", kv=QWEN_KV, n_prompt=32, config_id=4),
    "C5": dict(name="C5-full-4k-traffic", src=(3840, 2160), streams=1024, window=64, stride=8, gop=16,
               frames=None, scenes=["traffic"], kv=QWEN_KV, n_prompt=32, config_id=5),
    # NEXT-4: the similar-patch analysis of fig:mv_residual_analysis_cdf as a
    # second workload -- H.264-shaped AVMotionVector exports -> MB grid -> scores -> per-frame similar-patch
    # histograms over tau in {0.25, 0.5, 1, 2, 5} px; a step = one GOP (16 frames) of every stream
    "CDF": dict(name="NEXT4-cdf-1080p", src=(1920, 1080), streams=64, window=16, stride=16, gop=16, frames=None,
                scenes=["static", "low", "medium", "high"], kv=None, n_prompt=0, config_id=6,
                taus=(0.25, 0.5, 1.0, 2.0, 5.0), n_bins=20),
}


def scene_of(cfg: dict, stream_id: int) -> str:
    if cfg["scenes"] == "mixed":
        return "static" if stream_id % 2 == 0 else "high"
    sc = cfg["scenes"]
    return sc[stream_id % len(sc)]


def stream_seed(cfg: dict, stream_id: int, salt: int = 0) -> int:
    return 1000 * cfg["config_id"] + stream_id + 7919 * salt


def frame_types(n_frames: int, gop: int, first: int = 0) -> np.ndarray:
    """I-frame at every f % gop == 0, P otherwise (no B-frames, S:8)."""
    f = np.arange(first, first + n_frames)
    return np.where(f % gop == 0, FRAME_I, FRAME_P).astype(np.uint8)


# Scene kinds (SURVEY §8(d) generator table; SPEC S:516 kinds for parity).  Calibrated with the oracle
# (scripts/calibrate_synth.py, tests/test_synth_calibration.py) to the paper's per-motion-level pruning, P:563:
# 50 / 27 / 13 % of visual tokens pruned for low / medium / high motion (kept 0.50 / 0.73 / 0.87 of the patches of
# a 16-frame window, its I-frame included); traffic is "medium-high" (kept ~0.80).
#   k / v / size : moving objects (count, speed in px/frame, width as a fraction of the frame width)
#   tex / blobs  : fraction of the frame covered by textured background regions (foliage, water, screens) in
#                  `blobs` rectangles fixed per stream; each of their MBs flickers with a +-1 qpel vector (= tau, so
#                  dynamic) with probability p_tex per frame.  Sensor noise on real encoders is spatially persistent
#                  like this, not i.i.d. per frame (an i.i.d. 1-qpel MB anywhere would, under the GOP union of
#                  P:318, end up touching almost every patch within a GOP)
#   p_noise      : i.i.d. +-1 qpel MBs anywhere (only the SPEC "noise" kind and, sparsely, scene_cut)
SCENES = {
    "static": dict(k=(0, 0), v=(0.0, 0.0), p_noise=0.0, size=(0.05, 0.1)),
    "low": dict(k=(2, 4), v=(0.25, 1.0), p_noise=0.0, size=(0.15, 0.30), tex=0.15, blobs=(1, 3), p_tex=0.3),
    "medium": dict(k=(6, 8), v=(0.5, 3.5), p_noise=0.0, size=(0.16, 0.30), tex=0.25, blobs=(2, 3), p_tex=0.3),
    "high": dict(k=(11, 14), v=(1.5, 6.0), p_noise=0.0, size=(0.17, 0.32), tex=0.35, blobs=(2, 4), p_tex=0.3),
    "traffic": dict(k=(0, 0), v=(2.0, 8.0), p_noise=0.0, size=(0.042, 0.082), lanes=(4, 5), cars=(8, 20),
                    tex=0.05, blobs=(1, 2), p_tex=0.3),
    "translating_object": dict(k=(1, 1), v=(1.0, 2.0), p_noise=0.0, size=(0.15, 0.3)),
    "multi_object": dict(k=(3, 5), v=(0.25, 3.0), p_noise=0.0, size=(0.08, 0.2)),
    "noise": dict(k=(0, 0), v=(0.0, 0.0), p_noise=0.3, size=(0.05, 0.1)),
    "scene_cut": dict(k=(1, 2), v=(0.5, 2.0), p_noise=0.002, size=(0.1, 0.25), p_cut=0.15),
}


class StreamGen:
    """Per-stream seeded generator of P-frame macroblock metadata (one record set per consumed frame, Q25).

    Objects are axis-aligned boxes moving with a constant velocity (bouncing at the borders).  Macroblocks whose
    centre lies in a moving object get MV = round(4 v) qpel with +-1 qpel jitter (p = 0.2), type INTER,
    SAD ~ 256 U(8, 40); with p = 0.02 an object MB is INTRA (entering content).  Background MBs are SKIP with a
    zero MV and SAD 0, except flickering MBs of the stream's textured regions (p_tex per frame) and a fraction
    p_noise of i.i.d. MBs, both INTER with a +-1 qpel MV and SAD ~ 256 U(0, 3) (sensor noise).  "scene_cut"
    P-frames (probability p_cut) turn >= 80% of MBs INTRA."""

    def __init__(self, src_w: int, src_h: int, scene: str, seed: int, mb_size: int = 16):
        self.src_w, self.src_h, self.mb = src_w, src_h, mb_size
        self.cols, self.rows = -(-src_w // mb_size), -(-src_h // mb_size)
        self.scene = SCENES[scene]
        self.kind = scene
        self.rng = np.random.default_rng(seed)
        r = self.rng
        sc = self.scene
        objs = []
        if scene == "traffic":
            n_lanes = int(r.integers(sc["lanes"][0], sc["lanes"][1] + 1))
            for ln in range(n_lanes):
                y = (ln + 0.5) * src_h / n_lanes
                direction = 1.0 if ln % 2 == 0 else -1.0
                for _ in range(int(r.integers(sc["cars"][0], sc["cars"][1] + 1))):
                    w = r.uniform(*sc["size"]) * src_w * 1.6
                    h = w * 0.6
                    objs.append([r.uniform(0, src_w), y + r.uniform(-0.1, 0.1) * src_h / n_lanes, w, h,
                                 direction * r.uniform(*sc["v"]), 0.0])
        else:
            n = int(r.integers(sc["k"][0], sc["k"][1] + 1))
            for _ in range(n):
                w = r.uniform(*sc["size"]) * src_w
                h = w * r.uniform(0.6, 1.6)
                speed = r.uniform(*sc["v"])
                ang = r.uniform(0, 2 * math.pi)
                objs.append([r.uniform(0, src_w), r.uniform(0, src_h), w, h, speed * math.cos(ang),
                             speed * math.sin(ang)])
        self.objs = np.array(objs, dtype=np.float64).reshape(-1, 6)
        # textured background regions: `blobs` rectangles whose areas sum to ~tex of the frame, fixed per stream
        self.tex = np.zeros((self.rows, self.cols), bool)
        if sc.get("tex", 0.0) > 0:
            nb = int(r.integers(sc["blobs"][0], sc["blobs"][1] + 1))
            for _ in range(nb):
                area = sc["tex"] / nb * self.rows * self.cols
                aspect = r.uniform(0.5, 2.0)
                bh = max(1, int(round(math.sqrt(area / aspect))))
                bw = max(1, int(round(area / bh)))
                j0 = int(r.integers(0, max(1, self.rows - bh + 1)))
                i0 = int(r.integers(0, max(1, self.cols - bw + 1)))
                self.tex[j0:j0 + bh, i0:i0 + bw] = True
        self.cx = (np.arange(self.cols) * mb_size + mb_size / 2.0)[None, :]
        self.cy = (np.arange(self.rows) * mb_size + mb_size / 2.0)[:, None]

    def _advance(self):
        o = self.objs
        if len(o) == 0:
            return
        o[:, 0] += o[:, 4]
        o[:, 1] += o[:, 5]
        if self.kind == "traffic":
            o[:, 0] = np.mod(o[:, 0], self.src_w)
        else:
            for ax, vel, lim in ((0, 4, self.src_w), (1, 5, self.src_h)):
                lo = o[:, ax] < 0
                hi = o[:, ax] > lim
                o[lo | hi, vel] *= -1.0
                o[:, ax] = np.clip(o[:, ax], 0, lim)

    def next_frame(self) -> np.ndarray:
        """MB records [rows][cols] for the next consumed frame (also advances the scene)."""
        self._advance()
        r = self.rng
        sc = self.scene
        rec = np.zeros((self.rows, self.cols), MB_DTYPE)
        rec["type"] = MB_SKIP
        noise = None
        if sc["p_noise"] > 0:
            noise = r.random((self.rows, self.cols)) < sc["p_noise"]
        if sc.get("tex", 0.0) > 0:
            flick = self.tex & (r.random((self.rows, self.cols)) < sc["p_tex"])
            noise = flick if noise is None else (noise | flick)
        if noise is not None:
            if noise.any():
                k = int(noise.sum())
                mv = r.integers(-1, 2, size=(k, 2))
                zero = (mv[:, 0] == 0) & (mv[:, 1] == 0)
                mv[zero, 0] = 1
                rec["mvx"][noise] = mv[:, 0]
                rec["mvy"][noise] = mv[:, 1]
                rec["sad"][noise] = (256 * r.uniform(0, 3, size=k)).astype(np.uint16)
                rec["type"][noise] = MB_INTER
        for o in self.objs:
            x, y, w, h, vx, vy = o
            if vx == 0.0 and vy == 0.0:
                continue
            # MBs whose centre (16 i + 8, 16 j + 8) lies inside the box: a slice of the MB grid
            m = self.mb
            i0 = max(0, int(np.ceil((x - w / 2 - m / 2) / m)))
            i1 = min(self.cols - 1, int(np.floor((x + w / 2 - m / 2) / m)))
            j0 = max(0, int(np.ceil((y - h / 2 - m / 2) / m)))
            j1 = min(self.rows - 1, int(np.floor((y + h / 2 - m / 2) / m)))
            if i1 < i0 or j1 < j0:
                continue
            sl = rec[j0:j1 + 1, i0:i1 + 1]
            shp = sl.shape
            jit = (r.random(shp + (2,)) < 0.2) * r.choice(np.array([-1, 1]), size=shp + (2,))
            sl["mvx"] = np.clip(np.round(4 * vx) + jit[..., 0], -32768, 32767).astype(np.int16)
            sl["mvy"] = np.clip(np.round(4 * vy) + jit[..., 1], -32768, 32767).astype(np.int16)
            sl["sad"] = (256 * r.uniform(8, 40, size=shp)).astype(np.uint16)
            t = np.full(shp, MB_INTER, np.uint8)
            t[r.random(shp) < 0.02] = MB_INTRA
            sl["type"] = t
        if "p_cut" in sc and r.random() < sc["p_cut"]:
            cut = r.random((self.rows, self.cols)) < 0.85
            rec["type"][cut] = MB_INTRA
            rec["sad"][cut] = (256 * r.uniform(20, 60, size=int(cut.sum()))).astype(np.uint16)
        return rec


def random_mb(rows: int, cols: int, rng: np.random.Generator, p_intra: float = 0.05, mv_max: int = 12,
              p_bad_type: float = 0.0) -> np.ndarray:
    """Unstructured random MB records (edge cases: ties at 1 qpel, INTRA, extreme vectors)."""
    rec = np.zeros((rows, cols), MB_DTYPE)
    rec["mvx"] = rng.integers(-mv_max, mv_max + 1, size=(rows, cols))
    rec["mvy"] = rng.integers(-mv_max, mv_max + 1, size=(rows, cols))
    rec["sad"] = rng.integers(0, 65536, size=(rows, cols))
    t = rng.choice(np.array([MB_INTER, MB_SKIP], np.uint8), size=(rows, cols))
    t[rng.random((rows, cols)) < p_intra] = MB_INTRA
    if p_bad_type > 0:
        t[rng.random((rows, cols)) < p_bad_type] = 7
    rec["type"] = t
    return rec


def stream_metadata(src_w: int, src_h: int, scene: str, seed: int, n_frames: int, mb_size: int = 16) -> np.ndarray:
    """[n_frames][rows][cols] MB records of one stream (I-frame slots are filled but never read)."""
    gen = StreamGen(src_w, src_h, scene, seed, mb_size)
    return np.stack([gen.next_frame() for _ in range(n_frames)])


def random_bf16(shape, rng: np.random.Generator) -> np.ndarray:
    """N(0, 1) values truncated to bf16, returned as raw uint16 bits."""
    x = rng.standard_normal(size=shape, dtype=np.float32)
    return (x.view(np.uint32) >> 16).astype(np.uint16)


def random_frames(n: int, H: int, W: int, rng: np.random.Generator) -> list:
    """n model-input frames [3][H][W] (bf16 bits)."""
    return [random_bf16((3, H, W), rng) for _ in range(n)]


# FFmpeg's public AVMotionVector layout (libavutil/motion_vector.h), 40 B: the decoder's motion-vector export that
# codecsight_mv_rasterize ingests (NEXT-4).
AV_MV_DTYPE = np.dtype([("source", "<i4"), ("w", "u1"), ("h", "u1"), ("src_x", "<i2"), ("src_y", "<i2"),
                        ("dst_x", "<i2"), ("dst_y", "<i2"), ("pad0", "<u2"), ("flags", "<u8"), ("motion_x", "<i4"),
                        ("motion_y", "<i4"), ("motion_scale", "<u2"), ("pad1", "u1", (6,))])
assert AV_MV_DTYPE.itemsize == 40

# H.264 inter partition modes of a 16x16 MB (partition w, h) and their frequencies in the generated streams:
# 16x16 (skip and most inter MBs), 16x8, 8x16, 8x8 (P_8x8: libavcodec exports each 8x8 block as one 8x8 record with
# its first sub-partition's vector whatever its sub-partitioning -- checked against the real decoder,
# tests/test_real_h264.py -- so no sub-8x8 records are generated)
_PART_MODES = ((16, 16), (16, 8), (8, 16), (8, 8))
_PART_P = (0.55, 0.15, 0.15, 0.15)


def avmv_records(mb: np.ndarray, rng: np.random.Generator, mb_size: int = 16) -> np.ndarray:
    """AVMotionVector records of one P-frame, shaped like libavcodec's H.264 export, drawn from the frame's MB
    records `mb` [rows][cols] (the scene truth): an INTRA MB exports nothing; a SKIP MB one 16x16 record with its
    (predicted) vector; an INTER MB 1, 2 or 4 partitions (16x16 / 16x8 / 8x16 / 8x8) whose vectors are the MB's
    vector with +-1 qpel jitter on some partitions (p = 0.3).  motion_scale 4 (quarter pel),
    source -1 (past reference), dst = the partition centre in px.  Records are in raster order of MBs."""
    rows, cols = mb.shape
    jj, ii = np.nonzero(mb["type"] != MB_INTRA)
    mode = rng.choice(len(_PART_MODES), size=jj.size, p=_PART_P)
    mode[mb["type"][jj, ii] == MB_SKIP] = 0
    recs = []
    for m, (pw, ph) in enumerate(_PART_MODES):
        sel = mode == m
        if not sel.any():
            continue
        j, i = jj[sel], ii[sel]
        for oy in range(0, mb_size, ph):
            for ox in range(0, mb_size, pw):
                parts = [(np.ones(j.size, bool), ox, oy, pw, ph)]
                for msk, px, py, w, h in parts:
                    if not msk.any():
                        continue
                    jm, im = j[msk], i[msk]
                    a = np.zeros(jm.size, AV_MV_DTYPE)
                    a["source"] = -1
                    a["w"], a["h"] = w, h
                    a["dst_x"] = im * mb_size + px + w // 2
                    a["dst_y"] = jm * mb_size + py + h // 2
                    a["src_x"], a["src_y"] = a["dst_x"], a["dst_y"]
                    jit = (rng.random((jm.size, 2)) < 0.3) * rng.integers(-1, 2, size=(jm.size, 2))
                    skip = mb["type"][jm, im] == MB_SKIP
                    jit[skip] = 0
                    a["motion_x"] = mb["mvx"][jm, im].astype(np.int32) + jit[:, 0]
                    a["motion_y"] = mb["mvy"][jm, im].astype(np.int32) + jit[:, 1]
                    a["motion_scale"] = 4
                    a["src_x"] = (a["dst_x"] + a["motion_x"] // 4).astype(np.int16)
                    a["src_y"] = (a["dst_y"] + a["motion_y"] // 4).astype(np.int16)
                    recs.append((jm * cols + im, a))
    if not recs:
        return np.zeros(0, AV_MV_DTYPE)
    key = np.concatenate([k for k, _ in recs])
    out = np.concatenate([a for _, a in recs])
    return out[np.argsort(key, kind="stable")]
