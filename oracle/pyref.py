"""Second, independent transcription of the path in pure Python (TEST INFRASTRUCTURE ONLY).

Written separately from ``oracle/codecsight_ref.c`` (different structure: exact rationals, Python ints,
per-patch dictionaries) for tiny inputs only (<= 8x8 patch grids, <= 16 frames).  Tests require it to equal
the C oracle bit for bit; a transcription slip in either shows up as a disagreement.

Floating point follows the same IEEE single-precision operations the paper's definition implies
(Eq. 1-5): sqrt is correctly rounded (numpy float32 sqrt), fma is emulated exactly
(exact rational product-sum, then correct rounding to float32), the RoPE angle is a double product and
cos/sin are the platform libm's, as in the C oracle.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

INF = float("inf")


def f32(x) -> np.float32:
    return np.float32(x)


def round_f32(q: Fraction) -> np.float32:
    """Correctly rounded (ties-to-even) float32 nearest to the exact rational q."""
    if q == 0:
        return np.float32(0.0)
    x = np.float32(float(q))
    cands = [x, np.nextafter(x, np.float32(np.inf)), np.nextafter(x, np.float32(-np.inf))]
    best = None
    for c in cands:
        if not np.isfinite(c):
            continue
        d = abs(Fraction(float(c)) - q)
        key = (d, int(np.array(c, np.float32).view(np.uint32)) & 1)
        if best is None or key < best[0]:
            best = (key, c)
    return np.float32(best[1])


def fmaf(a, b, c) -> np.float32:
    return round_f32(Fraction(float(f32(a))) * Fraction(float(f32(b))) + Fraction(float(f32(c))))


def magnitude(dx: int, dy: int, t: int) -> np.float32:
    """Eq. 1 on quarter-pel vectors; INTRA/unknown -> +inf."""
    if t not in (0, 1):
        return np.float32(INF)
    return np.float32(np.sqrt(np.float32(dx * dx + dy * dy))) * np.float32(0.25)


def fields(g: dict, mb) -> dict:
    """{(r, c): (V, R, M)} for one P-frame.  mb: [rows][cols] structured records."""
    out = {}
    W, H, m = g["grid_w"], g["grid_h"], g["mb_size"]
    for r in range(H):
        for c in range(W):
            # patch rectangle in true (rational) source pixels
            x0, x1 = Fraction(c * g["src_w"], W), Fraction((c + 1) * g["src_w"], W)
            y0, y1 = Fraction(r * g["src_h"], H), Fraction((r + 1) * g["src_h"], H)
            vmax = None
            acc = Fraction(0)
            for j in range(g["mb_rows"]):
                for i in range(g["mb_cols"]):
                    ox = min(x1, (i + 1) * m) - max(x0, i * m)
                    oy = min(y1, (j + 1) * m) - max(y0, j * m)
                    if ox > 0 and oy > 0:
                        rec = mb[j][i]
                        v = magnitude(int(rec["mvx"]), int(rec["mvy"]), int(rec["type"]))
                        vmax = v if vmax is None or v > vmax else vmax
                        acc += ox * oy * Fraction(int(rec["sad"]), m * m)   # area x mean |residual|
            area = (x1 - x0) * (y1 - y0)
            R = np.float32(float(acc / area / 255))  # exact rational -> double -> float (as the definition)
            # the C oracle divides two exact doubles; the quotient's double rounding equals float(acc/area/255)
            M = np.float32(INF) if np.isinf(vmax) else fmaf(g["alpha"], R, vmax)
            out[(r, c)] = (np.float32(vmax), R, M)
    return out


def score_stream(g: dict, mbs, types, state=None):
    """GOP accumulation + group-complete for one stream.  Returns (keep [n][H][W] bool, kept [n], M [n][H][W],
    final (state_set, init_flag)).  ``state`` = (set of patch (r, c), init flag)."""
    W, H, G = g["grid_w"], g["grid_h"], g["group"]
    active, init = (set(), False) if state is None else (set(state[0]), state[1])
    keeps, kepts, scores = [], [], []
    for f, t in enumerate(types):
        if t != 1:  # I-frame (or unknown type, treated as I): all patches, state reset
            active, init = set(), True
            cur = {(r, c) for r in range(H) for c in range(W)}
            M = np.full((H, W), np.inf, np.float32)
        else:
            if not init:
                active, init = set(), True
            fl = fields(g, mbs[f])
            M = np.zeros((H, W), np.float32)
            for (r, c), (_, _, m) in fl.items():
                M[r, c] = m
                if m >= np.float32(g["tau"]):
                    active.add((r, c))
            cur = set(active)
        keep = np.zeros((H, W), bool)
        for gr in range(H // G):
            for gc in range(W // G):
                members = [(gr * G + a, gc * G + b) for a in range(G) for b in range(G)]
                if any(p in cur for p in members):
                    for p in members:
                        keep[p] = True
        keeps.append(keep)
        kepts.append(int(keep.sum()))
        scores.append(M)
    return np.array(keeps), np.array(kepts), np.array(scores), (active, init)


def tokens(g: dict, keep) -> list:
    """Kept groups of one frame, row-major (a group is a token if any of its patches is kept)."""
    G = g["group"]
    H, W = keep.shape
    return [(gr, gc) for gr in range(H // G) for gc in range(W // G)
            if keep[gr * G:(gr + 1) * G, gc * G:(gc + 1) * G].any()]


def plan(g: dict, keeps: dict, types: dict, w: int, s: int, k: int, n_prompt: int):
    """Prefill plan of window k.  keeps/types: frame index -> keep [H][W] / type.
    Returns list of (p_new, disposition, p_old) and (n_visual, n_reuse, n_anchor, n_new)."""
    NEW, ANCHOR, REUSE = 0, 1, 2
    prev = {}
    if k >= 1:
        pos = 0
        for f in range((k - 1) * s, (k - 1) * s + w):
            for t in tokens(g, keeps[f]):
                prev[(f, t)] = pos
                pos += 1
    out = []
    pos = 0
    for f in range(k * s, k * s + w):
        for t in tokens(g, keeps[f]):
            if k == 0 or (f, t) not in prev:
                d, po = NEW, -1
            elif types[f] == 0 or f == k * s:
                d, po = ANCHOR, prev[(f, t)]
            else:
                d, po = REUSE, prev[(f, t)]
            out.append((pos, d, po))
            pos += 1
    nv = pos
    for _ in range(n_prompt):
        out.append((pos, NEW, -1))
        pos += 1
    cnt = (nv, sum(1 for o in out if o[1] == REUSE), sum(1 for o in out if o[1] == ANCHOR),
           sum(1 for o in out if o[1] == NEW))
    return out, cnt


def rope_rotate(k, n_heads: int, head_dim: int, base: float, dp: int) -> np.ndarray:
    """Eq. 5 on fp32 vectors, rotate_half pairing (i, i + D/2)."""
    k = np.asarray(k, np.float32)
    out = np.zeros_like(k)
    half = head_dim // 2
    for h in range(n_heads):
        for i in range(half):
            inv = base ** (-2.0 * i / head_dim)
            ang = float(dp) * inv
            c, s = np.float32(math.cos(ang)), np.float32(math.sin(ang))
            x1, x2 = k[h * head_dim + i], k[h * head_dim + i + half]
            out[h * head_dim + i] = fmaf(x1, c, -(np.float32(x2 * s)))
            out[h * head_dim + i + half] = fmaf(x2, c, np.float32(x1 * s))
    return out
