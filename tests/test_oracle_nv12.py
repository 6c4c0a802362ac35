"""Pins of the fused preprocessing oracle (NEXT-2: NV12 -> RGB -> bilinear resize -> normalise).

Colour conversion against BT.601 closed forms; the resize against PyTorch's bilinear interpolation
(align_corners=False, antialias=False) as a library routine; the compaction of preprocessed patches against the
plain compaction of the fully preprocessed frame (index mapping)."""
import numpy as np
import pytest
import torch

from synth import make_grid


def _nv12(h, w, rng):
    Y = rng.integers(16, 236, size=(h, w), dtype=np.uint8)
    UV = rng.integers(16, 241, size=(h // 2, w), dtype=np.uint8)
    return Y, UV


def _bf16(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def test_bt601_closed_forms(ref):
    pre = ref.make_pre(2, 2)
    cases = {(16, 128, 128): (0, 0, 0), (235, 128, 128): (255, 255, 255),
             (81, 90, 240): (255, 0, 0), (145, 54, 34): (0, 255, 0), (41, 240, 110): (0, 0, 255)}
    for (y, u, v), rgb in cases.items():
        Y = np.full((2, 2), y, np.uint8)
        UV = np.array([[u, v]], np.uint8)
        got = ref.nv12_rgb(Y, UV, pre, 1, 1)
        assert np.abs(got - np.array(rgb, np.float32)).max() <= 1.5, ((y, u, v), got)
    # chroma siting: pixel (y, x) takes UV of (y//2, x//2)
    Y = np.full((4, 4), 128, np.uint8)
    UV = np.array([[128, 128, 200, 60], [128, 128, 128, 128]], np.uint8)
    assert (ref.nv12_rgb(Y, UV, pre, 1, 3) == ref.nv12_rgb(Y, UV, pre, 0, 2)).all()
    assert not (ref.nv12_rgb(Y, UV, pre, 2, 2) == ref.nv12_rgb(Y, UV, pre, 0, 2)).all()


@pytest.mark.parametrize("src", [(64, 48), (120, 90), (16, 12), (32, 32)])
def test_resize_matches_torch_bilinear(ref, src):
    sw, sh = src
    g = make_grid(sw, sh, grid_w=4, grid_h=4, patch=8, group=2)
    rng = np.random.default_rng(sw * 7 + sh)
    Y, UV = _nv12(sh, sw, rng)
    pre = ref.make_pre(sw, sh)
    rgb = np.zeros((3, sh, sw), np.float32)
    for y in range(sh):
        for x in range(sw):
            rgb[:, y, x] = ref.nv12_rgb(Y, UV, pre, y, x)
    res = torch.nn.functional.interpolate(torch.from_numpy(rgb)[None], size=(32, 32), mode="bilinear",
                                          align_corners=False, antialias=False)[0].numpy()
    mean = np.array(ref.CLIP_MEAN, np.float32)[:, None, None]
    std = np.array(ref.CLIP_STD, np.float32)[:, None, None]
    exp = _bf16(((res / np.float32(255.0)) - mean) / std)
    got = ref.preprocess_frame(g, pre, Y, UV)
    fe = (exp.astype(np.uint32) << 16).view(np.float32)
    fg = (got.astype(np.uint32) << 16).view(np.float32)
    ulp = np.abs(fe) * 2.0 ** -7 + 1e-30
    assert (np.abs(fg - fe) <= ulp).all()                     # within one bf16 ulp of PyTorch's bilinear
    assert (got == exp).mean() >= 0.99                         # and almost always bit-identical
    if src == (32, 32):                                        # identity scale: conversion only
        direct = _bf16(((rgb / np.float32(255.0)) - mean) / std)
        assert (got == direct).all()


def test_compact_nv12_equals_compact_of_preprocessed(ref):
    g = make_grid(120, 90, grid_w=8, grid_h=6, patch=6, group=2)
    rng = np.random.default_rng(3)
    S, n = 2, 2
    ys, uvs, planar = [], [], []
    pre = ref.make_pre(120, 90)
    for _ in range(S * n):
        Y, UV = _nv12(90, 120, rng)
        ys.append(Y)
        uvs.append(UV)
        planar.append(ref.preprocess_frame(g, pre, Y, UV))
    nw = 2
    km = rng.integers(0, 2**32, size=(S, n, nw), dtype=np.uint64).astype(np.uint32)
    fidx = np.arange(S * n, dtype=np.int32)
    a = ref.compact(g, km, fidx, planar, S * n * 48, S, n)
    b = ref.compact_nv12(g, pre, km, fidx, ys, uvs, S * n * 48, S, n)
    for key in ("packed", "pos_ids", "src_index", "frame_offsets"):
        assert (a[key] == b[key]).all(), key
    assert b["counters"][ref.C_PACKED_ROWS] == a["counters"][ref.C_PACKED_ROWS]


def _group_mask(g, groups):
    """Keep mask (one frame) with the given (gr, gc) groups set."""
    bits = np.zeros(g["grid_w"] * g["grid_h"], np.uint8)
    G = g["group"]
    for gr, gc in groups:
        for dy in range(G):
            for dx in range(G):
                bits[(gr * G + dy) * g["grid_w"] + gc * G + dx] = 1
    return np.packbits(bits, bitorder="little").view(np.uint32)


@pytest.mark.parametrize("src", [(64, 64), (128, 96)])
def test_nv12_source_sector_bytes(ref, src):
    """Algorithmic source bytes of the fused preprocessing (reading NEXT-2 bytes): the distinct 32-B sectors of the
    Y and UV planes that the kept groups' bilinear taps touch.  Closed forms at a 64 x 64 model input (grid 8 x 8,
    patch 8, 2 x 2 groups of 16 px):
      identity scale (src 64 x 64): taps of model px o are o and o + 1 (clamped), so group (0, 0) reads luma rows
        and columns 0..16 -> 17 rows x 1 sector + 9 UV rows x 1 sector = 26 sectors; every group -> all 64 rows x
        2 sectors + 32 UV rows x 2 = 192 sectors;
      src 128 x 96 (scale 2 x 1.5): group (0, 0) taps columns 2o, 2o + 1 for o < 16 -> 0..31 (sector 0) and rows
        floor(1.5 o + 0.25), +1 -> rows 0..23: 24 rows + 12 UV rows = 36 sectors.
    Pitches that are not multiples of 32 leave the source bytes uncounted."""
    g = make_grid(*src, grid_w=8, grid_h=8, patch=8, group=2)
    rng = np.random.default_rng(0)
    Y, UV = _nv12(src[1], src[0], rng)
    pre = ref.make_pre(*src)
    out_only = 4 * 2 + 4
    row = 3 * 8 * 8 * 2 + 16

    def bytes_for(groups, pre_=pre):
        km = _group_mask(g, groups)[None, None]
        o = ref.compact_nv12(g, pre_, km, np.zeros(1, np.int32), [Y], [UV], 64, 1, 1)
        return int(o["counters"][ref.C_BYTES_COMPACT]) - out_only - 4 * len(groups) * row

    one = 26 if src == (64, 64) else 36
    assert bytes_for([(0, 0)]) == one * 32
    if src == (64, 64):
        assert bytes_for([(r, c) for r in range(4) for c in range(4)]) == 192 * 32
    # vertically adjacent groups share their boundary rows: the union, not the sum
    if src == (64, 64):
        assert bytes_for([(0, 0), (1, 0)]) == (33 + 17) * 32     # luma rows 0..32, UV rows 0..16, one sector each
    else:                                                        # scale 1.5: group row 1 starts at luma row 24
        assert bytes_for([(0, 0), (1, 0)]) == 2 * one * 32
    # a pitch that is not a multiple of 32: outputs only
    Yp = np.zeros((src[1], src[0] + 8), np.uint8)
    Yp[:, :src[0]] = Y
    UVp = np.zeros((src[1] // 2, src[0] + 8), np.uint8)
    UVp[:, :src[0]] = UV
    pre2 = ref.make_pre(*src, y_pitch=src[0] + 8, uv_pitch=src[0] + 8)
    km = _group_mask(g, [(0, 0)])[None, None]
    o = ref.compact_nv12(g, pre2, km, np.zeros(1, np.int32), [Yp], [UVp], 64, 1, 1)
    assert int(o["counters"][ref.C_BYTES_COMPACT]) == out_only + 4 * row
