"""Pins of the temporal-patch compaction (NEXT-3, Qwen2-VL temporal_patch_size = 2).

The packed rows are pinned against the Hugging Face Qwen2-VL video processor itself (a library routine: with resize,
rescale and normalisation off it is exactly the flatten into [3][2][14][14] rows in merge-group order), the
pruning rule by a hand example (union over the unit's frames), and tp = 1 by equality with the plain compaction."""
import numpy as np
import pytest
import torch

import synth
from synth import make_grid


def _bf16_frames(n, h, w, rng):
    return [synth.random_frames(1, h, w, rng)[0] for _ in range(n)]


def _f32(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32)


def to_grouped(frame, g):
    p, G = g["patch"], g["group"]
    ngr, ngc = g["grid_h"] // G, g["grid_w"] // G
    x = frame.reshape(3, ngr, G, p, ngc, G, p)
    return np.ascontiguousarray(x.transpose(1, 4, 2, 5, 0, 3, 6)).reshape(-1)


def _hf_flatten(frames_u16):
    """Qwen2VLVideoProcessor on a [T][3][H][W] clip (values exact in bf16), transforms off."""
    from transformers.models.qwen2_vl.video_processing_qwen2_vl import Qwen2VLVideoProcessor
    vp = Qwen2VLVideoProcessor()
    v = torch.from_numpy(np.stack([_f32(f) for f in frames_u16]))
    out = vp(videos=[v], do_resize=False, do_rescale=False, do_normalize=False, do_sample_frames=False,
             return_tensors="pt")
    return out["pixel_values_videos"].numpy(), out["video_grid_thw"].numpy()[0]


@pytest.mark.parametrize("layout", [0, 1])
def test_tp2_all_kept_equals_hf_qwen2vl_processor(ref, layout):
    g = make_grid(448, 448, grid_w=8, grid_h=6, patch=14, group=2)
    rng = np.random.default_rng(5)
    T = 4
    fr = _bf16_frames(T, 6 * 14, 8 * 14, rng)
    hf, thw = _hf_flatten(fr)
    assert tuple(thw) == (2, 6, 8) and hf.shape == (96, 3 * 2 * 14 * 14)
    frames = fr if layout == 0 else [to_grouped(f, g) for f in fr]
    nw = 2
    km = np.full((1, T, nw), 0xFFFFFFFF, np.uint32)
    o = ref.compact_tp(g, 2, km, np.array([0, 1], np.int32), frames, 200, 1, 2, frame_layout=layout)
    assert o["rc"] == 0 and o["frame_offsets"].tolist() == [0, 48, 96]
    assert (_f32(o["packed"][:96]) == hf).all()
    assert o["pos_ids"][47].tolist() == [0, 5, 7] and o["pos_ids"][48].tolist() == [1, 0, 0]


def test_tp2_pruned_rows_are_hf_rows_and_union_rule(ref):
    g = make_grid(448, 448, grid_w=8, grid_h=6, patch=14, group=2)
    rng = np.random.default_rng(6)
    fr = _bf16_frames(4, 84, 112, rng)
    hf, _ = _hf_flatten(fr)
    km = np.zeros((1, 4, 2), np.uint32)
    km[0, 0, 0] = 1 << 0            # unit 0, frame 0: patch (0,0) -> group (0,0)
    km[0, 1, 0] = 1 << (1 * 8 + 7)  # unit 0, frame 1: patch (1,7) -> group (0,3)
    km[0, 3, 1] = 1 << (40 - 32)    # unit 1, frame 1: patch (5,0) -> group (2,0)
    o = ref.compact_tp(g, 2, km, np.array([7, 8], np.int32), fr, 100, 1, 2, want_unit_mask=True,
                       frame_type=np.array([[1, 1, 0, 1]], np.uint8))
    assert o["frame_offsets"].tolist() == [0, 8, 12]
    hw = [tuple(x) for x in o["pos_ids"][:12, 1:].tolist()]
    assert hw[:4] == [(0, 0), (0, 1), (1, 0), (1, 1)] and hw[4:8] == [(0, 6), (0, 7), (1, 6), (1, 7)]
    assert hw[8:12] == [(4, 0), (4, 1), (5, 0), (5, 1)]
    assert o["pos_ids"][:8, 0].tolist() == [7] * 8 and o["pos_ids"][8:12, 0].tolist() == [8] * 4
    # HF row index of (unit t, h, w) in merge-group order
    for n in range(12):
        t = 0 if n < 8 else 1
        h, w = hw[n]
        r = t * 48 + ((h // 2) * 4 + w // 2) * 4 + (h % 2) * 2 + (w % 2)
        assert (_f32(o["packed"][n]) == hf[r]).all()
        assert o["src_index"][n] == t * 48 + h * 8 + w
    assert o["unit_mask"][0, 0].tolist() == [1 | (1 << 15), 0] and o["unit_mask"][0, 1].tolist() == [0, 1 << 8]
    assert o["unit_type"][0].tolist() == [1, 0]          # (P, P) -> P; (I, P) -> I


def test_tp1_equals_plain_compaction(ref):
    g = make_grid(448, 448)
    rng = np.random.default_rng(8)
    S, n = 2, 3
    mb = np.stack([synth.stream_metadata(448, 448, "multi_object", 4 + i, n) for i in range(S)])
    types = np.stack([synth.frame_types(n, 16, 1)] * S)
    km = ref.score_patches(g, mb, types, np.zeros((S, 33), np.uint32))["keep_mask"]
    fr = [synth.random_frames(1, 448, 448, rng)[0] for _ in range(S * n)]
    fidx = np.tile(np.arange(n, dtype=np.int32), S)
    a = ref.compact(g, km, fidx, fr, S * n * 1024, S, n)
    b = ref.compact_tp(g, 1, km, fidx, fr, S * n * 1024, S, n)
    for k in ("packed", "pos_ids", "src_index", "frame_offsets", "counters"):
        assert (a[k] == b[k]).all(), k


def test_tp2_capacity_and_counters(ref):
    g = make_grid(448, 448, grid_w=4, grid_h=4, patch=2, group=2)
    rng = np.random.default_rng(9)
    fr = _bf16_frames(4, 8, 8, rng)
    km = np.full((1, 4, 1), 0xFFFF, np.uint32)
    o = ref.compact_tp(g, 2, km, np.array([0, 1], np.int32), fr, 10, 1, 2)
    assert o["status"] == 1 and o["frame_offsets"].tolist() == [0, 16, 32]
    row = 3 * 2 * 2 * 2
    assert int(o["counters"][11]) == 10
    assert int(o["counters"][9]) == 2 * (4 * 1 * 2 + 4) + 10 * (2 * row * 2 + 16)
