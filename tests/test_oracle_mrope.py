"""Pins of the M-RoPE position correction (NEXT-3: Qwen2-VL / Qwen3-VL multimodal rotary).

A reused visual token keeps its (h, w) position and moves in time by dt = -stride * t_per_frame, so Eq. 5 rotates
only the temporal frequency section.  Checked against an independent float64 transcription of the Hugging Face
`apply_multimodal_rotary_pos_emb` rule (cos/sin split into mrope_section * 2 chunks, chunk j from component j % 3)."""
import numpy as np
import pytest

import synth
from synth import make_grid
from test_oracle_pins import _masks_from_groups


def mrope_textbook(x, pos, base, sections):
    """x [H][D] float64; pos = (t, h, w); HF rule: split the duplicated cos/sin along D into sections*2 chunks."""
    H, D = x.shape
    inv = base ** (-np.arange(0, D, 2, dtype=np.float64) / D)            # [D/2]
    freqs = np.stack([p * inv for p in pos])                               # [3][D/2]
    emb = np.concatenate([freqs, freqs], axis=1)                           # [3][D]
    chunks = list(sections) * 2
    bounds = np.cumsum([0] + chunks)
    ang = np.concatenate([emb[j % 3, bounds[j]:bounds[j + 1]] for j in range(len(chunks))])
    cos, sin = np.cos(ang), np.sin(ang)
    rot_half = np.concatenate([-x[:, D // 2:], x[:, :D // 2]], axis=1)
    return x * cos + rot_half * sin


def _setup(dtype=1, H=2, D=16, sections=(2, 3, 3), tpf=1):
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    kept = [[0, 1, 2, 3], [1], [1, 3], [1, 3], [0, 1, 2, 3], [0], [0], [0, 2],
            [0, 1, 2, 3], [], [], [3], [0, 1, 2, 3], [2], [2], [2, 3]]
    masks = _masks_from_groups(g, kept)
    types = np.array([0 if f % 4 == 0 else 1 for f in range(16)], np.uint8)
    kv = dict(layers=2, kv_heads=H, head_dim=D, dtype=dtype, capacity=32, refresh_capacity=32, rope_base=1e4,
              n_prompt=2, rope_mode=1, mrope_section=sections, t_per_frame=tpf)
    return g, kept, masks, types, kv


def test_mrope_rotates_only_the_temporal_section(ref):
    g, kept, masks, types, kv = _setup()
    rng = np.random.default_rng(0)
    old = rng.standard_normal((2, 2, 32, 2, 16)).astype(np.float32)
    new = np.zeros_like(old)
    out = ref.kv_refresh(g, kv, dict(window=12, stride=4, step=1, ring_frames=16), masks[None], types[None],
                         [old], [new], None, 32)
    assert out["rc"] == 0 and out["status"] == 0
    reuse = [p for p in range(21) if out["disposition"][0, p] == 2]
    assert len(reuse) == 5
    for p in reuse:
        po = out["p_old"][0, p]
        for l in range(2):
            exp = mrope_textbook(old[l, 0, po].astype(np.float64), (-4, 0, 0), 1e4, (2, 3, 3))
            assert np.abs(new[l, 0, p] - exp).max() <= 2e-6
            # pairs of the h and w sections (i = 2..7 and i + 8) are untouched bit for bit
            for i in list(range(2, 8)):
                assert (new[l, 0, p][:, [i, i + 8]] == old[l, 0, po][:, [i, i + 8]]).all()
        assert (new[:, 1, p] == old[:, 1, po]).all()


def test_mrope_layer1_exactness(ref):
    """Keys stored as MRoPE(x, pos_old) and corrected by the oracle equal MRoPE(x, pos_new) (S:380 analogue)."""
    g, kept, masks, types, kv = _setup(H=2, D=32, sections=(4, 6, 6), tpf=2)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((32, 2, 32))                        # pre-rotation keys per old position
    old = np.zeros((2, 2, 32, 2, 32), np.float32)
    w, s = 12, 4
    # window 0 tokens: frame f, groups kept[f]; position (t = f * tpf, gr, gc)
    pos_of_old = {}
    p = 0
    for f in range(0, w):
        for q in kept[f]:
            gr, gc = divmod(q, 2)
            pos_of_old[p] = (f, q, (f * 2, gr, gc))
            for l in range(2):
                old[l, 0, p] = mrope_textbook(x[p], (f * 2, gr, gc), 1e4, (4, 6, 6))
            p += 1
    new = np.zeros_like(old)
    out = ref.kv_refresh(g, kv, dict(window=w, stride=s, step=1, ring_frames=16), masks[None], types[None],
                         [old], [new], None, 32)
    for pn in range(21):
        if out["disposition"][0, pn] != 2:
            continue
        po = out["p_old"][0, pn]
        f, q, (t, gr, gc) = pos_of_old[po]
        exp = mrope_textbook(x[po], ((f - s) * 2, gr, gc), 1e4, (4, 6, 6))
        assert np.abs(new[0, 0, pn] - exp).max() <= 1e-5


def test_mrope_validation(ref):
    g, kept, masks, types, kv = _setup()
    c = np.zeros((2, 2, 32, 2, 16), np.float32)
    bad = dict(kv, mrope_section=(2, 3, 4))                       # sections must cover D/2 pairs
    out = ref.kv_refresh(g, bad, dict(window=12, stride=4, step=1, ring_frames=16), masks[None], types[None],
                         [c], [c.copy()], None, 32)
    assert out["rc"] == -2


@pytest.mark.parametrize("dtype", [1, 0])
def test_mrope_paged_equals_out_of_place(ref, dtype):
    cfg = synth.CONFIGS["C1"]
    g = make_grid(448, 448)
    w, s, ring = 8, 2, 10
    n_prompt = 3
    cap = w * 256 + n_prompt
    kv = dict(layers=2, kv_heads=2, head_dim=32, dtype=dtype, capacity=cap, refresh_capacity=cap, rope_base=1e6,
              n_prompt=n_prompt, rope_mode=1, mrope_section=(4, 6, 6), t_per_frame=1)
    nf = 5 * s + w
    mb = synth.stream_metadata(448, 448, "multi_object", 5, nf)
    types = synth.frame_types(nf, 4)
    sc = ref.score_patches(g, mb[None], types[None], np.zeros((1, 33), np.uint32), want_score=False)
    rng = np.random.default_rng(2)

    def rc(rows):
        shp = (2, 2, rows, 2, 32)
        if dtype == 1:
            return rng.standard_normal(shp).astype(np.float32)
        return rng.integers(0, 65536, size=shp, dtype=np.uint16) & np.uint16(0xBFFF)

    pool = rc(cap)
    slot, oop_old = None, None
    for k in range(6):
        mring = np.zeros((1, ring, 32), np.uint32)
        tring = np.zeros((1, ring), np.uint8)
        for f in range(max(0, (k - 1) * s), k * s + w):
            mring[0, f % ring] = sc["keep_mask"][0, f]
            tring[0, f % ring] = types[f]
        win = dict(window=w, stride=s, step=k, ring_frames=ring)
        refr = rc(cap)
        oop_new = np.zeros_like(pool)
        o = ref.kv_refresh(g, kv, win, mring, tring, [oop_old] if k else None, [oop_new], [refr], cap)
        pg = ref.kv_refresh_paged(g, kv, win, mring, tring, [pool], slot, cap, [refr], cap)
        nt = int(o["n_tokens"][0, 0]) + n_prompt
        sn = pg["slot_new"][0, :nt]
        assert (pool[:, :, sn] == oop_new[:, :, :nt]).all()
        slot, oop_old = pg["slot_new"], oop_new


@pytest.mark.parametrize("paged", [False, True])
def test_mrope_hw_sections_keep_their_bits(ref, paged):
    """-0.0, +inf and NaN stored in the h / w sections survive a reuse bit for bit (they are not rotated by 0,
    which would turn -0 into +0 and inf into NaN); the temporal section is rotated."""
    g, kept, masks, types, kv = _setup()
    rng = np.random.default_rng(7)
    old = rng.standard_normal((2, 2, 32, 2, 16)).astype(np.float32)
    special = np.array([-0.0, np.inf, -np.inf, np.nan], np.float32)
    old[:, 0, :, :, 2:6] = special                       # pairs 2..5 (h section), first halves
    win = dict(window=12, stride=4, step=1, ring_frames=16)
    if paged:
        pool = old.copy()
        slot_old = np.arange(32, dtype=np.int32)[None]
        out = ref.kv_refresh_paged(g, kv, win, masks[None], types[None], [pool], slot_old, 32, None, 32)
        got = lambda p: pool[:, 0, out["slot_new"][0, p]]
    else:
        new = np.zeros_like(old)
        out = ref.kv_refresh(g, kv, win, masks[None], types[None], [old], [new], None, 32)
        got = lambda p: new[:, 0, p]
    reuse = [p for p in range(21) if out["disposition"][0, p] == 2]
    assert reuse
    for p in reuse:
        po = out["p_old"][0, p]
        a, b = got(p), old[:, 0, po]
        assert (a[..., 2:8].view(np.uint32) == b[..., 2:8].view(np.uint32)).all()
        assert (a[..., 10:16].view(np.uint32) == b[..., 10:16].view(np.uint32)).all()
        assert not (a[..., 0:2] == b[..., 0:2]).all()     # temporal pairs rotated


def test_mrope_paged_bytes_count_the_rotated_section(ref):
    """In place, a reused key moves only its temporal section: L * H * 2 * s_t elements read + written."""
    g, kept, masks, types, kv = _setup(dtype=1, H=2, D=16, sections=(2, 3, 3))
    pool = np.zeros((2, 2, 32, 2, 16), np.float32)
    out = ref.kv_refresh_paged(g, kv, dict(window=12, stride=4, step=1, ring_frames=16), masks[None], types[None],
                               [pool], np.arange(32, dtype=np.int32)[None], 32, None, 32)
    n_reuse = int(out["n_tokens"][0, 1])
    assert n_reuse == 5
    assert int(out["counters"][10]) == n_reuse * 2 * 2 * 2 * 2 * 4 * 2   # L * H * 2 s_t * 4 B * (r + w); no refreshed
