"""The C oracle against an independent pure-Python transcription (oracle/pyref.py), bit for bit, on tiny
inputs (<= 8x8 patches, <= 16 frames), plus randomized invariants."""
import numpy as np
import pytest

import oracle.pyref as py
from synth import MB_DTYPE, frame_types, make_grid, random_mb, stream_metadata

GEOMS = [
    # (src_w, src_h, mb, grid_w, grid_h, group)
    (40, 36, 8, 4, 4, 2),
    (64, 48, 16, 8, 6, 2),
    (30, 30, 8, 6, 6, 3),
    (56, 56, 16, 4, 4, 1),
    (100, 44, 16, 8, 8, 4),
]


@pytest.mark.parametrize("geom", GEOMS)
@pytest.mark.parametrize("alpha", [0.0, 0.25, 1.0, 5.0])
@pytest.mark.parametrize("tau", [0.0, 0.25, 1.0, 5.0])
def test_fields_and_scores_bit_exact(ref, geom, alpha, tau):
    sw, sh, m, gw, gh, G = geom
    g = make_grid(sw, sh, tau=tau, alpha=alpha, mb_size=m, grid_w=gw, grid_h=gh, group=G, patch=4)
    rng = np.random.default_rng(hash((geom, alpha, tau)) % 2**32)
    n = 6
    mb = np.stack([random_mb(g["mb_rows"], g["mb_cols"], rng, p_intra=0.03, mv_max=6) for _ in range(n)])
    ft = np.array([0, 1, 1, 0, 1, 1], np.uint8)
    nw = (gw * gh + 31) // 32
    out = ref.score_patches(g, mb[None], ft[None], np.zeros((1, nw + 1), np.uint32))
    keeps, kepts, scores, _ = py.score_stream(g, mb, ft)
    assert (out["kept_count"][0] == kepts).all()
    bits = np.unpackbits(out["keep_mask"][0].view(np.uint8), bitorder="little").reshape(n, nw * 32)[:, :gw * gh]
    assert (bits.reshape(n, gh, gw).astype(bool) == keeps).all()
    got = out["score"][0].reshape(n, gh, gw)
    assert (got.view(np.uint32) == scores.astype(np.float32).view(np.uint32)).all()
    # V and R individually
    V, R, M, _ = ref.patch_fields(g, mb[1])
    fl = py.fields(g, mb[1])
    for (r, c), (v, rr, mm) in fl.items():
        assert V[r, c] == v and R[r, c] == rr and M[r, c].view(np.uint32) == np.float32(mm).view(np.uint32)


def test_plan_vs_pyref_random(ref):
    rng = np.random.default_rng(123)
    for trial in range(60):
        G = int(rng.choice([1, 2]))
        gw, gh = int(rng.choice([2, 4])) * 2, int(rng.choice([2, 4])) * 2
        g = make_grid(64, 64, mb_size=16, grid_w=gw, grid_h=gh, group=G, patch=4)
        w = int(rng.integers(1, 9))
        s = int(rng.integers(1, w + 1))
        k = int(rng.integers(0, 4))
        gop = int(rng.integers(1, 7))
        ring = w + s + int(rng.integers(0, 3))
        nf = k * s + w
        keeps = {}
        types = {}
        nw = (gw * gh + 31) // 32
        ring_masks = np.zeros((ring, nw), np.uint32)
        ring_types = np.zeros(ring, np.uint8)
        dens = rng.random()
        for f in range(max(0, (k - 1) * s), nf):
            kp = rng.random((gh, gw)) < dens
            keeps[f] = kp
            types[f] = 0 if f % gop == 0 else 1
            bits = np.zeros(nw * 32, np.uint8)
            bits[:gw * gh] = kp.reshape(-1)
            ring_masks[f % ring] = np.packbits(bits, bitorder="little").view(np.uint32)
            ring_types[f % ring] = types[f]
        n_prompt = int(rng.integers(0, 4))
        kv = dict(layers=1, kv_heads=1, head_dim=4, dtype=1, capacity=4096, refresh_capacity=4096, rope_base=1e4,
                  n_prompt=n_prompt)
        old = rng.standard_normal((1, 2, 4096, 1, 4)).astype(np.float32)
        new = np.zeros_like(old)
        out = ref.kv_refresh(g, kv, dict(window=w, stride=s, step=k, ring_frames=ring), ring_masks[None],
                             ring_types[None], [old] if k else None, [new], None, 4096)
        assert out["rc"] == 0
        exp, cnt = py.plan(g, keeps, types, w, s, k, n_prompt)
        assert tuple(out["n_tokens"][0]) == cnt
        for (pn, d, po) in exp:
            assert out["disposition"][0, pn] == d and out["p_old"][0, pn] == po, (trial, pn)
        # Q12: dp is uniform over the REUSE/ANCHOR tokens of a stream-step
        dps = {pn - po for (pn, d, po) in exp if d != 0}
        assert len(dps) <= 1


def test_rope_vs_pyref(ref):
    rng = np.random.default_rng(7)
    for dp in [0, 1, -1, -9, -4096, 12345]:
        for base in [1e4, 1e6]:
            k = rng.standard_normal(2 * 16).astype(np.float32)
            a = ref.rope_rotate_f32(k, 2, 16, base, dp)
            b = py.rope_rotate(k, 2, 16, base, dp)
            assert (a.view(np.uint32) == b.view(np.uint32)).all()


@pytest.mark.parametrize("scene", ["static", "translating_object", "multi_object", "noise", "scene_cut", "low",
                                   "high"])
def test_invariants_on_synthetic_streams(ref, scene):
    """monotone growth within a GOP, group-completeness, kept % group^2 == 0, I-frames keep all."""
    g = make_grid(448, 448)
    n = 16
    mb = stream_metadata(448, 448, scene, 42, n)[None]
    ft = frame_types(n, 4)[None]
    out = ref.score_patches(g, mb, ft, np.zeros((1, 33), np.uint32))
    km = out["keep_mask"][0]
    kc = out["kept_count"][0]
    assert (kc % 4 == 0).all()
    bits = np.unpackbits(km.view(np.uint8), bitorder="little").reshape(n, 32, 32).astype(bool)
    for f in range(n):
        b = bits[f].reshape(16, 2, 16, 2)
        grp = b.any(axis=(1, 3))
        assert (b.all(axis=(1, 3)) == grp).all()                  # group-complete
        if ft[0, f] == 0:
            assert kc[f] == 1024
        elif ft[0, f - 1] == 1:
            assert (bits[f] | bits[f - 1] == bits[f]).all()        # monotone within the GOP
    if scene == "static":
        assert (kc[ft[0] == 1] == 0).all()


def test_validation_codes(ref):
    g = make_grid(448, 448)
    bad = dict(g, mb_cols=27)
    mb = np.zeros((1, 1, 28, 28), MB_DTYPE)
    assert ref.score_patches(bad, mb, np.zeros((1, 1), np.uint8), np.zeros((1, 33), np.uint32))["rc"] == -2
    bad = dict(g, group=3)
    assert ref.score_patches(bad, mb, np.zeros((1, 1), np.uint8), np.zeros((1, 33), np.uint32))["rc"] == -2
    bad = dict(g, tau=float("nan"))
    assert ref.score_patches(bad, mb, np.zeros((1, 1), np.uint8), np.zeros((1, 33), np.uint32))["rc"] == -1
    kv = dict(layers=1, kv_heads=1, head_dim=3, dtype=1, capacity=8, refresh_capacity=8, rope_base=1e4, n_prompt=0)
    c = np.zeros((1, 2, 8, 1, 3), np.float32)
    r = ref.kv_refresh(g, kv, dict(window=4, stride=2, step=0, ring_frames=4), np.zeros((1, 4, 32), np.uint32),
                       np.zeros((1, 4), np.uint8), None, [c], None, 8)
    assert r["rc"] == -3                                               # odd head_dim
    kv["head_dim"] = 4
    c = np.zeros((1, 2, 8, 1, 4), np.float32)
    r = ref.kv_refresh(g, kv, dict(window=4, stride=5, step=0, ring_frames=9), np.zeros((1, 9, 32), np.uint32),
                       np.zeros((1, 9), np.uint8), None, [c], None, 8)
    assert r["rc"] == -3                                               # s > w
    r = ref.kv_refresh(g, kv, dict(window=4, stride=2, step=1, ring_frames=5), np.zeros((1, 5, 32), np.uint32),
                       np.zeros((1, 5), np.uint8), [c], [c.copy()], None, 8)
    assert r["rc"] == -2                                               # ring shorter than w + s
