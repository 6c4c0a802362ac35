"""Pins of the in-place / paged KV refresh oracle (NEXT-1, "performs these updates in-place").

The paged variant must produce, through its slot map, exactly the cache the out-of-place oracle produces
(itself pinned in test_oracle_pins.py), while keeping every surviving token's slot, never touching values of
REUSE tokens, and handing the free slots to new tokens in ascending order."""
import numpy as np
import pytest

import synth
from synth import make_grid
from test_oracle_pins import _masks_from_groups


def _kv(cap, rcap, n_prompt, dtype=1, L=2, H=2, D=16, base=1e4):
    return dict(layers=L, kv_heads=H, head_dim=D, dtype=dtype, capacity=cap, refresh_capacity=rcap, rope_base=base,
                n_prompt=n_prompt)


def _rand_cache(kv, rng, rows):
    shape = (kv["layers"], 2, rows, kv["kv_heads"], kv["head_dim"])
    if kv["dtype"] == 1:
        return rng.standard_normal(shape).astype(np.float32)
    return rng.integers(0, 65536, size=shape, dtype=np.uint16) & np.uint16(0xBFFF)


def test_paged_hand_example_slots(ref):
    # the pruned plan of test_plan_hand_example_with_pruning: window 0 (k=0) then window 1 (k=1)
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    kept = [[0, 1, 2, 3], [1], [1, 3], [1, 3], [0, 1, 2, 3], [0], [0], [0, 2],
            [0, 1, 2, 3], [], [], [3], [0, 1, 2, 3], [2], [2], [2, 3]]
    masks = _masks_from_groups(g, kept)
    types = np.array([0 if f % 4 == 0 else 1 for f in range(16)], np.uint8)
    kv = _kv(cap=40, rcap=40, n_prompt=2)
    rng = np.random.default_rng(0)
    pool = _rand_cache(kv, rng, 40)
    refr = _rand_cache(kv, rng, 40)
    w0 = ref.kv_refresh_paged(g, kv, dict(window=12, stride=4, step=0, ring_frames=16), masks[None], types[None],
                              [pool], None, 32, [refr], 32)
    assert w0["rc"] == 0
    assert w0["slot_new"][0, :24].tolist() == list(range(24))       # empty pool: slots in p order
    refr2 = _rand_cache(kv, rng, 40)
    before = pool.copy()
    w1 = ref.kv_refresh_paged(g, kv, dict(window=12, stride=4, step=1, ring_frames=16), masks[None], types[None],
                              [pool], w0["slot_new"], 32, [refr2], 32)
    sn = w1["slot_new"][0, :23].tolist()
    # survivors (frames 4..11, p_old 9..21) keep their slots 9..21; new tokens take free slots 0..7, prompt 8 and 22
    assert sn[:13] == list(range(9, 22))
    assert sn[13:21] == list(range(0, 8)) and sn[21:23] == [8, 22]
    # REUSE values untouched in place, REUSE keys rotated by dp = -9
    re = [p for p in range(23) if w1["disposition"][0, p] == 2]
    assert len(re) == 5
    for p in re:
        s = sn[p]
        assert (pool[:, 1, s] == before[:, 1, s]).all()
        for l in range(2):
            exp = ref.rope_rotate_f32(before[l, 0, s].reshape(-1), 2, 16, 1e4, -9)
            assert (pool[l, 0, s].reshape(-1) == exp).all()
    # non-REUSE rows: r-th refreshed row in p_new order
    nonre = [p for p in range(23) if w1["disposition"][0, p] != 2]
    for r, p in enumerate(nonre):
        assert (pool[:, :, sn[p]] == refr2[:, :, r]).all()
    c = w1["counters"]
    row = 2 * 16 * 4
    assert c[ref.C_BYTES_KV] == (5 * 2 * 1 + 18 * 2 * 2) * row * 2


@pytest.mark.parametrize("dtype", [1, 0])
@pytest.mark.parametrize("scene", ["multi_object", "scene_cut", "noise"])
def test_paged_equals_out_of_place_through_slot_map(ref, dtype, scene):
    """Drive both oracles through 12 windows of a C1 stream (w=8, s=2, GOP 4); after every window the paged pool,
    read through slot_new, equals the out-of-place cache bit for bit (K rotated, V reused, refreshed rows)."""
    cfg = synth.CONFIGS["C1"]
    g = make_grid(448, 448)
    w, s, ring = 8, 2, 10
    n_prompt = 5
    cap = w * 256 + n_prompt
    kv = _kv(cap=cap + 300, rcap=cap, n_prompt=n_prompt, dtype=dtype, H=2, D=16 if dtype == 1 else 32)
    kv_oop = dict(kv, capacity=cap)
    nf = 11 * s + w
    mb = synth.stream_metadata(448, 448, scene, 77, nf)
    types = synth.frame_types(nf, 4)
    sc = ref.score_patches(g, mb[None], types[None], np.zeros((1, 33), np.uint32), want_score=False)
    rng = np.random.default_rng(1)
    pool = _rand_cache(kv, rng, kv["capacity"])
    slot = None
    oop_old = None
    for k in range(12):
        mring = np.zeros((1, ring, 32), np.uint32)
        tring = np.zeros((1, ring), np.uint8)
        for f in range(max(0, (k - 1) * s), k * s + w):
            mring[0, f % ring] = sc["keep_mask"][0, f]
            tring[0, f % ring] = types[f]
        win = dict(window=w, stride=s, step=k, ring_frames=ring)
        refr = _rand_cache(kv, rng, cap)
        oop_new = np.zeros_like(_rand_cache(kv_oop, rng, cap))
        o = ref.kv_refresh(g, kv_oop, win, mring, tring, [oop_old] if k else None, [oop_new], [refr], cap)
        pg = ref.kv_refresh_paged(g, kv, win, mring, tring, [pool], slot, cap, [refr], cap)
        assert o["status"] == 0 and pg["status"] == 0
        assert (o["disposition"] == pg["disposition"]).all() and (o["p_old"] == pg["p_old"]).all()
        assert (o["n_tokens"] == pg["n_tokens"]).all()
        nt = int(o["n_tokens"][0, 0]) + n_prompt
        sn = pg["slot_new"][0, :nt]
        assert len(set(sn.tolist())) == nt and sn.min() >= 0 and sn.max() < kv["capacity"]   # injective
        assert (pool[:, :, sn] == oop_new[:, :, :nt]).all()
        slot = pg["slot_new"]
        oop_old = oop_new


def test_paged_origin_and_capacity(ref):
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    masks = _masks_from_groups(g, [[0, 1, 2, 3]] * 8)
    types = np.array([0, 1, 1, 1, 1, 1, 1, 1], np.uint8)
    kv = _kv(cap=20, rcap=20, n_prompt=1)
    rng = np.random.default_rng(2)
    pool = _rand_cache(kv, rng, 20)
    win = dict(window=4, stride=2, step=1, ring_frames=8)
    bad = np.full((1, 32), 99, np.int32)                  # slots outside the pool -> ORIGIN
    out = ref.kv_refresh_paged(g, kv, win, masks[None], types[None], [pool], bad, 32, None, 32)
    assert out["status"] & ref.ST_ORIGIN
    small = dict(kv, capacity=6)                          # not enough free slots for the new tokens -> CAPACITY
    pool2 = _rand_cache(small, rng, 6)
    ok = np.arange(32, dtype=np.int32)[None] % 6
    out = ref.kv_refresh_paged(g, small, win, masks[None], types[None], [pool2], ok, 32, None, 32)
    assert out["status"] & ref.ST_CAPACITY
