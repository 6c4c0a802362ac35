"""The K/V checker the GPU parity tests rely on (tests/kvcheck.py) must reject every corruption class it claims
to catch: a flipped bit in an untouched row, in a refreshed (ANCHOR / NEW / prompt) row, in a reused value, or in
the non-rotated columns of a reused key, and a rotated key beyond the north star's bound.  The "GPU" result here is
the oracle's own output, corrupted on purpose."""
import numpy as np
import pytest

import kvcheck
from synth import make_grid
from test_oracle_pins import _masks_from_groups

KEPT = [[0, 1, 2, 3], [1], [1, 3], [1, 3], [0, 1, 2, 3], [0], [0], [0, 2],
        [0, 1, 2, 3], [], [], [3], [0, 1, 2, 3], [2], [2], [2, 3]]


def _rand(kv, rng, rows):
    shape = (kv["layers"], 2, rows, kv["kv_heads"], kv["head_dim"])
    if kv["dtype"] == 1:
        return rng.standard_normal(shape).astype(np.float32)
    return rng.integers(0, 65536, size=shape, dtype=np.uint16) & np.uint16(0xBFFF)


def _flip(a, idx):
    b = a.copy()
    u = b.view(np.uint16 if b.dtype == np.uint16 else np.uint32)
    u[idx] ^= 1
    return b


@pytest.mark.parametrize("dtype", [1, 0])
def test_pool_checker_catches_corruption(ref, dtype):
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    masks = _masks_from_groups(g, KEPT)
    types = np.array([0 if f % 4 == 0 else 1 for f in range(16)], np.uint8)
    kv = dict(layers=2, kv_heads=2, head_dim=16, dtype=dtype, capacity=40, refresh_capacity=40, rope_base=1e4,
              n_prompt=2)
    rng = np.random.default_rng(0)
    pool = _rand(kv, rng, 40)
    w0 = ref.kv_refresh_paged(g, kv, dict(window=12, stride=4, step=0, ring_frames=16), masks[None], types[None],
                              [pool], None, 32, [_rand(kv, rng, 40)], 32)
    pre = pool.copy()
    refr = _rand(kv, rng, 40)
    w1 = ref.kv_refresh_paged(g, kv, dict(window=12, stride=4, step=1, ring_frames=16), masks[None], types[None],
                              [pool], w0["slot_new"], 32, [refr], 32)
    exp, d, sl, n = pool, w1["disposition"][0], w1["slot_new"][0], 23
    stats = {}
    kvcheck.check_pool_step(exp, pre, exp, d, sl, n, kv, refr=refr, stats=stats)
    assert stats["not_bit_exact"] == 0 and stats["rotated"] == 5 * 2 * 2 * 16
    re_slot = sl[np.flatnonzero(d[:n] == 2)[0]]
    an_slot = sl[np.flatnonzero(d[:n] == 1)[0]]
    new_slot = sl[np.flatnonzero(d[:n] == 0)[-1]]          # a prompt row
    free = np.setdiff1d(np.arange(40), sl[:n])[0]          # a row no token of window 1 holds
    bad = [(0, 1, re_slot, 0, 0),     # reused value
           (1, 0, an_slot, 1, 3),     # anchor key (refreshed row)
           (0, 1, new_slot, 0, 15),   # prompt value (refreshed row)
           (1, 0, free, 0, 0),        # untouched row
           (0, 1, free, 1, 7)]
    for idx in bad:
        with pytest.raises(AssertionError):
            kvcheck.check_pool_step(_flip(exp, idx), pre, exp, d, sl, n, kv, refr=refr)
    # a rotated key one ulp off: within the bound, but counted as not bit-exact
    st = {}
    kvcheck.check_pool_step(_flip(exp, (0, 0, re_slot, 0, 0)), pre, exp, d, sl, n, kv, refr=refr, stats=st)
    assert st["not_bit_exact"] == 1
    # ... and beyond the bound: rejected
    far = exp.copy()
    if dtype == 1:
        far[0, 0, re_slot, 0, 0] += 1.0
    else:
        far[0, 0, re_slot, 0, 0] ^= np.uint16(0x4000)
    with pytest.raises(AssertionError):
        kvcheck.check_pool_step(far, pre, exp, d, sl, n, kv, refr=refr)
    # M-RoPE: the non-rotated (h / w) columns of a reused key are bit-checked
    kvm = dict(kv, rope_mode=1, mrope_section=(2, 3, 3), t_per_frame=1)
    _, keep = kvcheck.rot_cols(kvm)
    with pytest.raises(AssertionError):
        kvcheck.check_pool_step(_flip(exp, (0, 0, re_slot, 0, int(keep[0]))), pre, exp, d, sl, n, kvm, refr=refr)


@pytest.mark.parametrize("dtype", [1, 0])
def test_copy_checker_catches_corruption(ref, dtype):
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    masks = _masks_from_groups(g, KEPT)
    types = np.array([0 if f % 4 == 0 else 1 for f in range(16)], np.uint8)
    kv = dict(layers=2, kv_heads=2, head_dim=16, dtype=dtype, capacity=32, refresh_capacity=32, rope_base=1e4,
              n_prompt=2)
    rng = np.random.default_rng(1)
    old, refr = _rand(kv, rng, 32), _rand(kv, rng, 32)
    new = _rand(kv, rng, 32)
    pre = new.copy()
    out = ref.kv_refresh(g, kv, dict(window=12, stride=4, step=1, ring_frames=16), masks[None], types[None],
                         [old], [new], [refr], 32)
    d, po, n = out["disposition"][0], out["p_old"][0], 23
    kvcheck.check_copy_step(new, pre, new, d, po, n, kv, old=old, refr=refr)
    re = int(np.flatnonzero(d[:n] == 2)[0])
    an = int(np.flatnonzero(d[:n] == 1)[0])
    for idx in [(0, 1, re, 0, 0), (1, 0, an, 0, 1), (0, 1, n + 2, 0, 0), (1, 0, 22, 1, 2)]:
        with pytest.raises(AssertionError):
            kvcheck.check_copy_step(_flip(new, idx), pre, new, d, po, n, kv, old=old, refr=refr)
