"""Pins of the C oracle against what the paper and the mathematics fix (no GPU).

Each test names the passage it checks (P:n = PAPER.md line, S:n = SPEC.md line).  The expected values come
from the paper / SPEC worked examples (tests/golden/), hand derivations written out in the test, closed forms
and textbook formulas computed independently here in float64 — never from the oracle itself.
"""
import math
import os

import numpy as np
import pytest

from synth import MB_DTYPE, make_grid

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if line:
                rows.append(line)
    return rows


def mb_grid(g, fill_type=1):
    rec = np.zeros((g["mb_rows"], g["mb_cols"]), MB_DTYPE)
    rec["type"] = fill_type
    return rec


# ---------------------------------------------------------------- Eq. 1 -----------------------------------
def test_eq1_spec_examples(ref):
    # SPEC S:63-65 in integer pel; the ABI takes quarter-pel, so x4 on input (reading Q2)
    for line in golden("spec_examples.txt"):
        if line.startswith("magnitude"):
            _, dx, dy, _, exp = line.split()
            assert ref.mb_magnitude(4 * int(dx), 4 * int(dy)) == np.float32(float(exp))


def test_eq1_quarter_pel_ties_and_intra(ref):
    assert ref.mb_magnitude(1, 0) == np.float32(0.25)          # exactly tau -> dynamic (Q1)
    assert ref.mb_magnitude(0, -1) == np.float32(0.25)
    # sqrt(2)/4 correctly rounded to fp32
    assert ref.mb_magnitude(1, 1) == np.float32(math.sqrt(2) / 4)
    assert ref.mb_magnitude(1, 1) == np.float32(0.35355338)
    assert ref.mb_magnitude(12, 16) == np.float32(5.0)
    assert np.isinf(ref.mb_magnitude(3, 4, 2))                 # INTRA -> +inf (Q9)
    assert np.isinf(ref.mb_magnitude(0, 0, 9))                 # unknown type -> treated as INTRA
    assert ref.mb_magnitude(3, 4, 1) == np.float32(1.25)       # SKIP uses its exported MV (Q9)
    # extreme vectors do not overflow: |(-32768, -32768)| / 4 = 8192 sqrt 2
    assert ref.mb_magnitude(-32768, -32768) == np.float32(math.sqrt(2.0 * 32768 ** 2)) * np.float32(0.25)
    # exhaustive small range against float64 sqrt rounded once to fp32 (sqrt is correctly rounded)
    for dx in range(-20, 21):
        for dy in range(-20, 21):
            s = np.float32(dx * dx + dy * dy)
            assert ref.mb_magnitude(dx, dy) == np.float32(np.sqrt(np.float64(s))).astype(np.float32) * np.float32(0.25)


# ---------------------------------------------------------------- resampling ---------------------
def test_resample_block_equals_patch_grid(ref):
    # S:225 / S:222: when block grid = patch grid, V(i) is the block's own magnitude
    g = make_grid(64, 64, mb_size=16, grid_w=4, grid_h=4, patch=16)
    rng = np.random.default_rng(0)
    rec = mb_grid(g)
    rec["mvx"] = rng.integers(-40, 40, size=(4, 4))
    rec["mvy"] = rng.integers(-40, 40, size=(4, 4))
    V, R, M, st = ref.patch_fields(g, rec)
    for j in range(4):
        for i in range(4):
            assert V[j, i] == ref.mb_magnitude(int(rec["mvx"][j, i]), int(rec["mvy"][j, i]))
    assert (R == 0).all() and (M == V).all() and st == 0


def test_resample_max_over_four_blocks(ref):
    # patch spanning 4 blocks with magnitudes {0,0,1,5} -> V = 5.  At C1 geometry (448 px, 16-px MBs,
    # 14-px patches) patch (1,1) = px [14,28)^2 overlaps MBs (0,0),(0,1),(1,0),(1,1).
    g = make_grid(448, 448)
    rec = mb_grid(g)
    rec["mvx"][1, 0] = 4          # 1 px
    rec["mvx"][1, 1] = 12         # (3,4) px * 4 -> 5 px
    rec["mvy"][1, 1] = 16
    V, _, _, _ = ref.patch_fields(g, rec)
    assert V[1, 1] == np.float32(5.0)
    assert V[0, 0] == np.float32(0.0)   # patch (0,0) = [0,14)^2 lies in MB (0,0) only (magnitude 0)
    assert V[1, 0] == np.float32(1.0)   # patch (1,0) = X [0,14) x Y [14,28) overlaps MBs (0,0) and (1,0)
    assert V[0, 1] == np.float32(0.0)   # patch (0,1) = X [14,28) x Y [0,14) overlaps MBs (0,0) and (0,1)
    assert V[2, 2] == np.float32(5.0)   # patch (2,2) = [28,42)^2 overlaps MB (1,1) ([16,32)^2)
    assert V[3, 3] == np.float32(0.0)   # patch (3,3) = [42,56)^2 overlaps MBs (2..3, 2..3) only


def test_resample_hand_computed_R(ref):
    # Hand derivation (SURVEY §8(c) "Resample R"): patch (0,1) = X [14,28) x Y [0,14) px overlaps MB (0,0) with
    # area 2x14 = 28 px^2 and MB (0,1) with area 12x14 = 168 px^2.  SAD 2560 and 10240 -> per-pixel means 10
    # and 40.  R = (28*10 + 168*40) / 196 / 255 = 7000 / 49980 = 50/357.
    g = make_grid(448, 448, alpha=0.5)
    rec = mb_grid(g)
    rec["sad"][0, 0], rec["sad"][0, 1] = 2560, 10240
    rec["mvx"][0, 0], rec["mvy"][0, 0] = 3, 4      # 1.25 px
    rec["mvx"][0, 1], rec["mvy"][0, 1] = 0, -2     # 0.5 px
    V, R, M, _ = ref.patch_fields(g, rec)
    assert R[0, 1] == np.float32(50 / 357)
    assert R[0, 1] == np.float32(0.14005603)
    assert V[0, 1] == np.float32(1.25)
    # Eq. 3 with one rounding: M = fl32(1.25 + 0.5 * R) computed exactly in float64 then rounded
    assert M[0, 1] == np.float32(1.25 + 0.5 * np.float64(R[0, 1]))
    assert M[0, 1] == np.float32(1.3200281)
    # patch (0,0) = [0,14)^2 lies entirely in MB (0,0): R = 10/255, V = 1.25
    assert R[0, 0] == np.float32(10 / 255) and V[0, 0] == np.float32(1.25)


def test_resample_R_closed_form_uniform(ref):
    # a uniform SAD field gives R = sad / (mb^2 * 255) in every patch, whatever the geometry (area-weighted mean)
    for (sw, sh) in [(1920, 1080), (448, 448), (100, 60)]:
        g = make_grid(sw, sh, grid_w=8, grid_h=8)
        rec = mb_grid(g)
        rec["sad"] = 5100
        _, R, _, _ = ref.patch_fields(g, rec)
        assert (R == np.float32(5100 / (256 * 255))).all()


def test_resample_coded_grid_last_row_1080p(ref):
    # Reading Q3: 1080 rows -> 68 coded MB rows; the last row covers display rows 1072..1087 and must
    # influence only the last patch row (display rows 1046.25..1080).
    g = make_grid(1920, 1080)
    assert g["mb_rows"] == 68 and g["mb_cols"] == 120
    rec = mb_grid(g)
    rec["mvx"][67, 0] = 40
    V, _, _, _ = ref.patch_fields(g, rec)
    assert V[31, 0] == np.float32(10.0)
    assert (V[:31, :] == 0).all() and (V[31, 1:] == 0).all()


# ---------------------------------------------------------------- Eq. 3 / Eq. 4 --------------------------
def test_eq3_eq4_spec_examples(ref):
    # block = patch geometry so a patch's R is its own block's mean |residual| / 255
    g = make_grid(64, 64, mb_size=16, grid_w=4, grid_h=4, patch=16, alpha=1.0, tau=0.25)
    rec = mb_grid(g)
    rec["sad"][0, 0] = 32640          # mean 127.5 -> R = 0.5
    rec["sad"][0, 1] = 19584          # mean 76.5  -> R = 0.3
    rec["sad"][0, 2] = 13056          # mean 51.0  -> R = 0.2
    V, R, M, _ = ref.patch_fields(g, rec)
    assert M[0, 0] == np.float32(0.5)                 # S:235 V=0, alpha=1, R=0.5 -> 0.5
    assert M[0, 1] == np.float32(0.3)                 # S:243 0.3 >= 0.25 -> dynamic
    assert M[0, 2] == np.float32(0.2)                 # S:245 0.2 -> static
    S, n = 1, 2
    mb = np.stack([rec, rec])[None]
    out = ref.score_patches(g, mb, np.array([[0, 1]], np.uint8), np.zeros((1, 1 + 1), np.uint32))
    keep_p = np.unpackbits(out["keep_mask"][0, 1].view(np.uint8), bitorder="little")[:16].reshape(4, 4)
    # dynamic: (0,0) 0.5, (0,1) 0.3; static (0,2) 0.2 -> groups of 2x2: group (0,0) kept, group (0,1) has
    # (0,2) static and (0,3),(1,2),(1,3) zero -> dropped
    assert keep_p[0, 0] and keep_p[0, 1] and not keep_p[0, 2]
    # alpha = 0 -> M == V bit-identically
    g0 = dict(g, alpha=0.0)
    V0, _, M0, _ = ref.patch_fields(g0, rec)
    assert (M0 == V0).all()


def test_eq4_tau_zero_keeps_everything_and_inclusive(ref):
    # S:244 / S:269: tau = 0 -> every patch dynamic every frame (full compute)
    g = make_grid(448, 448, tau=0.0)
    rng = np.random.default_rng(1)
    n = 5
    mb = np.zeros((1, n, g["mb_rows"], g["mb_cols"]), MB_DTYPE)
    mb["type"] = 1
    ft = np.array([[0, 1, 1, 1, 1]], np.uint8)
    out = ref.score_patches(g, mb, ft, np.zeros((1, 33), np.uint32))
    assert (out["kept_count"] == 1024).all()
    # tau = 0.25 with every MB at exactly 1 qpel (0.25 px) -> all dynamic (inclusive >=, reading Q1)
    g2 = make_grid(448, 448, tau=0.25)
    mb2 = mb.copy()
    mb2["mvx"] = rng.choice([-1, 1], size=mb2.shape)
    out2 = ref.score_patches(g2, mb2, ft, np.zeros((1, 33), np.uint32))
    assert (out2["kept_count"] == 1024).all()
    assert out2["counters"][ref.C_NEAR_TAU] == 4 * 1024      # every P-frame patch sits exactly on tau


def test_threshold_monotone_in_tau(ref):
    # tau1 <= tau2 => dynamic set under tau2 subset of tau1 (checked on the accumulated keep masks)
    from synth import stream_metadata, frame_types
    mb = stream_metadata(448, 448, "multi_object", 5, 12)[None]
    ft = frame_types(12, 4)[None]
    prev = None
    for tau in [0.0, 0.25, 1.0, 5.0, float("inf")]:
        g = make_grid(448, 448, tau=tau)
        km = ref.score_patches(g, mb, ft, np.zeros((1, 33), np.uint32))["keep_mask"]
        if prev is not None:
            assert ((km & ~prev) == 0).all()
        prev = km


# ---------------------------------------------------------------- GOP accumulation --------------
def _patch_mb_for(g, patches, mag_qpel=8):
    """MB records (block = patch geometry) with motion on the listed patch indices."""
    rec = mb_grid(g)
    for i in patches:
        rec["mvx"][i // g["grid_w"], i % g["grid_w"]] = mag_qpel
    return rec


def test_gop_union_reset_and_empty(ref):
    g = make_grid(128, 128, mb_size=16, grid_w=8, grid_h=8, patch=16, group=1)
    frames = [_patch_mb_for(g, []), _patch_mb_for(g, [5]), _patch_mb_for(g, [9]), _patch_mb_for(g, []),
              _patch_mb_for(g, []), _patch_mb_for(g, [20])]
    ft = np.array([[0, 1, 1, 1, 0, 1]], np.uint8)
    out = ref.score_patches(g, np.stack(frames)[None], ft, np.zeros((1, 3), np.uint32))
    bits = lambda f: set(np.flatnonzero(np.unpackbits(out["keep_mask"][0, f].view(np.uint8), bitorder="little")))
    assert bits(0) == set(range(64))          # I-frame fully encoded
    assert bits(1) == {5}
    assert bits(2) == {5, 9}                  # S:252 union
    assert bits(3) == {5, 9}                  # S:254 empty detections keep the state
    assert bits(4) == set(range(64))          # I resets and outputs everything
    assert bits(5) == {20}                    # state restarted from empty after the I-frame (Q7)
    # final GOP state = {20} with the init flag
    st = out  # gop_state was updated in place in the array passed; recompute with an explicit array
    gs = np.zeros((1, 3), np.uint32)
    ref.score_patches(g, np.stack(frames)[None], ft, gs)
    assert gs[0, 0] == (1 << 20) and gs[0, 1] == 0 and gs[0, 2] == 1


def test_gop_state_carries_across_calls(ref):
    # splitting a stream into calls of n frames gives the same masks as one call (state in/out)
    from synth import stream_metadata, frame_types
    g = make_grid(448, 448)
    mb = stream_metadata(448, 448, "multi_object", 11, 16)
    ft = frame_types(16, 4)
    one = ref.score_patches(g, mb[None], ft[None], np.zeros((1, 33), np.uint32))
    gs = np.zeros((1, 33), np.uint32)
    parts = []
    for a in range(0, 16, 2):
        parts.append(ref.score_patches(g, mb[None, a:a + 2], ft[None, a:a + 2], gs)["keep_mask"][0])
    assert (np.concatenate(parts) == one["keep_mask"][0]).all()


def test_no_iframe_status(ref):
    g = make_grid(448, 448)
    mb = np.zeros((1, 2, 28, 28), MB_DTYPE)
    mb["type"] = 1
    out = ref.score_patches(g, mb, np.array([[1, 1]], np.uint8), np.zeros((1, 33), np.uint32))
    assert out["status"] & ref.ST_NO_IFRAME
    assert (out["kept_count"] == 0).all()
    out = ref.score_patches(g, mb, np.array([[3, 1]], np.uint8), np.zeros((1, 33), np.uint32))
    assert out["status"] & ref.ST_BAD_FRAME_TYPE and out["kept_count"][0, 0] == 1024


# ---------------------------------------------------------------- group-complete ----------------
def test_group_complete_spec_example(ref):
    # 8x8 grid, 2x2 groups, only patch (3,3) active -> the group covering rows 2-3, cols 2-3 is kept
    g = make_grid(128, 128, mb_size=16, grid_w=8, grid_h=8, patch=16, group=2)
    frames = [_patch_mb_for(g, []), _patch_mb_for(g, [3 * 8 + 3])]
    out = ref.score_patches(g, np.stack(frames)[None], np.array([[0, 1]], np.uint8), np.zeros((1, 3), np.uint32))
    bits = set(np.flatnonzero(np.unpackbits(out["keep_mask"][0, 1].view(np.uint8), bitorder="little")))
    assert bits == {2 * 8 + 2, 2 * 8 + 3, 3 * 8 + 2, 3 * 8 + 3}
    assert out["kept_count"][0, 1] == 4        # 1 group kept, 15 dropped
    assert out["kept_count"][0, 0] == 64        # S:262 all active -> all kept (I-frame)


def test_full_motion_frame_and_static_video(ref):
    # north star: a full-motion frame keeps every patch; S:270 / S:490: static video keeps only I-frames
    g = make_grid(1920, 1080)
    mb = np.zeros((1, 16, 68, 120), MB_DTYPE)
    mb["type"] = 1
    mb["mvx"][0, 5] = 1            # 0.25 px everywhere in frame 5 -> full motion
    ft = np.zeros((1, 16), np.uint8) + 1
    ft[0, 0] = 0
    out = ref.score_patches(g, mb, ft, np.zeros((1, 33), np.uint32))
    kc = out["kept_count"][0]
    assert kc[0] == 1024 and (kc[1:5] == 0).all() and (kc[5:] == 1024).all()
    c = out["counters"]
    assert c[ref.C_PATCHES] == 16 * 1024 and c[ref.C_KEPT] == kc.sum()   # kept + pruned = total
    # tau = inf: only I-frames (and INTRA MBs) survive
    g_inf = make_grid(1920, 1080, tau=float("inf"))
    out = ref.score_patches(g_inf, mb, ft, np.zeros((1, 33), np.uint32))
    assert list(out["kept_count"][0]) == [1024] + [0] * 15


# ---------------------------------------------------------------- compaction -----------------------------
def _frames(g, n, seed):
    rng = np.random.default_rng(seed)
    H, W = g["grid_h"] * g["patch"], g["grid_w"] * g["patch"]
    return [rng.integers(0, 65536, size=(3, H, W), dtype=np.uint16) for _ in range(n)]


def test_compact_round_trip_and_order(ref):
    from synth import stream_metadata, frame_types
    g = make_grid(448, 448)
    S, n = 2, 6
    mb = np.stack([stream_metadata(448, 448, sc, 3 + s, n) for s, sc in enumerate(["multi_object", "noise"])])
    ft = np.stack([frame_types(n, 4, 1), frame_types(n, 4, 1)])
    sc = ref.score_patches(g, mb, ft, np.zeros((S, 33), np.uint32))
    frames = _frames(g, S * n, 7)
    fidx = np.arange(S * n, dtype=np.int32) % n + 1
    cap = int(sc["kept_count"].sum())
    out = ref.compact(g, sc["keep_mask"], fidx, frames, cap, S, n)
    offs = out["frame_offsets"]
    assert offs[-1] == cap and (np.diff(offs) == sc["kept_count"].reshape(-1)).all()
    # order preserved: (slot, group row-major, patch in group) strictly increasing (reading Q14)
    si = out["src_index"].astype(np.int64)
    slot, rem = si // 1024, si % 1024
    h, w = rem // 32, rem % 32
    key = (((slot * 16 + h // 2) * 16 + w // 2) * 2 + h % 2) * 2 + w % 2
    assert (np.diff(key) > 0).all()
    # every emitted patch equals its source patch, pos ids match, group-major order within the frame
    p = 14
    for r in range(cap):
        slot, rem = divmod(int(out["src_index"][r]), 1024)
        h, w = divmod(rem, 32)
        assert tuple(out["pos_ids"][r]) == (fidx[slot], h, w)
        src = frames[slot][:, h * p:(h + 1) * p, w * p:(w + 1) * p].reshape(-1)
        assert (out["packed"][r] == src).all()
    # round trip: scattering packed back by src_index reproduces the kept patches and only those
    recon = [np.zeros_like(f) for f in frames]
    for r in range(cap):
        slot, rem = divmod(int(out["src_index"][r]), 1024)
        h, w = divmod(rem, 32)
        recon[slot][:, h * p:(h + 1) * p, w * p:(w + 1) * p] = out["packed"][r].reshape(3, p, p)
    for slot in range(S * n):
        keep = np.unpackbits(sc["keep_mask"].reshape(S * n, 32)[slot].view(np.uint8), bitorder="little").reshape(32, 32)
        m = np.kron(keep, np.ones((p, p), np.uint8)).astype(bool)
        assert (recon[slot][:, m] == frames[slot][:, m]).all()
        assert (recon[slot][:, ~m] == 0).all()
    # group-major order: rows 4q..4q+3 are the (dy,dx) = (0,0),(0,1),(1,0),(1,1) patches of one group
    for q in range(cap // 4):
        hw = [divmod(int(out["src_index"][4 * q + d]) % 1024, 32) for d in range(4)]
        (h0, w0) = hw[0]
        assert h0 % 2 == 0 and w0 % 2 == 0 and hw == [(h0, w0), (h0, w0 + 1), (h0 + 1, w0), (h0 + 1, w0 + 1)]


def to_grouped(frame, g):
    """planar [3][gh*p][gw*p] -> grouped [groups][dy][dx][3][p][p] by a numpy permutation (independent of the
    oracle's index arithmetic)."""
    p, G = g["patch"], g["group"]
    ngr, ngc = g["grid_h"] // G, g["grid_w"] // G
    x = frame.reshape(3, ngr, G, p, ngc, G, p)            # c, gr, dy, y, gc, dx, x
    return np.ascontiguousarray(x.transpose(1, 4, 2, 5, 0, 3, 6)).reshape(-1)


@pytest.mark.parametrize("geom", [(448, 448, 14, 2, 32), (64, 48, 4, 2, 8), (30, 30, 5, 3, 6), (56, 56, 14, 1, 4)])
def test_compact_grouped_layout_equals_planar(ref, geom):
    sw, sh, p, G, gw = geom
    g = make_grid(sw, sh, patch=p, group=G, grid_w=gw, grid_h=gw)
    rng = np.random.default_rng(4)
    nw = (gw * gw + 31) // 32
    km = rng.integers(0, 2**32, size=(2, 3, nw), dtype=np.uint64).astype(np.uint32)
    frames = [rng.integers(0, 65536, size=(3, gw * p, gw * p), dtype=np.uint16) for _ in range(6)]
    a = ref.compact(g, km, np.arange(6, dtype=np.int32), frames, 6 * gw * gw, 2, 3)
    b = ref.compact(g, km, np.arange(6, dtype=np.int32), [to_grouped(f, g) for f in frames], 6 * gw * gw, 2, 3,
                    frame_layout=1)
    for key in ("packed", "pos_ids", "src_index", "frame_offsets"):
        assert (a[key] == b[key]).all(), key


def test_compact_capacity_and_non_group_complete(ref):
    g = make_grid(128, 128, mb_size=16, grid_w=8, grid_h=8, patch=4, group=2)
    km = np.zeros((1, 1, 2), np.uint32)
    km[0, 0, 0] = 1 << 9          # patch (1,1) only: not group-complete -> its group (0,0) is emitted whole
    frames = _frames(g, 1, 1)
    out = ref.compact(g, km, np.array([0], np.int32), frames, 16, 1, 1)
    assert out["frame_offsets"].tolist() == [0, 4]
    assert out["src_index"][:4].tolist() == [0, 1, 8, 9]
    out = ref.compact(g, km, np.array([0], np.int32), frames, 2, 1, 1)
    assert out["status"] & ref.ST_CAPACITY and out["frame_offsets"].tolist() == [0, 4]
    assert out["src_index"].tolist() == [0, 1]
    # empty input
    out = ref.compact(g, np.zeros((0, 1, 2), np.uint32), np.zeros(0, np.int32), [], 0, 0, 1)
    assert out["rc"] == 0 and out["frame_offsets"].tolist() == [0]


# ---------------------------------------------------------------- KV plan --------------------
def _masks_from_groups(g, groups_per_frame):
    """keep masks (group-complete) from lists of kept group ids (row-major over the group grid)."""
    G = g["group"]
    gw = g["grid_w"] // G
    nw = (g["grid_w"] * g["grid_h"] + 31) // 32
    out = np.zeros((len(groups_per_frame), nw), np.uint32)
    for f, gl in enumerate(groups_per_frame):
        bits = np.zeros(nw * 32, np.uint8)
        for q in gl:
            gr, gc = divmod(q, gw)
            for dy in range(G):
                for dx in range(G):
                    bits[(gr * G + dy) * g["grid_w"] + gc * G + dx] = 1
        out[f] = np.packbits(bits, bitorder="little").view(np.uint32)
    return out


def _toy_kv(cap, rcap, n_prompt=0, dtype=1, L=2, H=2, D=16, base=1e4):
    return dict(layers=L, kv_heads=H, head_dim=D, dtype=dtype, capacity=cap, refresh_capacity=rcap,
                rope_base=base, n_prompt=n_prompt)


def _cache(kv, rng, cap=None):
    shape = (kv["layers"], 2, cap or kv["capacity"], kv["kv_heads"], kv["head_dim"])
    if kv["dtype"] == 1:
        return rng.standard_normal(shape).astype(np.float32)
    return rng.integers(0, 65536, size=shape, dtype=np.uint16) & np.uint16(0xBFFF)   # finite bf16 bits


def test_plan_paper_fig8_example(ref):
    rows = golden("fig_selective_kvc_refresh.txt")
    kvs = dict(r.split() for r in rows if len(r.split()) == 2)
    gop, w, s, k = int(kvs["gop"]), int(kvs["window"]), int(kvs["stride"]), int(kvs["step"])
    g = make_grid(448, 448)
    ring = w + s
    masks = np.full((ring, 32), 0xFFFFFFFF, np.uint32)    # no pruning
    types = np.array([0 if f % gop == 0 else 1 for f in range(ring)], np.uint8)
    kv = _toy_kv(cap=w * 256 + 8, rcap=w * 256 + 8, n_prompt=0)
    rng = np.random.default_rng(0)
    old, new = _cache(kv, rng), np.zeros_like(_cache(kv, rng))
    out = ref.kv_refresh(g, kv, dict(window=w, stride=s, step=k, ring_frames=ring), masks[None], types[None],
                         [old], [new], None, w * 256)
    names = {0: "NEW", 1: "ANCHOR", 2: "REUSE"}
    disp = out["disposition"][0]
    for r in rows:
        parts = r.split()
        if parts[0].startswith("F") and len(parts) == 2:
            f1 = int(parts[0][1:])               # 1-indexed frame of the figure
            f0 = f1 - 1
            q = (f0 - k * s) * 256               # first token of that frame in the new window
            assert {names[int(x)] for x in disp[q:q + 256]} == {parts[1]}, r
    nv, nr, na, nn = out["n_tokens"][0]
    assert nv == 12 * 256 and na == 2 * 256 and nr == 6 * 256 and nn == 4 * 256
    frac = float(kvs["overlap_fraction"])
    assert round((nr + na) / nv, 2) == frac       # P:344 "waste 67% of the FLOPs"
    # p_old = p_new + 4*256 for every overlap token (window slides by 4 unpruned frames)
    ov = np.arange(8 * 256)
    assert (out["p_old"][0, ov] == ov + 4 * 256).all() and (out["p_old"][0, 8 * 256:] == -1).all()


def test_plan_paper_window_80_16(ref):
    # P:115-116 + P:123 + P:269: w=80, s=16, 256 tokens/frame, 20,480 tokens per window, window 1 = [16, 96)
    nums = {r.split()[0]: r.split()[1:] for r in golden("paper_numbers.txt")}
    w, s = 80, 16
    g = make_grid(448, 448)
    ring = w + s
    masks = np.full((ring, 32), 0xFFFFFFFF, np.uint32)
    types = np.array([0 if f % 16 == 0 else 1 for f in range(ring)], np.uint8)
    kv = _toy_kv(cap=20480 + 32, rcap=20480 + 32, n_prompt=32, L=1, H=1, D=2)
    rng = np.random.default_rng(0)
    old, new = _cache(kv, rng), _cache(kv, rng)
    out = ref.kv_refresh(g, kv, dict(window=w, stride=s, step=1, ring_frames=ring), masks[None], types[None],
                         [old], [new], None, 20480 + 32)
    nv, nr, na, nn = out["n_tokens"][0]
    assert nv == int(nums["tokens_per_window_80"][0]) == 80 * int(nums["tokens_per_frame_448"][0])
    lo, hi = map(int, nums["window_k1_w80_s16"])
    assert (lo, hi) == (1 * s, 1 * s + w)
    # NEW frames [80, 96): 16 x 256 + 32 prompt; anchors: I-frames 16, 32, 48, 64 (16 is also the first frame)
    assert nn == 16 * 256 + 32 and na == 4 * 256 and nr == 60 * 256
    assert w / s == float(nums["window_80_stride_16_redundancy"][0])


def test_plan_hand_example_with_pruning(ref):
    # Hand derivation (SURVEY §8(c) "Plan, hand-computed with pruning"): 4x4 patches (2x2 groups), GOP 4,
    # w = 12, s = 4, window 0 = [0,12) -> window 1 = [4,16).
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    kept = [[0, 1, 2, 3], [1], [1, 3], [1, 3], [0, 1, 2, 3], [0], [0], [0, 2],
            [0, 1, 2, 3], [], [], [3], [0, 1, 2, 3], [2], [2], [2, 3]]
    masks = _masks_from_groups(g, kept)
    types = np.array([0 if f % 4 == 0 else 1 for f in range(16)], np.uint8)
    kv = _toy_kv(cap=32, rcap=32, n_prompt=2)
    rng = np.random.default_rng(3)
    old, new, refr = _cache(kv, rng), np.zeros_like(_cache(kv, rng)), _cache(kv, rng)
    out = ref.kv_refresh(g, kv, dict(window=12, stride=4, step=1, ring_frames=16), masks[None], types[None],
                         [old], [new], [refr], 32)
    nv, nr, na, nn = out["n_tokens"][0]
    assert (nv, nr, na, nn) == (21, 5, 8, 8 + 2)
    A, R, N = 1, 2, 0
    exp_disp = [A] * 4 + [R, R, R, R] + [A] * 4 + [R] + [N] * 8 + [N, N]
    exp_pold = [9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21] + [-1] * 10
    assert out["disposition"][0, :23].tolist() == exp_disp
    assert out["p_old"][0, :23].tolist() == exp_pold
    # REUSE rows: V bit-copied, K rotated by dp = -9; refreshed rows r = 0.. in p_new order
    reuse = [p for p in range(23) if exp_disp[p] == R]
    for p in reuse:
        po = exp_pold[p]
        assert (new[:, 1, p] == old[:, 1, po]).all()                     # P:361 value reuse
        for l in range(2):
            exp = ref.rope_rotate_f32(old[l, 0, po].reshape(-1), 2, 16, 1e4, p - po)
            assert (new[l, 0, p].reshape(-1) == exp).all()
    nonreuse = [p for p in range(23) if exp_disp[p] != R]
    for r, p in enumerate(nonreuse):
        assert (new[:, :, p] == refr[:, :, r]).all()
    c = out["counters"]
    assert c[ref.C_TOK_REUSE] == 5 and c[ref.C_TOK_ANCHOR] == 8 and c[ref.C_TOK_NEW] == 10
    assert c[ref.C_BYTES_KV] == 23 * 2 * 2 * (2 * 16 * 4) * 2


def test_plan_degenerate_cases(ref):
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    rng = np.random.default_rng(5)
    kept = [list(rng.choice(4, size=rng.integers(0, 5), replace=False)) for _ in range(16)]
    masks = _masks_from_groups(g, kept)
    types = np.array([0 if f % 4 == 0 else 1 for f in range(16)], np.uint8)
    kv = _toy_kv(cap=64, rcap=64, n_prompt=3)
    old = _cache(kv, rng)
    # s = w -> every token NEW
    out = ref.kv_refresh(g, kv, dict(window=4, stride=4, step=2, ring_frames=16), masks[None], types[None],
                         [old], [np.zeros_like(old)], None, 64)
    assert out["n_tokens"][0, 1] == 0 and out["n_tokens"][0, 2] == 0
    # k = 0 -> everything NEW, old cache never read
    out = ref.kv_refresh(g, kv, dict(window=6, stride=2, step=0, ring_frames=8), masks[None, :8], types[None, :8],
                         None, [np.zeros_like(old)], None, 64)
    assert (out["disposition"][0, :out["n_tokens"][0, 0] + 3] == 0).all()
    # zero-slide: dropped frames carry no tokens -> dp = 0 for every REUSE token -> K rows bit-identical (R(0)=I)
    kept2 = [[0, 1], [], [1], [1, 2], [], [], [2], [3]]
    masks2 = _masks_from_groups(g, kept2)
    types2 = np.array([0, 1, 1, 1, 1, 1, 1, 1], np.uint8)
    new = np.zeros_like(old)
    # window 1 = [1, 5): dropped frame 0 has 2 tokens -> use step 2 with s=1 : dropped frame 1 has none
    out = ref.kv_refresh(g, kv, dict(window=4, stride=1, step=2, ring_frames=8), masks2[None], types2[None],
                         [old], [new], None, 64)
    d, po = out["disposition"][0], out["p_old"][0]
    reuse = [p for p in range(out["n_tokens"][0, 0]) if d[p] == 2]
    assert reuse and all(po[p] == p for p in reuse)
    for p in reuse:
        assert (new[:, :, p] == old[:, :, p]).all()


def test_all_static_window_refreshes_nothing(ref):
    # north star: an all-static window (no I-frame inside, static P-frames) refreshes nothing
    g = make_grid(448, 448)
    n = 24
    mb = np.zeros((1, n, 28, 28), MB_DTYPE)
    mb["type"] = 1
    ft = np.ones((1, n), np.uint8)
    ft[0, 0] = 0                      # GOP longer than the stream: only frame 0 is an I-frame
    sc = ref.score_patches(g, mb, ft, np.zeros((1, 33), np.uint32))
    kv = _toy_kv(cap=4096, rcap=4096, n_prompt=4)
    rng = np.random.default_rng(0)
    old = _cache(kv, rng)
    out = ref.kv_refresh(g, kv, dict(window=8, stride=4, step=3, ring_frames=n), sc["keep_mask"], ft,
                         [old], [np.zeros_like(old)], None, 4096)
    nv, nr, na, nn = out["n_tokens"][0]
    assert nv == 0 and na == 0 and nr == 0 and nn == 4      # only the prompt is (re)computed


# ---------------------------------------------------------------- RoPE (Eq. 5) ---------------------------
def _rope_textbook(x, dp, base):
    """rotate_half RoPE in float64 (x*cos + rotate_half(x)*sin), independent of the oracle."""
    H, D = x.shape
    half = D // 2
    inv = base ** (-np.arange(half, dtype=np.float64) * 2.0 / D)
    ang = dp * inv
    cos = np.concatenate([np.cos(ang), np.cos(ang)])
    sin = np.concatenate([np.sin(ang), np.sin(ang)])
    x = x.astype(np.float64)
    rot_half = np.concatenate([-x[:, half:], x[:, :half]], axis=1)
    return x * cos + rot_half * sin


def test_rope_identity_inverse_norm_textbook(ref):
    rng = np.random.default_rng(2)
    H, D = 4, 128
    for base in (1e4, 1e6):
        k = rng.standard_normal(H * D).astype(np.float32)
        assert (ref.rope_rotate_f32(k, H, D, base, 0) == k).all()                      # S:378 R(0) = I bit-exact
        back = ref.rope_rotate_f32(ref.rope_rotate_f32(k, H, D, base, 3), H, D, base, -3)
        assert np.abs(back - k).max() <= 1e-6 * max(1.0, np.abs(k).max())
        for dp in (-16384, -4097, -9, 1, 777):
            r = ref.rope_rotate_f32(k, H, D, base, dp)
            exp = _rope_textbook(k.reshape(H, D), dp, base).reshape(-1)
            assert np.abs(r - exp).max() <= 2e-6                                       # textbook formula
            n0 = np.linalg.norm(k.reshape(H, D, ).astype(np.float64), axis=1)
            n1 = np.linalg.norm(r.reshape(H, D).astype(np.float64), axis=1)
            assert np.abs(n1 - n0).max() <= 1e-5 * n0.max()                             # S:420 norm preserved
        # composition: R(a) R(b) ~ R(a+b), layer-1 exactness rot(RoPE(k,p_old),dp) ~ RoPE(k,p_new)
        a, b = 1234, -987
        ab = ref.rope_rotate_f32(ref.rope_rotate_f32(k, H, D, base, a), H, D, base, b)
        assert np.abs(ab - ref.rope_rotate_f32(k, H, D, base, a + b)).max() <= 1e-5


def test_kv_bf16_rotation_vs_textbook(ref):
    # bf16 Qwen-shaped rows: REUSE K within 1e-2 of the fp64 textbook rotation of the stored key (north star)
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    kept = [[0, 1, 2, 3]] * 8
    masks = _masks_from_groups(g, kept)
    types = np.array([0, 1, 1, 1, 1, 1, 1, 1], np.uint8)
    kv = dict(layers=2, kv_heads=4, head_dim=128, dtype=0, capacity=32, refresh_capacity=32, rope_base=1e6,
              n_prompt=0)
    rng = np.random.default_rng(9)
    x = rng.standard_normal((2, 2, 32, 4, 128)).astype(np.float32)
    old = (x.view(np.uint32) >> 16).astype(np.uint16)
    new = np.zeros_like(old)
    out = ref.kv_refresh(g, kv, dict(window=4, stride=2, step=1, ring_frames=8), masks[None], types[None],
                         [old], [new], None, 32)
    d, po = out["disposition"][0], out["p_old"][0]
    as_f = lambda u: (u.astype(np.uint32) << 16).view(np.float32)
    cnt = 0
    for p in range(16):
        if d[p] != 2:
            continue
        cnt += 1
        for l in range(2):
            exp = _rope_textbook(as_f(old[l, 0, po[p]]), p - po[p], 1e6)
            assert np.abs(as_f(new[l, 0, p]) - exp).max() <= 1e-2
            assert (new[l, 1, p] == old[l, 1, po[p]]).all()
    assert cnt == 4   # window [2,6) after [0,4): f2 ANCHOR (first overlap frame), f3 REUSE (4), f4-f5 NEW


def test_bf16_rne_store(ref):
    """The bf16 store of a rotated key rounds to nearest, ties to EVEN (reading Q20).  Keys are chosen
    (tests/rne_ties.py) so that the fp32 result of Eq. 5 is exactly a bf16 tie, with both parities of the upper
    half; the expected bits come from PyTorch's own fp32 -> bf16 conversion, not from the oracle."""
    import rne_ties
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    masks = _masks_from_groups(g, [[0], [1], [0, 1], [2], [0], [0, 1, 2, 3], [1], [2]])
    types = np.ones(8, np.uint8)
    types[0] = 0
    D, base = 128, 1e4
    kv = dict(layers=1, kv_heads=1, head_dim=D, dtype=0, capacity=16, refresh_capacity=16, rope_base=base,
              n_prompt=0)
    # window k=2 ([4,8) after [2,6)): dropped frames 2, 3 carry 3 tokens -> dp = -3; f4 ANCHOR (first overlap
    # frame), f5's 4 tokens REUSE from p_old 4..7 to p_new 1..4
    rows, ties = rne_ties.tie_rows(4, D, base, -3)
    rng = np.random.default_rng(1)
    old = rng.integers(0, 65536, size=(1, 2, 16, 1, D), dtype=np.uint16) & np.uint16(0xBFFF)
    old[0, 0, 4:8, 0] = rows
    new = np.zeros_like(old)
    out = ref.kv_refresh(g, kv, dict(window=4, stride=2, step=2, ring_frames=8), masks[None], types[None],
                         [old], [new], None, 16)
    assert out["rc"] == 0 and out["status"] == 0
    assert list(out["disposition"][0, :6]) == [1, 2, 2, 2, 2, 0]
    assert list(out["p_old"][0, 1:5]) == [4, 5, 6, 7]
    n_even = n_odd = 0
    for j in range(4):
        idx = np.array([e for e, _ in ties[j]])
        o = np.array([v for _, v in ties[j]], np.float32)
        exp = rne_ties.rne_bf16(o)
        up = (o.view(np.uint32) >> 16).astype(np.uint16)
        assert ((exp == up) | (exp == up + 1)).all()               # a tie rounds to one of its neighbours
        assert (new[0, 0, 1 + j, 0, idx] == exp).all(), j          # ... the even one
        assert (new[0, 1, 1 + j] == old[0, 1, 4 + j]).all()        # V reused bit for bit
        n_even += int((up % 2 == 0).sum())
        n_odd += int((up % 2 == 1).sum())
    assert n_even >= 20 and n_odd >= 20, (n_even, n_odd)        # both directions of the tie rule exercised