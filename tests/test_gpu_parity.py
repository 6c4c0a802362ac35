"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element, on seeded inputs.

Bar (north star): masks, kept counts, compacted rows, position ids, source indices, offsets, dispositions, p_old
and token counts bit-exact; fp32 scores bit-exact (<= 1e-5 relative required); pure K/V copies bit-exact;
rotated K within 1e-2 abs (bf16) / 1e-5 (fp32), with the count of non-bit-exact elements reported.
"""
import numpy as np
import pytest
import torch

import synth
from synth import MB_DTYPE, make_grid

import kvcheck

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module")
def abi():
    import __graft_entry__ as ge
    ge.build_cuda()
    from paper_2604_06036_b200 import _abi
    _abi.lib()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return _abi


def d_mb(mb):
    return torch.from_numpy(np.ascontiguousarray(mb, dtype=MB_DTYPE).view(np.uint8)).to(DEV)


def u32(t):
    return t.cpu().numpy().view(np.uint32)


# ------------------------------------------------------------------------------------------------------------
# score_patches
# ------------------------------------------------------------------------------------------------------------
def run_score_both(abi, ref, g, mb, types, gop_h=None, frame_stride=None, want_score=True):
    """mb [S][n][rows][cols], types [S][frame_stride] -> (gpu dict, oracle dict)."""
    S, n = mb.shape[:2]
    nw = abi.grid_words(g)
    fs = n if frame_stride is None else frame_stride
    gop_h = np.zeros((S, nw + 1), np.uint32) if gop_h is None else gop_h
    gs_d = torch.from_numpy(gop_h.view(np.int32).copy()).to(DEV)
    km_d = torch.zeros(S, fs, nw, dtype=torch.int32, device=DEV)
    sc_d = torch.zeros(S, n, g["grid_w"] * g["grid_h"], dtype=torch.float32, device=DEV) if want_score else None
    kc_d = torch.zeros(S, n, dtype=torch.int32, device=DEV)
    cnt_d = torch.zeros(16, dtype=torch.int64, device=DEV)
    st_d = torch.zeros(1, dtype=torch.int32, device=DEV)
    ty_d = torch.from_numpy(np.ascontiguousarray(types, dtype=np.uint8)).to(DEV)
    abi.codecsight_score_patches(g, S, n, d_mb(mb), ty_d, km_d, fs, gs_d, sc_d, kc_d, cnt_d, st_d)
    o = ref.score_patches(g, mb, types, gop_h, frame_stride=fs, want_score=want_score)
    torch.cuda.synchronize()
    gpu = dict(keep_mask=u32(km_d), kept_count=kc_d.cpu().numpy(), score=None if sc_d is None else sc_d.cpu().numpy(),
               gop_state=u32(gs_d), counters=cnt_d.cpu().numpy().view(np.uint64), status=int(st_d.item()))
    o["gop_state"] = gop_h
    return gpu, o


def assert_score_equal(gpu, o, n, fs):
    assert gpu["status"] == o["status"]
    assert (gpu["keep_mask"][:, :n] == o["keep_mask"][:, :n]).all()
    assert (gpu["kept_count"] == o["kept_count"]).all()
    assert (gpu["gop_state"] == o["gop_state"]).all()
    assert (gpu["counters"] == o["counters"]).all(), (gpu["counters"], o["counters"])
    if o["score"] is not None:
        a, b = gpu["score"], o["score"]
        # scores: bit-exact expected (same IEEE operations); the gate is 1e-5 relative
        with np.errstate(invalid="ignore"):
            assert ((a == b) | (np.abs(a - b) <= 1e-5 * np.abs(b))).all()
        assert (a.view(np.uint32) == b.view(np.uint32)).all(), int((a.view(np.uint32) != b.view(np.uint32)).sum())


@pytest.mark.parametrize("scene", ["static", "translating_object", "multi_object", "noise", "scene_cut"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_score_c1_whole_stream(abi, ref, scene, seed):
    """C1: 448x448, 64 frames, GOP 4, first window of 8 then strides of 2 (state carried across calls)."""
    cfg = synth.CONFIGS["C1"]
    g = make_grid(448, 448)
    nf = cfg["frames"]
    mb = synth.stream_metadata(448, 448, scene, synth.stream_seed(cfg, seed), nf)
    types = synth.frame_types(nf, cfg["gop"])
    nw = abi.grid_words(g)
    gop_h = np.zeros((1, nw + 1), np.uint32)
    f0 = 0
    while f0 < nf:
        n = cfg["window"] if f0 == 0 else cfg["stride"]
        gpu, o = run_score_both(abi, ref, g, mb[None, f0:f0 + n], types[None, f0:f0 + n], gop_h.copy())
        assert_score_equal(gpu, o, n, n)
        gop_h = o["gop_state"]
        f0 += n


@pytest.mark.parametrize("geom", [(448, 448, 16, 32, 32, 2), (1920, 1080, 16, 32, 32, 2),
                                  (3840, 2160, 16, 32, 32, 2), (40, 36, 8, 4, 4, 2), (100, 44, 16, 8, 8, 4),
                                  (30, 30, 8, 6, 6, 3), (56, 56, 16, 4, 4, 1), (72, 40, 8, 12, 10, 2),
                                  (1000, 700, 16, 40, 30, 2), (4000, 300, 16, 64, 8, 2)])
@pytest.mark.parametrize("alpha,tau", [(0.0, 0.25), (0.5, 0.25), (1.0, 0.0), (5.0, 1.0), (0.25, 5.0),
                                       (0.0, float("inf"))])
def test_score_random_geometries(abi, ref, geom, alpha, tau):
    """Odd MB columns (non-bulk path), groups 1/2/3/4, partial last bitmap word, extreme MVs and bad types."""
    sw, sh, m, gw, gh, G = geom
    g = make_grid(sw, sh, tau=tau, alpha=alpha, mb_size=m, grid_w=gw, grid_h=gh, group=G, patch=4)
    rng = np.random.default_rng(abs(hash((geom, alpha, tau))) % 2**32)
    S, n = 3, 5
    mb = np.stack([np.stack([synth.random_mb(g["mb_rows"], g["mb_cols"], rng, p_intra=0.02, mv_max=3,
                                             p_bad_type=0.001) for _ in range(n)]) for _ in range(S)])
    mb["mvx"][0, 1, 0, 0] = -32768
    mb["mvy"][0, 1, 0, 0] = -32768
    types = np.array([[0, 1, 1, 1, 0], [1, 1, 0, 1, 1], [0, 1, 3, 1, 1]], np.uint8)  # NO_IFRAME, bad type
    gpu, o = run_score_both(abi, ref, g, mb, types)
    assert_score_equal(gpu, o, n, n)


def test_score_ring_stride_and_no_score(abi, ref):
    """keep_mask / frame_type addressed through frame_stride (ring slots), score output skipped."""
    g = make_grid(1920, 1080)
    S, n, fs = 4, 4, 20
    mb = np.stack([synth.stream_metadata(1920, 1080, "medium", 5 + s, n) for s in range(S)])
    types = np.zeros((S, fs), np.uint8)
    types[:, :n] = synth.frame_types(n, 16, 13)
    gpu, o = run_score_both(abi, ref, g, mb, types, frame_stride=fs, want_score=False)
    assert_score_equal(gpu, o, n, fs)
    assert (gpu["keep_mask"][:, n:] == 0).all()       # untouched slots


@pytest.mark.parametrize("cfg_name", ["C2", "C4", "C5"])
def test_score_full_size_batches(abi, ref, cfg_name):
    """BASELINE shapes: C2 32 streams x 4 frames 1080p; C4 mixed (sampled 16 streams); C5 4K traffic (8 streams,
    8 frames).  Launch configuration identical to the bench (one cluster per stream)."""
    cfg = synth.CONFIGS[cfg_name]
    sw, sh = cfg["src"]
    g = make_grid(sw, sh)
    S = {"C2": 32, "C4": 16, "C5": 8}[cfg_name]
    n = cfg["stride"]
    first = 3 * cfg["gop"] + 1
    mb = np.stack([synth.stream_metadata(sw, sh, synth.scene_of(cfg, s), synth.stream_seed(cfg, s), n)
                   for s in range(S)])
    types = np.stack([synth.frame_types(n, cfg["gop"], first) for _ in range(S)])
    nw = abi.grid_words(g)
    rng = np.random.default_rng(1)
    gop_h = np.zeros((S, nw + 1), np.uint32)
    gop_h[:, :nw] = rng.integers(0, 2**32, size=(S, nw), dtype=np.uint64).astype(np.uint32) & np.uint32(0x01010101)
    gop_h[:, nw] = 1
    gpu, o = run_score_both(abi, ref, g, mb, types, gop_h)
    assert_score_equal(gpu, o, n, n)


# ------------------------------------------------------------------------------------------------------------
# compact
# ------------------------------------------------------------------------------------------------------------
def to_grouped(frame, g):
    p, G = g["patch"], g["group"]
    ngr, ngc = g["grid_h"] // G, g["grid_w"] // G
    x = frame.reshape(3, ngr, G, p, ngc, G, p)
    return np.ascontiguousarray(x.transpose(1, 4, 2, 5, 0, 3, 6)).reshape(-1)


def run_compact_both(abi, ref, g, keep_mask, frame_index, frames, capacity, S, n, mfs, layout=0):
    nw = abi.grid_words(g)
    p = g["patch"]
    if layout == 1:
        frames = [to_grouped(f, g) for f in frames]
    km_d = torch.from_numpy(np.ascontiguousarray(keep_mask).view(np.int32)).to(DEV)
    fr_d = [torch.from_numpy(f.view(np.int16)).to(DEV) for f in frames]
    fptr = abi.ptr_array(fr_d, DEV) if fr_d else torch.zeros(1, dtype=torch.int64, device=DEV)
    fi_d = torch.from_numpy(np.ascontiguousarray(frame_index, dtype=np.int32)).to(DEV)
    cap = max(capacity, 1)
    packed = torch.full((cap, 3 * p * p), -1, dtype=torch.int16, device=DEV)
    pos = torch.full((cap, 3), -7, dtype=torch.int32, device=DEV)
    src = torch.full((cap,), -7, dtype=torch.int32, device=DEV)
    offs = torch.zeros(S * n + 1, dtype=torch.int32, device=DEV)
    cnt_d = torch.zeros(16, dtype=torch.int64, device=DEV)
    st_d = torch.zeros(1, dtype=torch.int32, device=DEV)
    abi.codecsight_compact(g, S, n, km_d, mfs, fi_d, fptr, capacity, packed, pos, src, offs, cnt_d, st_d,
                           frame_layout=layout)
    o = ref.compact(g, keep_mask, frame_index, frames, capacity, S, n, mask_frame_stride=mfs, frame_layout=layout)
    torch.cuda.synchronize()
    rows = min(int(o["frame_offsets"][-1]), capacity)
    assert int(st_d.item()) == o["status"]
    assert (offs.cpu().numpy() == o["frame_offsets"]).all()
    assert (packed.cpu().numpy().view(np.uint16)[:rows] == o["packed"][:rows]).all()
    assert (pos.cpu().numpy()[:rows] == o["pos_ids"][:rows]).all()
    assert (src.cpu().numpy()[:rows] == o["src_index"][:rows]).all()
    assert (cnt_d.cpu().numpy().view(np.uint64) == o["counters"]).all()
    if rows < cap:   # nothing written past the emitted rows
        assert (src.cpu().numpy()[rows:] == -7).all()
    return o


def scored_masks(ref, g, cfg, S, n, first):
    sw, sh = g["src_w"], g["src_h"]
    mb = np.stack([synth.stream_metadata(sw, sh, synth.scene_of(cfg, s), synth.stream_seed(cfg, s, 3), n)
                   for s in range(S)])
    types = np.stack([synth.frame_types(n, cfg["gop"], first) for _ in range(S)])
    nw = (g["grid_w"] * g["grid_h"] + 31) // 32
    gs = np.zeros((S, nw + 1), np.uint32)
    gs[:, nw] = 1
    return ref.score_patches(g, mb, types, gs, want_score=False)["keep_mask"]


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("cfg_name,S,n", [("C1", 1, 8), ("C1", 5, 2), ("C2", 32, 4), ("C4", 8, 4)])
def test_compact_configs(abi, ref, cfg_name, S, n, layout):
    cfg = synth.CONFIGS[cfg_name]
    g = make_grid(*cfg["src"])
    km = scored_masks(ref, g, cfg, S, n, first=1)
    rng = np.random.default_rng(11)
    frames = synth.random_frames(S * n, 448, 448, rng)
    fidx = np.tile(np.arange(100, 100 + n, dtype=np.int32), S)
    run_compact_both(abi, ref, g, km, fidx, frames, S * n * 1024, S, n, n, layout)


@pytest.mark.parametrize("layout", [0, 1])
def test_compact_edge_cases(abi, ref, layout):
    g = make_grid(448, 448)
    rng = np.random.default_rng(3)
    S, n = 3, 3
    km = rng.integers(0, 2**32, size=(S, n, 32), dtype=np.uint64).astype(np.uint32)  # not group-complete
    km[1] = 0                                   # an empty stream
    km[2, 1] = 0xFFFFFFFF                       # a full frame
    frames = synth.random_frames(S * n, 448, 448, rng)
    fidx = np.arange(S * n, dtype=np.int32)
    o = run_compact_both(abi, ref, g, km, fidx, frames, S * n * 1024, S, n, n, layout)
    total = int(o["frame_offsets"][-1])
    # capacity overflow in the middle of a group, and exactly at a group boundary
    run_compact_both(abi, ref, g, km, fidx, frames, total // 2 + 1, S, n, n, layout)
    run_compact_both(abi, ref, g, km, fidx, frames, (total // 8) * 4, S, n, n, layout)
    run_compact_both(abi, ref, g, km, fidx, frames, 0, S, n, n, layout)
    # mask stride (ring) addressing
    ring = np.zeros((S, 7, 32), np.uint32)
    ring[:, 2:2 + n] = km
    run_compact_both(abi, ref, g, ring[:, 2:].copy(), fidx, frames, S * n * 1024, S, n, 5, layout)
    # empty batch
    run_compact_both(abi, ref, g, np.zeros((0, n, 32), np.uint32), np.zeros(0, np.int32), [], 16, 0, n, n, layout)


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("geom", [(64, 48, 16, 8, 6, 2, 4), (30, 30, 8, 6, 6, 3, 6), (56, 56, 16, 4, 4, 1, 14),
                                  (100, 44, 16, 8, 8, 4, 8), (72, 40, 8, 12, 10, 2, 3)])
def test_compact_generic_geometries(abi, ref, geom, layout):
    """Generic (runtime patch/group) path, odd patch size (scalar loads), group 1/3/4."""
    sw, sh, m, gw, gh, G, p = geom
    g = make_grid(sw, sh, mb_size=m, grid_w=gw, grid_h=gh, group=G, patch=p)
    rng = np.random.default_rng(5)
    S, n = 2, 3
    nw = abi.grid_words(g)
    km = rng.integers(0, 2**32, size=(S, n, nw), dtype=np.uint64).astype(np.uint32)
    km &= rng.integers(0, 2**32, size=(S, n, nw), dtype=np.uint64).astype(np.uint32)
    frames = [rng.integers(0, 65536, size=(3, gh * p, gw * p), dtype=np.uint16) for _ in range(S * n)]
    fidx = np.arange(S * n, dtype=np.int32)
    run_compact_both(abi, ref, g, km, fidx, frames, S * n * gw * gh, S, n, n, layout)


# ------------------------------------------------------------------------------------------------------------
# score_compact (NEXT-2: scoring + compaction fused, decoupled look-back)
# ------------------------------------------------------------------------------------------------------------
def run_score_compact_both(abi, ref, g, mb, types, frames, capacity, layout=0, gop_h=None, frame_stride=None,
                           want_score=True, ws=None, check=True):
    S, n = mb.shape[:2]
    nw = abi.grid_words(g)
    p = g["patch"]
    fs = n if frame_stride is None else frame_stride
    gop_h = np.zeros((S, nw + 1), np.uint32) if gop_h is None else gop_h
    gs_d = torch.from_numpy(gop_h.view(np.int32).copy()).to(DEV)
    km_d = torch.zeros(S, fs, nw, dtype=torch.int32, device=DEV)
    sc_d = torch.zeros(S, n, g["grid_w"] * g["grid_h"], dtype=torch.float32, device=DEV) if want_score else None
    kc_d = torch.zeros(S, n, dtype=torch.int32, device=DEV)
    cnt_d = torch.zeros(16, dtype=torch.int64, device=DEV)
    st_d = torch.zeros(1, dtype=torch.int32, device=DEV)
    ty_d = torch.from_numpy(np.ascontiguousarray(types, dtype=np.uint8)).to(DEV)
    fr_h = [to_grouped(f, g) for f in frames] if layout == 1 else frames
    fr_d = [torch.from_numpy(f.view(np.int16)).to(DEV) for f in fr_h]
    fptr = abi.ptr_array(fr_d, DEV)
    fidx = np.tile(np.arange(7, 7 + n, dtype=np.int32), S)
    fi_d = torch.from_numpy(fidx).to(DEV)
    cap = max(capacity, 1)
    packed = torch.full((cap, 3 * p * p), -1, dtype=torch.int16, device=DEV)
    pos = torch.full((cap, 3), -7, dtype=torch.int32, device=DEV)
    src = torch.full((cap,), -7, dtype=torch.int32, device=DEV)
    offs = torch.full((S * n + 1,), -5, dtype=torch.int32, device=DEV)
    if ws is None:
        ws = torch.zeros(abi.score_compact_workspace_size(S), dtype=torch.uint8, device=DEV)
    abi.codecsight_score_compact(g, S, n, d_mb(mb), ty_d, km_d, fs, gs_d, sc_d, kc_d, fi_d, fptr, capacity, packed,
                                 pos, src, offs, ws, cnt_d, st_d, frame_layout=layout)
    so = ref.score_patches(g, mb, types, gop_h, frame_stride=fs, want_score=want_score)
    co = ref.compact(g, so["keep_mask"], fidx, fr_h, capacity, S, n, mask_frame_stride=fs, frame_layout=layout,
                     counters=so["counters"].copy())
    torch.cuda.synchronize()
    gpu = dict(keep_mask=u32(km_d), kept_count=kc_d.cpu().numpy(), score=None if sc_d is None else sc_d.cpu().numpy(),
               gop_state=u32(gs_d), counters=cnt_d.cpu().numpy().view(np.uint64), status=int(st_d.item()))
    so["gop_state"] = gop_h
    so["counters"] = co["counters"]
    so["status"] = so["status"] | co["status"]
    assert_score_equal(gpu, so, n, fs)
    rows = min(int(co["frame_offsets"][-1]), capacity)
    assert (offs.cpu().numpy() == co["frame_offsets"]).all()
    assert (packed.cpu().numpy().view(np.uint16)[:rows] == co["packed"][:rows]).all()
    assert (pos.cpu().numpy()[:rows] == co["pos_ids"][:rows]).all()
    assert (src.cpu().numpy()[:rows] == co["src_index"][:rows]).all()
    if rows < cap:
        assert (src.cpu().numpy()[rows:] == -7).all()
    assert (ws.cpu().numpy() == 0).all()            # the call leaves its workspace zeroed
    return co


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("cfg_name,S,n", [("C1", 3, 8), ("C2", 32, 4), ("C4", 16, 4), ("C4", 3, 16), ("C1", 2, 20)])
def test_score_compact_configs(abi, ref, cfg_name, S, n, layout):
    cfg = synth.CONFIGS[cfg_name]
    sw, sh = cfg["src"]
    g = make_grid(sw, sh)
    mb = np.stack([synth.stream_metadata(sw, sh, synth.scene_of(cfg, s), synth.stream_seed(cfg, s, 5), n)
                   for s in range(S)])
    types = np.stack([synth.frame_types(n, cfg["gop"], 3) for _ in range(S)])
    rng = np.random.default_rng(21)
    base = synth.random_frames(8, 448, 448, rng)
    frames = [base[i % 8] for i in range(S * n)]
    co = run_score_compact_both(abi, ref, g, mb, types, frames, S * n * 1024, layout)
    total = int(co["frame_offsets"][-1])
    # capacity truncation mid-group, want_score off, ring stride
    run_score_compact_both(abi, ref, g, mb, types, frames, total // 2 + 1, layout, want_score=False)
    ty_r = np.zeros((S, n + 3), np.uint8)
    ty_r[:, :n] = types
    run_score_compact_both(abi, ref, g, mb, ty_r, frames, total, layout, frame_stride=n + 3)


@pytest.mark.parametrize("geom", [(64, 48, 16, 8, 6, 2, 4), (30, 30, 8, 6, 6, 3, 6), (100, 44, 16, 8, 8, 4, 8),
                                  (72, 40, 8, 12, 10, 2, 3)])
def test_score_compact_generic(abi, ref, geom):
    sw, sh, m, gw, gh, G, p = geom
    g = make_grid(sw, sh, mb_size=m, grid_w=gw, grid_h=gh, group=G, patch=p)
    rng = np.random.default_rng(23)
    S, n = 5, 3
    mb = np.stack([np.stack([synth.random_mb(g["mb_rows"], g["mb_cols"], rng) for _ in range(n)])
                   for _ in range(S)])
    types = rng.integers(0, 2, size=(S, n)).astype(np.uint8)
    frames = [rng.integers(0, 65536, size=(3, gh * p, gw * p), dtype=np.uint16) for _ in range(S * n)]
    for layout in (0, 1):
        run_score_compact_both(abi, ref, g, mb, types, frames, S * n * gw * gh, layout)


def test_score_compact_many_streams_workspace_reuse(abi, ref):
    """300 streams (several waves of clusters, long look-back chains), the same workspace over 3 calls with the
    GOP state carried."""
    cfg = synth.CONFIGS["C4"]
    g = make_grid(1920, 1080)
    S, n = 300, 2
    nw = 32
    ws = torch.zeros(abi.score_compact_workspace_size(S), dtype=torch.uint8, device=DEV)
    gens = [synth.StreamGen(1920, 1080, synth.scene_of(cfg, i), synth.stream_seed(cfg, i)) for i in range(S)]
    rng = np.random.default_rng(4)
    base = synth.random_frames(4, 448, 448, rng)
    frames = [base[i % 4] for i in range(S * n)]
    gop_h = np.zeros((S, nw + 1), np.uint32)
    for call in range(3):
        mb = np.stack([np.stack([gn.next_frame() for _ in range(n)]) for gn in gens])
        types = np.stack([synth.frame_types(n, 16, call * n)] * S)
        # gop_h is uploaded, then advanced in place by the oracle: the state carries into the next call
        run_score_compact_both(abi, ref, g, mb, types, frames, S * n * 1024, 1, gop_h=gop_h, want_score=False, ws=ws)


# ------------------------------------------------------------------------------------------------------------
# compact_tp (NEXT-3 temporal patches)
# ------------------------------------------------------------------------------------------------------------
def run_compact_tp_both(abi, ref, g, tp, keep_mask, unit_index, frames, capacity, S, nu, mfs, layout=0,
                        want_unit_mask=True):
    nw = abi.grid_words(g)
    p = g["patch"]
    if layout == 1:
        frames = [to_grouped(f, g) for f in frames]
    km_d = torch.from_numpy(np.ascontiguousarray(keep_mask).view(np.int32)).to(DEV)
    fr_d = [torch.from_numpy(f.view(np.int16)).to(DEV) for f in frames]
    fptr = abi.ptr_array(fr_d, DEV) if fr_d else torch.zeros(1, dtype=torch.int64, device=DEV)
    ui_d = torch.from_numpy(np.ascontiguousarray(unit_index, dtype=np.int32)).to(DEV)
    cap = max(capacity, 1)
    packed = torch.full((cap, 3 * tp * p * p), -1, dtype=torch.int16, device=DEV)
    pos = torch.full((cap, 3), -7, dtype=torch.int32, device=DEV)
    src = torch.full((cap,), -7, dtype=torch.int32, device=DEV)
    offs = torch.zeros(S * nu + 1, dtype=torch.int32, device=DEV)
    um = torch.full((max(S, 1), nu, nw), -1, dtype=torch.int32, device=DEV) if want_unit_mask else None
    ft = np.random.default_rng(S + nu).integers(0, 3, size=(S, mfs)).astype(np.uint8) if want_unit_mask else None
    ft_d = torch.from_numpy(ft).to(DEV) if ft is not None else None
    ut = torch.full((max(S, 1), nu), 9, dtype=torch.uint8, device=DEV) if want_unit_mask else None
    cnt_d = torch.zeros(16, dtype=torch.int64, device=DEV)
    st_d = torch.zeros(1, dtype=torch.int32, device=DEV)
    abi.codecsight_compact_tp(g, tp, S, nu, km_d, mfs, ui_d, fptr, capacity, packed, pos, src, offs, cnt_d, st_d,
                              frame_layout=layout, unit_mask=um, unit_mask_stride=nu, frame_type=ft_d, unit_type=ut)
    o = ref.compact_tp(g, tp, keep_mask, unit_index, frames, capacity, S, nu, mask_frame_stride=mfs,
                       frame_layout=layout, want_unit_mask=want_unit_mask, frame_type=ft)
    torch.cuda.synchronize()
    rows = min(int(o["frame_offsets"][-1]), capacity)
    assert int(st_d.item()) == o["status"]
    assert (offs.cpu().numpy() == o["frame_offsets"]).all()
    assert (packed.cpu().numpy().view(np.uint16)[:rows] == o["packed"][:rows]).all()
    assert (pos.cpu().numpy()[:rows] == o["pos_ids"][:rows]).all()
    assert (src.cpu().numpy()[:rows] == o["src_index"][:rows]).all()
    assert (cnt_d.cpu().numpy().view(np.uint64) == o["counters"]).all()
    if want_unit_mask and S > 0:
        assert (um.cpu().numpy().view(np.uint32) == o["unit_mask"]).all()
        assert (ut.cpu().numpy() == o["unit_type"]).all()
    if rows < cap:
        assert (src.cpu().numpy()[rows:] == -7).all()
    return o


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("cfg_name,S,nu", [("C1", 2, 4), ("C4", 8, 2)])
def test_compact_tp2_configs(abi, ref, cfg_name, S, nu, layout):
    cfg = synth.CONFIGS[cfg_name]
    g = make_grid(*cfg["src"])
    km = scored_masks(ref, g, cfg, S, 2 * nu, first=1)
    rng = np.random.default_rng(12)
    frames = synth.random_frames(S * 2 * nu, 448, 448, rng)
    ui = np.tile(np.arange(50, 50 + nu, dtype=np.int32), S)
    o = run_compact_tp_both(abi, ref, g, 2, km, ui, frames, S * nu * 1024, S, nu, 2 * nu, layout)
    total = int(o["frame_offsets"][-1])
    run_compact_tp_both(abi, ref, g, 2, km, ui, frames, total // 2 + 1, S, nu, 2 * nu, layout)
    run_compact_tp_both(abi, ref, g, 2, km, ui, frames, 0, S, nu, 2 * nu, layout, want_unit_mask=False)


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("tp", [1, 2, 3])
@pytest.mark.parametrize("geom", [(64, 48, 16, 8, 6, 2, 4), (30, 30, 8, 6, 6, 3, 6), (56, 56, 16, 4, 4, 1, 14),
                                  (72, 40, 8, 12, 10, 2, 3)])
def test_compact_tp_generic(abi, ref, geom, tp, layout):
    sw, sh, m, gw, gh, G, p = geom
    g = make_grid(sw, sh, mb_size=m, grid_w=gw, grid_h=gh, group=G, patch=p)
    rng = np.random.default_rng(15 + tp)
    S, nu = 2, 2
    nw = abi.grid_words(g)
    mfs = nu * tp + 1
    km = rng.integers(0, 2**32, size=(S, mfs, nw), dtype=np.uint64).astype(np.uint32)
    km &= rng.integers(0, 2**32, size=(S, mfs, nw), dtype=np.uint64).astype(np.uint32)
    km &= rng.integers(0, 2**32, size=(S, mfs, nw), dtype=np.uint64).astype(np.uint32)
    frames = [rng.integers(0, 65536, size=(3, gh * p, gw * p), dtype=np.uint16) for _ in range(S * nu * tp)]
    ui = np.arange(S * nu, dtype=np.int32)
    run_compact_tp_both(abi, ref, g, tp, km, ui, frames, S * nu * gw * gh, S, nu, mfs, layout)


# ------------------------------------------------------------------------------------------------------------
# kv_refresh
# ------------------------------------------------------------------------------------------------------------
def _host_cache(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def run_kv_both(abi, ref, g, kv, win, mring, tring, old_d, new_d, ref_d, token_cap, sample=None):
    """Run GPU + oracle for one window step.  Returns (gpu dict, oracle dict, new_host_ref)."""
    S = mring.shape[0]
    dev = DEV
    old_h = [_host_cache(t) for t in old_d] if old_d is not None else None
    new_h = [_host_cache(t).copy() for t in new_d]
    pre_h = [t.copy() for t in new_h]
    ref_h = [_host_cache(t) for t in ref_d] if ref_d is not None else None
    m_d = torch.from_numpy(np.ascontiguousarray(mring).view(np.int32)).to(dev)
    t_d = torch.from_numpy(np.ascontiguousarray(tring)).to(dev)
    disp = torch.full((S, token_cap), 9, dtype=torch.uint8, device=dev)
    pold = torch.full((S, token_cap), -9, dtype=torch.int32, device=dev)
    ntok = torch.zeros(S, 4, dtype=torch.int32, device=dev)
    ws = torch.empty(abi.kv_workspace_size(kv, win, S), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(16, dtype=torch.int64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    abi.codecsight_kv_refresh(g, kv, win, S, m_d, t_d, abi.ptr_array(old_d, dev) if old_d is not None else None,
                              abi.ptr_array(new_d, dev), abi.ptr_array(ref_d, dev) if ref_d is not None else None,
                              token_cap, disp, pold, ntok, ws, cnt, st)
    o = ref.kv_refresh(g, kv, win, mring, tring, old_h, new_h, ref_h, token_cap)
    torch.cuda.synchronize()
    # the plan of every token (index outputs truncated at token_cap still have their rows written): per stream, the
    # oracle re-run with index outputs large enough for all tokens
    full = []
    for si in range(S):
        n_all = int(o["n_tokens"][si, 0]) + kv["n_prompt"]
        if n_all <= token_cap:
            full.append((o["disposition"][si], o["p_old"][si], n_all))
        else:
            f = ref.kv_refresh(g, kv, win, mring[si:si + 1], tring[si:si + 1],
                               [old_h[si]] if old_h is not None else None, [pre_h[si].copy()], None, n_all)
            full.append((f["disposition"][0], f["p_old"][0], n_all))
    gpu = dict(disposition=disp.cpu().numpy(), p_old=pold.cpu().numpy(), n_tokens=ntok.cpu().numpy(),
               counters=cnt.cpu().numpy().view(np.uint64), status=int(st.item()),
               pre=pre_h, old=old_h, refr=ref_h, full=full)
    return gpu, o, new_h


def _rot_cols(kv):
    return kvcheck.rot_cols(kv)


def assert_kv_equal(gpu, o, new_d, new_h, kv, stats=None):
    """Copy-mode step: indices bit-exact; cache rows split by kvcheck.check_copy_step (pure copies bit-exact,
    rotated keys within the bound, untouched rows unchanged)."""
    assert gpu["status"] == o["status"]
    assert (gpu["n_tokens"] == o["n_tokens"]).all()
    assert (gpu["counters"] == o["counters"]).all(), (gpu["counters"], o["counters"])
    S = len(new_d)
    tc = gpu["disposition"].shape[1]
    for s in range(S):
        nt = min(int(o["n_tokens"][s, 0]) + kv["n_prompt"], tc)
        assert (gpu["disposition"][s, :nt] == o["disposition"][s, :nt]).all()
        assert (gpu["p_old"][s, :nt] == o["p_old"][s, :nt]).all()
        assert (gpu["disposition"][s, nt:] == 9).all()        # nothing written past the tokens
        fd, fp, n_all = gpu["full"][s]
        kvcheck.check_copy_step(_host_cache(new_d[s]), gpu["pre"][s], new_h[s], fd, fp,
                                n_all, kv, old=gpu["old"][s] if gpu["old"] is not None else None,
                                refr=gpu["refr"][s] if gpu["refr"] is not None else None, stats=stats,
                                tag=f"stream {s}")


def stream_rings(ref, g, cfg, S, ring, k, w, s, scene_seed=0):
    """Score the frames of windows k-1 and k of S streams with the oracle and lay the masks out in rings."""
    sw, sh = g["src_w"], g["src_h"]
    nf = k * s + w
    nw = (g["grid_w"] * g["grid_h"] + 31) // 32
    mring = np.zeros((S, ring, nw), np.uint32)
    tring = np.zeros((S, ring), np.uint8)
    for si in range(S):
        mb = synth.stream_metadata(sw, sh, synth.scene_of(cfg, si), synth.stream_seed(cfg, si, scene_seed), nf)
        types = synth.frame_types(nf, cfg["gop"])
        out = ref.score_patches(g, mb[None], types[None], np.zeros((1, nw + 1), np.uint32), want_score=False)
        for f in range(max(0, (k - 1) * s), nf):
            mring[si, f % ring] = out["keep_mask"][0, f]
            tring[si, f % ring] = types[f]
    return mring, tring


def make_caches(kv, S, gen, with_refresh=True):
    dt = torch.bfloat16 if kv["dtype"] == 0 else torch.float32
    shape = (kv["layers"], 2, kv["capacity"], kv["kv_heads"], kv["head_dim"])
    rshape = (kv["layers"], 2, kv["refresh_capacity"], kv["kv_heads"], kv["head_dim"])
    old = [torch.randn(shape, generator=gen, device=DEV).to(dt) for _ in range(S)]
    new = [torch.full(shape, 7.0, device=DEV).to(dt) for _ in range(S)]
    refr = [torch.randn(rshape, generator=gen, device=DEV).to(dt) for _ in range(S)] if with_refresh else None
    return old, new, refr


@pytest.mark.parametrize("dtype", [1, 0])
def test_kv_c1_all_windows(abi, ref, dtype):
    """C1: 1 stream per scene kind, w=8, s=2, GOP 4, every window k = 0..28; toy fp32 and Qwen-shaped bf16."""
    cfg = synth.CONFIGS["C1"]
    g = make_grid(448, 448)
    w, s = cfg["window"], cfg["stride"]
    ring = w + s
    base = synth.TOY_KV if dtype == 1 else synth.QWEN_KV
    kv = dict(base, capacity=w * 256 + 32, refresh_capacity=w * 256 + 32, n_prompt=32)
    if dtype == 0:
        kv["layers"] = 2  # keep the oracle fast; the row shape (4 x 128 bf16) is the production one
    S = 5
    gen = torch.Generator(device=DEV)
    gen.manual_seed(0)
    stats = {}
    steps = range(0, 29) if dtype == 1 else [0, 1, 2, 3, 7, 28]
    for k in steps:
        mring, tring = stream_rings(ref, g, cfg, S, ring, k, w, s)
        old, new, refr = make_caches(kv, S, gen)
        gpu, o, new_h = run_kv_both(abi, ref, g, kv, dict(window=w, stride=s, step=k, ring_frames=ring), mring,
                                    tring, old if k else None, new, refr, kv["capacity"])
        assert_kv_equal(gpu, o, new, new_h, kv, stats)
    kvcheck.assert_rotation_bits(stats)


def test_kv_c3_sampled_streams(abi, ref):
    """C3 shape: 1080p masks, w=32, s=4, GOP 16, Qwen2-VL-7B bf16 (28 layers); 4 streams, a mid-stream window."""
    cfg = synth.CONFIGS["C3"]
    g = make_grid(1920, 1080)
    w, s, ring = 32, 4, 36
    kv = dict(synth.QWEN_KV, capacity=w * 256 + 32, refresh_capacity=10 * 256 + 32, n_prompt=32)
    S, k = 4, 9
    mring, tring = stream_rings(ref, g, cfg, S, ring, k, w, s)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(1)
    old, new, refr = make_caches(kv, S, gen)
    stats = {}
    gpu, o, new_h = run_kv_both(abi, ref, g, kv, dict(window=w, stride=s, step=k, ring_frames=ring), mring, tring,
                                old, new, refr, kv["capacity"])
    assert_kv_equal(gpu, o, new, new_h, kv, stats)
    kvcheck.assert_rotation_bits(stats)


def test_kv_edge_cases(abi, ref):
    g = make_grid(448, 448)
    cfg = synth.CONFIGS["C1"]
    w, s = 8, 2
    ring = w + s
    S = 5
    gen = torch.Generator(device=DEV)
    gen.manual_seed(3)
    mring, tring = stream_rings(ref, g, cfg, S, ring, 5, w, s)
    win = dict(window=w, stride=s, step=5, ring_frames=ring)
    # refreshed = NULL: non-REUSE rows untouched
    kv = dict(synth.TOY_KV, capacity=w * 256 + 32, refresh_capacity=w * 256 + 32, n_prompt=32)
    old, new, _ = make_caches(kv, S, gen, with_refresh=False)
    gpu, o, new_h = run_kv_both(abi, ref, g, kv, win, mring, tring, old, new, None, kv["capacity"])
    assert_kv_equal(gpu, o, new, new_h, kv)
    # small capacities: cache, refresh buffer and index outputs all overflow (CAPACITY / ORIGIN status)
    for cap, rcap, tc in [(300, 100, 250), (700, 5000, 2100), (64, 64, 64), (1, 0, 1)]:
        kv2 = dict(kv, capacity=cap, refresh_capacity=rcap)
        old, new, refr = make_caches(kv2, S, gen)
        gpu, o, new_h = run_kv_both(abi, ref, g, kv2, win, mring, tring, old, new, refr, tc)
        assert_kv_equal(gpu, o, new, new_h, kv2)
    # s = w: everything NEW
    mring2, tring2 = stream_rings(ref, g, cfg, S, 16, 3, 8, 8)
    old, new, refr = make_caches(kv, S, gen)
    gpu, o, new_h = run_kv_both(abi, ref, g, kv, dict(window=8, stride=8, step=3, ring_frames=16), mring2, tring2,
                                old, new, refr, kv["capacity"])
    assert_kv_equal(gpu, o, new, new_h, kv)
    assert (gpu["n_tokens"][:, 1] == 0).all() and (gpu["n_tokens"][:, 2] == 0).all()
    # odd-sized toy rows (scalar paths): D = 2, H = 1, fp32 and bf16
    for dt in (1, 0):
        kv3 = dict(layers=3, kv_heads=1, head_dim=2, dtype=dt, capacity=w * 256 + 4, refresh_capacity=w * 256 + 4,
                   rope_base=1e4, n_prompt=4)
        old, new, refr = make_caches(kv3, S, gen)
        gpu, o, new_h = run_kv_both(abi, ref, g, kv3, win, mring, tring, old, new, refr, kv3["capacity"])
        assert_kv_equal(gpu, o, new, new_h, kv3)
    # bf16 with head_dim 8 (half < 8: scalar rotation, 16-B copies)
    kv4 = dict(layers=2, kv_heads=2, head_dim=8, dtype=0, capacity=w * 256 + 4, refresh_capacity=w * 256 + 4,
               rope_base=1e6, n_prompt=4)
    old, new, refr = make_caches(kv4, S, gen)
    gpu, o, new_h = run_kv_both(abi, ref, g, kv4, win, mring, tring, old, new, refr, kv4["capacity"])
    assert_kv_equal(gpu, o, new, new_h, kv4)


def test_kv_zero_slide_bit_exact(abi, ref):
    """dp = 0 (dropped frames carry no tokens): REUSE keys must come back bit-identical (R(0) = I)."""
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    nw = 1
    mring = np.zeros((1, 8, nw), np.uint32)
    groups = [[0, 1], [], [1], [1, 2], [], [], [2], [3]]
    for f, gl in enumerate(groups):
        bits = 0
        for q in gl:
            gr, gc = divmod(q, 2)
            for dy in range(2):
                for dx in range(2):
                    bits |= 1 << ((gr * 2 + dy) * 4 + gc * 2 + dx)
        mring[0, f, 0] = bits
    tring = np.array([[0, 1, 1, 1, 1, 1, 1, 1]], np.uint8)
    kv = dict(layers=2, kv_heads=4, head_dim=128, dtype=0, capacity=64, refresh_capacity=64, rope_base=1e6,
              n_prompt=3)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(9)
    old, new, refr = make_caches(kv, 1, gen)
    gpu, o, new_h = run_kv_both(abi, ref, g, kv, dict(window=4, stride=1, step=2, ring_frames=8), mring, tring, old,
                                new, refr, 64)
    assert_kv_equal(gpu, o, new, new_h, kv)
    a = _host_cache(new[0])
    b = _host_cache(old[0])
    re = np.flatnonzero(gpu["disposition"][0] == 2)
    assert re.size and (a[:, :, re] == b[:, :, re]).all()


@pytest.mark.parametrize("H,D,dtype", [(8, 512, 0), (4, 512, 0), (4, 512, 1), (2, 384, 0)])
def test_kv_wide_heads(abi, ref, H, D, dtype):
    """head_dim in (256, 512]: the per-stage cos/sin table no longer leaves 3 TMA stages for 8 warps, so the gather
    runs with fewer warps per CTA (rows <= 8 KB) or the register path (rows > 8 KB) -- decided before the plan kernel
    is enqueued, never a failure after it.  Copy mode and paged, against the oracle."""
    g = make_grid(448, 448)
    cfg = synth.CONFIGS["C1"]
    w, s, ring, S = 8, 2, 10, 2
    mring, tring = stream_rings(ref, g, cfg, S, ring, 5, w, s)
    win = dict(window=w, stride=s, step=5, ring_frames=ring)
    cap = w * 256 + 8
    kv = dict(layers=2, kv_heads=H, head_dim=D, dtype=dtype, capacity=cap, refresh_capacity=cap, rope_base=1e6,
              n_prompt=8)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(17)
    old, new, refr = make_caches(kv, S, gen)
    stats = {}
    gpu, o, new_h = run_kv_both(abi, ref, g, kv, win, mring, tring, old, new, refr, cap)
    assert gpu["status"] == 0
    assert_kv_equal(gpu, o, new, new_h, kv, stats)
    rng = np.random.default_rng(4)
    slot_old = np.stack([rng.permutation(cap) for _ in range(S)]).astype(np.int32)
    _, _, st = run_paged_both(abi, ref, g, kv, win, mring, tring, old, slot_old, cap, refr, cap)
    for key in ("not_bit_exact", "rotated"):
        stats[key] = stats.get(key, 0) + st[key]
    kvcheck.assert_rotation_bits(stats)


def test_kv_misaligned_buffer_status(abi, ref):
    """A stream whose cache pointer is not 16-B aligned (a narrowed bf16 view): CS_STATUS_MISALIGNED, none of its
    rows move, its index outputs and every other stream are exactly as the oracle's (copy mode and paged)."""
    g = make_grid(448, 448)
    cfg = synth.CONFIGS["C1"]
    w, s, ring, S = 8, 2, 10, 3
    mring, tring = stream_rings(ref, g, cfg, S, ring, 5, w, s)
    win = dict(window=w, stride=s, step=5, ring_frames=ring)
    cap = w * 256 + 8
    kv = dict(synth.QWEN_KV, layers=2, capacity=cap, refresh_capacity=cap, n_prompt=8)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(23)
    old, new, refr = make_caches(kv, S, gen)
    shape = new[1].shape
    backing = torch.full((new[1].numel() + 8,), 7.0, device=DEV).to(torch.bfloat16)
    new[1] = backing[1:1 + new[1].numel()].view(shape)            # data_ptr % 16 == 2
    before = _host_cache(new[1]).copy()
    m_d = torch.from_numpy(mring.view(np.int32)).to(DEV)
    t_d = torch.from_numpy(tring).to(DEV)
    disp = torch.full((S, cap), 9, dtype=torch.uint8, device=DEV)
    pold = torch.full((S, cap), -9, dtype=torch.int32, device=DEV)
    ntok = torch.zeros(S, 4, dtype=torch.int32, device=DEV)
    ws = torch.empty(abi.kv_workspace_size(kv, win, S), dtype=torch.uint8, device=DEV)
    cnt = torch.zeros(16, dtype=torch.int64, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    abi.codecsight_kv_refresh(g, kv, win, S, m_d, t_d, abi.ptr_array(old, DEV), abi.ptr_array(new, DEV),
                              abi.ptr_array(refr, DEV), cap, disp, pold, ntok, ws, cnt, st)
    pre_h = [_host_cache(t).copy() for t in new]
    old_h = [_host_cache(t) for t in old]
    ref_h = [_host_cache(t) for t in refr]
    exp_h = [t.copy() for t in pre_h]
    o = ref.kv_refresh(g, kv, win, mring, tring, old_h, exp_h, ref_h, cap)
    torch.cuda.synchronize()
    assert int(st.item()) == o["status"] | abi.CS_STATUS_MISALIGNED
    assert (ntok.cpu().numpy() == o["n_tokens"]).all()
    for si in range(S):
        nt = int(o["n_tokens"][si, 0]) + 8
        assert (disp.cpu().numpy()[si, :nt] == o["disposition"][si, :nt]).all()
        assert (pold.cpu().numpy()[si, :nt] == o["p_old"][si, :nt]).all()
        if si == 1:
            assert (_host_cache(new[1]) == before).all()           # nothing moved in the misaligned stream
        else:
            kvcheck.check_copy_step(_host_cache(new[si]), pre_h[si], exp_h[si], o["disposition"][si],
                                    o["p_old"][si], nt, kv, old=old_h[si], refr=ref_h[si], tag=f"stream {si}")
    # paged: stream 2's pool misaligned
    pools = [t.clone() for t in old]
    pb = torch.empty(pools[2].numel() + 8, dtype=torch.bfloat16, device=DEV)
    pools[2] = pb[1:1 + pools[2].numel()].view(pools[2].shape)
    pools[2].copy_(old[2])
    pre2 = _host_cache(pools[2]).copy()
    sn_d = torch.full((S, cap), -7, dtype=torch.int32, device=DEV)
    so_d = torch.from_numpy(np.stack([np.arange(cap, dtype=np.int32)] * S)).to(DEV)
    wsp = torch.empty(abi.kv_paged_workspace_size(g, kv, win, S), dtype=torch.uint8, device=DEV)
    st.zero_()
    abi.codecsight_kv_refresh_paged(g, kv, win, S, m_d, t_d, abi.ptr_array(pools, DEV), so_d, sn_d, cap,
                                    abi.ptr_array(refr, DEV), cap, disp, pold, ntok, wsp, cnt, st)
    torch.cuda.synchronize()
    assert int(st.item()) & abi.CS_STATUS_MISALIGNED
    assert (_host_cache(pools[2]) == pre2).all()
    assert not (_host_cache(pools[0]) == _host_cache(old[0])).all()   # the aligned streams did move rows


def test_kv_bf16_rne_ties(abi, ref):
    """Rotated keys that land exactly on a bf16 tie (tests/rne_ties.py, both parities): the kernels' bf16 store
    must round them to even (reading Q20), bit-identical to PyTorch's fp32 -> bf16 conversion and to the oracle,
    in copy mode and in place (paged)."""
    import rne_ties
    g = make_grid(128, 128, mb_size=32, grid_w=4, grid_h=4, patch=4, group=2)
    nw = 1
    groups = [[0], [1], [0, 1], [2], [0], [0, 1, 2, 3], [1], [2]]
    mring = np.zeros((1, 8, nw), np.uint32)
    for f, gl in enumerate(groups):
        for q in gl:
            gr, gc = divmod(q, 2)
            for dy in range(2):
                for dx in range(2):
                    mring[0, f, 0] |= np.uint32(1 << ((gr * 2 + dy) * 4 + gc * 2 + dx))
    tring = np.array([[0, 1, 1, 1, 1, 1, 1, 1]], np.uint8)
    D = 128
    kv = dict(layers=1, kv_heads=1, head_dim=D, dtype=0, capacity=16, refresh_capacity=16, rope_base=1e4,
              n_prompt=0)
    rows, ties = rne_ties.tie_rows(4, D, 1e4, -3)     # window 2: dp = -3, p_old 4..7 -> p_new 1..4 (REUSE)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(2)
    old, new, refr = make_caches(kv, 1, gen)
    old[0][0, 0, 4:8, 0] = torch.from_numpy(rows.view(np.int16)).to(DEV).view(torch.bfloat16)
    win = dict(window=4, stride=2, step=2, ring_frames=8)
    gpu, o, new_h = run_kv_both(abi, ref, g, kv, win, mring, tring, old, new, refr, 16)
    assert_kv_equal(gpu, o, new, new_h, kv)
    got = _host_cache(new[0])
    # paged: the same keys rotated in place (window-1 slot map = identity)
    pool = [old[0].clone()]
    sn, _, _ = run_paged_both(abi, ref, g, kv, win, mring, tring, pool, np.arange(16, dtype=np.int32)[None], 16,
                              refr, 16)
    gotp = _host_cache(pool[0])
    for j in range(4):
        idx = np.array([e for e, _ in ties[j]])
        exp = rne_ties.rne_bf16(np.array([v for _, v in ties[j]], np.float32))
        assert gpu["disposition"][0, 1 + j] == 2 and gpu["p_old"][0, 1 + j] == 4 + j
        assert (got[0, 0, 1 + j, 0, idx] == exp).all(), j
        assert (gotp[0, 0, sn[0, 1 + j], 0, idx] == exp).all(), j


@pytest.mark.parametrize("overlap", [False, True])
def test_pipeline_end_to_end_c4_shape(abi, ref, overlap):
    """Pipeline (score -> compact -> kv_refresh) on a C4-shaped shard (4 streams: 2 static, 2 high-motion, 1080p,
    w=16, s=4, GOP 16) for 4 steps, every output compared with the oracle driven the same way."""
    from paper_2604_06036_b200.pipeline import Pipeline
    cfg = synth.CONFIGS["C4"]
    g = make_grid(1920, 1080)
    S, w, s, gop = 4, 16, 4, 16
    kvb = dict(synth.QWEN_KV, layers=2)
    pipe = Pipeline(g, S, w, s, gop, kvb, n_prompt=32, device=DEV, overlap=overlap)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(4)
    pipe.init_cache_fill(gen)
    nw = 32
    ring = pipe.ring
    gens = [synth.StreamGen(1920, 1080, synth.scene_of(cfg, si), synth.stream_seed(cfg, si)) for si in range(S)]
    gop_h = np.zeros((S, nw + 1), np.uint32)
    mring_h = np.zeros((S, ring, nw), np.uint32)
    tring_h = np.zeros((S, ring), np.uint8)
    rng = np.random.default_rng(0)
    frames_h = synth.random_frames(S * w, 448, 448, rng)
    frames_d = [torch.from_numpy(f.view(np.int16)).to(DEV) for f in frames_h]
    stats = {}
    for k in range(6 if overlap else 4):
        f0, n = pipe.new_frames(k)
        mb = np.stack([np.stack([gens[si].next_frame() for _ in range(n)]) for si in range(S)])
        types = np.stack([synth.frame_types(n, gop, f0) for _ in range(S)])
        fptr = abi.ptr_array(frames_d[:S * n], DEV)
        fidx = np.tile(np.arange(f0, f0 + n, dtype=np.int32), S)
        old_h = [_host_cache(c).copy() for c in pipe.caches[pipe.cur]]
        new_h = [_host_cache(c).copy() for c in pipe.caches[1 - pipe.cur]]   # content before the step
        pre_h = [c.copy() for c in new_h]
        ref_h = [_host_cache(c) for c in pipe.refreshed]
        pipe.step(k, d_mb(mb), fptr, torch.from_numpy(fidx).to(DEV), torch.from_numpy(types).to(DEV))
        torch.cuda.synchronize()
        # oracle, same sequence
        off = f0 % ring
        tring_h[:, off:off + n] = types
        so = ref.score_patches(g, mb, np.ascontiguousarray(tring_h[:, off:]), gop_h, want_score=False,
                               frame_stride=ring - off)
        mring_h[:, off:off + n] = so["keep_mask"][:, :n]
        assert (u32(pipe.mask_ring) == mring_h).all()
        assert (u32(pipe.gop_state) == gop_h).all()
        assert (pipe.kept_counts(n).cpu().numpy() == so["kept_count"]).all()
        co = ref.compact(g, mring_h[:, off:].copy(), fidx, frames_h[:S * n], pipe.capacity, S, n,
                         mask_frame_stride=ring - off)
        tot = int(co["frame_offsets"][-1])
        assert (pipe.frame_offsets[:S * n + 1].cpu().numpy() == co["frame_offsets"]).all()
        assert (pipe.src_index[:tot].cpu().numpy() == co["src_index"][:tot]).all()
        assert (pipe.pos_ids[:tot].cpu().numpy() == co["pos_ids"][:tot]).all()
        assert (pipe.packed[:tot].view(torch.int16).cpu().numpy().view(np.uint16) == co["packed"][:tot]).all()
        new_d = pipe.caches[pipe.cur]      # after the swap, cur holds window k
        prev = [_host_cache(c) for c in new_d]
        win = dict(window=w, stride=s, step=k, ring_frames=ring)
        ko = ref.kv_refresh(g, pipe.kv, win, mring_h, tring_h, old_h if k else None, new_h,
                            ref_h if k >= 1 else None, pipe.token_cap)
        gpu = dict(disposition=pipe.disposition.cpu().numpy(), p_old=pipe.p_old.cpu().numpy(),
                   n_tokens=pipe.n_tokens.cpu().numpy(), counters=ko["counters"], status=ko["status"])
        assert (gpu["n_tokens"] == ko["n_tokens"]).all()
        for si in range(S):
            nt = int(ko["n_tokens"][si, 0]) + 32
            assert (gpu["disposition"][si, :nt] == ko["disposition"][si, :nt]).all()
            assert (gpu["p_old"][si, :nt] == ko["p_old"][si, :nt]).all()
            kvcheck.check_copy_step(prev[si], pre_h[si], new_h[si], ko["disposition"][si], ko["p_old"][si], nt,
                                    pipe.kv, old=old_h[si] if k else None, refr=ref_h[si] if k >= 1 else None,
                                    stats=stats, tag=f"step {k} stream {si}")
    assert int(pipe.status.item()) == 0
    kvcheck.assert_rotation_bits(stats)


@pytest.mark.parametrize("kv_mode", ["paged", "copy"])
def test_pipeline_fused_overlap_matches_sequential(abi, ref, kv_mode):
    """Fused score+compact with overlap (kv_refresh of step k on its own stream, concurrent with score+compact of
    step k+1), every step enqueued without a host synchronisation, against the same steps run sequentially (itself
    parity-tested against the oracle): final GOP state, each frame's mask, the K/V cache state, slot maps and the
    last two steps' outputs (one per buffer set) must be bit-identical."""
    from paper_2604_06036_b200.pipeline import Pipeline
    cfg = synth.CONFIGS["C4"]
    g = make_grid(1920, 1080)
    S, w, s, gop = 6, 16, 4, 16
    kvb = dict(synth.QWEN_KV, layers=2)
    K = 9
    rng = np.random.default_rng(5)
    frames_h = synth.random_frames(S * w, 448, 448, rng)
    frames_d = [torch.from_numpy(to_grouped(f, g).view(np.int16)).to(DEV) for f in frames_h]
    gens = [synth.StreamGen(1920, 1080, synth.scene_of(cfg, si), synth.stream_seed(cfg, si)) for si in range(S)]
    inputs = []
    for k in range(K):
        f0, n = (0, w) if k == 0 else ((k - 1) * s + w, s)
        mb = np.stack([np.stack([gens[si].next_frame() for _ in range(n)]) for si in range(S)])
        types = np.stack([synth.frame_types(n, gop, f0) for _ in range(S)])
        fidx = np.tile(np.arange(f0, f0 + n, dtype=np.int32), S)
        inputs.append((d_mb(mb), abi.ptr_array(frames_d[:S * n], DEV), torch.from_numpy(fidx).to(DEV),
                       torch.from_numpy(types).to(DEV)))
    runs = {}
    for overlap in (False, True):
        pipe = Pipeline(g, S, w, s, gop, kvb, n_prompt=32, device=DEV, frame_layout=abi.CS_LAYOUT_GROUPED,
                        kv_mode=kv_mode, compact_chunk=s, fused=True, overlap=overlap)
        gen = torch.Generator(device=DEV)
        gen.manual_seed(9)
        pipe.init_cache_fill(gen)
        outs = {}
        for k in range(K):
            pipe.step(k, *inputs[k])
            if not overlap:
                torch.cuda.synchronize()
            if k >= K - 2:   # the last two steps' outputs live in different buffer sets with overlap
                bufs = (pipe.packed, pipe.pos_ids, pipe.src_index, pipe.frame_offsets, pipe.kept_count,
                        pipe.disposition, pipe.p_old, pipe.n_tokens)
                outs[k] = bufs if overlap else tuple(t.clone() for t in bufs)   # sequential: one buffer set
        pipe.join()
        torch.cuda.synchronize()
        f_last = (K - 1) * s + w   # frames 0 .. f_last-1 exist; masks of the last w + s frames by frame index
        masks = {f: pipe.mask_ring[:, f % pipe.ring].cpu().numpy() for f in range(f_last - w - s, f_last)}
        state = dict(gop=pipe.gop_state.cpu().numpy(), masks=masks, status=int(pipe.status.item()),
                     counters=pipe.counters.cpu().numpy(),
                     caches=[_host_cache(c).copy() for c in pipe.caches[pipe.cur if kv_mode == "copy" else 0]],
                     slots=pipe.slots[pipe.cur].cpu().numpy() if kv_mode == "paged" else None,
                     outs={k: [(t.view(torch.int16) if t.dtype == torch.bfloat16 else t).cpu().numpy().copy()
                               for t in v] for k, v in outs.items()})
        runs[overlap] = state
        del pipe
    a, b = runs[False], runs[True]
    assert a["status"] == b["status"] == 0
    assert (a["gop"] == b["gop"]).all()
    for f in a["masks"]:
        assert (a["masks"][f] == b["masks"][f]).all(), f
    assert (a["counters"] == b["counters"]).all()
    for x, y in zip(a["caches"], b["caches"]):
        assert (x.view(np.uint16) == y.view(np.uint16)).all()
    if kv_mode == "paged":
        assert (a["slots"] == b["slots"]).all()
    for k in a["outs"]:   # the valid part of each output (stale rows of earlier steps differ by buffer set)
        (pa, qa, sa, fa, ka, da, oa, na), (pb, qb, sb, fb, kb, db, ob, nb_) = a["outs"][k], b["outs"][k]
        assert (fa[:S * s + 1] == fb[:S * s + 1]).all(), k
        tot = int(fa[S * s])
        assert (pa[:tot].view(np.uint16) == pb[:tot].view(np.uint16)).all(), k
        assert (qa[:tot] == qb[:tot]).all() and (sa[:tot] == sb[:tot]).all(), k
        assert (ka.reshape(-1)[:S * s] == kb.reshape(-1)[:S * s]).all(), k
        assert (na == nb_).all(), k
        for si in range(S):
            nt = int(na[si, 0]) + 32
            assert (da[si, :nt] == db[si, :nt]).all() and (oa[si, :nt] == ob[si, :nt]).all(), (k, si)


@pytest.mark.parametrize("rope", ["1d", "mrope"])
def test_pipeline_temporal_patch2(abi, ref, rope):
    """Pipeline with Qwen2-VL temporal patches (tp = 2) on a C4-shaped shard, paged KV over token units: per-frame
    scoring, [3][2][14][14] unit rows with unit masks / types written into the unit ring, KV refresh with window
    w/2 and stride s/2 -- every output compared with the oracle driven the same way for 5 steps."""
    from paper_2604_06036_b200.pipeline import Pipeline
    cfg = synth.CONFIGS["C4"]
    g = make_grid(1920, 1080)
    S, w, s, gop, tp = 4, 16, 4, 16, 2
    kvb = dict(synth.QWEN_KV if rope == "1d" else synth.QWEN_MROPE_KV, layers=2)
    pipe = Pipeline(g, S, w, s, gop, kvb, n_prompt=32, device=DEV, kv_mode="paged", temporal_patch=tp,
                    frame_layout=abi.CS_LAYOUT_GROUPED)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(5)
    pipe.init_cache_fill(gen)
    nw, ring, uring = 32, pipe.ring, pipe.uring
    gens = [synth.StreamGen(1920, 1080, synth.scene_of(cfg, si), synth.stream_seed(cfg, si)) for si in range(S)]
    gop_h = np.zeros((S, nw + 1), np.uint32)
    mring_h = np.zeros((S, ring, nw), np.uint32)
    tring_h = np.zeros((S, ring), np.uint8)
    uring_h = np.zeros((S, uring, nw), np.uint32)
    utring_h = np.zeros((S, uring), np.uint8)
    rng = np.random.default_rng(2)
    frames_h = synth.random_frames(S * w, 448, 448, rng)
    frames_g = [to_grouped(f, g) for f in frames_h]
    frames_d = [torch.from_numpy(f.view(np.int16)).to(DEV) for f in frames_g]
    slot_h = None
    stats = {}
    for k in range(5):
        f0, n = pipe.new_frames(k)
        nu = n // tp
        mb = np.stack([np.stack([gens[si].next_frame() for _ in range(n)]) for si in range(S)])
        types = np.stack([synth.frame_types(n, gop, f0) for _ in range(S)])
        fptr = abi.ptr_array(frames_d[:S * n], DEV)
        uidx = np.tile(np.arange(f0 // tp, f0 // tp + nu, dtype=np.int32), S)
        pool_h = [_host_cache(c).copy() for c in pipe.caches[0]]
        pre_h = [c.copy() for c in pool_h]
        ref_h = [_host_cache(c) for c in pipe.refreshed]
        pipe.step(k, d_mb(mb), fptr, torch.from_numpy(uidx).to(DEV), torch.from_numpy(types).to(DEV))
        torch.cuda.synchronize()
        off, uoff = f0 % ring, (f0 % ring) // tp
        tring_h[:, off:off + n] = types
        so = ref.score_patches(g, mb, np.ascontiguousarray(tring_h[:, off:]), gop_h, want_score=False,
                               frame_stride=ring - off)
        mring_h[:, off:off + n] = so["keep_mask"][:, :n]
        assert (u32(pipe.mask_ring) == mring_h).all()
        co = ref.compact_tp(g, tp, mring_h[:, off:].copy(), uidx, frames_g[:S * n], pipe.capacity, S, nu,
                            mask_frame_stride=ring - off, frame_layout=1, want_unit_mask=True,
                            frame_type=np.ascontiguousarray(tring_h[:, off:]))
        uring_h[:, uoff:uoff + nu] = co["unit_mask"]
        utring_h[:, uoff:uoff + nu] = co["unit_type"]
        assert (u32(pipe.unit_ring) == uring_h).all()
        assert (pipe.unit_type_ring.cpu().numpy() == utring_h).all()
        tot = int(co["frame_offsets"][-1])
        assert (pipe.frame_offsets[:S * nu + 1].cpu().numpy() == co["frame_offsets"]).all()
        assert (pipe.pos_ids[:tot].cpu().numpy() == co["pos_ids"][:tot]).all()
        assert (pipe.src_index[:tot].cpu().numpy() == co["src_index"][:tot]).all()
        assert (pipe.packed[:tot].view(torch.int16).cpu().numpy().view(np.uint16) == co["packed"][:tot]).all()
        win = dict(window=w // tp, stride=s // tp, step=k, ring_frames=uring)
        ko = ref.kv_refresh_paged(g, pipe.kv, win, uring_h, utring_h, pool_h, slot_h, pipe.token_cap,
                                  ref_h if k >= 1 else None, pipe.token_cap)
        assert (pipe.n_tokens.cpu().numpy() == ko["n_tokens"]).all()
        sn = pipe.slots[pipe.cur].cpu().numpy()
        for si in range(S):
            nt = int(ko["n_tokens"][si, 0]) + 32
            assert (pipe.disposition.cpu().numpy()[si, :nt] == ko["disposition"][si, :nt]).all()
            assert (pipe.p_old.cpu().numpy()[si, :nt] == ko["p_old"][si, :nt]).all()
            assert (sn[si, :nt] == ko["slot_new"][si, :nt]).all()
            kvcheck.check_pool_step(_host_cache(pipe.caches[0][si]), pre_h[si], pool_h[si], ko["disposition"][si],
                                    ko["slot_new"][si], nt, pipe.kv, refr=ref_h[si] if k >= 1 else None,
                                    stats=stats, tag=f"step {k} stream {si}")
        slot_h = ko["slot_new"]
        if k >= 1:
            assert any((ko["disposition"][si, :int(ko["n_tokens"][si, 0])] == 2).any() for si in range(S))
    assert int(pipe.status.item()) == 0
    kvcheck.assert_rotation_bits(stats)


def test_pipeline_cuda_graphs(abi, ref):
    """Steps k >= 1 replayed as captured CUDA graphs (one per (ring phase, slot parity)), inputs staged into fixed
    buffers: 12 steps (graphs reused across two ring periods), fused score+compact + paged KV, every output compared
    with the oracle driven the same way."""
    from paper_2604_06036_b200.pipeline import Pipeline
    cfg = synth.CONFIGS["C4"]
    g = make_grid(1920, 1080)
    S, w, s, gop = 4, 16, 4, 16
    kvb = dict(synth.QWEN_KV, layers=2)
    pipe = Pipeline(g, S, w, s, gop, kvb, n_prompt=32, device=DEV, kv_mode="paged", fused=True,
                    frame_layout=abi.CS_LAYOUT_GROUPED)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(9)
    pipe.init_cache_fill(gen)
    nw, ring = 32, pipe.ring
    gens = [synth.StreamGen(1920, 1080, synth.scene_of(cfg, si), synth.stream_seed(cfg, si)) for si in range(S)]
    gop_h = np.zeros((S, nw + 1), np.uint32)
    mring_h = np.zeros((S, ring, nw), np.uint32)
    tring_h = np.zeros((S, ring), np.uint8)
    rng = np.random.default_rng(3)
    frames_h = [to_grouped(f, g) for f in synth.random_frames(S * s, 448, 448, rng)]
    frames_d = [torch.from_numpy(f.view(np.int16)).to(DEV) for f in frames_h]
    ptr_w = abi.ptr_array([frames_d[i % len(frames_d)] for i in range(S * w)], DEV)
    ptr_s = abi.ptr_array(frames_d, DEV)
    stage = [dict(mb=torch.empty(S * s * 68 * 120 * 8, dtype=torch.uint8, device=DEV),
                  ty=torch.empty(S, s, dtype=torch.uint8, device=DEV),
                  fi=torch.empty(S * s, dtype=torch.int32, device=DEV)) for _ in range(2)]
    slot_h = None
    stats = {}
    for k in range(12):
        f0, n = pipe.new_frames(k)
        mb = np.stack([np.stack([gn.next_frame() for _ in range(n)]) for gn in gens])
        types = np.stack([synth.frame_types(n, gop, f0) for _ in range(S)])
        fidx = np.tile(np.arange(f0, f0 + n, dtype=np.int32), S)
        pool_h = [_host_cache(c).copy() for c in pipe.caches[0]]
        pre_h = [c.copy() for c in pool_h]
        ref_h = [_host_cache(c) for c in pipe.refreshed]
        if k == 0:
            pipe.step(k, d_mb(mb), ptr_w, torch.from_numpy(fidx).to(DEV), torch.from_numpy(types).to(DEV))
        else:
            st = stage[k & 1]
            st["mb"].copy_(torch.from_numpy(mb.view(np.uint8).reshape(-1)))
            st["ty"].copy_(torch.from_numpy(types))
            st["fi"].copy_(torch.from_numpy(fidx))
            pipe.graph_step(k, st["mb"], ptr_s, st["fi"], st["ty"])
        torch.cuda.synchronize()
        off = f0 % ring
        tring_h[:, off:off + n] = types
        so = ref.score_patches(g, mb, np.ascontiguousarray(tring_h[:, off:]), gop_h, want_score=False,
                               frame_stride=ring - off)
        mring_h[:, off:off + n] = so["keep_mask"][:, :n]
        assert (u32(pipe.mask_ring) == mring_h).all()
        fr = [frames_h[i % len(frames_h)] for i in range(S * n)]
        co = ref.compact(g, mring_h[:, off:].copy(), fidx, fr, pipe.capacity, S, n, mask_frame_stride=ring - off,
                         frame_layout=1)
        tot = int(co["frame_offsets"][-1])
        assert (pipe.frame_offsets[:S * n + 1].cpu().numpy() == co["frame_offsets"]).all()
        assert (pipe.packed[:tot].view(torch.int16).cpu().numpy().view(np.uint16) == co["packed"][:tot]).all()
        assert (pipe.pos_ids[:tot].cpu().numpy() == co["pos_ids"][:tot]).all()
        win = dict(window=w, stride=s, step=k, ring_frames=ring)            # the true window index
        ko = ref.kv_refresh_paged(g, pipe.kv, win, mring_h, tring_h, pool_h, slot_h, pipe.token_cap,
                                  ref_h if k >= 1 else None, pipe.token_cap)
        assert (pipe.n_tokens.cpu().numpy() == ko["n_tokens"]).all()
        sn = pipe.slots[pipe.cur].cpu().numpy()
        for si in range(S):
            nt = int(ko["n_tokens"][si, 0]) + 32
            assert (pipe.disposition.cpu().numpy()[si, :nt] == ko["disposition"][si, :nt]).all()
            assert (pipe.p_old.cpu().numpy()[si, :nt] == ko["p_old"][si, :nt]).all()
            assert (sn[si, :nt] == ko["slot_new"][si, :nt]).all()
            kvcheck.check_pool_step(_host_cache(pipe.caches[0][si]), pre_h[si], pool_h[si], ko["disposition"][si],
                                    ko["slot_new"][si], nt, pipe.kv, refr=ref_h[si] if k >= 1 else None,
                                    stats=stats, tag=f"step {k} stream {si}")
        slot_h = ko["slot_new"]
    assert int(pipe.status.item()) == 0
    kvcheck.assert_rotation_bits(stats)
    assert 1 <= len(pipe._graphs) <= 10          # reused across ring periods: at most period x 2 captures


# ------------------------------------------------------------------------------------------------------------
# kv_refresh_paged (NEXT-1: in place, slot maps)
# ------------------------------------------------------------------------------------------------------------
def _full_paged_plan(ref, g, kv, win, mring, tring, pool, slot_old, slot_cap, n_all):
    """Disposition and slot of every token of one stream (the oracle run with index outputs large enough for all
    of them; slot_old padded with -1, which the oracle treats exactly like an index past slot_cap)."""
    cap2 = max(n_all, slot_cap)
    so = None
    if slot_old is not None:
        so = np.full((1, cap2), -1, np.int32)
        so[:, :slot_cap] = slot_old
    o = ref.kv_refresh_paged(g, kv, win, mring, tring, [pool.copy()], so, cap2, None, n_all)
    return o["disposition"][0], o["slot_new"][0]


def run_paged_both(abi, ref, g, kv, win, mring, tring, pools_d, slot_old_h, slot_cap, ref_d, token_cap):
    S = mring.shape[0]
    pools_h = [_host_cache(t).copy() for t in pools_d]
    pre_h = [t.copy() for t in pools_h]
    ref_h = [_host_cache(t) for t in ref_d] if ref_d is not None else None
    m_d = torch.from_numpy(np.ascontiguousarray(mring).view(np.int32)).to(DEV)
    t_d = torch.from_numpy(np.ascontiguousarray(tring)).to(DEV)
    so_d = torch.from_numpy(slot_old_h).to(DEV) if slot_old_h is not None else None
    sn_d = torch.full((S, slot_cap), -7, dtype=torch.int32, device=DEV)
    disp = torch.full((S, token_cap), 9, dtype=torch.uint8, device=DEV)
    pold = torch.full((S, token_cap), -9, dtype=torch.int32, device=DEV)
    ntok = torch.zeros(S, 4, dtype=torch.int32, device=DEV)
    ws = torch.empty(abi.kv_paged_workspace_size(g, kv, win, S), dtype=torch.uint8, device=DEV)
    cnt = torch.zeros(16, dtype=torch.int64, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    abi.codecsight_kv_refresh_paged(g, kv, win, S, m_d, t_d, abi.ptr_array(pools_d, DEV), so_d, sn_d, slot_cap,
                                    abi.ptr_array(ref_d, DEV) if ref_d is not None else None, token_cap, disp, pold,
                                    ntok, ws, cnt, st)
    o = ref.kv_refresh_paged(g, kv, win, mring, tring, pools_h, slot_old_h, slot_cap, ref_h, token_cap)
    torch.cuda.synchronize()
    assert int(st.item()) == o["status"]
    assert (ntok.cpu().numpy() == o["n_tokens"]).all()
    assert (cnt.cpu().numpy().view(np.uint64) == o["counters"]).all(), (cnt.cpu().numpy(), o["counters"])
    sn = sn_d.cpu().numpy()
    stats = {"not_bit_exact": 0, "max_diff": 0.0, "rotated": 0}
    for s in range(S):
        nt = min(int(o["n_tokens"][s, 0]) + kv["n_prompt"], token_cap)
        assert (disp.cpu().numpy()[s, :nt] == o["disposition"][s, :nt]).all()
        assert (pold.cpu().numpy()[s, :nt] == o["p_old"][s, :nt]).all()
        nsl = min(int(o["n_tokens"][s, 0]) + kv["n_prompt"], slot_cap)
        assert (sn[s, :nsl] == o["slot_new"][s, :nsl]).all()
        # every pool element: pure copies / untouched rows bit-identical, rotated keys within the bound
        n_all = int(o["n_tokens"][s, 0]) + kv["n_prompt"]
        if n_all <= min(token_cap, slot_cap):
            fd, fs = o["disposition"][s], o["slot_new"][s]
        else:   # index outputs truncated: the full plan of this stream from the oracle with uncapped outputs
            fd, fs = _full_paged_plan(ref, g, kv, win, mring[s:s + 1], tring[s:s + 1], pre_h[s],
                                      slot_old_h[s:s + 1] if slot_old_h is not None else None, slot_cap, n_all)
        kvcheck.check_pool_step(_host_cache(pools_d[s]), pre_h[s], pools_h[s], fd, fs, n_all, kv,
                                refr=ref_h[s] if ref_h is not None else None, stats=stats, tag=f"stream {s}")
    return sn, o, stats


@pytest.mark.parametrize("dtype", [1, 0])
def test_paged_c1_windows(abi, ref, dtype):
    """C1 streams of all 5 scene kinds, 14 consecutive windows, slot maps carried from step to step."""
    cfg = synth.CONFIGS["C1"]
    g = make_grid(448, 448)
    w, s, ring = 8, 2, 10
    base = synth.TOY_KV if dtype == 1 else dict(synth.QWEN_KV, layers=2)
    cap = w * 256 + 32
    kv = dict(base, capacity=cap + 64, refresh_capacity=cap, n_prompt=32)
    S = 5
    gen = torch.Generator(device=DEV)
    gen.manual_seed(5)
    dt = torch.bfloat16 if dtype == 0 else torch.float32
    shape = (kv["layers"], 2, kv["capacity"], kv["kv_heads"], kv["head_dim"])
    pools = [torch.randn(shape, generator=gen, device=DEV).to(dt) for _ in range(S)]
    slot = None
    tot = {"not_bit_exact": 0, "max_diff": 0.0}
    for k in range(14):
        mring, tring = stream_rings(ref, g, cfg, S, ring, k, w, s)
        _, _, refr = make_caches(kv, S, gen)
        sn, o, st = run_paged_both(abi, ref, g, kv, dict(window=w, stride=s, step=k, ring_frames=ring), mring, tring,
                                   pools, slot, cap, refr, cap)
        slot = sn
        for key in ("not_bit_exact", "rotated"):
            tot[key] = tot.get(key, 0) + st[key]
        tot["max_diff"] = max(tot["max_diff"], st["max_diff"])
    kvcheck.assert_rotation_bits(tot)


def test_paged_c5_shape(abi, ref):
    """C5 shape: 4K traffic masks, w=64, s=8, GOP 16, Qwen2-VL-7B rows (2 layers to bound the oracle), 2 streams,
    windows 0 and 1."""
    cfg = synth.CONFIGS["C5"]
    g = make_grid(3840, 2160)
    w, s, ring = 64, 8, 72
    cap = w * 256 + 32
    kv = dict(synth.QWEN_KV, layers=2, capacity=cap, refresh_capacity=13 * 256 + 32, n_prompt=32)
    S = 2
    gen = torch.Generator(device=DEV)
    gen.manual_seed(6)
    shape = (kv["layers"], 2, cap, 4, 128)
    pools = [torch.randn(shape, generator=gen, device=DEV).to(torch.bfloat16) for _ in range(S)]
    slot = None
    for k in range(2):
        mring, tring = stream_rings(ref, g, cfg, S, ring, k, w, s)
        _, _, refr = make_caches(dict(kv, refresh_capacity=cap) if k == 0 else kv, S, gen)
        sn, o, st = run_paged_both(abi, ref, g, dict(kv, refresh_capacity=cap) if k == 0 else kv,
                                   dict(window=w, stride=s, step=k, ring_frames=ring), mring, tring, pools, slot, cap,
                                   refr, cap)
        slot = sn


def test_paged_edge_cases(abi, ref):
    cfg = synth.CONFIGS["C1"]
    g = make_grid(448, 448)
    w, s, ring = 8, 2, 10
    S = 5
    gen = torch.Generator(device=DEV)
    gen.manual_seed(8)
    mring, tring = stream_rings(ref, g, cfg, S, ring, 3, w, s)
    win = dict(window=w, stride=s, step=3, ring_frames=ring)
    cap = w * 256 + 32
    rng = np.random.default_rng(2)
    for kvb, slot_cap, tc, pool_cap, with_ref in [
            (synth.TOY_KV, cap, cap, cap + 10, True),          # plain
            (synth.TOY_KV, cap, cap, cap + 10, False),         # refreshed = NULL
            (synth.TOY_KV, 300, 250, 400, True),               # small slot map / index / pool: CAPACITY
            (dict(layers=3, kv_heads=1, head_dim=2, dtype=1, rope_base=1e4), cap, cap, cap, True),   # scalar paths
            (dict(layers=2, kv_heads=2, head_dim=8, dtype=0, rope_base=1e6), cap, cap, cap, True)]:
        kv = dict(kvb, capacity=pool_cap, refresh_capacity=min(cap, 900), n_prompt=32)
        dt = torch.bfloat16 if kv["dtype"] == 0 else torch.float32
        shape = (kv["layers"], 2, pool_cap, kv["kv_heads"], kv["head_dim"])
        pools = [torch.randn(shape, generator=gen, device=DEV).to(dt) for _ in range(S)]
        # an arbitrary permutation of slots for window k-1 (some out of range -> ORIGIN)
        slot_old = np.stack([rng.permutation(pool_cap)[:slot_cap] for _ in range(S)]).astype(np.int32)
        slot_old[0, 5] = pool_cap + 3
        _, _, refr = make_caches(kv, S, gen)
        run_paged_both(abi, ref, g, kv, win, mring, tring, pools, slot_old, slot_cap, refr if with_ref else None, tc)


def _random_group_rings(g, S, ring, gop, rng, p_keep=0.5):
    """Group-complete masks (each 2x2 group kept with p_keep) and I/P types for a ring of frames."""
    ngr, ngc = g["grid_h"] // 2, g["grid_w"] // 2
    keep = rng.random((S, ring, ngr, ngc)) < p_keep
    bits = np.repeat(np.repeat(keep, 2, axis=2), 2, axis=3)            # [S][ring][32][32] patch bits
    words = (bits.astype(np.uint64) << np.arange(g["grid_w"], dtype=np.uint64)).sum(axis=-1).astype(np.uint32)
    types = np.where(np.arange(ring) % gop == 0, 0, 1).astype(np.uint8)
    return words, np.broadcast_to(types, (S, ring)).copy()


def test_paged_long_window_move_list_in_global(abi, ref):
    """w = 96: the plan's per-stream move list (96 x 256 + 32 entries, 197 KB) no longer fits the plan kernel's
    shared memory and is read back from the workspace instead (kv_plan_paged, P.mv_smem = 0)."""
    g = make_grid(448, 448)
    w, s = 96, 4
    ring = w + s
    S = 2
    rng = np.random.default_rng(21)
    mring, tring = _random_group_rings(g, S, ring, 16, rng)
    win = dict(window=w, stride=s, step=3, ring_frames=ring)
    cap = w * 256 + 32
    kv = dict(synth.TOY_KV, capacity=cap + 10, refresh_capacity=cap, n_prompt=32)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(4)
    shape = (kv["layers"], 2, cap + 10, kv["kv_heads"], kv["head_dim"])
    pools = [torch.randn(shape, generator=gen, device=DEV) for _ in range(S)]
    slot_old = np.stack([rng.permutation(cap + 10)[:cap] for _ in range(S)]).astype(np.int32)
    _, _, refr = make_caches(kv, S, gen)
    run_paged_both(abi, ref, g, kv, win, mring, tring, pools, slot_old, cap, refr, cap)


# ------------------------------------------------------------------------------------------------------------
# M-RoPE position correction (NEXT-3), both KV modes
# ------------------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [1, 0])
def test_mrope_gpu_both_modes(abi, ref, dtype):
    cfg = synth.CONFIGS["C1"]
    g = make_grid(448, 448)
    w, s, ring = 8, 2, 10
    cap = w * 256 + 32
    if dtype == 0:
        base = dict(synth.QWEN_MROPE_KV, layers=2)
    else:
        base = dict(synth.TOY_KV, rope_mode=1, mrope_section=(2, 3, 3), t_per_frame=3)
    kv = dict(base, capacity=cap, refresh_capacity=cap, n_prompt=32)
    S = 5
    gen = torch.Generator(device=DEV)
    gen.manual_seed(12)
    dt = torch.bfloat16 if dtype == 0 else torch.float32
    shape = (kv["layers"], 2, cap, kv["kv_heads"], kv["head_dim"])
    pools = [torch.randn(shape, generator=gen, device=DEV).to(dt) for _ in range(S)]
    _, keep = _rot_cols(kv)
    special = torch.tensor([-0.0, float("inf"), float("-inf"), float("nan")], device=DEV).to(dt)
    for t in pools:   # -0 / inf / NaN in the h / w sections must survive reuse bit for bit
        t[:, 0, :, :, keep[:4]] = special
    slot = None
    stats = {}
    for k in range(6):
        mring, tring = stream_rings(ref, g, cfg, S, ring, k, w, s)
        old, new, refr = make_caches(kv, S, gen)
        if k:
            for t in old:
                t[:, 0, :, :, keep[:4]] = special
        win = dict(window=w, stride=s, step=k, ring_frames=ring)
        gpu, o, new_h = run_kv_both(abi, ref, g, kv, win, mring, tring, old if k else None, new, refr, cap)
        assert_kv_equal(gpu, o, new, new_h, kv, stats)
        sn, _, st = run_paged_both(abi, ref, g, kv, win, mring, tring, pools, slot, cap, refr, cap)
        slot = sn
    kvcheck.assert_rotation_bits(stats)


# ------------------------------------------------------------------------------------------------------------
# fused preprocessing + compaction from NV12 (NEXT-2)
# ------------------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("geom", [(448, 448, 14, 2, 32, 32), (1920, 1080, 14, 2, 32, 32),
                                  (3840, 2160, 14, 2, 32, 32), (120, 90, 6, 2, 8, 6), (64, 48, 8, 2, 4, 4)])
@pytest.mark.parametrize("norm", ["clip", "odd", "exact"])
def test_compact_nv12(abi, ref, geom, norm):
    """norm: the CLIP mean/std; unusual stds on the guarded-reciprocal path (norm_bf16); a std outside
    [2^-20, 2^20], which takes the IEEE division for every pixel -- at every geometry, the 1080p / 4K ones on the
    staged kernel (pitches multiples of 16)."""
    sw, sh, p, G, gw, gh = geom
    mean, std = {"clip": (None, None), "odd": ((0.5, -0.25, 0.0), (0.0173, 3.7, 1.0)),
                 "exact": ((0.4815, 0.4578, 0.4082), (2.0 ** -21, 0.2613, 0.2758))}[norm]
    g = make_grid(sw, sh, patch=p, group=G, grid_w=gw, grid_h=gh)
    rng = np.random.default_rng(sw + sh)
    S, n = 2, 3
    nw = abi.grid_words(g)
    km = rng.integers(0, 2**32, size=(S, n, nw), dtype=np.uint64).astype(np.uint32)
    km &= rng.integers(0, 2**32, size=(S, n, nw), dtype=np.uint64).astype(np.uint32)
    pitch = sw + 64                                  # padded planes, as NVDEC allocates them
    ys = [rng.integers(16, 236, size=(sh, pitch), dtype=np.uint8) for _ in range(S * n)]
    uvs = [rng.integers(16, 241, size=(sh // 2, pitch), dtype=np.uint8) for _ in range(S * n)]
    pre_h = ref.make_pre(sw, sh, pitch, pitch) if mean is None else ref.make_pre(sw, sh, pitch, pitch, mean, std)
    pre = dict(src_w=sw, src_h=sh, y_pitch=pitch, uv_pitch=pitch)
    if mean is not None:
        pre.update(mean=mean, std=std)
    fidx = np.arange(S * n, dtype=np.int32) + 7
    for cap in (S * n * gw * gh, S * n * gw * gh // 3 + 1):
        y_d = [torch.from_numpy(a).to(DEV) for a in ys]
        uv_d = [torch.from_numpy(a).to(DEV) for a in uvs]
        km_d = torch.from_numpy(km.view(np.int32)).to(DEV)
        packed = torch.full((cap, 3 * p * p), -1, dtype=torch.int16, device=DEV)
        pos = torch.zeros(cap, 3, dtype=torch.int32, device=DEV)
        src = torch.zeros(cap, dtype=torch.int32, device=DEV)
        offs = torch.zeros(S * n + 1, dtype=torch.int32, device=DEV)
        cnt = torch.zeros(16, dtype=torch.int64, device=DEV)
        st = torch.zeros(1, dtype=torch.int32, device=DEV)
        abi.codecsight_compact_nv12(g, pre, S, n, km_d, n, torch.from_numpy(fidx).to(DEV), abi.ptr_array(y_d, DEV),
                                    abi.ptr_array(uv_d, DEV), cap, packed, pos, src, offs, cnt, st)
        o = ref.compact_nv12(g, pre_h, km, fidx, ys, uvs, cap, S, n)
        torch.cuda.synchronize()
        rows = min(int(o["frame_offsets"][-1]), cap)
        assert int(st.item()) == o["status"]
        assert (offs.cpu().numpy() == o["frame_offsets"]).all()
        assert (pos.cpu().numpy()[:rows] == o["pos_ids"][:rows]).all()
        assert (src.cpu().numpy()[:rows] == o["src_index"][:rows]).all()
        got = packed.cpu().numpy().view(np.uint16)[:rows]
        assert (got == o["packed"][:rows]).all(), int((got != o["packed"][:rows]).sum())
        assert (cnt.cpu().numpy().view(np.uint64) == o["counters"]).all()


@pytest.mark.parametrize("case", ["pitch8", "misaligned", "wide_span", "one_group", "ragged_cap"])
def test_compact_nv12_paths(abi, ref, case):
    """The launcher's NV12 paths beyond test_compact_nv12's: pitches that are not multiples of 16 (direct-load
    path), planes off 16-B alignment (staged path, byte-copied stages), a column span wider than 16 chunks (scale
    17: direct-load path), a batch with a single kept group (the staged ring's prologue / tail), and a capacity
    that ends inside a group."""
    sw, sh, gw, gh = 1920, 1080, 32, 32
    pitch = sw + 64
    if case == "pitch8":
        pitch = sw + 8
    if case == "wide_span":
        gw = gh = 8
    g = make_grid(sw, sh, patch=14, group=2, grid_w=gw, grid_h=gh)
    rng = np.random.default_rng(77)
    S, n = 2, 2
    nw = abi.grid_words(g)
    km = rng.integers(0, 2**32, size=(S, n, nw), dtype=np.uint64).astype(np.uint32)
    km &= rng.integers(0, 2**32, size=(S, n, nw), dtype=np.uint64).astype(np.uint32)
    if case == "one_group":
        km[:] = 0
        km[1, 1, 5] = 1 << 9
    off = 1 if case == "misaligned" else 0
    ys = [rng.integers(16, 236, size=(sh, pitch), dtype=np.uint8) for _ in range(S * n)]
    uvs = [rng.integers(16, 241, size=(sh // 2, pitch), dtype=np.uint8) for _ in range(S * n)]
    pre_h = ref.make_pre(sw, sh, pitch, pitch)
    pre = dict(src_w=sw, src_h=sh, y_pitch=pitch, uv_pitch=pitch)
    fidx = np.arange(S * n, dtype=np.int32) + 3
    cap = S * n * gw * gh if case != "ragged_cap" else 4 * 37 + 3
    # misaligned: each plane is a view 1 byte into its allocation
    y_d = [torch.from_numpy(np.concatenate([np.zeros(off, np.uint8), a.ravel()])).to(DEV)[off:] for a in ys]
    uv_d = [torch.from_numpy(np.concatenate([np.zeros(off, np.uint8), a.ravel()])).to(DEV)[off:] for a in uvs]
    if off:
        assert all(t.data_ptr() % 16 for t in y_d)
    km_d = torch.from_numpy(km.view(np.int32)).to(DEV)
    packed = torch.full((cap, 3 * 14 * 14), -1, dtype=torch.int16, device=DEV)
    pos = torch.zeros(cap, 3, dtype=torch.int32, device=DEV)
    src = torch.zeros(cap, dtype=torch.int32, device=DEV)
    offs = torch.zeros(S * n + 1, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(16, dtype=torch.int64, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    abi.codecsight_compact_nv12(g, pre, S, n, km_d, n, torch.from_numpy(fidx).to(DEV), abi.ptr_array(y_d, DEV),
                                abi.ptr_array(uv_d, DEV), cap, packed, pos, src, offs, cnt, st)
    o = ref.compact_nv12(g, pre_h, km, fidx, ys, uvs, cap, S, n)
    torch.cuda.synchronize()
    rows = min(int(o["frame_offsets"][-1]), cap)
    assert rows > 0
    assert int(st.item()) == o["status"]
    assert (offs.cpu().numpy() == o["frame_offsets"]).all()
    assert (pos.cpu().numpy()[:rows] == o["pos_ids"][:rows]).all()
    assert (src.cpu().numpy()[:rows] == o["src_index"][:rows]).all()
    got = packed.cpu().numpy().view(np.uint16)
    assert (got[:rows] == o["packed"][:rows]).all(), int((got[:rows] != o["packed"][:rows]).sum())
    assert (got[rows:] == 0xFFFF).all()   # nothing written past the packed rows / the capacity
    assert (cnt.cpu().numpy().view(np.uint64) == o["counters"]).all()


# ------------------------------------------------------------------------------------------------------------
# NEXT-4: AVMotionVector rasterisation and the similar-patch histogram
# ------------------------------------------------------------------------------------------------------------
def _random_avmv(ref, g, n_frames, rng, n_first=None):
    recs = []
    offs = [0]
    for f in range(n_frames):
        n = int(rng.integers(0, 3 * g["mb_rows"] * g["mb_cols"])) if (f or n_first is None) else n_first
        a = np.zeros(n, ref.AV_MV_DTYPE)
        a["source"] = rng.choice([-1, -1, -1, 1], size=n)
        a["w"] = rng.choice([4, 8, 16], size=n)
        a["h"] = rng.choice([4, 8, 16], size=n)
        a["dst_x"] = rng.integers(-8, g["src_w"] + 8, size=n)
        a["dst_y"] = rng.integers(-8, g["src_h"] + 8, size=n)
        a["motion_x"] = rng.integers(-40, 41, size=n)
        a["motion_y"] = rng.integers(-40, 41, size=n)
        a["motion_scale"] = rng.choice([1, 2, 4, 4, 4, 3, 8, 0], size=n)      # 4/2/1: shift path, else division
        big = rng.random(n) < 0.01
        a["motion_x"][big] = rng.integers(-40000, 40000, size=int(big.sum()))   # int16 clamp
        recs.append(a)
        offs.append(offs[-1] + n)
    return np.concatenate(recs), np.array(offs, np.int64)


@pytest.mark.parametrize("src", [(448, 448), (1920, 1080), (100, 60), (3840, 2160), (640, 360, 8), (500, 300, 12)])
def test_mv_rasterize_gpu(abi, ref, src):
    """Keys in shared memory (grids up to 12,288 MBs; 16-px MBs by shifts, other sizes by division; records past
    the ~20k whose vectors stay in shared memory decoded from global memory: 1080p's first frame has 24,479) and in
    global memory (4K: 32,400 MBs)."""
    g = make_grid(src[0], src[1], mb_size=src[2] if len(src) > 2 else 16)
    rng = np.random.default_rng(src[0])
    n = 1 if src[0] > 2000 else 5          # (the oracle's rasterisation is O(MBs x records) per frame)
    mvs, offs = _random_avmv(ref, g, n, rng, n_first=24479 if src == (1920, 1080) else None)
    out_d = torch.zeros(n * g["mb_rows"] * g["mb_cols"], dtype=torch.int64, device=DEV)
    abi.codecsight_mv_rasterize(g, n, torch.from_numpy(mvs.view(np.uint8)).to(DEV), torch.from_numpy(offs).to(DEV),
                                out_d)
    exp = ref.mv_rasterize(g, mvs, offs, n)
    torch.cuda.synchronize()
    got = out_d.cpu().numpy().view(MB_DTYPE).reshape(exp.shape)
    for f in ("mvx", "mvy", "sad", "type"):
        assert (got[f] == exp[f]).all(), f


def test_similar_hist_gpu(abi, ref):
    g = make_grid(1920, 1080)
    S, n = 8, 8
    mb = np.stack([synth.stream_metadata(1920, 1080, sc, 40 + i, n) for i, sc in
                   enumerate(["low", "medium", "high", "noise"] * 2)])
    types = np.stack([synth.frame_types(n, 16, 5)] * S)
    sc = ref.score_patches(g, mb, types, np.zeros((S, 33), np.uint32))["score"]
    taus = np.array([0.25, 0.5, 1.0, 2.0, 5.0], np.float32)
    hist_d = torch.zeros(5, 50, dtype=torch.int64, device=DEV)
    abi.codecsight_similar_hist(torch.from_numpy(sc.reshape(S * n, -1)).to(DEV),
                                torch.from_numpy(types.reshape(-1)).to(DEV), S * n, 1024,
                                torch.from_numpy(taus).to(DEV), 5, 50, hist_d)
    exp = ref.similar_hist(sc.reshape(S * n, -1), types.reshape(-1), taus, 50)
    torch.cuda.synchronize()
    assert (hist_d.cpu().numpy().view(np.uint64) == exp).all()


def test_cdf_workload_pipeline(abi, ref):
    """NEXT-4 workload as bench.py --workload cdf runs it: H.264-shaped AVMotionVector exports (synth.avmv_records)
    of whole GOPs -> mv_rasterize -> score_patches (scores out) -> similar_hist over 5 taus, against the oracle
    driven the same way: MB grids, scores, masks and the histogram bit-exact."""
    import bench_cdf
    cfg = dict(synth.CONFIGS["CDF"], tau=0.25, alpha=0.0, group=2)
    g = make_grid(*cfg["src"])
    S, F = 3, cfg["window"]
    gens = [synth.StreamGen(*cfg["src"], synth.scene_of(cfg, i), synth.stream_seed(cfg, i)) for i in range(S)]
    recs, offs, types = bench_cdf.gen_step(cfg, gens, np.random.default_rng(1))
    n = S * F
    nmb = g["mb_rows"] * g["mb_cols"]
    grid_d = torch.zeros(n * nmb, dtype=torch.int64, device=DEV)
    abi.codecsight_mv_rasterize(g, n, torch.from_numpy(recs.view(np.uint8)).to(DEV), torch.from_numpy(offs).to(DEV),
                                grid_d)
    gop = torch.zeros(S, 33, dtype=torch.int32, device=DEV)
    keep = torch.zeros(S, F, 32, dtype=torch.int32, device=DEV)
    score = torch.zeros(n, 1024, dtype=torch.float32, device=DEV)
    kept = torch.zeros(S, F, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(16, dtype=torch.int64, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    ty_d = torch.from_numpy(types).to(DEV)
    abi.codecsight_score_patches(g, S, F, grid_d, ty_d, keep, F, gop, score, kept, cnt, st)
    taus = np.array(cfg["taus"], np.float32)
    hist = torch.zeros(len(taus), cfg["n_bins"], dtype=torch.int64, device=DEV)
    abi.codecsight_similar_hist(score, ty_d, n, 1024, torch.from_numpy(taus).to(DEV), len(taus), cfg["n_bins"], hist)
    grid_o = ref.mv_rasterize(g, recs, offs, n)
    so = ref.score_patches(g, grid_o.reshape(S, F, g["mb_rows"], g["mb_cols"]), types, np.zeros((S, 33), np.uint32),
                           want_score=True)
    ho = ref.similar_hist(so["score"].reshape(n, -1), types.reshape(-1), taus, cfg["n_bins"])
    torch.cuda.synchronize()
    got = grid_d.cpu().numpy().view(MB_DTYPE).reshape(grid_o.shape)
    p = types.reshape(-1) == synth.FRAME_P
    for f in ("mvx", "mvy", "sad", "type"):
        assert (got[p][f] == grid_o[p][f]).all(), f
    assert (score.cpu().numpy().view(np.uint32)[p] == so["score"].reshape(n, -1).view(np.uint32)[p]).all()
    assert (u32(keep).reshape(S, F, -1) == so["keep_mask"]).all()
    assert (hist.cpu().numpy().astype(np.uint64) == ho).all()
    assert int(st.item()) == so["status"] == 0
    assert ho.sum() == len(taus) * p.sum()


def test_pipeline_pdl_matches_plain(abi, ref):
    """Prune-only (C2-shaped) pipeline with programmatic dependent launches (CS_LAUNCH_PDL): 10 steps enqueued back
    to back with no host synchronisation and no stream operation between the fused launches, so each step's stream
    ticket, MB loads and scoring passes really overlap the previous step's compaction.  Final GOP state, every mask
    of the ring, counters, status and the last step's outputs must equal the plain fused pipeline's (itself
    parity-tested against the oracle), and the last step's outputs the oracle's."""
    from paper_2604_06036_b200.pipeline import Pipeline
    cfg = synth.CONFIGS["C2"]
    g = make_grid(1920, 1080)
    S, w, s, gop, K = 12, 16, 4, 16, 10
    rng = np.random.default_rng(8)
    frames_h = [to_grouped(f, g) for f in synth.random_frames(S * s, 448, 448, rng)]
    frames_d = [torch.from_numpy(f.view(np.int16)).to(DEV) for f in frames_h]
    gens = [synth.StreamGen(1920, 1080, synth.scene_of(cfg, si), synth.stream_seed(cfg, si)) for si in range(S)]
    inputs, host = [], []
    for k in range(K):
        f0, n = (0, w) if k == 0 else ((k - 1) * s + w, s)
        mb = np.stack([np.stack([gens[si].next_frame() for _ in range(n)]) for si in range(S)])
        types = np.stack([synth.frame_types(n, gop, f0) for _ in range(S)])
        fidx = np.tile(np.arange(f0, f0 + n, dtype=np.int32), S)
        ptrs = abi.ptr_array([frames_d[i % len(frames_d)] for i in range(S * n)], DEV)
        inputs.append((d_mb(mb), ptrs, torch.from_numpy(fidx).to(DEV), torch.from_numpy(types).to(DEV)))
        host.append((mb, types, fidx))
    runs = {}
    for pdl in (False, True):
        pipe = Pipeline(g, S, w, s, gop, None, device=DEV, frame_layout=abi.CS_LAYOUT_GROUPED, fused=True, pdl=pdl)
        torch.cuda.synchronize()
        for k in range(K):
            pipe.step(k, *inputs[k])
        torch.cuda.synchronize()
        n = s
        tot = int(pipe.frame_offsets[S * n].item())
        runs[pdl] = dict(gop=u32(pipe.gop_state), ring=u32(pipe.mask_ring), counters=pipe.counters.cpu().numpy(),
                         status=int(pipe.status.item()), kept=pipe.kept_counts(n).cpu().numpy(),
                         offs=pipe.frame_offsets[:S * n + 1].cpu().numpy(),
                         packed=pipe.packed[:tot].view(torch.int16).cpu().numpy().view(np.uint16),
                         pos=pipe.pos_ids[:tot].cpu().numpy(), src=pipe.src_index[:tot].cpu().numpy())
        del pipe
    a, b = runs[False], runs[True]
    assert a["status"] == b["status"] == 0
    for key in ("gop", "ring", "counters", "kept", "offs", "packed", "pos", "src"):
        assert (a[key] == b[key]).all(), key
    # the last step against the oracle (the GOP state carried through all K steps)
    ring = w + s
    gop_h = np.zeros((S, 33), np.uint32)
    mring_h = np.zeros((S, ring, 32), np.uint32)
    tring_h = np.zeros((S, ring), np.uint8)
    for k in range(K):
        mb, types, fidx = host[k]
        f0, n = (0, w) if k == 0 else ((k - 1) * s + w, s)
        off = f0 % ring
        tring_h[:, off:off + n] = types
        so = ref.score_patches(g, mb, np.ascontiguousarray(tring_h[:, off:]), gop_h, want_score=False,
                               frame_stride=ring - off)
        mring_h[:, off:off + n] = so["keep_mask"][:, :n]
    assert (b["gop"] == gop_h).all() and (b["ring"] == mring_h).all()
    fr = [frames_h[i % len(frames_h)] for i in range(S * s)]
    co = ref.compact(g, mring_h[:, off:].copy(), fidx, fr, S * s * 1024, S, s, mask_frame_stride=ring - off,
                     frame_layout=1)
    assert (b["offs"] == co["frame_offsets"]).all()
    tot = int(co["frame_offsets"][-1])
    assert (b["packed"] == co["packed"][:tot]).all() and (b["pos"] == co["pos_ids"][:tot]).all()


@pytest.mark.parametrize("seed", list(range(24)))
def test_compact_nv12_random_geometries(abi, ref, seed):
    """The staged NV12 kernel over random geometries: source sizes from upscaling to ~8x downscaling (staged row
    pitch 144 or 256 B, spans that end at the plane's right edge), random grids of 2x2 groups of 14-px patches,
    pitches with and without 16-B multiples (staged vs direct path), random keep masks and capacities."""
    rng = np.random.default_rng(1000 + seed)
    gw, gh = int(rng.integers(2, 17)) * 2, int(rng.integers(2, 17)) * 2
    sw = int(rng.integers(16, 1921)) * 2
    sh = int(rng.integers(16, 1081)) * 2
    if sw > 8.4 * gw * 14:          # keep within the staged path's widest span (or it takes the direct path)
        sw = int(8.4 * gw * 14) // 2 * 2
    pitch = sw + int(rng.choice([0, 16, 48, 8, 2]))
    pitch += pitch % 2
    g = make_grid(sw, sh, patch=14, group=2, grid_w=gw, grid_h=gh)
    S, n = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    nw = abi.grid_words(g)
    km = rng.integers(0, 2**32, size=(S, n, nw), dtype=np.uint64).astype(np.uint32)
    km &= rng.integers(0, 2**32, size=(S, n, nw), dtype=np.uint64).astype(np.uint32)
    ys = [rng.integers(0, 256, size=(sh, pitch), dtype=np.uint8) for _ in range(S * n)]
    uvs = [rng.integers(0, 256, size=(sh // 2, pitch), dtype=np.uint8) for _ in range(S * n)]
    pre_h = ref.make_pre(sw, sh, pitch, pitch)
    pre = dict(src_w=sw, src_h=sh, y_pitch=pitch, uv_pitch=pitch)
    fidx = np.arange(S * n, dtype=np.int32)
    total = S * n * gw * gh
    cap = int(rng.choice([total, max(1, total // 2 + 1), 3]))
    y_d = [torch.from_numpy(a).to(DEV) for a in ys]
    uv_d = [torch.from_numpy(a).to(DEV) for a in uvs]
    km_d = torch.from_numpy(km.view(np.int32)).to(DEV)
    packed = torch.full((cap, 3 * 14 * 14), -1, dtype=torch.int16, device=DEV)
    pos = torch.zeros(cap, 3, dtype=torch.int32, device=DEV)
    src = torch.zeros(cap, dtype=torch.int32, device=DEV)
    offs = torch.zeros(S * n + 1, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(16, dtype=torch.int64, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    abi.codecsight_compact_nv12(g, pre, S, n, km_d, n, torch.from_numpy(fidx).to(DEV), abi.ptr_array(y_d, DEV),
                                abi.ptr_array(uv_d, DEV), cap, packed, pos, src, offs, cnt, st)
    o = ref.compact_nv12(g, pre_h, km, fidx, ys, uvs, cap, S, n)
    torch.cuda.synchronize()
    rows = min(int(o["frame_offsets"][-1]), cap)
    assert int(st.item()) == o["status"]
    assert (offs.cpu().numpy() == o["frame_offsets"]).all()
    assert (pos.cpu().numpy()[:rows] == o["pos_ids"][:rows]).all()
    assert (src.cpu().numpy()[:rows] == o["src_index"][:rows]).all()
    got = packed.cpu().numpy().view(np.uint16)
    assert (got[:rows] == o["packed"][:rows]).all(), (sw, sh, gw, gh, pitch, int((got[:rows] != o["packed"][:rows]).sum()))
    assert (got[rows:] == 0xFFFF).all()
    assert (cnt.cpu().numpy().view(np.uint64) == o["counters"]).all()
