"""The C-ABI library loads and exports every symbol include/codecsight.h declares; host-side validation
returns the documented codes without launching anything (no GPU needed)."""
import ctypes as C

import pytest
import torch

from synth import make_grid


@pytest.fixture(scope="module")
def abi():
    import __graft_entry__ as ge
    ge.build_cuda()
    from paper_2604_06036_b200 import _abi
    _abi.lib()
    return _abi


def test_exports_every_declared_symbol(abi):
    syms = abi.declared_symbols()
    assert set(syms) >= {"codecsight_score_patches", "codecsight_compact", "codecsight_kv_refresh"}
    for s in syms:
        assert hasattr(abi.lib(), s), s
    assert abi.lib().codecsight_version() == 100
    assert abi.lib().codecsight_strerror(-2) == b"shape / dimension mismatch"


def test_sm100a_cubin_only(abi):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_keeps_the_bulk_copy_pipelines(abi):
    """The hot kernels move data with Blackwell bulk copies behind mbarriers: the KV gather's per-warp
    TMA rings, the fused score+compact's MB ring and group ring, the grouped compaction's ring.  A change that
    silently falls back to register copies fails here (evidence: profiles/r02_sass.txt)."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    import sass_summary
    ks = sass_summary.parse(abi.LIB_PATH)
    need = {"void kv_gather_tma<unsigned short, 4, 128>": (1, 1), "void kv_gather_tma<float, 0, 0>": (1, 1),
            "void score_kernel<true>": (1, 1), "void score_kernel<false>": (1, 0), "compact_gather_tma": (1, 1)}
    for name, (g2s, s2g) in need.items():
        v = ks[name]
        assert v["UBLKCP.S.G"] >= g2s and v["UBLKCP.G.S"] >= s2g and v["SYNCS"] >= 1, (name, v)
        if name != "void score_kernel<false>":     # (the unfused score kernel is off the default path)
            assert v["stack"] == 0, (name, v)      # no local-memory spills in the hot kernels
    assert ks["compact_gather_band"]["LDGSTS"] >= 1 and ks["compact_gather_band"]["stack"] == 0  # planar: cp.async
    for rb in (144, 256):  # fused NV12 preprocessing: source rows staged with cp.async, no spills
        v = ks["void compact_nv12_staged<%d>" % rb]
        assert v["LDGSTS"] >= 2 and v["stack"] == 0 and v["local"] == 0, (rb, v)


FAKE = 0x1000  # never dereferenced: validation fails (or the device check does) before any launch


def _score(abi, g, n_streams=1, n_frames=2, frame_stride=2, mb=FAKE):
    L = abi.lib()
    return L.codecsight_score_patches(C.byref(abi.make_grid(g)), n_streams, n_frames, mb, FAKE, FAKE, frame_stride,
                                      FAKE, None, FAKE, FAKE, FAKE, None)


def test_score_validation(abi):
    g = make_grid(1920, 1080)
    assert _score(abi, dict(g, mb_rows=67)) == abi.CS_ERR_SHAPE          # coded grid must be ceil(src/16)
    assert _score(abi, dict(g, group=3)) == abi.CS_ERR_SHAPE             # group must divide the grid
    assert _score(abi, dict(g, tau=float("nan"))) == abi.CS_ERR_INVALID_ARGUMENT
    assert _score(abi, dict(g, alpha=-1.0)) == abi.CS_ERR_INVALID_ARGUMENT
    assert _score(abi, g, n_frames=0) == abi.CS_ERR_INVALID_ARGUMENT
    assert _score(abi, g, frame_stride=1) == abi.CS_ERR_INVALID_ARGUMENT
    assert _score(abi, g, n_streams=0) == abi.CS_OK                      # empty batch: nothing to do
    assert _score(abi, g, mb=FAKE + 4) == abi.CS_ERR_INVALID_ARGUMENT    # 8-B aligned records
    assert _score(abi, dict(g, grid_w=128, grid_h=64)) == abi.CS_ERR_SHAPE
    if not torch.cuda.is_available():
        assert _score(abi, g) == abi.CS_ERR_CUDA                          # no CPU fallback


def test_kv_validation(abi):
    L = abi.lib()
    g = make_grid(448, 448)

    def call(kv, win, ws_bytes=1 << 20, n_streams=1):
        return L.codecsight_kv_refresh(C.byref(abi.make_grid(g)), C.byref(abi.make_kv(kv)),
                                       C.byref(abi.make_window(win)), n_streams, FAKE, FAKE, FAKE, FAKE, None, 16,
                                       FAKE, FAKE, FAKE, FAKE, ws_bytes, FAKE, FAKE, None)

    kv = dict(layers=2, kv_heads=2, head_dim=16, dtype=1, capacity=64, refresh_capacity=64, rope_base=1e4,
              n_prompt=0)
    win = dict(window=8, stride=2, step=1, ring_frames=10)
    assert call(dict(kv, head_dim=15), win) == abi.CS_ERR_UNSUPPORTED    # odd head_dim
    assert call(dict(kv, dtype=7), win) == abi.CS_ERR_UNSUPPORTED
    assert call(kv, dict(win, stride=9, ring_frames=17)) == abi.CS_ERR_UNSUPPORTED   # s > w
    assert call(kv, dict(win, ring_frames=9)) == abi.CS_ERR_SHAPE        # ring < w + s
    assert call(kv, dict(win, step=0, ring_frames=8)) != abi.CS_ERR_SHAPE
    assert call(kv, win, ws_bytes=8) == abi.CS_ERR_INVALID_ARGUMENT      # workspace too small
    assert call(kv, win, n_streams=0) == abi.CS_OK
    assert call(dict(kv, rope_base=0.0), win) == abi.CS_ERR_INVALID_ARGUMENT
    ws = abi.kv_workspace_size(kv, win, 3)
    assert ws >= 16 + 3 * (16 + 9 * 16 + 8 * 8)


def test_compact_validation(abi):
    L = abi.lib()
    g = make_grid(448, 448)

    def call(g, cap=16, n_streams=1, n_frames=1, mfs=1, layout=0):
        return L.codecsight_compact(C.byref(abi.make_grid(g)), n_streams, n_frames, FAKE, mfs, FAKE, FAKE, layout,
                                    cap, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, None)

    assert call(g, cap=-1) == abi.CS_ERR_INVALID_ARGUMENT
    assert call(g, layout=2) == abi.CS_ERR_INVALID_ARGUMENT
    assert call(g, mfs=0) == abi.CS_ERR_INVALID_ARGUMENT
    assert call(dict(g, patch=40)) == abi.CS_ERR_SHAPE
    assert call(dict(g, patch=20)) == abi.CS_ERR_UNSUPPORTED     # group * patch > 32
    assert call(g, n_streams=1 << 20, n_frames=4096, mfs=4096) == abi.CS_ERR_UNSUPPORTED   # int32 offsets


def test_extension_validation(abi):
    """Argument checks of the extension entry points happen on the host, before any device work."""
    L = abi.lib()
    g = make_grid(448, 448)
    G = C.byref(abi.make_grid(g))
    nocuda = not torch.cuda.is_available()
    # fused score + compact (NEXT-2)
    ws_need = abi.score_compact_workspace_size(4)
    assert ws_need == 16 + 8 * 4

    def sc(n_streams=4, n_frames=2, fs=2, layout=1, cap=16, ws=FAKE, ws_bytes=1 << 10, mb=FAKE):
        return L.codecsight_score_compact(G, n_streams, n_frames, mb, FAKE, FAKE, fs, FAKE, None, FAKE, FAKE, FAKE,
                                          layout, cap, FAKE, FAKE, FAKE, FAKE, ws, ws_bytes, FAKE, FAKE, None)
    assert sc(ws_bytes=ws_need - 1) == abi.CS_ERR_INVALID_ARGUMENT        # workspace too small
    assert sc(ws=None) == abi.CS_ERR_INVALID_ARGUMENT
    assert sc(layout=3) == abi.CS_ERR_INVALID_ARGUMENT
    assert sc(fs=1) == abi.CS_ERR_INVALID_ARGUMENT                        # frame stride < n_frames
    assert sc(mb=FAKE + 2) == abi.CS_ERR_INVALID_ARGUMENT                  # 8-B aligned records
    assert sc(n_streams=0) == abi.CS_OK
    if nocuda:
        assert sc() == abi.CS_ERR_CUDA                                     # no CPU fallback

    # the extended call: type stride, chained launches (CS_LAUNCH_PDL needs a valid chain, no score output)
    def sce(flags=0, chain=None, ts=2, score=None):
        return L.codecsight_score_compact_ex(G, 4, 2, FAKE, FAKE, ts, FAKE, 2, FAKE, score, FAKE, FAKE, FAKE, 1, 16,
                                             FAKE, FAKE, FAKE, FAKE, FAKE, 1 << 10, FAKE, FAKE, flags, chain, None)
    good = abi.CsChain(FAKE, FAKE, 0, 4)
    assert sce(ts=1) == abi.CS_ERR_INVALID_ARGUMENT                        # type stride < n_frames
    assert sce(flags=2) == abi.CS_ERR_INVALID_ARGUMENT                     # unknown flag
    assert sce(flags=abi.CS_LAUNCH_PDL) == abi.CS_ERR_INVALID_ARGUMENT     # PDL without a chain
    for bad in (abi.CsChain(None, FAKE, 0, 4), abi.CsChain(FAKE, None, 0, 4), abi.CsChain(FAKE, FAKE, 0, 1),
                abi.CsChain(FAKE, FAKE, 0, 9)):
        assert sce(flags=abi.CS_LAUNCH_PDL, chain=C.byref(bad)) == abi.CS_ERR_INVALID_ARGUMENT
    assert sce(flags=abi.CS_LAUNCH_PDL, chain=C.byref(good), score=FAKE) == abi.CS_ERR_UNSUPPORTED
    if nocuda:
        assert sce(flags=abi.CS_LAUNCH_PDL, chain=C.byref(good)) == abi.CS_ERR_CUDA
    # temporal patches (NEXT-3)

    def tp(t=2, n_units=2, mfs=4, cap=16, um=None, ums=0, ft=None, ut=None):
        return L.codecsight_compact_tp(G, t, 1, n_units, FAKE, mfs, FAKE, FAKE, 0, cap, FAKE, FAKE, FAKE, FAKE, um,
                                       ums, ft, ut, FAKE, FAKE, None)
    assert tp(t=0) == abi.CS_ERR_UNSUPPORTED and tp(t=5) == abi.CS_ERR_UNSUPPORTED
    assert tp(mfs=3) == abi.CS_ERR_INVALID_ARGUMENT                        # n_units * tp frames needed
    assert tp(um=FAKE, ums=1) == abi.CS_ERR_INVALID_ARGUMENT               # unit mask stride < n_units
    assert tp(ft=FAKE) == abi.CS_ERR_INVALID_ARGUMENT                      # frame_type needs unit_type
    if nocuda:
        assert tp(um=FAKE, ums=2, ft=FAKE, ut=FAKE) == abi.CS_ERR_CUDA
    # MV rasterisation / similar histogram (NEXT-4)
    assert L.codecsight_mv_rasterize(G, -1, FAKE, FAKE, FAKE, None) == abi.CS_ERR_INVALID_ARGUMENT
    assert L.codecsight_mv_rasterize(G, 0, None, None, None, None) == abi.CS_OK
    assert L.codecsight_mv_rasterize(G, 2, FAKE, FAKE, FAKE + 4, None) == abi.CS_ERR_INVALID_ARGUMENT  # 8-B out
    assert L.codecsight_similar_hist(FAKE, FAKE, 4, 1024, FAKE, 0, 10, FAKE, None) == abi.CS_ERR_INVALID_ARGUMENT
    assert L.codecsight_similar_hist(FAKE, FAKE, 4, 1024, FAKE, 2, 0, FAKE, None) == abi.CS_ERR_INVALID_ARGUMENT
    assert L.codecsight_similar_hist(None, None, 0, 1024, None, 2, 10, None, None) == abi.CS_OK
    if nocuda:
        assert L.codecsight_mv_rasterize(G, 2, FAKE, FAKE, FAKE, None) == abi.CS_ERR_CUDA
        assert L.codecsight_similar_hist(FAKE, FAKE, 4, 1024, FAKE, 2, 10, FAKE, None) == abi.CS_ERR_CUDA


def test_nv12_validation(abi):
    L = abi.lib()
    G = C.byref(abi.make_grid(make_grid(1920, 1080)))

    def nv(**kw):
        pre = dict(dict(src_w=1920, src_h=1080), **kw)
        return L.codecsight_compact_nv12(G, C.byref(abi.make_preprocess(pre)), 1, 2, FAKE, 2, FAKE, FAKE, FAKE, 16,
                                         FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, None)
    assert nv(src_w=1921) == abi.CS_ERR_SHAPE                  # 4:2:0 needs even sizes
    assert nv(y_pitch=1900) == abi.CS_ERR_SHAPE                # pitch < width
    assert nv(color=1) == abi.CS_ERR_UNSUPPORTED
    assert nv(std=(0.2, 0.0, 0.2)) == abi.CS_ERR_INVALID_ARGUMENT
    assert nv(mean=(float("nan"), 0.4, 0.4)) == abi.CS_ERR_INVALID_ARGUMENT
    if not torch.cuda.is_available():
        assert nv() == abi.CS_ERR_CUDA
