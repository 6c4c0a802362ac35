"""ctypes binding of the C oracle ``oracle/libcodecsight_ref.so`` (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / ``--impl reference``) may import
this module.  It shares no code with the CUDA path: its ctypes structs are declared here, independently of
``paper_2604_06036_b200``.  All buffers are host numpy arrays.

The arithmetic lives in ``oracle/codecsight_ref.c``; this file only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcodecsight_ref.so")
SRC_PATH = os.path.join(HERE, "codecsight_ref.c")

MB_DTYPE = np.dtype([("mvx", "<i2"), ("mvy", "<i2"), ("sad", "<u2"), ("type", "u1"), ("rsv", "u1")])
assert MB_DTYPE.itemsize == 8

NCOUNTERS = 16
C_FRAMES, C_PFRAMES, C_PATCHES, C_KEPT, C_NEAR_TAU = 0, 1, 2, 3, 4
C_TOK_REUSE, C_TOK_ANCHOR, C_TOK_NEW = 5, 6, 7
C_BYTES_SCORE, C_BYTES_COMPACT, C_BYTES_KV, C_PACKED_ROWS, C_STREAM_STEPS = 8, 9, 10, 11, 12
DISP_NEW, DISP_ANCHOR, DISP_REUSE = 0, 1, 2
ST_CAPACITY, ST_NO_IFRAME, ST_ORIGIN, ST_BAD_FRAME_TYPE, ST_BAD_MB_TYPE = 1, 2, 4, 8, 16


class RefGrid(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("src_w", "src_h", "mb_size", "mb_cols", "mb_rows", "patch",
                                          "grid_w", "grid_h", "group")] + [("tau", C.c_float), ("alpha", C.c_float)]


class RefKv(C.Structure):
    _fields_ = [("layers", C.c_int32), ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("dtype", C.c_int32),
                ("capacity", C.c_int64), ("refresh_capacity", C.c_int64), ("rope_base", C.c_double),
                ("n_prompt", C.c_int32), ("rope_mode", C.c_int32), ("mrope_section", C.c_int32 * 3),
                ("t_per_frame", C.c_int32)]


class RefPre(C.Structure):
    _fields_ = [("src_w", C.c_int32), ("src_h", C.c_int32), ("y_pitch", C.c_int32), ("uv_pitch", C.c_int32),
                ("color", C.c_int32), ("mean", C.c_float * 3), ("stdv", C.c_float * 3)]


CLIP_MEAN = (0.48145466, 0.4578275, 0.40821073)   # Qwen2-VL / CLIP image normalisation
CLIP_STD = (0.26862954, 0.26130258, 0.27577711)


def make_pre(src_w, src_h, y_pitch=None, uv_pitch=None, mean=CLIP_MEAN, std=CLIP_STD, color=0) -> RefPre:
    return RefPre(src_w, src_h, y_pitch or src_w, uv_pitch or src_w, color, (C.c_float * 3)(*mean),
                  (C.c_float * 3)(*std))


class RefWindow(C.Structure):
    _fields_ = [("window", C.c_int32), ("stride", C.c_int32), ("step", C.c_int32), ("ring_frames", C.c_int32)]


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no FMA contraction, no vector intrinsics)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-Wall", "-fPIC", "-shared",
                               "-o", LIB_PATH, SRC_PATH, "-lm"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.codecsight_ref_mb_magnitude.restype = C.c_float
        L.codecsight_ref_mb_magnitude.argtypes = [C.c_int16, C.c_int16, C.c_uint8]
        L.codecsight_ref_patch_fields.restype = None
        L.codecsight_ref_patch_fields.argtypes = [C.POINTER(RefGrid), P, P, P, P, P]
        L.codecsight_ref_score_patches.restype = C.c_int
        L.codecsight_ref_score_patches.argtypes = [C.POINTER(RefGrid), C.c_int32, C.c_int32, P, P, P, C.c_int64,
                                                   P, P, P, P, P]
        L.codecsight_ref_compact.restype = C.c_int
        L.codecsight_ref_compact.argtypes = [C.POINTER(RefGrid), C.c_int32, C.c_int32, P, C.c_int64, P, P,
                                             C.c_int32, C.c_int64, P, P, P, P, P, P]
        L.codecsight_ref_compact_tp.restype = C.c_int
        L.codecsight_ref_compact_tp.argtypes = [C.POINTER(RefGrid), C.c_int32, C.c_int32, C.c_int32, P, C.c_int64, P,
                                                P, C.c_int32, C.c_int64, P, P, P, P, P, C.c_int64, P, P, P, P]
        L.codecsight_ref_kv_refresh.restype = C.c_int
        L.codecsight_ref_kv_refresh.argtypes = [C.POINTER(RefGrid), C.POINTER(RefKv), C.POINTER(RefWindow),
                                                C.c_int32, P, P, P, P, P, C.c_int64, P, P, P, P, P]
        L.codecsight_ref_kv_refresh_paged.restype = C.c_int
        L.codecsight_ref_kv_refresh_paged.argtypes = [C.POINTER(RefGrid), C.POINTER(RefKv), C.POINTER(RefWindow),
                                                      C.c_int32, P, P, P, P, P, C.c_int64, P, C.c_int64, P, P, P,
                                                      P, P]
        L.codecsight_ref_nv12_rgb.restype = None
        L.codecsight_ref_nv12_rgb.argtypes = [P, P, C.POINTER(RefPre), C.c_int64, C.c_int64, P]
        L.codecsight_ref_model_pixel.restype = C.c_float
        L.codecsight_ref_model_pixel.argtypes = [C.POINTER(RefGrid), C.POINTER(RefPre), P, P, C.c_int64, C.c_int64,
                                                 C.c_int64]
        L.codecsight_ref_preprocess_frame.restype = None
        L.codecsight_ref_preprocess_frame.argtypes = [C.POINTER(RefGrid), C.POINTER(RefPre), P, P, P]
        L.codecsight_ref_compact_nv12.restype = C.c_int
        L.codecsight_ref_compact_nv12.argtypes = [C.POINTER(RefGrid), C.POINTER(RefPre), C.c_int32, C.c_int32, P,
                                                  C.c_int64, P, P, P, C.c_int64, P, P, P, P, P, P]
        L.codecsight_ref_mv_rasterize.restype = C.c_int
        L.codecsight_ref_mv_rasterize.argtypes = [C.POINTER(RefGrid), C.c_int32, P, P, P]
        L.codecsight_ref_similar_hist.restype = C.c_int
        L.codecsight_ref_similar_hist.argtypes = [P, P, C.c_int64, C.c_int32, P, C.c_int32, C.c_int32, P]
        L.codecsight_ref_rope_rotate_f32.restype = None
        L.codecsight_ref_rope_rotate_f32.argtypes = [P, C.c_int32, C.c_int32, C.c_double, C.c_int64, P]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def make_grid(g: dict) -> RefGrid:
    return RefGrid(g["src_w"], g["src_h"], g["mb_size"], g["mb_cols"], g["mb_rows"], g["patch"], g["grid_w"],
                   g["grid_h"], g["group"], g["tau"], g["alpha"])


def grid_words(g: dict) -> int:
    return (g["grid_w"] * g["grid_h"] + 31) // 32


def mb_magnitude(dx: int, dy: int, mb_type: int = 0) -> np.float32:
    return np.float32(lib().codecsight_ref_mb_magnitude(dx, dy, mb_type))


def patch_fields(g: dict, mb2d: np.ndarray):
    """V, R, M ([grid_h, grid_w] fp32 each) of one P-frame's [mb_rows, mb_cols] MB records."""
    mb2d = np.ascontiguousarray(mb2d, dtype=MB_DTYPE)
    assert mb2d.shape == (g["mb_rows"], g["mb_cols"])
    V = np.zeros(g["grid_h"] * g["grid_w"], np.float32)
    R = np.zeros_like(V)
    M = np.zeros_like(V)
    st = np.zeros(1, np.int32)
    lib().codecsight_ref_patch_fields(C.byref(make_grid(g)), _p(mb2d), _p(V), _p(R), _p(M), _p(st))
    shp = (g["grid_h"], g["grid_w"])
    return V.reshape(shp), R.reshape(shp), M.reshape(shp), int(st[0])


def score_patches(g: dict, mb: np.ndarray, frame_type: np.ndarray, gop_state: np.ndarray,
                  keep_mask: np.ndarray | None = None, frame_stride: int | None = None, want_score: bool = True,
                  counters: np.ndarray | None = None, status: np.ndarray | None = None):
    """mb [S][n][mb_rows][mb_cols]; frame_type [S][frame_stride]; gop_state [S][words+1] (updated in place).

    Returns dict(keep_mask [S][frame_stride][words], kept_count [S][n], score [S][n][np] or None, counters,
    status, rc).  When ``keep_mask`` is given it is written in place (slot addressing as in the ABI)."""
    S, n = mb.shape[0], mb.shape[1]
    nw = grid_words(g)
    fs = n if frame_stride is None else frame_stride
    mb = np.ascontiguousarray(mb, dtype=MB_DTYPE)
    frame_type = np.ascontiguousarray(frame_type, dtype=np.uint8)
    assert frame_type.shape == (S, fs), frame_type.shape
    assert gop_state.dtype == np.uint32 and gop_state.flags.c_contiguous and gop_state.shape == (S, nw + 1)
    if keep_mask is None:
        keep_mask = np.zeros((S, fs, nw), np.uint32)
    score = np.zeros((S, n, g["grid_h"] * g["grid_w"]), np.float32) if want_score else None
    kept = np.zeros((S, n), np.int32)
    counters = np.zeros(NCOUNTERS, np.uint64) if counters is None else counters
    status = np.zeros(1, np.int32) if status is None else status
    rc = lib().codecsight_ref_score_patches(C.byref(make_grid(g)), S, n, _p(mb), _p(frame_type), _p(keep_mask), fs,
                                            _p(gop_state), _p(score), _p(kept), _p(counters), _p(status))
    return dict(rc=rc, keep_mask=keep_mask, kept_count=kept, score=score, counters=counters, status=int(status[0]))


def compact(g: dict, keep_mask: np.ndarray, frame_index: np.ndarray, frames: list, capacity: int,
            n_streams: int, n_frames: int, mask_frame_stride: int | None = None,
            counters: np.ndarray | None = None, frame_layout: int = 0):
    """keep_mask [S][mask_frame_stride][words]; frames: list of n_slots uint16 arrays (bf16 bits) in
    ``frame_layout`` (0 planar [3][H][W], 1 grouped [groups][group^2][3][p][p])."""
    nw = grid_words(g)
    mfs = n_frames if mask_frame_stride is None else mask_frame_stride
    keep_mask = np.ascontiguousarray(keep_mask, dtype=np.uint32).reshape(n_streams, mfs, nw)
    n_slots = n_streams * n_frames
    frame_index = np.ascontiguousarray(frame_index, dtype=np.int32).reshape(n_slots)
    frames = [np.ascontiguousarray(f, dtype=np.uint16) for f in frames]
    assert len(frames) == n_slots
    ptrs = (C.c_void_p * max(1, n_slots))(*[f.ctypes.data for f in frames])
    row = 3 * g["patch"] * g["patch"]
    packed = np.zeros((max(capacity, 0), row), np.uint16)
    pos = np.zeros((max(capacity, 0), 3), np.int32)
    src = np.zeros(max(capacity, 0), np.int32)
    offs = np.zeros(n_slots + 1, np.int32)
    counters = np.zeros(NCOUNTERS, np.uint64) if counters is None else counters
    status = np.zeros(1, np.int32)
    rc = lib().codecsight_ref_compact(C.byref(make_grid(g)), n_streams, n_frames, _p(keep_mask), mfs,
                                      _p(frame_index), C.cast(ptrs, C.c_void_p), frame_layout, capacity, _p(packed),
                                      _p(pos),
                                      _p(src), _p(offs), _p(counters), _p(status))
    return dict(rc=rc, packed=packed, pos_ids=pos, src_index=src, frame_offsets=offs, counters=counters,
                status=int(status[0]))


def compact_tp(g: dict, tp: int, keep_mask: np.ndarray, unit_index: np.ndarray, frames: list, capacity: int,
               n_streams: int, n_units: int, mask_frame_stride: int | None = None, frame_layout: int = 0,
               want_unit_mask: bool = False, counters: np.ndarray | None = None, frame_type: np.ndarray | None = None):
    """NEXT-3 temporal patches: keep_mask [S][mask_frame_stride][words] (per frame); frames: n_slots*tp arrays;
    frame_type [S][mask_frame_stride] (optional) -> unit_type [S][n_units]."""
    nw = grid_words(g)
    mfs = n_units * tp if mask_frame_stride is None else mask_frame_stride
    keep_mask = np.ascontiguousarray(keep_mask, dtype=np.uint32).reshape(n_streams, mfs, nw)
    n_slots = n_streams * n_units
    unit_index = np.ascontiguousarray(unit_index, dtype=np.int32).reshape(n_slots)
    frames = [np.ascontiguousarray(f, dtype=np.uint16) for f in frames]
    assert len(frames) == n_slots * tp
    ptrs = (C.c_void_p * max(1, len(frames)))(*[f.ctypes.data for f in frames])
    row = 3 * tp * g["patch"] * g["patch"]
    packed = np.zeros((max(capacity, 0), row), np.uint16)
    pos = np.zeros((max(capacity, 0), 3), np.int32)
    src = np.zeros(max(capacity, 0), np.int32)
    offs = np.zeros(n_slots + 1, np.int32)
    um = np.zeros((n_streams, n_units, nw), np.uint32) if want_unit_mask else None
    ft = None if frame_type is None else np.ascontiguousarray(frame_type, dtype=np.uint8).reshape(n_streams, mfs)
    ut = None if frame_type is None else np.zeros((n_streams, n_units), np.uint8)
    counters = np.zeros(NCOUNTERS, np.uint64) if counters is None else counters
    status = np.zeros(1, np.int32)
    rc = lib().codecsight_ref_compact_tp(C.byref(make_grid(g)), tp, n_streams, n_units, _p(keep_mask), mfs,
                                         _p(unit_index), C.cast(ptrs, C.c_void_p), frame_layout, capacity,
                                         _p(packed), _p(pos), _p(src), _p(offs), _p(um) if um is not None else None,
                                         n_units, _p(ft), _p(ut), _p(counters), _p(status))
    return dict(rc=rc, packed=packed, pos_ids=pos, src_index=src, frame_offsets=offs, unit_mask=um, unit_type=ut,
                counters=counters, status=int(status[0]))


def kv_desc(layers, kv_heads, head_dim, dtype, capacity, refresh_capacity, rope_base, n_prompt, rope_mode=0,
            mrope_section=(0, 0, 0), t_per_frame=1) -> RefKv:
    return RefKv(layers, kv_heads, head_dim, dtype, capacity, refresh_capacity, rope_base, n_prompt, rope_mode,
                 (C.c_int32 * 3)(*mrope_section), t_per_frame)


def _kvd(kv: dict) -> RefKv:
    return kv_desc(kv["layers"], kv["kv_heads"], kv["head_dim"], kv["dtype"], kv["capacity"],
                   kv["refresh_capacity"], kv["rope_base"], kv["n_prompt"], kv.get("rope_mode", 0),
                   tuple(kv.get("mrope_section", (0, 0, 0))), kv.get("t_per_frame", 1))


def kv_refresh(g: dict, kv: dict, win: dict, keep_mask_ring: np.ndarray, frame_type_ring: np.ndarray,
               old_cache: list | None, new_cache: list, refreshed: list | None, token_cap: int,
               counters: np.ndarray | None = None):
    """Caches are numpy arrays [L][2][cap][H][D] (uint16 bf16 bits or float32), modified in place (new_cache)."""
    S = len(new_cache)
    nw = grid_words(g)
    keep_mask_ring = np.ascontiguousarray(keep_mask_ring, dtype=np.uint32).reshape(S, win["ring_frames"], nw)
    frame_type_ring = np.ascontiguousarray(frame_type_ring, dtype=np.uint8).reshape(S, win["ring_frames"])
    for c in new_cache:
        assert c.flags.c_contiguous

    def arr(lst):
        if lst is None:
            return None
        a = (C.c_void_p * S)(*[x.ctypes.data for x in lst])
        return C.cast(a, C.c_void_p)

    disp = np.zeros((S, token_cap), np.uint8)
    pold = np.zeros((S, token_cap), np.int32)
    ntok = np.zeros((S, 4), np.int32)
    counters = np.zeros(NCOUNTERS, np.uint64) if counters is None else counters
    status = np.zeros(1, np.int32)
    kvd = _kvd(kv)
    w = RefWindow(win["window"], win["stride"], win["step"], win["ring_frames"])
    olds, news, refs = arr(old_cache), arr(new_cache), arr(refreshed)
    rc = lib().codecsight_ref_kv_refresh(C.byref(make_grid(g)), C.byref(kvd), C.byref(w), S, _p(keep_mask_ring),
                                         _p(frame_type_ring), olds, news, refs, token_cap, _p(disp), _p(pold),
                                         _p(ntok), _p(counters), _p(status))
    return dict(rc=rc, disposition=disp, p_old=pold, n_tokens=ntok, counters=counters, status=int(status[0]))


def kv_refresh_paged(g: dict, kv: dict, win: dict, keep_mask_ring: np.ndarray, frame_type_ring: np.ndarray,
                     pools: list, slot_old: np.ndarray | None, slot_cap: int, refreshed: list | None, token_cap: int,
                     counters: np.ndarray | None = None):
    """Pools are numpy arrays [L][2][capacity][H][D] updated in place; slot_old [S][slot_cap] (or None at k=0).
    Returns dict(slot_new [S][slot_cap], disposition, p_old, n_tokens, counters, status, rc)."""
    S = len(pools)
    nw = grid_words(g)
    keep_mask_ring = np.ascontiguousarray(keep_mask_ring, dtype=np.uint32).reshape(S, win["ring_frames"], nw)
    frame_type_ring = np.ascontiguousarray(frame_type_ring, dtype=np.uint8).reshape(S, win["ring_frames"])
    for c in pools:
        assert c.flags.c_contiguous
    pp = C.cast((C.c_void_p * S)(*[x.ctypes.data for x in pools]), C.c_void_p)
    rp = None if refreshed is None else C.cast((C.c_void_p * S)(*[x.ctypes.data for x in refreshed]), C.c_void_p)
    so = None if slot_old is None else np.ascontiguousarray(slot_old, dtype=np.int32)
    sn = np.full((S, slot_cap), -7, np.int32)
    disp = np.zeros((S, token_cap), np.uint8)
    pold = np.zeros((S, token_cap), np.int32)
    ntok = np.zeros((S, 4), np.int32)
    counters = np.zeros(NCOUNTERS, np.uint64) if counters is None else counters
    status = np.zeros(1, np.int32)
    kvd = _kvd(kv)
    w = RefWindow(win["window"], win["stride"], win["step"], win["ring_frames"])
    rc = lib().codecsight_ref_kv_refresh_paged(C.byref(make_grid(g)), C.byref(kvd), C.byref(w), S,
                                               _p(keep_mask_ring), _p(frame_type_ring), pp, _p(so), _p(sn),
                                               slot_cap, rp, token_cap, _p(disp), _p(pold), _p(ntok), _p(counters),
                                               _p(status))
    return dict(rc=rc, slot_new=sn, disposition=disp, p_old=pold, n_tokens=ntok, counters=counters,
                status=int(status[0]))


def rope_rotate_f32(k: np.ndarray, n_heads: int, head_dim: int, base: float, dp: int) -> np.ndarray:
    k = np.ascontiguousarray(k, dtype=np.float32)
    out = np.zeros_like(k)
    lib().codecsight_ref_rope_rotate_f32(_p(k), n_heads, head_dim, base, dp, _p(out))
    return out


def nv12_rgb(Y: np.ndarray, UV: np.ndarray, pre: RefPre, y: int, x: int) -> np.ndarray:
    out = np.zeros(3, np.float32)
    lib().codecsight_ref_nv12_rgb(_p(Y), _p(UV), C.byref(pre), y, x, _p(out))
    return out


def preprocess_frame(g: dict, pre: RefPre, Y: np.ndarray, UV: np.ndarray) -> np.ndarray:
    """Full-frame preprocessing -> planar [3][MH][MW] bf16 bits."""
    MH, MW = g["grid_h"] * g["patch"], g["grid_w"] * g["patch"]
    out = np.zeros((3, MH, MW), np.uint16)
    lib().codecsight_ref_preprocess_frame(C.byref(make_grid(g)), C.byref(pre), _p(np.ascontiguousarray(Y)),
                                          _p(np.ascontiguousarray(UV)), _p(out))
    return out


def compact_nv12(g: dict, pre: RefPre, keep_mask: np.ndarray, frame_index: np.ndarray, y_planes: list,
                 uv_planes: list, capacity: int, n_streams: int, n_frames: int,
                 mask_frame_stride: int | None = None, counters: np.ndarray | None = None):
    nw = grid_words(g)
    mfs = n_frames if mask_frame_stride is None else mask_frame_stride
    keep_mask = np.ascontiguousarray(keep_mask, dtype=np.uint32).reshape(n_streams, mfs, nw)
    n_slots = n_streams * n_frames
    frame_index = np.ascontiguousarray(frame_index, dtype=np.int32).reshape(n_slots)
    ys = [np.ascontiguousarray(a, dtype=np.uint8) for a in y_planes]
    uvs = [np.ascontiguousarray(a, dtype=np.uint8) for a in uv_planes]
    yp = (C.c_void_p * max(1, n_slots))(*[a.ctypes.data for a in ys])
    uvp = (C.c_void_p * max(1, n_slots))(*[a.ctypes.data for a in uvs])
    row = 3 * g["patch"] * g["patch"]
    packed = np.zeros((max(capacity, 0), row), np.uint16)
    pos = np.zeros((max(capacity, 0), 3), np.int32)
    src = np.zeros(max(capacity, 0), np.int32)
    offs = np.zeros(n_slots + 1, np.int32)
    counters = np.zeros(NCOUNTERS, np.uint64) if counters is None else counters
    status = np.zeros(1, np.int32)
    rc = lib().codecsight_ref_compact_nv12(C.byref(make_grid(g)), C.byref(pre), n_streams, n_frames, _p(keep_mask),
                                           mfs, _p(frame_index), C.cast(yp, C.c_void_p), C.cast(uvp, C.c_void_p),
                                           capacity, _p(packed), _p(pos), _p(src), _p(offs), _p(counters),
                                           _p(status))
    return dict(rc=rc, packed=packed, pos_ids=pos, src_index=src, frame_offsets=offs, counters=counters,
                status=int(status[0]))


AV_MV_DTYPE = np.dtype([("source", "<i4"), ("w", "u1"), ("h", "u1"), ("src_x", "<i2"), ("src_y", "<i2"),
                        ("dst_x", "<i2"), ("dst_y", "<i2"), ("pad0", "<u2"), ("flags", "<u8"), ("motion_x", "<i4"),
                        ("motion_y", "<i4"), ("motion_scale", "<u2"), ("pad1", "u1", (6,))])
assert AV_MV_DTYPE.itemsize == 40


def mv_rasterize(g: dict, mvs: np.ndarray, mv_offsets: np.ndarray, n_frames: int) -> np.ndarray:
    out = np.zeros((n_frames, g["mb_rows"], g["mb_cols"]), MB_DTYPE)
    mvs = np.ascontiguousarray(mvs, dtype=AV_MV_DTYPE)
    offs = np.ascontiguousarray(mv_offsets, dtype=np.int64)
    rc = lib().codecsight_ref_mv_rasterize(C.byref(make_grid(g)), n_frames, _p(mvs), _p(offs), _p(out))
    assert rc == 0
    return out


def similar_hist(score: np.ndarray, frame_type: np.ndarray, taus, n_bins: int) -> np.ndarray:
    score = np.ascontiguousarray(score, dtype=np.float32)
    n_frames, n_patches = score.shape
    taus = np.ascontiguousarray(taus, dtype=np.float32)
    hist = np.zeros((len(taus), n_bins), np.uint64)
    rc = lib().codecsight_ref_similar_hist(_p(score), _p(np.ascontiguousarray(frame_type, dtype=np.uint8)), n_frames,
                                           n_patches, _p(taus), len(taus), n_bins, _p(hist))
    assert rc == 0
    return hist
