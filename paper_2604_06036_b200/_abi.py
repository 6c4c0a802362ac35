"""Thin ctypes binding of ``libcodecsight.so`` (include/codecsight.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels behind the C ABI.  Tensors must
be CUDA tensors (device memory owned by PyTorch); the calls are enqueued on the current torch CUDA stream unless
``stream`` is given.  There is no CPU fallback: if the library is missing or there is no CUDA device the calls
raise.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcodecsight.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "codecsight.h")

CS_OK, CS_ERR_INVALID_ARGUMENT, CS_ERR_SHAPE, CS_ERR_UNSUPPORTED, CS_ERR_CUDA = 0, -1, -2, -3, -4
CS_STATUS_CAPACITY, CS_STATUS_NO_IFRAME, CS_STATUS_ORIGIN, CS_STATUS_BAD_FRAME_TYPE, CS_STATUS_BAD_MB_TYPE = \
    1, 2, 4, 8, 16
CS_STATUS_MISALIGNED = 32
CS_LAUNCH_PDL = 1
CS_FRAME_I, CS_FRAME_P = 0, 1
CS_MB_INTER, CS_MB_SKIP, CS_MB_INTRA = 0, 1, 2
CS_DISP_NEW, CS_DISP_ANCHOR, CS_DISP_REUSE = 0, 1, 2
CS_BF16, CS_FP32 = 0, 1
CS_LAYOUT_PLANAR, CS_LAYOUT_GROUPED = 0, 1
NCOUNTERS = 16
(CNT_FRAMES, CNT_PFRAMES, CNT_PATCHES, CNT_KEPT, CNT_NEAR_TAU, CNT_TOK_REUSE, CNT_TOK_ANCHOR, CNT_TOK_NEW,
 CNT_BYTES_SCORE, CNT_BYTES_COMPACT, CNT_BYTES_KV, CNT_PACKED_ROWS, CNT_STREAM_STEPS) = range(13)


class CodecSightError(RuntimeError):
    pass


class CsGrid(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("src_w", "src_h", "mb_size", "mb_cols", "mb_rows", "patch", "grid_w",
                                          "grid_h", "group")] + [("tau", C.c_float), ("alpha", C.c_float)]


class CsKvDesc(C.Structure):
    _fields_ = [("layers", C.c_int32), ("kv_heads", C.c_int32), ("head_dim", C.c_int32), ("dtype", C.c_int32),
                ("capacity", C.c_int64), ("refresh_capacity", C.c_int64), ("rope_base", C.c_double),
                ("n_prompt", C.c_int32), ("rope_mode", C.c_int32), ("mrope_section", C.c_int32 * 3),
                ("t_per_frame", C.c_int32)]


CS_ROPE_1D, CS_ROPE_MROPE = 0, 1


class CsPreprocess(C.Structure):
    _fields_ = [("src_w", C.c_int32), ("src_h", C.c_int32), ("y_pitch", C.c_int32), ("uv_pitch", C.c_int32),
                ("color", C.c_int32), ("mean", C.c_float * 3), ("std", C.c_float * 3)]


CLIP_MEAN = (0.48145466, 0.4578275, 0.40821073)
CLIP_STD = (0.26862954, 0.26130258, 0.27577711)


def make_preprocess(pre: dict) -> CsPreprocess:
    return CsPreprocess(pre["src_w"], pre["src_h"], pre.get("y_pitch", pre["src_w"]), pre.get("uv_pitch", pre["src_w"]),
                        pre.get("color", 0), (C.c_float * 3)(*pre.get("mean", CLIP_MEAN)),
                        (C.c_float * 3)(*pre.get("std", CLIP_STD)))


class CsWindow(C.Structure):
    _fields_ = [("window", C.c_int32), ("stride", C.c_int32), ("step", C.c_int32), ("ring_frames", C.c_int32)]


_lib = None


def lib():
    """Load libcodecsight.so (built in-tree by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CodecSightError(f"{LIB_PATH} not found: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
        L.codecsight_score_patches.restype = C.c_int
        L.codecsight_score_patches.argtypes = [C.POINTER(CsGrid), I32, I32, P, P, P, I64, P, P, P, P, P, P]
        L.codecsight_compact.restype = C.c_int
        L.codecsight_compact.argtypes = [C.POINTER(CsGrid), I32, I32, P, I64, P, P, I32, I64, P, P, P, P, P, P, P]
        L.codecsight_compact_nv12.restype = C.c_int
        L.codecsight_compact_nv12.argtypes = [C.POINTER(CsGrid), C.POINTER(CsPreprocess), I32, I32, P, I64, P, P, P,
                                              I64, P, P, P, P, P, P, P]
        L.codecsight_score_compact_workspace_size.restype = C.c_size_t
        L.codecsight_score_compact_workspace_size.argtypes = [I32]
        L.codecsight_score_compact.restype = C.c_int
        L.codecsight_score_compact.argtypes = [C.POINTER(CsGrid), I32, I32, P, P, P, I64, P, P, P, P, P, I32, I64, P,
                                               P, P, P, P, C.c_size_t, P, P, P]
        L.codecsight_score_compact_ex.restype = C.c_int
        L.codecsight_score_compact_ex.argtypes = [C.POINTER(CsGrid), I32, I32, P, P, I64, P, I64, P, P, P, P, P, I32,
                                                  I64, P, P, P, P, P, C.c_size_t, P, P, C.c_uint32,
                                                  C.POINTER(CsChain), P]
        L.codecsight_compact_tp.restype = C.c_int
        L.codecsight_compact_tp.argtypes = [C.POINTER(CsGrid), I32, I32, I32, P, I64, P, P, I32, I64, P, P, P, P, P,
                                            I64, P, P, P, P, P]
        L.codecsight_mv_rasterize.restype = C.c_int
        L.codecsight_mv_rasterize.argtypes = [C.POINTER(CsGrid), I32, P, P, P, P]
        L.codecsight_similar_hist.restype = C.c_int
        L.codecsight_similar_hist.argtypes = [P, P, I64, I32, P, I32, I32, P, P]
        L.codecsight_kv_refresh.restype = C.c_int
        L.codecsight_kv_refresh.argtypes = [C.POINTER(CsGrid), C.POINTER(CsKvDesc), C.POINTER(CsWindow), I32, P, P,
                                            P, P, P, I64, P, P, P, P, C.c_size_t, P, P, P]
        L.codecsight_kv_refresh_paged.restype = C.c_int
        L.codecsight_kv_refresh_paged.argtypes = [C.POINTER(CsGrid), C.POINTER(CsKvDesc), C.POINTER(CsWindow), I32,
                                                  P, P, P, P, P, I64, P, I64, P, P, P, P, C.c_size_t, P, P, P]
        L.codecsight_kv_refresh_paged_workspace_size.restype = C.c_size_t
        L.codecsight_kv_refresh_paged_workspace_size.argtypes = [C.POINTER(CsGrid), C.POINTER(CsKvDesc),
                                                                 C.POINTER(CsWindow), I32]
        L.codecsight_kv_refresh_workspace_size.restype = C.c_size_t
        L.codecsight_kv_refresh_workspace_size.argtypes = [C.POINTER(CsKvDesc), C.POINTER(CsWindow), I32]
        L.codecsight_strerror.restype = C.c_char_p
        L.codecsight_strerror.argtypes = [C.c_int]
        L.codecsight_version.restype = C.c_int
        _lib = L
    return _lib


def declared_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER) as f:
        txt = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(codecsight_\w+)\s*\(", txt, re.M)))


class CsChain(C.Structure):
    _fields_ = [("gop_ready", C.c_void_p), ("done", C.c_void_p), ("generation", C.c_uint32), ("depth", C.c_uint32)]


def make_grid(g: dict) -> CsGrid:
    return CsGrid(g["src_w"], g["src_h"], g["mb_size"], g["mb_cols"], g["mb_rows"], g["patch"], g["grid_w"],
                  g["grid_h"], g["group"], g["tau"], g["alpha"])


def make_kv(kv: dict) -> CsKvDesc:
    return CsKvDesc(kv["layers"], kv["kv_heads"], kv["head_dim"], kv["dtype"], kv["capacity"],
                    kv["refresh_capacity"], kv["rope_base"], kv["n_prompt"], kv.get("rope_mode", CS_ROPE_1D),
                    (C.c_int32 * 3)(*kv.get("mrope_section", (0, 0, 0))), kv.get("t_per_frame", 1))


def make_window(win: dict) -> CsWindow:
    return CsWindow(win["window"], win["stride"], win["step"], win["ring_frames"])


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if not t.is_cuda:
        raise CodecSightError("expected a CUDA tensor")
    return t.data_ptr()


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _check(rc: int, what: str):
    if rc != CS_OK:
        raise CodecSightError(f"{what}: {lib().codecsight_strerror(rc).decode()} ({rc})")


def ptr_array(tensors, device) -> torch.Tensor:
    """Device array of device pointers (for `frames`, `old_cache`, `new_cache`, `refreshed`)."""
    return torch.tensor([t.data_ptr() for t in tensors], dtype=torch.int64, device=device)


def grid_words(g: dict) -> int:
    return (g["grid_w"] * g["grid_h"] + 31) // 32


def codecsight_score_patches(g: dict, n_streams: int, n_frames: int, mb, frame_type, keep_mask, frame_stride: int,
                             gop_state, score, kept_count, counters, status, stream=None) -> None:
    rc = lib().codecsight_score_patches(C.byref(make_grid(g)), n_streams, n_frames, _ptr(mb), _ptr(frame_type),
                                        _ptr(keep_mask), frame_stride, _ptr(gop_state), _ptr(score),
                                        _ptr(kept_count), _ptr(counters), _ptr(status), _stream(stream))
    _check(rc, "codecsight_score_patches")


def codecsight_compact(g: dict, n_streams: int, n_frames: int, keep_mask, mask_frame_stride: int, frame_index,
                       frames_ptrs, capacity: int, packed, pos_ids, src_index, frame_offsets, counters, status,
                       stream=None, frame_layout: int = CS_LAYOUT_PLANAR) -> None:
    rc = lib().codecsight_compact(C.byref(make_grid(g)), n_streams, n_frames, _ptr(keep_mask), mask_frame_stride,
                                  _ptr(frame_index), _ptr(frames_ptrs), frame_layout, capacity, _ptr(packed),
                                  _ptr(pos_ids),
                                  _ptr(src_index), _ptr(frame_offsets), _ptr(counters), _ptr(status),
                                  _stream(stream))
    _check(rc, "codecsight_compact")


def codecsight_compact_nv12(g: dict, pre: dict, n_streams: int, n_frames: int, keep_mask, mask_frame_stride: int,
                            frame_index, y_ptrs, uv_ptrs, capacity: int, packed, pos_ids, src_index, frame_offsets,
                            counters, status, stream=None) -> None:
    rc = lib().codecsight_compact_nv12(C.byref(make_grid(g)), C.byref(make_preprocess(pre)), n_streams, n_frames,
                                       _ptr(keep_mask), mask_frame_stride, _ptr(frame_index), _ptr(y_ptrs),
                                       _ptr(uv_ptrs), capacity, _ptr(packed), _ptr(pos_ids), _ptr(src_index),
                                       _ptr(frame_offsets), _ptr(counters), _ptr(status), _stream(stream))
    _check(rc, "codecsight_compact_nv12")


def score_compact_workspace_size(n_streams: int) -> int:
    return int(lib().codecsight_score_compact_workspace_size(n_streams))


def codecsight_score_compact(g: dict, n_streams: int, n_frames: int, mb, frame_type, keep_mask, frame_stride: int,
                             gop_state, score, kept_count, frame_index, frames, capacity: int, packed, pos_ids,
                             src_index, frame_offsets, workspace, counters, status,
                             frame_layout: int = CS_LAYOUT_PLANAR, stream=None) -> None:
    rc = lib().codecsight_score_compact(C.byref(make_grid(g)), n_streams, n_frames, _ptr(mb), _ptr(frame_type),
                                        _ptr(keep_mask), frame_stride, _ptr(gop_state), _ptr(score),
                                        _ptr(kept_count), _ptr(frame_index), _ptr(frames), frame_layout, capacity,
                                        _ptr(packed), _ptr(pos_ids), _ptr(src_index), _ptr(frame_offsets),
                                        _ptr(workspace), workspace.numel() * workspace.element_size(),
                                        _ptr(counters), _ptr(status), _stream(stream))
    _check(rc, "codecsight_score_compact")


def codecsight_score_compact_ex(g: dict, n_streams: int, n_frames: int, mb, frame_type, type_stride: int, keep_mask,
                                frame_stride: int, gop_state, score, kept_count, frame_index, frames, capacity: int,
                                packed, pos_ids, src_index, frame_offsets, workspace, counters, status,
                                flags: int = 0, chain=None, frame_layout: int = CS_LAYOUT_PLANAR, stream=None) -> None:
    """chain = (gop_ready tensor [S] int32, done tensor [depth] int32, generation) with flags = CS_LAUNCH_PDL."""
    ch = None if chain is None else C.byref(CsChain(_ptr(chain[0]), _ptr(chain[1]), chain[2], chain[1].numel()))
    rc = lib().codecsight_score_compact_ex(C.byref(make_grid(g)), n_streams, n_frames, _ptr(mb), _ptr(frame_type),
                                           type_stride, _ptr(keep_mask), frame_stride, _ptr(gop_state), _ptr(score),
                                           _ptr(kept_count), _ptr(frame_index), _ptr(frames), frame_layout, capacity,
                                           _ptr(packed), _ptr(pos_ids), _ptr(src_index), _ptr(frame_offsets),
                                           _ptr(workspace), workspace.numel() * workspace.element_size(),
                                           _ptr(counters), _ptr(status), flags, ch, _stream(stream))
    _check(rc, "codecsight_score_compact_ex")


class BoundScoreCompact:
    """codecsight_score_compact_ex with every argument but the per-step inputs (mb, frame_index, frames, stream and,
    with types_per_call, frame_type) marshalled once: the Pipeline's per-step host cost is then one ctypes call (same
    C entry point, same checks).  flags = CS_LAUNCH_PDL: programmatic dependent launch."""

    def __init__(self, g: dict, n_streams: int, n_frames: int, frame_type, keep_mask, frame_stride: int, gop_state,
                 score, kept_count, capacity: int, packed, pos_ids, src_index, frame_offsets, workspace, counters,
                 status, frame_layout: int = CS_LAYOUT_PLANAR, flags: int = 0, type_stride: int | None = None,
                 chain=None):
        self._grid = make_grid(g)  # kept alive: passed by reference on every call
        self._fn = lib().codecsight_score_compact_ex
        self._head = (C.byref(self._grid), n_streams, n_frames)
        self._types_per_call = frame_type is None
        self._ty = None if frame_type is None else _ptr(frame_type)
        self._ts = frame_stride if type_stride is None else type_stride
        self._mid = (_ptr(keep_mask), frame_stride, _ptr(gop_state), _ptr(score), _ptr(kept_count))
        self._tail = (frame_layout, capacity, _ptr(packed), _ptr(pos_ids), _ptr(src_index), _ptr(frame_offsets),
                      _ptr(workspace), workspace.numel() * workspace.element_size(), _ptr(counters), _ptr(status),
                      flags)
        # chained calls (CS_LAUNCH_PDL): (gop_ready, done) tensors; the generation is given per call
        self._chain = None if chain is None else CsChain(_ptr(chain[0]), _ptr(chain[1]), 0, chain[1].numel())

    def __call__(self, mb, frame_index, frames, stream: int, frame_type=None, generation: int = 0) -> None:
        if not (mb.is_cuda and frame_index.is_cuda and frames.is_cuda):
            raise CodecSightError("expected CUDA tensors")
        ty = frame_type.data_ptr() if self._types_per_call else self._ty
        ch = None
        if self._chain is not None:
            self._chain.generation = generation & 0xFFFFFFFF
            ch = C.byref(self._chain)
        rc = self._fn(*self._head, mb.data_ptr(), ty, self._ts, *self._mid, frame_index.data_ptr(), frames.data_ptr(),
                      *self._tail, ch, stream)
        if rc != CS_OK:
            _check(rc, "codecsight_score_compact_ex")


def codecsight_compact_tp(g: dict, temporal_patch: int, n_streams: int, n_units: int, keep_mask,
                          mask_frame_stride: int, unit_index, frames, capacity: int, packed, pos_ids, src_index,
                          frame_offsets, counters, status, frame_layout: int = CS_LAYOUT_PLANAR, unit_mask=None,
                          unit_mask_stride: int = 0, frame_type=None, unit_type=None, stream=None) -> None:
    rc = lib().codecsight_compact_tp(C.byref(make_grid(g)), temporal_patch, n_streams, n_units, _ptr(keep_mask),
                                     mask_frame_stride, _ptr(unit_index), _ptr(frames), frame_layout, capacity,
                                     _ptr(packed), _ptr(pos_ids), _ptr(src_index), _ptr(frame_offsets),
                                     _ptr(unit_mask), unit_mask_stride, _ptr(frame_type), _ptr(unit_type),
                                     _ptr(counters), _ptr(status),
                                     _stream(stream))
    _check(rc, "codecsight_compact_tp")


def codecsight_mv_rasterize(g: dict, n_frames: int, mvs, mv_offsets, out, stream=None) -> None:
    rc = lib().codecsight_mv_rasterize(C.byref(make_grid(g)), n_frames, _ptr(mvs), _ptr(mv_offsets), _ptr(out),
                                       _stream(stream))
    _check(rc, "codecsight_mv_rasterize")


def codecsight_similar_hist(score, frame_type, n_frames: int, n_patches: int, taus, n_tau: int, n_bins: int, hist,
                            stream=None) -> None:
    rc = lib().codecsight_similar_hist(_ptr(score), _ptr(frame_type), n_frames, n_patches, _ptr(taus), n_tau, n_bins,
                                       _ptr(hist), _stream(stream))
    _check(rc, "codecsight_similar_hist")


def kv_workspace_size(kv: dict, win: dict, n_streams: int) -> int:
    return int(lib().codecsight_kv_refresh_workspace_size(C.byref(make_kv(kv)), C.byref(make_window(win)),
                                                          n_streams))


def codecsight_kv_refresh(g: dict, kv: dict, win: dict, n_streams: int, keep_mask_ring, frame_type_ring,
                          old_ptrs, new_ptrs, refreshed_ptrs, token_cap: int, disposition, p_old, n_tokens,
                          workspace, counters, status, stream=None) -> None:
    ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    rc = lib().codecsight_kv_refresh(C.byref(make_grid(g)), C.byref(make_kv(kv)), C.byref(make_window(win)),
                                     n_streams, _ptr(keep_mask_ring), _ptr(frame_type_ring), _ptr(old_ptrs),
                                     _ptr(new_ptrs), _ptr(refreshed_ptrs), token_cap, _ptr(disposition),
                                     _ptr(p_old), _ptr(n_tokens), _ptr(workspace), ws_bytes, _ptr(counters),
                                     _ptr(status), _stream(stream))
    _check(rc, "codecsight_kv_refresh")


def kv_paged_workspace_size(g: dict, kv: dict, win: dict, n_streams: int) -> int:
    return int(lib().codecsight_kv_refresh_paged_workspace_size(C.byref(make_grid(g)), C.byref(make_kv(kv)),
                                                                C.byref(make_window(win)), n_streams))


def codecsight_kv_refresh_paged(g: dict, kv: dict, win: dict, n_streams: int, keep_mask_ring, frame_type_ring,
                                pool_ptrs, slot_old, slot_new, slot_cap: int, refreshed_ptrs, token_cap: int,
                                disposition, p_old, n_tokens, workspace, counters, status, stream=None) -> None:
    ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    rc = lib().codecsight_kv_refresh_paged(C.byref(make_grid(g)), C.byref(make_kv(kv)), C.byref(make_window(win)),
                                           n_streams, _ptr(keep_mask_ring), _ptr(frame_type_ring), _ptr(pool_ptrs),
                                           _ptr(slot_old), _ptr(slot_new), slot_cap, _ptr(refreshed_ptrs), token_cap,
                                           _ptr(disposition), _ptr(p_old), _ptr(n_tokens), _ptr(workspace), ws_bytes,
                                           _ptr(counters), _ptr(status), _stream(stream))
    _check(rc, "codecsight_kv_refresh_paged")


# short aliases
kv_refresh_paged = codecsight_kv_refresh_paged
score_patches = codecsight_score_patches
compact = codecsight_compact
compact_nv12 = codecsight_compact_nv12
mv_rasterize = codecsight_mv_rasterize
compact_tp = codecsight_compact_tp
score_compact = codecsight_score_compact
similar_hist = codecsight_similar_hist
kv_refresh = codecsight_kv_refresh
