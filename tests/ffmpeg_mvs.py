"""Test helper: real FFmpeg motion-vector exports (AVMotionVector side data, AV_CODEC_FLAG2_EXPORT_MVS) from a clip
encoded here, through the FFmpeg libraries OpenCV bundles (opencv_python*.libs: libavformat / libavcodec /
libavutil), called with ctypes.  The image has no libx264 (and no PyAV / ffmpeg binary), so the clip is MPEG-4 Part 2
(OpenCV's 'mp4v' writer, FFmpeg's own encoder); the export format -- one 40-B AVMotionVector per predicted block,
dst = the block centre, w x h, motion = (src - dst) * motion_scale -- is FFmpeg's, shared by its H.264 and MPEG-4
decoders (libavcodec's mpegvideo / h264 export paths).

Only stable public ABI is touched: the functions' signatures, AVFrameSideData {type; data; size; ...}, AVPacket's
stream_index, AVFormatContext.streams and AVStream.codecpar (offsets unchanged since FFmpeg 4)."""
import ctypes as C
import glob
import os

import numpy as np

AV_FRAME_DATA_MOTION_VECTORS = 8
AVERROR_EAGAIN = -11
AVERROR_EOF = -0x20464F45  # FFERRTAG('E','O','F',' ')


def _libs():
    import cv2
    d = os.path.dirname(os.path.dirname(cv2.__file__))
    pats = {n: glob.glob(os.path.join(d, "opencv_python*.libs", f"lib{n}-*.so*")) for n in ("avutil", "avcodec",
                                                                                             "avformat")}
    if not all(pats.values()):
        return None
    mode = getattr(C, "RTLD_GLOBAL", 0)
    util = C.CDLL(pats["avutil"][0], mode=mode)
    codec = C.CDLL(pats["avcodec"][0], mode=mode)
    fmt = C.CDLL(pats["avformat"][0], mode=mode)
    return util, codec, fmt


def available() -> bool:
    try:
        return _libs() is not None
    except Exception:
        return False


def encode_clip(path, frames, fps=25):
    """frames: list of HxWx3 uint8 (BGR); MPEG-4 Part 2 in an .mp4 container (OpenCV's FFmpeg writer)."""
    import cv2
    h, w = frames[0].shape[:2]
    wr = cv2.VideoWriter(path, cv2.VideoWriter_fourcc(*"mp4v"), fps, (w, h))
    if not wr.isOpened():
        raise RuntimeError("no mp4v encoder")
    for f in frames:
        wr.write(f)
    wr.release()


def decode_mvs(path, av_mv_dtype):
    """Decode `path` with motion-vector export; returns a list (one entry per decoded frame, display order) of
    structured arrays of `av_mv_dtype` (the 40-B AVMotionVector layout); frames without side data give empty arrays."""
    util, codec, fmt = _libs()
    vp = C.c_void_p
    fmt.avformat_open_input.argtypes = [C.POINTER(vp), C.c_char_p, vp, vp]
    fmt.avformat_find_stream_info.argtypes = [vp, vp]
    fmt.av_find_best_stream.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp), C.c_int]
    fmt.av_read_frame.argtypes = [vp, vp]
    fmt.avformat_close_input.argtypes = [C.POINTER(vp)]
    codec.avcodec_alloc_context3.argtypes = [vp]
    codec.avcodec_alloc_context3.restype = vp
    codec.avcodec_parameters_to_context.argtypes = [vp, vp]
    codec.avcodec_open2.argtypes = [vp, vp, C.POINTER(vp)]
    codec.av_packet_alloc.restype = vp
    codec.av_packet_unref.argtypes = [vp]
    codec.av_packet_free.argtypes = [C.POINTER(vp)]
    codec.avcodec_send_packet.argtypes = [vp, vp]
    codec.avcodec_receive_frame.argtypes = [vp, vp]
    codec.avcodec_free_context.argtypes = [C.POINTER(vp)]
    util.av_frame_alloc.restype = vp
    util.av_frame_free.argtypes = [C.POINTER(vp)]
    util.av_frame_get_side_data.argtypes = [vp, C.c_int]
    util.av_frame_get_side_data.restype = vp
    util.av_dict_set.argtypes = [C.POINTER(vp), C.c_char_p, C.c_char_p, C.c_int]
    util.av_dict_free.argtypes = [C.POINTER(vp)]

    ic = vp()
    if fmt.avformat_open_input(C.byref(ic), path.encode(), None, None) < 0:
        raise RuntimeError("avformat_open_input failed")
    out = []
    try:
        if fmt.avformat_find_stream_info(ic, None) < 0:
            raise RuntimeError("avformat_find_stream_info failed")
        dec = vp()
        si = fmt.av_find_best_stream(ic, 0, -1, -1, C.byref(dec), 0)  # AVMEDIA_TYPE_VIDEO
        if si < 0 or not dec.value:
            raise RuntimeError("no video stream / decoder")
        streams = C.cast(ic.value + 48, C.POINTER(C.POINTER(vp))).contents   # AVFormatContext.streams
        st = streams[si]
        par = C.cast(st + 16, C.POINTER(vp)).contents                        # AVStream.codecpar
        ctx = vp(codec.avcodec_alloc_context3(dec))
        if codec.avcodec_parameters_to_context(ctx, par) < 0:
            raise RuntimeError("avcodec_parameters_to_context failed")
        opts = vp()
        util.av_dict_set(C.byref(opts), b"flags2", b"+export_mvs", 0)
        util.av_dict_set(C.byref(opts), b"threads", b"1", 0)
        if codec.avcodec_open2(ctx, dec, C.byref(opts)) < 0:
            raise RuntimeError("avcodec_open2 failed")
        util.av_dict_free(C.byref(opts))
        pkt = vp(codec.av_packet_alloc())
        frame = vp(util.av_frame_alloc())

        def drain():
            while True:
                r = codec.avcodec_receive_frame(ctx, frame)
                if r == AVERROR_EAGAIN or r == AVERROR_EOF or r < 0:
                    return
                sd = util.av_frame_get_side_data(frame, AV_FRAME_DATA_MOTION_VECTORS)
                if sd:
                    data = C.cast(sd + 8, C.POINTER(vp)).contents.value        # AVFrameSideData.data
                    size = C.cast(sd + 16, C.POINTER(C.c_size_t)).contents.value  # AVFrameSideData.size
                    buf = (C.c_ubyte * size).from_address(data)
                    out.append(np.frombuffer(bytes(buf), dtype=av_mv_dtype).copy())
                else:
                    out.append(np.zeros(0, av_mv_dtype))

        while fmt.av_read_frame(ic, pkt) >= 0:
            if C.cast(pkt.value + 36, C.POINTER(C.c_int)).contents.value == si:  # AVPacket.stream_index
                codec.avcodec_send_packet(ctx, pkt)
                drain()
            codec.av_packet_unref(pkt)
        codec.avcodec_send_packet(ctx, None)
        drain()
        util.av_frame_free(C.byref(frame))
        codec.av_packet_free(C.byref(pkt))
        codec.avcodec_free_context(C.byref(ctx))
    finally:
        fmt.avformat_close_input(C.byref(ic))
    return out


def moving_square_clip(w=128, h=96, n=12, dx=6, dy=2, size=32, seed=0):
    """A textured square translating by (dx, dy) px per frame over a static textured background."""
    rng = np.random.default_rng(seed)
    bg = rng.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    bg = (bg // 64 * 64).astype(np.uint8)                         # coarse texture: cheap to code, matchable
    sq = rng.integers(0, 256, size=(size, size, 3), dtype=np.uint8)
    frames = []
    for i in range(n):
        f = bg.copy()
        x0, y0 = 16 + dx * i, 16 + dy * i
        f[y0:y0 + size, x0:x0 + size] = sq
        frames.append(f)
    return frames
