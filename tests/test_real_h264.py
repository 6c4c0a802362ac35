"""NEXT-4 against FFmpeg's real H.264 decoder: an H.264 stream written here (tests/h264_writer.py: Baseline CAVLC,
an I_PCM IDR picture, then P pictures of P_L0_16x16 / P_L0_L0_16x8 / P_L0_L0_8x16 / P_8x8 macroblocks with chosen
quarter-pel motion vectors and no residual) is decoded by the libavcodec OpenCV bundles with motion-vector export
(tests/ffmpeg_mvs.py).  The vectors the decoder reconstructs pass through H.264's motion-vector prediction (the writer
codes differences against the standard's median / directional predictors), so an export equal to the written
vectors pins both sides.  Pinned on the real H.264 export:
  * one 40-B record per partition: w x h = the partition (16x16, 16x8, 8x16), dst = the partition centre,
    motion_scale = 4 (quarter pel), motion = the H.264 vector (src = dst + motion / 4), source = -1; a P_8x8 MB
    exports one 8x8 record per block carrying its FIRST sub-partition's vector (sub-8x8 partitions are not exported);
  * the oracle's rasterisation (reading NEXT-4): each MB takes its partition of largest |mv| -- in quarter pel, the
    written vector itself -- type INTER;
  * on the GPU, codecsight_mv_rasterize of the real records equals the oracle bit for bit."""
import numpy as np
import pytest

import ffmpeg_mvs as fm
import h264_writer as hw
import oracle.ref as ref
from synth import make_grid

pytestmark = pytest.mark.skipif(not fm.available(), reason="no FFmpeg libraries (OpenCV's bundled libav*)")

MBW, MBH, NP = 8, 6, 5


def _stream(seed):
    rng = np.random.default_rng(seed)

    def mv():
        return (int(rng.integers(-48, 49)), int(rng.integers(-48, 49)))

    frames = []
    for _ in range(NP):
        rows = []
        for _ in range(MBH):
            row = []
            for _ in range(MBW):
                t = int(rng.integers(0, 4))
                if t == 0:
                    row.append(mv())
                elif t < 3:
                    a, b = mv(), mv()
                    while a[0] ** 2 + a[1] ** 2 == b[0] ** 2 + b[1] ** 2:   # distinct magnitudes: no tie
                        b = mv()
                    row.append((t, [a, b]))
                else:                                                       # P_8x8 with random sub-partitions
                    sub = [int(rng.integers(0, 4)) for _ in range(4)]
                    mvs = [mv() for _ in hw.partitions(3, sub)]
                    row.append((3, mvs, sub))
                    firsts = _firsts(row[-1])
                    while len({v[0] ** 2 + v[1] ** 2 for v in firsts}) < 4:   # distinct exported magnitudes
                        mvs[:] = [mv() for _ in mvs]
                        firsts = _firsts(row[-1])
            rows.append(row)
        frames.append(rows)
    return frames


@pytest.fixture(scope="module", params=[3, 11])
def exported(request, tmp_path_factory):
    frames = _stream(request.param)
    path = str(tmp_path_factory.mktemp("h264") / "mvs.h264")
    hw.write_stream(path, MBW, MBH, frames, seed=request.param)
    per_frame = fm.decode_mvs(path, ref.AV_MV_DTYPE)
    assert len(per_frame) == NP + 1
    recs = np.concatenate(per_frame)
    offs = np.zeros(NP + 2, np.int64)
    offs[1:] = np.cumsum([len(p) for p in per_frame])
    return frames, per_frame, recs, offs


def _firsts(e):
    """P_8x8: the vector of each 8x8 block's first sub-partition (what FFmpeg exports for the block)."""
    out, k = [], 0
    for st in e[2]:
        out.append(e[1][k])
        k += len(hw.SUB_PARTS[st])
    return out


def _exported(e):
    """The (x, y, w, h) rectangles and vectors FFmpeg's H.264 export carries for one MB entry: every 16x16 / 16x8 /
    8x16 partition; for P_8x8 one 8x8 record per block with its first sub-partition's vector (libavcodec exports
    sub-8x8 partitions at 8x8 granularity -- found here, DESIGN §2 NEXT-4)."""
    if isinstance(e[1], int):
        return [((0, 0, 16, 16), e)]
    if e[0] != 3:
        return list(zip(hw.PARTS[e[0]], e[1]))
    return [((bx, by, 8, 8), v) for (bx, by), v in zip(hw.B8, _firsts(e))]


def test_h264_export_equals_the_written_vectors(exported):
    frames, per_frame, _, _ = exported
    assert len(per_frame[0]) == 0                           # the IDR picture exports no motion
    for i, p in enumerate(per_frame[1:]):
        assert (p["source"] == -1).all() and (p["motion_scale"] == 4).all()
        got = {(int(r["dst_x"]), int(r["dst_y"]), int(r["w"]), int(r["h"])): (int(r["motion_x"]), int(r["motion_y"]))
               for r in p}
        exp = {}
        for my in range(MBH):
            for mx in range(MBW):
                for (px, py, pw, ph), v in _exported(frames[i][my][mx]):
                    exp[(16 * mx + px + pw // 2, 16 * my + py + ph // 2, pw, ph)] = v   # dst = partition centre
        assert len(p) == len(exp) and got == exp
        exact = p["motion_x"] % 4 == 0
        assert (p["src_x"][exact] == p["dst_x"][exact] + p["motion_x"][exact] // 4).all()


def test_oracle_rasterises_the_h264_export(exported):
    frames, _, recs, offs = exported
    g = make_grid(16 * MBW, 16 * MBH)
    out = ref.mv_rasterize(g, recs, offs, NP + 1)
    assert (out[0]["type"] == 2).all()                       # IDR: no records -> INTRA
    for i in range(NP):
        for my in range(MBH):
            for mx in range(MBW):
                mvs = [v for _, v in _exported(frames[i][my][mx])]
                best = max(mvs, key=lambda v: v[0] ** 2 + v[1] ** 2)      # the MB's largest exported |mv| (qpel)
                o = out[i + 1, my, mx]
                assert (int(o["mvx"]), int(o["mvy"]), int(o["type"])) == (best[0], best[1], 0)


@pytest.mark.gpu
def test_gpu_rasterises_the_h264_export_like_the_oracle(exported):
    import torch
    from paper_2604_06036_b200 import _abi as abi
    _, _, recs, offs = exported
    g = make_grid(16 * MBW, 16 * MBH)
    n = NP + 1
    out_d = torch.zeros(n * g["mb_rows"] * g["mb_cols"], dtype=torch.int64, device="cuda")
    abi.codecsight_mv_rasterize(g, n, torch.from_numpy(recs.view(np.uint8)).to("cuda"),
                                torch.from_numpy(offs).to("cuda"), out_d)
    exp = ref.mv_rasterize(g, recs, offs, n)
    torch.cuda.synchronize()
    got = out_d.cpu().numpy().view(ref.MB_DTYPE).reshape(exp.shape)
    assert (got == exp).all()
