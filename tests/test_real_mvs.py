"""NEXT-4 against a real decoder export (the AVMotionVector semantics were checked only against
self-generated records).  A clip of a textured square moving by (+6, +2) px per frame over a smooth background is
encoded here (MPEG-4 Part 2 through OpenCV's bundled FFmpeg: the image has no libx264) and decoded by FFmpeg with
AV_CODEC_FLAG2_EXPORT_MVS (tests/ffmpeg_mvs.py).  Pinned, on FFmpeg's own output:
  * the record is the 40-B layout cs_av_mv / the oracle's AV_MV_DTYPE mirror (the side data size is a multiple of 40
    and every field decodes to a plausible value);
  * dst is the partition centre: [dst - w/2, dst - w/2 + w) is an aligned macroblock (reading NEXT-4);
  * motion = (src - dst) * motion_scale, i.e. the block came from src = dst + motion / motion_scale (the sign our
    magnitude ignores but the ingest keeps);
  * the oracle's rasterisation of the real records: every MB fully inside the moving square is INTER with
    trunc(4 * motion / motion_scale) = (-24, -8) quarter pel (the square moved +6, +2 px), and an MB with no record is
    INTRA;
  * on the GPU, codecsight_mv_rasterize of the real records equals the oracle bit for bit."""
import numpy as np
import pytest

import ffmpeg_mvs as fm
import oracle.ref as ref
from synth import make_grid

pytestmark = pytest.mark.skipif(not fm.available(), reason="no FFmpeg libraries (OpenCV's bundled libav*)")

W, H, N, DX, DY, SIZE, X0, Y0 = 160, 128, 10, 6, 2, 48, 20, 20


def _clip():
    yy, xx = np.mgrid[0:H, 0:W]
    bg = np.stack([(xx * 255 // W), (yy * 255 // H), np.full_like(xx, 60)], -1).astype(np.uint8)
    sy, sx = np.mgrid[0:SIZE, 0:SIZE]
    sq = np.stack([128 + 100 * np.sin(sx / 5.0), 128 + 100 * np.cos(sy / 4.0), 128 + 60 * np.sin((sx + sy) / 6.0)],
                  -1).astype(np.uint8)
    frames = []
    for i in range(N):
        f = bg.copy()
        f[Y0 + DY * i:Y0 + DY * i + SIZE, X0 + DX * i:X0 + DX * i + SIZE] = sq
        frames.append(f)
    return frames


@pytest.fixture(scope="module")
def exported(tmp_path_factory):
    path = str(tmp_path_factory.mktemp("clip") / "square.mp4")
    fm.encode_clip(path, _clip())
    per_frame = fm.decode_mvs(path, ref.AV_MV_DTYPE)
    assert len(per_frame) == N
    recs = np.concatenate(per_frame)
    offs = np.zeros(N + 1, np.int64)
    offs[1:] = np.cumsum([len(p) for p in per_frame])
    return per_frame, recs, offs


def _inside(i, bx, by, bs=16):
    x0, y0 = X0 + DX * i, Y0 + DY * i
    return bx >= x0 and bx + bs <= x0 + SIZE and by >= y0 and by + bs <= y0 + SIZE


def test_export_layout_and_semantics(exported):
    per_frame, recs, _ = exported
    assert ref.AV_MV_DTYPE.itemsize == 40
    assert len(per_frame[0]) == 0                        # the I-frame exports no motion
    assert all(len(p) > 0 for p in per_frame[1:])
    assert (recs["source"] == -1).all()                  # P-frames: past references only
    assert set(np.unique(recs["w"])) <= {8, 16} and (recs["w"] == recs["h"]).all()
    assert (recs["motion_scale"] == 2).all()             # MPEG-4 Part 2: half pel
    for p in per_frame[1:]:
        w = p["w"].astype(np.int64)
        x = p["dst_x"].astype(np.int64) - w // 2
        y = p["dst_y"].astype(np.int64) - p["h"].astype(np.int64) // 2
        assert ((x % w) == 0).all() and ((y % w) == 0).all()     # dst = the centre of an aligned block
        assert (x >= 0).all() and (x + w <= W).all() and (y >= 0).all() and (y + w <= H).all()
        exact = (p["motion_x"] % p["motion_scale"] == 0) & (p["motion_y"] % p["motion_scale"] == 0)
        assert (p["src_x"][exact] == p["dst_x"][exact] + p["motion_x"][exact] // p["motion_scale"][exact]).all()
        assert (p["src_y"][exact] == p["dst_y"][exact] + p["motion_y"][exact] // p["motion_scale"][exact]).all()


def test_oracle_rasterises_the_real_export(exported):
    per_frame, recs, offs = exported
    g = make_grid(W, H)
    out = ref.mv_rasterize(g, recs, offs, N)
    inside = 0
    for i in range(1, N):
        have = np.zeros((g["mb_rows"], g["mb_cols"]), bool)
        for r in per_frame[i]:
            x, y = int(r["dst_x"]) - int(r["w"]) // 2, int(r["dst_y"]) - int(r["h"]) // 2
            have[y // 16:(y + int(r["h"]) + 15) // 16, x // 16:(x + int(r["w"]) + 15) // 16] = True
        for my in range(g["mb_rows"]):
            for mx in range(g["mb_cols"]):
                o = out[i, my, mx]
                if not have[my, mx]:
                    assert o["type"] == 2                               # no record: intra coded
                elif _inside(i, 16 * mx, 16 * my):
                    inside += 1
                    assert (int(o["mvx"]), int(o["mvy"]), int(o["type"])) == (-4 * DX, -4 * DY, 0)
    assert inside >= 20


@pytest.mark.gpu
def test_gpu_rasterises_the_real_export_like_the_oracle(exported):
    import torch
    from paper_2604_06036_b200 import _abi as abi
    _, recs, offs = exported
    g = make_grid(W, H)
    out_d = torch.zeros(N * g["mb_rows"] * g["mb_cols"], dtype=torch.int64, device="cuda")
    abi.codecsight_mv_rasterize(g, N, torch.from_numpy(recs.view(np.uint8)).to("cuda"),
                                torch.from_numpy(offs).to("cuda"), out_d)
    exp = ref.mv_rasterize(g, recs, offs, N)
    torch.cuda.synchronize()
    got = out_d.cpu().numpy().view(ref.MB_DTYPE).reshape(exp.shape)
    assert (got == exp).all()
