"""Pins of NEXT-4: FFmpeg AVMotionVector rasterisation onto the MB grid, and the similar-patch-ratio histogram
behind fig:mv_residual_analysis_cdf."""
import numpy as np

import synth
from synth import make_grid


def _mv(ref, recs):
    a = np.zeros(len(recs), ref.AV_MV_DTYPE)
    for k, r in enumerate(recs):
        for name, v in r.items():
            a[name][k] = v
    return a


def test_rasterize_hand_example(ref):
    g = make_grid(64, 48)                    # 4 x 3 MBs
    recs = [
        dict(source=-1, w=16, h=16, dst_x=24, dst_y=24, motion_x=8, motion_y=-4, motion_scale=4),   # MB (1,1)
        dict(source=-1, w=8, h=8, dst_x=4, dst_y=4, motion_x=1, motion_y=0, motion_scale=4),        # MB (0,0)
        dict(source=-1, w=8, h=8, dst_x=12, dst_y=4, motion_x=-3, motion_y=4, motion_scale=4),      # MB (0,0) max
        dict(source=-1, w=16, h=8, dst_x=48, dst_y=4, motion_x=5, motion_y=5, motion_scale=2),      # MB (0,2) & (0,3)
        dict(source=1, w=16, h=16, dst_x=8, dst_y=40, motion_x=99, motion_y=99, motion_scale=4),    # future: ignored
        dict(source=-1, w=16, h=16, dst_x=56, dst_y=40, motion_x=0, motion_y=0, motion_scale=4),    # MB (2,3) skip
    ]
    out = ref.mv_rasterize(g, _mv(ref, recs), np.array([0, len(recs)]), 1)[0]
    assert (out["mvx"][1, 1], out["mvy"][1, 1], out["type"][1, 1]) == (8, -4, 0)
    assert (out["mvx"][0, 0], out["mvy"][0, 0], out["type"][0, 0]) == (-3, 4, 0)     # |(-3,4)| > |(1,0)|
    # partition [40, 56) x [0, 8) overlaps MB columns 2 and 3; motion 5 at scale 2 = 10 qpel
    assert (out["mvx"][0, 2], out["mvy"][0, 2]) == (10, 10) and (out["mvx"][0, 3], out["mvy"][0, 3]) == (10, 10)
    assert out["type"][2, 0] == 2                                                      # no past record: INTRA
    assert (out["mvx"][2, 3], out["mvy"][2, 3], out["type"][2, 3]) == (0, 0, 0)
    assert (out["sad"] == 0).all()


def test_rasterize_round_trip_of_synthetic_streams(ref):
    """cs_mb -> one 16x16 record per non-INTRA MB (motion in qpel, scale 4) -> rasterise -> same MVs and types."""
    for scene in ["multi_object", "noise", "high"]:
        src = synth.stream_metadata(448, 448, scene, 9, 3)
        g = make_grid(448, 448)
        recs, offs = [], [0]
        for f in range(3):
            for j in range(g["mb_rows"]):
                for i in range(g["mb_cols"]):
                    m = src[f, j, i]
                    if m["type"] == 2:
                        continue
                    recs.append(dict(source=-1, w=16, h=16, dst_x=16 * i + 8, dst_y=16 * j + 8,
                                     motion_x=int(m["mvx"]), motion_y=int(m["mvy"]), motion_scale=4))
            offs.append(len(recs))
        out = ref.mv_rasterize(g, _mv(ref, recs), np.array(offs), 3)
        intra = src["type"] == 2
        assert (out["type"][intra] == 2).all() and (out["type"][~intra] == 0).all()
        assert (out["mvx"][~intra] == src["mvx"][~intra]).all() and (out["mvy"][~intra] == src["mvy"][~intra]).all()


def test_similar_hist_closed_form(ref):
    n_p, n_bins = 100, 10
    score = np.tile(np.arange(n_p, dtype=np.float32) / 10, (4, 1))          # 0.0, 0.1, ..., 9.9
    types = np.array([0, 1, 1, 1], np.uint8)                                 # the I-frame is not counted
    hist = ref.similar_hist(score, types, [0.25, 1.0, 5.0, 100.0], n_bins)
    assert (hist.sum(axis=1) == 3).all()
    # tau 0.25: 3 patches below (0.0, 0.1, 0.2) -> ratio 0.03 -> bin 0; tau 1.0: 10 -> bin 1; tau 5: 50 -> bin 5
    assert hist[0, 0] == 3 and hist[1, 1] == 3 and hist[2, 5] == 3 and hist[3, 9] == 3


def test_similar_ratio_is_one_minus_dynamic_fraction(ref):
    """The similar ratio of a P-frame is 1 - |dynamic(i)| / n (Eq. 4 before GOP accumulation)."""
    g = make_grid(448, 448)
    mb = synth.stream_metadata(448, 448, "multi_object", 3, 5)
    for tau in (0.25, 1.0, 5.0):
        gt = dict(g, tau=tau)
        for f in range(1, 5):
            _, _, M, _ = ref.patch_fields(gt, mb[f])
            n_dyn = int((M >= np.float32(tau)).sum())
            hist = ref.similar_hist(M.reshape(1, -1), np.array([1], np.uint8), [tau], 1024)
            assert hist[0, 1024 - n_dyn if n_dyn > 0 else 1023] == 1
