"""Test helper: a minimal H.264 (Annex B, Baseline, CAVLC) bitstream writer whose P-frames carry CHOSEN motion
vectors, so that FFmpeg's real H.264 decoder can export them (the image has no H.264 encoder).

Stream: SPS + PPS; frame 0 an IDR picture of I_PCM macroblocks (raw samples); frames 1.. P pictures in which every
macroblock is P_L0_16x16, P_L0_L0_16x8, P_L0_L0_8x16 or P_8x8 (sub-partitions 8x8 / 8x4 / 4x8 / 4x4) with the
requested quarter-pel motion vectors,
coded_block_pattern 0 (no residual), one reference frame, deblocking off.  Each motion vector difference is coded
against the standard's prediction (ITU-T H.264 §8.4.1.3: neighbours A = left, B = above, C = above-right or D =
above-left of the partition; the directional rules of 16x8 / 8x16 partitions; else the median)."""
import numpy as np


class BitWriter:
    def __init__(self):
        self.bits = []

    def u(self, n, v):
        for i in range(n - 1, -1, -1):
            self.bits.append((v >> i) & 1)

    def ue(self, v):
        x = v + 1
        n = x.bit_length()
        self.u(n - 1, 0)
        self.u(n, x)

    def se(self, v):
        self.ue(2 * v - 1 if v > 0 else -2 * v)

    def align_zero(self):
        while len(self.bits) % 8:
            self.bits.append(0)

    def trailing(self):
        self.bits.append(1)
        self.align_zero()

    def bytes(self):
        assert len(self.bits) % 8 == 0
        out = bytearray()
        for i in range(0, len(self.bits), 8):
            b = 0
            for bit in self.bits[i:i + 8]:
                b = (b << 1) | bit
            out.append(b)
        return bytes(out)


def _nal(nal_ref_idc, nal_type, rbsp):
    # emulation prevention: 0x000000..0x000003 -> insert 0x03
    out = bytearray()
    zeros = 0
    for b in rbsp:
        if zeros >= 2 and b <= 3:
            out.append(3)
            zeros = 0
        out.append(b)
        zeros = zeros + 1 if b == 0 else 0
    return b"\x00\x00\x00\x01" + bytes([(nal_ref_idc << 5) | nal_type]) + bytes(out)


def _sps(mbw, mbh):
    w = BitWriter()
    w.u(8, 66)              # profile_idc: Baseline
    w.u(8, 0xC0)            # constraint_set0/1
    w.u(8, 30)              # level_idc
    w.ue(0)                 # seq_parameter_set_id
    w.ue(0)                 # log2_max_frame_num_minus4 -> 4-bit frame_num
    w.ue(2)                 # pic_order_cnt_type 2 (output order = decode order)
    w.ue(1)                 # max_num_ref_frames
    w.u(1, 0)               # gaps_in_frame_num_value_allowed_flag
    w.ue(mbw - 1)           # pic_width_in_mbs_minus1
    w.ue(mbh - 1)           # pic_height_in_map_units_minus1
    w.u(1, 1)               # frame_mbs_only_flag
    w.u(1, 1)               # direct_8x8_inference_flag
    w.u(1, 0)               # frame_cropping_flag
    w.u(1, 0)               # vui_parameters_present_flag
    w.trailing()
    return _nal(3, 7, w.bytes())


def _pps():
    w = BitWriter()
    w.ue(0)                 # pic_parameter_set_id
    w.ue(0)                 # seq_parameter_set_id
    w.u(1, 0)               # entropy_coding_mode_flag: CAVLC
    w.u(1, 0)               # bottom_field_pic_order_in_frame_present_flag
    w.ue(0)                 # num_slice_groups_minus1
    w.ue(0)                 # num_ref_idx_l0_default_active_minus1
    w.ue(0)                 # num_ref_idx_l1_default_active_minus1
    w.u(1, 0)               # weighted_pred_flag
    w.u(2, 0)               # weighted_bipred_idc
    w.se(0)                 # pic_init_qp_minus26
    w.se(0)                 # pic_init_qs_minus26
    w.se(0)                 # chroma_qp_index_offset
    w.u(1, 1)               # deblocking_filter_control_present_flag
    w.u(1, 0)               # constrained_intra_pred_flag
    w.u(1, 0)               # redundant_pic_cnt_present_flag
    w.trailing()
    return _nal(3, 8, w.bytes())


def _idr(mbw, mbh, luma, cb, cr):
    w = BitWriter()
    w.ue(0)                 # first_mb_in_slice
    w.ue(7)                 # slice_type: I (all slices of the picture)
    w.ue(0)                 # pic_parameter_set_id
    w.u(4, 0)               # frame_num
    w.ue(0)                 # idr_pic_id
    w.u(1, 0)               # no_output_of_prior_pics_flag
    w.u(1, 0)               # long_term_reference_flag
    w.se(0)                 # slice_qp_delta
    w.ue(1)                 # disable_deblocking_filter_idc: off
    for my in range(mbh):
        for mx in range(mbw):
            w.ue(25)        # mb_type I_PCM
            w.align_zero()  # pcm_alignment_zero_bit
            for v in luma[16 * my:16 * my + 16, 16 * mx:16 * mx + 16].reshape(-1):
                w.u(8, int(v))
            for plane in (cb, cr):
                for v in plane[8 * my:8 * my + 8, 8 * mx:8 * mx + 8].reshape(-1):
                    w.u(8, int(v))
    w.trailing()
    return _nal(3, 5, w.bytes())


def _median(a, b, c):
    return max(min(a, b), min(max(a, b), c))


class MvField:
    """Decoded luma 4x4 blocks of the current picture: their motion vectors (all reference index 0)."""

    def __init__(self, mbw, mbh):
        self.w, self.h = 4 * mbw, 4 * mbh
        self.mv = {}

    def get(self, x, y):  # luma sample location -> (available, mv)
        if x < 0 or y < 0 or x >= 4 * self.w or y >= 4 * self.h:
            return False, (0, 0)
        k = (x // 4, y // 4)
        return (True, self.mv[k]) if k in self.mv else (False, (0, 0))

    def put(self, x, y, pw, ph, mv):
        for by in range(y // 4, (y + ph) // 4):
            for bx in range(x // 4, (x + pw) // 4):
                self.mv[(bx, by)] = mv


def predict_partition(f, x, y, pw, ph, part_idx):
    """mvpLX of a partition at luma (x, y), pw x ph (H.264 §8.4.1.3, reference 0, one reference picture)."""
    a_ok, a = f.get(x - 1, y)
    b_ok, b = f.get(x, y - 1)
    c_ok, c = f.get(x + pw, y - 1)
    if not c_ok:
        c_ok, c = f.get(x - 1, y - 1)             # D replaces an unavailable C (8.4.1.3.2)
    # directional prediction of 16x8 / 8x16 partitions
    if (pw, ph) == (16, 8):
        if part_idx == 0 and b_ok:
            return b
        if part_idx == 1 and a_ok:
            return a
    if (pw, ph) == (8, 16):
        if part_idx == 0 and a_ok:
            return a
        if part_idx == 1 and c_ok:
            return c
    if not b_ok and not c_ok and a_ok:            # only A: B and C take A's motion (8.4.1.3.1)
        b, c, b_ok, c_ok = a, a, True, True
    refs = [a_ok, b_ok, c_ok]
    if sum(refs) == 1:                            # exactly one neighbour with the same reference index
        return [a, b, c][refs.index(True)]
    return (_median(a[0], b[0], c[0]), _median(a[1], b[1], c[1]))


PARTS = {0: [(0, 0, 16, 16)], 1: [(0, 0, 16, 8), (0, 8, 16, 8)], 2: [(0, 0, 8, 16), (8, 0, 8, 16)]}
# P_8x8 (mb_type 3): the four 8x8 blocks in order, each split by its sub_mb_type into these sub-partitions
SUB_PARTS = {0: [(0, 0, 8, 8)], 1: [(0, 0, 8, 4), (0, 4, 8, 4)], 2: [(0, 0, 4, 8), (4, 0, 4, 8)],
             3: [(0, 0, 4, 4), (4, 0, 4, 4), (0, 4, 4, 4), (4, 4, 4, 4)]}
B8 = [(0, 0), (8, 0), (0, 8), (8, 8)]


def partitions(mb_type, sub_types=None):
    """Luma rectangles (x, y, w, h) inside the MB, in decoding (and export) order."""
    if mb_type != 3:
        return PARTS[mb_type]
    return [(bx + x, by + y, w, h) for (bx, by), st in zip(B8, sub_types) for (x, y, w, h) in SUB_PARTS[st]]


def _p_slice(frame_num, mbw, mbh, mbs):
    """mbs[my][mx] = (mb_type, [mv per partition]) with mb_type 0 = 16x16, 1 = 16x8, 2 = 8x16."""
    w = BitWriter()
    w.ue(0)                 # first_mb_in_slice
    w.ue(5)                 # slice_type: P (all slices of the picture)
    w.ue(0)                 # pic_parameter_set_id
    w.u(4, frame_num % 16)  # frame_num
    w.u(1, 0)               # num_ref_idx_active_override_flag
    w.u(1, 0)               # ref_pic_list_modification_flag_l0
    w.u(1, 0)               # adaptive_ref_pic_marking_mode_flag
    w.se(0)                 # slice_qp_delta
    w.ue(1)                 # disable_deblocking_filter_idc: off
    f = MvField(mbw, mbh)
    for my in range(mbh):
        for mx in range(mbw):
            mb_type, mvs = mbs[my][mx][:2]
            sub = mbs[my][mx][2] if mb_type == 3 else None
            w.ue(0)         # mb_skip_run
            w.ue(mb_type)   # P_L0_16x16 / P_L0_L0_16x8 / P_L0_L0_8x16 / P_8x8 (one reference: no ref_idx)
            if mb_type == 3:
                for st in sub:
                    w.ue(st)  # sub_mb_type: 8x8 / 8x4 / 4x8 / 4x4
            for pi, (px, py, pw, ph) in enumerate(partitions(mb_type, sub)):
                x, y = 16 * mx + px, 16 * my + py
                pred = predict_partition(f, x, y, pw, ph, pi if mb_type in (1, 2) else 0)
                w.se(mvs[pi][0] - pred[0])   # mvd_l0 x (quarter pel)
                w.se(mvs[pi][1] - pred[1])   # mvd_l0 y
                f.put(x, y, pw, ph, mvs[pi])
            w.ue(0)         # coded_block_pattern 0 (inter me(v) code 0)
    w.trailing()
    return _nal(2, 1, w.bytes())


def write_stream(path, mbw, mbh, mv_frames, seed=0):
    """mv_frames: list over P-frames of [mbh][mbw] entries, each (mvx, mvy) (a 16x16 partition),
    (mb_type, [mv, mv]) (1: two 16x8, 2: two 8x16 partitions) or (3, [mv per sub-partition], [4 sub_mb_types])
    (P_8x8), quarter pel; writes SPS, PPS, an I_PCM IDR picture and one P picture per entry."""
    rng = np.random.default_rng(seed)
    luma = rng.integers(16, 236, size=(16 * mbh, 16 * mbw), dtype=np.uint8)
    cb = rng.integers(16, 240, size=(8 * mbh, 8 * mbw), dtype=np.uint8)
    cr = rng.integers(16, 240, size=(8 * mbh, 8 * mbw), dtype=np.uint8)
    data = _sps(mbw, mbh) + _pps() + _idr(mbw, mbh, luma, cb, cr)
    for i, mvs in enumerate(mv_frames, 1):
        mbs = [[(0, [e]) if isinstance(e[1], int) else e for e in row] for row in mvs]
        data += _p_slice(i, mbw, mbh, mbs)
    with open(path, "wb") as f:
        f.write(data)
