"""Time codecsight_compact_nv12 on a C4-shaped batch (256 streams x 4 frames of 1080p NV12, group masks with the
bench's kept fraction) for each library variant given on the command line (built with different
CS_NV12_BATCH / CS_NV12_CTAS).  One B200; CUDA events, 20 launches after 5 warm-up launches."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
from paper_2604_06036_b200 import _abi as abi  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    sw, sh = 1920, 1080
    g = synth.make_grid(sw, sh)
    S, n = 256, 4
    rng = np.random.default_rng(5)
    nw = abi.grid_words(g)
    # kept groups ~0.5: per frame a random set of 2x2 groups (group-complete masks)
    grp = rng.random((S, n, 16, 16)) < 0.53
    pm = np.repeat(np.repeat(grp, 2, axis=2), 2, axis=3)          # [S][n][32][32] patch bits
    km = np.packbits(pm.reshape(S, n, 32, 32)[..., ::-1], axis=-1, bitorder="big").view(">u4").astype(np.uint32)
    km = km.reshape(S, n, nw)
    gen = torch.Generator(device=dev)
    gen.manual_seed(3)
    nf = S * n
    ys = [torch.randint(16, 236, (sh, sw), dtype=torch.uint8, device=dev, generator=gen) for _ in range(nf)]
    uvs = [torch.randint(16, 241, (sh // 2, sw), dtype=torch.uint8, device=dev, generator=gen) for _ in range(nf)]
    km_d = torch.from_numpy(km.view(np.int32)).to(dev)
    fidx = torch.arange(nf, dtype=torch.int32, device=dev)
    cap = nf * 1024
    packed = torch.empty((cap, 588), dtype=torch.int16, device=dev)
    pos = torch.empty(cap, 3, dtype=torch.int32, device=dev)
    src = torch.empty(cap, dtype=torch.int32, device=dev)
    offs = torch.empty(nf + 1, dtype=torch.int32, device=dev)
    cnt = torch.zeros(16, dtype=torch.int64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    yp, uvp = abi.ptr_array(ys, dev), abi.ptr_array(uvs, dev)
    pre = dict(src_w=sw, src_h=sh, y_pitch=sw, uv_pitch=sw)
    ref_out = None
    for path in sys.argv[1:]:
        abi._lib = None
        abi.LIB_PATH = path
        run = lambda: abi.codecsight_compact_nv12(g, pre, S, n, km_d, n, fidx, yp, uvp, cap, packed, pos, src,  # noqa
                                                 offs, cnt, st)
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            run()
        b.record()
        torch.cuda.synchronize()
        rows = int(offs[-1].item())
        out = packed[:rows].clone()
        same = "" if ref_out is None else ("identical" if torch.equal(out, ref_out) else "DIFFERENT")
        ref_out = out if ref_out is None else ref_out
        print(f"{os.path.basename(path)}: {a.elapsed_time(b) / 20:.4f} ms, rows {rows} {same}", flush=True)


if __name__ == "__main__":
    main()
