"""Where the C2 step time goes beyond the fused kernel: the same steps enqueued with / without per-kernel timing
events, with / without the frame-type ring copy, and the bare fused call back to back (one B200)."""
import os
import sys
import types as _t

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2604_06036_b200 import _abi as abi  # noqa: E402
from paper_2604_06036_b200.pipeline import Pipeline  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    args = _t.SimpleNamespace(tau=0.25, alpha=0.0)
    cfg = bench.workload(os.environ.get("WL", "C2"), None, "paged", args)
    sw, sh = cfg["src"]
    g = synth.make_grid(sw, sh, tau=cfg["tau"], alpha=cfg["alpha"])
    S, w, s, gop = cfg["streams"], cfg["window"], cfg["stride"], cfg["gop"]
    pipe = Pipeline(g, S, w, s, gop, None, n_prompt=0, device=dev, frame_layout=abi.CS_LAYOUT_GROUPED,
                    kv_mode="paged", compact_chunk=s, fused=True)
    md = bench.gen_metadata(cfg, list(range(S)), 8)
    mb_dev = [torch.from_numpy(m.view(np.uint8).copy()).to(dev) for m in md]
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    H = g["grid_h"] * g["patch"]
    frames = [torch.randn(3, H, H, generator=gen, device=dev).to(torch.bfloat16) for _ in range(S * s)]
    ptr_w = abi.ptr_array([frames[i % len(frames)] for i in range(S * w)], dev)
    ptr_s = abi.ptr_array(frames, dev)
    N = 200
    tys, fis = [], []
    for k in range(N + 40):
        f0, n = bench.step_frames(cfg, k)
        tys.append(torch.from_numpy(np.stack([synth.frame_types(n, gop, f0)] * S)).to(dev))
        fis.append(torch.from_numpy(np.tile(np.arange(f0, f0 + n, dtype=np.int32), S)).to(dev))
    stream = torch.cuda.current_stream(dev)
    k = [0]

    def step(timing, with_types):
        kk = k[0]
        k[0] += 1
        mb = mb_dev[0] if kk == 0 else mb_dev[1 + (kk - 1) % 8]
        pipe.step(kk, mb, ptr_w if kk == 0 else ptr_s, fis[kk], tys[kk] if (with_types or kk < 2) else None,
                  timing=timing)

    for _ in range(20):
        step(False, True)
    torch.cuda.synchronize()

    def timeit(fn, n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(n):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3

    # NB: keep k advancing so the GOP / ring phases are those of a real run
    for name, fn in (("step timing=True  types copy", lambda: step(True, True)),
                     ("step timing=False types copy", lambda: step(False, True)),
                     ("step timing=False no types", lambda: step(False, False)),
                     ("step timing=True  types copy", lambda: step(True, True))):
        k[0] = 20
        print(f"{name}: {timeit(fn, 100):.1f} us/step", flush=True)
    # bare fused call, same ring slot, back to back
    f0, n = bench.step_frames(cfg, 20)
    off = f0 % pipe.ring
    call = pipe._bound[(off, n)]
    mb = mb_dev[1]
    print(f"bare fused call: {timeit(lambda: call(mb, fis[20], ptr_s, stream.cuda_stream), 100):.1f} us/call")
    x = torch.empty(S, n, dtype=torch.uint8, device=dev)
    print(f"types copy alone: {timeit(lambda: pipe.type_ring[:, off:off + n].copy_(x), 100):.1f} us")


if __name__ == "__main__":
    main()
