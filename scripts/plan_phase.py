"""Experiment: where kv_plan_paged's time goes.  kv_refresh.cu built with -DCS_PLAN_TIMING into
build/libcodecsight_plan.so stamps %globaltimer per CTA (one CTA = one stream) at the phase boundaries; this runs the
bench's pipeline on a workload (C4 default) for a few steps and prints the median / max phase lengths of the last
plan launch.  Phases: 0 start -> 1 masks loaded + per-frame counts -> 2 serial segment table -> 3 survivors (slots of
the previous window, move entries) -> 4 free-slot scan -> 5 NEW tokens -> 6 run starts counted + scanned -> 7 runs
written -> 8 cos/sin table + counters."""
import ctypes as C
import os
import sys
import types as _t

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2604_06036_b200 import _abi as abi  # noqa: E402

abi.LIB_PATH = os.path.join(ROOT, "build", "libcodecsight_plan.so")
from paper_2604_06036_b200.pipeline import Pipeline  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "C4"
    L = abi.lib()
    L.codecsight_debug_plan_phase.restype = C.c_int
    L.codecsight_debug_plan_phase.argtypes = [C.c_void_p, C.c_int]
    dev = torch.device("cuda", 0)
    cfg = bench.workload(wl, None, "paged", _t.SimpleNamespace(tau=0.25, alpha=0.0))
    sw, sh = cfg["src"]
    g = synth.make_grid(sw, sh)
    S, w, s, gop = cfg["streams"], cfg["window"], cfg["stride"], cfg["gop"]
    pipe = Pipeline(g, S, w, s, gop, cfg["kv"], n_prompt=cfg["n_prompt"], device=dev,
                    frame_layout=abi.CS_LAYOUT_GROUPED, kv_mode="paged", compact_chunk=s, fused=True)
    md = bench.gen_metadata(cfg, list(range(S)), 3)
    mb = [torch.from_numpy(m.view(np.uint8).copy()).to(dev) for m in md]
    fr = torch.randn(3, 448, 448, device=dev).to(torch.bfloat16)
    ptr_w = abi.ptr_array([fr] * (S * w), dev)
    ptr_s = abi.ptr_array([fr] * (S * s), dev)
    for k in range(6):
        f0, n = bench.step_frames(cfg, k)
        ty = torch.from_numpy(np.stack([synth.frame_types(n, gop, f0)] * S)).to(dev)
        fi = torch.from_numpy(np.tile(np.arange(f0, f0 + n, dtype=np.int32), S)).to(dev)
        pipe.step(k, mb[0] if k == 0 else mb[1 + (k - 1) % 3], ptr_w if k == 0 else ptr_s, fi, ty)
    torch.cuda.synchronize()
    h = np.zeros((S, 10), np.uint64)
    assert L.codecsight_debug_plan_phase(h.ctypes.data, S) == 0
    t0 = h[:, 0].min()
    print(f"{wl}: {S} CTAs, span {(h[:, 8].max() - t0) / 1e3:.1f} us (first start -> last end)")
    print(f"  start offsets: median {np.median(h[:, 0] - t0) / 1e3:.1f} us, max {(h[:, 0] - t0).max() / 1e3:.1f}")
    names = ["masks+counts", "serial table", "survivors", "free scan", "NEW tokens", "run count+scan", "runs write",
             "cos/sin+ctr"]
    for i, nm in enumerate(names):
        d = (h[:, i + 1].astype(np.int64) - h[:, i].astype(np.int64)) / 1e3
        print(f"  {i}->{i + 1} {nm:15s} median {np.median(d):7.2f} us   max {d.max():7.2f}")


if __name__ == "__main__":
    main()
