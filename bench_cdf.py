"""bench.py --workload cdf: the NEXT-4 workload.

The paper's motivation analysis (fig:mv_residual_analysis_cdf: "50% of frames contain patches
that are 77%~94% similar when evaluated under motion and residual thresholds") as a GPU pipeline over decoder
exports.  A step = one GOP (16 frames: an I-frame and 15 P-frames) of every stream of the rank:

  codecsight_mv_rasterize   H.264-shaped AVMotionVector records (synth.avmv_records: 16x16 ... 8x8 partitions, as
                            libavcodec exports them (sub-8x8 at 8x8 granularity, tests/test_real_h264.py),
                            skip MBs with their vector, intra MBs without a record) -> the MB grid
  codecsight_score_patches  the grid -> per-patch scores M(i) (Eq. 1-3) + keep masks (GOP state carried)
  codecsight_similar_hist   per P-frame similar-patch counts #{M(i) < tau} for tau in {0.25, 0.5, 1, 2, 5} px,
                            binned into a [n_tau][20] histogram (the CDF over frames is its running sum)

Inputs are device-resident for `value`; `e2e` adds, every step, the H2D copy of the step's records + offsets +
frame types from pinned memory and the D2H read of the histogram.  Algorithmic bytes per kernel (the roofline):
  mv_rasterize    40 B per record read + 8 offsets B per frame + 8 B per MB written
  score_patches   the library's CS_CNT_BYTES_SCORE (8 B per MB of a P-frame + masks, counts, 4 KB of scores)
  similar_hist    4 KB of scores + 1 B type per frame read, the histogram update
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def _grid(cfg):
    sw, sh = cfg["src"]
    return synth.make_grid(sw, sh, tau=cfg["tau"], alpha=cfg["alpha"], group=cfg["group"])


def gen_step(cfg, gens, rng):
    """One GOP of every stream: records [sum], offsets [S*F+1] (stream-major), frame types [S][F]."""
    F, gop = cfg["window"], cfg["gop"]
    types = synth.frame_types(F, gop)
    recs, offs = [], [0]
    for gn in gens:
        for f in range(F):
            mb = gn.next_frame()
            r = synth.avmv_records(mb, rng) if types[f] == synth.FRAME_P else np.zeros(0, synth.AV_MV_DTYPE)
            recs.append(r)
            offs.append(offs[-1] + r.size)
    return np.concatenate(recs), np.array(offs, np.int64), np.stack([types] * len(gens))


def cdf_summary(hist: np.ndarray, taus, n_bins: int) -> dict:
    """Per tau: P-frames counted, the median bin's similar ratio and the share of frames >= 77 % similar."""
    out = {}
    for t, tau in enumerate(taus):
        h = hist[t].astype(np.float64)
        n = h.sum()
        if n == 0:
            continue
        cdf = np.cumsum(h) / n
        med = int(np.searchsorted(cdf, 0.5))
        b77 = int(np.floor(0.77 * n_bins))
        out[str(tau)] = {"p_frames": int(n), "median_similar_ratio_bin": [med / n_bins, (med + 1) / n_bins],
                         "frac_frames_ge_77pct_similar": float(h[b77:].sum() / n)}
    return out


def oracle_sample(cfg, budget_s: float, max_streams: int = 64):
    """The oracle (as it stands) on whole GOPs of streams 0, 1, ...: rasterize + score + histogram, ~budget_s s."""
    import oracle.ref as ref
    g = _grid(cfg)
    nw = (g["grid_w"] * g["grid_h"] + 31) // 32
    taus = np.array(cfg["taus"], np.float32)
    t_tot, frames, si = 0.0, 0, 0
    rng = np.random.default_rng(7)
    while t_tot < budget_s and si < max_streams:
        gn = synth.StreamGen(*cfg["src"], synth.scene_of(cfg, si), synth.stream_seed(cfg, si))
        recs, offs, types = gen_step(cfg, [gn], rng)
        F = types.shape[1]
        t0 = time.perf_counter()
        grid = ref.mv_rasterize(g, recs, offs, F)
        so = ref.score_patches(g, grid[None], types, np.zeros((1, nw + 1), np.uint32), want_score=True)
        ref.similar_hist(so["score"].reshape(F, -1), types[0], taus, cfg["n_bins"])
        t_tot += time.perf_counter() - t0
        frames += F
        si += 1
    return dict(seconds=t_tot, frames=frames, streams=si)


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    per = max(1.0, args.cpu_seconds / max(1, args.steps))
    for _ in range(args.warmup):
        oracle_sample(cfg, 0.0, max_streams=1)
    tot = dict(seconds=0.0, frames=0, streams=0)
    for _ in range(args.steps):
        r = oracle_sample(cfg, per)
        for k in tot:
            tot[k] += r[k]
    fps = tot["frames"] / tot["seconds"]
    from bench import host_cpu_model
    print(json.dumps({
        "impl": "reference", "metric": "frames/sec (NEXT-4: MV ingest + score + similar-patch histogram)", "value": fps,
        "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * tot["seconds"] / args.steps, "higher_is_better": True, "scaling": cfg["scaling"],
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["name"], "streams_per_gpu": cfg["streams"], "gop": cfg["gop"],
                   "taus": list(cfg["taus"]), "n_bins": cfg["n_bins"]},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": 1, "kind": "oracle", "cpu_model": host_cpu_model(),
                         "sample": f"{tot['streams']} whole GOPs (16 frames) of streams 0.., single-threaded C oracle"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)


def run_ours(args, cfg, rank, world, local_rank):
    import torch

    from bench import ClockSampler, host_cpu_model, log, measured_peak_hbm, ncu_traffic
    from paper_2604_06036_b200 import _abi as abi
    from paper_2604_06036_b200 import shard

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    abi.lib()
    g = _grid(cfg)
    ids = shard.shard_ids(rank, world, cfg["streams"], "weak")
    S, F = len(ids), cfg["window"]
    n_fr = S * F
    nmb = g["mb_rows"] * g["mb_cols"]
    nw = abi.grid_words(g)
    taus = torch.tensor(cfg["taus"], dtype=torch.float32, device=dev)
    n_tau, n_bins = len(cfg["taus"]), cfg["n_bins"]
    t_setup = time.time()
    rng = np.random.default_rng(100 + rank)
    gens = [synth.StreamGen(*cfg["src"], synth.scene_of(cfg, gid), synth.stream_seed(cfg, gid)) for gid in ids]
    n_pool = 2
    pool_h, pool_d = [], []
    for _ in range(n_pool):
        recs, offs, types = gen_step(cfg, gens, rng)
        h = (torch.from_numpy(recs.view(np.uint8)).pin_memory(), torch.from_numpy(offs).pin_memory(),
             torch.from_numpy(types).pin_memory())
        pool_h.append(h)
        pool_d.append(tuple(t.to(dev) for t in h))
    grid_d = torch.zeros(n_fr * nmb, dtype=torch.int64, device=dev)          # cs_mb records, 8 B each
    gop_state = torch.zeros(S, nw + 1, dtype=torch.int32, device=dev)
    keep = torch.zeros(S, F, nw, dtype=torch.int32, device=dev)
    score = torch.zeros(n_fr, g["grid_w"] * g["grid_h"], dtype=torch.float32, device=dev)
    kept = torch.zeros(S, F, dtype=torch.int32, device=dev)
    hist = torch.zeros(n_tau, n_bins, dtype=torch.int64, device=dev)
    counters = torch.zeros(abi.NCOUNTERS, dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    if not args.quiet:
        log(f"[rank {rank}] cdf setup {time.time() - t_setup:.1f}s, records/step "
            f"{[int(p[1][-1]) for p in pool_h]}")

    def step(recs, offs, types, timing=False):
        evs = []

        def mark():
            if timing:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                evs.append(e)
        mark()
        abi.codecsight_mv_rasterize(g, n_fr, recs, offs, grid_d, stream)
        mark()
        abi.codecsight_score_patches(g, S, F, grid_d, types, keep, F, gop_state, score, kept, counters, status,
                                     stream)
        mark()
        abi.codecsight_similar_hist(score, types, n_fr, g["grid_w"] * g["grid_h"], taus, n_tau, n_bins, hist, stream)
        mark()
        return evs

    for k in range(args.warmup):
        step(*pool_d[k % n_pool])
    torch.cuda.synchronize()
    cnt0 = counters.clone()
    hist.zero_()
    clocks = ClockSampler(local_rank)
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
    clocks.idx = int(cvd[local_rank]) if len(cvd) > local_rank and cvd[local_rank].strip().isdigit() else local_rank
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    per = []
    ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ta.record(stream)
    for k in range(args.steps):
        per.append(step(*pool_d[k % n_pool], timing=True))
    tb.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = ta.elapsed_time(tb)
    dcnt = (counters - cnt0).cpu().numpy()
    kms = np.array([[e[i].elapsed_time(e[i + 1]) for i in range(3)] for e in per]).mean(axis=0)
    hist_h = hist.cpu().numpy().astype(np.uint64)
    st = int(status.item())

    # ---- e2e: records H2D every step, histogram D2H every step -----------------------------------------------
    e2e = None
    if not args.no_e2e:
        stage = [tuple(torch.empty_like(t) for t in pool_d[0]) for _ in range(2)]
        big = max(int(p[0].numel()) for p in pool_d)
        stage = [(torch.empty(big, dtype=torch.uint8, device=dev), torch.empty_like(pool_d[0][1]),
                  torch.empty_like(pool_d[0][2])) for _ in range(2)]
        res = [torch.empty(n_tau * n_bins, dtype=torch.int64).pin_memory() for _ in range(2)]
        cs = torch.cuda.Stream(dev)
        loaded = [torch.cuda.Event() for _ in range(2)]
        freed = [torch.cuda.Event() for _ in range(2)]
        torch.cuda.synchronize()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        h2d = 0
        for k in range(args.steps):
            b = k & 1
            rh, oh, th = pool_h[k % n_pool]
            with torch.cuda.stream(cs):
                if k >= 2:
                    cs.wait_event(freed[b])
                stage[b][0][:rh.numel()].copy_(rh, non_blocking=True)
                stage[b][1].copy_(oh, non_blocking=True)
                stage[b][2].copy_(th, non_blocking=True)
                loaded[b].record(cs)
            h2d = max(h2d, rh.numel() + oh.numel() * 8 + th.numel())
            stream.wait_event(loaded[b])
            step(stage[b][0], stage[b][1], stage[b][2])
            res[b].copy_(hist.view(-1), non_blocking=True)                    # D2H: the histogram
            freed[b].record(stream)
        eb.record(stream)
        torch.cuda.synchronize()
        e2e = dict(ms=ea.elapsed_time(eb), h2d=h2d, d2h=n_tau * n_bins * 8)

    tens = shard.reduce_max(torch.tensor([ms, e2e["ms"] if e2e else 0.0], dtype=torch.float64, device=dev))
    if rank != 0:
        return
    K = args.steps
    frames_total = S * world * F * K
    ms_max = float(tens[0])
    value = frames_total / (ms_max / 1e3)
    peak, peak_kind = measured_peak_hbm()
    n_rec = float(np.mean([p[1][-1].item() for p in pool_h]))
    b_rast = n_rec * 40 + (n_fr + 1) * 8 + n_fr * nmb * 8
    b_score = float(dcnt[abi.CNT_BYTES_SCORE]) / K
    b_hist = n_fr * (g["grid_w"] * g["grid_h"] * 4 + 1) + n_tau * 4
    rl = {}
    for name, byt, t in (("codecsight_mv_rasterize", b_rast, kms[0]), ("codecsight_score_patches", b_score, kms[1]),
                         ("codecsight_similar_hist", b_hist, kms[2])):
        a = byt / (t / 1e3) / 1e9
        key = {"codecsight_mv_rasterize": "rasterize", "codecsight_score_patches": "score_patches",
               "codecsight_similar_hist": "similar_hist"}[name]
        rl[name] = {"bound": "hbm", "kernel": name, "achieved": a, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                    "frac": a / peak, "ms": float(t), "algorithmic_bytes_per_launch": byt,
                    "traffic": ncu_traffic(key, cfg["name"])}
    dom = max(rl, key=lambda x: rl[x]["ms"])
    out = {
        "metric": "frames/sec (NEXT-4: H.264 MV ingest + score + similar-patch histogram), all GPUs",
        "value": value, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (H.264-shaped AVMotionVector exports drawn from the scene generator)",
        "config": {"workload": cfg["name"], "streams_per_gpu": S, "streams_total": S * world, "src": list(cfg["src"]),
                   "frames_per_step_per_stream": F, "gop": cfg["gop"], "taus": list(cfg["taus"]),
                   "n_bins": n_bins, "records_per_step": n_rec, "parallelism": f"stream-shard x{world}",
                   "l2": "inputs larger than L2 (records + grid + scores of one step)"},
        "per_kernel_ms": {k: v["ms"] for k, v in rl.items()},
        "roofline": rl[dom], "rooflines": rl,
        "cdf": cdf_summary(hist_h, cfg["taus"], n_bins),
        "paper_context": "P:211: 50% of UCF-Crime frames have 77-94% similar patches under motion/residual thresholds",
        "status": st, "gpu_launches": 3 * K, "clocks": clk, "host_cpu": host_cpu_model(),
    }
    if e2e:
        out["e2e"] = {"value": frames_total / (float(tens[1]) / 1e3), "unit": "frames/s",
                      "h2d_bytes_per_step": e2e["h2d"] * world, "d2h_bytes_per_step": e2e["d2h"] * world}
    if not args.no_cpu_baseline and world == 1:
        r = oracle_sample(cfg, min(args.cpu_seconds, 10.0))
        out["cpu_baseline"] = {"value": r["frames"] / r["seconds"], "unit": "frames/s", "cores": 1, "kind": "oracle",
                               "cpu_model": host_cpu_model(),
                               "sample": f"{r['streams']} whole GOPs of streams 0.., single-threaded C oracle "
                                         f"(rasterize + score + histogram), {r['seconds']:.1f} s"}
    print(json.dumps(out), flush=True)
