#!/usr/bin/env python3
"""Benchmark of the CodecSight hot path on B200 (BASELINE.json metric: codec-pruned frames/s per GPU and
streams/s at 1/2/4/8 GPUs, KV-refresh GB/s vs HBM).

A step = one pass of the whole hot path for every stream of the rank:
  codecsight_score_patches (s new frames/stream) -> codecsight_compact -> codecsight_kv_refresh (window k).
Workload (default C4, BASELINE configs[3]): 256 1080p streams in total, even ids static / odd ids high-motion,
w = 16, s = 4, GOP 16, Qwen2-VL-7B KV (28 x 4 x 128 bf16), 32 prompt rows, sharded over the N GPUs (strong scaling,
snake-order stream assignment, paper_2604_06036_b200/shard.py); C5 runs 128 4K streams per GPU (weak scaling).
No collective on the data path; one NCCL all_reduce of counters, a MAX of the device time and a gather of the
per-rank times after the timed loop.  --workload cdf: the NEXT-4 similar-patch analysis (bench_cdf.py).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4|C5|C3|C2|cdf] [--scaling strong|weak]
                    [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)   # 10 warm-up steps, >= 50 timed
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--streams", type=int, default=None,
                    help="streams: the total under --scaling strong, per GPU under weak (default: the config's)")
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"],
                    help="strong: the workload's streams split over the GPUs (C4: 256 streams 'sharded over 2/4/8 "
                         "B200'); weak: that many streams on every GPU (C5: 128 per GPU, 1,024 on 8).  Default: "
                         "strong for C4, weak otherwise")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tau", type=float, default=0.25, help="Eq. 4 threshold in source px (P:459)")
    ap.add_argument("--alpha", type=float, default=0.0, help="Eq. 3 residual weight (P:299)")
    ap.add_argument("--group-size", type=int, default=2,
                    help="patches per token edge (2x2 groups -> one LLM token, P:304; SPEC --group-size)")
    ap.add_argument("--window-frames", type=int, default=None, help="window w (default: the workload's)")
    ap.add_argument("--stride-frames", type=int, default=None, help="stride s (default: the workload's)")
    ap.add_argument("--gop", type=int, default=None, help="I-frame period (default: the workload's)")
    ap.add_argument("--pool", type=int, default=6, help="distinct metadata steps kept on the device")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--cpu-all-cores", action=argparse.BooleanOptionalAction, default=True,
                    help="also time the oracle as one process per host core (SURVEY §8(d)(ii))")
    ap.add_argument("--quiet", action="store_true")
    ap.add_argument("--overlap", action=argparse.BooleanOptionalAction, default=None,
                    help="run step k's compaction / kv_refresh on side streams while step k+1's scoring runs (default: "
                         "on for workloads with a KV refresh, unless --pdl / --graphs / --temporal-patch 2; measured, "
                         "same box: C4 6.43 -> 6.38 ms, 32 streams per GPU (C4 strong-scaled to 8 GPUs) 0.941 -> 0.917 "
                         "ms, NV12 C4 6.85 -> 6.72 ms; --no-overlap for the sequential step)")
    ap.add_argument("--fused", action=argparse.BooleanOptionalAction, default=True,
                    help="one codecsight_score_compact launch per step (NEXT-2, default) instead of score_patches + "
                         "compact (--no-fused)")
    ap.add_argument("--pdl", action=argparse.BooleanOptionalAction, default=None,
                    help="prune-only workloads (C2): launch each step's fused score+compact as a programmatic dependent "
                         "of the previous step's (CS_LAUNCH_PDL), so its scoring overlaps the previous compaction; the "
                         "kernel time is then the timed region / K (no per-kernel events between the launches); "
                         "default: on for prune-only workloads with the fused call and no --graphs")
    ap.add_argument("--chain-depth", type=int, default=4,
                    help="--pdl: output buffer sets the chained calls rotate (call g reuses call g - depth's)")
    ap.add_argument("--graphs", action="store_true",
                    help="replay steps k >= 1 as captured CUDA graphs (one per ring phase and slot parity)")
    ap.add_argument("--temporal-patch", type=int, default=1, choices=[1, 2],
                    help="frames per visual token (Qwen2-VL video: 2; NEXT-3); KV refresh over token units")
    ap.add_argument("--kv-mode", default="paged", choices=["paged", "copy"],
                    help="paged: codecsight_kv_refresh_paged (in place, NEXT-1); copy: out-of-place double buffer")
    ap.add_argument("--rope", default="1d", choices=["1d", "mrope"],
                    help="key position scheme: 1-D on compacted sequence indices (Q16) or Qwen2-VL M-RoPE (NEXT-3)")
    ap.add_argument("--frames", default="model", choices=["model", "nv12"],
                    help="model: preprocessed model-input frames; nv12: decoded NV12 frames, preprocessing fused into "
                         "the compaction (codecsight_compact_nv12, NEXT-2)")
    ap.add_argument("--frame-layout", default="grouped", choices=["grouped", "planar"],
                    help="layout of the preprocessed model-input frames handed to compact (DESIGN.md §6)")
    return ap.parse_args()


SCENE_KINDS = list(synth.SCENES)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------------------------------------------
# workload
# --------------------------------------------------------------------------------------------------------------
def workload(name: str, streams: int | None, kv_mode: str = "paged", args=None):
    name = name.upper()
    cfg = dict(synth.CONFIGS[name])
    # method parameters (SPEC CLI names): defaults are the paper's (tau 0.25 px, alpha 0)
    cfg["tau"] = getattr(args, "tau", 0.25)
    cfg["alpha"] = getattr(args, "alpha", 0.0)
    cfg["group"] = getattr(args, "group_size", 2)
    if cfg["group"] < 1 or 32 % cfg["group"] or cfg["group"] * 14 > 32:
        raise SystemExit("--group-size: 1 or 2 (it must divide the 32x32 patch grid, and group * patch <= 32 px is "
                         "the compaction's warp tile, include/codecsight.h); group 1 has 4x the tokens of group 2, so "
                         "the KV caches of a workload need 4x the memory (use --streams)")
    for key, opt in (("window", "window_frames"), ("stride", "stride_frames"), ("gop", "gop")):
        v = getattr(args, opt, None)
        if v is not None:
            cfg[key] = v
    if not 1 <= cfg["stride"] <= cfg["window"]:
        raise SystemExit("need 1 <= stride <= window (S:129)")
    if cfg["kv"] is None and name not in ("C2", "CDF"):
        raise SystemExit(f"workload {name} has no KV shape")
    if name == "C5":
        # BASELINE: 1,024 streams on 8 B200 -> 128 streams per GPU (weak scaling unit).  Out of place, 128 x 2 x
        # 941 MB caches exceed 180 GB: C5 runs with the in-place / paged refresh only.
        cfg["streams"] = 128
        if kv_mode != "paged":
            raise SystemExit("C5 needs --kv-mode paged (out-of-place caches do not fit one GPU)")
    if streams is not None:
        cfg["streams"] = streams
    # BASELINE configs[3] (C4): a fixed set of 256 streams sharded over 1/2/4/8 GPUs -> strong scaling; C5 is quoted
    # per GPU (1,024 streams on 8 = 128 each) -> weak; C2 / C3 are single-GPU configs (N > 1 replicates them)
    cfg["scaling"] = getattr(args, "scaling", None) or ("strong" if name == "C4" else "weak")
    return cfg


def host_cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def step_frames(cfg, k):
    w, s = cfg["window"], cfg["stride"]
    return (0, w) if k == 0 else ((k - 1) * s + w, s)


def gen_metadata(cfg, global_ids, n_pool):
    """MB metadata: entry 0 = the first window (w frames), entries 1..n_pool = stride steps (s frames each) that
    the timed loop cycles through.  Each stream's scene evolves in time; the first window re-uses the pool's
    frames (it is warm-up only)."""
    sw, sh = cfg["src"]
    w, s = cfg["window"], cfg["stride"]
    gens = [synth.StreamGen(sw, sh, synth.scene_of(cfg, gid), synth.stream_seed(cfg, gid)) for gid in global_ids]
    pool = [np.stack([np.stack([gn.next_frame() for _ in range(s)]) for gn in gens]) for _ in range(n_pool)]
    first = np.concatenate([pool[i % n_pool] for i in range(-(-w // s))], axis=1)[:, :w]
    return [np.ascontiguousarray(first)] + pool


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while the timed region runs."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic(kernel: str, workload: str):
    """DRAM bytes per launch of `kernel` from the committed ncu launch list, if it was captured on this workload."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        summ = json.load(f)
    d = summ.get(f"{kernel}@{workload}", summ.get(kernel, {}))
    return d.get("dram_bytes_per_launch") if d.get("workload") == workload else None


# --------------------------------------------------------------------------------------------------------------
# CPU oracle (baseline / reference arm)
# --------------------------------------------------------------------------------------------------------------
def oracle_sample(cfg, budget_s: float, max_steps: int = 64, kv_mode: str = "paged", tp: int = 1, sid0: int = 0,
                  sid_step: int = 1):
    """Run the oracle, as it stands, on a bounded sample of the workload: whole stream-steps (score + compact +
    kv_refresh) of streams sid0, sid0 + sid_step, ..., until ~budget_s seconds of single-threaded CPU work are
    spent."""
    import oracle.ref as ref
    sw, sh = cfg["src"]
    g = synth.make_grid(sw, sh, tau=cfg["tau"], alpha=cfg["alpha"], group=cfg["group"])
    w, s, gop = cfg["window"], cfg["stride"], cfg["gop"]
    ring = w + s
    nw = (g["grid_w"] * g["grid_h"] + 31) // 32
    kvb = cfg["kv"]
    groups = (g["grid_w"] // 2) * (g["grid_h"] // 2)
    wu, su, uring = w // tp, s // tp, ring // tp
    cap = wu * groups + cfg["n_prompt"]
    rcap = (su + 1 + math.ceil(max(0, wu - su) / max(1, gop // tp))) * groups + cfg["n_prompt"]
    kv = dict(kvb, capacity=cap, refresh_capacity=rcap, n_prompt=cfg["n_prompt"]) if kvb else None
    rng = np.random.default_rng(0)
    frames = synth.random_frames(w, g["grid_h"] * g["patch"], g["grid_w"] * g["patch"], rng)
    t_total, frames_done, steps_done, streams = 0.0, 0, 0, []
    k_meas = 4  # a steady-state window (k >= 1): s new frames + a KV refresh with reuse
    sid = sid0
    while t_total < budget_s and steps_done < max_steps:
        gid = sid
        sid += sid_step
        # stream state up to window k_meas-1 (setup, untimed), then the timed stream-step k_meas
        gen = synth.StreamGen(sw, sh, synth.scene_of(cfg, gid), synth.stream_seed(cfg, gid))
        gop_h = np.zeros((1, nw + 1), np.uint32)
        mring = np.zeros((1, ring, nw), np.uint32)
        tring = np.zeros((1, ring), np.uint8)
        umring = np.zeros((1, uring, nw), np.uint32) if tp > 1 else mring
        utring = np.zeros((1, uring), np.uint8) if tp > 1 else tring

        def do_step(k, timed):
            f0, n = step_frames(cfg, k)
            mb = np.stack([gen.next_frame() for _ in range(n)])[None]
            off = f0 % ring
            tring[0, off:off + n] = synth.frame_types(n, gop, f0)
            t0 = time.perf_counter()
            so = ref.score_patches(g, mb, np.ascontiguousarray(tring[:, off:]), gop_h, frame_stride=ring - off,
                                   want_score=False)
            mring[0, off:off + n] = so["keep_mask"][0, :n]
            if tp > 1:
                co = ref.compact_tp(g, tp, mring[:, off:].copy(), np.arange(f0 // tp, (f0 + n) // tp, dtype=np.int32),
                                    frames[:n], n // tp * g["grid_w"] * g["grid_h"], 1, n // tp,
                                    mask_frame_stride=ring - off, want_unit_mask=True,
                                    frame_type=np.ascontiguousarray(tring[:, off:]))
                umring[0, off // tp:(off + n) // tp] = co["unit_mask"][0]
                utring[0, off // tp:(off + n) // tp] = co["unit_type"][0]
            else:
                ref.compact(g, mring[:, off:].copy(), np.arange(f0, f0 + n, dtype=np.int32), frames[:n],
                            n * g["grid_w"] * g["grid_h"], 1, n, mask_frame_stride=ring - off)
            t1 = time.perf_counter()
            return t1 - t0, mb

        for k in range(k_meas):
            do_step(k, False)
        dt, _ = do_step(k_meas, True)
        if kv is not None:
            dtp = np.uint16 if kv["dtype"] == 0 else np.float32
            shape = (kv["layers"], 2, cap, kv["kv_heads"], kv["head_dim"])
            rshape = (kv["layers"], 2, rcap, kv["kv_heads"], kv["head_dim"])
            old = np.zeros(shape, dtp)
            if dtp == np.uint16:
                old[...] = rng.integers(0, 65536, size=(1,), dtype=np.uint16)  # content irrelevant to the timing
            new = np.zeros(shape, dtp)
            refr = np.zeros(rshape, dtp)
            win = dict(window=wu, stride=su, step=k_meas, ring_frames=uring)
            if kv_mode == "paged":
                slot_old = np.arange(cap, dtype=np.int32)[None]     # any valid slot map of window k-1
                t0 = time.perf_counter()
                ref.kv_refresh_paged(g, kv, win, umring, utring, [old], slot_old, cap, [refr], cap)
                dt += time.perf_counter() - t0
            else:
                t0 = time.perf_counter()
                ref.kv_refresh(g, kv, win, umring, utring, [old], [new], [refr], cap)
                dt += time.perf_counter() - t0
        t_total += dt
        frames_done += s
        steps_done += 1
        streams.append(synth.scene_of(cfg, gid))
    return dict(seconds=t_total, frames=frames_done, stream_steps=steps_done, scenes=streams)


def _oracle_worker(a):
    cfg, budget_s, max_steps, kv_mode, tp, sid0 = a
    return oracle_sample(cfg, budget_s, max_steps=max_steps, kv_mode=kv_mode, tp=tp, sid0=sid0)


class OraclePool:
    """one single-threaded oracle process per host core (bounded by host memory and 32).  Each
    `run` gives worker i its own consecutive streams (2000 i + offset, 2000 i + offset + 1, ...: the same scene mix
    as the single-core sample) for ~budget_s seconds; the aggregate rate is the sum of frames over the max of the
    workers' oracle seconds (they run concurrently)."""

    def __init__(self, cfg, kv_mode: str, tp: int):
        import concurrent.futures as cf
        import multiprocessing as mp
        self.cfg, self.kv_mode, self.tp, self.offset = cfg, kv_mode, tp, 0
        self.host_cpus = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
        kvb = cfg["kv"]
        per_proc = 0.7e9
        if kvb is not None:   # old + new cache + recompute buffer of one stream, bf16
            rows = (cfg["window"] // tp) * (32 // cfg.get("group", 2)) ** 2 + cfg["n_prompt"]
            per_proc += 3.0 * rows * kvb["layers"] * 2 * kvb["kv_heads"] * kvb["head_dim"] * 2
        try:
            with open("/proc/meminfo") as f:
                avail = next(int(ln.split()[1]) * 1024 for ln in f if ln.startswith("MemAvailable"))
        except (OSError, StopIteration):
            avail = 16e9
        self.P = int(max(1, min(self.host_cpus, 32, avail * 0.5 // per_proc)))
        self.ex = cf.ProcessPoolExecutor(max_workers=self.P, mp_context=mp.get_context("spawn"))

    def run(self, budget_s: float, max_steps: int = 64):
        args = [(self.cfg, budget_s, max_steps, self.kv_mode, self.tp, 2000 * i + self.offset) for i in range(self.P)]
        rs = list(self.ex.map(_oracle_worker, args))
        self.offset += 2 * max_steps
        return dict(frames=sum(r["frames"] for r in rs), stream_steps=sum(r["stream_steps"] for r in rs),
                    seconds=max(r["seconds"] for r in rs))

    def close(self):
        self.ex.shutdown()


def oracle_all_cores(cfg, budget_s: float, kv_mode: str, tp: int):
    """The all-cores oracle rate on one bounded sample; None if the processes cannot be started."""
    try:
        pool = OraclePool(cfg, kv_mode, tp)
        try:
            r = pool.run(budget_s)
        finally:
            pool.close()
    except Exception as e:  # noqa: BLE001
        log(f"[rank 0] all-cores oracle baseline unavailable: {e}")
        return None
    return dict(value=r["frames"] / r["seconds"], processes=pool.P, host_cpus=pool.host_cpus, **r)


def run_reference(args, cfg, rank, world):
    """The reference arm: the oracle, as it stands, on the host cores (one single-threaded process per core, see
    OraclePool; --no-cpu-all-cores: one process), each step a bounded sample of the workload."""
    if rank != 0:
        return
    per_step = max(1.0, args.cpu_seconds / max(1, args.steps))
    pool = None
    if args.cpu_all_cores:
        try:
            pool = OraclePool(cfg, args.kv_mode, args.temporal_patch)
        except Exception as e:  # noqa: BLE001
            log(f"[reference] process pool unavailable ({e}); single process")

    def sample(budget, max_steps):
        if pool is not None:
            return pool.run(budget, max_steps=max_steps)
        return oracle_sample(cfg, budget, max_steps=max_steps, kv_mode=args.kv_mode, tp=args.temporal_patch)

    for _ in range(args.warmup):
        sample(0.0, 1)
    tot = dict(seconds=0.0, frames=0, stream_steps=0)
    for _ in range(args.steps):
        r = sample(per_step, 4)
        for kk in tot:
            tot[kk] += r[kk]
    cores = pool.P if pool is not None else 1
    if pool is not None:
        pool.close()
    fps = tot["frames"] / tot["seconds"]
    out = {"impl": "reference", "metric": "codec-pruned frames/sec (whole hot path: score+compact+kv_refresh), all GPUs",
           "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1000.0 * tot["seconds"] / args.steps, "higher_is_better": True,
           "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
           "config": {"workload": cfg["name"], "streams_total": cfg["streams"] * (1 if cfg["scaling"] == "strong"
                                                                                   else world),
                      "window": cfg["window"],
                      "stride": cfg["stride"], "gop": cfg["gop"], "tau": cfg["tau"], "alpha": cfg["alpha"], "group": cfg["group"],
                      "temporal_patch": args.temporal_patch},
           "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "oracle",
                            "cpu_model": host_cpu_model(),
                            "sample": f"{tot['stream_steps']} whole stream-steps (k=4) of alternating "
                                      f"static/high-motion streams, {cores} concurrent single-threaded C oracle "
                                      f"process(es)"},
           "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------------------------------------------
def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2604_06036_b200 import _abi as abi
    from paper_2604_06036_b200 import shard
    from paper_2604_06036_b200.pipeline import Pipeline

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    abi.lib()
    sw, sh = cfg["src"]
    g = synth.make_grid(sw, sh, tau=cfg["tau"], alpha=cfg["alpha"], group=cfg["group"])
    w, s, gop = cfg["window"], cfg["stride"], cfg["gop"]
    scaling = cfg["scaling"]
    global_ids = shard.shard_ids(rank, world, cfg["streams"], scaling)
    S = len(global_ids)                     # this rank's streams
    S_total = cfg["streams"] if scaling == "strong" else cfg["streams"] * world
    if S == 0:
        raise SystemExit(f"rank {rank}: no streams ({cfg['streams']} streams over {world} ranks)")
    kvb = cfg["kv"]
    if kvb is not None and args.rope == "mrope":
        kvb = dict(kvb, rope_mode=1, mrope_section=(16, 24, 24), t_per_frame=1)
    layout = abi.CS_LAYOUT_GROUPED if args.frame_layout == "grouped" else abi.CS_LAYOUT_PLANAR
    pre = dict(src_w=sw, src_h=sh, y_pitch=sw, uv_pitch=sw) if args.frames == "nv12" else None
    if args.pdl is None:  # default: chained steps for prune-only workloads
        args.pdl = kvb is None and args.fused and not args.graphs and not args.overlap and args.temporal_patch == 1 \
            and args.frames == "model"
    if args.overlap is None:  # default: pipelined steps wherever the Pipeline supports them
        args.overlap = kvb is not None and not args.pdl and not args.graphs and args.temporal_patch == 1
    if args.pdl and (kvb is not None or not args.fused or args.overlap or args.graphs):
        raise SystemExit("--pdl: prune-only workload (C2), fused score+compact, no --overlap / --graphs")
    pipe = Pipeline(g, S, w, s, gop, kvb, n_prompt=cfg["n_prompt"], device=dev, frame_layout=layout,
                    kv_mode=args.kv_mode, compact_chunk=s, preprocess=pre, overlap=args.overlap,
                    temporal_patch=args.temporal_patch, fused=args.fused, pdl=args.pdl, chain_depth=args.chain_depth)
    tp = args.temporal_patch
    # --graphs: steps k >= 1 are CUDA graph replays, one graph per (ring phase, slot parity); the warm-up covers a
    # whole cycle of keys so that no capture happens inside a timed region
    period = pipe.uring // math.gcd(pipe.uring, pipe.su)
    warm = max(args.warmup, 2 * period + 2) if args.graphs else args.warmup
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    pipe.init_cache_fill(gen)
    t_setup = time.time()
    # metadata pool: step 0 (w frames) + `pool` stride steps, cycled during the run
    n_pool = max(1, min(args.pool if cfg["src"][0] < 3000 else min(args.pool, 3), warm + args.steps))
    md = gen_metadata(cfg, global_ids, n_pool)
    mb_host = [torch.from_numpy(m.view(np.uint8).copy()).pin_memory() for m in md]
    mb_dev = [t.to(dev) for t in mb_host]
    # frames: S*s distinct model-input frames [3][448][448] bf16 (pointer array aliases them for the first window)
    H, W = g["grid_h"] * g["patch"], g["grid_w"] * g["patch"]
    if args.frames == "nv12":
        # decoded frames as NVDEC delivers them: Y [sh][sw] + interleaved UV [sh/2][sw], u8
        ys = [torch.randint(16, 236, (sh, sw), dtype=torch.uint8, device=dev, generator=gen) for _ in range(S * s)]
        uvs = [torch.randint(16, 241, (sh // 2, sw), dtype=torch.uint8, device=dev, generator=gen)
               for _ in range(S * s)]
        ptr_w = (abi.ptr_array([ys[i % len(ys)] for i in range(S * w)], dev),
                 abi.ptr_array([uvs[i % len(uvs)] for i in range(S * w)], dev))
        ptr_s = (abi.ptr_array(ys, dev), abi.ptr_array(uvs, dev))
    else:
        frames = [torch.randn(3, H, W, generator=gen, device=dev).to(torch.bfloat16) for _ in range(S * s)]
        ptr_w = abi.ptr_array([frames[i % len(frames)] for i in range(S * w)], dev)
        ptr_s = abi.ptr_array(frames, dev)
    # eager sequential steps after the timed loop whose per-kernel events give the per-call times and rooflines (the
    # timed steps record no events: an event between two calls costs a few us of a small step; inside graphs there
    # are none; in overlap mode a side-stream call's events would also cover the time it waits for SMs held by the
    # other stream's kernel).  Chained (--pdl) calls overlap each other: their time is the timed region / K.
    calib = 2 * period if args.graphs else (0 if args.pdl else min(max(args.steps, 4), 10))
    total_steps = warm + args.steps + calib
    types_dev, fidx_dev, types_host = [], [], []
    for k in range(total_steps + 1):
        f0, n = step_frames(cfg, k)
        t = np.stack([synth.frame_types(n, gop, f0)] * S)
        types_host.append(torch.from_numpy(t).pin_memory())
        types_dev.append(types_host[-1].to(dev))
        fidx_dev.append(torch.from_numpy(np.tile(np.arange(f0 // tp, (f0 + n) // tp, dtype=np.int32), S)).to(dev))
    torch.cuda.synchronize()
    if not args.quiet:
        free, tot = torch.cuda.mem_get_info(dev)
        log(f"[rank {rank}] setup {time.time() - t_setup:.1f}s, device memory used {(tot - free) / 1e9:.1f} GB")

    stream = torch.cuda.current_stream(dev)

    def md_for(k):
        return mb_dev[0] if k == 0 else mb_dev[1 + (k - 1) % n_pool]

    # ---- device-resident timed loop ------------------------------------------------------------------------
    ev = {name: [] for name in ("score", "compact", "kv")}

    # fixed staging buffers (graph inputs; the e2e loop uploads into the same ones)
    stage = [dict(mb=torch.empty_like(mb_dev[1 if len(mb_dev) > 1 else 0]), ty=torch.empty_like(types_dev[1]),
                  fi=torch.empty_like(fidx_dev[1])) for _ in range(2)]

    def run_step_eager(k):
        evs = pipe.step(k, md_for(k), ptr_s, fidx_dev[k], types_dev[k], timing=True)
        for name in ("score", "compact", "kv"):
            if name in evs:
                ev[name].append(evs[name])

    def run_step(k, timed):
        _, n = step_frames(cfg, k)
        ptrs = ptr_w if k == 0 else ptr_s
        if args.graphs and k >= 1:
            st = stage[k & 1]
            st["mb"].copy_(md_for(k), non_blocking=True)    # stage this step's inputs (device copies)
            st["ty"].copy_(types_dev[k], non_blocking=True)
            st["fi"].copy_(fidx_dev[k], non_blocking=True)
            pipe.graph_step(k, st["mb"], ptrs, st["fi"], st["ty"])
            return
        pipe.step(k, md_for(k), ptrs, fidx_dev[k], types_dev[k])

    for k in range(warm):
        run_step(k, False)
    pipe.join(stream)
    torch.cuda.synchronize()
    cnt0 = pipe.counters.clone()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(torch.cuda.get_device_properties(dev).index if hasattr(
        torch.cuda.get_device_properties(dev), "index") else local_rank)
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
    clocks.idx = int(cvd[local_rank]) if len(cvd) > local_rank and cvd[local_rank].strip().isdigit() else local_rank
    clocks.start()
    time.sleep(0.3)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    h0 = time.perf_counter()
    for k in range(warm, warm + args.steps):
        run_step(k, True)
    pipe.join(stream)
    t_end.record(stream)
    host_ms = (time.perf_counter() - h0) * 1e3  # host time to enqueue the K steps (>= device time: host-bound)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end)
    dcnt = (pipe.counters - cnt0)
    if calib:
        # per-kernel times of the timed steps: the same kernels timed eagerly and sequentially with events right
        # after (counters of these steps are excluded from dcnt above)
        pipe.overlap = False  # (the ring and buffers stay as they are; steps run on one stream)
        for k in range(warm + args.steps, warm + args.steps + calib):
            run_step_eager(k)
        torch.cuda.synchronize()
        pipe.overlap = args.overlap
    per = {kname: [a.elapsed_time(b) for a, b in lst] for kname, lst in ev.items()}
    if args.pdl:  # back-to-back overlapping launches: the average launch duration is the timed region / K
        per["score"] = [ms / args.steps] * args.steps
    status = int(pipe.status.item())

    # ---- compact alone on the last step's masks, both frame layouts (context for the layout choice) ---------
    layouts = {}
    k_last = warm + args.steps + calib - 1
    off_l = pipe.ring_slot(k_last)

    def time_compact(fn, reps=10):
        fn()  # warm-up launch (lazy module loading, smem attributes) outside the timed region
        torch.cuda.synchronize()
        c0 = pipe.counters.clone()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        for _ in range(reps):
            fn()
        eb.record(stream)
        torch.cuda.synchronize()
        t_ms = ea.elapsed_time(eb) / reps
        byt = float((pipe.counters - c0)[abi.CNT_BYTES_COMPACT].item()) / reps
        return {"ms": t_ms, "gbs": byt / (t_ms / 1e3) / 1e9}

    if args.frames == "nv12":
        # fused (kept groups only) vs unfused (preprocess every group of every frame into grouped model frames,
        # then compact them) on the last step's frames and masks
        full = torch.full((S, s, abi.grid_words(g)), -1, dtype=torch.int32, device=dev)
        model_frames = torch.empty(S * s, 3 * H * W, dtype=torch.bfloat16, device=dev)
        mf_ptrs = abi.ptr_array([model_frames[i] for i in range(S * s)], dev)
        offs_full = torch.zeros(S * s + 1, dtype=torch.int32, device=dev)
        pos_full = torch.empty(S * s * pipe.np, 3, dtype=torch.int32, device=dev)
        src_full = torch.empty(S * s * pipe.np, dtype=torch.int32, device=dev)

        def fused():
            abi.codecsight_compact_nv12(g, pre, S, s, pipe.mask_ring[:, off_l:], pipe.ring, fidx_dev[k_last],
                                        ptr_s[0], ptr_s[1], pipe.capacity, pipe.packed, pipe.pos_ids,
                                        pipe.src_index, pipe.frame_offsets[:S * s + 1], pipe.counters, pipe.status)

        def unfused():
            abi.codecsight_compact_nv12(g, pre, S, s, full, s, fidx_dev[k_last], ptr_s[0], ptr_s[1],
                                        S * s * pipe.np, model_frames, pos_full, src_full, offs_full, pipe.counters,
                                        pipe.status)
            abi.codecsight_compact(g, S, s, pipe.mask_ring[:, off_l:], pipe.ring, fidx_dev[k_last], mf_ptrs,
                                   pipe.capacity, pipe.packed, pipe.pos_ids, pipe.src_index,
                                   pipe.frame_offsets[:S * s + 1], pipe.counters, pipe.status,
                                   frame_layout=abi.CS_LAYOUT_GROUPED)

        layouts["nv12_fused"] = time_compact(fused)
        layouts["nv12_preprocess_all_then_compact"] = time_compact(unfused)
        del model_frames
    elif tp > 1:
        for lname, lid in (("grouped", abi.CS_LAYOUT_GROUPED), ("planar", abi.CS_LAYOUT_PLANAR)):
            layouts[lname] = time_compact(lambda lid=lid: abi.codecsight_compact_tp(
                g, tp, S, s // tp, pipe.mask_ring[:, off_l:], pipe.ring, fidx_dev[k_last], ptr_s, pipe.capacity,
                pipe.packed, pipe.pos_ids, pipe.src_index, pipe.frame_offsets[:S * s // tp + 1], pipe.counters,
                pipe.status, frame_layout=lid))
    else:
        for lname, lid in (("grouped", abi.CS_LAYOUT_GROUPED), ("planar", abi.CS_LAYOUT_PLANAR)):
            layouts[lname] = time_compact(lambda lid=lid: abi.codecsight_compact(
                g, S, s, pipe.mask_ring[:, off_l:], pipe.ring, fidx_dev[k_last], ptr_s, pipe.capacity, pipe.packed,
                pipe.pos_ids, pipe.src_index, pipe.frame_offsets[:S * s + 1], pipe.counters, pipe.status,
                frame_layout=lid))

    # ---- end-to-end through the public API with host buffers ----------------------------------------------
    # Every step: the step's codec metadata, frame types and frame indices go H2D from pinned host memory (copy
    # stream, double-buffered staging so step k+1's upload overlaps step k's kernels), the three calls run on the
    # compute stream, and the step's results (token counts per stream, kept counts, packed rows) come back D2H;
    # the host waits for step k-1's results while step k runs (a streaming server's pipeline).
    e2e = None
    scene_acc = [0.0] * (2 * len(SCENE_KINDS))
    if not args.no_e2e:
        k0 = warm + args.steps + calib
        nsteps = args.steps
        in_mb, in_ty, in_fi = [], [], []
        for k in range(k0, k0 + nsteps):
            f0, n = step_frames(cfg, k)
            in_mb.append(mb_host[1 + (k - 1) % n_pool])
            in_ty.append(torch.from_numpy(np.stack([synth.frame_types(n, gop, f0)] * S)).pin_memory())
            in_fi.append(torch.from_numpy(np.tile(np.arange(f0 // tp, (f0 + n) // tp, dtype=np.int32),
                                                  S)).pin_memory())
        # the timed loop's staging buffers (same addresses, so graph keys match): slot b = k & 1
        st_mb = [stage[0]["mb"], stage[1]["mb"]]
        st_ty = [stage[0]["ty"], stage[1]["ty"]]
        st_fi = [stage[0]["fi"], stage[1]["fi"]]
        res = [torch.empty(S * 4 + S * s + 1, dtype=torch.int32).pin_memory() for _ in range(2)]
        snap = [torch.zeros(S * 4 + S * s + 1, dtype=torch.int32, device=dev) for _ in range(2)]
        copy_stream = torch.cuda.Stream(dev)
        loaded = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e_a = torch.cuda.Event(enable_timing=True)
        e_b = torch.cuda.Event(enable_timing=True)
        checksum = 0
        kept_acc = np.zeros(S, np.int64)   # per-stream kept patches of the e2e steps (results the host reads)
        t0 = time.perf_counter()
        e_a.record(copy_stream)
        res_stream = torch.cuda.Stream(dev)
        for i in range(nsteps):
            k = k0 + i
            b = k & 1
            _, n = step_frames(cfg, k)
            with torch.cuda.stream(copy_stream):
                if i >= 2:
                    copy_stream.wait_event(consumed[b])
                st_mb[b].copy_(in_mb[i], non_blocking=True)              # H2D: this step's codec metadata
                st_ty[b].copy_(in_ty[i], non_blocking=True)
                st_fi[b].copy_(in_fi[i], non_blocking=True)
                loaded[b].record(copy_stream)
            stream.wait_event(loaded[b])
            if args.overlap:
                # double-buffered outputs (parity b) were last read back by step i-2's results copy
                evs = pipe.step(k, st_mb[b], ptr_s, st_fi[b], st_ty[b], wait_events=[done[b]] if i >= 2 else [])
            else:
                if args.graphs:
                    pipe.graph_step(k, st_mb[b], ptr_s, st_fi[b], st_ty[b])
                else:
                    pipe.step(k, st_mb[b], ptr_s, st_fi[b], st_ty[b])
                # the outputs are single-buffered: snapshot the step's results on the compute stream (device
                # copies, stream-ordered before step i+1 overwrites them) into slot b, free once step i-2's
                # read-back of slot b is done; the D2H then runs off the compute stream's critical path
                if i >= 2:
                    stream.wait_event(done[b])
                if pipe.kv is not None:
                    snap[b][:S * 4].copy_(pipe.n_tokens.view(-1), non_blocking=True)
                snap[b][S * 4:S * 4 + S * n].copy_(pipe.kept_counts(n).reshape(-1), non_blocking=True)
                snap[b][-1:].copy_(pipe.frame_offsets[S * n // tp:S * n // tp + 1], non_blocking=True)
                e_step = torch.cuda.Event()
                e_step.record(stream)
                evs = {"step": (None, e_step)}
            # results stream: waits for the step, reads the results back (D2H), releases the staging slot
            for name in ("score", "compact", "kv", "step"):
                if name in evs:
                    res_stream.wait_event(evs[name][1])
            with torch.cuda.stream(res_stream):
                if args.overlap:
                    if pipe.kv is not None:                                # D2H: the step's results
                        res[b][:S * 4].copy_(pipe.n_tokens.view(-1), non_blocking=True)
                    res[b][S * 4:S * 4 + S * n].copy_(pipe.kept_counts(n).reshape(-1), non_blocking=True)
                    res[b][-1:].copy_(pipe.frame_offsets[S * n // tp:S * n // tp + 1], non_blocking=True)
                else:
                    res[b].copy_(snap[b], non_blocking=True)               # D2H: the step's results
                consumed[b].record(res_stream)
                done[b].record(res_stream)
            if i >= 1:
                done[1 - b].synchronize()                                  # the host consumes step k-1's result
                checksum += int(res[1 - b][-1])
                kept_acc += res[1 - b][S * 4:S * 4 + S * s].numpy().reshape(S, s).sum(axis=1)
        stream.wait_stream(res_stream)
        e_b.record(stream)
        done[(k0 + nsteps - 1) & 1].synchronize()
        checksum += int(res[(k0 + nsteps - 1) & 1][-1])
        kept_acc += res[(k0 + nsteps - 1) & 1][S * 4:S * 4 + S * s].numpy().reshape(S, s).sum(axis=1)
        torch.cuda.synchronize()
        wall_ms = (time.perf_counter() - t0) * 1e3
        e2e_ms = e_a.elapsed_time(e_b)
        h2d = in_mb[0].numel() + in_ty[0].numel() + in_fi[0].numel() * 4
        d2h = (S * 4 + S * s + 1) * 4
        # the link's own rate for this upload: back-to-back pinned copies of one step's metadata buffer, nothing else
        # on the GPU (the e2e rate above is bounded by it whenever a step's upload outlasts its kernels)
        with torch.cuda.stream(copy_stream):
            st_mb[0].copy_(in_mb[0], non_blocking=True)
            c_a, c_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c_a.record(copy_stream)
            for i in range(8):
                st_mb[i & 1].copy_(in_mb[i % len(in_mb)], non_blocking=True)
            c_b.record(copy_stream)
        torch.cuda.synchronize()
        link_gbs = 8 * in_mb[0].numel() / (c_a.elapsed_time(c_b) / 1e3) / 1e9
        e2e = dict(ms=e2e_ms, wall_ms=wall_ms, steps=nsteps, h2d=h2d, d2h=d2h, checksum=checksum, link_gbs=link_gbs)
        # per scene kind: kept patches / patches over the e2e steps (calibration check against P:563)
        for i, gid in enumerate(global_ids):
            j = SCENE_KINDS.index(synth.scene_of(cfg, gid))
            scene_acc[2 * j] += float(kept_acc[i])
            scene_acc[2 * j + 1] += float(nsteps * s * pipe.np)

    # ---- reduce over ranks --------------------------------------------------------------------------------
    scene_tot = shard.reduce_counters(torch.tensor(scene_acc, dtype=torch.float64, device=dev)).cpu().numpy()
    tens = shard.reduce_max(torch.tensor([ms, e2e["ms"] if e2e else 0.0, e2e["wall_ms"] if e2e else 0.0],
                                         dtype=torch.float64, device=dev))
    # per-rank device times and shard sizes (load imbalance across ranks)
    per_rank = shard.gather_per_rank(torch.tensor([ms, float(S), e2e["ms"] if e2e else 0.0], dtype=torch.float64,
                                                  device=dev))
    cnt_all = shard.reduce_counters(dcnt)
    ms_max, e2e_ms_max = float(tens[0]), float(tens[1])
    if e2e:
        e2e["wall_ms"] = float(tens[2])  # the slowest rank's host wall clock (all ranks' frames are counted)
    if rank != 0:
        return
    c = cnt_all.cpu().numpy().astype(np.int64)
    K = args.steps
    frames_total = S_total * s * K
    value = frames_total / (ms_max / 1e3)
    stream_steps = S_total * K / (ms_max / 1e3)
    kv_ms = float(np.mean(per["kv"])) if per["kv"] else 0.0
    kv_bytes_launch = float(dcnt[abi.CNT_BYTES_KV].item()) / K
    peak, peak_kind = measured_peak_hbm()
    achieved = kv_bytes_launch / (kv_ms / 1e3) / 1e9 if kvb else 0.0
    sc_ms = float(np.mean(per["score"]))
    sc_bytes = float(dcnt[abi.CNT_BYTES_SCORE].item()) / K
    cmp_bytes = float(dcnt[abi.CNT_BYTES_COMPACT].item()) / K
    # ncu_summary.json keys of this run's kernels (traffic of a variant is only reported when it was captured)
    kv_key = ("kv_refresh_paged" if args.kv_mode == "paged" else "kv_refresh_copy") + \
        ("+mrope" if args.rope == "mrope" else "") + ("+tp2" if tp == 2 else "")
    cmp_key = ("compact_nv12" if args.frames == "nv12" else "compact_tp" if tp == 2 else
               "score_compact" if args.fused else "compact_gather") + ("+planar" if args.frame_layout == "planar" else "")
    if args.fused:   # one launch does both: its time and the bytes of both calls
        cmp_ms = sc_ms
        cmp_bytes += sc_bytes
    else:
        cmp_ms = float(np.mean(per["compact"]))
    cmp_gbs = cmp_bytes / (cmp_ms / 1e3) / 1e9
    step_bytes = float(dcnt[abi.CNT_BYTES_SCORE].item() + dcnt[abi.CNT_BYTES_COMPACT].item() +
                       dcnt[abi.CNT_BYTES_KV].item()) / K
    kept_frac = float(dcnt[abi.CNT_KEPT].item()) / max(1.0, float(dcnt[abi.CNT_PATCHES].item()))
    out = {
        "metric": "codec-pruned frames/sec (whole hot path: score+compact+kv_refresh), all GPUs",
        "value": value, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": warm,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": {"workload": cfg["name"], "streams_per_gpu": S if scaling == "weak" else
                   [int(r[1]) for r in per_rank], "streams_total": S_total, "src": list(cfg["src"]),
                   "model_input": [448, 448], "window": w, "stride": s, "gop": gop, "tau": cfg["tau"], "alpha": cfg["alpha"], "group": cfg["group"],
                   "kv": "Qwen2-VL-7B 28x4x128 bf16" if kvb else None, "n_prompt": cfg["n_prompt"],
                   "frame_layout": args.frame_layout, "kv_mode": args.kv_mode, "rope": args.rope,
                   "frames": args.frames, "overlap": args.overlap, "temporal_patch": tp, "fused": args.fused,
                   "pdl": args.pdl, "chain_depth": args.chain_depth if args.pdl else None,
                   "graphs": args.graphs,
                   "parallelism": f"stream-shard x{world}",
                   "l2": "inputs larger than L2 (KV caches, frames and metadata of one step exceed the 126 MB L2; "
                         "see per-step bytes)"},
        "streams_per_sec": stream_steps,
        "per_gpu": {"frames_per_sec": value / world, "streams_per_sec": stream_steps / world},
        "per_rank": [{"rank": i, "streams": int(r[1]), "ms_per_step": r[0] / K,
                      "frames_per_sec": r[1] * s * K / (r[0] / 1e3), "e2e_ms_per_step": r[2] / K if e2e else None}
                     for i, r in enumerate(per_rank)],
        "host_cpu": host_cpu_model(),
        "host_enqueue_ms_per_step": host_ms / K,
        "kv_refresh_gbs": achieved,
        "per_kernel_ms": ({"score_compact": sc_ms, "kv_refresh": kv_ms} if args.fused else
                          {"score_patches": sc_ms, "compact": cmp_ms, "kv_refresh": kv_ms}),
        "per_kernel_gbs": {"score_patches" if not args.fused else "score_compact":
                           (sc_bytes if not args.fused else cmp_bytes) / (sc_ms / 1e3) / 1e9, "compact": cmp_gbs,
                           "kv_refresh": achieved},
        "frame_layout": args.frame_layout,
        "compact_by_layout": layouts,
        "kept_fraction": kept_frac,
        # per scene kind over the e2e steps; calibration targets kept 0.50 / 0.73 / 0.87 for low / medium / high
        # motion (50 / 27 / 13 % of visual tokens pruned), traffic "medium-high" ~0.80, static = I-frames only
        "kept_fraction_by_scene": {kind: scene_tot[2 * j] / scene_tot[2 * j + 1]
                                   for j, kind in enumerate(SCENE_KINDS) if scene_tot[2 * j + 1] > 0},
        "tokens_per_step": {"reuse": int(c[abi.CNT_TOK_REUSE]) // K, "anchor": int(c[abi.CNT_TOK_ANCHOR]) // K,
                            "new": int(c[abi.CNT_TOK_NEW]) // K},
        "near_tau_patches": int(c[abi.CNT_NEAR_TAU]),
        "status": status,
        "kv_mode": args.kv_mode,
        "roofline": ({"bound": "hbm", "kernel": ("codecsight_kv_refresh_paged (kv_plan_paged + kv_prefix + "
                                                 "kv_gather_tma)") if args.kv_mode == "paged" else
                      "codecsight_kv_refresh (kv_plan + kv_prefix + kv_gather_tma)",
                      "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                      "frac": achieved / peak,
                      "traffic": ncu_traffic(kv_key, cfg["name"]),
                      "algorithmic_bytes_per_launch": kv_bytes_launch} if kvb else
                     {"bound": "hbm", "kernel": ("codecsight_score_compact (score_kernel<fused>)" if args.fused else
                                                 "codecsight_compact (compact_scan + compact_gather)"),
                      "achieved": cmp_gbs, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                      "frac": cmp_gbs / peak,
                      "traffic": ncu_traffic(cmp_key, cfg["name"]),
                      "algorithmic_bytes_per_launch": cmp_bytes}),
        "secondary_roofline": {"kernel": {"compact_nv12": "codecsight_compact_nv12", "compact_tp": "codecsight_compact_tp",
                                          "score_compact": "codecsight_score_compact"}.get(cmp_key.split("+")[0],
                                                                                            "codecsight_compact"),
                               "achieved": cmp_gbs, "peak": peak,
                               "frac": cmp_gbs / peak, "unit": "GB/s", "algorithmic_bytes_per_launch": cmp_bytes,
                               "traffic": ncu_traffic(cmp_key, cfg["name"])},
        # the whole step against the same roofline: every call's algorithmic bytes per step / the step's time
        "step_roofline": {"bytes_per_step": step_bytes, "achieved": step_bytes / (ms_max / K / 1e3) / 1e9,
                          "peak": peak, "unit": "GB/s", "frac": step_bytes / (ms_max / K / 1e3) / 1e9 / peak},
        "gpu_launches": K * pipe.kernel_launches_per_step(1),
        # the paper's own numbers for this path (context, not the target): per-request overheads of its Python
        # implementation on vLLM/LMCache, InternVL3 on 2 x A100 40GB SXM4; a request there is
        # one window of one stream, i.e. one stream-step here
        "paper_context": {"hardware": "NVIDIA A100 40GB SXM4 (InternVL3-14B, TP=2)",
                          "token_pruning_ms_per_request": 48.9, "kvc_refresh_ms_per_request": 0.6, "cite": "P:714",
                          "ours_ms_per_stream_step": ms_max / K / S},
        "clocks": clk,
    }
    if args.frames == "nv12":
        # the fused NV12 preprocessing is bound by its exact fp32 arithmetic, not by bytes: its FP32-pipe
        # roofline from the guide's unit counts -- 148 SMs x 128 FP32 lanes x the max SM clock -- and the kernel's
        # static count of 91 packed FP32 instructions (FMUL2 / FFMA2 / FADD2, 2 lane-ops each) per item (a pair of
        # output rows of a kept group: 14 per group) over the warp's 32 lanes
        groups = float(dcnt[abi.CNT_PACKED_ROWS].item()) / K / 4.0
        lane_ops = groups * 14 * 32 * 91 * 2
        sm_mhz = (json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0)
                  if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1965.0)
        fp32_peak = torch.cuda.get_device_properties(dev).multi_processor_count * 128 * sm_mhz * 1e6
        nv_ms = cmp_ms  # the codecsight_compact_nv12 call in the step (count + scan included), as the secondary roofline
        out["compute_roofline"] = {"bound": "fp32_pipe", "kernel": "codecsight_compact_nv12 (compact_nv12_staged)",
                                   "achieved": lane_ops / (nv_ms / 1e3) / 1e12, "peak": fp32_peak / 1e12,
                                   "unit": "T fp32 lane-ops/s", "frac": lane_ops / (nv_ms / 1e3) / fp32_peak,
                                   "lane_ops_per_launch": lane_ops, "peak_kind": "guide unit counts x sm_max_mhz"}
    if e2e:
        out["e2e"] = {"value": frames_total / (e2e_ms_max / 1e3), "unit": "frames/s",
                      "h2d_bytes_per_step": e2e["h2d"] * S_total // S, "d2h_bytes_per_step": e2e["d2h"] * S_total // S,
                      "wall_clock_value": frames_total / (e2e["wall_ms"] / 1e3),
                      "pipelining": "H2D of step k+1 on a copy stream overlaps step k; host reads step k-1's result",
                      # upload rate the e2e steps achieved vs the pinned H2D rate of the same buffer measured alone
                      "h2d_gbs": e2e["h2d"] * e2e["steps"] / (e2e["ms"] / 1e3) / 1e9,
                      "h2d_link_gbs": e2e["link_gbs"]}
    if not args.no_cpu_baseline and world == 1:  # the oracle baseline is timed at N = 1 only
        log("[rank 0] timing the CPU oracle on a bounded sample ...")
        r = oracle_sample(cfg, args.cpu_seconds, kv_mode=args.kv_mode, tp=tp)
        out["cpu_baseline"] = {"value": r["frames"] / r["seconds"], "unit": "frames/s", "cores": 1, "kind": "oracle",
                               "cpu_model": host_cpu_model(),
                               "sample": f"{r['stream_steps']} whole stream-steps (window k=4: {s} new frames + "
                                         f"KV refresh) of streams {r['scenes'][:4]}..., single-threaded C oracle, "
                                         f"{r['seconds']:.1f} s"}
        if args.cpu_all_cores:
            log("[rank 0] timing the CPU oracle on all host cores ...")
            ra = oracle_all_cores(cfg, args.cpu_seconds, args.kv_mode, tp)
            if ra is not None:
                out["cpu_baseline_all_cores"] = {
                    "value": ra["value"], "unit": "frames/s", "cores": ra["processes"], "kind": "oracle",
                    "host_cpus": ra["host_cpus"], "cpu_model": host_cpu_model(),
                    "sample": f"{ra['processes']} concurrent single-threaded oracle processes (one per core, capped "
                              f"by host memory and 32), {ra['stream_steps']} whole stream-steps (k=4) of disjoint "
                              f"streams, ~{ra['seconds']:.1f} s each"}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: CS_BENCH_SHARED_GPU=1 runs every rank on GPU 0 with the gloo backend (exercises the multi-rank
    # sharding / barrier / max-over-ranks / counter all-reduce path on a one-GPU box; never used for numbers)
    shared = os.environ.get("CS_BENCH_SHARED_GPU") == "1"
    if shared:
        local_rank = 0
    cfg = workload(args.workload, args.streams, args.kv_mode, args)
    # the fused score+compact kernel takes model frames, one frame per token
    args.fused = bool(args.fused and args.frames == "model" and args.temporal_patch == 1)
    if cfg["name"].startswith("NEXT4"):
        import bench_cdf
        if args.impl == "reference":
            bench_cdf.run_reference(args, cfg, rank, world)
            return
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo" if shared else "nccl")
        bench_cdf.run_ours(args, cfg, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("gloo" if shared else "nccl")
    run_ours(args, cfg, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
