"""Multi-stream state of the hot path on one GPU (plumbing only: device buffers + the three ABI calls).

One ``Pipeline`` owns, for its shard of camera streams, everything the path keeps between sliding-window steps
(SURVEY §5 "per-stream state = gop_state + mask/type ring + KV buffers"):

  gop_state   [S][grid_words + 1]      GOP accumulation state
  mask_ring   [S][ring][grid_words]    keep masks of the last ring = w + s frames (decode-once)
  type_ring   [S][ring]                I/P frame types
  caches      kv_mode "copy":  2 x S buffers [L][2][capacity][H][D] (window k-1 / window k, swapped every step)
              kv_mode "paged": S row pools [L][2][capacity][H][D] updated in place + 2 x [S][capacity] slot maps
  refreshed   S buffers [L][2][refresh_capacity][H][D] (rows the prefill recomputes: anchors, new, prompt)

``step(k, ...)`` enqueues, on the current CUDA stream and without any host synchronisation:
  codecsight_score_patches -> codecsight_compact -> codecsight_kv_refresh.
Window k consumes frames [k s, k s + w); the new frames of step k are [(k-1)s + w, k s + w) (all w at k = 0).
"""
from __future__ import annotations

import math

import torch

from . import _abi as abi


class Pipeline:
    def __init__(self, grid: dict, n_streams: int, window: int, stride: int, gop: int, kv: dict | None,
                 n_prompt: int = 0, device=None, want_score: bool = False, packed_capacity: int | None = None,
                 with_refreshed: bool = True, frame_layout: int = abi.CS_LAYOUT_PLANAR, kv_mode: str = "copy",
                 compact_chunk: int | None = None, preprocess: dict | None = None, overlap: bool = False,
                 temporal_patch: int = 1, fused: bool = False, pdl: bool = False, chain_depth: int = 4):
        self.g = dict(grid)
        # Ring slots: frame f lives in slot f % ring and a step's n new frames are handed to the kernels as ONE
        # contiguous run of slots [off, off + n) (the calls take a pointer and a frame stride, not a modular index).
        # The run of step k >= 1 starts at ((k-1)s + w) % ring; with s dividing w (and hence the ring, w + s or
        # w + 2s) it always ends inside the ring.  Otherwise some step would write past the ring's last slot (into
        # the next stream's ring row), so such windows are rejected here rather than corrupted (SPEC allows any
        # 1 <= s <= w; every BASELINE config has s | w).
        if not (1 <= stride <= window) or window % stride != 0:
            raise ValueError(f"Pipeline needs 1 <= stride <= window and stride | window (got w={window}, s={stride}): "
                             "a step's new frames must be one contiguous run of ring slots")
        # fused: one codecsight_score_compact launch per step (NEXT-2) instead of score_patches + compact
        self.fused = fused
        # pdl: step k's fused launch is chained call k (CS_LAUNCH_PDL, cs_chain): a programmatic dependent of step
        # k-1's that overlaps it (scoring during k-1's compaction, then compaction alongside k-1's tail).  Prune-only
        # pipelines (no KV refresh between the launches); the step's frame types are read straight from the caller's
        # [S][n] tensor (no ring copy between the launches); workspaces and output buffer sets alternate by parity.
        self.pdl = pdl
        if pdl:
            assert fused and kv is None and not overlap, "pdl: fused score+compact, no KV refresh, no overlap mode"
        if fused:
            assert temporal_patch == 1 and preprocess is None, "fused score+compact: model frames, temporal_patch 1"
        # temporal patches (NEXT-3, Qwen2-VL temporal_patch_size): a token unit = tp consecutive frames; scoring stays
        # per frame, compaction emits [3][tp][p][p] rows per unit (codecsight_compact_tp) and writes the unit masks /
        # types into a unit ring, and the KV refresh runs over units (window w/tp, stride s/tp)
        self.tp = tp = temporal_patch
        if tp > 1:
            assert window % tp == 0 and stride % tp == 0, "window and stride must be multiples of temporal_patch"
            assert preprocess is None and not overlap, "temporal patches: planar/grouped frames, no overlap mode"
            assert compact_chunk is None or compact_chunk % tp == 0
        self.frame_layout = frame_layout
        self.kv_mode = kv_mode
        # preprocess set: frames are decoded NV12 (frame_ptrs = (y_ptrs, uv_ptrs)) and compaction runs the fused
        # NV12 -> RGB -> resize -> normalise kernel (codecsight_compact_nv12, NEXT-2)
        self.preprocess = preprocess
        # frames per compaction call (the first window's w frames are compacted s at a time when set)
        self.compact_chunk = compact_chunk
        self.S, self.w, self.s, self.gop = n_streams, window, stride, gop
        # overlap: compact and kv_refresh of step k run on their own streams concurrently with the scoring of step
        # k+1 (fused: kv_refresh of step k concurrently with the score+compact of step k+1); the ring then holds w + 2s frames so that step k+1's new masks never land on slots kv_refresh(k)
        # still reads (frames [(k-1)s, ks+w) and the next s frames are w + 2s distinct slots)
        self.overlap = overlap
        self.ring = window + (2 * stride if overlap else stride)
        self.dev = torch.device(device if device is not None else "cuda")
        self.nw = abi.grid_words(grid)
        self.np = grid["grid_w"] * grid["grid_h"]
        self.groups = (grid["grid_w"] // grid["group"]) * (grid["grid_h"] // grid["group"])
        d = self.dev
        S, ring, nw = n_streams, self.ring, self.nw
        self.gop_state = torch.zeros(S, nw + 1, dtype=torch.int32, device=d)
        self.mask_ring = torch.zeros(S, ring, nw, dtype=torch.int32, device=d)
        self.type_ring = torch.zeros(S, ring, dtype=torch.uint8, device=d)
        # per-step outputs alternate between nb buffer sets (step parity; chained PDL calls: step mod chain depth)
        self.chain_depth = chain_depth
        nb = self.chain_depth if pdl else (2 if overlap else 1)
        self._kept_count = [torch.zeros(S, window, dtype=torch.int32, device=d) for _ in range(nb)]
        self.kept_count = self._kept_count[0]
        self.score = torch.zeros(S, window, self.np, dtype=torch.float32, device=d) if want_score else None
        self.counters = torch.zeros(abi.NCOUNTERS, dtype=torch.int64, device=d)
        self.status = torch.zeros(1, dtype=torch.int32, device=d)
        # packed ViT input: enough rows for the first window (every patch kept)
        p = grid["patch"]
        chunk = compact_chunk if (compact_chunk is not None and not fused) else window
        self.capacity = packed_capacity if packed_capacity is not None else S * (chunk // tp) * self.np
        self._packed = [torch.empty(self.capacity, 3 * tp * p * p, dtype=torch.bfloat16, device=d)
                        for _ in range(nb)]
        self._pos_ids = [torch.empty(self.capacity, 3, dtype=torch.int32, device=d) for _ in range(nb)]
        self._src_index = [torch.empty(self.capacity, dtype=torch.int32, device=d) for _ in range(nb)]
        self._frame_offsets = [torch.zeros(S * (window // tp) + 1, dtype=torch.int32, device=d) for _ in range(nb)]
        self.packed, self.pos_ids = self._packed[0], self._pos_ids[0]
        self.src_index, self.frame_offsets = self._src_index[0], self._frame_offsets[0]
        self.frame_index = torch.zeros(S * window, dtype=torch.int32, device=d)
        # KV token units: frames (tp = 1) or frame tuples with their own mask / type ring
        self.wu, self.su, self.uring = window // tp, stride // tp, ring // tp
        if tp > 1:
            self.unit_ring = torch.zeros(S, self.uring, nw, dtype=torch.int32, device=d)
            self.unit_type_ring = torch.zeros(S, self.uring, dtype=torch.uint8, device=d)
        else:
            self.unit_ring, self.unit_type_ring = self.mask_ring, self.type_ring
        self.kv = None
        if kv is not None:
            self.n_prompt = n_prompt
            wu, su = self.wu, self.su
            cap = wu * self.groups + n_prompt
            anchors = 1 + math.ceil(max(0, wu - su) / max(1, gop // tp))
            rcap = (su + anchors) * self.groups + n_prompt
            self.kv = dict(kv, capacity=cap, refresh_capacity=rcap, n_prompt=n_prompt)
            dt = torch.bfloat16 if kv["dtype"] == abi.CS_BF16 else torch.float32
            shape = (kv["layers"], 2, cap, kv["kv_heads"], kv["head_dim"])
            n_sets = 1 if kv_mode == "paged" else 2
            self.caches = [[torch.empty(shape, dtype=dt, device=d) for _ in range(S)] for _ in range(n_sets)]
            self.cache_ptrs = [abi.ptr_array(c, d) for c in self.caches]
            if kv_mode == "paged":
                self.slots = [torch.full((S, cap), -1, dtype=torch.int32, device=d) for _ in range(2)]
            rshape = (kv["layers"], 2, rcap, kv["kv_heads"], kv["head_dim"])
            self.refreshed = [torch.empty(rshape, dtype=dt, device=d) for _ in range(S)] if with_refreshed else None
            self.refreshed_ptrs = abi.ptr_array(self.refreshed, d) if with_refreshed else None
            self.token_cap = cap
            self._disposition = [torch.zeros(S, cap, dtype=torch.uint8, device=d) for _ in range(nb)]
            self._p_old = [torch.zeros(S, cap, dtype=torch.int32, device=d) for _ in range(nb)]
            self._n_tokens = [torch.zeros(S, 4, dtype=torch.int32, device=d) for _ in range(nb)]
            self.disposition, self.p_old, self.n_tokens = self._disposition[0], self._p_old[0], self._n_tokens[0]
            win1 = dict(window=self.wu, stride=self.su, step=1, ring_frames=self.uring)
            nbytes = (abi.kv_paged_workspace_size(grid, self.kv, win1, S) if kv_mode == "paged"
                      else abi.kv_workspace_size(self.kv, win1, S))
            self.workspace = torch.empty((nbytes + 15) // 16 * 16, dtype=torch.uint8, device=d)
        self.cur = 0  # which cache set holds window k-1
        if fused:
            self.sc_workspace = torch.zeros(abi.score_compact_workspace_size(S), dtype=torch.uint8, device=d)
            # chained calls rotate three workspaces (a call takes its stream tickets while the two before it may
            # still run); chain state: per-stream GOP-state generations + per-parity completed-call generations
            nws = self.chain_depth + 1 if pdl else 1
            self._sc_ws = [self.sc_workspace] + [torch.zeros_like(self.sc_workspace) for _ in range(nws - 1)]
            if pdl:
                self._chain = (torch.zeros(S, dtype=torch.int32, device=d),
                               torch.zeros(self.chain_depth, dtype=torch.int32, device=d))
        self._side_done = {}  # step -> events closing its compact / kv_refresh work (overlap mode)
        self._graphs = {}     # graph_step: key -> captured torch.cuda.CUDAGraph
        self._bound = {}      # (ring slot, frames, buffer parity) -> abi.BoundScoreCompact
        self._type_views = {}
        if overlap:
            self.stream_compact = torch.cuda.Stream(d)
            self.stream_kv = torch.cuda.Stream(d)

    # ------------------------------------------------------------------------------------------------------
    def new_frames(self, k: int) -> tuple[int, int]:
        """(first new frame index, number of new frames) of step k."""
        if k == 0:
            return 0, self.w
        return (k - 1) * self.s + self.w, self.s

    def ring_slot(self, k: int) -> int:
        f0, _ = self.new_frames(k)
        return f0 % self.ring

    def init_cache_fill(self, gen: torch.Generator | None = None):
        """Random K/V content (the prefill's output is out of scope; bits only need to be non-degenerate)."""
        if self.kv is None:
            return
        for lst in self.caches + ([self.refreshed] if self.refreshed is not None else []):
            for t in lst:
                t.normal_(generator=gen)

    def kept_counts(self, n: int) -> torch.Tensor:
        """[S][n] kept-patch counts of a step's n new frames: the calls write a contiguous [n_streams][n_frames]
        array, i.e. the first S*n elements of the buffer (not the strided [:, :n] slice of its [S][window] shape)."""
        return self.kept_count.view(-1)[: self.S * n].view(self.S, n)

    def scores(self, n: int):
        """[S][n][patches] scores of a step's n new frames (contiguous prefix of the buffer), or None."""
        return None if self.score is None else self.score.view(-1)[: self.S * n * self.np].view(self.S, n, self.np)

    def step(self, k: int, mb: torch.Tensor, frame_ptrs: torch.Tensor, frame_index: torch.Tensor | None = None,
             types: torch.Tensor | None = None, use_refreshed: bool | None = None, do_kv: bool = True,
             stream=None, timing: bool = False, wait_events=()):
        """Enqueue one sliding-window step.  ``mb``: [S][n_new][mb_rows][mb_cols] cs_mb records (uint8 view or any
        dtype, contiguous, device); ``types``: [S][n_new] uint8 written into the ring (None = already there);
        ``frame_ptrs``: device int64 [S*n_new] pointers to [3][H][W] bf16 frames (a (Y, UV) pair with NV12).
        Returns {"score"|"compact"|"kv": (start_event, end_event)} (timing events when ``timing``)."""
        g = self.g
        f0, n = self.new_frames(k)
        off = f0 % self.ring
        main = torch.cuda.current_stream(self.dev) if stream is None else stream

        def ev(st):
            e = torch.cuda.Event(enable_timing=timing)
            e.record(st)
            return e

        out = {}
        if self.overlap:
            # this step's output buffers (parity k & 1) and ring slots were last used by step k-2: wait for its
            # side-stream work (and any consumer events the caller passes) before writing them again
            b = k & 1
            self.kept_count, self.packed, self.pos_ids = self._kept_count[b], self._packed[b], self._pos_ids[b]
            self.src_index, self.frame_offsets = self._src_index[b], self._frame_offsets[b]
            if self.kv is not None:
                self.disposition, self.p_old, self.n_tokens = self._disposition[b], self._p_old[b], self._n_tokens[b]
            for e in self._side_done.pop(k - 2, []) + list(wait_events):
                main.wait_event(e)
        if self.pdl:
            # no stream operation between two fused launches (an event or a copy would cancel the overlap)
            assert types is not None, "pdl: pass the step's frame types"
            b, nws = k % self.chain_depth, len(self._sc_ws)
            self.kept_count, self.packed, self.pos_ids = self._kept_count[b], self._packed[b], self._pos_ids[b]
            self.src_index, self.frame_offsets = self._src_index[b], self._frame_offsets[b]
            key = (off, n, b, k % nws)
            call = self._bound.get(key)
            if call is None:
                call = abi.BoundScoreCompact(
                    g, self.S, n, None, self.mask_ring[:, off:], self.ring, self.gop_state, None,
                    self.kept_counts(n), self.capacity, self.packed, self.pos_ids, self.src_index,
                    self.frame_offsets[: self.S * n + 1], self._sc_ws[k % nws], self.counters, self.status,
                    frame_layout=self.frame_layout, flags=abi.CS_LAUNCH_PDL, type_stride=n, chain=self._chain)
                self._bound[key] = call
            fi = self.frame_index[: self.S * n] if frame_index is None else frame_index
            if timing:
                s0 = ev(main)
            call(mb, fi, frame_ptrs, main.cuda_stream, frame_type=types, generation=k)
            return {"score": (s0, ev(main))} if timing else {}
        with torch.cuda.stream(main):
            if types is not None:
                tv = self._type_views.get((off, n))
                if tv is None:
                    tv = self._type_views[(off, n)] = self.type_ring[:, off:off + n]
                tv.copy_(types, non_blocking=True)
            s0 = ev(main)
            if self.fused:
                fi = self.frame_index[: self.S * n] if frame_index is None else frame_index
                key = (off, n, k & 1 if self.overlap else 0)
                call = self._bound.get(key)
                if call is None:  # arguments of this ring slot (and output buffer set) marshalled once
                    call = abi.BoundScoreCompact(
                        g, self.S, n, self.type_ring[:, off:], self.mask_ring[:, off:], self.ring, self.gop_state,
                        self.scores(n), self.kept_counts(n), self.capacity, self.packed, self.pos_ids,
                        self.src_index, self.frame_offsets[: self.S * n + 1], self.sc_workspace, self.counters,
                        self.status, frame_layout=self.frame_layout)
                    self._bound[key] = call
                call(mb, fi, frame_ptrs, main.cuda_stream)
            else:
                abi.codecsight_score_patches(g, self.S, n, mb, self.type_ring[:, off:], self.mask_ring[:, off:],
                                             self.ring, self.gop_state,
                                             self.scores(n),
                                             self.kept_counts(n), self.counters, self.status, main)
            out["score"] = (s0, ev(main))
        cs_stream = self.stream_compact if self.overlap else main
        kv_stream = self.stream_kv if self.overlap else main
        if self.overlap:
            cs_stream.wait_event(out["score"][1])
        if not self.fused:
            with torch.cuda.stream(cs_stream):
                c0 = ev(cs_stream)
                self.compact(k, n, off, frame_ptrs, frame_index, cs_stream)
                out["compact"] = (c0, ev(cs_stream))
        if self.kv is not None and do_kv:
            if self.overlap:
                kv_stream.wait_event(out["score"][1])
            with torch.cuda.stream(kv_stream):
                k0 = ev(kv_stream)
                self.kv_refresh(k, use_refreshed, kv_stream)
                out["kv"] = (k0, ev(kv_stream))
        if self.overlap:
            self._side_done[k] = [out[x][1] for x in ("compact", "kv") if x in out]
        return out

    def join(self, stream=None):
        """Make `stream` (default: current) wait for everything enqueued on the side streams."""
        if not self.overlap:
            return
        main = torch.cuda.current_stream(self.dev) if stream is None else stream
        main.wait_stream(self.stream_compact)
        main.wait_stream(self.stream_kv)

    def compact(self, k, n, off, frame_ptrs, frame_index=None, stream=None):
        """codecsight_compact of the step's n new frames, in chunks of compact_chunk frames when set (the packed
        buffer then holds one chunk at a time, as a streaming ViT would consume it)."""
        g = self.g
        # frame_index: [S * n] stream-local frame indices, or [S * n / tp] unit indices with temporal patches
        fi = self.frame_index[: self.S * n // self.tp] if frame_index is None else frame_index
        c = n if self.compact_chunk is None else min(n, self.compact_chunk)
        for j0 in range(0, n, c):
            nj = min(c, n - j0)
            ptrs = frame_ptrs if isinstance(frame_ptrs, (tuple, list)) else (frame_ptrs,)
            if nj == n:
                fptrs, fidx = ptrs, fi
            else:  # frames / indices of the chunk: per stream the slots j0..j0+nj-1 of [S][n]
                fptrs = tuple(p.view(self.S, n)[:, j0:j0 + nj].contiguous().view(-1) for p in ptrs)
                tp = self.tp
                fidx = fi.view(self.S, n // tp)[:, j0 // tp:(j0 + nj) // tp].contiguous().view(-1)
            if self.tp > 1:
                tp, uoff = self.tp, (off + j0) // self.tp
                abi.codecsight_compact_tp(g, tp, self.S, nj // tp, self.mask_ring[:, off + j0:], self.ring, fidx,
                                          fptrs[0], self.capacity, self.packed, self.pos_ids, self.src_index,
                                          self.frame_offsets[: self.S * (nj // tp) + 1], self.counters, self.status,
                                          frame_layout=self.frame_layout, unit_mask=self.unit_ring[:, uoff:],
                                          unit_mask_stride=self.uring, frame_type=self.type_ring[:, off + j0:],
                                          unit_type=self.unit_type_ring[:, uoff:], stream=stream)
            elif self.preprocess is not None:
                abi.codecsight_compact_nv12(g, self.preprocess, self.S, nj, self.mask_ring[:, off + j0:], self.ring,
                                            fidx, fptrs[0], fptrs[1], self.capacity, self.packed, self.pos_ids,
                                            self.src_index, self.frame_offsets[: self.S * nj + 1], self.counters,
                                            self.status, stream)
            else:
                abi.codecsight_compact(g, self.S, nj, self.mask_ring[:, off + j0:], self.ring, fidx, fptrs[0],
                                       self.capacity, self.packed, self.pos_ids, self.src_index,
                                       self.frame_offsets[: self.S * nj + 1], self.counters, self.status, stream,
                                       frame_layout=self.frame_layout)

    def kv_step(self, k: int) -> int:
        """Window index handed to kv_refresh.  A plan depends on k only through k == 0 and the ring phase -- every
        frame index it uses is relative to ks and read through slot f % ring -- so k >= 1 is folded into
        [1, period] with period = ring / gcd(ring, s) (in token units).  Equivalent by construction (every parity
        test runs through it); it is what lets one captured CUDA graph serve all steps of a phase."""
        if k == 0:
            return 0
        period = self.uring // math.gcd(self.uring, self.su)
        return (k - 1) % period + 1

    def graph_key(self, k: int):
        """Steps with equal keys run identical kernel sequences with identical arguments (given fixed inputs)."""
        return (self.kv_step(k), self.ring_slot(k), self.cur)

    def graph_step(self, k: int, mb, frame_ptrs, frame_index, types, use_refreshed=None):
        """Step k >= 1 as one CUDA graph replay (captured on first use of its key).  The inputs must be the same
        tensors (addresses) for every step that shares a key -- callers stage per-step data into fixed buffers."""
        assert k >= 1 and not self.overlap and self.preprocess is None
        use_r = (k >= 1) if use_refreshed is None else use_refreshed
        key = self.graph_key(k) + (mb.data_ptr(), frame_index.data_ptr(), types.data_ptr(),
                                   frame_ptrs.data_ptr(), use_r)
        gr = self._graphs.get(key)
        if gr is None:
            cur0 = self.cur
            gr = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(self.dev)
            side.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.graph(gr, stream=side):
                self.step(k, mb, frame_ptrs, frame_index, types, use_refreshed)
            torch.cuda.current_stream(self.dev).wait_stream(side)
            self.cur = cur0  # capture recorded the step without running it; the replay below runs it
            self._graphs[key] = gr
        gr.replay()
        if self.kv is not None:
            self.cur = 1 - self.cur

    def kv_refresh(self, k, use_refreshed=None, stream=None):
        g = self.g
        win = dict(window=self.wu, stride=self.su, step=self.kv_step(k), ring_frames=self.uring)
        use_r = (k >= 1) if use_refreshed is None else use_refreshed
        ref = self.refreshed_ptrs if use_r else None
        if self.kv_mode == "paged":
            so, sn = self.slots[self.cur], self.slots[1 - self.cur]
            abi.codecsight_kv_refresh_paged(g, self.kv, win, self.S, self.unit_ring, self.unit_type_ring,
                                            self.cache_ptrs[0], so if k >= 1 else None, sn, self.token_cap, ref,
                                            self.token_cap, self.disposition, self.p_old, self.n_tokens,
                                            self.workspace, self.counters, self.status, stream)
        else:
            old, new = self.cache_ptrs[self.cur], self.cache_ptrs[1 - self.cur]
            abi.codecsight_kv_refresh(g, self.kv, win, self.S, self.unit_ring, self.unit_type_ring, old, new, ref,
                                      self.token_cap, self.disposition, self.p_old, self.n_tokens, self.workspace,
                                      self.counters, self.status, stream)
        self.cur = 1 - self.cur

    def kernel_launches_per_step(self, k: int) -> int:
        """Kernels of this library launched by one step (score 1 or fused score+compact 1, compact 3 per chunk:
        count + scan + gather, kv_refresh 3: plan + prefix + gather)."""
        _, nf = self.new_frames(k)
        c = nf if self.compact_chunk is None else min(nf, self.compact_chunk)
        n = 1 if self.fused else 1 + 3 * ((nf + c - 1) // c)
        if self.kv is not None:
            n += 3
        return n
