// group_ring.cuh — one warp's TMA bulk ring over a range of kept 2x2 groups of a compaction batch (internal).
//
// Shared by codecsight_compact (compact_gather_tma) and the fused score+compact kernel's grid-balanced compaction:
// 2x2 groups of 14-px patches on a 32 x 32 patch grid, grouped frames (a kept group is one contiguous 4,704-B
// block of its frame and of the packed output, reading Q14).  The batch's kept groups are numbered in packed order
// (slot, group row-major); frame_offsets[slot] (rows, = 4 x groups) is the exclusive prefix.  Lane 0 walks the
// range [q, q1): cp.async.bulk global -> smem completes on the stage's mbarrier, cp.async.bulk smem -> global
// (bulk_group) writes the packed rows, and a stage is refilled once wait_group.read says its store has read it;
// every lane writes position ids / source indices.  Groups that cannot take the bulk path (capacity-truncated,
// misaligned frame) are copied by the warp.  Mask and offset reads are plain (coherent) loads: in the fused kernel
// they were written by the same grid.
#pragma once

#include "cs_internal.cuh"

namespace cs {

constexpr unsigned kRingGroupBytes = 4704u;  // 4 patches x 3 x 14 x 14 bf16
constexpr unsigned kRingStageAlloc = 4736u;  // rounded up to 128 B

struct RingGroup {
  long long n0;     // first packed row
  int slot;         // frame slot
  int gi;           // group index gr * 16 + gc
  int t_index;      // pos id t
  int kind;         // 0 bulk, 1 direct (warp copy), 2 beyond the capacity, -1 end of work
  const uint16_t* src;
};

struct RingBatch {
  const int32_t* frame_offsets;  // [n_slots + 1]
  int n_slots, n_frames;         // slot = stream * n_frames + frame
  const uint32_t* keep_mask;     // frame f of stream s at keep_mask + (s * mask_frame_stride + f) * 32
  long long mask_frame_stride;
  const void* const* frames;     // [n_slots] grouped bf16 frames
  const int32_t* frame_index;    // [n_slots] pos id t
  long long capacity;
  uint16_t* packed;
  int32_t* pos_ids;
  int32_t* src_index;
};

// Returns the packed rows this warp wrote (lane 0's count; capacity-clamped).
// smask: a 16-B aligned per-warp shared buffer of 32 words (the current slot's keep mask, copied once per slot so
// that walking its group rows costs no global-memory latency on the ring's critical path).
CS_DEV long long group_ring(const RingBatch& B, long long q, long long q1, unsigned char* stages, int nst,
                            uint64_t* full, RingGroup* desc, uint32_t* smask, int lane) {
  if (q >= q1) return 0;
  constexpr int kNgr = 16;
  const long long row_el = 3ll * 14 * 14;
  const long long q_first = q;
  int slot = 0, gr = 0, t_index = 0;
  uint32_t ybits = 0u;
  const uint16_t* frame = nullptr;
  bool aligned = false;
  auto mask_of = [&](int sl) {
    const int s = sl / B.n_frames, f = sl - s * B.n_frames;
    return B.keep_mask + ((long long)s * B.mask_frame_stride + f) * 32;
  };
  auto load_row = [&]() {
    const uint32_t x = smask[2 * gr] | smask[2 * gr + 1];
    ybits = (x | (x >> 1)) & 0x55555555u;  // bit 2*gc set iff group (gr, gc) is kept
  };
  auto load_slot = [&]() {
    frame = static_cast<const uint16_t*>(B.frames[slot]);
    t_index = B.frame_index[slot];
    aligned = (reinterpret_cast<uintptr_t>(frame) & 15u) == 0;
    const uint32_t* m = mask_of(slot);
    if ((reinterpret_cast<uintptr_t>(m) & 15u) == 0) {
      uint4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = reinterpret_cast<const uint4*>(m)[i];
#pragma unroll
      for (int i = 0; i < 8; ++i) reinterpret_cast<uint4*>(smask)[i] = v[i];
    } else {
      for (int i = 0; i < 32; ++i) smask[i] = m[i];
    }
  };
  bool more = true;
  if (lane == 0) {
    int lo = 0, hi = B.n_slots;  // largest slot with frame_offsets[slot] <= q * 4
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (static_cast<long long>(B.frame_offsets[mid]) <= q * 4) lo = mid; else hi = mid;
    }
    slot = lo;
    long long skip = q - B.frame_offsets[slot] / 4;
    load_slot();
    load_row();
    while (skip >= __popc(ybits)) {
      skip -= __popc(ybits);
      ++gr;  // stays inside the slot: the slot holds more than `skip` kept groups
      load_row();
    }
    for (; skip > 0; --skip) ybits &= ybits - 1u;
    for (int st = 0; st < nst; ++st) mbar_init(&full[st], 1);
    fence_mbar_init();
    fence_proxy_async_smem();  // the stages may have been used through the generic proxy before
  }
  __syncwarp();

  auto issue = [&](int st) {  // lane 0: next kept group of the range into stage st
    RingGroup d;
    if (q >= q1) {
      d.kind = -1;
      desc[st] = d;
      mbar_arrive(&full[st]);
      more = false;
      return;
    }
    while (ybits == 0u) {
      if (++gr == kNgr) {
        gr = 0;
        ++slot;
        load_slot();
      }
      load_row();
    }
    const int b = __ffs(ybits) - 1;
    ybits &= ybits - 1u;
    d.n0 = q * 4;
    d.slot = slot;
    d.gi = gr * 16 + (b >> 1);
    d.t_index = t_index;
    d.src = frame + (long long)d.gi * 4 * row_el;
    ++q;
    if (d.n0 + 4 <= B.capacity && aligned) {
      d.kind = 0;
      desc[st] = d;
      mbar_arrive_expect_tx(&full[st], kRingGroupBytes);
      bulk_g2s(stages + (size_t)st * kRingStageAlloc, d.src, kRingGroupBytes, &full[st]);
    } else {
      d.kind = d.n0 < B.capacity ? 1 : 2;
      desc[st] = d;
      mbar_arrive(&full[st]);
    }
  };
  if (lane == 0)
    for (int st = 0; st < nst && more; ++st) issue(st);

  for (int it = 0;; ++it) {
    const int st = it % nst;
    mbar_wait(&full[st], (it / nst) & 1);
    const RingGroup d = desc[st];
    if (d.kind < 0) break;
    long long nvalid = B.capacity - d.n0;
    nvalid = nvalid < 0 ? 0 : (nvalid > 4 ? 4 : nvalid);
    if (d.kind == 0) {
      if (lane == 0) bulk_s2g(B.packed + d.n0 * row_el, stages + (size_t)st * kRingStageAlloc, kRingGroupBytes);
    } else if (d.kind == 1) {
      uint16_t* dst = B.packed + d.n0 * row_el;
      const int nel = static_cast<int>(nvalid * row_el);
      for (int e = lane; e < nel; e += 32) dst[e] = d.src[e];
    }
    if (lane < nvalid) {
      const int gr_ = d.gi >> 4, gc_ = d.gi & 15;
      const int h = gr_ * 2 + (lane >> 1), w = gc_ * 2 + (lane & 1);
      const long long n = d.n0 + lane;
      B.pos_ids[3 * n + 0] = d.t_index;
      B.pos_ids[3 * n + 1] = h;
      B.pos_ids[3 * n + 2] = w;
      B.src_index[n] = d.slot * 1024 + h * 32 + w;
    }
    __syncwarp();
    if (lane == 0) {
      bulk_commit();  // one (possibly empty) bulk group per consumed stage keeps the group count aligned
      if (it >= 1 && more) {
        bulk_wait_read<1>();  // the store of item it-1 has read its stage
        issue((it - 1) % nst);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    bulk_wait_all<0>();
    asm volatile("fence.proxy.async.global;" ::: "memory");  // bulk (async-proxy) writes before later generic sync
  }
  long long r = B.capacity - q_first * 4;
  r = r < 0 ? 0 : (r > (q1 - q_first) * 4 ? (q1 - q_first) * 4 : r);
  return r;
}

}  // namespace cs
