// compact.cu — codecsight_compact on sm_100a: stream compaction of kept patches into the packed ViT input
// ("executes the ViT only on the selected patches"; order = reading Q14, pos ids = Q15).
//
// Two launches:
//   compact_scan    one CTA: per-slot emitted-patch counts (groups with any keep bit x group^2) -> block-wide
//                   exclusive scan with a running carry -> frame_offsets (cu_seqlens); capacity status; counters.
//   compact_gather  persistent grid (a multiple of the SM count), one WARP per contiguous range of the flat
//                   kept-group index space [0, total/group^2), so every warp moves the same number of bytes
//                   whatever the per-frame kept fraction.  A warp locates its first slot by binary search over
//                   frame_offsets, enumerates that slot's kept groups with ballots, gathers each group's
//                   3 x (group*patch)^2 pixels from the bf16 frame with 8-byte loads into a per-warp shared
//                   memory tile laid out in packed order, and writes the tile out with coalesced 16-byte stores
//                   (a 2x2 group of 14-px patches = 4,704 B = 294 x 16 B, so every group starts 16-B aligned).
// Pixels of pruned patches are never read.
#include <cstdlib>

#include "cs_internal.cuh"

namespace {

constexpr int kScanThreads = 1024;
constexpr int kGatherThreads = 256;
constexpr int kWarpsPerCta = kGatherThreads / 32;

constexpr int kLayoutNV12 = 2;  // internal: frames are decoded NV12 planes, preprocessing fused (NEXT-2)
#ifndef CS_NV12_BATCH
#define CS_NV12_BATCH 2
#endif
#ifndef CS_NV12_CTAS
#define CS_NV12_CTAS 4
#endif
constexpr int kNvBatch = CS_NV12_BATCH;  // output pixels per lane in flight (fused NV12 fast path)
constexpr int kNvCtas = CS_NV12_CTAS;    // resident CTAs per SM of the fused NV12 kernel (register budget)
constexpr float kInv255 = 1.0f / 255.0f;  // RN(1/255)

// per-warp tile of one group in packed order: 3 x tp x (group*patch)^2 bf16, padded to 16 B
__host__ __device__ __forceinline__ int tile_bytes_of(int p, int G, int tp = 1) {
  return ((3 * tp * G * G * p * p * 2) + 15) & ~15;
}

struct CompactParams {
  int grid_w, grid_h, G, p, np, nw, ngc, ngroups;
  int n_streams, n_frames, n_slots;  // n_frames = token units per stream (frames when tp == 1)
  int tp;                             // temporal patch: frames per token unit (NEXT-3, Qwen2-VL: 2)
  long long mask_frame_stride;
  uint32_t* unit_mask;                // optional [n_streams][unit_mask_stride][nw] OR of the unit's masks
  long long unit_mask_stride;
  const uint8_t* frame_type;          // optional [n_streams][mask_frame_stride] -> unit_type
  uint8_t* unit_type;                 // optional [n_streams][unit_mask_stride]: I iff any frame is not P
  long long capacity;
  int FH, FW;  // model-input frame height / width in pixels
  int vec_out;
  int layout;  // CS_LAYOUT_PLANAR | CS_LAYOUT_GROUPED | kLayoutNV12
  // NV12 source (fused preprocessing, NEXT-2)
  int src_w, src_h, y_pitch, uv_pitch;
  float scale_y, scale_x;  // src / model, fp32 (computed once on the host, IEEE division)
  float mean[3], stdv[3];
  float rstd[3];  // RN(1 / std[c]) (host IEEE division)
  int fast_div;   // every std in [2^-20, 2^20]: bf16((t - mean) / std) through the guarded reciprocal (norm_bf16)
  const void* const* uv_planes;
  const uint32_t* keep_mask;
  const int32_t* frame_index;
  const void* const* frames;
  uint16_t* packed;
  int32_t* pos_ids;
  int32_t* src_index;
  int32_t* frame_offsets;
  unsigned long long* counters;
  int32_t* status;
};

// mask of frame f of token unit `slot` (frame j*tp + f of its stream)
__device__ __forceinline__ const uint32_t* slot_mask(const CompactParams& P, int slot, int f = 0) {
  const int s = slot / P.n_frames, j = slot - s * P.n_frames;
  return P.keep_mask + ((long long)s * P.mask_frame_stride + (long long)j * P.tp + f) * P.nw;
}

// word t of the unit mask: OR over the unit's tp frames (a group is emitted iff kept in any of them)
__device__ __forceinline__ uint32_t unit_word(const CompactParams& P, int slot, int t) {
  const uint32_t* m = slot_mask(P, slot);
  uint32_t w = __ldg(m + t);
  for (int f = 1; f < P.tp; ++f) w |= __ldg(m + (long long)f * P.nw + t);
  return w;
}

__device__ __forceinline__ void put_unit_word(const CompactParams& P, int slot, int t, uint32_t w) {
  const int s = slot / P.n_frames, j = slot - s * P.n_frames;
  P.unit_mask[((long long)s * P.unit_mask_stride + j) * P.nw + t] = w;
}

// Per-slot emitted-patch counts, one WARP per slot over the whole grid (lane l holds word l of the mask on 32-wide
// grids); the count goes to frame_offsets[slot] and is turned into the exclusive offset by compact_scan.  Also
// writes the unit masks / types of temporal patches.
constexpr int kCountThreads = 256;
__global__ void __launch_bounds__(kCountThreads) compact_count(const __grid_constant__ CompactParams P) {
  __shared__ uint32_t s_m[kCountThreads / 32][128];  // per-warp unit mask (grid_words <= 128)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = blockIdx.x * (kCountThreads / 32) + warp;
  if (slot >= P.n_slots) return;
  const int gs2 = P.G * P.G;
  int c = 0;
  if (P.G == 2 && P.grid_w == 32 && P.nw <= 32) {
    // word r = patch row r; group row g = rows 2g, 2g+1; fold horizontal pairs onto even bits
    const uint32_t wv = lane < P.nw ? (P.tp == 1 ? __ldg(slot_mask(P, slot) + lane) : unit_word(P, slot, lane)) : 0u;
    if (P.unit_mask && lane < P.nw) put_unit_word(P, slot, lane, wv);
    const uint32_t x = wv | __shfl_down_sync(0xffffffffu, wv, 1);
    c = (lane & 1) == 0 ? __popc((x | (x >> 1)) & 0x55555555u) : 0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) c += __shfl_down_sync(0xffffffffu, c, d);
  } else {
    const uint32_t* m = slot_mask(P, slot);
    if (P.tp > 1 || P.unit_mask) {
      for (int t = lane; t < P.nw; t += 32) {
        const uint32_t w = unit_word(P, slot, t);
        s_m[warp][t] = w;
        if (P.unit_mask) put_unit_word(P, slot, t, w);
      }
      __syncwarp();
      m = s_m[warp];
    }
    for (int q0 = 0; q0 < P.ngroups; q0 += 32) {
      const int q = q0 + lane;
      c += __popc(__ballot_sync(0xffffffffu, q < P.ngroups && cs::group_kept(m, q, P.ngc, P.G, P.grid_w)));
    }
  }
  if (lane == 0) {
    P.frame_offsets[slot] = c * gs2;
    if (P.unit_type) {
      const int s = slot / P.n_frames, j = slot - s * P.n_frames;
      const uint8_t* ft = P.frame_type + (long long)s * P.mask_frame_stride + (long long)j * P.tp;
      uint8_t ty = CS_FRAME_P;
      for (int f = 0; f < P.tp; ++f)
        if (ft[f] != CS_FRAME_P) ty = CS_FRAME_I;
      P.unit_type[(long long)s * P.unit_mask_stride + j] = ty;
    }
  }
}

// One CTA: frame_offsets[slot] (counts) -> exclusive scan in place (block-wide, running carry) + the total, capacity
// status and counters.
__global__ void __launch_bounds__(kScanThreads) compact_scan(const __grid_constant__ CompactParams P) {
  __shared__ int s_warp[kScanThreads / 32];
  __shared__ int s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < P.n_slots; base += kScanThreads) {
    const int slot = base + tid;
    const int cnt = slot < P.n_slots ? P.frame_offsets[slot] : 0;
    int inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += v;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      int v = s_warp[lane];
      int w = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += u;
      }
      s_warp[lane] = w - v;  // exclusive prefix of warp totals
    }
    __syncthreads();
    const int excl = s_carry + s_warp[warp] + inc - cnt;
    if (slot < P.n_slots) P.frame_offsets[slot] = excl;
    __syncthreads();
    if (tid == kScanThreads - 1) s_carry = excl + cnt;
    __syncthreads();
  }
  if (tid == 0) {
    const long long total = s_carry;
    P.frame_offsets[P.n_slots] = static_cast<int32_t>(total);
    const long long rows = total < P.capacity ? total : P.capacity;
    if (total > P.capacity) cs::atomic_or_status(P.status, CS_STATUS_CAPACITY);
    const unsigned long long row_bytes = 3ull * P.tp * P.p * P.p * 2ull;
    cs::atomic_add_u64(&P.counters[CS_CNT_PACKED_ROWS], static_cast<unsigned long long>(rows));
    // per packed row: its bytes read from the frame and written (+16 B of ids); with the fused NV12 path the
    // source pixels depend on the scale and are not counted here (write side only, as in the oracle)
    const unsigned long long per_row = (P.layout == kLayoutNV12 ? 1ull : 2ull) * row_bytes + 16ull;
    cs::atomic_add_u64(&P.counters[CS_CNT_BYTES_COMPACT],
                       static_cast<unsigned long long>(P.n_slots) * (4ull * P.nw * P.tp + 4ull) +
                           (P.unit_mask ? static_cast<unsigned long long>(P.n_slots) * 4ull * P.nw : 0ull) +
                           (P.unit_type ? static_cast<unsigned long long>(P.n_slots) * (P.tp + 1ull) : 0ull) +
                           static_cast<unsigned long long>(rows) * per_row);
  }
}


// ---- fused preprocessing (NEXT-2): NV12 -> RGB (BT.601 limited) -> bilinear resize -> /255 -> normalise ------
// Same fp32 operations in the same order as the oracle (oracle/codecsight_ref.c, codecsight_ref_model_pixel).
__device__ __forceinline__ void nv12_axis(int o, int src, float scale, int& i0, int& i1, float& l) {
  float f = __fsub_rn(__fmul_rn(__fadd_rn(static_cast<float>(o), 0.5f), scale), 0.5f);
  f = f < 0.0f ? 0.0f : f;
  i0 = static_cast<int>(f);
  i1 = i0 + (i0 < src - 1 ? 1 : 0);
  l = __fsub_rn(f, static_cast<float>(i0));
}

// bf16 bits of RN_bf16(RN_f32(a / std)) -- the oracle's fp32 division then round-to-nearest-even to bf16 --
// without the IEEE division in the common case.  q = RN(a * RN(1/std)) is within 2.5 ulp of a / std (relative
// error < 2^-23 + 2^-48; |q - RN(a/std)| <= 5 fp32 steps even across a binade edge), so q and RN(a/std) round to
// the same bf16 unless a bf16 rounding midpoint (low 16 bits 0x8000) lies within 8 steps of q; only then is the
// exact division taken.  Valid for std in [2^-20, 2^20] and |mean| <= 2^60 (fast_div: q stays normal, no overflow); the
// outputs are never NaN.  Pinned in scripts/check_norm_bf16.c / tests/test_div255.py.
__device__ __forceinline__ uint16_t norm_bf16(float a, float stdv, float rstd, bool fast) {
  float q;
  if (fast) {
    q = __fmul_rn(a, rstd);
    if ((__float_as_uint(q) & 0xffffu) - 0x7ff8u <= 16u) q = __fdiv_rn(a, stdv);
  } else {
    q = __fdiv_rn(a, stdv);
  }
  return cs::f32_to_bf16_cvt(q);
}

// Gather one kept group (gr, gc) of `frame` into the warp tile and write it to packed rows [n0, n0 + G^2).
// TT = frames per token unit (temporal patch, NEXT-3); 0 = runtime P.tp.  With TT > 1 the packed row is
// [3][TT][p][p] and tile element (patch q, c, f, y, x) sits at ((q*3 + c)*TT + f)*p*p + y*p + x.
template <int TP, int TG, int LAYOUT, int TT>
__device__ __forceinline__ void gather_group(const CompactParams& P, const uint16_t* __restrict__ frame,
                                             bool vec_in, int gr, int gc, long long n0, int slot, int t_index,
                                             uint16_t* tile, int lane) {
  const int p = TP > 0 ? TP : P.p;
  const int G = TG > 0 ? TG : P.G;
  const int tp = TT > 0 ? TT : P.tp;
  const int gp = G * p;  // group edge in pixels
  const int pp = p * p;
  const long long FW = P.FW;
  const long long plane = (long long)P.FH * FW;
  if (LAYOUT == CS_LAYOUT_GROUPED && tp > 1) {
    // direct, no staging: every 16-B store of the group's output rows [q][3][tp][p][p] is assembled from two 8-B loads of the
    // unit's frames (a p*p segment is a multiple of 4 elements, so a 4-element half never straddles segments)
    const int gs2 = G * G;
    long long nvalid = P.capacity - n0;
    nvalid = nvalid < 0 ? 0 : (nvalid > gs2 ? gs2 : nvalid);
    const int row_el = 3 * tp * pp;
    const long long goff = ((long long)gr * P.ngc + gc) * ((long long)gs2 * 3 * pp);
    const uint16_t* fb[4];
#pragma unroll
    for (int f = 0; f < 4; ++f)
      fb[f] = f < tp ? (f == 0 ? frame : static_cast<const uint16_t*>(P.frames[(long long)slot * tp + f])) + goff
                     : frame;
    auto src_of = [&](int el) -> const uint16_t* {
      const int q = el / row_el, r = el - q * row_el;
      const int c = r / (tp * pp), r2 = r - c * tp * pp;
      const int f = r2 / pp, x = r2 - f * pp;
      const uint16_t* b = f == 0 ? fb[0] : (f == 1 ? fb[1] : (f == 2 ? fb[2] : fb[3]));
      return b + (q * 3 + c) * pp + x;
    };
    uint16_t* dst = P.packed + n0 * row_el;
    const int nel = static_cast<int>(nvalid) * row_el;
    const int n16 = nel / 8;
    if (!(vec_in && P.vec_out)) {  // unaligned frames or rows: element copies
      for (int e = lane; e < nel; e += 32) dst[e] = *src_of(e);
    } else {
    for (int e = n16 * 8 + lane; e < nel; e += 32) dst[e] = *src_of(e);  // tail of a truncated group
    constexpr int kU = TP > 0 ? 4 : 1;  // the generic (runtime-shape) instance stays within 64 registers
    for (int e0 = 0; e0 < n16; e0 += 32 * kU) {
      uint2 lo[kU], hi[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * 32 + lane;
        if (e < n16) {
          lo[u] = cs::ld_nc_v2(src_of(8 * e));
          hi[u] = cs::ld_nc_v2(src_of(8 * e + 4));
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * 32 + lane;
        if (e < n16) reinterpret_cast<uint4*>(dst)[e] = make_uint4(lo[u].x, lo[u].y, hi[u].x, hi[u].y);
      }
    }
    }
    if (lane < nvalid) {
      const int dy = lane / G, dx = lane - dy * G;
      const int h = gr * G + dy, w = gc * G + dx;
      const long long n = n0 + lane;
      P.pos_ids[3 * n + 0] = t_index;
      P.pos_ids[3 * n + 1] = h;
      P.pos_ids[3 * n + 2] = w;
      P.src_index[n] = slot * P.np + h * P.grid_w + w;
    }
    return;
  }
  if (LAYOUT == CS_LAYOUT_GROUPED) {
    // the kept group is one contiguous block already in packed order: straight 16-B copy (no smem staging)
    const int gs2 = G * G;
    long long nvalid = P.capacity - n0;
    nvalid = nvalid < 0 ? 0 : (nvalid > gs2 ? gs2 : nvalid);
    const long long row_el = 3ll * pp;
    const uint16_t* blk = frame + ((long long)gr * P.ngc + gc) * gs2 * row_el;
    uint16_t* dst = P.packed + n0 * row_el;
    if (vec_in && P.vec_out) {
      const int nel = static_cast<int>(nvalid * row_el);
      const int n16 = nel / 8;
      for (int e = n16 * 8 + lane; e < nel; e += 32) dst[e] = blk[e];  // tail of a truncated group
      const uint4* s4 = reinterpret_cast<const uint4*>(blk);
      uint4* d4 = reinterpret_cast<uint4*>(dst);
      constexpr int kU = 5;
      for (int e0 = 0; e0 < n16; e0 += 32 * kU) {
        uint4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int e = e0 + u * 32 + lane;
          if (e < n16) v[u] = cs::ld_nc_v4(s4 + e);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int e = e0 + u * 32 + lane;
          if (e < n16) d4[e] = v[u];
        }
      }
    } else {
      const int nel = static_cast<int>(nvalid * row_el);
      for (int e = lane; e < nel; e += 32) dst[e] = blk[e];
    }
    if (lane < nvalid) {
      const int dy = lane / G, dx = lane - dy * G;
      const int h = gr * G + dy, w = gc * G + dx;
      const long long n = n0 + lane;
      P.pos_ids[3 * n + 0] = t_index;
      P.pos_ids[3 * n + 1] = h;
      P.pos_ids[3 * n + 2] = w;
      P.src_index[n] = slot * P.np + h * P.grid_w + w;
    }
    return;
  }
  if (LAYOUT == kLayoutNV12) {
    // preprocess only the kept group's 3 x gp x gp model pixels straight from the decoded NV12 frame
    const uint8_t* Yp = reinterpret_cast<const uint8_t*>(frame);
    const uint8_t* UVp = static_cast<const uint8_t*>(P.uv_planes[slot]);
    const float kY = 1.164383f, kRV = 1.596027f, kGU = 0.391762f, kGV = 0.812968f, kBU = 2.017232f;
    if (TP > 0 && TG == 2 && gp <= 32) {
      // fast path (issue-bound: every instruction per pixel counts).  The source taps of output column xx / row yy
      // are computed once per group by lane xx / yy and fetched with shuffles; the pixel's (yy, xx) advance by
      // (32 / gp, 32 % gp) per round; the bf16 store is the hardware RNE conversion (the outputs are never NaN:
      // std > 0 and mean is not NaN are checked on the host, so it equals the oracle's rounding bit for bit).
      int ax0 = 0, ay0 = 0;
      float alx = 0.0f, aly = 0.0f;
      if (lane < gp) {
        int i1;
        nv12_axis(gc * gp + lane, P.src_w, P.scale_x, ax0, i1, alx);
        nv12_axis(gr * gp + lane, P.src_h, P.scale_y, ay0, i1, aly);
      }
      int yy = lane / gp, xx = lane - (lane / gp) * gp;
      // two output pixels per lane per iteration (rounds e0 and e0 + 32): their 16 loads are all in flight
      // before either is converted (the kernel is latency-bound on these scattered byte loads)
      const int npx = gp * gp;
      for (int e0 = 0; e0 < npx; e0 += 32 * kNvBatch) {  // warp-uniform trip count (the shuffles need every lane)
        uint32_t yv[kNvBatch][4], uvv[kNvBatch][4];
        float lxv[kNvBatch], lyv[kNvBatch];
        int pxx[kNvBatch], pyy[kNvBatch];
        bool valid[kNvBatch];
#pragma unroll
        for (int b = 0; b < kNvBatch; ++b) {
          // lanes past the group's end fetch an in-group pixel (valid addresses) and do not emit it
          valid[b] = e0 + 32 * b + lane < npx;
          pxx[b] = valid[b] ? xx : 0;
          pyy[b] = valid[b] ? yy : 0;
          const int x0 = __shfl_sync(0xffffffffu, ax0, pxx[b]), y0 = __shfl_sync(0xffffffffu, ay0, pyy[b]);
          lxv[b] = __shfl_sync(0xffffffffu, alx, pxx[b]);
          lyv[b] = __shfl_sync(0xffffffffu, aly, pyy[b]);
          const int x1 = x0 + (x0 < P.src_w - 1 ? 1 : 0), y1 = y0 + (y0 < P.src_h - 1 ? 1 : 0);
          const uint8_t* r0 = Yp + (long long)y0 * P.y_pitch;
          const uint8_t* r1 = Yp + (long long)y1 * P.y_pitch;
          const uint8_t* c0 = UVp + (long long)(y0 >> 1) * P.uv_pitch;
          const uint8_t* c1 = UVp + (long long)(y1 >> 1) * P.uv_pitch;
          yv[b][0] = __ldg(r0 + x0);
          yv[b][1] = __ldg(r0 + x1);
          yv[b][2] = __ldg(r1 + x0);
          yv[b][3] = __ldg(r1 + x1);
          uvv[b][0] = __ldg(reinterpret_cast<const uint16_t*>(c0 + 2 * (x0 >> 1)));
          uvv[b][1] = __ldg(reinterpret_cast<const uint16_t*>(c0 + 2 * (x1 >> 1)));
          uvv[b][2] = __ldg(reinterpret_cast<const uint16_t*>(c1 + 2 * (x0 >> 1)));
          uvv[b][3] = __ldg(reinterpret_cast<const uint16_t*>(c1 + 2 * (x1 >> 1)));
          // (yy, xx) of this lane's next pixel (32 further in row-major order)
          xx += 32 % gp;
          yy += 32 / gp;
          if (xx >= gp) {
            xx -= gp;
            ++yy;
          }
        }
#pragma unroll
        for (int b = 0; b < kNvBatch; ++b) {
          if (!valid[b]) continue;
          float rgb[4][3];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float c = static_cast<float>(static_cast<int>(yv[b][q]) - 16);
            const float d = static_cast<float>(static_cast<int>(uvv[b][q] & 0xffu) - 128);
            const float ee = static_cast<float>(static_cast<int>(uvv[b][q] >> 8) - 128);
            rgb[q][0] = fminf(fmaxf(__fadd_rn(__fmul_rn(kY, c), __fmul_rn(kRV, ee)), 0.0f), 255.0f);
            rgb[q][1] = fminf(fmaxf(__fsub_rn(__fsub_rn(__fmul_rn(kY, c), __fmul_rn(kGU, d)), __fmul_rn(kGV, ee)),
                                    0.0f), 255.0f);
            rgb[q][2] = fminf(fmaxf(__fadd_rn(__fmul_rn(kY, c), __fmul_rn(kBU, d)), 0.0f), 255.0f);
          }
          const float lx = lxv[b], ly = lyv[b];
          const float hx = __fsub_rn(1.0f, lx), hy = __fsub_rn(1.0f, ly);
          const int dy = pyy[b] >= p ? 1 : 0, y = pyy[b] - dy * p, dx = pxx[b] >= p ? 1 : 0, x = pxx[b] - dx * p;
          uint16_t* tq = tile + (dy * G + dx) * 3 * pp + y * p + x;
          float an[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const float top = __fadd_rn(__fmul_rn(hx, rgb[0][c]), __fmul_rn(lx, rgb[1][c]));
            const float bot = __fadd_rn(__fmul_rn(hx, rgb[2][c]), __fmul_rn(lx, rgb[3][c]));
            const float v = __fadd_rn(__fmul_rn(hy, top), __fmul_rn(ly, bot));
            // v / 255 correctly rounded without a division: q = v * RN(1/255), one fma residual correction.
            // Exhaustively verified equal to IEEE v / 255 for every fp32 v in [0, 512] (scripts/check_div255.c)
            const float q255 = __fmul_rn(v, kInv255);
            const float t = __fmaf_rn(__fmaf_rn(-q255, 255.0f, v), kInv255, q255);
            an[c] = __fsub_rn(t, P.mean[c]);
          }
          // (t - mean) / std -> bf16 (norm_bf16), the three channels' midpoint guards folded into one branch
          float on[3];
          uint32_t near_mid = 0u;
          if (P.fast_div) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              on[c] = __fmul_rn(an[c], P.rstd[c]);
              near_mid |= static_cast<uint32_t>((__float_as_uint(on[c]) & 0xffffu) - 0x7ff8u <= 16u);
            }
          }
          if (!P.fast_div || near_mid) {
#pragma unroll
            for (int c = 0; c < 3; ++c) on[c] = __fdiv_rn(an[c], P.stdv[c]);
          }
#pragma unroll
          for (int c = 0; c < 3; ++c) tq[c * pp] = cs::f32_to_bf16_cvt(on[c]);
        }
      }
    } else {
    // generic path: batches of 4 output pixels per lane: the 4 x (4 luma bytes + 4 chroma pairs) loads of a batch
    // are all issued before any is consumed (memory-level parallelism), then converted, interpolated, normalised
    constexpr int kB = 4;
    for (int e0 = 0; e0 < gp * gp; e0 += 32 * kB) {
      uint32_t yv[kB][4], uvv[kB][4];
      float lyv[kB], lxv[kB];
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int e = e0 + b * 32 + lane;
        if (e < gp * gp) {
          const int yy = e / gp, xx = e - yy * gp;
          int y0, y1, x0, x1;
          nv12_axis(gr * gp + yy, P.src_h, P.scale_y, y0, y1, lyv[b]);
          nv12_axis(gc * gp + xx, P.src_w, P.scale_x, x0, x1, lxv[b]);
          const int ys[4] = {y0, y0, y1, y1}, xs[4] = {x0, x1, x0, x1};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            yv[b][q] = __ldg(Yp + (long long)ys[q] * P.y_pitch + xs[q]);
            uvv[b][q] = __ldg(reinterpret_cast<const uint16_t*>(UVp + (long long)(ys[q] >> 1) * P.uv_pitch +
                                                                2 * (xs[q] >> 1)));
          }
        }
      }
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int e = e0 + b * 32 + lane;
        if (e >= gp * gp) continue;
        float rgb[4][3];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float c = static_cast<float>(static_cast<int>(yv[b][q]) - 16);
          const float d = static_cast<float>(static_cast<int>(uvv[b][q] & 0xffu) - 128);
          const float ee = static_cast<float>(static_cast<int>(uvv[b][q] >> 8) - 128);
          rgb[q][0] = fminf(fmaxf(__fadd_rn(__fmul_rn(kY, c), __fmul_rn(kRV, ee)), 0.0f), 255.0f);
          rgb[q][1] = fminf(fmaxf(__fsub_rn(__fsub_rn(__fmul_rn(kY, c), __fmul_rn(kGU, d)), __fmul_rn(kGV, ee)), 0.0f),
                            255.0f);
          rgb[q][2] = fminf(fmaxf(__fadd_rn(__fmul_rn(kY, c), __fmul_rn(kBU, d)), 0.0f), 255.0f);
        }
        const float lx = lxv[b], ly = lyv[b];
        const float hx = __fsub_rn(1.0f, lx), hy = __fsub_rn(1.0f, ly);
        const int yy = e / gp, xx = e - yy * gp;
        const int dy = yy / p, y = yy - dy * p, dx = xx / p, x = xx - dx * p;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float top = __fadd_rn(__fmul_rn(hx, rgb[0][c]), __fmul_rn(lx, rgb[1][c]));
          const float bot = __fadd_rn(__fmul_rn(hx, rgb[2][c]), __fmul_rn(lx, rgb[3][c]));
          const float v = __fadd_rn(__fmul_rn(hy, top), __fmul_rn(ly, bot));
          const float q255 = __fmul_rn(v, kInv255);
          const float t = __fmaf_rn(__fmaf_rn(-q255, 255.0f, v), kInv255, q255);
          tile[((dy * G + dx) * 3 + c) * pp + y * p + x] =
              norm_bf16(__fsub_rn(t, P.mean[c]), P.stdv[c], P.rstd[c], P.fast_div != 0);
        }
      }
    }
    }
  } else if (vec_in) {
    // 8-byte loads: each group row segment is gp pixels = gp/4 pieces of 4 bf16.  Pairs of pixels never
    // straddle a patch boundary (p even), so the tile is written with 4-byte stores.
   for (int f = 0; f < tp; ++f) {
    const uint16_t* src0 = (f == 0 ? frame : static_cast<const uint16_t*>(P.frames[(long long)slot * tp + f])) +
                           (long long)(gr * gp) * FW + (long long)gc * gp;
    const int cpr = gp / 4;
    const int total = 3 * gp * cpr;
    constexpr int kUnroll = (TP > 0) ? 10 : 4;  // 588 8-B pieces of a 2x2 group of 14-px patches: 2 rounds
    for (int e0 = 0; e0 < total; e0 += 32 * kUnroll) {
      uint2 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int e = e0 + u * 32 + lane;
        if (e < total) {
          const int row = e / cpr, piece = e - row * cpr;
          const int c = row / gp, yy = row - c * gp;
          v[u] = cs::ld_nc_v2(src0 + c * plane + (long long)yy * FW + piece * 4);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int e = e0 + u * 32 + lane;
        if (e < total) {
          const int row = e / cpr, piece = e - row * cpr;
          const int c = row / gp, yy = row - c * gp;
          const int dy = yy / p, y = yy - dy * p;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int x = piece * 4 + 2 * k;
            const int dx = x / p, xx = x - dx * p;
            const int idx = (((dy * G + dx) * 3 + c) * tp + f) * pp + y * p + xx;
            *reinterpret_cast<uint32_t*>(tile + idx) = k == 0 ? v[u].x : v[u].y;
          }
        }
      }
    }
   }
  } else {
    for (int f = 0; f < tp; ++f) {
      const uint16_t* src0 = (f == 0 ? frame : static_cast<const uint16_t*>(P.frames[(long long)slot * tp + f])) +
                             (long long)(gr * gp) * FW + (long long)gc * gp;
      const int total = 3 * gp * gp;
      for (int e = lane; e < total; e += 32) {
        const int row = e / gp, x = e - row * gp;
        const int c = row / gp, yy = row - c * gp;
        const int dy = yy / p, y = yy - dy * p, dx = x / p, xx = x - dx * p;
        tile[(((dy * G + dx) * 3 + c) * tp + f) * pp + y * p + xx] = src0[c * plane + (long long)yy * FW + x];
      }
    }
  }
  __syncwarp();
  const int gs2 = G * G;
  long long nvalid = P.capacity - n0;
  nvalid = nvalid < 0 ? 0 : (nvalid > gs2 ? gs2 : nvalid);
  const long long row_el = 3ll * tp * pp;
  uint16_t* dst = P.packed + n0 * row_el;
  if (P.vec_out) {
    const int nel = static_cast<int>(nvalid * row_el);
    const int n16 = nel / 8;
    const uint4* t4 = reinterpret_cast<const uint4*>(tile);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int e = lane; e < n16; e += 32) d4[e] = t4[e];
    for (int e = n16 * 8 + lane; e < nel; e += 32) dst[e] = tile[e];  // tail of a truncated group
  } else {
    const int nel = static_cast<int>(nvalid * row_el);
    for (int e = lane; e < nel; e += 32) dst[e] = tile[e];
  }
  if (lane < nvalid) {
    const int dy = lane / G, dx = lane - dy * G;
    const int h = gr * G + dy, w = gc * G + dx;
    const long long n = n0 + lane;
    P.pos_ids[3 * n + 0] = t_index;
    P.pos_ids[3 * n + 1] = h;
    P.pos_ids[3 * n + 2] = w;
    P.src_index[n] = slot * P.np + h * P.grid_w + w;
  }
  __syncwarp();  // tile reusable
}

template <int TP, int TG, int LAYOUT, int TT>
__global__ void __launch_bounds__(kGatherThreads, (LAYOUT == CS_LAYOUT_GROUPED && TP > 0) ? 4 : (LAYOUT == kLayoutNV12 && TP > 0) ? kNvCtas : 2)
    compact_gather(const __grid_constant__ CompactParams P) {
  extern __shared__ __align__(16) unsigned char g_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int G = TG > 0 ? TG : P.G;
  const int gs2 = G * G;
  const long long total_groups = static_cast<long long>(P.frame_offsets[P.n_slots]) / gs2;
  const long long nwarps = static_cast<long long>(gridDim.x) * kWarpsPerCta;
  const long long wid = static_cast<long long>(blockIdx.x) * kWarpsPerCta + wib;
  long long q = total_groups * wid / nwarps;
  const long long q1 = total_groups * (wid + 1) / nwarps;
  if (q >= q1) return;
  const int tp = TT > 0 ? TT : P.tp;
  const int tile_bytes = LAYOUT == CS_LAYOUT_GROUPED ? 0 : tile_bytes_of(TP > 0 ? TP : P.p, G, tp);
  uint16_t* tile = reinterpret_cast<uint16_t*>(g_smem + (size_t)wib * tile_bytes);
  uint32_t* mask = reinterpret_cast<uint32_t*>(g_smem + (size_t)kWarpsPerCta * tile_bytes) + wib * P.nw;

  // slot containing group q: largest slot with frame_offsets[slot] <= q * gs2
  int lo = 0, hi = P.n_slots;  // invariant: off[lo] <= x < off[hi]
  const long long x = q * gs2;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (static_cast<long long>(__ldg(P.frame_offsets + mid)) <= x) lo = mid; else hi = mid;
  }
  int slot = lo;
  long long skip = q - __ldg(P.frame_offsets + slot) / gs2;  // kept groups of the slot before q

  while (q < q1 && slot < P.n_slots) {
    for (int t = lane; t < P.nw; t += 32) mask[t] = tp == 1 ? __ldg(slot_mask(P, slot) + t) : unit_word(P, slot, t);
    const uint16_t* frame = static_cast<const uint16_t*>(P.frames[(long long)slot * tp]);
    const int t_index = __ldg(P.frame_index + slot);
    const int pe = TP > 0 ? TP : P.p;
    uintptr_t align_or = reinterpret_cast<uintptr_t>(frame);
    for (int f = 1; f < tp; ++f) align_or |= reinterpret_cast<uintptr_t>(P.frames[(long long)slot * tp + f]);
    const bool vec_in =
        LAYOUT == CS_LAYOUT_GROUPED
            ? (tp == 1 ? (((align_or & 15u) == 0) && ((3 * G * G * pe * pe * 2) % 16 == 0))
                       : (((align_or & 7u) == 0) && ((pe * pe) % 4 == 0)))
            : (((align_or & 7u) == 0) && ((P.FW & 3) == 0) && (((G * pe) & 3) == 0) && ((pe & 1) == 0));
    __syncwarp();
    for (int base = 0; base < P.ngroups && q < q1; base += 32) {
      const int qq = base + lane;
      const bool kept = qq < P.ngroups && cs::group_kept(mask, qq, P.ngc, G, P.grid_w);
      uint32_t bal = __ballot_sync(0xffffffffu, kept);
      const int nb = __popc(bal);
      if (skip >= nb) {
        skip -= nb;
        continue;
      }
      while (skip > 0) {  // drop the groups before q
        bal &= bal - 1;
        --skip;
      }
      while (bal && q < q1) {
        const int b = __ffs(bal) - 1;
        bal &= bal - 1;
        const int gi = base + b;
        const int gr = gi / P.ngc, gc = gi - gr * P.ngc;
        const long long n0 = q * gs2;
        if (n0 < P.capacity) gather_group<TP, TG, LAYOUT, TT>(P, frame, vec_in, gr, gc, n0, slot, t_index, tile, lane);
        ++q;
      }
    }
    ++slot;
    skip = 0;
  }
}

// ---- grouped frames, 2x2 groups of 14-px patches on a 32-wide grid: TMA bulk copies ------------------------
// A kept group is one contiguous 4,704-B block of the frame and of the packed output (16-B aligned): each warp is
// an independent TMA ring (lane 0 drives it, like kv_gather_tma): cp.async.bulk global -> smem completes on the
// stage's mbarrier, cp.async.bulk smem -> global (bulk_group) writes the packed rows, and the stage is refilled once
// wait_group.read says the store has read it.  Groups that cannot take the bulk path (a capacity-truncated group, a
// misaligned frame) are copied by the warp with ordinary loads/stores in the same order.
constexpr int kTmaWarps = kWarpsPerCta;
constexpr int kTmaMaxStages = 8;
constexpr unsigned kTmaGroupBytes = 4704u;  // 4 patches x 3 x 14 x 14 bf16
constexpr unsigned kTmaStageAlloc = 4736u;  // rounded up to 128 B

struct TmaGroup {
  long long n0;     // first packed row
  int slot;         // frame slot
  int gi;           // group index gr * ngc + gc
  int t_index;      // pos id t
  int kind;         // 0 bulk, 1 direct (warp copy), -1 end of work
  const uint16_t* src;
};

__global__ void __launch_bounds__(kGatherThreads, 1) compact_gather_tma(const __grid_constant__ CompactParams P,
                                                                        int nst) {
  extern __shared__ __align__(128) unsigned char t_smem[];
  __shared__ TmaGroup s_desc[kTmaWarps][kTmaMaxStages];
  __shared__ __align__(8) uint64_t s_full[kTmaWarps][kTmaMaxStages];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* stages = t_smem + (size_t)wib * nst * kTmaStageAlloc;
  uint64_t* full = s_full[wib];
  TmaGroup* desc = s_desc[wib];
  const long long total_groups = static_cast<long long>(__ldg(P.frame_offsets + P.n_slots)) / 4;
  const long long nwarps = static_cast<long long>(gridDim.x) * kTmaWarps;
  const long long wid = static_cast<long long>(blockIdx.x) * kTmaWarps + wib;
  long long q = total_groups * wid / nwarps;
  const long long q1 = total_groups * (wid + 1) / nwarps;
  if (q >= q1) return;  // the warp's range is empty (no block-wide synchronisation below)
  constexpr int kNgr = 16;  // group rows of a 32 x 32 patch grid
  const long long row_el = 3ll * 14 * 14;

  // ---- generator state (lane 0): current slot, group row, remaining kept-group bits of that row -------------
  int slot = 0, gr = 0, t_index = 0;
  uint32_t ybits = 0u;
  const uint16_t* frame = nullptr;
  bool aligned = false;
  auto load_row = [&]() {
    const uint32_t* m = slot_mask(P, slot);
    const uint32_t x = __ldg(m + 2 * gr) | __ldg(m + 2 * gr + 1);
    ybits = (x | (x >> 1)) & 0x55555555u;  // bit 2*gc set iff group (gr, gc) is kept
  };
  auto load_slot = [&]() {
    frame = static_cast<const uint16_t*>(P.frames[slot]);
    t_index = __ldg(P.frame_index + slot);
    aligned = (reinterpret_cast<uintptr_t>(frame) & 15u) == 0;
  };
  bool more = true;
  if (lane == 0) {
    int lo = 0, hi = P.n_slots;  // largest slot with frame_offsets[slot] <= q * 4
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (static_cast<long long>(__ldg(P.frame_offsets + mid)) <= q * 4) lo = mid; else hi = mid;
    }
    slot = lo;
    long long skip = q - __ldg(P.frame_offsets + slot) / 4;
    load_slot();
    load_row();
    while (skip >= __popc(ybits)) {
      skip -= __popc(ybits);
      ++gr;  // stays inside the slot: the slot holds more than `skip` kept groups
      load_row();
    }
    for (; skip > 0; --skip) ybits &= ybits - 1u;
    for (int st = 0; st < nst; ++st) cs::mbar_init(&full[st], 1);
    cs::fence_mbar_init();
  }
  __syncwarp();

  auto issue = [&](int st) {  // lane 0: next kept group of the range into stage st
    TmaGroup d;
    if (q >= q1) {
      d.kind = -1;
      desc[st] = d;
      cs::mbar_arrive(&full[st]);
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
    if (d.n0 + 4 <= P.capacity && aligned) {
      d.kind = 0;
      desc[st] = d;
      cs::mbar_arrive_expect_tx(&full[st], kTmaGroupBytes);
      cs::bulk_g2s(stages + (size_t)st * kTmaStageAlloc, d.src, kTmaGroupBytes, &full[st]);
    } else {
      d.kind = d.n0 < P.capacity ? 1 : 2;  // 2: entirely beyond the capacity, nothing to write
      desc[st] = d;
      cs::mbar_arrive(&full[st]);
    }
  };
  if (lane == 0)
    for (int st = 0; st < nst && more; ++st) issue(st);

  for (int it = 0;; ++it) {
    const int st = it % nst;
    cs::mbar_wait(&full[st], (it / nst) & 1);
    const TmaGroup d = desc[st];
    if (d.kind < 0) break;
    long long nvalid = P.capacity - d.n0;
    nvalid = nvalid < 0 ? 0 : (nvalid > 4 ? 4 : nvalid);
    if (d.kind == 0) {
      if (lane == 0) cs::bulk_s2g(P.packed + d.n0 * row_el, stages + (size_t)st * kTmaStageAlloc, kTmaGroupBytes);
    } else if (d.kind == 1) {
      uint16_t* dst = P.packed + d.n0 * row_el;
      const int nel = static_cast<int>(nvalid * row_el);
      for (int e = lane; e < nel; e += 32) dst[e] = d.src[e];
    }
    if (lane < nvalid) {
      const int gr_ = d.gi >> 4, gc_ = d.gi & 15;
      const int h = gr_ * 2 + (lane >> 1), w = gc_ * 2 + (lane & 1);
      const long long n = d.n0 + lane;
      P.pos_ids[3 * n + 0] = d.t_index;
      P.pos_ids[3 * n + 1] = h;
      P.pos_ids[3 * n + 2] = w;
      P.src_index[n] = d.slot * P.np + h * 32 + w;
    }
    __syncwarp();
    if (lane == 0) {
      cs::bulk_commit();  // one (possibly empty) bulk group per consumed stage keeps the group count aligned
      if (it >= 1 && more) {
        cs::bulk_wait_read<1>();  // the store of item it-1 has read its stage
        issue((it - 1) % nst);
      }
    }
    __syncwarp();
  }
  if (lane == 0) cs::bulk_wait_all<0>();
}

}  // namespace

static int launch_compact(const cs_grid* g, const cs_preprocess* pre, int32_t tp, int32_t n_streams,
                          int32_t n_frames, const uint32_t* keep_mask, int64_t mask_frame_stride,
                          const int32_t* frame_index, const void* const* frames, const void* const* uv_planes,
                          int32_t frame_layout, int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                          int32_t* frame_offsets, uint32_t* unit_mask, int64_t unit_mask_stride,
                          const uint8_t* frame_type, uint8_t* unit_type, unsigned long long* counters,
                          int32_t* status, cudaStream_t stream) {
  CompactParams P{};
  P.grid_w = g->grid_w;
  P.grid_h = g->grid_h;
  P.G = g->group;
  P.p = g->patch;
  P.np = g->grid_w * g->grid_h;
  P.nw = (P.np + 31) / 32;
  P.ngc = g->grid_w / g->group;
  P.ngroups = (g->grid_h / g->group) * P.ngc;
  P.n_streams = n_streams;
  P.n_frames = n_frames;
  P.n_slots = n_streams * n_frames;
  P.tp = tp;
  P.unit_mask = unit_mask;
  P.unit_mask_stride = unit_mask_stride;
  P.frame_type = frame_type;
  P.unit_type = unit_type;
  P.mask_frame_stride = mask_frame_stride;
  P.capacity = capacity;
  P.FH = g->grid_h * g->patch;
  P.FW = g->grid_w * g->patch;
  const long long row_bytes = 3ll * tp * g->patch * g->patch * 2ll;
  // every group starts at row n0 = q * group^2, i.e. at byte n0 * row_bytes: 16-B aligned iff a whole group is
  // a multiple of 16 B (4,704 B for 2x2 groups of 14-px patches); a capacity-truncated group ends with a tail
  P.vec_out = ((reinterpret_cast<uintptr_t>(packed) & 15u) == 0 &&
               ((row_bytes * g->group * g->group) % 16) == 0) ? 1 : 0;
  P.layout = frame_layout;
  if (pre) {
    P.src_w = pre->src_w;
    P.src_h = pre->src_h;
    P.y_pitch = pre->y_pitch;
    P.uv_pitch = pre->uv_pitch;
    P.scale_y = static_cast<float>(pre->src_h) / static_cast<float>(P.FH);
    P.scale_x = static_cast<float>(pre->src_w) / static_cast<float>(P.FW);
    P.fast_div = 1;
    for (int c = 0; c < 3; ++c) {
      P.mean[c] = pre->mean[c];
      P.stdv[c] = pre->std[c];
      P.rstd[c] = 1.0f / pre->std[c];
      if (!(pre->std[c] >= 0x1p-20f && pre->std[c] <= 0x1p20f && fabsf(pre->mean[c]) <= 0x1p60f)) P.fast_div = 0;
    }
    P.uv_planes = uv_planes;
  }
  P.keep_mask = keep_mask;
  P.frame_index = frame_index;
  P.frames = frames;
  P.packed = static_cast<uint16_t*>(packed);
  P.pos_ids = pos_ids;
  P.src_index = src_index;
  P.frame_offsets = frame_offsets;
  P.counters = counters;
  P.status = status;

  if (P.n_slots > 0) {
    compact_count<<<(P.n_slots + kCountThreads / 32 - 1) / (kCountThreads / 32), kCountThreads, 0, stream>>>(P);
    if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
  }
  compact_scan<<<1, kScanThreads, 0, stream>>>(P);
  if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
  if (P.n_slots == 0 || capacity == 0) return CS_OK;
  const bool grouped = frame_layout == CS_LAYOUT_GROUPED;
  const bool nv12 = frame_layout == kLayoutNV12;
  const size_t smem =
      (size_t)kWarpsPerCta * ((grouped ? 0 : tile_bytes_of(g->patch, g->group, tp)) + 4 * P.nw);
  const bool fast = g->patch == 14 && g->group == 2 && (tp == 1 || tp == 2);
  const int grid = cs_num_sms() * (grouped ? 8 : (nv12 && fast) ? kNvCtas : 4);  // resident CTAs per SM
  const void* fn;
  int slot;
#define CS_PICK(TP, TG, LY, TT, SL) \
  do {                                                                                   \
    fn = reinterpret_cast<const void*>(compact_gather<TP, TG, LY, TT>);                  \
    slot = SL;                                                                           \
  } while (0)
  if (nv12) {
    if (fast) CS_PICK(14, 2, kLayoutNV12, 1, 15); else CS_PICK(0, 0, kLayoutNV12, 1, 16);
  } else if (grouped) {
    if (fast) {
      if (tp == 1) CS_PICK(14, 2, 1, 1, 12); else CS_PICK(14, 2, 1, 2, 17);
    } else {
      CS_PICK(0, 0, 1, 0, 14);
    }
  } else {
    if (fast) {
      if (tp == 1) CS_PICK(14, 2, 0, 1, 11); else CS_PICK(14, 2, 0, 2, 18);
    } else {
      CS_PICK(0, 0, 0, 0, 13);
    }
  }
#undef CS_PICK
  if (grouped && tp == 1 && fast && g->grid_w == 32 && g->grid_h % 2 == 0 && g->grid_h == 32 && P.vec_out) {
    {
      const int nst = 5;
      const size_t tsmem = (size_t)kTmaWarps * nst * kTmaStageAlloc;
      const void* tf = reinterpret_cast<const void*>(compact_gather_tma);
      if (cs_set_smem_attr(tf, 20, 200 * 1024)) return CS_ERR_CUDA;  // + 2.5 KB static <= 227 KB
      compact_gather_tma<<<cs_num_sms(), kGatherThreads, tsmem, stream>>>(P, nst);
      if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
      return CS_OK;
    }
  }
  if (cs_set_smem_attr(fn, slot, 227 * 1024)) return CS_ERR_CUDA;
  void* args[] = {&P};
  if (cudaLaunchKernel(fn, dim3(grid), dim3(kGatherThreads), args, smem, stream) != cudaSuccess) return CS_ERR_CUDA;
  if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
  return CS_OK;
}

int cs_launch_compact(const cs_grid* g, int32_t n_streams, int32_t n_frames, const uint32_t* keep_mask,
                      int64_t mask_frame_stride, const int32_t* frame_index, const void* const* frames,
                      int32_t frame_layout, int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                      int32_t* frame_offsets, unsigned long long* counters, int32_t* status, cudaStream_t stream) {
  return launch_compact(g, nullptr, 1, n_streams, n_frames, keep_mask, mask_frame_stride, frame_index, frames,
                        nullptr, frame_layout, capacity, packed, pos_ids, src_index, frame_offsets, nullptr, 0,
                        nullptr, nullptr, counters, status, stream);
}

int cs_launch_compact_tp(const cs_grid* g, int32_t tp, int32_t n_streams, int32_t n_units, const uint32_t* keep_mask,
                         int64_t mask_frame_stride, const int32_t* unit_index, const void* const* frames,
                         int32_t frame_layout, int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                         int32_t* frame_offsets, uint32_t* unit_mask, int64_t unit_mask_stride,
                         const uint8_t* frame_type, uint8_t* unit_type, unsigned long long* counters,
                         int32_t* status, cudaStream_t stream) {
  return launch_compact(g, nullptr, tp, n_streams, n_units, keep_mask, mask_frame_stride, unit_index, frames,
                        nullptr, frame_layout, capacity, packed, pos_ids, src_index, frame_offsets, unit_mask,
                        unit_mask_stride, frame_type, unit_type, counters, status, stream);
}

int cs_launch_compact_nv12(const cs_grid* g, const cs_preprocess* pp, int32_t n_streams, int32_t n_frames,
                           const uint32_t* keep_mask, int64_t mask_frame_stride, const int32_t* frame_index,
                           const void* const* y_planes, const void* const* uv_planes, int64_t capacity,
                           void* packed, int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets,
                           unsigned long long* counters, int32_t* status, cudaStream_t stream) {
  return launch_compact(g, pp, 1, n_streams, n_frames, keep_mask, mask_frame_stride, frame_index, y_planes,
                        uv_planes, kLayoutNV12, capacity, packed, pos_ids, src_index, frame_offsets, nullptr, 0,
                        nullptr, nullptr, counters, status, stream);
}
