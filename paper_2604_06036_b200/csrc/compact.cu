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
#include "group_ring.cuh"

#include <algorithm>
#include <atomic>
#include <memory>
#include <vector>

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
constexpr int kNvRows = CS_NV12_BATCH;   // output rows per warp iteration, loads all in flight (fused NV12 fast path)
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
  float one, negone;  // 1.0f / -1.0f: the uncontractable packed add / subtract (cs::add1 / cs::sub1)
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

// Source bytes of the fused NV12 preprocessing (algorithmic bytes, reading NEXT-2 bytes): per frame, the distinct
// 32-B sectors of the Y and UV planes holding a bilinear tap of a kept group's model pixel.  With pitches that are
// multiples of 32 a sector is (row, x / 32) in both planes (a chroma pair 2(x/2), 2(x/2)+1 shares luma x's sector).
// The taps of model row o depend only on o, so every source row r is touched by a contiguous range of group rows
// (its mask over gr), and every sector column by a range of group columns.  Rows with the same mask form a class
// (at most 2 per group row); the frame's sector count is sum over (row class, column class) of rows x columns x
// [some kept group lies in mask_r x mask_c].  The classes are geometry only (host, once per call).
struct NvClass {
  unsigned long long mask;  // group rows (row classes) / group columns (column classes)
  int n;                    // source rows / sector columns in the class
  int plane;                // row classes: 0 = Y, 1 = UV
};
constexpr int kNvMaxRowClasses = 256, kNvMaxColClasses = 128;
struct NvSrcClasses {
  int enabled, n_rows, n_cols;
  NvClass rows[kNvMaxRowClasses];
  NvClass cols[kNvMaxColClasses];
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
__global__ void __launch_bounds__(kCountThreads) compact_count(const __grid_constant__ CompactParams P,
                                                                const __grid_constant__ NvSrcClasses C) {
  __shared__ uint32_t s_m[kCountThreads / 32][128];  // per-warp unit mask (grid_words <= 128)
  __shared__ unsigned long long s_k[kCountThreads / 32][64];  // NV12 source count: kept group columns per group row
  __shared__ NvClass s_rc[kNvMaxRowClasses];  // the row / column classes, staged once per CTA: a lane-indexed
  __shared__ NvClass s_cc[kNvMaxColClasses];  // read of the parameter bank serialises its cache misses
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = blockIdx.x * (kCountThreads / 32) + warp;
  if (C.enabled) {
    // warp-uniform parameter reads (one address per warp instruction, the warps' misses in flight together)
    for (int i = warp; i < C.n_rows; i += kCountThreads / 32) {
      const NvClass v = C.rows[i];
      if (lane == 0) s_rc[i] = v;
    }
    for (int j = warp; j < C.n_cols; j += kCountThreads / 32) {
      const NvClass v = C.cols[j];
      if (lane == 0) s_cc[j] = v;
    }
    __syncthreads();
  }
  if (slot >= P.n_slots) return;
  if (C.enabled) {
    // the slot's keep mask in shared memory first (the group tests below would otherwise be dependent global loads)
    const uint32_t* mg = slot_mask(P, slot);
    for (int t = lane; t < P.nw; t += 32) s_m[warp][t] = __ldg(mg + t);
    __syncwarp();
    const uint32_t* m = s_m[warp];
    const int ngr = P.grid_h / P.G;
    if (P.G == 2 && P.grid_w == 32) {
      // kept group columns of group row gr: OR of patch rows 2gr, 2gr+1 (one word each), pairs folded onto even
      // bits, even bits compressed to 16
      for (int gr = lane; gr < ngr; gr += 32) {
        const uint32_t x = m[2 * gr] | m[2 * gr + 1];
        uint32_t y = (x | (x >> 1)) & 0x55555555u;
        y = (y | (y >> 1)) & 0x33333333u;
        y = (y | (y >> 2)) & 0x0F0F0F0Fu;
        y = (y | (y >> 4)) & 0x00FF00FFu;
        y = (y | (y >> 8)) & 0x0000FFFFu;
        s_k[warp][gr] = y;
      }
    } else {
      for (int gr = lane; gr < ngr; gr += 32) {
        unsigned long long k = 0ull;
        for (int gc = 0; gc < P.ngc; ++gc)
          if (cs::group_kept(m, gr * P.ngc + gc, P.ngc, P.G, P.grid_w)) k |= 1ull << gc;
        s_k[warp][gr] = k;
      }
    }
    __syncwarp();
    // lanes take row classes (i = lane + 32 t): K = the kept group columns of the class's group rows, then one
    // AND per column class (shared-memory broadcast reads); short per-lane chains, all lanes busy
    unsigned long long sectors = 0ull;
    for (int i = lane; i < C.n_rows; i += 32) {
      const NvClass rc = s_rc[i];
      unsigned long long K = 0ull;
      for (unsigned long long bm = rc.mask; bm; bm &= bm - 1) K |= s_k[warp][__ffsll(static_cast<long long>(bm)) - 1];
      unsigned long long cols = 0ull;
      for (int j = 0; j < C.n_cols; ++j) cols += (K & s_cc[j].mask) ? static_cast<unsigned long long>(s_cc[j].n) : 0ull;
      sectors += cols * static_cast<unsigned long long>(rc.n);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sectors += __shfl_xor_sync(0xffffffffu, sectors, d);
    if (lane == 0 && sectors) cs::atomic_add_u64(&P.counters[CS_CNT_BYTES_COMPACT], sectors * 32ull);
  }
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

// One pair of output rows (yy0, yy0 + 1) of a kept group, fused NV12 preprocessing, lanes on output columns: the
// 4 luma taps yv and 4 chroma pairs uvv of both rows (loaded by the caller from global or shared memory) -> the
// normalised fp32 model pixels of the lane's column (on[c] = (row yy0, row yy0 + 1) of channel c, before the bf16
// rounding).  The two output rows are the two halves of packed fp32 pairs (FADD2 / FMUL2 / FFMA2: one issue per
// pair, each half the same IEEE operation as the oracle's); a sum of products is an FFMA2 with a runtime 1.0
// (cs::add1: ptxas would contract a plain packed add into the product, cs_internal.cuh).  Bytes become floats
// exactly: float(2^23 + b) - (2^23 + 16) = b - 16 (PRMT + FADD).
__device__ __forceinline__ void nv12_pair_an(const CompactParams& P, const uint32_t (&yv)[2][4],
                                             const uint32_t (&uvv)[2][4], const float (&lyv)[2], float lx, float hx,
                                             float2 (&an)[3]) {
  const float kY = 1.164383f, kRV = 1.596027f, kGU = 0.391762f, kGV = 0.812968f, kBU = 2.017232f;
  constexpr float kBiasY = 8388624.0f, kBiasC = 8388736.0f;  // 2^23 + 16, 2^23 + 128
  const float2 kY2 = make_float2(kY, kY), kRV2 = make_float2(kRV, kRV), kGU2 = make_float2(kGU, kGU);
  const float2 kGV2 = make_float2(kGV, kGV), kBU2 = make_float2(kBU, kBU);
  const float2 bY = make_float2(kBiasY, kBiasY), bC = make_float2(kBiasC, kBiasC);
  auto bytes2 = [](uint32_t v0, uint32_t v1, uint32_t sel) {
    return make_float2(__uint_as_float(__byte_perm(v0, 0x4B000000u, sel)),
                       __uint_as_float(__byte_perm(v1, 0x4B000000u, sel)));
  };
  // sums / differences of products: FFMA2 with the runtime 1.0 (cs::add1 / cs::sub1, never contracted)
  const float2 one = make_float2(P.one, P.one), neg = make_float2(P.negone, P.negone);
  float2 rgb[4][3];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 d = cs::sub2(bytes2(uvv[0][q], uvv[1][q], 0x7540u), bC);
    const float2 e = cs::sub2(bytes2(uvv[0][q], uvv[1][q], 0x7541u), bC);
    const float2 yk = cs::mul2(kY2, cs::sub2(bytes2(yv[0][q], yv[1][q], 0x7540u), bY));
    // the sums are never NaN or -0.0 (integer-valued c, d, e; x + (-x) = +0 in RN): the one-instruction clamp
    rgb[q][0] = cs::clamp255_relu2(cs::add1(yk, cs::mul2(kRV2, e), one));
    rgb[q][1] = cs::clamp255_relu2(cs::sub1(cs::sub1(yk, cs::mul2(kGU2, d), neg), cs::mul2(kGV2, e), neg));
    rgb[q][2] = cs::clamp255_relu2(cs::add1(yk, cs::mul2(kBU2, d), one));
  }
  const float2 lx2 = make_float2(lx, lx), hx2 = make_float2(hx, hx);
  const float2 ly2 = make_float2(lyv[0], lyv[1]);
  const float2 hy2 = cs::sub2(make_float2(1.0f, 1.0f), ly2);
  const float2 inv255 = make_float2(kInv255, kInv255), n255 = make_float2(255.0f, 255.0f);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float2 top = cs::add1(cs::mul2(hx2, rgb[0][c]), cs::mul2(lx2, rgb[1][c]), one);
    const float2 bot = cs::add1(cs::mul2(hx2, rgb[2][c]), cs::mul2(lx2, rgb[3][c]), one);
    const float2 v = cs::add1(cs::mul2(hy2, top), cs::mul2(ly2, bot), one);
    // v / 255 correctly rounded without a division: q = v * RN(1/255), one fma residual correction.
    // Exhaustively verified equal to IEEE v / 255 for every fp32 v in [0, 512] (scripts/check_div255.c)
    const float2 q255 = cs::mul2(v, inv255);
    const float2 res = cs::fma2(make_float2(-q255.x, -q255.y), n255, v);
    const float2 t = cs::fma2(res, inv255, q255);
    an[c] = cs::sub2(t, make_float2(P.mean[c], P.mean[c]));
  }
}

// (t - mean) / std -> bf16 (norm_bf16) for a pair's six values through the guarded reciprocal: on = an * RN(1/std);
// returns nonzero when any product lies within 8 fp32 steps of a bf16 rounding midpoint (or fast_div is off), in
// which case the caller takes nv12_norm_exact for it (one branch for any number of pairs).
__device__ __forceinline__ uint32_t nv12_norm_fast(const CompactParams& P, const float2 (&an)[3], float2 (&on)[3]) {
  uint32_t near_mid = P.fast_div ? 0u : 1u;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    on[c] = cs::mul2(an[c], make_float2(P.rstd[c], P.rstd[c]));
    near_mid |= static_cast<uint32_t>((__float_as_uint(on[c].x) & 0xffffu) - 0x7ff8u <= 16u);
    near_mid |= static_cast<uint32_t>((__float_as_uint(on[c].y) & 0xffffu) - 0x7ff8u <= 16u);
  }
  return near_mid;
}
__device__ __forceinline__ void nv12_norm_exact(const CompactParams& P, const float2 (&an)[3], float2 (&on)[3]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) on[c] = make_float2(__fdiv_rn(an[c].x, P.stdv[c]), __fdiv_rn(an[c].y, P.stdv[c]));
}
__device__ __forceinline__ void nv12_pair_px(const CompactParams& P, const uint32_t (&yv)[2][4],
                                             const uint32_t (&uvv)[2][4], const float (&lyv)[2], float lx, float hx,
                                             float2 (&on)[3]) {
  float2 an[3];
  nv12_pair_an(P, yv, uvv, lyv, lx, hx, an);
  if (nv12_norm_fast(P, an, on)) nv12_norm_exact(P, an, on);
}

// nv12_pair_px, then the bf16 pixels into the warp's group tile (tcol = the lane column's tile base)
__device__ __forceinline__ void nv12_pair(const CompactParams& P, const uint32_t (&yv)[2][4], const uint32_t (&uvv)[2][4],
                                          const float (&lyv)[2], float lx, float hx, uint16_t* tcol, int yy0,
                                          bool store) {
  constexpr int p = 14, pp = 196, G = 2, kNvRows = 2;
  float2 on[3];
  nv12_pair_px(P, yv, uvv, lyv, lx, hx, on);
  if (store) {
#pragma unroll
    for (int r = 0; r < kNvRows; ++r) {
      const int yy = yy0 + r, dyp = yy >= p ? 1 : 0;
      uint16_t* tq = tcol + dyp * G * 3 * pp + (yy - dyp * p) * p;
#pragma unroll
      for (int c = 0; c < 3; ++c) tq[c * pp] = cs::f32_to_bf16_cvt(r == 0 ? on[c].x : on[c].y);
    }
  }
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
    if (TP > 0 && TG == 2 && gp <= 32 && gp % kNvRows == 0) {
      // fast path (issue-bound: every instruction per pixel counts).  Lanes run along the group's output columns
      // (lane xx < gp = 28; lanes 28..31 duplicate the last column and store nothing) and every iteration handles
      // kNvRows output rows: a column's source taps, weights and chroma offsets are per-lane constants, a row's
      // are warp-uniform (computed once per row by the whole warp), so a pixel costs no index arithmetic beyond
      // its eight loads.  Bytes become floats exactly with the 2^23 trick: float(2^23 + b) - (2^23 + 16) = b - 16
      // (one PRMT + one FADD instead of integer subtract + I2F); when both tap rows of an output row fall in the
      // same chroma row (uniform), the two lower taps reuse the upper taps' chroma terms.  Same fp32 operations
      // in the same order as the oracle; the bf16 store is the hardware RNE conversion (outputs are never NaN:
      // std > 0 and mean not NaN are checked on the host).
      const int xx = lane < gp ? lane : gp - 1;
      int x0, x1;
      float lx;
      nv12_axis(gc * gp + xx, P.src_w, P.scale_x, x0, x1, lx);
      const float hx = __fsub_rn(1.0f, lx);
      const uint8_t* yc0 = Yp + x0;
      const uint8_t* yc1 = Yp + x1;
      const uint8_t* cc0 = UVp + 2 * (x0 >> 1);
      const uint8_t* cc1 = UVp + 2 * (x1 >> 1);
      const int dxp = xx >= p ? 1 : 0;
      uint16_t* tcol = tile + dxp * 3 * pp + (xx - dxp * p);
      const bool store = lane < gp;
      static_assert(kNvRows == 2, "nv12_pair: pairs of output rows");
      // per pair of output rows: its 16 loads are all issued before any is consumed (software-pipelining the next
      // pair's loads, or prefetching a group's source band into L2, measured slower: DESIGN §6)
      for (int yy0 = 0; yy0 < gp; yy0 += kNvRows) {
        uint32_t yv[kNvRows][4], uvv[kNvRows][4];
        float lyv[kNvRows];
        bool cshare[kNvRows];
#pragma unroll
        for (int r = 0; r < kNvRows; ++r) {
          int y0, y1;
          nv12_axis(gr * gp + yy0 + r, P.src_h, P.scale_y, y0, y1, lyv[r]);
          const long long o0 = (long long)y0 * P.y_pitch, o1 = (long long)y1 * P.y_pitch;
          const long long c0 = (long long)(y0 >> 1) * P.uv_pitch, c1 = (long long)(y1 >> 1) * P.uv_pitch;
          cshare[r] = (y0 >> 1) == (y1 >> 1);
          yv[r][0] = __ldg(yc0 + o0);
          yv[r][1] = __ldg(yc1 + o0);
          yv[r][2] = __ldg(yc0 + o1);
          yv[r][3] = __ldg(yc1 + o1);
          uvv[r][0] = __ldg(reinterpret_cast<const uint16_t*>(cc0 + c0));
          uvv[r][1] = __ldg(reinterpret_cast<const uint16_t*>(cc1 + c0));
          if (!cshare[r]) {
            uvv[r][2] = __ldg(reinterpret_cast<const uint16_t*>(cc0 + c1));
            uvv[r][3] = __ldg(reinterpret_cast<const uint16_t*>(cc1 + c1));
          } else {
            uvv[r][2] = uvv[r][0];
            uvv[r][3] = uvv[r][1];
          }
        }
        nv12_pair(P, yv, uvv, lyv, lx, hx, tcol, yy0, store);
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

// ---- planar CHW frames, 2x2 groups of 14-px patches on a 32 x 32 grid: band-staged gather --------------------
// A kept group of a planar frame is 84 row segments of 56 B (3 channels x 28 rows) at 8-B alignment.  Fetched one
// group at a time, every segment drags in the rest of its 128-B lines, which are only useful if the neighbouring
// group is kept AND still cached when its turn comes (measured round 1: DRAM reads 3.2x the algorithmic bytes,
// 0.41 of the roofline).  Here a warp takes RUNS of up to kBandRun consecutive kept groups of one group row (the
// packed order puts them in consecutive rows) and stages the run's band -- for each of the 84 source rows the one
// contiguous span covering all of the run's groups, widened to 16-B alignment -- into a stage of its ring with 16-B
// asynchronous copies (cp.async, commit / wait groups), so each source line is requested once, by one warp, while
// the next run's copies are in flight.  (1-D bulk copies, one per row span, were measured 2-4 % slower: 84
// requests per run keep the TMA unit busy.)  The warp then writes each group's 4,704 output bytes with 16-B stores,
// every 16-B chunk assembled from four 4-B pixel pairs of the staged rows (a pair never straddles a 14-px patch
// row) through a per-CTA table of staged-row offsets.
#ifndef CS_BAND_RUN
#define CS_BAND_RUN 3
#define CS_BAND_WARPS 7
#define CS_BAND_STAGES 2
#endif
constexpr int kBandRun = CS_BAND_RUN;                                 // groups per run
constexpr int kBandRowBytes = ((8 + 56 * kBandRun) + 15) & ~15;      // staged row pitch (3 groups: 176 B)
constexpr int kBandStage = 84 * kBandRowBytes;                        // 3 channels x 28 rows
constexpr int kBandWarps = CS_BAND_WARPS;                             // 7 x 2 stages x 14.8 KB: one CTA per SM
constexpr int kBandMaxStages = CS_BAND_STAGES;
static_assert(kBandWarps * kBandMaxStages * kBandStage <= 220 * 1024, "band stages exceed shared memory");

struct BandRun {
  long long n0;          // first packed row of the run
  const uint16_t* row0;  // frame element of (c = 0, y = 28 gr, x = 28 gc_a), i.e. the run's first source pixel
  int slot, gr, gc, k;   // frame slot, group row, first group column, groups in the run (0: end of work)
  int t_index, lead;     // pos id t; bytes between the 16-B aligned copy start and the run's first pixel
};

__global__ void __launch_bounds__(kBandWarps * 32, 1) compact_gather_band(const __grid_constant__ CompactParams P,
                                                                          int nst) {
  extern __shared__ __align__(128) unsigned char b_smem[];
  __shared__ BandRun s_run[kBandWarps][kBandMaxStages];
  __shared__ uint4 s_tab[294];  // per 16-B output chunk of a group: 4 pixel pairs -> (staged row, byte) as u16 pairs
  __shared__ __align__(16) uint32_t s_mask[kBandWarps][32];  // the current slot's keep mask (lane 0's generator)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  constexpr int p = 14, pp = 196, row_el = 588;
  constexpr long long FW = 448, plane = 448ll * 448;
  // table: element i = 8 e + 2 t of a group -> patch q, channel c, (py, px) -> staged row c*28 + dy*14 + py and the
  // byte offset 2 (dx*14 + px) within the group's 56 bytes (the run offset j*56 + lead is added per group)
  for (int e = threadIdx.x; e < 294; e += blockDim.x) {
    uint32_t w[4];
    for (int t = 0; t < 4; ++t) {
      const int i = 8 * e + 2 * t, q = i / row_el, r = i - q * row_el, c = r / pp, r2 = r - c * pp;
      const int py = r2 / p, px = r2 - py * p, dy = q >> 1, dx = q & 1;
      w[t] = static_cast<uint32_t>((c * 28 + dy * 14 + py) * kBandRowBytes) | (static_cast<uint32_t>(2 * (dx * 14 + px)) << 16);
    }
    s_tab[e] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  __syncthreads();
  const long long total_groups = static_cast<long long>(__ldg(P.frame_offsets + P.n_slots)) / 4;
  const long long nwarps = static_cast<long long>(gridDim.x) * kBandWarps;
  const long long wid = static_cast<long long>(blockIdx.x) * kBandWarps + wib;
  long long q = total_groups * wid / nwarps;
  const long long q1 = total_groups * (wid + 1) / nwarps;
  if (q >= q1) return;
  unsigned char* stages = b_smem + (size_t)wib * nst * kBandStage;
  BandRun* runs = s_run[wib];

  // ---- generator (lane 0): slot, group row, remaining kept-group bits of the row -------------------------------
  int slot = 0, gr = 0, t_index = 0;
  uint32_t ybits = 0u;
  const uint16_t* frame = nullptr;
  // the slot's 32 mask words are copied to shared memory once per slot (8 x 16-B loads), so walking its group rows
  // costs no global-memory latency on the ring's critical path
  uint32_t* smask = s_mask[wib];
  auto load_row = [&]() {
    const uint32_t x = smask[2 * gr] | smask[2 * gr + 1];
    ybits = (x | (x >> 1)) & 0x55555555u;  // bit 2*gc set iff group (gr, gc) is kept
  };
  auto load_slot = [&]() {
    frame = static_cast<const uint16_t*>(P.frames[slot]);
    t_index = __ldg(P.frame_index + slot);
    const uint4* m4 = reinterpret_cast<const uint4*>(slot_mask(P, slot));
    uint4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldg(m4 + i);
#pragma unroll
    for (int i = 0; i < 8; ++i) reinterpret_cast<uint4*>(smask)[i] = v[i];
  };
  if (lane == 0) {
    int lo = 0, hi = P.n_slots;
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
      ++gr;
      load_row();
    }
    for (; skip > 0; --skip) ybits &= ybits - 1u;
  }
  __syncwarp();
  bool more = true;  // (lane 0)
  // next run into stage st: lane 0 forms it and arms the barrier, then the lanes issue the 84 row copies
  auto issue = [&](int st) {
    BandRun r;
    uint32_t bytes = 0;
    if (lane == 0) {
      if (q >= q1) {
        r.k = 0;
        more = false;
      } else {
        while (ybits == 0u) {
          if (++gr == 16) {
            gr = 0;
            ++slot;
            load_slot();
          }
          load_row();
        }
        const int gc = (__ffs(ybits) - 1) >> 1;
        int k = 0;  // consecutive kept groups gc, gc+1, ... of this row, within the warp's range and the run cap
        while (k < kBandRun && q + k < q1 && gc + k < 16 && ((ybits >> (2 * (gc + k))) & 1u)) ++k;
        ybits &= ~((1u << (2 * (gc + k))) - 1u);
        r.n0 = q * 4;
        r.slot = slot;
        r.gr = gr;
        r.gc = gc;
        r.k = k;
        r.t_index = t_index;
        r.row0 = frame + (long long)(gr * 28) * FW + gc * 28;
        const uintptr_t a = reinterpret_cast<uintptr_t>(r.row0);
        r.lead = static_cast<int>(a & 15u);
        bytes = static_cast<uint32_t>(((r.lead + k * 56) + 15) & ~15);  // per row, 16-B multiple
        q += k;
        runs[st] = r;
      }
      if (r.k == 0) runs[st].k = 0;
    }
    __syncwarp();
    bytes = __shfl_sync(0xffffffffu, bytes, 0);
    if (bytes) {  // the 84 row spans as 16-B asynchronous copies spread over the lanes
      const BandRun rr = runs[st];
      const unsigned char* base = reinterpret_cast<const unsigned char*>(rr.row0) - rr.lead;
      const int nch = static_cast<int>(bytes >> 4);
      unsigned char* sb = stages + (size_t)st * kBandStage;
      for (int e = lane; e < 84 * nch; e += 32) {
        const int row = e / nch, ch = e - row * nch;
        const int c = row / 28, y = row - c * 28;
        cs::cp_async16(sb + row * kBandRowBytes + ch * 16, base + (c * plane + (long long)y * FW) * 2 + ch * 16);
      }
    }
    cs::cp_async_commit();  // one (possibly empty) group per issued item keeps the wait count uniform
  };
  for (int st = 0; st < nst; ++st) {
    const bool m = __shfl_sync(0xffffffffu, more ? 1 : 0, 0);
    if (!m) break;
    issue(st);
  }
  for (int it = 0;; ++it) {
    const int st = it % nst;
    cs::cp_async_wait<kBandMaxStages - 1>();  // this lane's copies of item `it` have landed (nst == kBandMaxStages)
    __syncwarp();                             // ... and every lane's
    const BandRun r = runs[st];
    if (r.k == 0) break;
    const unsigned char* stg = stages + (size_t)st * kBandStage;
    for (int j = 0; j < r.k; ++j) {
      const long long n0 = r.n0 + 4 * j;
      long long nvalid = P.capacity - n0;
      nvalid = nvalid < 0 ? 0 : (nvalid > 4 ? 4 : nvalid);
      if (nvalid > 0) {
        const unsigned char* g0 = stg + r.lead + j * 56;
        uint16_t* dst = P.packed + n0 * row_el;
        if (nvalid == 4) {
          uint4* d4 = reinterpret_cast<uint4*>(dst);
          for (int e = lane; e < 294; e += 32) {
            const uint4 t = s_tab[e];
            uint4 v;
            v.x = *reinterpret_cast<const uint32_t*>(g0 + (t.x & 0xffffu) + (t.x >> 16));
            v.y = *reinterpret_cast<const uint32_t*>(g0 + (t.y & 0xffffu) + (t.y >> 16));
            v.z = *reinterpret_cast<const uint32_t*>(g0 + (t.z & 0xffffu) + (t.z >> 16));
            v.w = *reinterpret_cast<const uint32_t*>(g0 + (t.w & 0xffffu) + (t.w >> 16));
            d4[e] = v;
          }
        } else {  // capacity-truncated group: element stores of its first nvalid rows
          for (int i = lane; i < nvalid * row_el; i += 32) {
            const int qq = i / row_el, rr = i - qq * row_el, c = rr / pp, r2 = rr - c * pp;
            const int py = r2 / p, px = r2 - py * p;
            dst[i] = *reinterpret_cast<const uint16_t*>(g0 + (c * 28 + (qq >> 1) * 14 + py) * kBandRowBytes +
                                                        2 * ((qq & 1) * 14 + px));
          }
        }
        if (lane < nvalid) {
          const int h = r.gr * 2 + (lane >> 1), w = (r.gc + j) * 2 + (lane & 1);
          const long long n = n0 + lane;
          P.pos_ids[3 * n + 0] = r.t_index;
          P.pos_ids[3 * n + 1] = h;
          P.pos_ids[3 * n + 2] = w;
          P.src_index[n] = r.slot * 1024 + h * 32 + w;
        }
      }
    }
    __syncwarp();  // the stage is consumed (generic-proxy reads) before it is refilled by the async proxy
    const bool m = __shfl_sync(0xffffffffu, more ? 1 : 0, 0);
    if (m) issue(st);
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
constexpr unsigned kTmaStageAlloc = cs::kRingStageAlloc;

__global__ void __launch_bounds__(kGatherThreads, 1) compact_gather_tma(const __grid_constant__ CompactParams P,
                                                                        int nst) {
  extern __shared__ __align__(128) unsigned char t_smem[];
  __shared__ cs::RingGroup s_desc[kTmaWarps][kTmaMaxStages];
  __shared__ __align__(8) uint64_t s_full[kTmaWarps][kTmaMaxStages];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long total_groups = static_cast<long long>(__ldg(P.frame_offsets + P.n_slots)) / 4;
  const long long nwarps = static_cast<long long>(gridDim.x) * kTmaWarps;
  const long long wid = static_cast<long long>(blockIdx.x) * kTmaWarps + wib;
  cs::RingBatch B;
  B.frame_offsets = P.frame_offsets;
  B.n_slots = P.n_slots;
  B.n_frames = P.n_frames;
  B.keep_mask = P.keep_mask;
  B.mask_frame_stride = P.mask_frame_stride;
  B.frames = P.frames;
  B.frame_index = P.frame_index;
  B.capacity = P.capacity;
  B.packed = P.packed;
  B.pos_ids = P.pos_ids;
  B.src_index = P.src_index;
  __shared__ __align__(16) uint32_t s_mask[kTmaWarps][32];
  cs::group_ring(B, total_groups * wid / nwarps, total_groups * (wid + 1) / nwarps,
                 t_smem + (size_t)wib * nst * kTmaStageAlloc, nst, s_full[wib], s_desc[wib], s_mask[wib], lane);
}

// ---- fused NV12 preprocessing, source rows staged in shared memory (NEXT-2; 2x2 groups of 14-px patches) -------
// The work of a warp is a flat sequence of ITEMS -- one pair of output rows of one kept group, 14 per group, the
// warp's kept groups in packed order -- taken two at a time: pair j of a group = items j and j + 7, i.e. rows
// (2j, 2j + 1) of patch rows dy = 0 and 1, so the pair's 12 bf16 stores are immediates off one per-lane base.  An
// item reads 8 source rows: the luma tap rows y0(r), y1(r) of its two output rows r and their chroma rows, each over
// the group's column span [xs, xs + 16 nch) (xs = the group's first luma tap rounded down to 16 B; nch chunks cover
// the last column's luma and chroma taps).  PRODUCER: lane l copies staged row l/4 of each item, chunks (l%4) + 4m,
// with predicated 16-B cp.async into a stage of the warp's ring, kNvsStages - 1 pairs ahead of the compute, across
// group boundaries (the next group comes from the warp's kept-group enumeration when the producer reaches it; its
// descriptor is published in shared memory).  CONSUMER: lanes on the group's 28 output columns (nv12_pair_an, as
// the direct-load path), every tap one shared-memory load at a per-lane constant offset, no 64-bit index arithmetic;
// one midpoint-guard branch per pair; predicated 2-B stores straight to the packed rows (a pair covers 56 contiguous
// bytes per channel and patch row, so sectors fill in L2).  Row taps / weights come from per-CTA tables (one
// nv12_axis per model row per launch).  16 warps x ~107 registers, one CTA per SM (measured against 8-24 warps and a
// 64-register budget, which rematerialised the lane constants every pair).  Requires pitches that are
// multiples of 16; a slot whose planes are not 16-B aligned is staged with byte copies.
constexpr int kNvsWarps = 16;
constexpr int kNvsStages = 3;  // ring stages per warp (kNvsStages - 1 pairs in flight)
constexpr int kNvsPairs = 7;   // item pairs (4 output rows) per 28-row group; a ring stage holds one pair

struct NvsGroup {  // a kept group of the warp's range (warp-uniform)
  long long n0;    // first packed row
  const uint8_t* Y;
  const uint8_t* UV;
  int slot, gr, gc;
};

template <int RB>  // staged row pitch in bytes (16 * max chunks: 144 covers scale_x <= 4.6, 256 up to 8.6)
__global__ void __launch_bounds__(kNvsWarps * 32, 1) compact_nv12_staged(const __grid_constant__ CompactParams P) {
  constexpr int p = 14, gp = 28, row_el = 588, kItem = 8 * RB, kStage = 2 * kItem;
  extern __shared__ __align__(128) unsigned char n_smem[];
  __shared__ __align__(16) uint32_t s_mask[kNvsWarps][64];
  __shared__ NvsGroup s_grp[kNvsWarps][2];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* stages = n_smem + (size_t)wib * kNvsStages * kStage;
  // per model row o: luma tap rows y0 | y1 << 16, chroma rows (y0 / 2) | (y1 / 2) << 16, the weight ly
  uint32_t* s_y01 = reinterpret_cast<uint32_t*>(n_smem + (size_t)kNvsWarps * kNvsStages * kStage);
  uint32_t* s_c01 = s_y01 + P.FH;
  float* s_ly = reinterpret_cast<float*>(s_c01 + P.FH);
  for (int o = threadIdx.x; o < P.FH; o += blockDim.x) {
    int y0, y1;
    float ly;
    nv12_axis(o, P.src_h, P.scale_y, y0, y1, ly);
    s_y01[o] = static_cast<uint32_t>(y0) | (static_cast<uint32_t>(y1) << 16);
    s_c01[o] = static_cast<uint32_t>(y0 >> 1) | (static_cast<uint32_t>(y1 >> 1) << 16);
    s_ly[o] = ly;
  }
  __syncthreads();

  const long long total_groups = static_cast<long long>(__ldg(P.frame_offsets + P.n_slots)) / 4;
  const long long nwarps = static_cast<long long>(gridDim.x) * kNvsWarps;
  const long long wid = static_cast<long long>(blockIdx.x) * kNvsWarps + wib;
  long long q = total_groups * wid / nwarps;
  const long long q1 = total_groups * (wid + 1) / nwarps;
  if (q >= q1) return;
  uint32_t* mask = s_mask[wib];

  // ---- the warp's kept-group enumeration (producer side): slot, 32-group chunk `base`, its remaining ballot bits
  int g_slot, g_base = 0;
  uint32_t g_bal = 0u;
  auto load_mask = [&](int slot) {
    __syncwarp();
    for (int t = lane; t < P.nw; t += 32) mask[t] = __ldg(slot_mask(P, slot) + t);
    __syncwarp();
  };
  auto ballot_chunk = [&]() {
    const int qq = g_base + lane;
    const bool kept = qq < P.ngroups && cs::group_kept(mask, qq, P.ngc, 2, P.grid_w);
    g_bal = __ballot_sync(0xffffffffu, kept);
  };
  {
    int lo = 0, hi = P.n_slots;  // largest slot with frame_offsets[slot] <= q * 4
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (static_cast<long long>(__ldg(P.frame_offsets + mid)) <= q * 4) lo = mid; else hi = mid;
    }
    g_slot = lo;
    long long skip = q - __ldg(P.frame_offsets + g_slot) / 4;  // kept groups of the slot before q
    load_mask(g_slot);
    ballot_chunk();
    while (skip >= __popc(g_bal)) {  // the slot holds more than `skip` kept groups
      skip -= __popc(g_bal);
      g_base += 32;
      ballot_chunk();
    }
    for (; skip > 0; --skip) g_bal &= g_bal - 1u;
  }
  auto next_group = [&]() -> NvsGroup {
    while (g_bal == 0u) {
      g_base += 32;
      if (g_base >= P.ngroups) {
        g_base = 0;
        ++g_slot;
        load_mask(g_slot);
      }
      ballot_chunk();
    }
    const int gi = g_base + __ffs(g_bal) - 1;
    g_bal &= g_bal - 1u;
    NvsGroup d;
    d.n0 = q * 4;
    ++q;
    d.slot = g_slot;
    d.gr = gi / P.ngc;
    d.gc = gi - d.gr * P.ngc;
    d.Y = static_cast<const uint8_t*>(P.frames[g_slot]);
    d.UV = static_cast<const uint8_t*>(P.uv_planes[g_slot]);
    return d;
  };
  // the group's column span start (16-B aligned), identical on the producer and consumer sides
  auto span_start = [&](int gc) {
    int x0, x1;
    float lx;
    nv12_axis(gc * gp, P.src_w, P.scale_x, x0, x1, lx);
    return x0 & ~15;
  };

  // ---- producer (lane: staged row k = lane / 4 of each item, chunks cl + 4m; rows 0-3 luma, 4-7 chroma)
  const int k = lane >> 2, cl = lane & 3;
  const uint32_t p_pitch = static_cast<uint32_t>(k < 4 ? P.y_pitch : P.uv_pitch);
  const uint32_t p_sel = (k & 1) ? 0x4432u : 0x4410u;  // PRMT: the y1 / y0 half of a row-table entry
  const uint32_t p_dst = cs::smem_u32(stages) + k * RB + 16 * cl;
  const uint8_t* p_src = nullptr;  // this lane's first chunk in source row 0 of its plane
  const uint32_t* p_tab = nullptr; // the lane's row-table entry of item 0 of the producer's group
  int p_nch = 0;                   // 16-B chunks of the group's span
  bool p_aligned = true;
  auto produce_group = [&](const NvsGroup& d) {
    int x0, x1, xa, xb;
    float l;
    nv12_axis(d.gc * gp, P.src_w, P.scale_x, x0, x1, l);
    nv12_axis(d.gc * gp + gp - 1, P.src_w, P.scale_x, xa, xb, l);
    const int xs = x0 & ~15;
    p_nch = ((2 * (xb >> 1) + 1 - xs) >> 4) + 1;  // the host sized RB for the widest group (<= RB / 16)
    p_src = (k < 4 ? d.Y : d.UV) + xs + 16 * cl;
    p_tab = (k < 4 ? s_y01 : s_c01) + d.gr * gp + ((k >> 1) & 1);
    p_aligned = ((reinterpret_cast<uintptr_t>(d.Y) | reinterpret_cast<uintptr_t>(d.UV)) & 15u) == 0;
  };
  // items j and j + 7 (patch rows dy = 0 and 1) of the producer's group into the stage at byte offset soff of the
  // warp's ring
  auto produce_pair = [&](int j, uint32_t soff) {
    uint32_t y[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) y[h] = __byte_perm(p_tab[2 * j + 14 * h], 0u, p_sel);
    if (p_aligned) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint8_t* src = p_src + y[h] * p_pitch;
        const uint32_t dst = p_dst + soff + h * kItem;
#pragma unroll
        for (int m = 0; m < RB / 64 + 1; ++m) cs::cp_async16_if(dst + 64 * m, src + 64 * m, cl + 4 * m < p_nch);
      }
    } else {
      for (int h = 0; h < 2; ++h) {
        const uint8_t* src = p_src + y[h] * p_pitch;
        unsigned char* d8 = stages + (p_dst - cs::smem_u32(stages)) + soff + h * kItem;
        for (int m = 0; m < RB / 64 + 1; ++m)
          if (cl + 4 * m < p_nch)
            for (int b = 0; b < 16; ++b) d8[64 * m + b] = __ldg(src + 64 * m + b);
      }
    }
  };

  // ---- producer sequence: pair pj of the producer's current group into ring stage ps; a new group is fetched
  // (and its descriptor published in s_grp[wib][pg & 1]) when pj wraps.  The producer runs kNvsStages - 1 pairs
  // ahead of the consumer, i.e. at most one group ahead.
  long long p_left = q1 - q;  // groups the producer has yet to fetch
  int pj = 0, ps = 0, pg = 0;
  auto produce_next = [&]() {
    if (pj == 0) {
      if (p_left == 0) return;
      --p_left;
      const NvsGroup d = next_group();
      if (lane == 0) s_grp[wib][pg & 1] = d;
      ++pg;
      produce_group(d);
    }
    produce_pair(pj, static_cast<uint32_t>(ps * kStage));
    pj = pj == kNvsPairs - 1 ? 0 : pj + 1;
    ps = ps == kNvsStages - 1 ? 0 : ps + 1;
  };

  // ---- consumer (lane: output column xx of the group)
  const int xx = lane < gp ? lane : gp - 1;
  const int dx = xx >= p ? 1 : 0, xin = xx - dx * p;
  const long long n_groups = q1 - q;
  for (int u = 0; u < kNvsStages - 1; ++u) {
    produce_next();
    cs::cp_async_commit();  // one (possibly empty) group per pair keeps the wait count uniform
  }
  int cs_ = 0;  // ring stage of the pair being computed
  for (long long g = 0; g < n_groups; ++g) {
    __syncwarp();  // the group's descriptor (published at least one pair ago) is visible
    const NvsGroup& dg = s_grp[wib][g & 1];
    const long long n0 = dg.n0;
    const int slot = dg.slot, gr = dg.gr, gc = dg.gc;
    int x0, x1;
    float lx;
    nv12_axis(gc * gp + xx, P.src_w, P.scale_x, x0, x1, lx);
    const float hx = __fsub_rn(1.0f, lx);
    const int xs = span_start(gc);
    const int ox0 = x0 - xs, ox1 = x1 - xs, cx0 = 2 * (x0 >> 1) - xs, cx1 = 2 * (x1 >> 1) - xs;
    uint16_t* out = P.packed + (n0 + dx) * row_el + xin;  // this lane's column, patch row dy = 0
    const bool st[2] = {lane < gp && n0 + dx < P.capacity, lane < gp && n0 + 2 + dx < P.capacity};
    const float* lyp = s_ly + gr * gp;
#pragma unroll 1
    for (int j = 0; j < kNvsPairs; ++j) {
      cs::cp_async_wait<kNvsStages - 2>();  // this lane's copies of pair j have landed
      __syncwarp();  // ... and every lane's; every lane is done with the stage the next copies go to (pair j - 1's)
      produce_next();
      cs::cp_async_commit();
      const uint32_t J = static_cast<uint32_t>(cs_ * kStage);
      cs_ = cs_ == kNvsStages - 1 ? 0 : cs_ + 1;
      const unsigned char* sb = stages + J;
      float2 an[2][3], on[2][3];
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // item j + 7h: output rows 2j, 2j + 1 of patch row dy = h
        const unsigned char* ib = sb + h * kItem;
        uint32_t yv[2][4], uvv[2][4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const unsigned char* ry0 = ib + (2 * r) * RB;
          const unsigned char* ry1 = ib + (2 * r + 1) * RB;
          const unsigned char* rc0 = ib + (4 + 2 * r) * RB;
          const unsigned char* rc1 = ib + (5 + 2 * r) * RB;
          yv[r][0] = ry0[ox0];
          yv[r][1] = ry0[ox1];
          yv[r][2] = ry1[ox0];
          yv[r][3] = ry1[ox1];
          uvv[r][0] = *reinterpret_cast<const uint16_t*>(rc0 + cx0);
          uvv[r][1] = *reinterpret_cast<const uint16_t*>(rc0 + cx1);
          uvv[r][2] = *reinterpret_cast<const uint16_t*>(rc1 + cx0);
          uvv[r][3] = *reinterpret_cast<const uint16_t*>(rc1 + cx1);
        }
        const float2 ly = *reinterpret_cast<const float2*>(lyp + 2 * j + 14 * h);
        const float lyv[2] = {ly.x, ly.y};
        nv12_pair_an(P, yv, uvv, lyv, lx, hx, an[h]);
      }
      if (nv12_norm_fast(P, an[0], on[0]) | nv12_norm_fast(P, an[1], on[1])) {
        nv12_norm_exact(P, an[0], on[0]);
        nv12_norm_exact(P, an[1], on[1]);
      }
      uint16_t* o = out + 28 * j;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          cs::st_b16_if(o + h * 2 * row_el + c * p * p, cs::f32_to_bf16_cvt(on[h][c].x), st[h]);
          cs::st_b16_if(o + h * 2 * row_el + c * p * p + p, cs::f32_to_bf16_cvt(on[h][c].y), st[h]);
        }
    }
    if (lane < 4) {
      const long long n = n0 + lane;
      if (n < P.capacity) {
        const int h = gr * 2 + (lane >> 1), w = gc * 2 + (lane & 1);
        P.pos_ids[3 * n + 0] = __ldg(P.frame_index + slot);
        P.pos_ids[3 * n + 1] = h;
        P.pos_ids[3 * n + 2] = w;
        P.src_index[n] = slot * P.np + h * P.grid_w + w;
      }
    }
  }
  cs::cp_async_wait<0>();
}

}  // namespace

// model coordinate o -> its two source taps along an axis (the device's nv12_axis, in the same fp32 operations)
static void host_axis(int o, int src, float scale, int* i0, int* i1) {
  volatile float t = static_cast<float>(o) + 0.5f;  // separate roundings, never contracted
  t = t * scale;
  t = t - 0.5f;
  float f = t;
  f = f < 0.0f ? 0.0f : f;
  *i0 = static_cast<int>(f);
  *i1 = *i0 + (*i0 < src - 1 ? 1 : 0);
}

// Row / column classes of the NV12 source-byte count (see NvSrcClasses); false = count only the outputs (pitches
// that are not multiples of 32)
static bool nv12_classes(const CompactParams& P, NvSrcClasses* C) {
  if (P.y_pitch % 32 != 0 || P.uv_pitch % 32 != 0) return false;
  const int gp = P.G * P.p, ncol = (P.src_w + 31) / 32;
  std::vector<unsigned long long> ry(P.src_h, 0ull), ruv((P.src_h + 1) / 2, 0ull), cm(ncol, 0ull);
  for (int o = 0; o < P.FH; ++o) {
    int a, b;
    host_axis(o, P.src_h, P.scale_y, &a, &b);
    const unsigned long long bit = 1ull << (o / gp);
    ry[a] |= bit;
    ry[b] |= bit;
    ruv[a / 2] |= bit;
    ruv[b / 2] |= bit;
  }
  for (int o = 0; o < P.FW; ++o) {
    int a, b;
    host_axis(o, P.src_w, P.scale_x, &a, &b);
    const unsigned long long bit = 1ull << (o / gp);
    cm[a / 32] |= bit;
    cm[b / 32] |= bit;
  }
  // classes: runs of equal masks (a row's group range is monotone in the row, so equal masks are contiguous;
  // merging runs of the same mask anyway keeps the tables small)
  auto add = [](NvClass* t, int* n, int cap, unsigned long long mask, int plane) -> bool {
    if (!mask) return true;
    for (int i = 0; i < *n; ++i)
      if (t[i].mask == mask && t[i].plane == plane) {
        ++t[i].n;
        return true;
      }
    if (*n >= cap) return false;
    t[*n].mask = mask;
    t[*n].n = 1;
    t[*n].plane = plane;
    ++*n;
    return true;
  };
  C->n_rows = C->n_cols = 0;
  for (unsigned long long m : ry)
    if (!add(C->rows, &C->n_rows, kNvMaxRowClasses, m, 0)) return false;
  for (unsigned long long m : ruv)
    if (!add(C->rows, &C->n_rows, kNvMaxRowClasses, m, 1)) return false;
  for (unsigned long long m : cm)
    if (!add(C->cols, &C->n_cols, kNvMaxColClasses, m, 0)) return false;
  C->enabled = 1;
  return true;
}

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
    P.one = 1.0f;
    P.negone = -1.0f;
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

  static NvSrcClasses none{};  // (zero: no source-byte count)
  NvSrcClasses* cls = &none;
  std::unique_ptr<NvSrcClasses> nvc;
  if (pre) {
    nvc.reset(new NvSrcClasses{});
    if (nv12_classes(P, nvc.get())) cls = nvc.get();
  }
  if (P.n_slots > 0) {
    compact_count<<<(P.n_slots + kCountThreads / 32 - 1) / (kCountThreads / 32), kCountThreads, 0, stream>>>(P,
                                                                                                          *cls);
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
  if (!grouped && !nv12 && tp == 1 && fast && g->grid_w == 32 && g->grid_h == 32 && P.vec_out &&
      (reinterpret_cast<uintptr_t>(keep_mask) & 15u) == 0) {
    // planar frames: band-staged gather (runs of consecutive kept groups, their 84 row spans staged with cp.async)
    const int nst = kBandMaxStages;  // (the cp.async wait count assumes exactly kBandMaxStages stages)
    const size_t bsmem = (size_t)kBandWarps * nst * kBandStage;
    const void* bf = reinterpret_cast<const void*>(compact_gather_band);
    if (cs_set_smem_attr(bf, 22, static_cast<int>(bsmem))) return CS_ERR_CUDA;
    compact_gather_band<<<cs_num_sms(), kBandWarps * 32, bsmem, stream>>>(P, nst);
    if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
    return CS_OK;
  }
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
  if (nv12 && tp == 1 && fast && P.y_pitch % 16 == 0 && P.uv_pitch % 16 == 0 && P.nw <= 64 &&
      static_cast<long long>(std::max(P.y_pitch, P.uv_pitch)) * P.src_h < (1ll << 31)) {
    // staged fused preprocessing: the widest column span of a group (16-B chunks, luma and chroma) picks the
    // staged row pitch
    int nch = 0;
    for (int gc = 0; gc < P.ngc; ++gc) {
      int a, b, c, d;
      host_axis(gc * 28, P.src_w, P.scale_x, &a, &b);
      host_axis(gc * 28 + 27, P.src_w, P.scale_x, &c, &d);
      const int xs = a & ~15;
      nch = std::max(nch, ((2 * (d >> 1) + 1 - xs) >> 4) + 1);
    }
    if (nch <= 16) {
      const int rb = nch <= 9 ? 144 : 256;
      const size_t nsmem = (size_t)kNvsWarps * kNvsStages * 16 * rb + (size_t)P.FH * 12;
      if (nsmem > 200 * 1024) goto nv12_direct;  // (a tall model input with the widest span: direct loads)
      const void* sf = rb == 144 ? reinterpret_cast<const void*>(compact_nv12_staged<144>)
                                 : reinterpret_cast<const void*>(compact_nv12_staged<256>);
      if (cs_set_smem_attr(sf, rb == 144 ? 23 : 24, 220 * 1024)) return CS_ERR_CUDA;
      static std::atomic<int> carveout_done[2];
      if (!carveout_done[rb == 144 ? 0 : 1].load(std::memory_order_acquire)) {
        // 4 CTAs x ~44 KB: ask for the largest shared-memory carveout (the kernel reads nothing through L1 twice)
        if (cudaFuncSetAttribute(sf, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared) != cudaSuccess)
          return CS_ERR_CUDA;
        carveout_done[rb == 144 ? 0 : 1].store(1, std::memory_order_release);
      }
      int per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sf, kNvsWarps * 32, nsmem) != cudaSuccess ||
          per_sm < 1)
        per_sm = 1;
      const int ngrid = cs_num_sms() * per_sm;
      if (rb == 144) compact_nv12_staged<144><<<ngrid, kNvsWarps * 32, nsmem, stream>>>(P);
      else compact_nv12_staged<256><<<ngrid, kNvsWarps * 32, nsmem, stream>>>(P);
      if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
      return CS_OK;
    }
  }
nv12_direct:
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
