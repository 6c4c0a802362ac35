// analysis.cu — NEXT-4 on sm_100a:
//   codecsight_mv_rasterize   FFmpeg AVMotionVector partitions -> the cs_mb grid consumed by score_patches
//                             (real H.264 metadata ingest; the decoder's MV extraction)
//   codecsight_similar_hist   per P-frame similar-patch ratio histogram for a set of thresholds
//                             (fig:mv_residual_analysis_cdf)
// Definitions: include/codecsight.h; oracle: codecsight_ref_mv_rasterize / codecsight_ref_similar_hist.
#include "cs_internal.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int qpel(int motion, int scale) {
  // trunc(4 * motion / scale) clamped to int16.  H.264 exports use scale 4 (quarter pel) -- and 2 / 1 for half /
  // full pel -- for which the quotient is exact (no rounding): shifts instead of the 64-bit division (the kernel is
  // issue-bound, ncu: 71 % issue slots), the general case keeps the division.
  long long v;
  if (scale == 4) v = motion;
  else if (scale == 2) v = 2ll * motion;
  else if (scale == 1) v = 4ll * motion;
  else v = (static_cast<long long>(motion) * 4) / (scale > 0 ? scale : 1);  // truncation toward zero
  v = v > 32767 ? 32767 : (v < -32768 ? -32768 : v);
  return static_cast<int>(v);
}

// One CTA per frame.  The output MB records double as 64-bit arbitration words: each past-reference partition
// atomicMax-es (|mv|^2 + 1) << 32 | ~record into every MB it overlaps (largest magnitude wins, ties -> the first
// record), then every MB decodes its winner in place (no winner: INTRA).
__global__ void __launch_bounds__(kThreads) mv_rasterize(int mb, int cols, int rows, const cs_av_mv* __restrict__ mvs,
                                                          const long long* __restrict__ offs, cs_mb* out) {
  const int f = blockIdx.x;
  const long long n_mb = static_cast<long long>(rows) * cols;
  unsigned long long* key = reinterpret_cast<unsigned long long*>(out + f * n_mb);
  for (long long e = threadIdx.x; e < n_mb; e += blockDim.x) key[e] = 0ull;
  __syncthreads();
  const long long r0 = offs[f], r1 = offs[f + 1];
  for (long long r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const cs_av_mv m = mvs[r];
    if (m.source >= 0) continue;
    const int x0 = static_cast<int>(m.dst_x) - m.w / 2, y0 = static_cast<int>(m.dst_y) - m.h / 2;
    const int x1 = x0 + m.w, y1 = y0 + m.h;  // [x0, x1) x [y0, y1)
    const int qx = qpel(m.motion_x, m.motion_scale), qy = qpel(m.motion_y, m.motion_scale);
    const unsigned long long sq = static_cast<unsigned long long>(static_cast<long long>(qx) * qx +
                                                                  static_cast<long long>(qy) * qy);
    const unsigned long long k = ((sq + 1ull) << 32) | (0xffffffffull - static_cast<unsigned long long>(r - r0));
    const int i_lo = max(0, (x0 >= 0 ? x0 : x0 - mb + 1) / mb), i_hi = min(cols - 1, (x1 - 1) / mb);
    const int j_lo = max(0, (y0 >= 0 ? y0 : y0 - mb + 1) / mb), j_hi = min(rows - 1, (y1 - 1) / mb);
    if (x1 <= 0 || y1 <= 0) continue;
    for (int j = j_lo; j <= j_hi; ++j)
      for (int i = i_lo; i <= i_hi; ++i) {
        const int ox = min(x1, mb * (i + 1)) - max(x0, mb * i);
        const int oy = min(y1, mb * (j + 1)) - max(y0, mb * j);
        if (ox > 0 && oy > 0) atomicMax(&key[static_cast<long long>(j) * cols + i], k);
      }
  }
  __syncthreads();
  for (long long e = threadIdx.x; e < n_mb; e += blockDim.x) {
    const unsigned long long k = key[e];
    cs_mb o;
    o.sad = 0;
    o.reserved = 0;
    if (k == 0ull) {
      o.mvx_qpel = 0;
      o.mvy_qpel = 0;
      o.mb_type = CS_MB_INTRA;
    } else {
      const long long r = r0 + static_cast<long long>(0xffffffffull - (k & 0xffffffffull));
      o.mvx_qpel = static_cast<int16_t>(qpel(mvs[r].motion_x, mvs[r].motion_scale));
      o.mvy_qpel = static_cast<int16_t>(qpel(mvs[r].motion_y, mvs[r].motion_scale));
      o.mb_type = CS_MB_INTER;
    }
    out[f * n_mb + e] = o;
  }
}

// The same arbitration with the frame's keys in shared memory (grids up to kSmemMbs MBs: 1080p's 8,160 MBs are 65 KB):
// shared-memory atomics instead of L2 atomics, and the output written once, coalesced.  Each record's quarter-pel
// vector is also kept in shared memory (the frame's first qcap records), so decoding a winner reads no global
// memory; MB_SHIFT > 0: the MB size is 1 << MB_SHIFT (H.264: 16) and the partition -> MB range is two shifts.
constexpr int kSmemMbs = 12288;
constexpr int kRastThreads = 1024;  // the per-thread record loop and the winner decode are latency chains: wide CTAs
template <int MB_SHIFT>
__global__ void __launch_bounds__(kRastThreads, 1) mv_rasterize_smem(int mb, int cols, int rows,
                                                                  const cs_av_mv* __restrict__ mvs,
                                                                  const long long* __restrict__ offs, cs_mb* out,
                                                                  int qcap) {
  extern __shared__ unsigned long long s_key[];
  uint32_t* s_q = reinterpret_cast<uint32_t*>(s_key + rows * cols);  // (qx & 0xffff) | qy << 16 per record
  const int f = blockIdx.x;
  const int n_mb = rows * cols;
  for (int e = threadIdx.x; e < n_mb; e += blockDim.x) s_key[e] = 0ull;
  __syncthreads();
  const long long r0 = offs[f], r1 = offs[f + 1];
  // a record's fields as four 8-B loads (bytes 0-15: source, w, h, src, dst; 24-31: motion; 32-39: scale; the
  // flags word is never read), the next record's loads in flight while this one is arbitrated
  struct Rec {
    uint2 a, b, c, d;
  };
  auto load = [&](long long r) {
    const uint2* p = reinterpret_cast<const uint2*>(mvs + r);
    return Rec{__ldg(p), __ldg(p + 1), __ldg(p + 3), __ldg(p + 4)};
  };
  long long r = r0 + threadIdx.x;
  Rec cur{};
  if (r < r1) cur = load(r);
  for (; r < r1; r += blockDim.x) {
    Rec nxt{};
    if (r + blockDim.x < r1) nxt = load(r + blockDim.x);
    const Rec m = cur;
    cur = nxt;
    if (static_cast<int>(m.a.x) >= 0) continue;  // source: past references only
    const int w = m.a.y & 0xffu, h = (m.a.y >> 8) & 0xffu;
    const int x0 = static_cast<int>(static_cast<int16_t>(m.b.x >> 16)) - w / 2;
    const int y0 = static_cast<int>(static_cast<int16_t>(m.b.y & 0xffffu)) - h / 2;
    const int x1 = x0 + w, y1 = y0 + h;  // [x0, x1) x [y0, y1)
    if (x1 <= 0 || y1 <= 0) continue;
    const int scale = static_cast<int>(m.d.x & 0xffffu);
    const int qx = qpel(static_cast<int>(m.c.x), scale), qy = qpel(static_cast<int>(m.c.y), scale);
    if (r - r0 < qcap) s_q[r - r0] = (static_cast<uint32_t>(qx) & 0xffffu) | (static_cast<uint32_t>(qy) << 16);
    const unsigned long long sq = static_cast<unsigned long long>(static_cast<long long>(qx) * qx +
                                                                  static_cast<long long>(qy) * qy);
    const unsigned long long k = ((sq + 1ull) << 32) | (0xffffffffull - static_cast<unsigned long long>(r - r0));
    // MBs i with [mb i, mb (i + 1)) meeting [x0, x1) in positive length: floor(x0 / mb) .. floor((x1 - 1) / mb),
    // clamped to the grid (x1 > 0 and y1 > 0 here; a partition right of / below the grid gives an empty range)
    int i_lo, i_hi, j_lo, j_hi;
    if (MB_SHIFT > 0) {
      i_lo = max(0, x0 >> MB_SHIFT);  // arithmetic shift = floor division
      i_hi = min(cols - 1, (x1 - 1) >> MB_SHIFT);
      j_lo = max(0, y0 >> MB_SHIFT);
      j_hi = min(rows - 1, (y1 - 1) >> MB_SHIFT);
    } else {
      i_lo = max(0, (x0 >= 0 ? x0 : x0 - mb + 1) / mb);
      i_hi = min(cols - 1, (x1 - 1) / mb);
      j_lo = max(0, (y0 >= 0 ? y0 : y0 - mb + 1) / mb);
      j_hi = min(rows - 1, (y1 - 1) / mb);
    }
    for (int j = j_lo; j <= j_hi; ++j)
      for (int i = i_lo; i <= i_hi; ++i) atomicMax(&s_key[j * cols + i], k);
  }
  __syncthreads();
  cs_mb* o = out + static_cast<long long>(f) * n_mb;
  for (int e = threadIdx.x; e < n_mb; e += blockDim.x) {
    const unsigned long long k = s_key[e];
    cs_mb v;
    v.sad = 0;
    v.reserved = 0;
    if (k == 0ull) {
      v.mvx_qpel = 0;
      v.mvy_qpel = 0;
      v.mb_type = CS_MB_INTRA;
    } else {
      const long long i = static_cast<long long>(0xffffffffull - (k & 0xffffffffull));
      if (i < qcap) {
        const uint32_t qq = s_q[i];
        v.mvx_qpel = static_cast<int16_t>(qq & 0xffffu);
        v.mvy_qpel = static_cast<int16_t>(qq >> 16);
      } else {
        v.mvx_qpel = static_cast<int16_t>(qpel(mvs[r0 + i].motion_x, mvs[r0 + i].motion_scale));
        v.mvy_qpel = static_cast<int16_t>(qpel(mvs[r0 + i].motion_y, mvs[r0 + i].motion_scale));
      }
      v.mb_type = CS_MB_INTER;
    }
    o[e] = v;
  }
}

// One warp per (frame, threshold): ballot-count patches with score < tau, bin = count * n_bins / n_patches.
__global__ void __launch_bounds__(kThreads) similar_hist(const float* __restrict__ score,
                                                          const uint8_t* __restrict__ frame_type, long long n_frames,
                                                          int n_patches, const float* __restrict__ taus, int n_tau,
                                                          int n_bins, unsigned long long* hist) {
  const int lane = threadIdx.x & 31;
  const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= n_frames * n_tau) return;
  const long long f = w / n_tau;
  const int t = static_cast<int>(w - f * n_tau);
  if (frame_type[f] != CS_FRAME_P) return;
  const float tau = taus[t];
  const float* s = score + f * n_patches;
  long long cnt = 0;
  for (int i0 = 0; i0 < n_patches; i0 += 32) {
    const int i = i0 + lane;
    cnt += __popc(__ballot_sync(0xffffffffu, i < n_patches && s[i] < tau));
  }
  if (lane == 0) {
    long long bin = cnt * n_bins / n_patches;
    if (bin >= n_bins) bin = n_bins - 1;
    atomicAdd(&hist[static_cast<long long>(t) * n_bins + bin], 1ull);
  }
}

}  // namespace

int cs_launch_mv_rasterize(const cs_grid* g, int32_t n_frames, const cs_av_mv* mvs, const int64_t* mv_offsets,
                           cs_mb* out, cudaStream_t stream) {
  if (n_frames == 0) return CS_OK;
  const long long n_mb = static_cast<long long>(g->mb_rows) * g->mb_cols;
  if (n_mb <= kSmemMbs) {
    // keys of the whole grid + the frame's first qcap quarter-pel vectors; one CTA per SM leaves ~80 KB of L1
    const int qcap = static_cast<int>((144 * 1024 - n_mb * 8) / 4);
    const size_t smem = static_cast<size_t>(n_mb) * 8 + static_cast<size_t>(qcap) * 4;
    const bool h264 = g->mb_size == 16;
    const void* fn = h264 ? reinterpret_cast<const void*>(mv_rasterize_smem<4>)
                          : reinterpret_cast<const void*>(mv_rasterize_smem<0>);
    if (cs_set_smem_attr(fn, h264 ? 21 : 25, 144 * 1024)) return CS_ERR_CUDA;
    const long long* offs = reinterpret_cast<const long long*>(mv_offsets);
    if (h264) mv_rasterize_smem<4><<<n_frames, kRastThreads, smem, stream>>>(16, g->mb_cols, g->mb_rows, mvs, offs, out, qcap);
    else mv_rasterize_smem<0><<<n_frames, kRastThreads, smem, stream>>>(g->mb_size, g->mb_cols, g->mb_rows, mvs, offs, out,
                                                                  qcap);
    return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
  }
  mv_rasterize<<<n_frames, kThreads, 0, stream>>>(g->mb_size, g->mb_cols, g->mb_rows, mvs,
                                                  reinterpret_cast<const long long*>(mv_offsets), out);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}

int cs_launch_similar_hist(const float* score, const uint8_t* frame_type, int64_t n_frames, int32_t n_patches,
                           const float* taus, int32_t n_tau, int32_t n_bins, unsigned long long* hist,
                           cudaStream_t stream) {
  const long long warps = n_frames * n_tau;
  if (warps == 0) return CS_OK;
  const long long blocks = (warps * 32 + kThreads - 1) / kThreads;
  similar_hist<<<static_cast<unsigned>(blocks), kThreads, 0, stream>>>(score, frame_type, n_frames, n_patches, taus,
                                                                        n_tau, n_bins, hist);
  return cudaGetLastError() == cudaSuccess ? CS_OK : CS_ERR_CUDA;
}
