// kv_refresh.cu — codecsight_kv_refresh on sm_100a: selective KVC refresh for one sliding-window step
// (Eq. 5 at P:354-357; SPEC plan_refresh S:390-398, selective_prefill S:399-402).
//
// Two launches:
//   kv_plan    one CTA per stream.  Stages the stream's (w + s) ring masks in shared memory, counts tokens per
//              frame with warp ballots, builds the per-frame segments of window k (reading Q12 makes every
//              segment a contiguous run in both the old and the new cache, with one uniform dp per stream-step),
//              writes the index outputs (disposition, p_old by p_new, n_tokens), clamps the data moves to the
//              capacities (status bits), and leaves in the workspace: a header, the segment list and the fp32
//              (cos, sin) table of R(dp) computed once per stream-step from fp64 angles (reading Q20).
//   kv_prefix  one CTA: the item prefix over the streams (items per stream from the plans' row counts) and the
//              gather's work counter zeroed.
//   kv_gather  persistent grid (one CTA per SM; production path kv_gather_tma: a TMA bulk ring per warp).  The
//              work items are (stream, 64-row block, layer, K|V), claimed dynamically by the warps from the work
//              counter (guided claim sizes, see kClaimMax).  Each item walks the segments that overlap its row block: REUSE K runs
//              are rotated (rotate_half pairs (i, i + D/2) loaded as two 16-B vectors, fp32 fma, RNE store),
//              REUSE V runs and refreshed rows are contiguous 16-B vector copies.  No tensor cores: nothing here
//              is a contraction; the kernel is HBM-bound.
#include <math_constants.h>
#include <stdio.h>
#include <stdlib.h>

#include "cs_internal.cuh"

namespace {

#ifndef CS_PLAN_THREADS
#define CS_PLAN_THREADS 512
#endif
constexpr int kPlanThreads = CS_PLAN_THREADS;  // one CTA per stream (512: measured faster than 256 / 1024)
constexpr int kGatherThreads = 256;
constexpr size_t kPlanSmem = 188 * 1024;  // kv_plan_paged dynamic shared memory limit (+ 33 KB static <= 227 KB)

#ifdef CS_PLAN_TIMING
// experiment build only (scripts/experiments/plan_phase.py): per-CTA %globaltimer stamps of kv_plan_paged
__device__ unsigned long long g_cs_plan_phase[4096][10];
#define CS_PLAN_PHASE(k)                                                              \
  do {                                                                                \
    __syncthreads();                                                                  \
    if (threadIdx.x == 0 && blockIdx.x < 4096) {                                      \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      g_cs_plan_phase[blockIdx.x][k] = t_;                                            \
    }                                                                                 \
  } while (0)
#else
#define CS_PLAN_PHASE(k)
#endif
// rows per gather work item (stream, row block, layer, K|V): 64 balances the grid's tail with guided claims at 32
// streams per GPU (0.896 -> 0.861 ms per step vs 128) and costs nothing at 256 / C5 (measured, round 2)
constexpr int kRowBlock = 64;
constexpr int kMaxSeg = 1025;  // w + 1 with w + s <= 1024

enum { SEG_SKIP = 0, SEG_COPY = 1, SEG_REUSE = 2 };

struct KvHdr {
  int n_rows;  // rows of the new cache that can be touched: min(n_total, capacity)
  int n_seg;
  int dp;
  int pad;
};
struct KvSeg {
  int p_new;  // first token (p_new) of the run
  int len;    // tokens (already clamped to the capacities)
  int kind;   // SEG_COPY (refreshed rows) | SEG_REUSE (old cache, K rotated, V copied) | SEG_SKIP
  int src;    // first source row (old cache / pool row for REUSE, refreshed-buffer row for COPY)
  int dst;    // first destination row (= p_new out of place; the pool slot in the paged variant)
  int pad[3];  // 32 B: keeps the cos/sin table that follows the run list 16-B aligned (TMA source)
};
static_assert(sizeof(KvSeg) == 32, "KvSeg must stay 32 bytes");
struct PlanSeg {  // per-frame index segment inside the plan kernels (shared memory)
  int p_new, len, kind, src;
};

struct KvParams {
  int grid_w, grid_h, G, nw, ngc, ngroups;
  int w, s, k, ring;
  int L, H, D, esz;
  long long cap, rcap, token_cap;
  int n_prompt, n_streams, max_seg, has_refreshed;
  int vec_rot, vec_copy;  // 16-B vector paths usable: (D/2) % (16/esz) == 0, row bytes % 16 == 0
  long long ws_stride;
  const uint32_t* mring;
  const uint8_t* tring;
  const void* const* old_cache;
  void* const* new_cache;
  const void* const* refreshed;
  uint8_t* disposition;
  int32_t* p_old;
  int32_t* n_tokens;
  unsigned char* ws;
  unsigned long long* counters;
  int32_t* status;
  // paged (in-place) variant
  void* const* pool;
  const int32_t* slot_old;
  int32_t* slot_new;
  long long slot_cap;
  int max_tok;      // w * groups + n_prompt: entries of the per-stream move list
  int mv_smem;      // kv_plan_paged: the move list is also staged in shared memory (runs pass reads it there)
  int prefix_mode;  // kv_prefix items: 0 = (stream, kRowBlock-row block, layer, K|V), 1 = tokens
  int paged;        // 1: REUSE runs rotate keys in place and leave values alone
  int rope_mode;    // CS_ROPE_1D | CS_ROPE_MROPE
  int mrope_t;      // M-RoPE: pairs of the temporal section (rotated by dt); the h / w sections stay
  long long mrope_dt;  // M-RoPE: temporal position change of a reused token (-stride * t_per_frame)
  int rot_pairs;       // pairs (i, i + D/2) of a reused key that Eq. 5 rewrites: D/2 (1-D), s_t (M-RoPE); the
                       // others keep their stored bits (reading NEXT-3)
  int partial_mode;    // paged with rot_pairs < D/2: a REUSE key chunk is rotated in place (its rotated pairs only)
                       // straight in global memory by the ring's warp instead of a TMA round trip of whole rows
  long long mv_off;  // byte offset of the move list inside a stream's workspace slice
  double inv_freq[cs::kMaxHeadDim / 2];  // base^(-2i/D), computed on the host
};

__device__ __forceinline__ unsigned char* stream_ws(const KvParams& P, int s) { return P.ws + 16 + (long long)s * P.ws_stride; }

// Rows are moved with 16-B vectors / TMA bulk copies whenever a row is a multiple of 16 B: every cache, pool and
// recompute buffer of a stream must then be 16-B aligned (element-aligned otherwise).  Device pointer arrays cannot
// be checked on the host, so each plan CTA checks its stream's buffers and, if one is misaligned, raises
// CS_STATUS_MISALIGNED and moves no row of that stream (a misaligned vector access would be a sticky fault).
__device__ __forceinline__ bool kv_misaligned(const KvParams& P, int sidx) {
  const uintptr_t a = P.vec_copy ? 15u : static_cast<uintptr_t>(P.esz - 1);
  uintptr_t m = reinterpret_cast<uintptr_t>(P.new_cache[sidx]);
  if (P.k >= 1) m |= reinterpret_cast<uintptr_t>(P.old_cache[sidx]);
  if (P.has_refreshed) m |= reinterpret_cast<uintptr_t>(P.refreshed[sidx]);
  return (m & a) != 0;
}

// ------------------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kPlanThreads) kv_plan(const __grid_constant__ KvParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_n[cs::kMaxWindowPlusStride];       // tokens per frame of [lo, hi)
  __shared__ uint8_t s_t[cs::kMaxWindowPlusStride];   // frame types
  __shared__ PlanSeg s_seg[kMaxSeg];                  // index segments (unclamped), one per frame + prompt
  __shared__ int s_pold[kMaxSeg];                     // p_old of the first token of the segment (-1: NEW)
  __shared__ int s_disp[kMaxSeg];
  __shared__ int s_nseg;
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(smem);  // [nfr][nw]

  const int sidx = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int k = P.k, w = P.w, s = P.s;
  const int lo = k >= 1 ? (k - 1) * s : 0;
  const int ks = k * s, hi = ks + w;
  const int nfr = hi - lo;
  const int nw = P.nw;

  for (int e = tid; e < nfr * nw; e += blockDim.x) {
    const int fi = e / nw, t = e - fi * nw;
    const int f = lo + fi;
    s_mask[e] = __ldg(P.mring + ((long long)sidx * P.ring + (f % P.ring)) * nw + t);
  }
  for (int fi = tid; fi < nfr; fi += blockDim.x) s_t[fi] = __ldg(P.tring + (long long)sidx * P.ring + ((lo + fi) % P.ring));
  __syncthreads();
  // tokens per frame = groups with any keep bit (same rule as codecsight_compact)
  for (int fi = warp; fi < nfr; fi += nwarp) {
    int n = 0;
    for (int base = 0; base < P.ngroups; base += 32) {
      const int q = base + lane;
      const bool kept = q < P.ngroups && cs::group_kept(s_mask + fi * nw, q, P.ngc, P.G, P.grid_w);
      n += __popc(__ballot_sync(0xffffffffu, kept));
    }
    if (lane == 0) s_n[fi] = n;
  }
  __syncthreads();
  // ---- (cos, sin) of R(dp), fp64 angle rounded to fp32 (reading Q20): warps 1.. while thread 0 builds the
  //      segment table (one sincos per pair) --------------------------------------------------------------------
  if (warp >= 1) {
    long long drop = 0;
    for (int f = lo; f < ks; ++f) drop += s_n[f - lo];
    float2* cs_tab = reinterpret_cast<float2*>(stream_ws(P, sidx) + sizeof(KvHdr) + sizeof(KvSeg) * P.max_seg);
    for (int i = tid - 32; i < P.D / 2; i += blockDim.x - 32) {
      // position change of pair i: the sequence-index change (1-D RoPE) or its section's component (M-RoPE)
      const long long delta = P.rope_mode == CS_ROPE_MROPE ? (i < P.mrope_t ? P.mrope_dt : 0ll) : -drop;
      double sn, cs;
      sincos(static_cast<double>(delta) * P.inv_freq[i], &sn, &cs);
      cs_tab[i] = make_float2(__double2float_rn(cs), __double2float_rn(sn));
    }
  }

  if (tid == 0) {
    // ---- serial segment construction over <= w + 1 entries -------------------------------------------
    long long drop = 0;  // tokens of the dropped frames [(k-1)s, ks)
    for (int f = lo; f < ks; ++f) drop += s_n[f - lo];
    const int new_first = (k - 1) * s + w;  // frames >= new_first arrived with this stride
    long long pnew = 0, rrow = 0, n_reuse = 0, n_anchor = 0, n_new = 0;
    int nseg = 0;
    for (int f = ks; f < hi; ++f) {
      const int n = s_n[f - lo];
      int disp, pold;
      if (k == 0 || f >= new_first) {
        disp = CS_DISP_NEW;
        pold = -1;
      } else {
        disp = (s_t[f - lo] != CS_FRAME_P || f == ks) ? CS_DISP_ANCHOR : CS_DISP_REUSE;  // P:346, Q17
        pold = static_cast<int>(drop + pnew);
      }
      s_seg[nseg].p_new = static_cast<int>(pnew);
      s_seg[nseg].len = n;
      s_seg[nseg].kind = disp;
      s_seg[nseg].src = disp == CS_DISP_REUSE ? pold : static_cast<int>(rrow);
      s_pold[nseg] = pold;
      s_disp[nseg] = disp;
      ++nseg;
      if (disp != CS_DISP_REUSE) rrow += n;
      if (disp == CS_DISP_REUSE) n_reuse += n;
      else if (disp == CS_DISP_ANCHOR) n_anchor += n;
      else n_new += n;
      pnew += n;
    }
    const long long n_visual = pnew;
    // prompt rows, always NEW
    s_seg[nseg].p_new = static_cast<int>(pnew);
    s_seg[nseg].len = P.n_prompt;
    s_seg[nseg].kind = CS_DISP_NEW;
    s_seg[nseg].src = static_cast<int>(rrow);
    s_pold[nseg] = -1;
    s_disp[nseg] = CS_DISP_NEW;
    ++nseg;
    n_new += P.n_prompt;
    const long long n_total = n_visual + P.n_prompt;
    s_nseg = nseg;

    int* nt = P.n_tokens + (long long)sidx * 4;
    nt[0] = static_cast<int>(n_visual);
    nt[1] = static_cast<int>(n_reuse);
    nt[2] = static_cast<int>(n_anchor);
    nt[3] = static_cast<int>(n_new);

    // ---- clamp the data moves (same rules as the oracle, per row) ---------------------------------------
    int st = 0;
    if (n_total > P.token_cap) st |= CS_STATUS_CAPACITY;
    const bool mis = kv_misaligned(P, sidx);
    if (mis) st |= CS_STATUS_MISALIGNED;
    unsigned char* ws = stream_ws(P, sidx);
    KvSeg* wseg = reinterpret_cast<KvSeg*>(ws + sizeof(KvHdr));
    int nout = 0;
    long long moved = 0;
    for (int i = 0; i < nseg; ++i) {
      const long long pn = s_seg[i].p_new, len = s_seg[i].len, src = s_seg[i].src;
      long long valid = 0;
      int kind = SEG_SKIP;
      if (len == 0) continue;
      if (s_disp[i] == CS_DISP_REUSE) {
        // rows t with pn + t >= cap: CAPACITY; rows with pn + t < cap <= src + t: ORIGIN (src >= pn)
        const long long in_cap = P.cap - pn;  // rows with p_new < cap
        if (len > (in_cap > 0 ? in_cap : 0)) st |= CS_STATUS_CAPACITY;
        valid = P.cap - src;
        valid = valid < 0 ? 0 : (valid > len ? len : valid);
        const long long lim = in_cap < len ? (in_cap > 0 ? in_cap : 0) : len;
        if (lim > valid) st |= CS_STATUS_ORIGIN;
        kind = SEG_REUSE;
      } else if (P.has_refreshed) {
        const long long a = P.cap - pn, b = P.rcap - src;
        valid = a < b ? a : b;
        valid = valid < 0 ? 0 : (valid > len ? len : valid);
        if (valid < len) st |= CS_STATUS_CAPACITY;
        kind = SEG_COPY;
      }
      if (valid > 0 && !mis) {
        wseg[nout].p_new = static_cast<int>(pn);
        wseg[nout].len = static_cast<int>(valid);
        wseg[nout].kind = kind;
        wseg[nout].src = static_cast<int>(src);
        wseg[nout].dst = static_cast<int>(pn);
        ++nout;
        moved += valid;
      }
    }
    KvHdr* hdr = reinterpret_cast<KvHdr*>(ws);
    hdr->n_rows = static_cast<int>(n_total < P.cap ? n_total : P.cap);
    hdr->n_seg = nout;
    hdr->dp = static_cast<int>(-drop);
    hdr->pad = 0;
    cs::atomic_or_status(P.status, st);
    cs::atomic_add_u64(&P.counters[CS_CNT_TOK_REUSE], static_cast<unsigned long long>(n_reuse));
    cs::atomic_add_u64(&P.counters[CS_CNT_TOK_ANCHOR], static_cast<unsigned long long>(n_anchor));
    cs::atomic_add_u64(&P.counters[CS_CNT_TOK_NEW], static_cast<unsigned long long>(n_new));
    cs::atomic_add_u64(&P.counters[CS_CNT_BYTES_KV], static_cast<unsigned long long>(moved) * P.L * 2ull *
                                                         (unsigned long long)(P.H * P.D * P.esz) * 2ull);
    cs::atomic_add_u64(&P.counters[CS_CNT_STREAM_STEPS], 1ull);
  }
  __syncthreads();

  // ---- index outputs by p_new: disposition, p_old --------------------------------------------------------
  const int nseg = s_nseg;
  uint8_t* dsp = P.disposition + (long long)sidx * P.token_cap;
  int32_t* po = P.p_old + (long long)sidx * P.token_cap;
  for (int i = warp; i < nseg; i += nwarp) {
    const long long pn = s_seg[i].p_new;
    const int len = s_seg[i].len, d = s_disp[i], pold = s_pold[i];
    for (int t = lane; t < len; t += 32) {
      const long long p = pn + t;
      if (p < P.token_cap) {
        dsp[p] = static_cast<uint8_t>(d);
        po[p] = d == CS_DISP_NEW ? -1 : pold + t;
      }
    }
  }

}

// ------------------------------------------------------------------------------------------------------------
// gather: rotate/copy contiguous row runs
// ------------------------------------------------------------------------------------------------------------
template <typename T>
struct Vec;  // 16-B vector of cache elements
template <>
struct Vec<uint16_t> {
  static constexpr int N = 8;
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
};

__device__ __forceinline__ void rot8_bf16(uint4& a, uint4& b, const float* c, const float* s) {
  uint32_t* pa = reinterpret_cast<uint32_t*>(&a);
  uint32_t* pb = reinterpret_cast<uint32_t*>(&b);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float x1l = cs::bf16_lo(pa[q]), x1h = cs::bf16_hi(pa[q]);
    const float x2l = cs::bf16_lo(pb[q]), x2h = cs::bf16_hi(pb[q]);
    const float cl = c[2 * q], ch = c[2 * q + 1], sl = s[2 * q], sh = s[2 * q + 1];
    const float o1l = __fmaf_rn(x1l, cl, -__fmul_rn(x2l, sl));
    const float o2l = __fmaf_rn(x2l, cl, __fmul_rn(x1l, sl));
    const float o1h = __fmaf_rn(x1h, ch, -__fmul_rn(x2h, sh));
    const float o2h = __fmaf_rn(x2h, ch, __fmul_rn(x1h, sh));
    pa[q] = cs::f32_to_bf16_rne(o1l) | (cs::f32_to_bf16_rne(o1h) << 16);
    pb[q] = cs::f32_to_bf16_rne(o2l) | (cs::f32_to_bf16_rne(o2h) << 16);
  }
}

__device__ __forceinline__ void rot4_f32(uint4& a, uint4& b, const float* c, const float* s) {
  float* pa = reinterpret_cast<float*>(&a);
  float* pb = reinterpret_cast<float*>(&b);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float x1 = pa[q], x2 = pb[q];
    pa[q] = __fmaf_rn(x1, c[q], -__fmul_rn(x2, s[q]));
    pb[q] = __fmaf_rn(x2, c[q], __fmul_rn(x1, s[q]));
  }
}

// Rotate `nrows` contiguous K rows (Eq. 5).  Work unit = one pair of 16-B vectors (elements j*VE.. of the first
// and second half of one head).  TH/TD > 0: compile-time head count / head dim (production shape).
template <typename T, int TH, int TD>
__device__ __forceinline__ void rotate_run(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                                           int nrows, int rH, int rD, const float* s_c, const float* s_s,
                                           int rot_pairs) {
  constexpr int VE = Vec<T>::N;
  const int H = TH > 0 ? TH : rH;
  const int D = TD > 0 ? TD : rD;
  const int half = D / 2;
  const int vph = half / VE;  // vectors per half-head
  const int upr = H * vph;    // units per row
  const int rowb = H * D * static_cast<int>(sizeof(T));
  const int total = nrows * upr;
  constexpr int kU = 4;
  for (int e0 = threadIdx.x; e0 < total; e0 += kU * blockDim.x) {
    uint4 a[kU], b[kU];
    int off1[kU], jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < total) {
        const int row = e / upr, un = e - row * upr;
        const int h = un / vph, j = un - h * vph;
        off1[u] = row * rowb + (h * D + j * VE) * static_cast<int>(sizeof(T));
        jv[u] = j;
        a[u] = cs::ld_nc_v4(src + off1[u]);
        b[u] = cs::ld_nc_v4(src + off1[u] + half * static_cast<int>(sizeof(T)));
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < total) {
        const float* c = s_c + jv[u] * VE;
        const float* s = s_s + jv[u] * VE;
        if (jv[u] * VE < rot_pairs) {  // else: a pair of an unchanged M-RoPE section, copied bit for bit
          if constexpr (sizeof(T) == 2) rot8_bf16(a[u], b[u], c, s);
          else rot4_f32(a[u], b[u], c, s);
        }
        cs::st_na_v4(dst + off1[u], a[u]);
        cs::st_na_v4(dst + off1[u] + half * static_cast<int>(sizeof(T)), b[u]);
      }
    }
  }
}

// contiguous copy of `bytes` (multiple of 16) with 4 vectors in flight per thread
__device__ __forceinline__ void copy_run(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                                         long long bytes) {
  const long long n = bytes >> 4;
  constexpr int kU = 4;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (long long e0 = threadIdx.x; e0 < n; e0 += kU * blockDim.x) {
    uint4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long e = e0 + (long long)u * blockDim.x;
      if (e < n) v[u] = cs::ld_nc_v4(s4 + e);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long e = e0 + (long long)u * blockDim.x;
      if (e < n) cs::st_na_v4(d4 + e, v[u]);
    }
  }
}

// generic fallbacks (toy shapes): element-pair rotation and 4-byte copies
template <typename T>
__device__ __forceinline__ void rotate_run_scalar(const unsigned char* __restrict__ src,
                                                  unsigned char* __restrict__ dst, int nrows, int H, int D,
                                                  const float* s_c, const float* s_s, int rot_pairs) {
  const int half = D / 2;
  const int total = nrows * H * half;
  const T* sp = reinterpret_cast<const T*>(src);
  T* dp = reinterpret_cast<T*>(dst);
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int row = e / (H * half), r = e - row * H * half;
    const int h = r / half, i = r - h * half;
    const long long o1 = (long long)row * H * D + h * D + i, o2 = o1 + half;
    if (i >= rot_pairs) {  // unchanged M-RoPE section: bit copy
      dp[o1] = sp[o1];
      dp[o2] = sp[o2];
      continue;
    }
    float x1, x2;
    if constexpr (sizeof(T) == 2) {
      x1 = __uint_as_float(static_cast<uint32_t>(sp[o1]) << 16);
      x2 = __uint_as_float(static_cast<uint32_t>(sp[o2]) << 16);
    } else {
      x1 = sp[o1];
      x2 = sp[o2];
    }
    const float y1 = __fmaf_rn(x1, s_c[i], -__fmul_rn(x2, s_s[i]));
    const float y2 = __fmaf_rn(x2, s_c[i], __fmul_rn(x1, s_s[i]));
    if constexpr (sizeof(T) == 2) {
      dp[o1] = static_cast<T>(cs::f32_to_bf16_rne(y1));
      dp[o2] = static_cast<T>(cs::f32_to_bf16_rne(y2));
    } else {
      dp[o1] = y1;
      dp[o2] = y2;
    }
  }
}

__device__ __forceinline__ void copy_run_u32(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst,
                                             long long bytes) {
  const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
  uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
  for (long long e = threadIdx.x; e < (bytes >> 2); e += blockDim.x) d4[e] = s4[e];
}

template <typename T, int TH, int TD>
__global__ void __launch_bounds__(kGatherThreads) kv_gather_ldg(const __grid_constant__ KvParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  long long* s_pref = reinterpret_cast<long long*>(smem);                         // [n_streams + 1]
  KvSeg* s_seg = reinterpret_cast<KvSeg*>(smem + 8 * ((P.n_streams + 2) & ~1));  // [max_seg]
  float* s_c = reinterpret_cast<float*>(s_seg + P.max_seg);                       // [D/2]
  float* s_s = s_c + P.D / 2;
  __shared__ long long s_carry;
  __shared__ int s_nseg, s_cur;

  const int tid = threadIdx.x;
  const int items_per_block = P.L * 2;
  // ---- item prefix over streams (identical in every CTA) --------------------------------------------------
  if (tid == 0) {
    s_carry = 0;
    s_cur = -1;
  }
  __syncthreads();
  __shared__ long long s_wsum[kGatherThreads / 32];
  const int lane = tid & 31, warp = tid >> 5;
  for (int base = 0; base < P.n_streams; base += blockDim.x) {
    const int si = base + tid;
    long long v = 0;
    if (si < P.n_streams) {
      const KvHdr* h = reinterpret_cast<const KvHdr*>(stream_ws(P, si));
      const long long rows = h->n_seg > 0 ? h->n_rows : 0;
      v = (rows + kRowBlock - 1) / kRowBlock * items_per_block;
    }
    long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long u = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += u;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    long long woff = s_carry;
    for (int q = 0; q < warp; ++q) woff += s_wsum[q];
    if (si < P.n_streams) s_pref[si + 1] = woff + inc;
    __syncthreads();
    if (tid == blockDim.x - 1) s_carry = woff + inc;
    __syncthreads();
  }
  if (tid == 0) s_pref[0] = 0;
  __syncthreads();
  const long long V = s_pref[P.n_streams];
  const long long it0 = V * blockIdx.x / gridDim.x, it1 = V * (blockIdx.x + 1) / gridDim.x;
  const long long row_bytes = (long long)P.H * P.D * sizeof(T);

  int sidx = 0;
  for (long long it = it0; it < it1; ++it) {
    while (s_pref[sidx + 1] <= it) ++sidx;  // uniform across the CTA
    if (sidx != s_cur) {
      __syncthreads();
      const unsigned char* ws = stream_ws(P, sidx);
      const KvHdr* h = reinterpret_cast<const KvHdr*>(ws);
      const KvSeg* g = reinterpret_cast<const KvSeg*>(ws + sizeof(KvHdr));
      const int nseg = h->n_seg;
      for (int i = tid; i < nseg; i += blockDim.x) s_seg[i] = g[i];
      const float2* tab = reinterpret_cast<const float2*>(ws + sizeof(KvHdr) + sizeof(KvSeg) * P.max_seg);
      for (int i = tid; i < P.D / 2; i += blockDim.x) {
        const float2 cs2 = tab[i];
        s_c[i] = cs2.x;
        s_s[i] = cs2.y;
      }
      if (tid == 0) {
        s_nseg = nseg;
        s_cur = sidx;
      }
      __syncthreads();
    }
    const long long local = it - s_pref[sidx];
    const int blk = static_cast<int>(local / items_per_block);
    const int lk = static_cast<int>(local - (long long)blk * items_per_block);
    const int l = lk >> 1, kv = lk & 1;
    const int a = blk * kRowBlock, b = a + kRowBlock;
    unsigned char* nc = static_cast<unsigned char*>(P.new_cache[sidx]);
    const unsigned char* oc = P.k >= 1 ? static_cast<const unsigned char*>(P.old_cache[sidx]) : nullptr;
    const unsigned char* rf = P.has_refreshed ? static_cast<const unsigned char*>(P.refreshed[sidx]) : nullptr;
    const long long plane_new = ((long long)(l * 2 + kv)) * P.cap;
    for (int i = 0; i < s_nseg; ++i) {
      const KvSeg sg = s_seg[i];
      const int x0 = max(a, sg.p_new), x1 = min(b, sg.p_new + sg.len);
      if (x0 >= x1) continue;
      const int n = x1 - x0;
      const long long srow = sg.src + (x0 - sg.p_new);
      unsigned char* dst = nc + (plane_new + x0) * row_bytes;
      if (sg.kind == SEG_REUSE) {
        const unsigned char* src = oc + (plane_new + srow) * row_bytes;
        if (kv == 0) {  // Eq. 5
          if (P.vec_rot) rotate_run<T, TH, TD>(src, dst, n, P.H, P.D, s_c, s_s, P.rot_pairs);
          else rotate_run_scalar<T>(src, dst, n, P.H, P.D, s_c, s_s, P.rot_pairs);
        } else {  // value reuse
          if (TH > 0 || P.vec_copy) copy_run(src, dst, n * row_bytes);
          else copy_run_u32(src, dst, n * row_bytes);
        }
      } else {
        const unsigned char* src = rf + (((long long)(l * 2 + kv)) * P.rcap + srow) * row_bytes;
        if (TH > 0 || P.vec_copy) copy_run(src, dst, n * row_bytes);
        else copy_run_u32(src, dst, n * row_bytes);
      }
    }
  }
}


// ------------------------------------------------------------------------------------------------------------
// TMA bulk-copy pipelines (production path), one per WARP.  Every contiguous row run is cut into <= 8 KB chunks
// that stream global -> shared (cp.async.bulk, mbarrier complete_tx) -> global (cp.async.bulk bulk_group store)
// through the warp's NST-deep ring; REUSE K chunks are rotated in shared memory in between (Eq. 5) by the warp's
// 32 lanes.  Lane 0 drives the ring (chunk generation, load/store issue).  Eight independent rings per CTA keep
// the issue overhead off the critical path and ~8 x NST x 8 KB in flight per SM without register staging.
// ------------------------------------------------------------------------------------------------------------
constexpr int kTmaChunk = 8192;
// Dynamic work claims are GUIDED: a warp claims max(1, min(kClaimMax, remaining / (kClaimDiv * warps))) items,
// sizing from the counter value it last saw, so claims shrink to single items at the end of the kernel (the tail
// imbalance is then about one item, not one 4-item claim = up to 512 KB = ~90 us of a warp's ring at 32 streams per
// GPU), while large batches (C5: 3.7 M items) keep few atomics on the shared counter.
constexpr int kClaimMax = 16;
constexpr int kClaimDiv = 8;
constexpr int kWarpsPerGather = kGatherThreads / 32;
constexpr int kMaxStages = 6;
constexpr int kPartialRows = 32;  // rows per in-place partial (M-RoPE temporal section) rotation item

struct ChunkDesc {
  unsigned char* dst;
  uint32_t bytes;  // 0 = end of the sequence
  int rotate;      // 1: K rows of a REUSE run (rotate by R(dp))
  int rows;
  int pad;
};

struct ChunkGen {  // generator state, owned by lane 0 of a warp
  long long it, it1;
  int sidx, seg, x, active;
  int nseg, a, b, l, kv;
  int c_sidx, c_blk, c_seg;  // cache: stream whose pointers are loaded; (stream, block) of the last run search
  long long V;               // total items
  long long next_claim;      // start of the next claimed range (claimed one range ahead), >= V when exhausted
  int next_size;             // items in that range
  int claim_div;             // kClaimDiv x the grid's warps
  unsigned long long* ctr;   // work counter in the workspace header (zeroed by kv_prefix)
  const KvSeg* segs;
  unsigned char* nc;
  const unsigned char* oc;
  const unsigned char* rf;
  const void* tab;
};

// claim the next range (lane 0 of the warp); `seen` = the largest counter value this warp has observed
__device__ __forceinline__ void claim(ChunkGen& g, long long seen) {
  const long long rem = g.V - seen;
  const int sz = static_cast<int>(rem <= 0 ? 1 : min(static_cast<long long>(kClaimMax), max(1ll, rem / g.claim_div)));
  g.next_size = sz;
  g.next_claim = static_cast<long long>(atomicAdd(g.ctr, static_cast<unsigned long long>(sz)));
}

__device__ __forceinline__ const int* ws_prefix(const KvParams& P) {
  return reinterpret_cast<const int*>(P.ws + 16 + (long long)P.n_streams * P.ws_stride);
}

__device__ __forceinline__ bool gen_next(const KvParams& P, const int* pref, ChunkGen& g, int cr,
                                         long long row_bytes, const unsigned char*& src, ChunkDesc& d,
                                         const void*& tab) {
  const int ipb = P.L * 2;
  for (;;) {
    if (g.it >= g.it1) {
      // dynamic balancing: take the range claimed earlier, claim the next one now (latency hidden by the ring)
      if (g.next_claim >= g.V) return false;
      g.it = g.next_claim;
      g.it1 = min(g.V, g.it + g.next_size);
      claim(g, g.it1);
      if (__ldg(pref + g.sidx) > g.it) g.sidx = 0;  // (claims only increase; defensive)
      g.active = 0;
    }
    if (!g.active) {
      // items of one stream are contiguous and ordered (block, layer, K|V): stream pointers and the run search
      // of a block are cached across the 2L items that share them
      if (__ldg(pref + g.sidx + 1) <= g.it) {  // find the stream of item g.it: pref[s] <= it < pref[s + 1]
        int lo = g.sidx + 1, hi = P.n_streams;
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (__ldg(pref + mid) <= g.it) lo = mid; else hi = mid;
        }
        g.sidx = lo;
        while (__ldg(pref + g.sidx + 1) <= g.it) ++g.sidx;
      }
      const long long local = g.it - __ldg(pref + g.sidx);
      const int blk = static_cast<int>(local / ipb);
      const int lk = static_cast<int>(local - (long long)blk * ipb);
      g.l = lk >> 1;
      g.kv = lk & 1;
      g.a = blk * kRowBlock;
      g.b = g.a + kRowBlock;
      if (g.sidx != g.c_sidx) {
        const unsigned char* ws = stream_ws(P, g.sidx);
        g.nseg = reinterpret_cast<const KvHdr*>(ws)->n_seg;
        g.segs = reinterpret_cast<const KvSeg*>(ws + sizeof(KvHdr));
        g.tab = ws + sizeof(KvHdr) + sizeof(KvSeg) * P.max_seg;
        g.nc = static_cast<unsigned char*>(P.new_cache[g.sidx]);
        g.oc = P.k >= 1 ? static_cast<const unsigned char*>(P.old_cache[g.sidx]) : nullptr;
        g.rf = P.has_refreshed ? static_cast<const unsigned char*>(P.refreshed[g.sidx]) : nullptr;
        g.c_sidx = g.sidx;
        g.c_blk = -1;
      }
      if (blk != g.c_blk) {
        // first run that ends after the block start (runs are sorted by p_new and disjoint)
        int lo = 0, hi = g.nseg;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const KvSeg m = g.segs[mid];
          if (m.p_new + m.len <= g.a) lo = mid + 1; else hi = mid;
        }
        g.c_blk = blk;
        g.c_seg = lo;
      }
      g.seg = g.c_seg;
      g.x = g.a;
      g.active = 1;
    }
    while (g.seg < g.nseg) {
      const KvSeg sg = g.segs[g.seg];
      if (sg.p_new >= g.b) {
        g.seg = g.nseg;
        break;
      }
      const int x0 = max(g.x, sg.p_new), x1 = min(g.b, sg.p_new + sg.len);
      if (x0 >= x1 || sg.kind == SEG_SKIP || (P.paged && sg.kind == SEG_REUSE && g.kv == 1)) {
        ++g.seg;
        continue;
      }
      // in place with M-RoPE only the temporal section of a reused key changes: no TMA round trip of the whole
      // row, the warp rotates those pairs straight in global memory (rotate = 2), in larger row batches
      const bool partial = P.partial_mode && sg.kind == SEG_REUSE && g.kv == 0;
      const int n = min(partial ? kPartialRows : cr, x1 - x0);
      const long long plane = static_cast<long long>(g.l * 2 + g.kv);
      const long long srow = sg.src + (x0 - sg.p_new);
      const long long drow = sg.dst + (x0 - sg.p_new);
      d.dst = g.nc + (plane * P.cap + drow) * row_bytes;
      d.bytes = static_cast<uint32_t>(n * row_bytes);
      d.rows = n;
      if (sg.kind == SEG_REUSE) {
        src = g.oc + (plane * P.cap + srow) * row_bytes;
        d.rotate = partial ? 2 : (g.kv == 0);
      } else {
        src = g.rf + (plane * P.rcap + srow) * row_bytes;
        d.rotate = 0;
      }
      tab = g.tab;
      g.x = x0 + n;
      if (g.x >= x1) ++g.seg;
      return true;
    }
    ++g.it;
    g.active = 0;
  }
}

// 1 CTA: item prefix over streams into the workspace (item = stream x kRowBlock-row block x layer x K|V)
__global__ void __launch_bounds__(1024) kv_prefix(const __grid_constant__ KvParams P) {
  __shared__ int s_wsum[32];
  __shared__ int s_carry;
  int* pref = const_cast<int*>(ws_prefix(P));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ipb = P.L * 2;
  if (tid == 0) {
    s_carry = 0;
    pref[0] = 0;
    *reinterpret_cast<unsigned long long*>(P.ws) = 0ull;  // work counter of the gather (dynamic claims)
  }
  __syncthreads();
  for (int base = 0; base < P.n_streams; base += blockDim.x) {
    const int si = base + tid;
    int v = 0;
    if (si < P.n_streams) {
      const KvHdr* h = reinterpret_cast<const KvHdr*>(stream_ws(P, si));
      if (P.prefix_mode == 1) {
        v = h->n_rows;  // paged: one item per token (all layers)
      } else {
        const int rows = h->n_seg > 0 ? h->n_rows : 0;
        v = (rows + kRowBlock - 1) / kRowBlock * ipb;
      }
    }
    int inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += u;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    int woff = s_carry;
    for (int q = 0; q < warp; ++q) woff += s_wsum[q];
    if (si < P.n_streams) pref[si + 1] = woff + inc;
    __syncthreads();
    if (tid == blockDim.x - 1) s_carry = woff + inc;
    __syncthreads();
  }
}

__device__ __forceinline__ void rot8_bf16_pack(uint4& a, uint4& b, const float* c, const float* s) {
  uint32_t* pa = reinterpret_cast<uint32_t*>(&a);
  uint32_t* pb = reinterpret_cast<uint32_t*>(&b);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float x1l = cs::bf16_lo(pa[q]), x1h = cs::bf16_hi(pa[q]);
    const float x2l = cs::bf16_lo(pb[q]), x2h = cs::bf16_hi(pb[q]);
    const float cl = c[2 * q], ch = c[2 * q + 1], sl = s[2 * q], sh = s[2 * q + 1];
    const float o1l = __fmaf_rn(x1l, cl, -__fmul_rn(x2l, sl));
    const float o2l = __fmaf_rn(x2l, cl, __fmul_rn(x1l, sl));
    const float o1h = __fmaf_rn(x1h, ch, -__fmul_rn(x2h, sh));
    const float o2h = __fmaf_rn(x2h, ch, __fmul_rn(x1h, sh));
    pa[q] = cs::pack_bf16x2_rn(o1l, o1h);  // cvt.rn.bf16x2.f32: round to nearest even
    pb[q] = cs::pack_bf16x2_rn(o2l, o2h);
  }
}

// rotate the K rows of one chunk in shared memory; executed by the 32 lanes of one warp
template <typename T, int TH, int TD>
__device__ __forceinline__ void rotate_smem_warp(unsigned char* buf, const float2* tab, int rows, int rH, int rD,
                                                 int rot_pairs, int lane) {
  constexpr int VE = Vec<T>::N;
  const int H = TH > 0 ? TH : rH;
  const int D = TD > 0 ? TD : rD;
  const int half = D / 2;
  const int vph = rot_pairs / VE;  // rotated vectors per half-head (the rest of the row is already in place)
  const int upr = H * vph;
  const int rowb = H * D * static_cast<int>(sizeof(T));
  const int total = rows * upr;
  for (int e = lane; e < total; e += 32) {
    const int row = e / upr, un = e - row * upr;
    const int h = un / vph, j = un - h * vph;
    unsigned char* p1 = buf + row * rowb + (h * D + j * VE) * static_cast<int>(sizeof(T));
    unsigned char* p2 = p1 + half * static_cast<int>(sizeof(T));
    uint4 a = *reinterpret_cast<const uint4*>(p1);
    uint4 b = *reinterpret_cast<const uint4*>(p2);
    float c[VE], s[VE];
#pragma unroll
    for (int v = 0; v < VE; v += 2) {
      const float4 t = *reinterpret_cast<const float4*>(tab + j * VE + v);
      c[v] = t.x;
      s[v] = t.y;
      c[v + 1] = t.z;
      s[v + 1] = t.w;
    }
    if constexpr (sizeof(T) == 2) rot8_bf16_pack(a, b, c, s);
    else rot4_f32(a, b, c, s);
    *reinterpret_cast<uint4*>(p1) = a;
    *reinterpret_cast<uint4*>(p2) = b;
  }
}

// In-place rotation of the first rot_pairs pairs (i, i + D/2) of every head of `rows` contiguous key rows, straight
// in global memory (M-RoPE: the temporal section; the h / w sections are not touched).  All loads of a batch are
// issued before any rotation (memory-level parallelism); executed by the 32 lanes of one warp.
template <typename T, int TH, int TD>
__device__ __forceinline__ void rotate_partial_global(unsigned char* base, const float2* tab, int rows, int rH, int rD,
                                                      int rot_pairs, int lane) {
  constexpr int VE = Vec<T>::N;
  const int H = TH > 0 ? TH : rH;
  const int D = TD > 0 ? TD : rD;
  const int half = D / 2;
  const int vph = rot_pairs / VE;
  const int upr = H * vph;
  const int rowb = H * D * static_cast<int>(sizeof(T));
  const int total = rows * upr;
  constexpr int kU = 8;
  for (int e0 = lane; e0 < total; e0 += 32 * kU) {
    uint4 a[kU], b[kU];
    int off[kU], jv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * 32;
      if (e < total) {
        const int row = e / upr, un = e - row * upr;
        const int h = un / vph, j = un - h * vph;
        off[u] = row * rowb + (h * D + j * VE) * static_cast<int>(sizeof(T));
        jv[u] = j;
        a[u] = *reinterpret_cast<const uint4*>(base + off[u]);
        b[u] = *reinterpret_cast<const uint4*>(base + off[u] + half * static_cast<int>(sizeof(T)));
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * 32;
      if (e < total) {
        float c[VE], sn[VE];
#pragma unroll
        for (int v = 0; v < VE; ++v) {
          const float2 t = tab[jv[u] * VE + v];
          c[v] = t.x;
          sn[v] = t.y;
        }
        if constexpr (sizeof(T) == 2) rot8_bf16_pack(a[u], b[u], c, sn);
        else rot4_f32(a[u], b[u], c, sn);
        cs::st_na_v4(base + off[u], a[u]);
        cs::st_na_v4(base + off[u] + half * static_cast<int>(sizeof(T)), b[u]);
      }
    }
  }
}

template <typename T, int TH, int TD>
__global__ void __launch_bounds__(kGatherThreads, 1) kv_gather_tma(const __grid_constant__ KvParams P, int nst,
                                                                   unsigned stage_bytes, unsigned tab_bytes) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ ChunkDesc s_desc[kWarpsPerGather][kMaxStages];
  __shared__ __align__(8) uint64_t s_full[kWarpsPerGather][kMaxStages];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* stages = smem + (size_t)wib * nst * (stage_bytes + tab_bytes);  // this warp's ring
  unsigned char* tabs = stages + (size_t)nst * stage_bytes;
  uint64_t* full = s_full[wib];
  ChunkDesc* desc = s_desc[wib];
  const long long row_bytes = (long long)P.H * P.D * sizeof(T);
  const int cr = static_cast<int>(stage_bytes / row_bytes);
  const int* pref = ws_prefix(P);

  const long long V = __ldg(pref + P.n_streams);
  ChunkGen gen{};
  gen.V = V;
  gen.ctr = reinterpret_cast<unsigned long long*>(P.ws);
  gen.c_sidx = -1;
  gen.c_blk = -1;
  gen.sidx = 0;
  gen.claim_div = kClaimDiv * static_cast<int>(gridDim.x) * static_cast<int>(blockDim.x / 32);
  if (lane == 0) {
    claim(gen, 0);
    gen.it = gen.it1 = 0;  // empty: the first gen_next takes the claimed range
    for (int s = 0; s < nst; ++s) cs::mbar_init(&full[s], 1);
    cs::fence_mbar_init();
  }
  __syncwarp();

  bool more = true;
  auto issue = [&](int st) {
    const unsigned char* src = nullptr;
    const void* tab = nullptr;
    ChunkDesc d;
    if (!gen_next(P, pref, gen, cr, row_bytes, src, d, tab)) {
      desc[st].bytes = 0;
      cs::mbar_arrive(&full[st]);
      more = false;
      return;
    }
    desc[st] = d;
    if (d.rotate == 2) {  // partial in-place rotation: only the cos/sin table goes through the stage
      cs::mbar_arrive_expect_tx(&full[st], tab_bytes);
      cs::bulk_g2s(tabs + (size_t)st * tab_bytes, tab, tab_bytes, &full[st]);
      return;
    }
    cs::mbar_arrive_expect_tx(&full[st], d.bytes + (d.rotate ? tab_bytes : 0u));
    cs::bulk_g2s(stages + (size_t)st * stage_bytes, src, d.bytes, &full[st]);
    if (d.rotate) cs::bulk_g2s(tabs + (size_t)st * tab_bytes, tab, tab_bytes, &full[st]);
  };
  if (lane == 0)
    for (int st = 0; st < nst && more; ++st) issue(st);

  for (int q = 0;; ++q) {
    const int st = q % nst;
    cs::mbar_wait(&full[st], (q / nst) & 1);
    const ChunkDesc d = desc[st];
    if (d.bytes == 0) break;
    unsigned char* buf = stages + (size_t)st * stage_bytes;
    if (d.rotate == 2) {
      rotate_partial_global<T, TH, TD>(d.dst, reinterpret_cast<const float2*>(tabs + (size_t)st * tab_bytes), d.rows,
                                       P.H, P.D, P.rot_pairs, lane);
    } else if (d.rotate) {
      rotate_smem_warp<T, TH, TD>(buf, reinterpret_cast<const float2*>(tabs + (size_t)st * tab_bytes), d.rows, P.H,
                                  P.D, P.rot_pairs, lane);
      cs::fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk store
    }
    __syncwarp();
    if (lane == 0) {
      if (d.rotate != 2) cs::bulk_s2g(d.dst, buf, d.bytes);
      cs::bulk_commit();  // (an empty group for a partial item keeps the wait_group accounting per item)
      if (q >= 1 && more) {
        cs::bulk_wait_read<1>();  // the store of chunk q-1 has read its stage
        issue((q - 1) % nst);
      }
    }
    __syncwarp();
  }
  if (lane == 0) cs::bulk_wait_all<0>();
}

// ============================================================================================================
// Paged / in-place variant (NEXT-1; "maintains the previous window's KV cache resident in GPU memory and
// performs these updates in-place").  Rows live in a per-stream pool; slot maps give each token's row.
// REUSE: key rotated in place, value untouched.  ANCHOR: keeps its slot, rows overwritten from `refreshed`.
// NEW (new frames + prompt): the free slots in ascending order.
// ============================================================================================================
struct MoveEntry {
  int slot;  // pool row, -1 = none
  int src;   // -1: rotate the key in place (REUSE); >= 0: copy K and V from refreshed row src; -2: nothing
};

__device__ __forceinline__ MoveEntry* stream_moves(const KvParams& P, int s) {
  return reinterpret_cast<MoveEntry*>(stream_ws(P, s) + P.mv_off);
}

// exclusive scan of n ints in shared memory (in place), block-wide; returns the total
__device__ int block_exclusive_scan(int* a, int n) {
  __shared__ int s_part[33];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int b = tid * per, e = min(n, b + per);
  int sum = 0;
  for (int i = b; i < e; ++i) sum += a[i];
  // warp scan of the per-thread sums, then of the warp totals
  const int lane = tid & 31, warp = tid >> 5;
  int inc = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += u;
  }
  if (lane == 31) s_part[warp] = inc;
  __syncthreads();
  if (tid == 0) {
    int c = 0;
    for (int q = 0; q < (nt + 31) / 32; ++q) {
      const int v = s_part[q];
      s_part[q] = c;
      c += v;
    }
    s_part[32] = c;
  }
  __syncthreads();
  int run = s_part[warp] + inc - sum;
  for (int i = b; i < e; ++i) {
    const int v = a[i];
    a[i] = run;
    run += v;
  }
  __syncthreads();
  return s_part[32];
}

__global__ void __launch_bounds__(kPlanThreads) kv_plan_paged(const __grid_constant__ KvParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_n[cs::kMaxWindowPlusStride];
  __shared__ uint8_t s_t[cs::kMaxWindowPlusStride];
  __shared__ PlanSeg s_seg[kMaxSeg];
  __shared__ int s_pold[kMaxSeg];
  __shared__ int s_disp[kMaxSeg];
  __shared__ int s_nseg, s_ntotal, s_p0, s_n_old, s_r0, s_st, s_mis;
  __shared__ unsigned long long s_rot, s_cop;

  const int sidx = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int k = P.k, w = P.w, s = P.s;
  const int lo = k >= 1 ? (k - 1) * s : 0;
  const int ks = k * s, hi = ks + w;
  const int nfr = hi - lo;
  const int nw = P.nw;
  const int cw = static_cast<int>((P.cap + 31) / 32);  // words of the slot bitmap
  CS_PLAN_PHASE(0);
  uint32_t* s_mask = reinterpret_cast<uint32_t*>(smem);                 // [nfr][nw]
  uint32_t* s_used = s_mask + nfr * nw;                                 // [cw]
  int* s_free = reinterpret_cast<int*>(s_used + cw);                    // [cw + 1] free-slot prefix
  MoveEntry* s_mv = reinterpret_cast<MoveEntry*>(  // [max_tok] if P.mv_smem, 8-B aligned after s_free
      smem + ((static_cast<size_t>(nfr * nw + 2 * cw + 1) * 4 + 7) & ~static_cast<size_t>(7)));

  {  // the window's masks: up to 8 words per thread in flight at once
    constexpr int kM = 8;
    for (int e0 = tid; e0 < nfr * nw; e0 += kM * blockDim.x) {
      uint32_t v[kM];
#pragma unroll
      for (int u = 0; u < kM; ++u) {
        const int e = e0 + u * blockDim.x;
        const int fi = e / nw, t = e - fi * nw;
        v[u] = e < nfr * nw ? __ldg(P.mring + ((long long)sidx * P.ring + ((lo + fi) % P.ring)) * nw + t) : 0u;
      }
#pragma unroll
      for (int u = 0; u < kM; ++u)
        if (e0 + u * blockDim.x < nfr * nw) s_mask[e0 + u * blockDim.x] = v[u];
    }
  }
  for (int fi = tid; fi < nfr; fi += blockDim.x) s_t[fi] = __ldg(P.tring + (long long)sidx * P.ring + ((lo + fi) % P.ring));
  for (int i = tid; i < cw; i += blockDim.x) s_used[i] = 0u;
  if (tid == 0) {
    s_rot = 0ull;
    s_cop = 0ull;
    s_st = 0;
  }
  __syncthreads();
  if (P.G == 2 && P.grid_w == 32 && (P.grid_h & 1) == 0 && P.grid_h <= 64) {
    // 2x2 groups of a 32-wide grid: word r = patch row r; a group row's kept groups = popc of the OR of its two
    // words folded onto even bits.  One lane per group row, one warp per frame.
    const int ngr = P.grid_h / 2;
    for (int fi = warp; fi < nfr; fi += nwarp) {
      int n = 0;
      for (int gr = lane; gr < ngr; gr += 32) {
        const uint32_t x = s_mask[fi * nw + 2 * gr] | s_mask[fi * nw + 2 * gr + 1];
        n += __popc((x | (x >> 1)) & 0x55555555u);
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) n += __shfl_xor_sync(0xffffffffu, n, d);
      if (lane == 0) s_n[fi] = n;
    }
  } else {
    for (int fi = warp; fi < nfr; fi += nwarp) {
      int n = 0;
      for (int base = 0; base < P.ngroups; base += 32) {
        const int q = base + lane;
        const bool kept = q < P.ngroups && cs::group_kept(s_mask + fi * nw, q, P.ngc, P.G, P.grid_w);
        n += __popc(__ballot_sync(0xffffffffu, kept));
      }
      if (lane == 0) s_n[fi] = n;
    }
  }
  __syncthreads();
  // (cos, sin) of R(dp), dp = -(tokens of the s dropped frames): warps 1.. compute it while thread 0 builds the
  // segment table below (64 double-precision sincos calls were the longest phase of this kernel, measured)
  float2* cs_tab = reinterpret_cast<float2*>(stream_ws(P, sidx) + sizeof(KvHdr) + sizeof(KvSeg) * P.max_seg);
  if (warp >= 1) {
    long long drop = 0;
    if (k >= 1)
      for (int f = lo; f < ks; ++f) drop += s_n[f - lo];
    for (int i = tid - 32; i < P.D / 2; i += blockDim.x - 32) {
      // position change of pair i: the sequence-index change (1-D RoPE) or its section's component (M-RoPE)
      const long long delta = P.rope_mode == CS_ROPE_MROPE ? (i < P.mrope_t ? P.mrope_dt : 0ll) : -drop;
      double sn, cs;
      sincos(static_cast<double>(delta) * P.inv_freq[i], &sn, &cs);
      cs_tab[i] = make_float2(__double2float_rn(cs), __double2float_rn(sn));
    }
  }
  CS_PLAN_PHASE(1);

  if (tid == 0) {
    long long drop = 0, n_old = 0;
    if (k >= 1) {
      for (int f = lo; f < ks; ++f) drop += s_n[f - lo];
      for (int f = lo; f < lo + w; ++f) n_old += s_n[f - lo];
      n_old += P.n_prompt;
    }
    const int new_first = (k - 1) * s + w;
    long long pnew = 0, rrow = 0, n_reuse = 0, n_anchor = 0, n_new = 0, p0 = -1, r0 = 0;
    int nseg = 0;
    for (int f = ks; f < hi; ++f) {
      const int n = s_n[f - lo];
      int disp, pold;
      if (k == 0 || f >= new_first) {
        disp = CS_DISP_NEW;
        pold = -1;
      } else {
        disp = (s_t[f - lo] != CS_FRAME_P || f == ks) ? CS_DISP_ANCHOR : CS_DISP_REUSE;
        pold = static_cast<int>(drop + pnew);
      }
      if (disp == CS_DISP_NEW && p0 < 0) {
        p0 = pnew;
        r0 = rrow;
      }
      s_seg[nseg].p_new = static_cast<int>(pnew);
      s_seg[nseg].len = n;
      s_seg[nseg].kind = disp;
      s_seg[nseg].src = static_cast<int>(rrow);
      s_pold[nseg] = pold;
      s_disp[nseg] = disp;
      ++nseg;
      if (disp != CS_DISP_REUSE) rrow += n;
      if (disp == CS_DISP_REUSE) n_reuse += n;
      else if (disp == CS_DISP_ANCHOR) n_anchor += n;
      else n_new += n;
      pnew += n;
    }
    const long long n_visual = pnew;
    if (p0 < 0) {
      p0 = pnew;
      r0 = rrow;
    }
    s_seg[nseg].p_new = static_cast<int>(pnew);
    s_seg[nseg].len = P.n_prompt;
    s_seg[nseg].kind = CS_DISP_NEW;
    s_seg[nseg].src = static_cast<int>(rrow);
    s_pold[nseg] = -1;
    s_disp[nseg] = CS_DISP_NEW;
    ++nseg;
    n_new += P.n_prompt;
    const long long n_total = n_visual + P.n_prompt;
    s_nseg = nseg;
    s_ntotal = static_cast<int>(n_total);
    s_p0 = static_cast<int>(p0);
    s_r0 = static_cast<int>(r0);
    s_n_old = static_cast<int>(n_old);
    int* nt = P.n_tokens + (long long)sidx * 4;
    nt[0] = static_cast<int>(n_visual);
    nt[1] = static_cast<int>(n_reuse);
    nt[2] = static_cast<int>(n_anchor);
    nt[3] = static_cast<int>(n_new);
    int st = 0;
    if (n_total > P.token_cap || n_total > P.slot_cap) st |= CS_STATUS_CAPACITY;
    s_mis = kv_misaligned(P, sidx) ? 1 : 0;
    if (s_mis) st |= CS_STATUS_MISALIGNED;
    s_st = st;
    KvHdr* hdr = reinterpret_cast<KvHdr*>(stream_ws(P, sidx));
    hdr->n_rows = static_cast<int>(n_total < P.max_tok ? n_total : P.max_tok);
    hdr->n_seg = nseg;
    hdr->dp = static_cast<int>(-drop);
    hdr->pad = 0;
    cs::atomic_add_u64(&P.counters[CS_CNT_TOK_REUSE], static_cast<unsigned long long>(n_reuse));
    cs::atomic_add_u64(&P.counters[CS_CNT_TOK_ANCHOR], static_cast<unsigned long long>(n_anchor));
    cs::atomic_add_u64(&P.counters[CS_CNT_TOK_NEW], static_cast<unsigned long long>(n_new));
    cs::atomic_add_u64(&P.counters[CS_CNT_STREAM_STEPS], 1ull);
  }
  __syncthreads();

  CS_PLAN_PHASE(2);
  const int nseg = s_nseg, n_total = s_ntotal, p0 = s_p0, n_old = s_n_old;
  MoveEntry* mv = stream_moves(P, sidx);
  int32_t* slot_new = P.slot_new + (long long)sidx * P.slot_cap;
  uint8_t* dsp = P.disposition + (long long)sidx * P.token_cap;
  int32_t* po_out = P.p_old + (long long)sidx * P.token_cap;
  int st_local = 0;
  unsigned long long rot = 0, cop = 0;
  // ---- surviving tokens (REUSE, ANCHOR) keep their slots; index outputs of every token ---------------------
  for (int i = warp; i < nseg; i += nwarp) {
    const PlanSeg sg = s_seg[i];
    const int d = s_disp[i], pold = s_pold[i];
    // the previous window's slots of 4 x 32 tokens are loaded before any is used (one latency per batch)
    constexpr int kU = 4;
    for (int t0 = lane; t0 < sg.len; t0 += 32 * kU) {
      int slv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int t = t0 + 32 * u;
        const long long q = (long long)pold + t;
        slv[u] = (d != CS_DISP_NEW && t < sg.len && q < P.slot_cap && q < n_old)
                     ? __ldg(P.slot_old + (long long)sidx * P.slot_cap + q) : -1;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int t = t0 + 32 * u;
        if (t >= sg.len) break;
        const long long p = (long long)sg.p_new + t;
        if (p < P.token_cap) {
          dsp[p] = static_cast<uint8_t>(d);
          po_out[p] = d == CS_DISP_NEW ? -1 : pold + t;
        }
        if (d == CS_DISP_NEW) continue;
        int sl = slv[u];
        if (sl < 0 || sl >= P.cap) {
          sl = -1;
          st_local |= CS_STATUS_ORIGIN;
        } else {
          atomicOr(&s_used[sl >> 5], 1u << (sl & 31));
        }
        if (p < P.slot_cap) slot_new[p] = sl;
        MoveEntry me;
        me.slot = sl;
        if (d == CS_DISP_REUSE) {
          me.src = sl >= 0 ? -1 : -2;
          rot += sl >= 0;
        } else {
          const long long r = (long long)sg.src + t;
          const bool ok = P.has_refreshed && sl >= 0 && r < P.rcap;
          if (P.has_refreshed && sl >= 0 && r >= P.rcap) st_local |= CS_STATUS_CAPACITY;
          me.src = ok ? static_cast<int>(r) : -2;
          cop += ok;
        }
        if (p < P.max_tok) {
          mv[p] = me;
          if (P.mv_smem) s_mv[p] = me;
        }
      }
    }
  }
  __syncthreads();
  CS_PLAN_PHASE(3);
  // ---- free slots (not held by a survivor), ascending -> NEW tokens in p_new order -------------------------
  for (int i = tid; i < cw; i += blockDim.x) {
    uint32_t valid = 0xffffffffu;
    if ((long long)(i + 1) * 32 > P.cap) valid = (1u << (P.cap - (long long)i * 32)) - 1u;
    s_free[i] = __popc(~s_used[i] & valid);
  }
  __syncthreads();
  const int total_free = block_exclusive_scan(s_free, cw);
  if (tid == 0) s_free[cw] = total_free;
  __syncthreads();
  CS_PLAN_PHASE(4);
  for (int p = p0 + tid; p < n_total; p += blockDim.x) {
    const int i = p - p0;  // index among the NEW tokens
    int sl = -1;
    if (i < total_free) {
      int a = 0, b = cw;  // s_free[a] <= i < s_free[b]
      while (b - a > 1) {
        const int m = (a + b) >> 1;
        if (s_free[m] <= i) a = m; else b = m;
      }
      const uint32_t fr = ~s_used[a];
      const int j = i - s_free[a];
      sl = a * 32 + static_cast<int>(__fns(fr, 0, j + 1));
    } else {
      st_local |= CS_STATUS_CAPACITY;
    }
    if (p < P.slot_cap) slot_new[p] = sl;
    const long long r = (long long)s_r0 + i;
    const bool ok = P.has_refreshed && sl >= 0 && r < P.rcap;
    if (P.has_refreshed && sl >= 0 && r >= P.rcap) st_local |= CS_STATUS_CAPACITY;
    MoveEntry me;
    me.slot = sl;
    me.src = ok ? static_cast<int>(r) : -2;
    cop += ok;
    if (p < P.max_tok) {
        mv[p] = me;
        if (P.mv_smem) s_mv[p] = me;
      }
  }
  // ---- runs for the bulk-copy gather: maximal token ranges with one action and consecutive slots (and
  //      consecutive refreshed rows for copies); skipped tokens form SKIP runs so runs tile [0, n_total) -------
  __syncthreads();  // move entries of every token written
  CS_PLAN_PHASE(5);
  {
    __shared__ int s_cnt[kPlanThreads];
    const int nmv = min(n_total, P.max_tok);
    const int per = (nmv + blockDim.x - 1) / blockDim.x;
    const int b = tid * per, e = min(nmv, b + per);
    auto cls = [](const MoveEntry& m) { return (m.slot < 0 || m.src == -2) ? 0 : (m.src == -1 ? 1 : 2); };
    // the thread's entries are read in batches of kB (+ the one before), all loads in flight at once: a run
    // start depends on the entry and its predecessor only
    constexpr int kB = 8;
    auto batch = [&](int p0, MoveEntry (&m)[kB + 1]) {
#pragma unroll
      for (int u = 0; u <= kB; ++u) {
        const int p = p0 - 1 + u;
        m[u] = (p >= 0 && p < e) ? (P.mv_smem ? s_mv[p] : mv[p]) : MoveEntry{-1, -2};
      }
    };
    auto is_start = [&](const MoveEntry& a, const MoveEntry& c, int p) {
      if (p == 0) return true;
      const int ca = cls(a), cc = cls(c);
      if (ca != cc) return true;
      if (cc == 0) return false;
      if (c.slot != a.slot + 1) return true;
      return cc == 2 && c.src != a.src + 1;
    };
    int cnt = 0;
    for (int p0 = b; p0 < e; p0 += kB) {
      MoveEntry m[kB + 1];
      batch(p0, m);
#pragma unroll
      for (int u = 1; u <= kB; ++u)
        if (p0 - 1 + u < e) cnt += is_start(m[u - 1], m[u], p0 - 1 + u) ? 1 : 0;
    }
    s_cnt[tid] = cnt;
    __syncthreads();
    const int nruns = block_exclusive_scan(s_cnt, blockDim.x);
    CS_PLAN_PHASE(6);
    KvSeg* runs = reinterpret_cast<KvSeg*>(stream_ws(P, sidx) + sizeof(KvHdr));
    int idx = s_cnt[tid];
    for (int p0 = b; p0 < e; p0 += kB) {
      MoveEntry m[kB + 1];
      batch(p0, m);
#pragma unroll
      for (int u = 1; u <= kB; ++u) {
        const int p = p0 - 1 + u;
        if (p >= e || !is_start(m[u - 1], m[u], p)) continue;
        const int c = cls(m[u]);
        KvSeg r;
        r.p_new = p;
        r.len = 0;
        r.kind = c == 0 ? SEG_SKIP : (c == 1 ? SEG_REUSE : SEG_COPY);
        r.src = c == 2 ? m[u].src : m[u].slot;
        r.dst = m[u].slot;
        runs[idx++] = r;
      }
    }
    __syncthreads();
    for (int i = tid; i < nruns; i += blockDim.x) runs[i].len = (i + 1 < nruns ? runs[i + 1].p_new : nmv) - runs[i].p_new;
    if (tid == 0) reinterpret_cast<KvHdr*>(stream_ws(P, sidx))->n_seg = s_mis ? 0 : nruns;
  }
  CS_PLAN_PHASE(7);
  // per-warp reductions first: one shared atomic per warp instead of one per thread
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    st_local |= __shfl_xor_sync(0xffffffffu, st_local, d);
    rot += __shfl_xor_sync(0xffffffffu, rot, d);
    cop += __shfl_xor_sync(0xffffffffu, cop, d);
  }
  if (lane == 0) {
    if (st_local) atomicOr(&s_st, st_local);
    if (rot) atomicAdd(&s_rot, rot);
    if (cop) atomicAdd(&s_cop, cop);
  }
  __syncthreads();
  if (tid == 0 && s_mis) {  // misaligned buffers: no row of this stream moves (kv_prefix then counts no item)
    KvHdr* hdr = reinterpret_cast<KvHdr*>(stream_ws(P, sidx));
    hdr->n_rows = 0;
    hdr->n_seg = 0;
    s_rot = s_cop = 0;
  }
  if (tid == 0) {
    cs::atomic_or_status(P.status, s_st);
    const unsigned long long rowb = (unsigned long long)(P.H * P.D * P.esz);
    // REUSE: the rotated pairs of the key rows (M-RoPE: the temporal section only); refreshed rows: K and V
    const unsigned long long rotb = (unsigned long long)P.H * 2ull * P.rot_pairs * P.esz;
    cs::atomic_add_u64(&P.counters[CS_CNT_BYTES_KV], (s_rot * P.L * rotb + s_cop * P.L * 2ull * rowb) * 2ull);
  }
  CS_PLAN_PHASE(8);
}

// One token per warp iteration: REUSE -> rotate the key rows of all layers in place; copy -> K and V rows of all
// layers from the refreshed buffer.  Layers are unrolled by 4 for memory-level parallelism.
template <typename T, int TH, int TD>
__global__ void __launch_bounds__(kGatherThreads) kv_gather_paged(const __grid_constant__ KvParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int VE = Vec<T>::N;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int H = TH > 0 ? TH : P.H;
  const int D = TD > 0 ? TD : P.D;
  const int half = D / 2;
  const int rowb = H * D * static_cast<int>(sizeof(T));
  float2* tab = reinterpret_cast<float2*>(smem) + wib * (P.D / 2);  // this warp's (cos, sin) table
  const int* pref = ws_prefix(P);
  const long long V = __ldg(pref + P.n_streams);
  const long long nwarps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  const long long gw = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + wib;
  long long it = V * gw / nwarps;
  const long long it1 = V * (gw + 1) / nwarps;
  if (it >= it1) return;
  int sidx = 0;
  {
    int lo = 0, hi = P.n_streams;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(pref + mid) <= it) lo = mid; else hi = mid;
    }
    sidx = lo;
  }
  int cur = -1;
  const long long plane = P.cap * rowb;       // bytes of one (layer, K|V) plane of the pool
  const long long rplane = P.rcap * rowb;     // ... of the refreshed buffer
  unsigned char* pl = nullptr;
  const unsigned char* rf = nullptr;
  const MoveEntry* mv = nullptr;
  for (; it < it1; ++it) {
    while (__ldg(pref + sidx + 1) <= it) ++sidx;
    if (sidx != cur) {
      cur = sidx;
      pl = static_cast<unsigned char*>(P.pool[sidx]);
      rf = P.has_refreshed ? static_cast<const unsigned char*>(P.refreshed[sidx]) : nullptr;
      mv = stream_moves(P, sidx);
      const float2* g = reinterpret_cast<const float2*>(stream_ws(P, sidx) + sizeof(KvHdr) + sizeof(KvSeg) * P.max_seg);
      __syncwarp();
      for (int i = lane; i < P.D / 2; i += 32) tab[i] = g[i];
      __syncwarp();
    }
    const int p = static_cast<int>(it - __ldg(pref + sidx));
    const MoveEntry me = mv[p];
    if (me.src == -2 || me.slot < 0) continue;
    if (me.src == -1) {
      // Eq. 5 in place on the key rows (plane 2l) of every layer
      unsigned char* base = pl + (long long)me.slot * rowb;
      if (P.vec_rot && P.vec_copy) {
        const int vphr = P.rot_pairs / VE;  // rotated vectors per half-head (M-RoPE: the temporal section)
        const int total = H * vphr;         // units per row
        for (int l0 = 0; l0 < P.L; l0 += 4) {
          for (int e = lane; e < total; e += 32) {
            const int h = e / vphr, j = e - h * vphr;
            const int off1 = (h * D + j * VE) * static_cast<int>(sizeof(T));
            const int off2 = off1 + half * static_cast<int>(sizeof(T));
            uint4 a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (l0 + u < P.L) {
                unsigned char* r = base + (long long)(2 * (l0 + u)) * plane;
                a[u] = *reinterpret_cast<const uint4*>(r + off1);
                b[u] = *reinterpret_cast<const uint4*>(r + off2);
              }
            }
            float c[VE], sn[VE];
#pragma unroll
            for (int v = 0; v < VE; ++v) {
              const float2 cs2 = tab[j * VE + v];
              c[v] = cs2.x;
              sn[v] = cs2.y;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (l0 + u < P.L) {
                if constexpr (sizeof(T) == 2) rot8_bf16_pack(a[u], b[u], c, sn);
                else rot4_f32(a[u], b[u], c, sn);
                unsigned char* r = base + (long long)(2 * (l0 + u)) * plane;
                *reinterpret_cast<uint4*>(r + off1) = a[u];
                *reinterpret_cast<uint4*>(r + off2) = b[u];
              }
            }
          }
        }
      } else {
        for (int l = 0; l < P.L; ++l) {
          T* r = reinterpret_cast<T*>(base + (long long)(2 * l) * plane);
          for (int e = lane; e < H * P.rot_pairs; e += 32) {
            const int h = e / P.rot_pairs, i = e - h * P.rot_pairs;
            float x1, x2;
            if constexpr (sizeof(T) == 2) {
              x1 = __uint_as_float(static_cast<uint32_t>(r[h * D + i]) << 16);
              x2 = __uint_as_float(static_cast<uint32_t>(r[h * D + i + half]) << 16);
            } else {
              x1 = r[h * D + i];
              x2 = r[h * D + i + half];
            }
            const float2 cs2 = tab[i];
            const float y1 = __fmaf_rn(x1, cs2.x, -__fmul_rn(x2, cs2.y));
            const float y2 = __fmaf_rn(x2, cs2.x, __fmul_rn(x1, cs2.y));
            if constexpr (sizeof(T) == 2) {
              r[h * D + i] = static_cast<T>(cs::f32_to_bf16_rne(y1));
              r[h * D + i + half] = static_cast<T>(cs::f32_to_bf16_rne(y2));
            } else {
              r[h * D + i] = y1;
              r[h * D + i + half] = y2;
            }
          }
        }
      }
    } else {
      // refreshed rows -> slot, K and V of every layer
      unsigned char* dst = pl + (long long)me.slot * rowb;
      const unsigned char* src = rf + (long long)me.src * rowb;
      if (P.vec_copy) {
        const int n16 = rowb / 16;
        for (int l0 = 0; l0 < 2 * P.L; l0 += 4) {
          for (int e = lane; e < n16; e += 32) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (l0 + u < 2 * P.L) v[u] = cs::ld_nc_v4(src + (long long)(l0 + u) * rplane + e * 16);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (l0 + u < 2 * P.L) *reinterpret_cast<uint4*>(dst + (long long)(l0 + u) * plane + e * 16) = v[u];
          }
        }
      } else {
        for (int l = 0; l < 2 * P.L; ++l) {
          const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src + (long long)l * rplane);
          uint32_t* d4 = reinterpret_cast<uint32_t*>(dst + (long long)l * plane);
          for (int e = lane; e < rowb / 4; e += 32) d4[e] = s4[e];
        }
      }
    }
  }
}


// Geometry of the TMA ring gather: warps per CTA x stages x 8 KB stages (one CTA per SM).  8 warps with as many
// stages (<= 6) as fit; a row set whose per-stage cos/sin table leaves fewer than 3 stages per warp (head_dim > 256)
// halves the warps until 3 fit.  Computed before ANY kernel of the call is enqueued: a configuration no geometry
// serves takes the register-path gather instead (never a failure after the plan kernel ran, codecsight.h:24).
struct TmaGeom {
  int warps, nst;
  unsigned stage_bytes, tab_bytes;
};

static bool tma_geometry(const KvParams& P, TmaGeom* t) {
  const long long row_bytes = static_cast<long long>(P.H) * P.D * P.esz;
  if (!(P.vec_rot && P.vec_copy && row_bytes <= kTmaChunk && (P.D % 4) == 0)) return false;
  t->stage_bytes = static_cast<unsigned>(kTmaChunk);  // >= one row, so every chunk carries >= 1 row
  t->tab_bytes = static_cast<unsigned>(((8 * (P.D / 2)) + 127) & ~127);
  for (int warps = kWarpsPerGather; warps >= 2; warps /= 2) {
    int nst = static_cast<int>((216u * 1024u) / (warps * (t->stage_bytes + t->tab_bytes)));
    if (nst > kMaxStages) nst = kMaxStages;
    if (nst >= 3) {
      t->warps = warps;
      t->nst = nst;
      return true;
    }
  }
  return false;
}

// Launch the TMA ring gather with a geometry from tma_geometry().
static int launch_gather_tma(const KvParams& P, const cs_kv_desc* kv, const TmaGeom& t, cudaStream_t stream) {
  const int warps = t.warps, nst = t.nst;
  const unsigned stage_bytes = t.stage_bytes, tab_bytes = t.tab_bytes;
  const size_t smem = static_cast<size_t>(warps) * nst * (stage_bytes + tab_bytes);
  const int grid = cs_num_sms();
  const bool qwen = kv->dtype == CS_BF16 && kv->kv_heads == 4 && kv->head_dim == 128;
  const void* fn = qwen ? reinterpret_cast<const void*>(kv_gather_tma<uint16_t, 4, 128>)
                        : (kv->dtype == CS_BF16 ? reinterpret_cast<const void*>(kv_gather_tma<uint16_t, 0, 0>)
                                                : reinterpret_cast<const void*>(kv_gather_tma<float, 0, 0>));
  const int slot = qwen ? 7 : (kv->dtype == CS_BF16 ? 8 : 9);
  if (cs_set_smem_attr(fn, slot, 220 * 1024)) return CS_ERR_CUDA;
  const int threads = warps * 32;
  if (qwen)
    kv_gather_tma<uint16_t, 4, 128><<<grid, threads, smem, stream>>>(P, nst, stage_bytes, tab_bytes);
  else if (kv->dtype == CS_BF16)
    kv_gather_tma<uint16_t, 0, 0><<<grid, threads, smem, stream>>>(P, nst, stage_bytes, tab_bytes);
  else
    kv_gather_tma<float, 0, 0><<<grid, threads, smem, stream>>>(P, nst, stage_bytes, tab_bytes);
  return CS_OK;
}

}  // namespace

size_t cs_kv_workspace_bytes(const cs_kv_desc* kv, const cs_window* win, int32_t n_streams) {
  const size_t max_seg = static_cast<size_t>(win->window) + 1;
  size_t stride = sizeof(KvHdr) + sizeof(KvSeg) * max_seg + 8 * static_cast<size_t>(kv->head_dim / 2);
  stride = (stride + 15) & ~static_cast<size_t>(15);
  return 16 + stride * static_cast<size_t>(n_streams) + 4 * (static_cast<size_t>(n_streams) + 1);
}

static void fill_params(KvParams& P, const cs_grid* g, const cs_kv_desc* kv, const cs_window* win,
                        int32_t n_streams, const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring,
                        const void* const* old_cache, void* const* new_cache, const void* const* refreshed,
                        int64_t token_cap, uint8_t* disposition, int32_t* p_old, int32_t* n_tokens, void* workspace,
                        unsigned long long* counters, int32_t* status) {
  P.grid_w = g->grid_w;
  P.grid_h = g->grid_h;
  P.G = g->group;
  P.nw = (g->grid_w * g->grid_h + 31) / 32;
  P.ngc = g->grid_w / g->group;
  P.ngroups = (g->grid_h / g->group) * P.ngc;
  P.w = win->window;
  P.s = win->stride;
  P.k = win->step;
  P.ring = win->ring_frames;
  P.L = kv->layers;
  P.H = kv->kv_heads;
  P.D = kv->head_dim;
  P.esz = kv->dtype == CS_BF16 ? 2 : 4;
  P.cap = kv->capacity;
  P.rcap = kv->refresh_capacity;
  P.token_cap = token_cap;
  P.n_prompt = kv->n_prompt;
  P.n_streams = n_streams;
  P.max_seg = win->window + 1;
  P.has_refreshed = refreshed != nullptr;
  {
    const int ve = 16 / P.esz;
    P.rot_pairs = kv->rope_mode == CS_ROPE_MROPE ? kv->mrope_section[0] : kv->head_dim / 2;
    P.vec_rot = ((P.D / 2) % ve) == 0 && (P.rot_pairs % ve) == 0;
    P.vec_copy = ((static_cast<long long>(P.H) * P.D * P.esz) % 16) == 0;
  }
  const size_t max_seg = static_cast<size_t>(P.max_seg);
  size_t stride = sizeof(KvHdr) + sizeof(KvSeg) * max_seg + 8 * static_cast<size_t>(kv->head_dim / 2);
  P.ws_stride = static_cast<long long>((stride + 15) & ~static_cast<size_t>(15));
  P.mring = keep_mask_ring;
  P.tring = frame_type_ring;
  P.old_cache = old_cache;
  P.new_cache = new_cache;
  P.refreshed = refreshed;
  P.disposition = disposition;
  P.p_old = p_old;
  P.n_tokens = n_tokens;
  P.ws = static_cast<unsigned char*>(workspace);
  P.counters = counters;
  P.status = status;
  for (int i = 0; i < kv->head_dim / 2; ++i)
    P.inv_freq[i] = pow(kv->rope_base, -2.0 * static_cast<double>(i) / static_cast<double>(kv->head_dim));
  P.rope_mode = kv->rope_mode;
  P.mrope_t = kv->mrope_section[0];
  P.mrope_dt = -static_cast<long long>(win->stride) * kv->t_per_frame;

}

int cs_launch_kv_refresh(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, int32_t n_streams,
                         const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring,
                         const void* const* old_cache, void* const* new_cache, const void* const* refreshed,
                         int64_t token_cap, uint8_t* disposition, int32_t* p_old, int32_t* n_tokens,
                         void* workspace, size_t workspace_bytes, unsigned long long* counters, int32_t* status,
                         cudaStream_t stream) {
  (void)workspace_bytes;
  KvParams P{};
  fill_params(P, g, kv, win, n_streams, keep_mask_ring, frame_type_ring, old_cache, new_cache, refreshed, token_cap,
              disposition, p_old, n_tokens, workspace, counters, status);
  const size_t max_seg = static_cast<size_t>(P.max_seg);
  const int lo = win->step >= 1 ? (win->step - 1) * win->stride : 0;
  const int nfr = win->step * win->stride + win->window - lo;
  const size_t plan_smem = static_cast<size_t>(nfr) * P.nw * 4;
  TmaGeom geom{};
  const bool tma_ok = tma_geometry(P, &geom);
  if (cs_set_smem_attr(reinterpret_cast<const void*>(kv_plan), 3, 128 * 1024)) return CS_ERR_CUDA;
  kv_plan<<<n_streams, kPlanThreads, plan_smem, stream>>>(P);
  if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;

  const int sms = cs_num_sms();
  kv_prefix<<<1, 1024, 0, stream>>>(P);
  if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
  if (tma_ok) {
    const int rc = launch_gather_tma(P, kv, geom, stream);
    if (rc) return rc;
  } else {
    const size_t gsmem = 8 * static_cast<size_t>((n_streams + 2) & ~1) + sizeof(KvSeg) * max_seg +
                         8 * static_cast<size_t>(kv->head_dim / 2);
    const int grid = sms * 4;
    const void* fn = kv->dtype == CS_BF16 ? reinterpret_cast<const void*>(kv_gather_ldg<uint16_t, 0, 0>)
                                          : reinterpret_cast<const void*>(kv_gather_ldg<float, 0, 0>);
    if (cs_set_smem_attr(fn, kv->dtype == CS_BF16 ? 5 : 6, 160 * 1024)) return CS_ERR_CUDA;
    if (kv->dtype == CS_BF16) kv_gather_ldg<uint16_t, 0, 0><<<grid, kGatherThreads, gsmem, stream>>>(P);
    else kv_gather_ldg<float, 0, 0><<<grid, kGatherThreads, gsmem, stream>>>(P);
  }
  if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
  return CS_OK;
}

static size_t paged_stride(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, long long* mv_off,
                           int* max_tok) {
  const long long groups = static_cast<long long>(g->grid_w / g->group) * (g->grid_h / g->group);
  const long long mt = static_cast<long long>(win->window) * groups + kv->n_prompt;
  size_t off = sizeof(KvHdr) + sizeof(KvSeg) * (static_cast<size_t>(mt) + 1) +
               8 * static_cast<size_t>(kv->head_dim / 2);
  off = (off + 15) & ~static_cast<size_t>(15);
  if (mv_off) *mv_off = static_cast<long long>(off);
  if (max_tok) *max_tok = static_cast<int>(mt);
  size_t stride = off + sizeof(MoveEntry) * static_cast<size_t>(mt);
  return (stride + 15) & ~static_cast<size_t>(15);
}

size_t cs_kv_paged_workspace_bytes(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win,
                                   int32_t n_streams) {
  const size_t stride = paged_stride(g, kv, win, nullptr, nullptr);
  return 16 + stride * static_cast<size_t>(n_streams) + 4 * (static_cast<size_t>(n_streams) + 1);
}

int cs_launch_kv_refresh_paged(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, int32_t n_streams,
                               const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring, void* const* pool,
                               const int32_t* slot_old, int32_t* slot_new, int64_t slot_cap,
                               const void* const* refreshed, int64_t token_cap, uint8_t* disposition,
                               int32_t* p_old, int32_t* n_tokens, void* workspace, unsigned long long* counters,
                               int32_t* status, cudaStream_t stream) {
  KvParams P{};
  fill_params(P, g, kv, win, n_streams, keep_mask_ring, frame_type_ring, nullptr, nullptr, refreshed, token_cap,
              disposition, p_old, n_tokens, workspace, counters, status);
  P.pool = pool;
  P.slot_old = slot_old;
  P.slot_new = slot_new;
  P.slot_cap = slot_cap;
  P.ws_stride = static_cast<long long>(paged_stride(g, kv, win, &P.mv_off, &P.max_tok));
  P.max_seg = P.max_tok + 1;  // run list capacity (also locates the cos/sin table)
  P.paged = 1;
  P.partial_mode = 0;
  P.old_cache = pool;  // REUSE runs read and write the same pool rows
  P.new_cache = pool;
  TmaGeom geom{};
  const bool tma_ok = tma_geometry(P, &geom);
  P.partial_mode = (tma_ok && P.rot_pairs < P.D / 2) ? 1 : 0;
  P.prefix_mode = tma_ok ? 0 : 1;
  const int lo = win->step >= 1 ? (win->step - 1) * win->stride : 0;
  const int nfr = win->step * win->stride + win->window - lo;
  const long long cw = (kv->capacity + 31) / 32;
  size_t plan_smem = static_cast<size_t>(nfr) * P.nw * 4 + static_cast<size_t>(cw) * 4 +
                     static_cast<size_t>(cw + 1) * 4;
  plan_smem = (plan_smem + 7) & ~static_cast<size_t>(7);
  if (plan_smem > kPlanSmem) return CS_ERR_UNSUPPORTED;
  // the move list staged in shared memory too when it fits (the runs pass then reads it there, not from L2)
  const size_t mv_bytes = static_cast<size_t>(P.max_tok) * sizeof(MoveEntry);
  P.mv_smem = plan_smem + mv_bytes <= kPlanSmem ? 1 : 0;
  if (P.mv_smem) plan_smem += mv_bytes;
  if (cs_set_smem_attr(reinterpret_cast<const void*>(kv_plan_paged), 10, kPlanSmem)) return CS_ERR_CUDA;
  kv_plan_paged<<<n_streams, kPlanThreads, plan_smem, stream>>>(P);
  if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
  kv_prefix<<<1, 1024, 0, stream>>>(P);
  if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
  if (tma_ok) {
    const int rc = launch_gather_tma(P, kv, geom, stream);
    if (rc) return rc;
  } else {
    const int grid = cs_num_sms() * 4;
    const size_t gsmem = static_cast<size_t>(kGatherThreads / 32) * 8 * static_cast<size_t>(kv->head_dim / 2);
    if (kv->dtype == CS_BF16) kv_gather_paged<uint16_t, 0, 0><<<grid, kGatherThreads, gsmem, stream>>>(P);
    else kv_gather_paged<float, 0, 0><<<grid, kGatherThreads, gsmem, stream>>>(P);
  }
  if (cudaGetLastError() != cudaSuccess) return CS_ERR_CUDA;
  return CS_OK;
}

#ifdef CS_PLAN_TIMING
extern "C" int codecsight_debug_plan_phase(unsigned long long* host, int n_ctas) {
  if (n_ctas > 4096) n_ctas = 4096;
  return cudaMemcpyFromSymbol(host, g_cs_plan_phase, sizeof(unsigned long long) * 10 * n_ctas) == cudaSuccess ? 0 : -1;
}
#endif
