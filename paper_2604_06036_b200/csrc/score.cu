// score.cu — codecsight_score_patches on sm_100a.
//
// Computes, per P-frame, the patch motion score M(i) = V(i) + alpha R(i) (Eq. 1-3), the
// dynamic mask M(i) >= tau (Eq. 4), the GOP-accumulated active set and the group-complete
// keep mask.  Readings: DESIGN.md Q1-Q13.
//
// Layout of the work: one thread-block CLUSTER per camera stream, one CTA per (group of) new frame(s) of that
// stream.  Each CTA streams its frames' macroblock records from HBM into shared memory with the TMA bulk-copy
// engine (cp.async.bulk, mbarrier-tracked, NSTAGE-deep ring of MB-row chunks), reduces MB -> patch with a
// separable two-pass scheme (MB row -> patch column partial max / area-weighted SAD sums in smem, then patch
// rows), and ballots the per-patch threshold decisions into 32-bit words.  The GOP accumulation is a segmented
// OR-scan over the stream's frames in time order: after a cluster barrier every CTA reads the dynamic words of
// the earlier frames of its stream straight out of the other CTAs' shared memory (DSMEM).
//
// Parity-relevant arithmetic is spelled out with IEEE intrinsics (no fast-math): the sqrt is correctly rounded,
// R is one correctly rounded double division of two exact integers, M is one fp32 fma.
#include <cooperative_groups.h>
#include <math_constants.h>

#include "cs_internal.cuh"
#include "group_ring.cuh"

namespace cg = cooperative_groups;

namespace {

#ifndef CS_FUSED_SMEM_KB
#define CS_FUSED_SMEM_KB 68u  // fused kernel dynamic shared memory per CTA (3 CTAs per SM; registers allow no 4th)
#endif
constexpr int kThreads = 256;
constexpr uint32_t kIntraSq = 0xffffffffu;  // > any |mv|^2 (<= 2^31)

struct ScoreParams {
  int src_w, src_h, mb, mb_cols, mb_rows, grid_w, grid_h, G;
  int np, nw;
  float tau, alpha;
  double denom;  // mb^2 * 255 * src_w * src_h (exact)
  int n_streams, n_frames, fpc, cluster;
  long long frame_stride;
  long long type_stride;  // row stride of frame_type (frame_stride unless the types come from their own array)
  int pdl;                // chained call launched as a programmatic dependent of the preceding one (see below)
  unsigned* gop_ready;    // chain: [n_streams] generation of each stream's GOP state
  unsigned* chain_done;   // chain: [depth] per g mod depth, generation + 1 of the last completed call of that class
  unsigned chain_depth;   // chain: output buffer sets the calls rotate (call g writes what call g - depth wrote)
  unsigned generation;    // chain: this call's index g
  int phase_slot;         // CS_PHASE_TIMING builds only
  int use_bulk, chunk_rows, n_chunks, nstage;
  unsigned row_bytes, chunk_alloc;
  int want_score;
  int use_r;     // alpha != 0: R(i) is needed (with alpha == 0, M = fma(0, R, V) = V exactly, R is skipped)
  int gw_shift;  // log2(grid_w) when grid_w is a power of two, else -1
  unsigned off_col, off_row;  // smem: per patch column (i0, i1), per patch row (j0, j1)
  const cs_mb* mb_ptr;
  const uint8_t* frame_type;
  uint32_t* keep_mask;
  uint32_t* gop_state;
  float* score;
  int32_t* kept_count;
  unsigned long long* counters;
  int32_t* status;
  unsigned off_vrow, off_srow, off_dyn, off_bar, off_stage;
  // ---- fused compaction (NEXT-2: codecsight_score_compact) ----
  int fused;
  int layout;            // CS_LAYOUT_PLANAR | CS_LAYOUT_GROUPED
  int patch, FW, FH, ngc, vec_out;
  long long capacity;
  const int32_t* frame_index;
  const void* const* frames;
  uint16_t* packed;
  int32_t* pos_ids;
  int32_t* src_index;
  int32_t* frame_offsets;
  unsigned* ws_ctr;              // [0] ticket, [1] CTAs done, [2] CTAs whose frame offsets are published
  int global_compact;            // every cluster co-resident: compaction balanced over the whole grid (see below)
  unsigned long long* ws_flags;  // [n_streams] look-back words: (state << 62) | rows, state 1 = aggregate, 2 = prefix
  unsigned total_ctas;
  int tma_stages;  // 4,736-B TMA stages that fit the score's staging memory (fused compaction ring)
};

#ifdef CS_PHASE_TIMING
// experiment build only (scripts/phase_timing.py): per-CTA %globaltimer stamps at the phase boundaries
// (two slots, alternating per launch, so that back-to-back launches -- PDL overlap -- can be compared)
__device__ unsigned long long g_cs_phase[2][16384][12];
static int g_cs_phase_launch = 0;
__device__ unsigned g_cs_smid[16384];
__device__ __forceinline__ void cs_phase(int slot, int k) {
  if (threadIdx.x == 0 && blockIdx.x < 16384) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_cs_phase[slot][blockIdx.x][k] = t;
    if (k == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      g_cs_smid[blockIdx.x] = sm;
    }
  }
}
#define CS_PHASE(k) cs_phase(P.phase_slot, k)
#else
#define CS_PHASE(k)
#endif

constexpr int kFusedMaxStages = 42;  // 200 KB of 4,736-B stages (one-wave grids, see launch_score)
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagPre = 2ull << 62, kFlagVal = (1ull << 62) - 1;

// programmatic dependent launch (sm_90+): allow the next grid on the stream to launch now
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One kept group (gr, gc) of frame `fr` -> packed rows [n0, n0 + G^2) (rows >= capacity dropped); returns rows
// written.  Same bytes and order as codecsight_compact (reading Q14/Q15).
__device__ __forceinline__ int fused_copy_group(const ScoreParams& P, const uint16_t* __restrict__ fr, bool vec_in,
                                                int gr, int gc, long long n0, long long slot, int t_index,
                                                int lane) {
  const int G = P.G, p = P.patch, pp = p * p, gs2 = G * G;
  long long nvalid = P.capacity - n0;
  nvalid = nvalid < 0 ? 0 : (nvalid > gs2 ? gs2 : nvalid);
  if (nvalid == 0) return 0;
  const long long row_el = 3ll * pp;
  uint16_t* dst = P.packed + n0 * row_el;
  const int nel = static_cast<int>(nvalid * row_el);
  if (P.layout == CS_LAYOUT_GROUPED) {
    const uint16_t* blk = fr + ((long long)gr * P.ngc + gc) * gs2 * row_el;
    if (vec_in && P.vec_out) {
      const int n16 = nel / 8;
      for (int e = n16 * 8 + lane; e < nel; e += 32) dst[e] = blk[e];
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
      for (int e = lane; e < nel; e += 32) dst[e] = blk[e];
    }
  } else {
    // planar CHW: element (q, c, y, x) of the packed group reads pixel (c, (gr*G + dy)*p + y, (gc*G + dx)*p + x)
    const long long plane = (long long)P.FH * P.FW;
    for (int e = lane; e < nel; e += 32) {
      const int q = e / (3 * pp), r = e - q * 3 * pp;
      const int c = r / pp, r2 = r - c * pp;
      const int y = r2 / p, x = r2 - y * p;
      const int dy = q / G, dx = q - dy * G;
      dst[e] = fr[c * plane + (long long)((gr * G + dy) * p + y) * P.FW + (gc * G + dx) * p + x];
    }
  }
  if (lane < nvalid) {
    const int dy = lane / G, dx = lane - dy * G;
    const int h = gr * G + dy, w = gc * G + dx;
    const long long n = n0 + lane;
    P.pos_ids[3 * n + 0] = t_index;
    P.pos_ids[3 * n + 1] = h;
    P.pos_ids[3 * n + 2] = w;
    P.src_index[n] = static_cast<int32_t>(slot * P.np + h * P.grid_w + w);
  }
  return static_cast<int>(nvalid);
}

template <bool FUSED>
__global__ void __launch_bounds__(kThreads) score_kernel(const __grid_constant__ ScoreParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint8_t s_types[cs::kMaxFramesPerCall];
  __shared__ int s_plist[cs::kMaxFramesPerCall];
  __shared__ uint32_t s_state[cs::kMaxGridWords + 1];
  __shared__ uint32_t s_out[cs::kMaxGridWords];
  __shared__ uint32_t s_keep[cs::kMaxGridWords];
  __shared__ int s_np, s_kept, s_badmb;
  __shared__ unsigned long long s_near;

  __shared__ int s_sidx;
  CS_PHASE(0);
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank());
  int sidx_ = blockIdx.x / P.cluster;
  if (FUSED && !(P.global_compact && !P.pdl)) {
    // streams are taken in ticket order (cluster start order), so every stream a look-back waits for belongs to a
    // cluster that is already running: the decoupled look-back below cannot deadlock.  (A grid-balanced call has
    // every cluster resident -- its grid barrier relies on that already -- so it takes its stream from blockIdx and
    // starts its MB loads one atomic round trip earlier; chained calls keep the ticket, their predecessor's CTAs
    // may still hold SMs.)
    if (rank == 0 && threadIdx.x == 0) s_sidx = static_cast<int>(atomicAdd(&P.ws_ctr[0], 1u));
    cluster.sync();
    sidx_ = *cluster.map_shared_rank(&s_sidx, 0);
  }
  const int sidx = sidx_;
  CS_PHASE(1);
  const int tid = threadIdx.x, lane = tid & 31;
  const int nthr = blockDim.x;

  unsigned char* stage = smem + P.off_stage;
  uint32_t* Vrow = reinterpret_cast<uint32_t*>(smem + P.off_vrow);  // max |mv|^2 per (MB row, patch col)
  uint32_t* Srow = reinterpret_cast<uint32_t*>(smem + P.off_srow);
  uint32_t* dyn = reinterpret_cast<uint32_t*>(smem + P.off_dyn);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P.off_bar);

  const int f_begin = rank * P.fpc;
  const int f_end = min(P.n_frames, f_begin + P.fpc);
  const int nw = P.nw;

  // ---- prologue: warp 0 reads this CTA's frame types, lists its P-frames and starts the MB loads at once; the
  // other warps meanwhile stage the frame types of the whole stream (the scan needs the earlier frames), the GOP
  // state and the MB column / row ranges of the patch columns / rows ----
  const cs_mb* stream_mb = P.mb_ptr + (long long)sidx * P.n_frames * P.mb_rows * P.mb_cols;
  int2* s_col = reinterpret_cast<int2*>(smem + P.off_col);  // [grid_w] MB column range of each patch column
  int2* s_row = reinterpret_cast<int2*>(smem + P.off_row);  // [grid_h] MB row range of each patch row
  // producer (thread 0) walks the chunk sequence with its own counters: frame list index, chunk in frame, stage
  int pf = 0, pc = 0, ps = 0;
  auto issue_next = [&]() {
    const int f = s_plist[pf];
    const int r0 = pc * P.chunk_rows;
    const int nrows = min(P.chunk_rows, P.mb_rows - r0);
    const uint32_t bytes = static_cast<uint32_t>(nrows) * P.row_bytes;
    cs::mbar_arrive_expect_tx(&bars[ps], bytes);
    cs::bulk_g2s(stage + (size_t)ps * P.chunk_alloc, stream_mb + ((long long)f * P.mb_rows + r0) * P.mb_cols, bytes,
                 &bars[ps]);
    if (++pc == P.n_chunks) { pc = 0; ++pf; }
    if (++ps == P.nstage) ps = 0;
  };
  if (tid < 32) {
    const int f = f_begin + lane;  // fpc <= kMaxFramesPerCall / 8 = 32
    const bool isP = f < f_end && P.frame_type[(long long)sidx * P.type_stride + f] == CS_FRAME_P;
    uint32_t pm = __ballot_sync(0xffffffffu, isP);
    if (lane == 0) {
      int n = 0;
      for (; pm; pm &= pm - 1u) s_plist[n++] = f_begin + __ffs(pm) - 1;
      s_np = n;
      s_badmb = 0;
      s_near = 0ull;
      if (P.use_bulk) {
        for (int st = 0; st < P.nstage; ++st) cs::mbar_init(&bars[st], 1);
        cs::fence_mbar_init();
        for (int q = 0; q < min(n * P.n_chunks, P.nstage); ++q) issue_next();
      }
    }
  } else {
    const int t0 = tid - 32, nt = nthr - 32;
    for (int f = t0; f < P.n_frames; f += nt) s_types[f] = P.frame_type[(long long)sidx * P.type_stride + f];
    if (!(FUSED && P.pdl))  // (chained: the GOP state -- the preceding call's output -- is read once it is ready)
      for (int t = t0; t <= nw; t += nt) s_state[t] = P.gop_state[(long long)sidx * (nw + 1) + t];
    const int cw = P.mb * P.grid_w, ch = P.mb * P.grid_h;  // MB width / height in scaled units
    for (int c = t0; c < P.grid_w; c += nt) s_col[c] = make_int2((c * P.src_w) / cw, ((c + 1) * P.src_w - 1) / cw);
    for (int r = t0; r < P.grid_h; r += nt) s_row[r] = make_int2((r * P.src_h) / ch, ((r + 1) * P.src_h - 1) / ch);
  }
  __syncthreads();
  const int T = s_np * P.n_chunks;  // chunk sequence over this CTA's P-frames
  // every chunk of every P-frame of this CTA is in flight at once: warps need not wait for each other per chunk
  const bool resident = T <= P.nstage;

  CS_PHASE(2);
  unsigned long long near_local = 0;
  const int lane_w = tid >> 5, nwarps = nthr >> 5;
  const int cw = P.mb * P.grid_w;
  int cf = 0, cc = 0, cs_ = 0, cph = 0;  // consumer: frame list index, chunk in frame, stage, stage phase
  for (int q = 0; q < T; ++q) {
    const int f = s_plist[cf];
    const int r0 = cc * P.chunk_rows;
    const int nrows = min(P.chunk_rows, P.mb_rows - r0);
    const uint2* buf = reinterpret_cast<const uint2*>(stage + (size_t)cs_ * P.chunk_alloc);
    if (P.use_bulk) {
      cs::mbar_wait(&bars[cs_], cph);
      if (q == 0) CS_PHASE(3);
      if (q == T - 1) CS_PHASE(10);
    } else {
      const uint2* g = reinterpret_cast<const uint2*>(stream_mb + ((long long)f * P.mb_rows + r0) * P.mb_cols);
      uint2* d = reinterpret_cast<uint2*>(stage + (size_t)cs_ * P.chunk_alloc);
      for (int e = tid; e < nrows * P.mb_cols; e += nthr) d[e] = g[e];
      __syncthreads();
    }
    // ---- pass 1: MB row j -> per patch column c: max |mv|^2 and sum_i ox(c,i) * sad_m (exact, u32) --------
    // v = fl(sqrt(fl(dx^2 + dy^2))) / 4 is monotone in dx^2 + dy^2, so max_m v_m = v(max_m |mv_m|^2): the sqrt
    // is taken once per patch in pass 2 (bit-identical to the max of per-MB magnitudes).  INTRA -> sentinel.
    int badmb = 0;
    for (int c = lane; c < P.grid_w; c += 32) {
      const int px0 = c * P.src_w, px1 = px0 + P.src_w;
      const int2 ic = s_col[c];
      for (int row = lane_w; row < nrows; row += nwarps) {
        uint32_t msq = 0u, ssum = 0u;
        const uint2* rr = buf + row * P.mb_cols;
        for (int i = ic.x; i <= ic.y; ++i) {
          const uint2 rec = rr[i];
          const int dx = static_cast<int16_t>(rec.x & 0xffffu);
          const int dy = static_cast<int16_t>(rec.x >> 16);
          const uint32_t type = (rec.y >> 16) & 0xffu;
          if (type <= CS_MB_SKIP) {
            const uint32_t sq = static_cast<uint32_t>(dx * dx) + static_cast<uint32_t>(dy * dy);
            msq = sq > msq ? sq : msq;
          } else {
            msq = kIntraSq;  // INTRA (or unknown) -> maximally dynamic (Q9)
            badmb |= (type > CS_MB_INTRA);
          }
          if (P.use_r) {
            const int ox = min(px1, cw * (i + 1)) - max(px0, cw * i);
            ssum += static_cast<uint32_t>(ox) * (rec.y & 0xffffu);
          }
        }
        const int j = r0 + row;
        Vrow[j * P.grid_w + c] = msq;
        if (P.use_r) Srow[j * P.grid_w + c] = ssum;
      }
    }
    if (badmb) s_badmb = 1;
    if (!resident) {
      __syncthreads();  // chunk fully consumed (its stage is refilled below), Vrow/Srow rows complete
      if (P.use_bulk && tid == 0 && q + P.nstage < T) issue_next();
    }
    if (++cs_ == P.nstage) { cs_ = 0; cph ^= 1; }

    if (++cc == P.n_chunks) {
      cc = 0;
      ++cf;
      // ---- pass 2: patch rows; Eq. 3 and Eq. 4; ballot into dynamic words ------------------------------
      if (resident) __syncthreads();  // Vrow/Srow rows of the frame complete
      CS_PHASE(9);
      const int lf = f - f_begin;
      const int ch = P.mb * P.grid_h;  // MB height in scaled y units
      for (int i = tid; i < nw * 32; i += nthr) {
        bool d = false, nr = false;
        if (i < P.np) {
          const int r = P.gw_shift >= 0 ? (i >> P.gw_shift) : i / P.grid_w;
          const int c = i - r * P.grid_w;
          const int py0 = r * P.src_h, py1 = py0 + P.src_h;
          const int2 jr = s_row[r];
          uint32_t msq = 0u;
          unsigned long long S = 0ull;
          for (int j = jr.x; j <= jr.y; ++j) {
            const uint32_t mj = Vrow[j * P.grid_w + c];
            msq = mj > msq ? mj : msq;
            if (P.use_r) {
              const int oy = min(py1, ch * (j + 1)) - max(py0, ch * j);
              S += static_cast<unsigned long long>(oy) * Srow[j * P.grid_w + c];
            }
          }
          // Eq. 1: V(i) = max over overlapping MBs of |mv| / 4 px
          const float V = msq == kIntraSq ? CUDART_INF_F : __fmul_rn(__fsqrt_rn(__uint2float_rn(msq)), 0.25f);
          float M;
          if (isinf(V)) {
            M = CUDART_INF_F;
          } else if (P.use_r) {
            const float R = __double2float_rn(__ddiv_rn(static_cast<double>(S), P.denom));
            M = __fmaf_rn(P.alpha, R, V);  // Eq. 3
          } else {
            M = V;  // alpha == 0: fma(0, R, V) == V for every finite R >= 0 and V >= 0
          }
          d = (M >= P.tau);  // Eq. 4 (inclusive, Q1)
          nr = isfinite(M) && fabsf(__fsub_rn(M, P.tau)) <= 1e-5f;
          if (P.want_score) P.score[((long long)sidx * P.n_frames + f) * P.np + i] = M;
        }
        const uint32_t word = __ballot_sync(0xffffffffu, d);
        const uint32_t nword = __ballot_sync(0xffffffffu, nr);
        if (lane == 0) {
          dyn[lf * nw + (i >> 5)] = word;
          near_local += __popc(nword);
        }
      }
      __syncthreads();  // Vrow/Srow free for the next frame
    }
  }
  // scores of I-frames: +inf (Q10)
  if (P.want_score)
    for (int f = f_begin; f < f_end; ++f)
      if (s_types[f] != CS_FRAME_P)
        for (int i = tid; i < P.np; i += nthr) P.score[((long long)sidx * P.n_frames + f) * P.np + i] = CUDART_INF_F;

  CS_PHASE(11);
  if (FUSED && P.pdl) {
    // Chained call (CS_LAUNCH_PDL): everything above (stream ticket in this call's own workspace, MB loads, passes
    // 1 and 2 into shared memory) read only inputs staged before the preceding call started, so it overlapped that
    // call.  The GOP state is the preceding call's output: wait until its generation says it is final, and (the
    // outputs below go to buffers call g-d used, d = chain depth) until call g-d has completed (done[g mod d]: calls
    // of one class complete in order).  Both are published with release stores; the calls we wait for are resident
    // (this grid launched after all of g-1's CTAs passed this point, g-1 after all of g-2's, ...), so the spins
    // cannot deadlock.  (The stream ticket above used this call's workspace before any wait: calls g-1 .. g-d may
    // still run, so chained calls rotate d + 1 workspaces.)
    if (tid == 0) {
      while (ld_acquire_u32(&P.gop_ready[sidx]) != P.generation) __nanosleep(32);
      const unsigned cls = P.generation % P.chain_depth;
      while (static_cast<int>(ld_acquire_u32(&P.chain_done[cls]) - (P.generation - P.chain_depth + 1u)) < 0)
        __nanosleep(32);
    }
    __syncthreads();
    for (int t = tid; t <= nw; t += nthr) s_state[t] = P.gop_state[(long long)sidx * (nw + 1) + t];
    __syncthreads();
    pdl_launch_dependents();  // the next call may launch once every CTA of this one is here
  }
  CS_PHASE(4);
  cluster.sync();  // every CTA's dynamic words are published

  // ---- segmented OR-scan over time (GOP accumulation) + group-complete expansion ----------
  int st_bits = 0;
  if (tid == 0) {
    if (s_badmb) st_bits |= CS_STATUS_BAD_MB_TYPE;
    int flag = s_state[nw] & 1u;
    for (int f = 0; f < f_end; ++f) {
      const uint8_t ty = s_types[f];
      if (ty == CS_FRAME_P) {
        if (!flag && f >= f_begin) st_bits |= CS_STATUS_NO_IFRAME;
        flag = 1;
      } else {
        if (ty != CS_FRAME_I && f >= f_begin) st_bits |= CS_STATUS_BAD_FRAME_TYPE;
        flag = 1;
      }
    }
  }
  unsigned long long kept_total = 0;
  for (int f = f_begin; f < f_end; ++f) {
    const bool isP = (s_types[f] == CS_FRAME_P);
    for (int t = tid; t < nw; t += nthr) {
      uint32_t acc = s_state[t];
      uint32_t flag = s_state[nw] & 1u;
      for (int f2 = 0; f2 <= f; ++f2) {
        if (s_types[f2] != CS_FRAME_P) {
          acc = 0u;  // I-frame: state := empty (Q7)
          flag = 1u;
        } else {
          if (!flag) {
            acc = 0u;  // P-frame on an uninitialised stream (Q11)
            flag = 1u;
          }
          const uint32_t* rd = cluster.map_shared_rank(dyn, f2 / P.fpc);
          acc |= rd[(f2 % P.fpc) * nw + t];
        }
      }
      uint32_t full = 0xffffffffu;
      if ((t + 1) * 32 > P.np) full = (P.np - t * 32 >= 32) ? 0xffffffffu : ((1u << (P.np - t * 32)) - 1u);
      s_out[t] = isP ? acc : full;
      if (f == P.n_frames - 1) {  // final GOP state of the stream
        P.gop_state[(long long)sidx * (nw + 1) + t] = acc;
        if (t == 0) P.gop_state[(long long)sidx * (nw + 1) + nw] = s_state[nw] | 1u;
        if (FUSED && P.pdl) __threadfence();  // (chained: ordered before the generation published below)
      }
    }
    if (tid == 0) s_kept = 0;
    __syncthreads();
    if (FUSED && P.pdl && f == P.n_frames - 1 && tid == 0)  // chained: the stream's final state, to call g+1
      st_release_u32(&P.gop_ready[sidx], P.generation + 1u);
    if (P.G == 2 && P.grid_w == 32) {
      // word r = patch row r: a group row is rows 2g, 2g+1; fold horizontal pairs, spread back to both columns
      for (int gr = tid; gr < P.grid_h / 2; gr += nthr) {
        const uint32_t x = s_out[2 * gr] | s_out[2 * gr + 1];
        const uint32_t y = (x | (x >> 1)) & 0x55555555u;
        const uint32_t kw = y | (y << 1);
        s_keep[2 * gr] = kw;
        s_keep[2 * gr + 1] = kw;
        atomicAdd(&s_kept, 2 * __popc(kw));
      }
    } else {
      const int ngc = P.grid_w / P.G;
      for (int i = tid; i < nw * 32; i += nthr) {
        bool k = false;
        if (i < P.np) {
          const int h = i / P.grid_w, w = i - h * P.grid_w;
          k = cs::group_kept(s_out, (h / P.G) * ngc + (w / P.G), ngc, P.G, P.grid_w);
        }
        const uint32_t word = __ballot_sync(0xffffffffu, k);
        if (lane == 0) {
          s_keep[i >> 5] = word;
          atomicAdd(&s_kept, __popc(word));
        }
      }
    }
    __syncthreads();
    const long long slot = (long long)sidx * P.frame_stride + f;
    for (int t = tid; t < nw; t += nthr) P.keep_mask[slot * nw + t] = s_keep[t];
    if (tid == 0) {
      P.kept_count[(long long)sidx * P.n_frames + f] = s_kept;
      kept_total += static_cast<unsigned long long>(s_kept);
    }
    __syncthreads();
  }

  // ---- counters / status -------------------------------------------------------------------------------
  CS_PHASE(5);
  if (near_local) atomicAdd(&s_near, near_local);
  __syncthreads();
  if (tid == 0) {
    const unsigned long long nf = static_cast<unsigned long long>(f_end - f_begin);
    const unsigned long long npf = static_cast<unsigned long long>(s_np);
    const unsigned long long per_frame = 4ull * nw + 4ull + (P.want_score ? 4ull * P.np : 0ull);
    unsigned long long bytes = nf * per_frame + npf * 8ull * P.mb_rows * P.mb_cols;
    if (rank == 0) bytes += 2ull * 4ull * (nw + 1);
    cs::atomic_add_u64(&P.counters[CS_CNT_FRAMES], nf);
    cs::atomic_add_u64(&P.counters[CS_CNT_PFRAMES], npf);
    cs::atomic_add_u64(&P.counters[CS_CNT_PATCHES], nf * P.np);
    cs::atomic_add_u64(&P.counters[CS_CNT_KEPT], kept_total);
    cs::atomic_add_u64(&P.counters[CS_CNT_NEAR_TAU], s_near);
    cs::atomic_add_u64(&P.counters[CS_CNT_BYTES_SCORE], bytes);
    cs::atomic_or_status(P.status, st_bits);
  }
  if (FUSED) {
    // ---- NEXT-2: compaction fused into the scoring pass -----------------------------------------------------
    // (1) stream-local prefix of emitted patches over the stream's frames (kept counts are group-complete, so a
    //     frame emits exactly kept_count rows); (2) the stream's offset in the batch by a decoupled look-back over
    //     the streams (ticket order = stream order); (3) the cluster's warps split the stream's kept groups evenly
    //     and copy them (frame -> packed rows), exactly as codecsight_compact would.
    __shared__ int s_lp[cs::kMaxFramesPerCall + 1];
    __shared__ long long s_prefix;
    __shared__ int s_written;
    cluster.sync();  // the stream's keep masks and kept counts are in global memory (cluster-scope acquire)
    if (tid < 32) {  // s_lp = exclusive prefix of the stream's kept counts (warp scan, 32 frames per round)
      int carry = 0;
      for (int f0 = 0; f0 < P.n_frames; f0 += 32) {
        const int f = f0 + lane;
        int v = f < P.n_frames ? P.kept_count[(long long)sidx * P.n_frames + f] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, v, d);
          if (lane >= d) v += u;
        }
        if (f < P.n_frames) s_lp[f + 1] = carry + v;
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
      if (lane == 0) {
        s_lp[0] = 0;
        s_written = 0;
      }
    }
    __syncthreads();
    if (rank == 0 && tid < 32) {
      // warp-parallel decoupled look-back: lane l inspects stream (j - l); the closest PREFIX flag ends the walk
      const unsigned long long tot = static_cast<unsigned long long>(s_lp[P.n_frames]);
      unsigned long long excl = 0;
      if (sidx == 0) {
        if (lane == 0) st_release_u64(&P.ws_flags[0], kFlagPre | tot);
      } else {
        if (lane == 0) st_release_u64(&P.ws_flags[sidx], kFlagAgg | tot);
        int j = sidx - 1;
        while (true) {
          const int jj = j - lane;
          unsigned long long v = jj >= 0 ? ld_acquire_u64(&P.ws_flags[jj]) : kFlagPre;  // before stream 0: prefix 0
          const uint32_t pre_mask = __ballot_sync(0xffffffffu, (v & ~kFlagVal) == kFlagPre);
          const uint32_t bad_mask = __ballot_sync(0xffffffffu, (v & ~kFlagVal) == 0ull);
          const int stop = pre_mask ? __ffs(pre_mask) - 1 : 32;  // lanes [0, stop] are summed (stop: the prefix)
          const uint32_t need = stop >= 31 ? 0xffffffffu : ((2u << stop) - 1u);
          if (bad_mask & need) continue;  // a stream in the window has not published yet: re-read
          unsigned long long add = (lane <= stop && jj >= 0) ? (v & kFlagVal) : 0ull;
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) add += __shfl_xor_sync(0xffffffffu, add, d);
          excl += add;
          if (pre_mask) break;
          j -= 32;
        }
        if (lane == 0) st_release_u64(&P.ws_flags[sidx], kFlagPre | (excl + tot));
      }
      if (lane == 0) {
        s_prefix = static_cast<long long>(excl);
        if (static_cast<long long>(excl + tot) > P.capacity) cs::atomic_or_status(P.status, CS_STATUS_CAPACITY);
        if (sidx == P.n_streams - 1)
          P.frame_offsets[(long long)P.n_streams * P.n_frames] = static_cast<int32_t>(excl + tot);
      }
    }
    cluster.sync();
    const long long pre = *cluster.map_shared_rank(&s_prefix, 0);
    CS_PHASE(6);
    for (int f = f_begin + tid; f < f_end; f += nthr)
      P.frame_offsets[(long long)sidx * P.n_frames + f] = static_cast<int32_t>(pre + s_lp[f]);
    const int gs2 = P.G * P.G;
    const long long groups = s_lp[P.n_frames] / gs2;
    const int ngroups = (P.grid_h / P.G) * P.ngc;
    // enumerate, for one warp, the stream's kept groups q in [q, q1) in packed order and call fn on each
    auto for_each_group = [&](long long q, long long q1, auto&& fn) {
      if (q >= q1) return;
      int f = 0;
      while (f + 1 < P.n_frames && s_lp[f + 1] / gs2 <= q) ++f;
      long long skip = q - s_lp[f] / gs2;
      for (; f < P.n_frames && q < q1; ++f, skip = 0) {
        const long long slot = (long long)sidx * P.n_frames + f;
        const uint32_t* m = P.keep_mask + ((long long)sidx * P.frame_stride + f) * nw;
        for (int base = 0; base < ngroups && q < q1; base += 32) {
          const int qq = base + lane;
          const bool kept = qq < ngroups && cs::group_kept(m, qq, P.ngc, P.G, P.grid_w);
          uint32_t bal = __ballot_sync(0xffffffffu, kept);
          const int nb = __popc(bal);
          if (skip >= nb) {
            skip -= nb;
            continue;
          }
          while (skip > 0) {
            bal &= bal - 1;
            --skip;
          }
          while (bal && q < q1) {
            const int b = __ffs(bal) - 1;
            bal &= bal - 1;
            const int gi = base + b;
            fn(slot, gi / P.ngc, gi - (gi / P.ngc) * P.ngc, pre + q * gs2);
            ++q;
          }
        }
      }
    };
    int written = 0;
    bool tma = false;  // per-stream TMA ring: only thread 0 holds the CTA's count
    if (P.global_compact) {
      // Grid-balanced compaction (every cluster is co-resident, checked on the host): each stream's cluster would
      // otherwise copy only its own stream's kept groups, and streams with more motion keep more (measured at C2:
      // CTAs end 36-55 us apart).  Publish this CTA's frame offsets, wait until every CTA of the grid has, then
      // every ring warp of the grid takes an equal share of ALL the batch's kept groups (the layout
      // codecsight_compact's TMA gather uses, cs::group_ring).
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        atomicAdd(&P.ws_ctr[2], 1u);
        while (ld_acquire_u32(&P.ws_ctr[2]) < P.total_ctas) __nanosleep(64);
      }
      __syncthreads();
      __shared__ __align__(8) uint64_t s_gfull[kFusedMaxStages];
      __shared__ cs::RingGroup s_gdesc[kFusedMaxStages];
      __shared__ __align__(16) uint32_t s_gmask[kThreads / 32][32];
      const int R = min(nthr >> 5, P.tma_stages / 3);  // ring warps of >= 3 stages each
      const int wq = tid >> 5;
      if (wq < R) {
        const int nst = P.tma_stages / R;
        cs::RingBatch B;
        B.frame_offsets = P.frame_offsets;
        B.n_slots = P.n_streams * P.n_frames;
        B.n_frames = P.n_frames;
        B.keep_mask = P.keep_mask;
        B.mask_frame_stride = P.frame_stride;
        B.frames = P.frames;
        B.frame_index = P.frame_index;
        B.capacity = P.capacity;
        B.packed = P.packed;
        B.pos_ids = P.pos_ids;
        B.src_index = P.src_index;
        const long long T = static_cast<long long>(P.frame_offsets[B.n_slots]) / 4;
        const long long NW = static_cast<long long>(gridDim.x) * R, gw = static_cast<long long>(blockIdx.x) * R + wq;
        const long long rows = cs::group_ring(B, T * gw / NW, T * (gw + 1) / NW,
                                              smem + P.off_stage + (size_t)wq * nst * cs::kRingStageAlloc, nst,
                                              s_gfull + wq * nst, s_gdesc + wq * nst, s_gmask[wq], lane);
        if (lane == 0) written = static_cast<int>(rows);
      }
    } else {
    tma = P.layout == CS_LAYOUT_GROUPED && P.vec_out && P.patch == 14 && P.G == 2 && P.grid_w == 32 &&
                     P.grid_h == 32 && P.tma_stages >= 9;  // R = stages/3 rings of >= 3 stages each, else direct copies (measured)
    if (tma) {
      // the CTA's share of the stream's kept groups: thread 0 runs a TMA bulk ring over it (4,704-B groups,
      // global -> smem on an mbarrier, smem -> global as a bulk group, the stage reused once the store has read
      // it) in the score's staging memory, which is free now; warps 1.. write the position ids / source indices
      const long long qa0 = groups * rank / P.cluster, qb0 = groups * (rank + 1) / P.cluster;
      // R ring warps (lane 0 of each drives its own TMA ring over its own stages and share of the range)
      const int R = min(4, P.tma_stages / 3);
      const int wq = tid >> 5;
      const long long qa = qa0 + (qb0 - qa0) * min(wq, R) / R, qb = qa0 + (qb0 - qa0) * min(wq + 1, R) / R;
      __shared__ __align__(8) uint64_t s_tfull_all[kFusedMaxStages];
      __shared__ long long s_tn0_all[kFusedMaxStages];
      __shared__ const uint16_t* s_tsrc_all[kFusedMaxStages];
      if (wq < R && lane == 0 && qa < qb) {
        const int nst = P.tma_stages / R, sb = wq * nst;
        uint64_t* s_tfull = s_tfull_all + sb;
        long long* s_tn0 = s_tn0_all + sb;
        const uint16_t** s_tsrc = s_tsrc_all + sb;
        unsigned char* tbase = smem + P.off_stage + (size_t)sb * 4736u;
        const long long row_el = 3ll * 14 * 14;
        for (int st = 0; st < nst; ++st) cs::mbar_init(&s_tfull[st], 1);
        cs::fence_mbar_init();
        cs::fence_proxy_async_smem();  // the staging memory was last used through the generic proxy
        int f = 0;
        while (f + 1 < P.n_frames && s_lp[f + 1] / 4 <= qa) ++f;
        long long skip = qa - s_lp[f] / 4;
        int gr = 0;
        uint32_t ybits = 0u;
        const uint16_t* fr = nullptr;
        bool aligned = false;
        auto load_row = [&]() {
          const uint32_t* m = P.keep_mask + ((long long)sidx * P.frame_stride + f) * nw;
          const uint32_t x = m[2 * gr] | m[2 * gr + 1];
          ybits = (x | (x >> 1)) & 0x55555555u;
        };
        auto load_frame = [&]() {
          fr = static_cast<const uint16_t*>(P.frames[(long long)sidx * P.n_frames + f]);
          aligned = (reinterpret_cast<uintptr_t>(fr) & 15u) == 0;
        };
        load_frame();
        load_row();
        while (skip >= __popc(ybits)) {
          skip -= __popc(ybits);
          ++gr;
          load_row();
        }
        for (; skip > 0; --skip) ybits &= ybits - 1u;
        long long q = qa;
        bool more = true;
        auto issue = [&](int st) {
          if (q >= qb) {
            s_tn0[st] = -1;
            cs::mbar_arrive(&s_tfull[st]);
            more = false;
            return;
          }
          while (ybits == 0u) {
            if (++gr == 16) {
              gr = 0;
              ++f;
              load_frame();
            }
            load_row();
          }
          const int b = __ffs(ybits) - 1;
          ybits &= ybits - 1u;
          const long long n0 = pre + q * 4;
          const uint16_t* src = fr + (long long)(gr * 16 + (b >> 1)) * 4 * row_el;
          ++q;
          s_tn0[st] = n0;
          s_tsrc[st] = src;
          if (n0 + 4 <= P.capacity && aligned) {
            cs::mbar_arrive_expect_tx(&s_tfull[st], 4704u);
            cs::bulk_g2s(tbase + (size_t)st * 4736u, src, 4704u, &s_tfull[st]);
          } else {
            cs::mbar_arrive(&s_tfull[st]);  // copied directly below (truncated group / misaligned frame)
          }
        };
        for (int st = 0; st < nst && more; ++st) issue(st);
        for (int it = 0;; ++it) {
          const int st = it % nst;
          cs::mbar_wait(&s_tfull[st], (it / nst) & 1);
          const long long n0 = s_tn0[st];
          if (n0 < 0) break;
          if (n0 + 4 <= P.capacity) {
            if (s_tsrc[st] && (reinterpret_cast<uintptr_t>(s_tsrc[st]) & 15u) == 0) {
              cs::bulk_s2g(P.packed + n0 * row_el, tbase + (size_t)st * 4736u, 4704u);
            } else {
              for (long long e = 0; e < 4 * row_el; ++e) P.packed[n0 * row_el + e] = s_tsrc[st][e];
            }
          } else if (n0 < P.capacity) {
            for (long long e = 0; e < (P.capacity - n0) * row_el; ++e) P.packed[n0 * row_el + e] = s_tsrc[st][e];
          }
          cs::bulk_commit();  // one (possibly empty) bulk group per item
          if (it >= 1 && more) {
            cs::bulk_wait_read<1>();
            issue((it - 1) % nst);
          }
        }
        cs::bulk_wait_all<0>();
      } else if (wq >= R && qa0 < qb0) {
        const long long nw7 = (nthr >> 5) - R, w7 = wq - R;
        for_each_group(qa0 + (qb0 - qa0) * w7 / nw7, qa0 + (qb0 - qa0) * (w7 + 1) / nw7,
                       [&](long long slot, int gr, int gc, long long n0) {
                         const int t_index = P.frame_index[slot];
                         if (lane < 4 && n0 + lane < P.capacity) {
                           const int h = gr * 2 + (lane >> 1), w = gc * 2 + (lane & 1);
                           const long long n = n0 + lane;
                           P.pos_ids[3 * n + 0] = t_index;
                           P.pos_ids[3 * n + 1] = h;
                           P.pos_ids[3 * n + 2] = w;
                           P.src_index[n] = static_cast<int32_t>(slot * P.np + h * P.grid_w + w);
                         }
                       });
      }
      if (tid == 0) {
        long long r = P.capacity - (pre + qa0 * 4);
        r = r < 0 ? 0 : (r > (qb0 - qa0) * 4 ? (qb0 - qa0) * 4 : r);
        written = static_cast<int>(r);
      }
    } else {
      const long long nwarp_c = static_cast<long long>(P.cluster) * (nthr >> 5);
      const long long wid = static_cast<long long>(rank) * (nthr >> 5) + (tid >> 5);
      for_each_group(groups * wid / nwarp_c, groups * (wid + 1) / nwarp_c,
                     [&](long long slot, int gr, int gc, long long n0) {
                       const uint16_t* fr = static_cast<const uint16_t*>(P.frames[slot]);
                       const bool vec_in = ((reinterpret_cast<uintptr_t>(fr) & 15u) == 0) &&
                                           ((3 * gs2 * P.patch * P.patch * 2) % 16 == 0);
                       written += fused_copy_group(P, fr, vec_in, gr, gc, n0, slot, P.frame_index[slot], lane);
                     });
    }
    }  // (per-stream compaction)
    if ((lane == 0 || tma) && written) atomicAdd(&s_written, written);
    if (P.pdl) __threadfence();  // (chained: every output write ordered before the completion published below)
    __syncthreads();
    CS_PHASE(7);
    if (tid == 0) {
      const unsigned long long rows = static_cast<unsigned long long>(s_written);
      const unsigned long long row_bytes = 3ull * P.patch * P.patch * 2ull;
      const unsigned long long nf = static_cast<unsigned long long>(f_end - f_begin);
      cs::atomic_add_u64(&P.counters[CS_CNT_PACKED_ROWS], rows);
      cs::atomic_add_u64(&P.counters[CS_CNT_BYTES_COMPACT], nf * (4ull * nw + 4ull) + rows * (2ull * row_bytes + 16ull));
      // the last CTA out returns the workspace to zero (every look-back has completed by then)
      __threadfence();
      if (atomicAdd(&P.ws_ctr[1], 1u) == P.total_ctas - 1) {
        for (int j = 0; j < P.n_streams; ++j) P.ws_flags[j] = 0ull;
        P.ws_ctr[0] = 0u;
        P.ws_ctr[1] = 0u;
        P.ws_ctr[2] = 0u;
        __threadfence();
        if (P.pdl) st_release_u32(&P.chain_done[P.generation % P.chain_depth], P.generation + 1u);  // call complete
      }
    }
  }
  CS_PHASE(8);
  cluster.sync();  // keep this CTA's shared memory alive until every DSMEM reader is done
}

}  // namespace

constexpr unsigned kWideSmem = 200u * 1024u;  // the kernels' dynamic shared memory limit (set once per device)

// true when all n_streams clusters of `cfg` are co-resident with kWideSmem bytes of dynamic shared memory per CTA
// (cudaOccupancyMaxActiveClusters; the answer for the last (device, cluster size) is cached)
// clusters of this launch configuration that can be resident at once with `smem` dynamic bytes per CTA (cached)
static int max_active_clusters(const void* fn, const cudaLaunchConfig_t& cfg, size_t smem) {
  static thread_local int c_dev = -1, c_cluster = -1, c_max = 0;
  static thread_local size_t c_smem = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  const int cl = static_cast<int>(cfg.attrs[0].val.clusterDim.x);
  if (dev != c_dev || cl != c_cluster || smem != c_smem) {
    cudaLaunchConfig_t q = cfg;
    q.dynamicSmemBytes = smem;
    q.numAttrs = 1;  // (the cluster dimension only)
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &q) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    c_dev = dev;
    c_cluster = cl;
    c_smem = smem;
    c_max = n;
  }
  return c_max;
}

static bool fused_one_wave(const void* fn, const cudaLaunchConfig_t& cfg, int32_t n_streams) {
  static thread_local int c_dev = -1, c_cluster = -1, c_max = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const int cl = static_cast<int>(cfg.attrs[0].val.clusterDim.x);
  if (dev != c_dev || cl != c_cluster) {
    cudaLaunchConfig_t q = cfg;
    q.dynamicSmemBytes = kWideSmem;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &q) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    c_dev = dev;
    c_cluster = cl;
    c_max = n;
  }
  return n_streams <= c_max;
}

static int launch_score(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                        const uint8_t* frame_type, uint32_t* keep_mask, int64_t frame_stride, uint32_t* gop_state,
                        float* score, int32_t* kept_count, unsigned long long* counters, int32_t* status,
                        const ScoreParams* fuse, cudaStream_t stream) {
  ScoreParams P{};
  if (fuse) P = *fuse;
  P.src_w = g->src_w;
  P.src_h = g->src_h;
  P.mb = g->mb_size;
  P.mb_cols = g->mb_cols;
  P.mb_rows = g->mb_rows;
  P.grid_w = g->grid_w;
  P.grid_h = g->grid_h;
  P.G = g->group;
  P.np = g->grid_w * g->grid_h;
  P.nw = (P.np + 31) / 32;
  P.tau = g->tau;
  P.alpha = g->alpha;
  P.denom = static_cast<double>(g->mb_size) * static_cast<double>(g->mb_size) * 255.0 *
            static_cast<double>(g->src_w) * static_cast<double>(g->src_h);
  P.n_streams = n_streams;
  P.n_frames = n_frames;
  int cluster = n_frames < 8 ? n_frames : 8;
  P.fpc = (n_frames + cluster - 1) / cluster;
  cluster = (n_frames + P.fpc - 1) / P.fpc;
  P.cluster = cluster;
  P.frame_stride = frame_stride;
  if (!fuse || P.type_stride <= 0) P.type_stride = frame_stride;
#ifdef CS_PHASE_TIMING
  P.phase_slot = g_cs_phase_launch & 1;
  ++g_cs_phase_launch;
#endif
  P.row_bytes = static_cast<unsigned>(g->mb_cols) * 8u;
  P.use_bulk = ((reinterpret_cast<uintptr_t>(mb) & 15u) == 0 && (P.row_bytes % 16u) == 0) ? 1 : 0;
  const unsigned target = 8192u;
  P.chunk_rows = static_cast<int>(P.row_bytes >= target ? 1u : target / P.row_bytes);
  if (P.chunk_rows > P.mb_rows) P.chunk_rows = P.mb_rows;
  P.n_chunks = (P.mb_rows + P.chunk_rows - 1) / P.chunk_rows;
  P.chunk_alloc = (static_cast<unsigned>(P.chunk_rows) * P.row_bytes + 127u) & ~127u;
  P.want_score = score != nullptr;
  P.use_r = g->alpha != 0.0f;
  P.gw_shift = -1;
  for (int sh = 0; sh < 13; ++sh)
    if ((1 << sh) == g->grid_w) P.gw_shift = sh;
  P.mb_ptr = mb;
  P.frame_type = frame_type;
  P.keep_mask = keep_mask;
  P.gop_state = gop_state;
  P.score = score;
  P.kept_count = kept_count;
  P.counters = counters;
  P.status = status;
  P.total_ctas = static_cast<unsigned>(n_streams) * static_cast<unsigned>(cluster);
  const void* fn = P.fused ? reinterpret_cast<const void*>(score_kernel<true>)
                          : reinterpret_cast<const void*>(score_kernel<false>);
  if (cs_set_smem_attr(fn, P.fused ? 19 : 0, kWideSmem) != 0) return CS_ERR_CUDA;

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(n_streams) * static_cast<unsigned>(cluster), 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (P.fused && P.pdl) {  // may start while the preceding call on `stream` runs (chained by generations, above)
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 2;
  }

  // dynamic shared memory budget per CTA: 50 KB for score_patches (4 CTAs/SM, register-limited anyway), 68 KB for
  // the fused kernel (3 CTAs/SM; the compaction's TMA rings reuse the staging memory), and the SM's whole 200 KB
  // when all the fused grid's clusters are co-resident even then (one wave at one CTA per SM, e.g. C2): deeper
  // rings, more bytes in flight per SM (measured)
  unsigned budget = P.fused ? CS_FUSED_SMEM_KB * 1024u : 50u * 1024u;
  // (PDL: two calls' CTAs must fit an SM together, so no whole-SM budget)
  if (P.fused && !P.pdl && fused_one_wave(fn, cfg, n_streams)) budget = kWideSmem;

  // layout: small regions first, then the MB staging ring, Vrow, Srow (only with alpha != 0); the MB ring takes
  // whatever the budget leaves (all of a frame's chunks in flight when they fit, at most 16 mbarriers, >= 2 stages)
  unsigned off = 0;
  P.off_dyn = off;
  off += ((static_cast<unsigned>(P.fpc * P.nw) * 4u + 127u) & ~127u);
  P.off_bar = off;
  off += 128u;
  P.off_col = off;
  off += ((static_cast<unsigned>(g->grid_w) * 8u + 127u) & ~127u);
  P.off_row = off;
  off += ((static_cast<unsigned>(g->grid_h) * 8u + 127u) & ~127u);
  P.off_stage = off;
  const unsigned vr_bytes = (static_cast<unsigned>(P.mb_rows * P.grid_w) * 4u + 127u) & ~127u;
  const unsigned fixed = off + vr_bytes + (P.use_r ? vr_bytes : 0u);
  int nst = fixed + 2u * P.chunk_alloc <= budget ? static_cast<int>((budget - fixed) / P.chunk_alloc) : 2;
  nst = nst > P.n_chunks ? P.n_chunks : nst;
  nst = nst > 16 ? 16 : (nst < 2 ? 2 : nst);
  P.nstage = P.use_bulk ? nst : 1;
  off += P.nstage * P.chunk_alloc;
  P.off_vrow = off;
  off += vr_bytes;
  P.off_srow = off;
  off += P.use_r ? vr_bytes : 0u;
  size_t smem = off;
  if (smem > kWideSmem) return CS_ERR_UNSUPPORTED;
  if (P.fused) {
    // the compaction's TMA rings: 4,736-B stages from off_stage up to the budget
    const size_t want = smem < budget ? budget : smem;
    unsigned st = static_cast<unsigned>((want - P.off_stage) / 4736u);
    if (st > static_cast<unsigned>(kFusedMaxStages)) st = kFusedMaxStages;
    P.tma_stages = static_cast<int>(st);
    const size_t need = P.off_stage + static_cast<size_t>(st) * 4736u;
    if (need > smem) smem = need;
  }
  cfg.dynamicSmemBytes = smem;
  // grid-balanced compaction when every cluster of the grid is resident at once (its CTAs wait for each other)
  P.global_compact = (P.fused && P.layout == CS_LAYOUT_GROUPED && P.vec_out && P.patch == 14 && P.G == 2 &&
                      P.grid_w == 32 && P.grid_h == 32 && P.tma_stages >= 3 &&
                      n_streams <= max_active_clusters(fn, cfg, smem)) ? 1 : 0;
  void* args[] = {&P};
  if (cudaLaunchKernelExC(&cfg, fn, args) != cudaSuccess) return CS_ERR_CUDA;
  return CS_OK;
}

int cs_launch_score(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                    const uint8_t* frame_type, uint32_t* keep_mask, int64_t frame_stride, uint32_t* gop_state,
                    float* score, int32_t* kept_count, unsigned long long* counters, int32_t* status,
                    cudaStream_t stream) {
  return launch_score(g, n_streams, n_frames, mb, frame_type, keep_mask, frame_stride, gop_state, score, kept_count,
                      counters, status, nullptr, stream);
}

size_t cs_score_compact_workspace_bytes(int32_t n_streams) {
  return n_streams < 0 ? 0 : 16u + 8u * static_cast<size_t>(n_streams);
}

int cs_launch_score_compact(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                            const uint8_t* frame_type, int64_t type_stride, uint32_t* keep_mask,
                            int64_t frame_stride, uint32_t* gop_state, float* score, int32_t* kept_count,
                            const int32_t* frame_index, const void* const* frames, int32_t frame_layout,
                            int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                            int32_t* frame_offsets, void* workspace, unsigned long long* counters, int32_t* status,
                            const cs_chain* chain, cudaStream_t stream) {
  ScoreParams F{};
  F.fused = 1;
  F.type_stride = type_stride;
  F.pdl = chain ? 1 : 0;
  if (chain) {
    F.gop_ready = chain->gop_ready;
    F.chain_done = chain->done;
    F.generation = chain->generation;
    F.chain_depth = chain->depth;
  }
  F.layout = frame_layout;
  F.patch = g->patch;
  F.FW = g->grid_w * g->patch;
  F.FH = g->grid_h * g->patch;
  F.ngc = g->grid_w / g->group;
  const long long group_bytes = 3ll * g->patch * g->patch * 2ll * g->group * g->group;
  F.vec_out = ((reinterpret_cast<uintptr_t>(packed) & 15u) == 0 && group_bytes % 16 == 0) ? 1 : 0;
  F.capacity = capacity;
  F.frame_index = frame_index;
  F.frames = frames;
  F.packed = static_cast<uint16_t*>(packed);
  F.pos_ids = pos_ids;
  F.src_index = src_index;
  F.frame_offsets = frame_offsets;
  F.ws_ctr = static_cast<unsigned*>(workspace);
  F.ws_flags = reinterpret_cast<unsigned long long*>(static_cast<unsigned char*>(workspace) + 16);
  return launch_score(g, n_streams, n_frames, mb, frame_type, keep_mask, frame_stride, gop_state, score, kept_count,
                      counters, status, &F, stream);
}

#ifdef CS_PHASE_TIMING
extern "C" int codecsight_debug_phase(unsigned long long* host, int n_ctas) {  // slot of the last launch
  if (n_ctas > 16384) n_ctas = 16384;
  const size_t off = sizeof(unsigned long long) * 12 * 16384 * ((g_cs_phase_launch + 1) & 1);
  return cudaMemcpyFromSymbol(host, g_cs_phase, sizeof(unsigned long long) * 12 * n_ctas, off) == cudaSuccess ? 0 : -1;
}
extern "C" int codecsight_debug_smid(unsigned* host, int n_ctas) {  // SM of each CTA of the last launch
  if (n_ctas > 16384) n_ctas = 16384;
  return cudaMemcpyFromSymbol(host, g_cs_smid, sizeof(unsigned) * n_ctas) == cudaSuccess ? 0 : -1;
}
extern "C" int codecsight_debug_phase_slot(unsigned long long* host, int n_ctas, int slot) {
  if (n_ctas > 16384) n_ctas = 16384;
  const size_t off = sizeof(unsigned long long) * 12 * 16384 * (slot & 1);
  return cudaMemcpyFromSymbol(host, g_cs_phase, sizeof(unsigned long long) * 12 * n_ctas, off) == cudaSuccess ? 0 : -1;
}
#endif
