// cs_internal.cuh — internal helpers of libcodecsight (sm_100a).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "codecsight.h"

#define CS_DEV __device__ __forceinline__

namespace cs {

constexpr int kMaxGridPatches = 4096;
constexpr int kMaxGridWords = kMaxGridPatches / 32;
constexpr int kMaxMbRowsTimesGridW = 8192;
constexpr int kMaxFramesPerCall = 256;
constexpr int kMaxHeadDim = 512;
constexpr int kMaxWindowPlusStride = 1024;

// ---------------------------------------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA engine) PTX wrappers
// ---------------------------------------------------------------------------------------------------------
CS_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

CS_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

CS_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

CS_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

CS_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

CS_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared (this CTA), completion signalled on `bar` (tx bytes).
// dst, src 16-B aligned; bytes a multiple of 16.
CS_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 1-D bulk copy shared (this CTA) -> global, tracked by the issuing thread's bulk async-groups.
CS_DEV void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
CS_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N committed bulk groups of this thread still READ their shared-memory source
template <int N>
CS_DEV void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// wait until at most N committed bulk groups of this thread are still in flight (writes performed)
template <int N>
CS_DEV void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// Ampere-style asynchronous 16-B copy global -> shared (LDGSTS; src and dst 16-B aligned), tracked per thread by
// commit / wait groups.  Many small row segments: one instruction moves 512 B per warp, where a 1-D bulk copy per
// segment pays the TMA unit's per-request cost (measured).
CS_DEV void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// predicated form (no branch around the copy): dst is a shared-space address (smem_u32)
CS_DEV void cp_async16_if(uint32_t dst, const void* src, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p cp.async.cg.shared.global [%0], [%1], 16;\n}" ::"r"(dst),
      "l"(src), "r"(static_cast<int>(pred))
      : "memory");
}
// predicated 2-B global store (no branch around it)
CS_DEV void st_b16_if(void* p, uint16_t v, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.b16 [%0], %1;\n}" ::"l"(p), "h"(v),
               "r"(static_cast<int>(pred))
               : "memory");
}
CS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
CS_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

CS_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------------------------------------------------
// vector memory helpers
// ---------------------------------------------------------------------------------------------------------
CS_DEV uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
CS_DEV uint2 ld_nc_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
CS_DEV void st_na_v4(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

CS_DEV float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
CS_DEV float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// fp32 -> bf16 bits, round to nearest even (NaN -> quiet NaN), same rule as the stored cache dtype.
CS_DEV uint32_t f32_to_bf16_rne(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu) != 0) return (u >> 16) | 0x0040u;
  u += 0x7fffu + ((u >> 16) & 1u);
  return u >> 16;
}

// Blackwell packed fp32 pairs (FADD2 / FMUL2 / FFMA2: two IEEE round-to-nearest fp32 operations, one per half, in
// one instruction issue -- each half is bit-identical to __fadd_rn / __fmul_rn / __fmaf_rn on it).
// CAUTION (measured, ptxas 12.9): ptxas contracts mul.rn.f32x2 feeding add/sub.rn.f32x2 into FFMA2 -- even with
// -fmad=false, and even through fma(x, 1, y) -- which changes the rounding.  So a sum or difference whose operand is
// a packed product must use add1 / sub1 below (FFMA2 with a runtime 1.0) or the scalar per-half forms addp / subp
// (scalar FADD is never fused with FMUL2).
CS_DEV unsigned long long f2pk(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
CS_DEV float2 f2upk(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
CS_DEV float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pk(a)), "l"(f2pk(b)));
  return f2upk(r);
}
CS_DEV float2 sub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pk(a)), "l"(f2pk(b)));
  return f2upk(r);
}
CS_DEV float2 mul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2pk(a)), "l"(f2pk(b)));
  return f2upk(r);
}
CS_DEV float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2pk(a)), "l"(f2pk(b)), "l"(f2pk(c)));
  return f2upk(r);
}
CS_DEV float2 addp(float2 a, float2 b) { return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y)); }
CS_DEV float2 subp(float2 a, float2 b) { return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y)); }
// Packed sum / difference in ONE issue that ptxas cannot contract: FFMA2 with a multiplier of exactly 1.0 that
// ptxas cannot see (`one` = a kernel parameter set to 1.0f / -1.0f on the host).  a * 1 and b * -1 are exact, so
// the single rounding of the fma is the IEEE sum / difference; and a product feeding it stays a separately rounded
// FMUL2 (the FFMA2 already spends its multiply on `one`).  Same bits as addp / subp, half the fma-pipe issues.
CS_DEV float2 add1(float2 a, float2 b, float2 one) { return fma2(a, one, b); }
CS_DEV float2 sub1(float2 a, float2 b, float2 negone) { return fma2(b, negone, a); }
CS_DEV float2 clamp255_2(float2 a) {
  return make_float2(fminf(fmaxf(a.x, 0.0f), 255.0f), fminf(fmaxf(a.y, 0.0f), 255.0f));
}
// clamp to [0, 255] in one ALU instruction per half (VIMNMX.RELU on the bit patterns): for non-negative floats the
// signed-int order of the bits is the float order, a negative float is a negative int (relu -> +0.0f).  Equal to
// clamp255_2 for every non-NaN input except -0.0f (-> +0.0f instead of -0.0f); callers guarantee no NaN / -0.0f.
CS_DEV float2 clamp255_relu2(float2 a) {
  int x, y;
  asm("min.relu.s32 %0, %1, %2;" : "=r"(x) : "r"(__float_as_int(a.x)), "r"(0x437F0000));
  asm("min.relu.s32 %0, %1, %2;" : "=r"(y) : "r"(__float_as_int(a.y)), "r"(0x437F0000));
  return make_float2(__int_as_float(x), __int_as_float(y));
}

// fp32 -> bf16 bits, round to nearest even, one cvt.rn.bf16.f32 (equal to f32_to_bf16_rne for every non-NaN f)
CS_DEV uint16_t f32_to_bf16_cvt(float f) {
  uint16_t r;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(f));
  return r;
}

// two fp32 -> packed bf16x2 (low half = lo), round to nearest even (cvt.rn.bf16x2.f32)
CS_DEV uint32_t pack_bf16x2_rn(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

CS_DEV void atomic_or_status(int32_t* status, int bits) {
  if (bits) atomicOr(reinterpret_cast<int*>(status), bits);
}

CS_DEV void atomic_add_u64(unsigned long long* p, unsigned long long v) {
  if (v) atomicAdd(p, v);
}

// warp-level group-bit enumeration helper: is group q (row-major over the group grid) kept in mask `m`
// (a group is kept iff any of its G x G patches has its bit set).
CS_DEV bool group_kept(const uint32_t* m, int q, int ngc, int G, int grid_w) {
  const int gr = q / ngc, gc = q - gr * ngc;
  bool any = false;
  for (int dy = 0; dy < G; ++dy) {
    const int base = (gr * G + dy) * grid_w + gc * G;
    for (int dx = 0; dx < G; ++dx) {
      const int i = base + dx;
      any |= ((m[i >> 5] >> (i & 31)) & 1u) != 0;
    }
  }
  return any;
}

}  // namespace cs

// launchers (one per .cu), called by abi.cu after validation
int cs_launch_score(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                    const uint8_t* frame_type, uint32_t* keep_mask, int64_t frame_stride, uint32_t* gop_state,
                    float* score, int32_t* kept_count, unsigned long long* counters, int32_t* status,
                    cudaStream_t stream);
int cs_launch_compact(const cs_grid* g, int32_t n_streams, int32_t n_frames, const uint32_t* keep_mask,
                      int64_t mask_frame_stride, const int32_t* frame_index, const void* const* frames,
                      int32_t frame_layout, int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets,
                      unsigned long long* counters, int32_t* status, cudaStream_t stream);
int cs_launch_compact_nv12(const cs_grid* g, const cs_preprocess* pp, int32_t n_streams, int32_t n_frames,
                           const uint32_t* keep_mask, int64_t mask_frame_stride, const int32_t* frame_index,
                           const void* const* y_planes, const void* const* uv_planes, int64_t capacity,
                           void* packed, int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets,
                           unsigned long long* counters, int32_t* status, cudaStream_t stream);
int cs_launch_compact_tp(const cs_grid* g, int32_t tp, int32_t n_streams, int32_t n_units, const uint32_t* keep_mask,
                         int64_t mask_frame_stride, const int32_t* unit_index, const void* const* frames,
                         int32_t frame_layout, int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                         int32_t* frame_offsets, uint32_t* unit_mask, int64_t unit_mask_stride,
                         const uint8_t* frame_type, uint8_t* unit_type, unsigned long long* counters,
                         int32_t* status, cudaStream_t stream);
int cs_launch_kv_refresh(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, int32_t n_streams,
                         const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring,
                         const void* const* old_cache, void* const* new_cache, const void* const* refreshed,
                         int64_t token_cap, uint8_t* disposition, int32_t* p_old, int32_t* n_tokens,
                         void* workspace, size_t workspace_bytes, unsigned long long* counters, int32_t* status,
                         cudaStream_t stream);
size_t cs_kv_workspace_bytes(const cs_kv_desc* kv, const cs_window* win, int32_t n_streams);
int cs_launch_kv_refresh_paged(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, int32_t n_streams,
                               const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring, void* const* pool,
                               const int32_t* slot_old, int32_t* slot_new, int64_t slot_cap,
                               const void* const* refreshed, int64_t token_cap, uint8_t* disposition,
                               int32_t* p_old, int32_t* n_tokens, void* workspace, unsigned long long* counters,
                               int32_t* status, cudaStream_t stream);
size_t cs_kv_paged_workspace_bytes(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win,
                                   int32_t n_streams);
int cs_launch_mv_rasterize(const cs_grid* g, int32_t n_frames, const cs_av_mv* mvs, const int64_t* mv_offsets,
                           cs_mb* out, cudaStream_t stream);
int cs_launch_similar_hist(const float* score, const uint8_t* frame_type, int64_t n_frames, int32_t n_patches,
                           const float* taus, int32_t n_tau, int32_t n_bins, unsigned long long* hist,
                           cudaStream_t stream);
size_t cs_score_compact_workspace_bytes(int32_t n_streams);
int cs_launch_score_compact(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                            const uint8_t* frame_type, int64_t type_stride, uint32_t* keep_mask,
                            int64_t frame_stride, uint32_t* gop_state, float* score, int32_t* kept_count,
                            const int32_t* frame_index, const void* const* frames, int32_t frame_layout,
                            int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                            int32_t* frame_offsets, void* workspace, unsigned long long* counters, int32_t* status,
                            const cs_chain* chain, cudaStream_t stream);
int cs_num_sms();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel slot, device); 0 on success
int cs_set_smem_attr(const void* func, int slot, int bytes);
