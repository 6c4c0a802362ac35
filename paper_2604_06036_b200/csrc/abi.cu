// abi.cu — the C ABI of libcodecsight: host-side argument validation, then the launchers of score.cu,
// compact.cu and kv_refresh.cu.  Declarations and the contract of every call: include/codecsight.h.
#include <math.h>

#include <atomic>

#include "cs_internal.cuh"

namespace {

constexpr int kMaxDevices = 64;
std::atomic<int> g_sms[kMaxDevices];
std::atomic<unsigned> g_attr_done[kMaxDevices];  // bit per kernel slot

int grid_ok(const cs_grid* g) {
  if (!g) return CS_ERR_INVALID_ARGUMENT;
  if (g->src_w < 1 || g->src_h < 1 || g->src_w > 16384 || g->src_h > 16384) return CS_ERR_SHAPE;
  if (g->mb_size < 1 || g->mb_size > 64) return CS_ERR_SHAPE;
  if (g->mb_cols != (g->src_w + g->mb_size - 1) / g->mb_size) return CS_ERR_SHAPE;
  if (g->mb_rows != (g->src_h + g->mb_size - 1) / g->mb_size) return CS_ERR_SHAPE;
  if (g->grid_w < 1 || g->grid_h < 1 || static_cast<long long>(g->grid_w) * g->grid_h > cs::kMaxGridPatches)
    return CS_ERR_SHAPE;
  if (g->group < 1 || g->grid_w % g->group != 0 || g->grid_h % g->group != 0) return CS_ERR_SHAPE;
  if (static_cast<long long>(g->mb_rows) * g->grid_w > cs::kMaxMbRowsTimesGridW) return CS_ERR_UNSUPPORTED;
  if (g->patch < 1 || g->patch > 32) return CS_ERR_SHAPE;
  if (isnan(g->tau) || g->tau < 0.0f) return CS_ERR_INVALID_ARGUMENT;
  if (isnan(g->alpha) || isinf(g->alpha) || g->alpha < 0.0f) return CS_ERR_INVALID_ARGUMENT;
  return CS_OK;
}

int device_ok() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    cudaGetLastError();
    return CS_ERR_CUDA;
  }
  return CS_OK;
}

}  // namespace

int cs_num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int n = g_sms[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    g_sms[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

int cs_set_smem_attr(const void* func, int slot, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  const unsigned bit = 1u << slot;
  if (g_attr_done[dev].load(std::memory_order_acquire) & bit) return 0;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return -1;
  g_attr_done[dev].fetch_or(bit, std::memory_order_release);
  return 0;
}

extern "C" {

static int kv_args_ok(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, int32_t n_streams,
                      int64_t token_cap);

int codecsight_version(void) { return 100; }

const char* codecsight_strerror(int code) {
  switch (code) {
    case CS_OK: return "ok";
    case CS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case CS_ERR_SHAPE: return "shape / dimension mismatch";
    case CS_ERR_UNSUPPORTED: return "unsupported configuration";
    case CS_ERR_CUDA: return "CUDA error";
    default: return "unknown error";
  }
}

int codecsight_score_patches(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                             const uint8_t* frame_type, uint32_t* keep_mask, int64_t frame_stride,
                             uint32_t* gop_state, float* score, int32_t* kept_count,
                             unsigned long long* counters, int32_t* status, cudaStream_t stream) {
  int rc = grid_ok(g);
  if (rc) return rc;
  if (n_streams < 0 || n_frames < 1 || n_frames > cs::kMaxFramesPerCall || frame_stride < n_frames)
    return CS_ERR_INVALID_ARGUMENT;
  if (n_streams == 0) return CS_OK;
  if (!mb || !frame_type || !keep_mask || !gop_state || !kept_count || !counters || !status)
    return CS_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(mb) & 7u) != 0) return CS_ERR_INVALID_ARGUMENT;
  if (g->mb_cols > 4096) return CS_ERR_UNSUPPORTED;
  if (static_cast<long long>(n_streams) * 8 > 0x7fffffffLL) return CS_ERR_UNSUPPORTED;
  if ((rc = device_ok())) return rc;
  return cs_launch_score(g, n_streams, n_frames, mb, frame_type, keep_mask, frame_stride, gop_state, score,
                         kept_count, counters, status, stream);
}

size_t codecsight_score_compact_workspace_size(int32_t n_streams) { return cs_score_compact_workspace_bytes(n_streams); }

int codecsight_score_compact_ex(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                                const uint8_t* frame_type, int64_t type_stride, uint32_t* keep_mask,
                                int64_t frame_stride, uint32_t* gop_state, float* score, int32_t* kept_count,
                                const int32_t* frame_index, const void* const* frames, int32_t frame_layout,
                                int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                                int32_t* frame_offsets, void* workspace, size_t workspace_bytes,
                                unsigned long long* counters, int32_t* status, uint32_t flags, const cs_chain* chain,
                                cudaStream_t stream) {
  int rc = grid_ok(g);
  if (rc) return rc;
  if (n_streams < 0 || n_frames < 1 || n_frames > cs::kMaxFramesPerCall || frame_stride < n_frames ||
      type_stride < n_frames || capacity < 0)
    return CS_ERR_INVALID_ARGUMENT;
  if ((flags & ~static_cast<uint32_t>(CS_LAUNCH_PDL)) != 0) return CS_ERR_INVALID_ARGUMENT;
  const bool pdl = (flags & CS_LAUNCH_PDL) != 0;
  if (pdl && (!chain || !chain->gop_ready || !chain->done || chain->depth < 2 || chain->depth > 8))
    return CS_ERR_INVALID_ARGUMENT;
  if (pdl && score) return CS_ERR_UNSUPPORTED;  // chained calls: no score output (it would race call g-2's)
  if (n_streams == 0) return CS_OK;
  if (!mb || !frame_type || !keep_mask || !gop_state || !kept_count || !counters || !status) return CS_ERR_INVALID_ARGUMENT;
  if (!frame_index || !frames || !frame_offsets || !workspace) return CS_ERR_INVALID_ARGUMENT;
  if (capacity > 0 && (!packed || !pos_ids || !src_index)) return CS_ERR_INVALID_ARGUMENT;
  if (frame_layout != CS_LAYOUT_PLANAR && frame_layout != CS_LAYOUT_GROUPED) return CS_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < cs_score_compact_workspace_bytes(n_streams)) return CS_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(workspace) & 7u) != 0) return CS_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(mb) & 7u) != 0) return CS_ERR_INVALID_ARGUMENT;
  if (g->mb_cols > 4096) return CS_ERR_UNSUPPORTED;
  const long long n_slots = static_cast<long long>(n_streams) * n_frames;
  if (n_slots * g->grid_w * g->grid_h >= 2147483648LL) return CS_ERR_UNSUPPORTED;
  if (g->group * g->patch > 32) return CS_ERR_UNSUPPORTED;
  if ((rc = device_ok())) return rc;
  return cs_launch_score_compact(g, n_streams, n_frames, mb, frame_type, type_stride, keep_mask, frame_stride,
                                 gop_state, score, kept_count, frame_index, frames, frame_layout, capacity, packed,
                                 pos_ids, src_index, frame_offsets, workspace, counters, status,
                                 pdl ? chain : nullptr, stream);
}

int codecsight_score_compact(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                             const uint8_t* frame_type, uint32_t* keep_mask, int64_t frame_stride,
                             uint32_t* gop_state, float* score, int32_t* kept_count, const int32_t* frame_index,
                             const void* const* frames, int32_t frame_layout, int64_t capacity, void* packed,
                             int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets, void* workspace,
                             size_t workspace_bytes, unsigned long long* counters, int32_t* status,
                             cudaStream_t stream) {
  return codecsight_score_compact_ex(g, n_streams, n_frames, mb, frame_type, frame_stride, keep_mask, frame_stride,
                                     gop_state, score, kept_count, frame_index, frames, frame_layout, capacity,
                                     packed, pos_ids, src_index, frame_offsets, workspace, workspace_bytes, counters,
                                     status, 0u, nullptr, stream);
}

int codecsight_compact(const cs_grid* g, int32_t n_streams, int32_t n_frames, const uint32_t* keep_mask,
                       int64_t mask_frame_stride, const int32_t* frame_index, const void* const* frames,
                       int32_t frame_layout, int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                       int32_t* frame_offsets, unsigned long long* counters, int32_t* status,
                       cudaStream_t stream) {
  int rc = grid_ok(g);
  if (rc) return rc;
  if (n_streams < 0 || n_frames < 1 || mask_frame_stride < n_frames || capacity < 0)
    return CS_ERR_INVALID_ARGUMENT;
  if (frame_layout != CS_LAYOUT_PLANAR && frame_layout != CS_LAYOUT_GROUPED) return CS_ERR_INVALID_ARGUMENT;
  const long long n_slots = static_cast<long long>(n_streams) * n_frames;
  if (n_slots * g->grid_w * g->grid_h >= 2147483648LL) return CS_ERR_UNSUPPORTED;
  if (g->group * g->patch > 32) return CS_ERR_UNSUPPORTED;
  if (!frame_offsets || !counters || !status) return CS_ERR_INVALID_ARGUMENT;
  if (n_slots > 0 && (!keep_mask || !frame_index || !frames)) return CS_ERR_INVALID_ARGUMENT;
  if (capacity > 0 && (!packed || !pos_ids || !src_index)) return CS_ERR_INVALID_ARGUMENT;
  if ((rc = device_ok())) return rc;
  return cs_launch_compact(g, n_streams, n_frames, keep_mask, mask_frame_stride, frame_index, frames, frame_layout,
                           capacity,
                           packed, pos_ids, src_index, frame_offsets, counters, status, stream);
}

int codecsight_compact_tp(const cs_grid* g, int32_t temporal_patch, int32_t n_streams, int32_t n_units,
                          const uint32_t* keep_mask, int64_t mask_frame_stride, const int32_t* unit_index,
                          const void* const* frames, int32_t frame_layout, int64_t capacity, void* packed,
                          int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets, uint32_t* unit_mask,
                          int64_t unit_mask_stride, const uint8_t* frame_type, uint8_t* unit_type,
                          unsigned long long* counters, int32_t* status, cudaStream_t stream) {
  int rc = grid_ok(g);
  if (rc) return rc;
  if (temporal_patch < 1 || temporal_patch > 4) return CS_ERR_UNSUPPORTED;
  if (n_streams < 0 || n_units < 1 || capacity < 0) return CS_ERR_INVALID_ARGUMENT;
  if (mask_frame_stride < static_cast<long long>(n_units) * temporal_patch) return CS_ERR_INVALID_ARGUMENT;
  if ((unit_mask || unit_type) && unit_mask_stride < n_units) return CS_ERR_INVALID_ARGUMENT;
  if ((frame_type == nullptr) != (unit_type == nullptr)) return CS_ERR_INVALID_ARGUMENT;
  if (frame_layout != CS_LAYOUT_PLANAR && frame_layout != CS_LAYOUT_GROUPED) return CS_ERR_INVALID_ARGUMENT;
  const long long n_slots = static_cast<long long>(n_streams) * n_units;
  if (n_slots * g->grid_w * g->grid_h >= 2147483648LL) return CS_ERR_UNSUPPORTED;
  if (g->group * g->patch > 32) return CS_ERR_UNSUPPORTED;
  // per-warp staging tile of one group (x 8 warps) must fit the 227 KB of shared memory
  const long long tile = (3ll * temporal_patch * g->group * g->group * g->patch * g->patch * 2 + 15) & ~15ll;
  if (8 * (tile + 4ll * ((g->grid_w * g->grid_h + 31) / 32)) > 227 * 1024) return CS_ERR_UNSUPPORTED;
  if (!frame_offsets || !counters || !status) return CS_ERR_INVALID_ARGUMENT;
  if (n_slots > 0 && (!keep_mask || !unit_index || !frames)) return CS_ERR_INVALID_ARGUMENT;
  if (capacity > 0 && (!packed || !pos_ids || !src_index)) return CS_ERR_INVALID_ARGUMENT;
  if ((rc = device_ok())) return rc;
  return cs_launch_compact_tp(g, temporal_patch, n_streams, n_units, keep_mask, mask_frame_stride, unit_index, frames,
                              frame_layout, capacity, packed, pos_ids, src_index, frame_offsets, unit_mask,
                              unit_mask_stride, frame_type, unit_type, counters, status, stream);
}

int codecsight_kv_refresh_paged(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, int32_t n_streams,
                                const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring, void* const* pool,
                                const int32_t* slot_old, int32_t* slot_new, int64_t slot_cap,
                                const void* const* refreshed, int64_t token_cap, uint8_t* disposition,
                                int32_t* p_old, int32_t* n_tokens, void* workspace, size_t workspace_bytes,
                                unsigned long long* counters, int32_t* status, cudaStream_t stream) {
  int rc = kv_args_ok(g, kv, win, n_streams, token_cap);
  if (rc == 1) return CS_OK;
  if (rc) return rc;
  if (slot_cap < 0) return CS_ERR_INVALID_ARGUMENT;
  if (kv->capacity > 262144) return CS_ERR_UNSUPPORTED;
  if (!keep_mask_ring || !frame_type_ring || !pool || !slot_new || !disposition || !p_old || !n_tokens ||
      !counters || !status || !workspace)
    return CS_ERR_INVALID_ARGUMENT;
  if (win->step >= 1 && !slot_old) return CS_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15u) != 0) return CS_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < cs_kv_paged_workspace_bytes(g, kv, win, n_streams)) return CS_ERR_INVALID_ARGUMENT;
  if ((rc = device_ok())) return rc;
  return cs_launch_kv_refresh_paged(g, kv, win, n_streams, keep_mask_ring, frame_type_ring, pool, slot_old,
                                    slot_new, slot_cap, refreshed, token_cap, disposition, p_old, n_tokens,
                                    workspace, counters, status, stream);
}

size_t codecsight_kv_refresh_paged_workspace_size(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win,
                                                  int32_t n_streams) {
  if (!g || !kv || !win || n_streams < 0 || win->window < 1 || kv->head_dim < 2 || kv->head_dim > cs::kMaxHeadDim ||
      g->group < 1 || kv->n_prompt < 0)
    return 0;
  return cs_kv_paged_workspace_bytes(g, kv, win, n_streams);
}

int codecsight_compact_nv12(const cs_grid* g, const cs_preprocess* pp, int32_t n_streams, int32_t n_frames,
                            const uint32_t* keep_mask, int64_t mask_frame_stride, const int32_t* frame_index,
                            const void* const* y_planes, const void* const* uv_planes, int64_t capacity,
                            void* packed, int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets,
                            unsigned long long* counters, int32_t* status, cudaStream_t stream) {
  int rc = grid_ok(g);
  if (rc) return rc;
  if (!pp) return CS_ERR_INVALID_ARGUMENT;
  if (pp->src_w < 2 || pp->src_h < 2 || (pp->src_w & 1) || (pp->src_h & 1) || pp->src_w > 16384 ||
      pp->src_h > 16384 || pp->y_pitch < pp->src_w || pp->uv_pitch < pp->src_w)
    return CS_ERR_SHAPE;
  if (pp->color != CS_COLOR_BT601_LIMITED) return CS_ERR_UNSUPPORTED;
  for (int c = 0; c < 3; ++c)
    if (!(pp->std[c] > 0.0f) || isnan(pp->mean[c])) return CS_ERR_INVALID_ARGUMENT;
  if (n_streams < 0 || n_frames < 1 || mask_frame_stride < n_frames || capacity < 0) return CS_ERR_INVALID_ARGUMENT;
  const long long n_slots = static_cast<long long>(n_streams) * n_frames;
  if (n_slots * g->grid_w * g->grid_h >= 2147483648LL) return CS_ERR_UNSUPPORTED;
  if (g->group * g->patch > 32) return CS_ERR_UNSUPPORTED;
  if (g->grid_w / g->group > 64 || g->grid_h / g->group > 64) return CS_ERR_UNSUPPORTED;  // source-byte count masks
  if (!frame_offsets || !counters || !status) return CS_ERR_INVALID_ARGUMENT;
  if (n_slots > 0 && (!keep_mask || !frame_index || !y_planes || !uv_planes)) return CS_ERR_INVALID_ARGUMENT;
  if (capacity > 0 && (!packed || !pos_ids || !src_index)) return CS_ERR_INVALID_ARGUMENT;
  if ((rc = device_ok())) return rc;
  return cs_launch_compact_nv12(g, pp, n_streams, n_frames, keep_mask, mask_frame_stride, frame_index, y_planes,
                                uv_planes, capacity, packed, pos_ids, src_index, frame_offsets, counters, status,
                                stream);
}

int codecsight_mv_rasterize(const cs_grid* g, int32_t n_frames, const cs_av_mv* mvs, const int64_t* mv_offsets,
                            cs_mb* out, cudaStream_t stream) {
  int rc = grid_ok(g);
  if (rc) return rc;
  if (n_frames < 0) return CS_ERR_INVALID_ARGUMENT;
  if (n_frames == 0) return CS_OK;
  if (!mvs || !mv_offsets || !out) return CS_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(out) & 7u) != 0) return CS_ERR_INVALID_ARGUMENT;
  if ((rc = device_ok())) return rc;
  return cs_launch_mv_rasterize(g, n_frames, mvs, mv_offsets, out, stream);
}

int codecsight_similar_hist(const float* score, const uint8_t* frame_type, int64_t n_frames, int32_t n_patches,
                            const float* taus, int32_t n_tau, int32_t n_bins, unsigned long long* hist,
                            cudaStream_t stream) {
  if (n_frames < 0 || n_patches < 1 || n_tau < 1 || n_bins < 1) return CS_ERR_INVALID_ARGUMENT;
  if (n_frames == 0) return CS_OK;
  if (!score || !frame_type || !taus || !hist) return CS_ERR_INVALID_ARGUMENT;
  if (n_frames * n_tau > (1ll << 40)) return CS_ERR_UNSUPPORTED;
  int rc;
  if ((rc = device_ok())) return rc;
  return cs_launch_similar_hist(score, frame_type, n_frames, n_patches, taus, n_tau, n_bins, hist, stream);
}

size_t codecsight_kv_refresh_workspace_size(const cs_kv_desc* kv, const cs_window* win, int32_t n_streams) {
  if (!kv || !win || n_streams < 0 || win->window < 1 || kv->head_dim < 2 || kv->head_dim > cs::kMaxHeadDim)
    return 0;
  return cs_kv_workspace_bytes(kv, win, n_streams);
}

static int kv_args_ok(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, int32_t n_streams,
                      int64_t token_cap) {
  int rc = grid_ok(g);
  if (rc) return rc;
  if (!kv || !win) return CS_ERR_INVALID_ARGUMENT;
  if (n_streams < 0 || token_cap < 0) return CS_ERR_INVALID_ARGUMENT;
  if (kv->dtype != CS_BF16 && kv->dtype != CS_FP32) return CS_ERR_UNSUPPORTED;
  if (kv->layers < 1 || kv->kv_heads < 1 || kv->head_dim < 2 || kv->head_dim > cs::kMaxHeadDim)
    return CS_ERR_UNSUPPORTED;
  if (kv->head_dim % 2 != 0) return CS_ERR_UNSUPPORTED;  // S:376 "odd head_dim"
  if (kv->capacity < 0 || kv->refresh_capacity < 0 || kv->n_prompt < 0) return CS_ERR_INVALID_ARGUMENT;
  if (!(kv->rope_base > 0.0)) return CS_ERR_INVALID_ARGUMENT;
  if (kv->rope_mode != CS_ROPE_1D && kv->rope_mode != CS_ROPE_MROPE) return CS_ERR_UNSUPPORTED;
  if (kv->rope_mode == CS_ROPE_MROPE) {
    if (kv->mrope_section[0] < 0 || kv->mrope_section[1] < 0 || kv->mrope_section[2] < 0 || kv->t_per_frame < 1)
      return CS_ERR_INVALID_ARGUMENT;
    if (kv->mrope_section[0] + kv->mrope_section[1] + kv->mrope_section[2] != kv->head_dim / 2) return CS_ERR_SHAPE;
  }
  const long long w = win->window, s = win->stride, k = win->step;
  if (w < 1 || s < 1 || k < 0) return CS_ERR_INVALID_ARGUMENT;
  if (s > w) return CS_ERR_UNSUPPORTED;
  if (win->ring_frames < (k >= 1 ? w + s : w)) return CS_ERR_SHAPE;
  if (w + s > cs::kMaxWindowPlusStride) return CS_ERR_UNSUPPORTED;
  if (n_streams == 0) return 1;  /* nothing to do */
  if (n_streams > 8192) return CS_ERR_UNSUPPORTED;
  const long long nw = (static_cast<long long>(g->grid_w) * g->grid_h + 31) / 32;
  if ((w + s) * nw * 4 > 96 * 1024) return CS_ERR_UNSUPPORTED;
  const long long ngroups = static_cast<long long>(g->grid_w / g->group) * (g->grid_h / g->group);
  if (w * ngroups + kv->n_prompt >= 2147483647LL || kv->capacity >= 2147483647LL ||
      kv->refresh_capacity >= 2147483647LL || (k * s + w) >= 2147483647LL)
    return CS_ERR_UNSUPPORTED;
  return CS_OK;
}

int codecsight_kv_refresh(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, int32_t n_streams,
                          const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring,
                          const void* const* old_cache, void* const* new_cache, const void* const* refreshed,
                          int64_t token_cap, uint8_t* disposition, int32_t* p_old, int32_t* n_tokens,
                          void* workspace, size_t workspace_bytes, unsigned long long* counters,
                          int32_t* status, cudaStream_t stream) {
  int rc = kv_args_ok(g, kv, win, n_streams, token_cap);
  if (rc == 1) return CS_OK;
  if (rc) return rc;
  const long long k = win->step;
  if (!keep_mask_ring || !frame_type_ring || !new_cache || !disposition || !p_old || !n_tokens || !counters ||
      !status || !workspace)
    return CS_ERR_INVALID_ARGUMENT;
  if (k >= 1 && !old_cache) return CS_ERR_INVALID_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15u) != 0) return CS_ERR_INVALID_ARGUMENT;
  if (workspace_bytes < cs_kv_workspace_bytes(kv, win, n_streams)) return CS_ERR_INVALID_ARGUMENT;
  if ((rc = device_ok())) return rc;
  return cs_launch_kv_refresh(g, kv, win, n_streams, keep_mask_ring, frame_type_ring, old_cache, new_cache,
                              refreshed, token_cap, disposition, p_old, n_tokens, workspace, workspace_bytes,
                              counters, status, stream);
}

}  // extern "C"
