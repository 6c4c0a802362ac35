/*
 * oracle/codecsight_ref.h — the CodecSight hot-path ORACLE (test infrastructure only).
 *
 * A plain, slow, single-threaded CPU definition of what the path computes, written from the paper
 * (PAPER.md, cited P:n) and the readings recorded in DESIGN.md.  It shares no code, header, helper or
 * constant with the CUDA library: every type here is declared independently.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may load it.
 *
 * Host memory only.  Layouts match include/codecsight.h by specification, not by inclusion.
 */
#ifndef CODECSIGHT_REF_H_
#define CODECSIGHT_REF_H_
#include <stdint.h>

#define REF_FRAME_I 0
#define REF_FRAME_P 1
#define REF_MB_INTER 0
#define REF_MB_SKIP 1
#define REF_MB_INTRA 2
#define REF_DISP_NEW 0
#define REF_DISP_ANCHOR 1
#define REF_DISP_REUSE 2
#define REF_LAYOUT_PLANAR 0
#define REF_LAYOUT_GROUPED 1
#define REF_BF16 0
#define REF_FP32 1

#define REF_ST_CAPACITY 1
#define REF_ST_NO_IFRAME 2
#define REF_ST_ORIGIN 4
#define REF_ST_BAD_FRAME_TYPE 8
#define REF_ST_BAD_MB_TYPE 16

/* counter slots */
#define REF_C_FRAMES 0
#define REF_C_PFRAMES 1
#define REF_C_PATCHES 2
#define REF_C_KEPT 3
#define REF_C_NEAR_TAU 4
#define REF_C_TOK_REUSE 5
#define REF_C_TOK_ANCHOR 6
#define REF_C_TOK_NEW 7
#define REF_C_BYTES_SCORE 8
#define REF_C_BYTES_COMPACT 9
#define REF_C_BYTES_KV 10
#define REF_C_PACKED_ROWS 11
#define REF_C_STREAM_STEPS 12
#define REF_NCOUNTERS 16

typedef struct {
  int16_t mvx_qpel, mvy_qpel;
  uint16_t sad;
  uint8_t mb_type, reserved;
} ref_mb;

typedef struct {
  int32_t src_w, src_h, mb_size, mb_cols, mb_rows, patch, grid_w, grid_h, group;
  float tau, alpha;
} ref_grid;

typedef struct {
  int32_t layers, kv_heads, head_dim, dtype;
  int64_t capacity, refresh_capacity;
  double rope_base;
  int32_t n_prompt, rope_mode;
  int32_t mrope_section[3];
  int32_t t_per_frame;
} ref_kv;
#define REF_ROPE_1D 0
#define REF_ROPE_MROPE 1

typedef struct {
  int32_t window, stride, step, ring_frames;
} ref_window;

/* Eq. 1 for one macroblock. */
float codecsight_ref_mb_magnitude(int16_t dx_qpel, int16_t dy_qpel, uint8_t mb_type);

/* Resampling + Eq. 3 for one P-frame: V, R, M per patch ([grid_h*grid_w] each, any may be NULL). */
void codecsight_ref_patch_fields(const ref_grid* g, const ref_mb* mb, float* V, float* R, float* M,
                                 int32_t* status);

/* The three entry points (host pointers; same argument meaning as include/codecsight.h). */
int codecsight_ref_score_patches(const ref_grid* g, int32_t n_streams, int32_t n_frames, const ref_mb* mb,
                                 const uint8_t* frame_type, uint32_t* keep_mask, int64_t frame_stride,
                                 uint32_t* gop_state, float* score, int32_t* kept_count,
                                 unsigned long long* counters, int32_t* status);

int codecsight_ref_compact(const ref_grid* g, int32_t n_streams, int32_t n_frames, const uint32_t* keep_mask,
                           int64_t mask_frame_stride, const int32_t* frame_index, const void* const* frames,
                           int32_t frame_layout, int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                           int32_t* frame_offsets, unsigned long long* counters, int32_t* status);

int codecsight_ref_kv_refresh(const ref_grid* g, const ref_kv* kv, const ref_window* win, int32_t n_streams,
                              const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring,
                              const void* const* old_cache, void* const* new_cache,
                              const void* const* refreshed, int64_t token_cap, uint8_t* disposition,
                              int32_t* p_old, int32_t* n_tokens, unsigned long long* counters, int32_t* status);

/* NEXT-1: in-place / paged variant (per-stream row pools + slot maps). */
int codecsight_ref_kv_refresh_paged(const ref_grid* g, const ref_kv* kv, const ref_window* win, int32_t n_streams,
                                    const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring,
                                    void* const* pool, const int32_t* slot_old, int32_t* slot_new, int64_t slot_cap,
                                    const void* const* refreshed, int64_t token_cap, uint8_t* disposition,
                                    int32_t* p_old, int32_t* n_tokens, unsigned long long* counters,
                                    int32_t* status);

/* NEXT-2: NV12 -> RGB -> bilinear resize -> normalise, fused into the compaction. */
typedef struct {
  int32_t src_w, src_h, y_pitch, uv_pitch;
  int32_t color; /* 0 = BT.601 limited range */
  float mean[3], stdv[3];
} ref_pre;
void codecsight_ref_nv12_rgb(const uint8_t* Y, const uint8_t* UV, const ref_pre* pp, int64_t y, int64_t x,
                             float rgb[3]);
float codecsight_ref_model_pixel(const ref_grid* g, const ref_pre* pp, const uint8_t* Y, const uint8_t* UV, int64_t c,
                                 int64_t yo, int64_t xo);
void codecsight_ref_preprocess_frame(const ref_grid* g, const ref_pre* pp, const uint8_t* Y, const uint8_t* UV,
                                     uint16_t* out);
int codecsight_ref_compact_nv12(const ref_grid* g, const ref_pre* pp, int32_t n_streams, int32_t n_frames,
                                const uint32_t* keep_mask, int64_t mask_frame_stride, const int32_t* frame_index,
                                const void* const* y_planes, const void* const* uv_planes, int64_t capacity,
                                void* packed, int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets,
                                unsigned long long* counters, int32_t* status);

/* NEXT-3: temporal patches (Qwen2-VL temporal_patch_size): a token unit = tp consecutive frames, row [3][tp][p][p];
 * a group is emitted iff any of its patches is kept in any frame of the unit; unit masks (OR) optionally written,
 * and unit types (I iff any frame of the unit is not a P-frame) when frame_type and unit_type are given. */
int codecsight_ref_compact_tp(const ref_grid* g, int32_t tp, int32_t n_streams, int32_t n_units,
                              const uint32_t* keep_mask, int64_t mask_frame_stride, const int32_t* unit_index,
                              const void* const* frames, int32_t frame_layout, int64_t capacity, void* packed,
                              int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets, uint32_t* unit_mask,
                              int64_t unit_mask_stride, const uint8_t* frame_type, uint8_t* unit_type,
                              unsigned long long* counters, int32_t* status);

/* NEXT-4: FFmpeg AVMotionVector records -> MB grid; similar-patch-ratio histogram. */
typedef struct {
  int32_t source;
  uint8_t w, h;
  int16_t src_x, src_y, dst_x, dst_y;
  uint64_t flags;
  int32_t motion_x, motion_y;
  uint16_t motion_scale;
} ref_av_mv;
int codecsight_ref_mv_rasterize(const ref_grid* g, int32_t n_frames, const ref_av_mv* mvs, const int64_t* mv_offsets,
                                ref_mb* out);
int codecsight_ref_similar_hist(const float* score, const uint8_t* frame_type, int64_t n_frames, int32_t n_patches,
                                const float* taus, int32_t n_tau, int32_t n_bins, unsigned long long* hist);

/* Eq. 5 on one fp32 key vector of n_heads x head_dim: out = R(dp) k (rotate_half pairing). */
void codecsight_ref_rope_rotate_f32(const float* k, int32_t n_heads, int32_t head_dim, double base, int64_t dp,
                                    float* out);

#endif
