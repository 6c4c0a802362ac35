/*
 * codecsight.h — C ABI of the CodecSight hot path on B200 (sm_100a).
 *
 * Paper: "CodecSight: Leveraging Video Codec Signals for Efficient Streaming VLM Inference"
 * (arXiv 2604.06036).  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n.
 *
 * The library implements three calls, each a plain-pointer, asynchronous, stream-ordered operation:
 *
 *   codecsight_score_patches  per-macroblock codec metadata -> patch scores -> keep mask
 *                             (Eq. 1-4, GOP accumulation, group-complete expansion)
 *   codecsight_compact        keep mask + frames -> packed ViT input, position ids, source index,
 *                             per-frame offsets ("executes the ViT only on the selected patches")
 *   codecsight_kv_refresh     sliding-window reuse/anchor/new token index + K/V gather with RoPE key
 *                             correction (Eq. 5) and value reuse, refreshed-row scatter
 *
 * Conventions (all calls):
 *  - Ownership: the caller owns every buffer.  The library allocates nothing, frees nothing and keeps no
 *    pointer after a call returns (SPEC single-owner stream state).
 *  - Pointers named "device" must be CUDA device (or managed) memory valid on the current device; host
 *    structs (cs_grid, cs_kv_desc, cs_window) are read during the call only.
 *  - Execution: every call validates its arguments on the host, then enqueues kernels on `stream` and returns
 *    without synchronising.  Calls are reentrant; concurrent calls on different streams with disjoint output
 *    buffers are allowed.
 *  - Synchronous errors: a negative return code means NOTHING was enqueued (except CS_ERR_CUDA, returned when a
 *    launch itself failed).  Device-detected conditions are OR-ed as CS_STATUS_* bits into the caller-owned
 *    device int32 `status` (never cleared by the library); read it after the stream is synchronised.
 *  - Counters: `counters` is a caller-owned device array of CS_NCOUNTERS u64, accumulated with atomic adds.
 *  - There is no CPU fallback: without a CUDA device the calls return CS_ERR_CUDA.
 */
#ifndef CODECSIGHT_H_
#define CODECSIGHT_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- synchronous return codes -------------------------------------------------------------------------- */
enum {
  CS_OK = 0,
  CS_ERR_INVALID_ARGUMENT = -1, /* NULL required pointer, negative count, NaN/negative tau or alpha             */
  CS_ERR_SHAPE = -2,            /* SPEC "dimension mismatch": mb grid != ceil(src/mb), group does
                                   not divide the patch grid, ring shorter than w+s, ...                          */
  CS_ERR_UNSUPPORTED = -3,      /* dtype not in {bf16,fp32}, odd head_dim, s > w, sizes above the
                                   documented limits                                                              */
  CS_ERR_CUDA = -4              /* a CUDA launch failed (cudaGetLastError), or no device                          */
};

/* ---- asynchronous status bits (OR-ed into *status on the device) ---------------------------------------- */
enum {
  CS_STATUS_CAPACITY = 1,       /* an output capacity was exceeded; writes beyond it were dropped (offsets and
                                   counts still report the full, unclamped sizes)                                */
  CS_STATUS_NO_IFRAME = 2,      /* a P-frame arrived on a stream whose GOP state was never initialised by an
                                   I-frame; the accumulated state is taken as empty (reading Q11)                */
  CS_STATUS_ORIGIN = 4,         /* an ANCHOR/REUSE token's p_old lies outside the old cache's capacity (the
                                   previous window was truncated; SPEC "origin mismatch"); row skipped    */
  CS_STATUS_BAD_FRAME_TYPE = 8, /* frame type not in {I, P} (B-frames are out of scope, S:8); treated as I       */
  CS_STATUS_BAD_MB_TYPE = 16,   /* macroblock type not in {INTER, SKIP, INTRA}; treated as INTRA (dynamic)        */
  CS_STATUS_MISALIGNED = 32     /* kv_refresh: a stream's cache / pool / refreshed buffer violates the alignment
                                   rule below; no K/V row of that stream is moved (its index outputs are written)  */
};

enum { CS_FRAME_I = 0, CS_FRAME_P = 1 };
enum { CS_MB_INTER = 0, CS_MB_SKIP = 1, CS_MB_INTRA = 2 };
enum { CS_DISP_NEW = 0, CS_DISP_ANCHOR = 1, CS_DISP_REUSE = 2 };
enum { CS_BF16 = 0, CS_FP32 = 1 };
enum { CS_LAYOUT_PLANAR = 0, CS_LAYOUT_GROUPED = 1 }; /* model-input frame layouts accepted by codecsight_compact */

/* ---- counters (u64 each) -------------------------------------------------------------------------------- */
enum {
  CS_CNT_FRAMES = 0,        /* frames scored (I + P)                                                          */
  CS_CNT_PFRAMES = 1,       /* P-frames scored                                                                */
  CS_CNT_PATCHES = 2,       /* patches scored (= frames x grid_h x grid_w)                                    */
  CS_CNT_KEPT = 3,          /* patches kept (group-complete mask)                                             */
  CS_CNT_NEAR_TAU = 4,      /* P-frame patches with finite M and |M - tau| <= 1e-5 (north star)               */
  CS_CNT_TOK_REUSE = 5,     /* kv_refresh: REUSE tokens                                                       */
  CS_CNT_TOK_ANCHOR = 6,    /* kv_refresh: ANCHOR tokens                                                      */
  CS_CNT_TOK_NEW = 7,       /* kv_refresh: NEW tokens including prompt rows                                   */
  CS_CNT_BYTES_SCORE = 8,   /* algorithmic bytes of score_patches             */
  CS_CNT_BYTES_COMPACT = 9, /* algorithmic bytes of compact                                                    */
  CS_CNT_BYTES_KV = 10,     /* algorithmic bytes of the K/V row moves of kv_refresh                            */
  CS_CNT_PACKED_ROWS = 11,  /* compact: packed rows written                                                   */
  CS_CNT_STREAM_STEPS = 12, /* kv_refresh: stream-window steps processed                                       */
  CS_NCOUNTERS = 16
};

/* One coded macroblock of a P-frame (D2 in SURVEY §2.2).  8 bytes, no padding.
 *   mvx_qpel, mvy_qpel : motion vector in QUARTER-pel units of the source (displayed) frame (reading Q2)
 *   sad                : sum of absolute differences of the block vs its prediction (Eq. 2)
 *   mb_type            : CS_MB_INTER | CS_MB_SKIP | CS_MB_INTRA                                           */
typedef struct {
  int16_t mvx_qpel;
  int16_t mvy_qpel;
  uint16_t sad;
  uint8_t mb_type;
  uint8_t reserved;
} cs_mb;

/* Frame / macroblock / patch geometry and the pruning policy parameters.
 * Limits: 1 <= src_w, src_h <= 16384; 1 <= mb_size <= 64; mb_cols == ceil(src_w/mb_size) and
 * mb_rows == ceil(src_h/mb_size) (coded grid, reading Q3); 1 <= grid_w, grid_h; grid_w*grid_h <= 4096;
 * group >= 1 divides grid_w and grid_h; mb_rows*grid_w <= 8192; 1 <= patch and group*patch <= 32 (the
 * compaction calls: a group's pixel rows fit one warp; else CS_ERR_UNSUPPORTED);
 * tau >= 0 (may be +inf), alpha >= 0 finite.                                                                 */
typedef struct {
  int32_t src_w, src_h;     /* displayed source size in px (448x448, 1920x1080, 3840x2160)                   */
  int32_t mb_size;          /* 16                                                                           */
  int32_t mb_cols, mb_rows; /* coded MB grid = ceil(src/mb_size): 28x28, 120x68, 240x135                     */
  int32_t patch;            /* ViT patch edge in model px (14)                                              */
  int32_t grid_w, grid_h;   /* patch grid of the model input (32x32 for 448x448)                             */
  int32_t group;            /* spatial merge group edge (2: 2x2 patches -> one LLM token)             */
  float tau;                /* threshold in source px, default 0.25; dynamic iff M >= tau (Eq. 4)   */
  float alpha;              /* residual weight of Eq. 3, default 0                                  */
} cs_grid;

/* grid_words = ceil(grid_w*grid_h / 32): u32 words of one patch bitmap; patch i = h*grid_w + w is bit (i%32)
 * of word (i/32).                                                                                            */

/* ------------------------------------------------------------------------------------------------------------
 * codecsight_score_patches — Eq. 1-4 + GOP accumulation + group-complete expansion.
 *
 * Per stream sigma and new frame j (time order), for a P-frame:
 *   v_m   = |mv_m| / 4 px (Eq. 1); INTRA (or unknown type) MBs have v_m = +inf.
 *   V(i)  = max of v_m over MBs whose rectangle overlaps patch i with positive area; R(i) = area-weighted
 *           mean per-pixel |residual| / 255 (resampling).
 *   M(i)  = V(i) + alpha*R(i) (Eq. 3, one fp32 fma), dynamic(i) = M(i) >= tau (Eq. 4).
 *   state = state OR dynamic (GOP accumulation); out = state.
 * For an I-frame: state = empty, out = all patches, score = +inf, metadata not read (reading Q7, Q10).
 * keep = group-complete expansion of out: a group is kept iff any of its patches is in out.
 *
 *   g            host   geometry and policy
 *   n_streams    >= 0   streams in this call (0 = no-op)
 *   n_frames     1..256 new frames per stream (the stride s; w for the first window)
 *   mb           device [n_streams][n_frames][mb_rows][mb_cols] cs_mb; I-frame slots are not read.
 *                       16-B alignment of `mb` enables the bulk-copy (TMA) path.
 *   frame_type   device [n_streams][frame_stride] u8 CS_FRAME_*, frame j of stream sigma at sigma*frame_stride+j
 *   keep_mask    device [n_streams][frame_stride][grid_words] u32 out (same slot addressing as frame_type,
 *                       so a caller can point both at the slots of a per-stream ring)
 *   frame_stride >= n_frames
 *   gop_state    device [n_streams][grid_words+1] u32 in/out: accumulated patch bits, then a flag word whose
 *                       bit 0 = "initialised by an I-frame".  Zero-initialise for a new stream.
 *   score        device [n_streams][n_frames][grid_h*grid_w] fp32 out: M(i) (+inf for I-frames); NULL = skip
 *   kept_count   device [n_streams][n_frames] i32 out: kept patches (a multiple of group^2)
 *   counters     device [CS_NCOUNTERS] u64 (FRAMES, PFRAMES, PATCHES, KEPT, NEAR_TAU, BYTES_SCORE)
 *   status       device i32 (NO_IFRAME, BAD_FRAME_TYPE, BAD_MB_TYPE)
 * --------------------------------------------------------------------------------------------------------- */
int codecsight_score_patches(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                             const uint8_t* frame_type, uint32_t* keep_mask, int64_t frame_stride,
                             uint32_t* gop_state, float* score, int32_t* kept_count,
                             unsigned long long* counters, int32_t* status, cudaStream_t stream);

/* ------------------------------------------------------------------------------------------------------------
 * codecsight_compact — stream compaction of kept patches into the packed ViT input.
 *
 * The batch is n_streams x n_frames frames, flattened stream-major: slot = sigma*n_frames + j.
 * A group (group x group patches) is emitted iff any of its patches has its keep bit set; every emitted group
 * contributes all group^2 patches (group-complete, idempotent on masks produced by score_patches).
 * Order (reading Q14, "group-major"): slot, then group row-major, then patch (dy, dx) row-major in the group.
 * For the n-th emitted patch (h, w) of slot `slot` whose stream-local frame index is t:
 *   packed[n][c][y][x] = frame[slot][c][patch*h + y][patch*w + x]   (bit copy, c < 3, y, x < patch)
 *   pos_ids[n]         = (t, h, w)                                   (reading Q15)
 *   src_index[n]       = slot*grid_h*grid_w + h*grid_w + w
 * frame_offsets[slot] = exclusive scan of emitted patches per slot; frame_offsets[n_slots] = total
 * (cu_seqlens for a varlen ViT).  Rows n >= capacity are not written (CS_STATUS_CAPACITY); offsets are not clamped.
 *
 *   keep_mask         device [n_streams][mask_frame_stride][grid_words] u32, frame j of stream sigma at
 *                            sigma*mask_frame_stride + j (mask_frame_stride >= n_frames)
 *   frame_index       device [n_slots] i32 stream-local absolute frame index (pos id t)
 *   frames            device [n_slots] array of device pointers to bf16 model-input frames (the preprocessed
 *                            frames) in `frame_layout`:
 *                            CS_LAYOUT_PLANAR  [3][grid_h*patch][grid_w*patch] (the usual CHW tensor)
 *                            CS_LAYOUT_GROUPED [n_groups][group*group][3][patch][patch]: groups row-major, the
 *                              patches of a group (dy, dx) row-major -- i.e. already in packed order, so a kept
 *                              group is one contiguous block (what a fused resize/normalise stage can emit, NEXT-2)
 *                            8-B (planar) / 16-B (grouped) alignment enables wide loads
 *   frame_layout      CS_LAYOUT_PLANAR | CS_LAYOUT_GROUPED (results are identical for both)
 *   capacity          rows available in packed / pos_ids / src_index
 *   packed            device [capacity][3*patch*patch] bf16 out
 *   pos_ids           device [capacity][3] i32 out
 *   src_index         device [capacity] i32 out
 *   frame_offsets     device [n_slots+1] i32 out
 *   counters          BYTES_COMPACT, PACKED_ROWS;  status: CAPACITY
 * n_slots * grid_h * grid_w must be < 2^31.
 * --------------------------------------------------------------------------------------------------------- */
int codecsight_compact(const cs_grid* g, int32_t n_streams, int32_t n_frames, const uint32_t* keep_mask,
                       int64_t mask_frame_stride, const int32_t* frame_index, const void* const* frames,
                       int32_t frame_layout, int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                       int32_t* frame_offsets, unsigned long long* counters, int32_t* status,
                       cudaStream_t stream);

/* ------------------------------------------------------------------------------------------------------------
 * codecsight_score_compact — NEXT-2: scoring and compaction fused into ONE kernel pass ("single batched operation",
 * P:268, over the pruned patches).  Results are bit-identical to codecsight_score_patches followed by
 * codecsight_compact(keep_mask, mask_frame_stride = frame_stride) on the same arguments -- every output of both
 * calls (keep_mask, gop_state, score, kept_count, packed, pos_ids, src_index, frame_offsets), the counters of both
 * and the status bits of both.  Each stream's cluster scores its frames, then finds its offset in the packed batch
 * by a decoupled look-back over the streams (no separate scan pass, no mask round trip through a second launch) and
 * copies its kept groups.
 *   workspace       device, >= codecsight_score_compact_workspace_size(n_streams) bytes, 8-B aligned, ZERO-FILLED
 *                   once by the caller before first use; every call leaves it zeroed again.  One call at a time
 *                   per workspace (calls on different CUDA streams need different workspaces).
 *   other arguments as codecsight_score_patches and codecsight_compact (frame_index / frames / frame_layout /
 *   capacity / packed / pos_ids / src_index / frame_offsets over the n_streams x n_frames slots).
 * n_streams == 0 enqueues nothing (frame_offsets untouched).
 * --------------------------------------------------------------------------------------------------------- */
/* codecsight_score_compact_ex — the same call with two launch options:
 *   type_stride   row stride (frames) of frame_type, which may then be the step's own [n_streams][type_stride]
 *                 input array instead of the mask ring's type slots (codecsight_score_compact: = frame_stride)
 *   flags         CS_LAUNCH_PDL: a CHAINED call g (chain->generation = g = 0, 1, 2, ... on one chain of depth
 *                 d = chain->depth, 2 <= d <= 8), launched as a programmatic dependent of the preceding kernel on
 *                 `stream` (the preceding chained call g-1): its stream ticket, MB loads and scoring passes run
 *                 while earlier calls are still compacting; it then waits until chain->gop_ready[s] == g (call g-1
 *                 published stream s's final GOP state) and until chain->done[g mod d] >= g-d+1 (call g-d, whose
 *                 output buffers it reuses, has completed), computes, and publishes gop_ready[s] = g+1 and, when
 *                 its last CTA finishes, done[g mod d] = g+1 (release stores; the waits are acquire spins on calls
 *                 that are already resident, so they cannot deadlock).  Successive chained calls therefore overlap
 *                 each other's scoring and compaction.  Requirements: gop_ready [n_streams] and done [d] device
 *                 u32, zero before call 0, the same n_streams on every call of a chain; call g's workspace differs
 *                 from calls g-1 .. g-d's (rotate d + 1); call g writes the outputs kept_count, packed, pos_ids,
 *                 src_index and frame_offsets that call g-d wrote (rotate d sets); mb, frame_type and frames are
 *                 not written by the preceding kernels; score must be NULL (else CS_ERR_UNSUPPORTED).  Results are
 *                 identical to plain calls.  (Other flag bits, or CS_LAUNCH_PDL without a valid chain:
 *                 CS_ERR_INVALID_ARGUMENT.)
 */
enum { CS_LAUNCH_PDL = 1 };
typedef struct {
  uint32_t* gop_ready;  /* device [n_streams]  */
  uint32_t* done;       /* device [depth]      */
  uint32_t generation;  /* this call's index g */
  uint32_t depth;       /* output buffer sets  */
} cs_chain;
int codecsight_score_compact_ex(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                                const uint8_t* frame_type, int64_t type_stride, uint32_t* keep_mask,
                                int64_t frame_stride, uint32_t* gop_state, float* score, int32_t* kept_count,
                                const int32_t* frame_index, const void* const* frames, int32_t frame_layout,
                                int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                                int32_t* frame_offsets, void* workspace, size_t workspace_bytes,
                                unsigned long long* counters, int32_t* status, uint32_t flags,
                                const cs_chain* chain, cudaStream_t stream);
size_t codecsight_score_compact_workspace_size(int32_t n_streams);
int codecsight_score_compact(const cs_grid* g, int32_t n_streams, int32_t n_frames, const cs_mb* mb,
                             const uint8_t* frame_type, uint32_t* keep_mask, int64_t frame_stride,
                             uint32_t* gop_state, float* score, int32_t* kept_count, const int32_t* frame_index,
                             const void* const* frames, int32_t frame_layout, int64_t capacity, void* packed,
                             int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets, void* workspace,
                             size_t workspace_bytes, unsigned long long* counters, int32_t* status,
                             cudaStream_t stream);

/* ------------------------------------------------------------------------------------------------------------
 * codecsight_compact_tp — NEXT-3: temporal patches.  Qwen2-VL / Qwen3-VL embed video with
 * temporal_patch_size 2: one visual token covers `temporal_patch` consecutive frames and its patch row is
 * [3][temporal_patch][patch][patch] (channel, frame, y, x -- the Hugging Face processor's flatten order).
 * Token unit u of stream sigma = frames u*tp .. u*tp+tp-1 of the stream: their bf16 frames are
 * frames[(sigma*n_units + u)*tp + f] and their masks keep_mask[sigma][u*tp + f] (f < tp).  Reading: a group of the
 * unit is emitted iff any of its patches is kept in ANY frame of the unit (the union keeps every dynamic pixel).
 *   packed[n][c][f][y][x] = frame f of the unit, pixel (c, patch*h + y, patch*w + x)
 *   pos_ids[n] = (unit_index[slot], h, w); src_index[n] = slot*grid_h*grid_w + h*grid_w + w; slot = sigma*n_units+u
 *   unit_mask  optional device [n_streams][unit_mask_stride][grid_words] u32 out: OR of the unit's frame masks
 *              (the per-unit mask a token-unit KV ring is built from); NULL = not written
 *   frame_type, unit_type  optional together: frame_type device [n_streams][mask_frame_stride] u8 (the frame type
 *              ring), unit_type device [n_streams][unit_mask_stride] u8 out = CS_FRAME_P iff every frame of the
 *              unit is a P-frame, else CS_FRAME_I (a unit holding an I-frame is an anchor of the KV refresh)
 * Order, offsets, capacity and status as codecsight_compact (rows of 3*tp*patch^2 bf16); temporal_patch = 1 is
 * codecsight_compact.  A clip whose length is not a multiple of tp repeats its last frame (pass the same pointer
 * and mask twice), as the Hugging Face processor does.  Limits: 1 <= temporal_patch <= 4; 8 tiles of
 * 3*tp*(group*patch)^2 bf16 fit 227 KB of shared memory (else CS_ERR_UNSUPPORTED).
 *   counters: BYTES_COMPACT (+ 4*tp*grid_words+4 per unit, + 4*grid_words per unit mask and tp+1 per unit type
 *             written), PACKED_ROWS
 * --------------------------------------------------------------------------------------------------------- */
int codecsight_compact_tp(const cs_grid* g, int32_t temporal_patch, int32_t n_streams, int32_t n_units,
                          const uint32_t* keep_mask, int64_t mask_frame_stride, const int32_t* unit_index,
                          const void* const* frames, int32_t frame_layout, int64_t capacity, void* packed,
                          int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets, uint32_t* unit_mask,
                          int64_t unit_mask_stride, const uint8_t* frame_type, uint8_t* unit_type,
                          unsigned long long* counters, int32_t* status, cudaStream_t stream);

/* ------------------------------------------------------------------------------------------------------------
 * codecsight_compact_nv12 — NEXT-2: the GPU preprocessing fused into the compaction ("Resizing, color-space
 * conversion, and normalization are fused into a single batched operation over all frames"): the frames are the
 * decoder's NV12 output and only the kept groups are converted, resized and normalised -- pruned patches are never
 * preprocessed.  A model-input pixel (c, y, x) of the (grid_h*patch) x (grid_w*patch) input is, in fp32 and in
 * this order:
 *   colour  BT.601 limited range: R = 1.164383(Y-16) + 1.596027(V-128), G = (1.164383(Y-16) - 0.391762(U-128))
 *           - 0.812968(V-128), B = 1.164383(Y-16) + 2.017232(U-128), each clamped to [0, 255]; the chroma of
 *           source pixel (y, x) is UV[y/2][2(x/2)], UV[y/2][2(x/2)+1]
 *   resize  bilinear with half-pixel centres (PyTorch interpolate, align_corners=False, no antialias):
 *           f = (o + 0.5)(src/M) - 0.5 clamped at 0, i0 = floor f, i1 = i0 + (i0 < src-1), l = f - i0,
 *           v = (1-ly)((1-lx)p00 + lx p01) + ly((1-lx)p10 + lx p11)
 *   scale   out = (v/255 - mean[c]) / std[c], stored bf16 (RNE)
 * Outputs, order and capacity semantics are those of codecsight_compact.
 *   pp         host  source geometry and normalisation
 *   y_planes   device [n_slots] device pointers to Y planes   [src_h][y_pitch] u8
 *   uv_planes  device [n_slots] device pointers to UV planes  [src_h/2][uv_pitch] u8 (U, V interleaved)
 * --------------------------------------------------------------------------------------------------------- */
enum { CS_COLOR_BT601_LIMITED = 0 };
typedef struct {
  int32_t src_w, src_h;      /* decoded frame size in px, even, <= 16384                                     */
  int32_t y_pitch, uv_pitch; /* bytes per row of the Y and UV planes (>= src_w)                              */
  int32_t color;             /* CS_COLOR_BT601_LIMITED                                                       */
  float mean[3], std[3];     /* per-channel normalisation of v/255 (Qwen2-VL / CLIP: 0.4815 0.4578 0.4082,
                                0.2686 0.2613 0.2758)                                                        */
} cs_preprocess;

int codecsight_compact_nv12(const cs_grid* g, const cs_preprocess* pp, int32_t n_streams, int32_t n_frames,
                            const uint32_t* keep_mask, int64_t mask_frame_stride, const int32_t* frame_index,
                            const void* const* y_planes, const void* const* uv_planes, int64_t capacity,
                            void* packed, int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets,
                            unsigned long long* counters, int32_t* status, cudaStream_t stream);

/* KV cache description.  One cache buffer (one stream, one window) is laid out as
 *   [layers][2 (K, V)][capacity][kv_heads][head_dim]  of dtype,
 * so one (token, layer, K-or-V) row is kv_heads*head_dim contiguous elements.                                */
typedef struct {
  int32_t layers, kv_heads, head_dim; /* 28, 4, 128 (Qwen2-VL-7B shape) | toy 2, 2, 16; head_dim even <= 512 */
  int32_t dtype;                      /* CS_BF16 | CS_FP32                                                    */
  int64_t capacity;                   /* token rows per cache buffer                                          */
  int64_t refresh_capacity;           /* token rows per refreshed (recompute) buffer                          */
  double rope_base;                   /* 1e4 (S:355 default) | 1e6 (Qwen2)                                    */
  int32_t n_prompt;                   /* prompt rows after the visual tokens; always NEW        */
  int32_t rope_mode;                  /* CS_ROPE_1D | CS_ROPE_MROPE (below)                                   */
  int32_t mrope_section[3];           /* M-RoPE: frequency pairs of the t / h / w sections, sum = head_dim/2
                                         (Qwen2-VL: 16, 24, 24)                                               */
  int32_t t_per_frame;                /* M-RoPE: temporal position units per consumed frame (>= 1)            */
} cs_kv_desc;

/* Rotary position schemes of the cached keys (Eq. 5; reading Q19 and NEXT-3):
 *   CS_ROPE_1D    one position per token = its compacted sequence index (reading Q16); R(dp) rotates every
 *                 frequency pair i by dp * base^(-2i/D), dp = p_new - p_old.
 *   CS_ROPE_MROPE multimodal RoPE (Qwen2-VL / Qwen3-VL): a visual token of frame f, group (gr, gc) has position
 *                 (t, h, w) = ((f - ks) * t_per_frame, gr, gc) in window k, pair i < s_t rotates with t, the next
 *                 s_h pairs with h, the last s_w with w.  A reused token keeps (h, w) and moves in time by
 *                 dt = -stride * t_per_frame, so only the temporal section is rotated.                          */
enum { CS_ROPE_1D = 0, CS_ROPE_MROPE = 1 };

/* Sliding window: window k covers frames [k*stride, k*stride + window).                   */
typedef struct {
  int32_t window, stride; /* w, s with 1 <= s <= w                                                 */
  int32_t step;           /* k >= 0 (window index)                                                         */
  int32_t ring_frames;    /* slots in the per-stream mask/type ring; frame f lives in slot f % ring_frames;
                             must be >= w + s for k >= 1 (>= w for k = 0)                                   */
} cs_window;

/* ------------------------------------------------------------------------------------------------------------
 * codecsight_kv_refresh — selective KVC refresh for window k of every stream.
 *
 * Tokens of window k (reading Q16): visual tokens in (frame, group row-major) order over frames [ks, ks+w),
 * one per emitted group (as in codecsight_compact), followed by n_prompt prompt rows.  n_f = tokens of frame f.
 *   p_new(f, g) = sum_{f' in [ks, f)} n_f' + rank_f(g);  p_old(f, g) = sum_{f' in [(k-1)s, f)} n_f' + rank_f(g)
 *   disposition: f >= (k-1)s + w          -> NEW      (frames that arrived with this stride)
 *                else type(f) == I or f == ks -> ANCHOR (I-frame anchors; first overlap frame, Q17)
 *                else                      -> REUSE
 *   prompt rows: p_new = n_visual + j, NEW.  k == 0: every token NEW.
 * REUSE (Eq. 5), for every layer l:  K_new[l][p_new] = R(p_new - p_old) K_old[l][p_old]  (rotate_half
 *   pairing (i, i + D/2), inv_freq_i = base^(-2i/D), fp64 angle -> fp32 cos/sin, fp32 fma, RNE store; Q19-Q21)
 *   and V_new[l][p_new] = V_old[l][p_old] (bit copy).
 * Non-REUSE tokens (ANCHOR, NEW, prompt), in p_new order, take row r = 0, 1, ... of `refreshed` (bit copy of K and
 * V for all layers) if `refreshed` is not NULL; otherwise those rows of new_cache are left untouched for the
 * prefill (Q18).
 *
 *   keep_mask_ring    device [n_streams][ring_frames][grid_words] u32 (masks from score_patches)
 *   frame_type_ring   device [n_streams][ring_frames] u8
 *   Alignment: when a row (H * D * element size bytes) is a multiple of 16 B, rows move by 16-B vectors and TMA
 *   bulk copies, so every old_cache / new_cache / refreshed pointer must be 16-B aligned; otherwise element
 *   aligned.  The pointers live in device arrays, so this is checked on the device: a stream that violates it
 *   raises CS_STATUS_MISALIGNED and none of its rows move (never a misaligned-access fault).
 *   old_cache         device array [n_streams] of device pointers to window k-1 caches (not read when k == 0)
 *   new_cache         device array [n_streams] of device pointers to window k caches; must not alias old_cache
 *   refreshed         device array [n_streams] of device pointers to [layers][2][refresh_capacity][H][D]
 *                            recompute buffers, or NULL
 *   token_cap         per-stream capacity of the index outputs
 *   disposition       device [n_streams][token_cap] u8 out, indexed by p_new
 *   p_old             device [n_streams][token_cap] i32 out, -1 for NEW
 *   n_tokens          device [n_streams][4] i32 out: n_visual, n_reuse, n_anchor, n_new (incl. prompt)
 *   workspace         device scratch of >= codecsight_kv_refresh_workspace_size() bytes, 16-B aligned; its
 *                            content is undefined after the call (the per-stream plan segments)
 *   counters          TOK_REUSE, TOK_ANCHOR, TOK_NEW, BYTES_KV, STREAM_STEPS;  status: CAPACITY, ORIGIN
 * Rows with p_new >= min(capacity, token_cap) and refreshed rows r >= refresh_capacity are dropped
 * (CS_STATUS_CAPACITY); n_tokens reports the unclamped counts.
 * --------------------------------------------------------------------------------------------------------- */
int codecsight_kv_refresh(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, int32_t n_streams,
                          const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring,
                          const void* const* old_cache, void* const* new_cache, const void* const* refreshed,
                          int64_t token_cap, uint8_t* disposition, int32_t* p_old, int32_t* n_tokens,
                          void* workspace, size_t workspace_bytes, unsigned long long* counters,
                          int32_t* status, cudaStream_t stream);

/* ------------------------------------------------------------------------------------------------------------
 * codecsight_kv_refresh_paged — the same window step with the KV cache kept resident and updated IN PLACE
 * ("maintains the previous window's KV cache resident in GPU memory and performs these updates in-place", P:363;
 * SURVEY NEXT-1).  Each stream owns a pool of kv->capacity physical rows, laid out like a cache buffer
 * [layers][2][capacity][H][D]; a window's token p lives in row slot_map[p].
 *   tokens, dispositions, p_old, n_tokens: exactly as codecsight_kv_refresh.
 *   REUSE  : keeps slot_old[p_old]; its key rows are rotated in place by R(p_new - p_old) (Eq. 5); values are not
 *            touched.
 *   ANCHOR : keeps slot_old[p_old]; its K and V rows are overwritten with refreshed row r (if refreshed != NULL).
 *   NEW    : (new frames, then prompt rows) take the free slots -- slots not held by a REUSE/ANCHOR token --
 *            in ascending slot order, in p_new order; rows copied from refreshed row r (if refreshed != NULL).
 * Only keys of reused tokens move: 57,344 B per reused token instead of 114,688 B (Qwen2-VL-7B bf16).
 *
 *   pool        device array [n_streams] of device pointers to the row pools (in/out; pool and refreshed
 *               pointers follow codecsight_kv_refresh's alignment rule, else CS_STATUS_MISALIGNED)
 *   slot_old    device [n_streams][slot_cap] i32: slots of window k-1 (read when k >= 1; entries outside
 *               [0, capacity) raise CS_STATUS_ORIGIN and the token gets no row)
 *   slot_new    device [n_streams][slot_cap] i32 out: slots of window k (-1 = no row); must not alias slot_old
 *   slot_cap    per-stream length of the slot maps
 *   workspace   >= codecsight_kv_refresh_paged_workspace_size() bytes, 16-B aligned
 *   other arguments as codecsight_kv_refresh.  CS_STATUS_CAPACITY when a NEW token finds no free slot.
 * Limits: capacity <= 262144 rows per stream.
 * --------------------------------------------------------------------------------------------------------- */
int codecsight_kv_refresh_paged(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win, int32_t n_streams,
                                const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring, void* const* pool,
                                const int32_t* slot_old, int32_t* slot_new, int64_t slot_cap,
                                const void* const* refreshed, int64_t token_cap, uint8_t* disposition,
                                int32_t* p_old, int32_t* n_tokens, void* workspace, size_t workspace_bytes,
                                unsigned long long* counters, int32_t* status, cudaStream_t stream);

/* Bytes of device workspace codecsight_kv_refresh_paged needs (0 on bad args). */
size_t codecsight_kv_refresh_paged_workspace_size(const cs_grid* g, const cs_kv_desc* kv, const cs_window* win,
                                                  int32_t n_streams);

/* ------------------------------------------------------------------------------------------------------------
 * NEXT-4 — real H.264 metadata ingest and the similar-patch analysis.
 *
 * cs_av_mv is FFmpeg's AVMotionVector (libavutil/motion_vector.h, 40 bytes): the per-partition motion a software
 * H.264 decoder exports (the "MV extraction" of the Codec Processor).
 *
 * codecsight_mv_rasterize: frame f's records mvs[mv_offsets[f] .. mv_offsets[f+1]) -> out[f] = its
 * [mb_rows][mb_cols] cs_mb grid (the input of codecsight_score_patches).  Partition = destination rectangle
 * [dst_x - w/2, dst_x - w/2 + w) x [dst_y - h/2, ...) px; an MB takes the motion vector of largest magnitude among
 * the past-reference partitions (source < 0) overlapping it with positive area (ties: the earliest record) -- the
 * conservative max of the patch resampling -- in quarter pel, trunc(4 * motion / motion_scale) clamped to
 * int16, type INTER; an MB no partition covers was intra coded (FFmpeg exports no motion for it): INTRA.  SAD is not
 * exported by FFmpeg: 0 (use alpha = 0).
 *   mvs         device cs_av_mv records;  mv_offsets device [n_frames+1] i64;  out device [n_frames][rows][cols],
 *               8-B aligned (used as scratch while arbitrating).
 *
 * codecsight_similar_hist: fig:mv_residual_analysis_cdf.  For every P-frame f and threshold
 * taus[t]: count = #{i : score[f][i] < taus[t]} ("similar" patches), bin = min(count * n_bins / n_patches,
 * n_bins - 1), hist[t][bin] += 1 (u64, accumulated).  The CDF over frames is the running sum of a row.
 *   score device [n_frames][n_patches] fp32 (codecsight_score_patches' optional output); frame_type device
 *   [n_frames]; taus device [n_tau] fp32; hist device [n_tau][n_bins] u64.
 * --------------------------------------------------------------------------------------------------------- */
typedef struct {
  int32_t source;       /* < 0: past reference, > 0: future (B-frames, ignored)                            */
  uint8_t w, h;         /* partition size in px                                                           */
  int16_t src_x, src_y; /* source position (unused)                                                      */
  int16_t dst_x, dst_y; /* centre of the partition in the current frame, px                              */
  uint64_t flags;
  int32_t motion_x, motion_y; /* motion in 1/motion_scale px                                             */
  uint16_t motion_scale;
} cs_av_mv;

int codecsight_mv_rasterize(const cs_grid* g, int32_t n_frames, const cs_av_mv* mvs, const int64_t* mv_offsets,
                            cs_mb* out, cudaStream_t stream);

int codecsight_similar_hist(const float* score, const uint8_t* frame_type, int64_t n_frames, int32_t n_patches,
                            const float* taus, int32_t n_tau, int32_t n_bins, unsigned long long* hist,
                            cudaStream_t stream);

/* Bytes of device workspace codecsight_kv_refresh needs for this window and stream count (0 on bad args). */
size_t codecsight_kv_refresh_workspace_size(const cs_kv_desc* kv, const cs_window* win, int32_t n_streams);

/* Static string for a return code. */
const char* codecsight_strerror(int code);

/* Library ABI version (major*100 + minor). */
int codecsight_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CODECSIGHT_H_ */
