/*
 * oracle/codecsight_ref.c — ORACLE for the CodecSight hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded C, compiled with `gcc -O2 -ffp-contract=off` (no FMA contraction, no SIMD
 * intrinsics).  Every function follows the paper's definitions in the paper's order, written as loops
 * so a reader can check it against PAPER.md by eye.  Readings of silent or ambiguous passages are the
 * Q-numbered readings of DESIGN.md (taken from SURVEY.md §8(c)).
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference) may load this
 * library.  It shares no code with the CUDA path (paper_2604_06036_b200/csrc), and the CUDA path never
 * calls it.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py (worked examples of the paper
 * and SPEC, hand-derived examples, closed forms, invariants and an independent pure-Python transcription,
 * oracle/pyref.py).  No function is "parity unpinned".
 */
#include "codecsight_ref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------------------------------- */
/* small helpers: bit access on u32 words, bf16 <-> fp32                                               */
/* ---------------------------------------------------------------------------------------------------- */
static int64_t ref_words(const ref_grid* g) { return ((int64_t)g->grid_w * g->grid_h + 31) / 32; }
static int ref_bit(const uint32_t* w, int64_t i) { return (int)((w[i / 32] >> (i % 32)) & 1u); }
static void ref_set(uint32_t* w, int64_t i) { w[i / 32] |= (1u << (i % 32)); }

static float ref_bf16_to_f32(uint16_t h) {
  uint32_t u = ((uint32_t)h) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* fp32 -> bf16, round to nearest, ties to even (reading Q20: "RNE store"). */
static uint16_t ref_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu) != 0) return (uint16_t)((u >> 16) | 0x0040u); /* NaN */
  uint32_t lsb = (u >> 16) & 1u;
  u = u + 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

static int ref_grid_ok(const ref_grid* g) {
  if (!g) return -1;
  if (g->src_w < 1 || g->src_h < 1 || g->src_w > 16384 || g->src_h > 16384) return -2;
  if (g->mb_size < 1 || g->mb_size > 64) return -2;
  if (g->mb_cols != (g->src_w + g->mb_size - 1) / g->mb_size) return -2;
  if (g->mb_rows != (g->src_h + g->mb_size - 1) / g->mb_size) return -2;
  if (g->grid_w < 1 || g->grid_h < 1 || (int64_t)g->grid_w * g->grid_h > 4096) return -2;
  if (g->group < 1 || g->grid_w % g->group != 0 || g->grid_h % g->group != 0) return -2;
  if ((int64_t)g->mb_rows * g->grid_w > 8192) return -3;
  if (g->patch < 1 || g->patch > 32) return -2;
  if (isnan(g->tau) || g->tau < 0.0f) return -1;
  if (isnan(g->alpha) || isinf(g->alpha) || g->alpha < 0.0f) return -1;
  return 0;
}

/* ---------------------------------------------------------------------------------------------------- */
/* Eq. 1: V_t^m = ||v_t^m||.  The MV is in quarter-pel units, so the magnitude in source     */
/* pixels is sqrt(dx^2 + dy^2) / 4 (reading Q2).  INTRA macroblocks have no motion vector; they are      */
/* treated as maximally dynamic, v = +inf (reading Q9).  Unknown types are treated as INTRA.            */
/* ---------------------------------------------------------------------------------------------------- */
float codecsight_ref_mb_magnitude(int16_t dx_qpel, int16_t dy_qpel, uint8_t mb_type) {
  if (mb_type != REF_MB_INTER && mb_type != REF_MB_SKIP) return INFINITY;
  uint32_t sq = (uint32_t)((int32_t)dx_qpel * (int32_t)dx_qpel) + (uint32_t)((int32_t)dy_qpel * (int32_t)dy_qpel);
  return sqrtf((float)sq) * 0.25f;
}

/* ---------------------------------------------------------------------------------------------------- */
/* Resampling onto the patch grid followed by Eq. 3.                      */
/* Coordinates are scaled by (grid_w, grid_h) so every rectangle edge is an integer (reading Q3):        */
/*   patch (r, c):  X [c*src_w, (c+1)*src_w)            Y [r*src_h, (r+1)*src_h)                          */
/*   MB (j, i):     X [mb*i*grid_w, mb*(i+1)*grid_w)    Y [mb*j*grid_h, mb*(j+1)*grid_h)                  */
/* V(i) = max of v_m over MBs with positive-area overlap ("max over blocks overlapping").           */
/* R(i) = sum_m a(i,m) * sad_m / (mb^2 * 255 * src_w * src_h): the area-weighted mean of the per-pixel    */
/*        |residual| (uniform inside an MB: sad/mb^2) over the patch (area src_w*src_h in scaled units), */
/*        normalised to [0,1] by /255.  Numerator and denominator are exact in double.     */
/* M(i) = V(i) + alpha R(i) as one fp32 fma; +inf stays +inf.                                             */
/* ---------------------------------------------------------------------------------------------------- */
void codecsight_ref_patch_fields(const ref_grid* g, const ref_mb* mb, float* V, float* R, float* M,
                                 int32_t* status) {
  const int64_t gw = g->grid_w, gh = g->grid_h, mbs = g->mb_size;
  const double denom = (double)mbs * (double)mbs * 255.0 * (double)g->src_w * (double)g->src_h;
  for (int64_t r = 0; r < gh; ++r) {
    for (int64_t c = 0; c < gw; ++c) {
      const int64_t px0 = c * g->src_w, px1 = (c + 1) * g->src_w;
      const int64_t py0 = r * g->src_h, py1 = (r + 1) * g->src_h;
      float v = -INFINITY;
      int64_t area_sad = 0;
      for (int64_t j = 0; j < g->mb_rows; ++j) {
        const int64_t my0 = mbs * j * gh, my1 = mbs * (j + 1) * gh;
        const int64_t oy = (py1 < my1 ? py1 : my1) - (py0 > my0 ? py0 : my0);
        if (oy <= 0) continue;
        for (int64_t i = 0; i < g->mb_cols; ++i) {
          const int64_t mx0 = mbs * i * gw, mx1 = mbs * (i + 1) * gw;
          const int64_t ox = (px1 < mx1 ? px1 : mx1) - (px0 > mx0 ? px0 : mx0);
          if (ox <= 0) continue;
          const ref_mb* b = &mb[j * g->mb_cols + i];
          if (b->mb_type > REF_MB_INTRA && status) *status |= REF_ST_BAD_MB_TYPE;
          const float vm = codecsight_ref_mb_magnitude(b->mvx_qpel, b->mvy_qpel, b->mb_type);
          if (vm > v) v = vm;
          area_sad += ox * oy * (int64_t)b->sad;
        }
      }
      const float rr = (float)((double)area_sad / denom);
      const float mm = isinf(v) ? INFINITY : fmaf(g->alpha, rr, v);
      if (V) V[r * gw + c] = v;
      if (R) R[r * gw + c] = rr;
      if (M) M[r * gw + c] = mm;
    }
  }
}

/* ---------------------------------------------------------------------------------------------------- */
/* score_patches: Eq. 4 threshold, GOP accumulation, group-complete expansion */
/* ---------------------------------------------------------------------------------------------------- */
int codecsight_ref_score_patches(const ref_grid* g, int32_t n_streams, int32_t n_frames, const ref_mb* mb,
                                 const uint8_t* frame_type, uint32_t* keep_mask, int64_t frame_stride,
                                 uint32_t* gop_state, float* score, int32_t* kept_count,
                                 unsigned long long* counters, int32_t* status) {
  int rc = ref_grid_ok(g);
  if (rc) return rc;
  if (n_streams < 0 || n_frames < 1 || n_frames > 256 || frame_stride < n_frames) return -1;
  if (n_streams == 0) return 0;
  if (!mb || !frame_type || !keep_mask || !gop_state || !kept_count || !counters || !status) return -1;

  const int64_t np = (int64_t)g->grid_w * g->grid_h, nw = ref_words(g), G = g->group;
  const int64_t n_mb = (int64_t)g->mb_rows * g->mb_cols;
  float* M = (float*)malloc(sizeof(float) * np);
  uint32_t* out = (uint32_t*)malloc(sizeof(uint32_t) * nw);
  uint32_t* keep = (uint32_t*)malloc(sizeof(uint32_t) * nw);
  if (!M || !out || !keep) { free(M); free(out); free(keep); return -1; }

  for (int64_t s = 0; s < n_streams; ++s) {
    uint32_t* st = gop_state + s * (nw + 1); /* accumulated bits, then the flag word */
    for (int64_t j = 0; j < n_frames; ++j) {
      const int64_t slot = s * frame_stride + j;
      const uint8_t type = frame_type[slot];
      int is_i = (type == REF_FRAME_I);
      if (type != REF_FRAME_I && type != REF_FRAME_P) { *status |= REF_ST_BAD_FRAME_TYPE; is_i = 1; }
      counters[REF_C_FRAMES] += 1;
      if (is_i) {
        /* "I-frames are always fully encoded" and reset the mask: output every patch,
           accumulation state := empty (reading Q7), score = +inf, metadata not read (Q10). */
        for (int64_t w = 0; w < nw; ++w) st[w] = 0;
        st[nw] |= 1u;
        for (int64_t w = 0; w < nw; ++w) out[w] = 0;
        for (int64_t i = 0; i < np; ++i) ref_set(out, i);
        if (score)
          for (int64_t i = 0; i < np; ++i) score[(s * n_frames + j) * np + i] = INFINITY;
      } else {
        counters[REF_C_PFRAMES] += 1;
        if (!(st[nw] & 1u)) { /* reading Q11 */
          *status |= REF_ST_NO_IFRAME;
          for (int64_t w = 0; w < nw; ++w) st[w] = 0;
          st[nw] |= 1u;
        }
        codecsight_ref_patch_fields(g, mb + (s * n_frames + j) * n_mb, NULL, NULL, M, status);
        for (int64_t i = 0; i < np; ++i) {
          /* Eq. 4: dynamic(i) = M_t(i) >= tau (inclusive, reading Q1) */
          if (M[i] >= g->tau) ref_set(st, i);
          /* union with the preceding P-frames of the GOP is the |= above */
          if (isfinite(M[i]) && fabsf(M[i] - g->tau) <= 1e-5f) counters[REF_C_NEAR_TAU] += 1;
        }
        for (int64_t w = 0; w < nw; ++w) out[w] = st[w];
        if (score)
          for (int64_t i = 0; i < np; ++i) score[(s * n_frames + j) * np + i] = M[i];
      }
      /* group-complete expansion: keep every patch of a group with any active patch */
      for (int64_t w = 0; w < nw; ++w) keep[w] = 0;
      for (int64_t gr = 0; gr < g->grid_h / G; ++gr)
        for (int64_t gc = 0; gc < g->grid_w / G; ++gc) {
          int any = 0;
          for (int64_t dy = 0; dy < G; ++dy)
            for (int64_t dx = 0; dx < G; ++dx) any |= ref_bit(out, (gr * G + dy) * g->grid_w + gc * G + dx);
          if (any)
            for (int64_t dy = 0; dy < G; ++dy)
              for (int64_t dx = 0; dx < G; ++dx) ref_set(keep, (gr * G + dy) * g->grid_w + gc * G + dx);
        }
      int64_t kept = 0;
      for (int64_t i = 0; i < np; ++i) kept += ref_bit(keep, i);
      for (int64_t w = 0; w < nw; ++w) keep_mask[slot * nw + w] = keep[w];
      kept_count[s * n_frames + j] = (int32_t)kept;
      counters[REF_C_PATCHES] += (unsigned long long)np;
      counters[REF_C_KEPT] += (unsigned long long)kept;
      counters[REF_C_BYTES_SCORE] +=
          (unsigned long long)((is_i ? 0 : 8 * n_mb) + 4 * nw + 4 + (score ? 4 * np : 0));
    }
    counters[REF_C_BYTES_SCORE] += (unsigned long long)(2 * 4 * (nw + 1));
  }
  free(M);
  free(out);
  free(keep);
  return 0;
}

/* ---------------------------------------------------------------------------------------------------- */
/* compact: "executes the ViT only on the selected patches" — the packed, group-major ViT input. */
/* ---------------------------------------------------------------------------------------------------- */
int codecsight_ref_compact(const ref_grid* g, int32_t n_streams, int32_t n_frames, const uint32_t* keep_mask,
                           int64_t mask_frame_stride, const int32_t* frame_index, const void* const* frames,
                           int32_t frame_layout, int64_t capacity, void* packed, int32_t* pos_ids, int32_t* src_index,
                           int32_t* frame_offsets, unsigned long long* counters, int32_t* status) {
  int rc = ref_grid_ok(g);
  if (rc) return rc;
  if (n_streams < 0 || n_frames < 1 || mask_frame_stride < n_frames || capacity < 0) return -1;
  if (frame_layout != REF_LAYOUT_PLANAR && frame_layout != REF_LAYOUT_GROUPED) return -1;
  const int64_t np = (int64_t)g->grid_w * g->grid_h, nw = ref_words(g), G = g->group, p = g->patch;
  const int64_t n_slots = (int64_t)n_streams * n_frames;
  if (n_slots * np >= 2147483648LL) return -3;
  if (!frame_offsets || !counters || !status) return -1;
  if (n_slots > 0 && (!keep_mask || !frame_index || !frames)) return -1;
  if (capacity > 0 && (!packed || !pos_ids || !src_index)) return -1;

  const int64_t fh = g->grid_h * p, fw = g->grid_w * p; /* model-input frame [3][fh][fw] bf16 */
  const int64_t row = 3 * p * p;                         /* elements of one packed patch row */
  uint16_t* out = (uint16_t*)packed;
  int64_t off = 0, written = 0;
  for (int64_t s = 0; s < n_streams; ++s)
    for (int64_t j = 0; j < n_frames; ++j) {
      const int64_t slot = s * n_frames + j;
      const uint32_t* m = keep_mask + (s * mask_frame_stride + j) * nw;
      const uint16_t* fr = (const uint16_t*)frames[slot];
      frame_offsets[slot] = (int32_t)off;
      for (int64_t gr = 0; gr < g->grid_h / G; ++gr)
        for (int64_t gc = 0; gc < g->grid_w / G; ++gc) {
          int any = 0;
          for (int64_t dy = 0; dy < G; ++dy)
            for (int64_t dx = 0; dx < G; ++dx) any |= ref_bit(m, (gr * G + dy) * g->grid_w + gc * G + dx);
          if (!any) continue;
          for (int64_t dy = 0; dy < G; ++dy)
            for (int64_t dx = 0; dx < G; ++dx) {
              const int64_t h = gr * G + dy, w = gc * G + dx, n = off++;
              if (n >= capacity) { *status |= REF_ST_CAPACITY; continue; }
              for (int64_t c = 0; c < 3; ++c)
                for (int64_t y = 0; y < p; ++y)
                  for (int64_t x = 0; x < p; ++x) {
                    /* pixel (c, p*h + y, p*w + x) of the frame, in the frame's layout */
                    int64_t src;
                    if (frame_layout == REF_LAYOUT_PLANAR)
                      src = c * fh * fw + (h * p + y) * fw + (w * p + x);
                    else /* grouped: [group (gr,gc)][patch (dy,dx)][c][y][x] */
                      src = (((gr * (g->grid_w / G) + gc) * G * G + dy * G + dx) * 3 + c) * p * p + y * p + x;
                    out[n * row + c * p * p + y * p + x] = fr[src];
                  }
              pos_ids[3 * n + 0] = frame_index[slot];
              pos_ids[3 * n + 1] = (int32_t)h;
              pos_ids[3 * n + 2] = (int32_t)w;
              src_index[n] = (int32_t)(slot * np + h * g->grid_w + w);
              ++written;
            }
        }
    }
  frame_offsets[n_slots] = (int32_t)off;
  counters[REF_C_PACKED_ROWS] += (unsigned long long)written;
  counters[REF_C_BYTES_COMPACT] +=
      (unsigned long long)(n_slots * (4 * nw + 4) + written * (2 * row * 2 + 16));
  return 0;
}

/* ---------------------------------------------------------------------------------------------------- */
/* NEXT-3: temporal patches.  Qwen2-VL embeds video with temporal_patch_size = 2 (P:399 names the
 * Qwen-VL models): one visual token covers tp consecutive frames and its patch row is [3][tp][p][p] (channel, then
 * frame, then pixels -- the Hugging Face processor's flatten order).  Pruning reading: a group of a unit is emitted
 * iff any of its patches is kept in ANY of the unit's frames (the union keeps every dynamic pixel).  Unit u of
 * stream s uses frames[(s*n_units + u)*tp + f] and masks keep_mask[s][u*tp + f], f < tp.                     */
/* ---------------------------------------------------------------------------------------------------- */
int codecsight_ref_compact_tp(const ref_grid* g, int32_t tp, int32_t n_streams, int32_t n_units,
                              const uint32_t* keep_mask, int64_t mask_frame_stride, const int32_t* unit_index,
                              const void* const* frames, int32_t frame_layout, int64_t capacity, void* packed,
                              int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets, uint32_t* unit_mask,
                              int64_t unit_mask_stride, const uint8_t* frame_type, uint8_t* unit_type,
                              unsigned long long* counters, int32_t* status) {
  int rc = ref_grid_ok(g);
  if (rc) return rc;
  if (tp < 1 || tp > 4) return -3;
  if (n_streams < 0 || n_units < 1 || mask_frame_stride < (int64_t)n_units * tp || capacity < 0) return -1;
  if ((unit_mask || unit_type) && unit_mask_stride < n_units) return -1;
  if ((frame_type == 0) != (unit_type == 0)) return -1;
  if (frame_layout != REF_LAYOUT_PLANAR && frame_layout != REF_LAYOUT_GROUPED) return -1;
  const int64_t np = (int64_t)g->grid_w * g->grid_h, nw = ref_words(g), G = g->group, p = g->patch;
  const int64_t n_slots = (int64_t)n_streams * n_units;
  if (n_slots * np >= 2147483648LL) return -3;
  if (!frame_offsets || !counters || !status) return -1;
  if (n_slots > 0 && (!keep_mask || !unit_index || !frames)) return -1;
  if (capacity > 0 && (!packed || !pos_ids || !src_index)) return -1;

  const int64_t fh = g->grid_h * p, fw = g->grid_w * p;
  const int64_t row = 3 * tp * p * p; /* elements of one packed row: [3][tp][p][p] */
  uint16_t* out = (uint16_t*)packed;
  int64_t off = 0, written = 0;
  for (int64_t s = 0; s < n_streams; ++s)
    for (int64_t u = 0; u < n_units; ++u) {
      const int64_t slot = s * n_units + u;
      frame_offsets[slot] = (int32_t)off;
      if (unit_mask)
        for (int64_t t = 0; t < nw; ++t) {
          uint32_t w = 0;
          for (int64_t f = 0; f < tp; ++f) w |= keep_mask[(s * mask_frame_stride + u * tp + f) * nw + t];
          unit_mask[(s * unit_mask_stride + u) * nw + t] = w;
        }
      if (unit_type) { /* a unit holding an I-frame (or an unknown type, read as I) is an I unit */
        uint8_t ty = REF_FRAME_P;
        for (int64_t f = 0; f < tp; ++f)
          if (frame_type[s * mask_frame_stride + u * tp + f] != REF_FRAME_P) ty = REF_FRAME_I;
        unit_type[s * unit_mask_stride + u] = ty;
      }
      for (int64_t gr = 0; gr < g->grid_h / G; ++gr)
        for (int64_t gc = 0; gc < g->grid_w / G; ++gc) {
          int any = 0;
          for (int64_t f = 0; f < tp; ++f) {
            const uint32_t* m = keep_mask + (s * mask_frame_stride + u * tp + f) * nw;
            for (int64_t dy = 0; dy < G; ++dy)
              for (int64_t dx = 0; dx < G; ++dx) any |= ref_bit(m, (gr * G + dy) * g->grid_w + gc * G + dx);
          }
          if (!any) continue;
          for (int64_t dy = 0; dy < G; ++dy)
            for (int64_t dx = 0; dx < G; ++dx) {
              const int64_t h = gr * G + dy, w = gc * G + dx, n = off++;
              if (n >= capacity) { *status |= REF_ST_CAPACITY; continue; }
              for (int64_t c = 0; c < 3; ++c)
                for (int64_t f = 0; f < tp; ++f) {
                  const uint16_t* fr = (const uint16_t*)frames[slot * tp + f];
                  for (int64_t y = 0; y < p; ++y)
                    for (int64_t x = 0; x < p; ++x) {
                      int64_t src;
                      if (frame_layout == REF_LAYOUT_PLANAR)
                        src = c * fh * fw + (h * p + y) * fw + (w * p + x);
                      else
                        src = (((gr * (g->grid_w / G) + gc) * G * G + dy * G + dx) * 3 + c) * p * p + y * p + x;
                      out[n * row + ((c * tp + f) * p + y) * p + x] = fr[src];
                    }
                }
              pos_ids[3 * n + 0] = unit_index[slot];
              pos_ids[3 * n + 1] = (int32_t)h;
              pos_ids[3 * n + 2] = (int32_t)w;
              src_index[n] = (int32_t)(slot * np + h * g->grid_w + w);
              ++written;
            }
        }
    }
  frame_offsets[n_slots] = (int32_t)off;
  counters[REF_C_PACKED_ROWS] += (unsigned long long)written;
  counters[REF_C_BYTES_COMPACT] += (unsigned long long)(n_slots * (4 * nw * tp + 4) + written * (2 * row * 2 + 16) +
                                                        (unit_mask ? n_slots * 4 * nw : 0) +
                                                        (unit_type ? n_slots * (tp + 1) : 0));
  return 0;
}

/* ---------------------------------------------------------------------------------------------------- */
/* Eq. 5: K^_t(j) = R(p_new - p_old) K_{t-1}(j), rotate_half pairing (reading Q19-Q21).      */
/* ---------------------------------------------------------------------------------------------------- */
static void ref_rot_pair(float x1, float x2, int64_t i, int64_t D, double base, int64_t dp, float* o1, float* o2) {
  const double inv = pow(base, -2.0 * (double)i / (double)D);
  const double ang = (double)dp * inv;
  const float c = (float)cos(ang), s = (float)sin(ang);
  *o1 = fmaf(x1, c, -(x2 * s));
  *o2 = fmaf(x2, c, x1 * s);
}

/* The position difference that rotates frequency pair i (Eq. 5): 1-D RoPE rotates every pair by the
 * sequence-position difference; M-RoPE (reading NEXT-3) rotates pair i by the difference of the position component
 * its section belongs to: i < s_t -> t, next s_h -> h, last s_w -> w. */
static int64_t ref_pair_delta(const ref_kv* kv, int64_t i, int64_t dp_seq, const int64_t dpos[3]) {
  if (kv->rope_mode != REF_ROPE_MROPE) return dp_seq;
  if (i < kv->mrope_section[0]) return dpos[0];
  if (i < kv->mrope_section[0] + kv->mrope_section[1]) return dpos[1];
  return dpos[2];
}

static int ref_rope_ok(const ref_kv* kv) {
  if (kv->rope_mode == REF_ROPE_1D) return 0;
  if (kv->rope_mode != REF_ROPE_MROPE) return -3;
  if (kv->mrope_section[0] < 0 || kv->mrope_section[1] < 0 || kv->mrope_section[2] < 0) return -1;
  if (kv->mrope_section[0] + kv->mrope_section[1] + kv->mrope_section[2] != kv->head_dim / 2) return -2;
  if (kv->t_per_frame < 1) return -1;
  return 0;
}

void codecsight_ref_rope_rotate_f32(const float* k, int32_t n_heads, int32_t head_dim, double base, int64_t dp,
                                    float* out) {
  const int64_t half = head_dim / 2;
  for (int64_t h = 0; h < n_heads; ++h)
    for (int64_t i = 0; i < half; ++i)
      ref_rot_pair(k[h * head_dim + i], k[h * head_dim + i + half], i, head_dim, base, dp,
                   &out[h * head_dim + i], &out[h * head_dim + i + half]);
}

static int64_t ref_tokens_of(const ref_grid* g, const uint32_t* m) {
  /* one token per emitted group (same rule as compaction, "(2x2) group ... projected into a token") */
  const int64_t G = g->group;
  int64_t n = 0;
  for (int64_t gr = 0; gr < g->grid_h / G; ++gr)
    for (int64_t gc = 0; gc < g->grid_w / G; ++gc) {
      int any = 0;
      for (int64_t dy = 0; dy < G; ++dy)
        for (int64_t dx = 0; dx < G; ++dx) any |= ref_bit(m, (gr * G + dy) * g->grid_w + gc * G + dx);
      n += any;
    }
  return n;
}

/* ---------------------------------------------------------------------------------------------------- */
/* kv_refresh: critical-token refresh + position-consistent reuse.               */
/* ---------------------------------------------------------------------------------------------------- */
int codecsight_ref_kv_refresh(const ref_grid* g, const ref_kv* kv, const ref_window* win, int32_t n_streams,
                              const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring,
                              const void* const* old_cache, void* const* new_cache,
                              const void* const* refreshed, int64_t token_cap, uint8_t* disposition,
                              int32_t* p_old, int32_t* n_tokens, unsigned long long* counters, int32_t* status) {
  int rc = ref_grid_ok(g);
  if (rc) return rc;
  if (!kv || !win) return -1;
  if (n_streams < 0 || token_cap < 0) return -1;
  if (kv->dtype != REF_BF16 && kv->dtype != REF_FP32) return -3;
  if (kv->layers < 1 || kv->kv_heads < 1 || kv->head_dim < 2 || kv->head_dim > 512) return -3;
  if (kv->head_dim % 2 != 0) return -3;
  if (kv->capacity < 0 || kv->refresh_capacity < 0 || kv->n_prompt < 0) return -1;
  if (!(kv->rope_base > 0.0)) return -1;
  if ((rc = ref_rope_ok(kv))) return rc;
  const int64_t w = win->window, s = win->stride, k = win->step;
  if (w < 1 || s < 1 || k < 0) return -1;
  if (s > w) return -3;
  if (win->ring_frames < (k >= 1 ? w + s : w)) return -2;
  if (n_streams == 0) return 0;
  if (!keep_mask_ring || !frame_type_ring || !new_cache || !disposition || !p_old || !n_tokens || !counters ||
      !status)
    return -1;
  if (k >= 1 && !old_cache) return -1;

  const int64_t nw = ref_words(g), G = g->group, ring = win->ring_frames;
  const int64_t L = kv->layers, H = kv->kv_heads, D = kv->head_dim, cap = kv->capacity;
  const int64_t rowel = H * D, esz = (kv->dtype == REF_BF16) ? 2 : 4;
  const int64_t ks = k * s, new_first = (k - 1) * s + w; /* frames >= new_first arrived with this stride */

  for (int64_t sg = 0; sg < n_streams; ++sg) {
    const uint32_t* mring = keep_mask_ring + sg * ring * nw;
    const uint8_t* tring = frame_type_ring + sg * ring;
    /* sum of n_f over the dropped frames [(k-1)s, ks): p_old(f) = drop + sum_{[ks, f)} n_f' */
    int64_t drop = 0;
    if (k >= 1)
      for (int64_t f = (k - 1) * s; f < ks; ++f) drop += ref_tokens_of(g, mring + (f % ring) * nw);

    int64_t pn = 0, before = 0, n_reuse = 0, n_anchor = 0, n_new = 0, rrow = 0, moved = 0;
    const uint8_t* oc = k >= 1 ? (const uint8_t*)old_cache[sg] : NULL;
    uint8_t* nc = (uint8_t*)new_cache[sg];
    const uint8_t* rf = refreshed ? (const uint8_t*)refreshed[sg] : NULL;

    /* visual tokens in (frame, group row-major) order, then the prompt rows */
    for (int64_t f = ks; f < ks + w + 1; ++f) {
      const int is_prompt = (f == ks + w);
      const uint32_t* m = is_prompt ? NULL : mring + (f % ring) * nw;
      const uint8_t type = is_prompt ? 0 : tring[f % ring];
      const int64_t nslots = is_prompt ? kv->n_prompt : (g->grid_h / G) * (g->grid_w / G);
      int64_t rank = 0;
      for (int64_t q = 0; q < nslots; ++q) {
        if (!is_prompt) {
          const int64_t gr = q / (g->grid_w / G), gc = q % (g->grid_w / G);
          int any = 0;
          for (int64_t dy = 0; dy < G; ++dy)
            for (int64_t dx = 0; dx < G; ++dx) any |= ref_bit(m, (gr * G + dy) * g->grid_w + gc * G + dx);
          if (!any) continue;
        }
        const int64_t p_new = pn++;
        int disp;
        int64_t po;
        if (is_prompt || k == 0 || f >= new_first) {
          disp = REF_DISP_NEW;
          po = -1;
        } else {
          /* I-frame tokens are anchors; the first overlap frame anchors the boundary (Q17) */
          disp = (type == REF_FRAME_I || f == ks) ? REF_DISP_ANCHOR : REF_DISP_REUSE;
          po = drop + before + rank; /* before = sum of n_f' over [ks, f) */
        }
        ++rank;
        if (disp == REF_DISP_REUSE) ++n_reuse;
        else if (disp == REF_DISP_ANCHOR) ++n_anchor;
        else ++n_new;
        if (p_new < token_cap) {
          disposition[sg * token_cap + p_new] = (uint8_t)disp;
          p_old[sg * token_cap + p_new] = (int32_t)po;
        } else {
          *status |= REF_ST_CAPACITY;
        }
        /* K/V rows of this token, all layers */
        if (disp == REF_DISP_REUSE) {
          if (p_new >= cap) { *status |= REF_ST_CAPACITY; continue; }
          if (po >= cap) { *status |= REF_ST_ORIGIN; continue; }
          const int64_t dp = p_new - po;
          /* M-RoPE positions of this token in windows k-1 and k: (t, h, w) = (frame offset * t_per_frame, gr, gc) */
          const int64_t gr = q / (g->grid_w / G), gc = q % (g->grid_w / G);
          const int64_t pos_old[3] = {(f - (k - 1) * s) * kv->t_per_frame, gr, gc};
          const int64_t pos_new[3] = {(f - ks) * kv->t_per_frame, gr, gc};
          const int64_t dpos[3] = {pos_new[0] - pos_old[0], pos_new[1] - pos_old[1], pos_new[2] - pos_old[2]};
          for (int64_t l = 0; l < L; ++l) {
            /* value reuse: V^_t(j) = V_{t-1}(j) */
            memcpy(nc + ((l * 2 + 1) * cap + p_new) * rowel * esz, oc + ((l * 2 + 1) * cap + po) * rowel * esz,
                   (size_t)(rowel * esz));
            /* key correction (Eq. 5) */
            for (int64_t h = 0; h < H; ++h)
              for (int64_t i = 0; i < D / 2; ++i) {
                const int64_t e1 = h * D + i, e2 = h * D + i + D / 2;
                const int64_t src = ((l * 2 + 0) * cap + po) * rowel, dst = ((l * 2 + 0) * cap + p_new) * rowel;
                float x1, x2, o1, o2;
                if (kv->rope_mode == REF_ROPE_MROPE && i >= kv->mrope_section[0]) {
                  /* h / w sections: the token's (h, w) are unchanged -> the stored bits are kept (NEXT-3) */
                  memcpy(nc + (dst + e1) * esz, oc + (src + e1) * esz, (size_t)esz);
                  memcpy(nc + (dst + e2) * esz, oc + (src + e2) * esz, (size_t)esz);
                  continue;
                }
                if (esz == 2) {
                  x1 = ref_bf16_to_f32(((const uint16_t*)oc)[src + e1]);
                  x2 = ref_bf16_to_f32(((const uint16_t*)oc)[src + e2]);
                } else {
                  x1 = ((const float*)oc)[src + e1];
                  x2 = ((const float*)oc)[src + e2];
                }
                ref_rot_pair(x1, x2, i, D, kv->rope_base, ref_pair_delta(kv, i, dp, dpos), &o1, &o2);
                if (esz == 2) {
                  ((uint16_t*)nc)[dst + e1] = ref_f32_to_bf16(o1);
                  ((uint16_t*)nc)[dst + e2] = ref_f32_to_bf16(o2);
                } else {
                  ((float*)nc)[dst + e1] = o1;
                  ((float*)nc)[dst + e2] = o2;
                }
              }
          }
          ++moved;
        } else {
          const int64_t r = rrow++; /* r-th non-REUSE token in p_new order (reading Q18) */
          if (!rf) continue;
          if (p_new >= cap || r >= kv->refresh_capacity) { *status |= REF_ST_CAPACITY; continue; }
          for (int64_t l = 0; l < L; ++l)
            for (int64_t h2 = 0; h2 < 2; ++h2)
              memcpy(nc + ((l * 2 + h2) * cap + p_new) * rowel * esz,
                     rf + ((l * 2 + h2) * kv->refresh_capacity + r) * rowel * esz, (size_t)(rowel * esz));
          ++moved;
        }
      }
      if (!is_prompt) before += rank; /* rank == n_f once the frame is done */
    }
    const int64_t n_visual = pn - kv->n_prompt;
    n_tokens[sg * 4 + 0] = (int32_t)n_visual;
    n_tokens[sg * 4 + 1] = (int32_t)n_reuse;
    n_tokens[sg * 4 + 2] = (int32_t)n_anchor;
    n_tokens[sg * 4 + 3] = (int32_t)n_new;
    counters[REF_C_TOK_REUSE] += (unsigned long long)n_reuse;
    counters[REF_C_TOK_ANCHOR] += (unsigned long long)n_anchor;
    counters[REF_C_TOK_NEW] += (unsigned long long)n_new;
    counters[REF_C_BYTES_KV] += (unsigned long long)(moved * L * 2 * rowel * esz * 2);
    counters[REF_C_STREAM_STEPS] += 1;
  }
  return 0;
}

/* ---------------------------------------------------------------------------------------------------- */
/* kv_refresh_paged (NEXT-1): the same window step with the previous window's KV kept resident and        */
/* updated IN PLACE ("maintains the previous window's KV cache resident in GPU memory and performs these  */
/* updates in-place").  Each stream owns a pool of `capacity` physical rows; a token's rows live at */
/* slot_map[p].  REUSE tokens keep their slot, their keys are rotated in place by R(dp) (Eq. 5) and their */
/* values are not touched.  ANCHOR tokens keep their slot and are overwritten with their          */
/* recomputed rows.  NEW tokens (new frames, prompt) take the free slots (slots not held by a token       */
/* surviving from window k-1) in ascending slot order, in p_new order.                                    */
/* ---------------------------------------------------------------------------------------------------- */
int codecsight_ref_kv_refresh_paged(const ref_grid* g, const ref_kv* kv, const ref_window* win, int32_t n_streams,
                                    const uint32_t* keep_mask_ring, const uint8_t* frame_type_ring,
                                    void* const* pool, const int32_t* slot_old, int32_t* slot_new, int64_t slot_cap,
                                    const void* const* refreshed, int64_t token_cap, uint8_t* disposition,
                                    int32_t* p_old, int32_t* n_tokens, unsigned long long* counters,
                                    int32_t* status) {
  int rc = ref_grid_ok(g);
  if (rc) return rc;
  if (!kv || !win) return -1;
  if (n_streams < 0 || token_cap < 0 || slot_cap < 0) return -1;
  if (kv->dtype != REF_BF16 && kv->dtype != REF_FP32) return -3;
  if (kv->layers < 1 || kv->kv_heads < 1 || kv->head_dim < 2 || kv->head_dim > 512) return -3;
  if (kv->head_dim % 2 != 0) return -3;
  if (kv->capacity < 0 || kv->refresh_capacity < 0 || kv->n_prompt < 0) return -1;
  if (!(kv->rope_base > 0.0)) return -1;
  if ((rc = ref_rope_ok(kv))) return rc;
  const int64_t w = win->window, s = win->stride, k = win->step;
  if (w < 1 || s < 1 || k < 0) return -1;
  if (s > w) return -3;
  if (win->ring_frames < (k >= 1 ? w + s : w)) return -2;
  if (n_streams == 0) return 0;
  if (!keep_mask_ring || !frame_type_ring || !pool || !slot_new || !disposition || !p_old || !n_tokens ||
      !counters || !status)
    return -1;
  if (k >= 1 && !slot_old) return -1;

  const int64_t nw = ref_words(g), ring = win->ring_frames;
  const int64_t L = kv->layers, H = kv->kv_heads, D = kv->head_dim, cap = kv->capacity;
  const int64_t rowel = H * D, esz = (kv->dtype == REF_BF16) ? 2 : 4;
  const int64_t ks = k * s, new_first = (k - 1) * s + w;
  const int64_t max_tok = w * (g->grid_h / g->group) * (g->grid_w / g->group) + kv->n_prompt;
  int32_t* tdisp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(max_tok + 1));
  int64_t* tpold = (int64_t*)malloc(sizeof(int64_t) * (size_t)(max_tok + 1));
  int64_t* tslot = (int64_t*)malloc(sizeof(int64_t) * (size_t)(max_tok + 1));
  int64_t* tfrm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(max_tok + 1));
  uint8_t* used = (uint8_t*)malloc((size_t)(cap + 1));
  if (!tdisp || !tpold || !tslot || !used || !tfrm) {
    free(tdisp); free(tpold); free(tslot); free(used); free(tfrm);
    return -1;
  }

  for (int64_t sg = 0; sg < n_streams; ++sg) {
    const uint32_t* mring = keep_mask_ring + sg * ring * nw;
    const uint8_t* tring = frame_type_ring + sg * ring;
    /* 1. the tokens of window k, in p_new order: disposition and p_old (same rules as kv_refresh) */
    int64_t drop = 0, n_old = 0;
    if (k >= 1) {
      for (int64_t f = (k - 1) * s; f < ks; ++f) drop += ref_tokens_of(g, mring + (f % ring) * nw);
      for (int64_t f = (k - 1) * s; f < (k - 1) * s + w; ++f) n_old += ref_tokens_of(g, mring + (f % ring) * nw);
      n_old += kv->n_prompt; /* tokens of window k-1, prompt included */
    }
    int64_t nt = 0, before = 0;
    for (int64_t f = ks; f < ks + w; ++f) {
      const uint8_t type = tring[f % ring];
      const int64_t nf = ref_tokens_of(g, mring + (f % ring) * nw);
      for (int64_t t = 0; t < nf; ++t) {
        if (k == 0 || f >= new_first) {
          tdisp[nt] = REF_DISP_NEW;
          tpold[nt] = -1;
        } else {
          tdisp[nt] = (type == REF_FRAME_I || f == ks) ? REF_DISP_ANCHOR : REF_DISP_REUSE;
          tpold[nt] = drop + before + t;
        }
        tfrm[nt] = f;
        ++nt;
      }
      before += nf;
    }
    const int64_t n_visual = nt;
    for (int64_t j = 0; j < kv->n_prompt; ++j) {
      tdisp[nt] = REF_DISP_NEW;
      tpold[nt] = -1;
      ++nt;
    }
    /* 2. slots held by tokens that survive from window k-1 (REUSE and ANCHOR keep their rows' slots) */
    for (int64_t i = 0; i < cap; ++i) used[i] = 0;
    for (int64_t p = 0; p < nt; ++p) {
      tslot[p] = -1;
      if (tdisp[p] == REF_DISP_NEW) continue;
      const int64_t po = tpold[p];
      const int64_t sl = (po < slot_cap && po < n_old) ? slot_old[sg * slot_cap + po] : -1;
      if (sl < 0 || sl >= cap) { *status |= REF_ST_ORIGIN; continue; }
      tslot[p] = sl;
      used[sl] = 1;
    }
    /* 3. NEW tokens take the free slots in ascending order */
    int64_t next_free = 0;
    for (int64_t p = 0; p < nt; ++p) {
      if (tdisp[p] != REF_DISP_NEW) continue;
      while (next_free < cap && used[next_free]) ++next_free;
      if (next_free >= cap) { *status |= REF_ST_CAPACITY; continue; }
      tslot[p] = next_free;
      used[next_free] = 1;
    }
    /* 4. outputs and row updates */
    const uint8_t* rf = refreshed ? (const uint8_t*)refreshed[sg] : NULL;
    uint8_t* pl = (uint8_t*)pool[sg];
    /* In place, a reused key is rewritten only where Eq. 5 changes it: every pair for 1-D RoPE; for M-RoPE only
     * the s_t pairs of the temporal section -- (h, w) of a reused token do not change, so the h / w sections keep
     * their stored bits (R(0) = identity; reading NEXT-3). */
    const int64_t rot_pairs = kv->rope_mode == REF_ROPE_MROPE ? kv->mrope_section[0] : D / 2;
    int64_t n_reuse = 0, n_anchor = 0, n_new = 0, rrow = 0, rot = 0, cop = 0, dp = 0;
    for (int64_t p = 0; p < nt; ++p) {
      const int d = tdisp[p];
      if (d == REF_DISP_REUSE) ++n_reuse;
      else if (d == REF_DISP_ANCHOR) ++n_anchor;
      else ++n_new;
      if (p < token_cap) {
        disposition[sg * token_cap + p] = (uint8_t)d;
        p_old[sg * token_cap + p] = (int32_t)tpold[p];
      } else {
        *status |= REF_ST_CAPACITY;
      }
      if (p < slot_cap) slot_new[sg * slot_cap + p] = (int32_t)tslot[p];
      else *status |= REF_ST_CAPACITY;
      const int64_t sl = tslot[p];
      if (d == REF_DISP_REUSE) {
        if (sl < 0) continue;
        dp = p - tpold[p];
        /* M-RoPE: t moves with the window, (h, w) of a reused token (same frame, same group) do not */
        const int64_t dpos[3] = {((tfrm[p] - ks) - (tfrm[p] - (k - 1) * s)) * kv->t_per_frame, 0, 0};
        for (int64_t l = 0; l < L; ++l)
          for (int64_t h = 0; h < H; ++h)
            for (int64_t i = 0; i < rot_pairs; ++i) {
              const int64_t base = ((l * 2 + 0) * cap + sl) * rowel; /* the key row, rotated in place */
              const int64_t e1 = base + h * D + i, e2 = base + h * D + i + D / 2;
              float x1, x2, o1, o2;
              if (esz == 2) {
                x1 = ref_bf16_to_f32(((uint16_t*)pl)[e1]);
                x2 = ref_bf16_to_f32(((uint16_t*)pl)[e2]);
              } else {
                x1 = ((float*)pl)[e1];
                x2 = ((float*)pl)[e2];
              }
              ref_rot_pair(x1, x2, i, D, kv->rope_base, ref_pair_delta(kv, i, dp, dpos), &o1, &o2);
              if (esz == 2) {
                ((uint16_t*)pl)[e1] = ref_f32_to_bf16(o1);
                ((uint16_t*)pl)[e2] = ref_f32_to_bf16(o2);
              } else {
                ((float*)pl)[e1] = o1;
                ((float*)pl)[e2] = o2;
              }
            }
        ++rot;
      } else {
        const int64_t r = rrow++;
        if (!rf || sl < 0) continue;
        if (r >= kv->refresh_capacity) { *status |= REF_ST_CAPACITY; continue; }
        for (int64_t l = 0; l < L; ++l)
          for (int64_t h2 = 0; h2 < 2; ++h2)
            memcpy(pl + ((l * 2 + h2) * cap + sl) * rowel * esz,
                   rf + ((l * 2 + h2) * kv->refresh_capacity + r) * rowel * esz, (size_t)(rowel * esz));
        ++cop;
      }
    }
    (void)dp;
    n_tokens[sg * 4 + 0] = (int32_t)n_visual;
    n_tokens[sg * 4 + 1] = (int32_t)n_reuse;
    n_tokens[sg * 4 + 2] = (int32_t)n_anchor;
    n_tokens[sg * 4 + 3] = (int32_t)n_new;
    counters[REF_C_TOK_REUSE] += (unsigned long long)n_reuse;
    counters[REF_C_TOK_ANCHOR] += (unsigned long long)n_anchor;
    counters[REF_C_TOK_NEW] += (unsigned long long)n_new;
    /* REUSE: the rotated pairs of the key rows (read + write); refreshed rows: keys and values (read + write) */
    counters[REF_C_BYTES_KV] += (unsigned long long)((rot * L * H * 2 * rot_pairs + cop * L * 2 * rowel) * esz * 2);
    counters[REF_C_STREAM_STEPS] += 1;
  }
  free(tdisp);
  free(tpold);
  free(tslot);
  free(used);
  free(tfrm);
  return 0;
}

/* ---------------------------------------------------------------------------------------------------- */
/* NEXT-2: GPU preprocessing fused into the compaction ("Resizing, color-space conversion, and      */
/* normalization are fused into a single batched operation over all frames").  Decoded frames arrive as   */
/* NV12 (NVDEC's output: a Y plane and an interleaved 2x2-subsampled UV plane).  A model-input pixel      */
/* (c, y, x) of the MH x MW input (MH = grid_h*patch, MW = grid_w*patch) is defined, in fp32 and in this   */
/* order (reading NEXT-2):                                                                                 */
/*   colour  BT.601 limited range: R = kY(Y-16) + kRV(V-128), G = (kY(Y-16) - kGU(U-128)) - kGV(V-128),     */
/*           B = kY(Y-16) + kBU(U-128), clamped to [0, 255]; chroma of pixel (y, x) at UV row y/2, col x/2  */
/*   resize  bilinear, half-pixel centres (PyTorch interpolate align_corners=False, antialias=False):      */
/*           f = (o + 0.5) * (src/M) - 0.5, clamped at 0; i0 = floor(f), i1 = i0 + (i0 < src-1),           */
/*           l = f - i0; value = (1-ly)((1-lx) p00 + lx p01) + ly((1-lx) p10 + lx p11)                     */
/*   scale   t = value / 255; out = (t - mean_c) / std_c; stored as bf16 (RNE).                            */
/* ---------------------------------------------------------------------------------------------------- */
static const float REF_KY = 1.164383f, REF_KRV = 1.596027f, REF_KGU = 0.391762f, REF_KGV = 0.812968f,
                   REF_KBU = 2.017232f;

static float ref_clamp255(float v) { return v < 0.0f ? 0.0f : (v > 255.0f ? 255.0f : v); }

void codecsight_ref_nv12_rgb(const uint8_t* Y, const uint8_t* UV, const ref_pre* pp, int64_t y, int64_t x,
                             float rgb[3]) {
  const float c = (float)((int32_t)Y[y * pp->y_pitch + x] - 16);
  const float d = (float)((int32_t)UV[(y / 2) * pp->uv_pitch + 2 * (x / 2)] - 128);
  const float e = (float)((int32_t)UV[(y / 2) * pp->uv_pitch + 2 * (x / 2) + 1] - 128);
  rgb[0] = ref_clamp255(REF_KY * c + REF_KRV * e);
  rgb[1] = ref_clamp255((REF_KY * c - REF_KGU * d) - REF_KGV * e);
  rgb[2] = ref_clamp255(REF_KY * c + REF_KBU * d);
}

/* source index pair and weight of model coordinate o along an axis of `src` source and `m` model pixels */
static void ref_axis(int64_t o, int64_t src, int64_t m, int64_t* i0, int64_t* i1, float* l) {
  const float scale = (float)src / (float)m;
  float f = ((float)o + 0.5f) * scale - 0.5f;
  if (f < 0.0f) f = 0.0f;
  *i0 = (int64_t)f; /* f >= 0: truncation is floor */
  *i1 = *i0 + (*i0 < src - 1 ? 1 : 0);
  *l = f - (float)*i0;
}

float codecsight_ref_model_pixel(const ref_grid* g, const ref_pre* pp, const uint8_t* Y, const uint8_t* UV, int64_t c,
                                 int64_t yo, int64_t xo) {
  const int64_t MH = (int64_t)g->grid_h * g->patch, MW = (int64_t)g->grid_w * g->patch;
  int64_t y0, y1, x0, x1;
  float ly, lx;
  ref_axis(yo, pp->src_h, MH, &y0, &y1, &ly);
  ref_axis(xo, pp->src_w, MW, &x0, &x1, &lx);
  float p00[3], p01[3], p10[3], p11[3];
  codecsight_ref_nv12_rgb(Y, UV, pp, y0, x0, p00);
  codecsight_ref_nv12_rgb(Y, UV, pp, y0, x1, p01);
  codecsight_ref_nv12_rgb(Y, UV, pp, y1, x0, p10);
  codecsight_ref_nv12_rgb(Y, UV, pp, y1, x1, p11);
  const float hx = 1.0f - lx, hy = 1.0f - ly;
  const float top = hx * p00[c] + lx * p01[c];
  const float bot = hx * p10[c] + lx * p11[c];
  const float v = hy * top + ly * bot;
  const float t = v / 255.0f;
  return (t - pp->mean[c]) / pp->stdv[c];
}

static int ref_pre_ok(const ref_pre* pp) {
  if (!pp) return -1;
  if (pp->src_w < 2 || pp->src_h < 2 || pp->src_w % 2 || pp->src_h % 2 || pp->src_w > 16384 || pp->src_h > 16384)
    return -2;
  if (pp->y_pitch < pp->src_w || pp->uv_pitch < pp->src_w) return -2;
  if (pp->color != 0) return -3;
  for (int c = 0; c < 3; ++c)
    if (!(pp->stdv[c] > 0.0f) || isnan(pp->mean[c])) return -1;
  return 0;
}

void codecsight_ref_preprocess_frame(const ref_grid* g, const ref_pre* pp, const uint8_t* Y, const uint8_t* UV,
                                     uint16_t* out) {
  const int64_t MH = (int64_t)g->grid_h * g->patch, MW = (int64_t)g->grid_w * g->patch;
  for (int64_t c = 0; c < 3; ++c)
    for (int64_t y = 0; y < MH; ++y)
      for (int64_t x = 0; x < MW; ++x)
        out[(c * MH + y) * MW + x] = ref_f32_to_bf16(codecsight_ref_model_pixel(g, pp, Y, UV, c, y, x));
}

/* Distinct 32-B source sectors (Y plane: row y, byte x; UV plane: row y/2, bytes 2(x/2), 2(x/2)+1 -- the same
 * sector) touched by the four taps of every model pixel of every kept group, summed over the frames, x 32 B. */
static unsigned long long ref_nv12_source_bytes(const ref_grid* g, const ref_pre* pp, const uint32_t* keep_mask,
                                                int64_t mask_frame_stride, int32_t n_streams, int32_t n_frames) {
  const int64_t MH = (int64_t)g->grid_h * g->patch, MW = (int64_t)g->grid_w * g->patch, G = g->group;
  const int64_t gp = G * g->patch, nw = ref_words(g), sc = (pp->src_w + 31) / 32;
  const int64_t yrows = pp->src_h, uvrows = (pp->src_h + 1) / 2;
  uint8_t* ys = (uint8_t*)malloc((size_t)(yrows * sc));
  uint8_t* uvs = (uint8_t*)malloc((size_t)(uvrows * sc));
  unsigned long long total = 0;
  if (!ys || !uvs) { free(ys); free(uvs); return 0; }
  for (int64_t s = 0; s < n_streams; ++s)
    for (int64_t j = 0; j < n_frames; ++j) {
      const uint32_t* m = keep_mask + (s * mask_frame_stride + j) * nw;
      memset(ys, 0, (size_t)(yrows * sc));
      memset(uvs, 0, (size_t)(uvrows * sc));
      for (int64_t gr = 0; gr < g->grid_h / G; ++gr)
        for (int64_t gc = 0; gc < g->grid_w / G; ++gc) {
          int any = 0;
          for (int64_t dy = 0; dy < G; ++dy)
            for (int64_t dx = 0; dx < G; ++dx) any |= ref_bit(m, (gr * G + dy) * g->grid_w + gc * G + dx);
          if (!any) continue;
          for (int64_t yo = gr * gp; yo < (gr + 1) * gp; ++yo)
            for (int64_t xo = gc * gp; xo < (gc + 1) * gp; ++xo) {
              int64_t y0, y1, x0, x1;
              float ly, lx;
              ref_axis(yo, pp->src_h, MH, &y0, &y1, &ly);
              ref_axis(xo, pp->src_w, MW, &x0, &x1, &lx);
              const int64_t yy[2] = {y0, y1}, xx[2] = {x0, x1};
              for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b) {
                  ys[yy[a] * sc + xx[b] / 32] = 1;
                  uvs[(yy[a] / 2) * sc + (2 * (xx[b] / 2)) / 32] = 1;
                }
            }
        }
      for (int64_t i = 0; i < yrows * sc; ++i) total += ys[i];
      for (int64_t i = 0; i < uvrows * sc; ++i) total += uvs[i];
    }
  free(ys);
  free(uvs);
  return total * 32ull;
}

int codecsight_ref_compact_nv12(const ref_grid* g, const ref_pre* pp, int32_t n_streams, int32_t n_frames,
                                const uint32_t* keep_mask, int64_t mask_frame_stride, const int32_t* frame_index,
                                const void* const* y_planes, const void* const* uv_planes, int64_t capacity,
                                void* packed, int32_t* pos_ids, int32_t* src_index, int32_t* frame_offsets,
                                unsigned long long* counters, int32_t* status) {
  int rc = ref_grid_ok(g);
  if (rc) return rc;
  if ((rc = ref_pre_ok(pp))) return rc;
  if (n_streams < 0 || n_frames < 1 || mask_frame_stride < n_frames || capacity < 0) return -1;
  const int64_t np = (int64_t)g->grid_w * g->grid_h, nw = ref_words(g), G = g->group, p = g->patch;
  const int64_t n_slots = (int64_t)n_streams * n_frames;
  if (n_slots * np >= 2147483648LL) return -3;
  if (!frame_offsets || !counters || !status) return -1;
  if (n_slots > 0 && (!keep_mask || !frame_index || !y_planes || !uv_planes)) return -1;
  if (capacity > 0 && (!packed || !pos_ids || !src_index)) return -1;
  const int64_t row = 3 * p * p;
  uint16_t* out = (uint16_t*)packed;
  int64_t off = 0, written = 0;
  for (int64_t s = 0; s < n_streams; ++s)
    for (int64_t j = 0; j < n_frames; ++j) {
      const int64_t slot = s * n_frames + j;
      const uint32_t* m = keep_mask + (s * mask_frame_stride + j) * nw;
      const uint8_t* Y = (const uint8_t*)y_planes[slot];
      const uint8_t* UV = (const uint8_t*)uv_planes[slot];
      frame_offsets[slot] = (int32_t)off;
      for (int64_t gr = 0; gr < g->grid_h / G; ++gr)
        for (int64_t gc = 0; gc < g->grid_w / G; ++gc) {
          int any = 0;
          for (int64_t dy = 0; dy < G; ++dy)
            for (int64_t dx = 0; dx < G; ++dx) any |= ref_bit(m, (gr * G + dy) * g->grid_w + gc * G + dx);
          if (!any) continue;
          for (int64_t dy = 0; dy < G; ++dy)
            for (int64_t dx = 0; dx < G; ++dx) {
              const int64_t h = gr * G + dy, w = gc * G + dx, n = off++;
              if (n >= capacity) { *status |= REF_ST_CAPACITY; continue; }
              for (int64_t c = 0; c < 3; ++c)
                for (int64_t y = 0; y < p; ++y)
                  for (int64_t x = 0; x < p; ++x)
                    out[n * row + c * p * p + y * p + x] =
                        ref_f32_to_bf16(codecsight_ref_model_pixel(g, pp, Y, UV, c, h * p + y, w * p + x));
              pos_ids[3 * n + 0] = frame_index[slot];
              pos_ids[3 * n + 1] = (int32_t)h;
              pos_ids[3 * n + 2] = (int32_t)w;
              src_index[n] = (int32_t)(slot * np + h * g->grid_w + w);
              ++written;
            }
        }
    }
  frame_offsets[n_slots] = (int32_t)off;
  counters[REF_C_PACKED_ROWS] += (unsigned long long)written;
  /* algorithmic bytes: masks + offsets, per written row its output (+16 B of ids), and the source the kept groups
     read: per frame, every distinct 32-B sector of the Y and UV planes (offsets from the plane start) holding a
     bilinear tap of a kept group's model pixel (reading NEXT-2 bytes; counted when both pitches are multiples of
     32, so that a sector is (row, byte column / 32)) */
  counters[REF_C_BYTES_COMPACT] += (unsigned long long)(n_slots * (4 * nw + 4) + written * (row * 2 + 16));
  if (pp->y_pitch % 32 == 0 && pp->uv_pitch % 32 == 0)
    counters[REF_C_BYTES_COMPACT] += ref_nv12_source_bytes(g, pp, keep_mask, mask_frame_stride, n_streams, n_frames);
  return 0;
}

/* ---------------------------------------------------------------------------------------------------- */
/* NEXT-4 (a): real H.264 metadata ingest.  FFmpeg exports a frame's motion as AVMotionVector records      */
/* (libavutil/motion_vector.h) per coded partition (4x4 .. 16x16, the decoder's "MV extraction"):  */
/* destination centre (dst_x, dst_y), size w x h, motion (motion_x, motion_y) / motion_scale pixels.       */
/* Rasterised onto the 16x16 MB grid (reading NEXT-4): an MB takes the motion vector of largest magnitude  */
/* among the past-reference partitions (source < 0) overlapping it with positive area (ties: the first     */
/* record) -- the same conservative max that the patch resampling uses -- converted to quarter     */
/* pel, mv_q = trunc(4 * motion / motion_scale) clamped to int16, type INTER; an MB that no partition      */
/* covers was intra coded (no motion exported): type INTRA.  SAD is not exported by FFmpeg: 0.             */
/* ---------------------------------------------------------------------------------------------------- */
static int32_t ref_qpel(int32_t motion, int32_t scale) {
  int64_t v = ((int64_t)motion * 4) / (scale > 0 ? scale : 1); /* C division truncates toward zero */
  if (v > 32767) v = 32767;
  if (v < -32768) v = -32768;
  return (int32_t)v;
}

int codecsight_ref_mv_rasterize(const ref_grid* g, int32_t n_frames, const ref_av_mv* mvs, const int64_t* mv_offsets,
                                ref_mb* out) {
  if (!g || n_frames < 0 || (n_frames > 0 && (!mvs || !mv_offsets || !out))) return -1;
  const int64_t cols = g->mb_cols, rows = g->mb_rows, mb = g->mb_size;
  for (int64_t f = 0; f < n_frames; ++f) {
    for (int64_t j = 0; j < rows; ++j)
      for (int64_t i = 0; i < cols; ++i) {
        int64_t best = -1, best_sq = -1;
        for (int64_t r = mv_offsets[f]; r < mv_offsets[f + 1]; ++r) {
          const ref_av_mv* m = &mvs[r];
          if (m->source >= 0) continue;
          /* partition rectangle [dst - size/2, dst - size/2 + size) in pixels */
          const int64_t x0 = (int64_t)m->dst_x - m->w / 2, y0 = (int64_t)m->dst_y - m->h / 2;
          const int64_t ox = (x0 + m->w < mb * (i + 1) ? x0 + m->w : mb * (i + 1)) - (x0 > mb * i ? x0 : mb * i);
          const int64_t oy = (y0 + m->h < mb * (j + 1) ? y0 + m->h : mb * (j + 1)) - (y0 > mb * j ? y0 : mb * j);
          if (ox <= 0 || oy <= 0) continue;
          const int64_t qx = ref_qpel(m->motion_x, m->motion_scale), qy = ref_qpel(m->motion_y, m->motion_scale);
          const int64_t sq = qx * qx + qy * qy;
          if (sq > best_sq) { best_sq = sq; best = r; }
        }
        ref_mb* o = &out[(f * rows + j) * cols + i];
        o->sad = 0;
        o->reserved = 0;
        if (best < 0) {
          o->mvx_qpel = 0;
          o->mvy_qpel = 0;
          o->mb_type = REF_MB_INTRA;
        } else {
          o->mvx_qpel = (int16_t)ref_qpel(mvs[best].motion_x, mvs[best].motion_scale);
          o->mvy_qpel = (int16_t)ref_qpel(mvs[best].motion_y, mvs[best].motion_scale);
          o->mb_type = REF_MB_INTER;
        }
      }
  }
  return 0;
}

/* ---------------------------------------------------------------------------------------------------- */
/* NEXT-4 (b): the similar-patch-ratio distribution of fig:mv_residual_analysis_cdf: */
/* for every P-frame and threshold tau_t, the ratio of patches whose score is below tau_t ("similar") --   */
/* count / n_patches -- falls in bin floor(count * n_bins / n_patches) (the last bin holds ratio 1);        */
/* hist[t][bin] counts frames.  The CDF is the running sum of a row.                                       */
/* ---------------------------------------------------------------------------------------------------- */
int codecsight_ref_similar_hist(const float* score, const uint8_t* frame_type, int64_t n_frames, int32_t n_patches,
                                const float* taus, int32_t n_tau, int32_t n_bins, unsigned long long* hist) {
  if (n_frames < 0 || n_patches < 1 || n_tau < 1 || n_bins < 1) return -1;
  for (int64_t f = 0; f < n_frames; ++f) {
    if (frame_type[f] != REF_FRAME_P) continue;
    for (int32_t t = 0; t < n_tau; ++t) {
      int64_t cnt = 0;
      for (int32_t i = 0; i < n_patches; ++i) cnt += (score[f * n_patches + i] < taus[t]) ? 1 : 0;
      int64_t bin = cnt * n_bins / n_patches;
      if (bin >= n_bins) bin = n_bins - 1;
      hist[(int64_t)t * n_bins + bin] += 1;
    }
  }
  return 0;
}
