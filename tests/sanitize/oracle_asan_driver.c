/* oracle_asan_driver.c -- TEST INFRASTRUCTURE ("oracle under -fsanitize=address,undefined").
 *
 * Drives every entry point of the C oracle (oracle/codecsight_ref.c) through a C1-shaped stream (448x448, w = 8,
 * s = 2, GOP 4, toy fp32 KV and a bf16 Qwen-layout KV) and a ragged geometry, with capacity truncation, so that
 * AddressSanitizer / UndefinedBehaviorSanitizer see every loop and index of the oracle.  Built and run by
 * tests/test_oracle_sanitizers.py with gcc -fsanitize=address,undefined -fno-sanitize-recover=all; exit code 0
 * means every call returned its expected code and no sanitizer fired.  Inputs come from a fixed LCG.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "codecsight_ref.h"

static uint64_t g_rng = 0x9e3779b97f4a7c15ull;
static uint32_t rnd(void) {
  g_rng = g_rng * 6364136223846793005ull + 1442695040888963407ull;
  return (uint32_t)(g_rng >> 33);
}

static int g_fail = 0;
#define CHECK(cond, ...)                                   \
  do {                                                     \
    if (!(cond)) {                                         \
      fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      fprintf(stderr, __VA_ARGS__);                        \
      fprintf(stderr, "\n");                               \
      g_fail = 1;                                          \
    }                                                      \
  } while (0)

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) {
    fprintf(stderr, "out of memory\n");
    exit(2);
  }
  return p;
}

static void fill_mb(ref_mb* mb, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t r = rnd();
    if (r % 1000 < 985) { /* mostly static background (SKIP, zero MV): pruning happens */
      mb[i].mvx_qpel = mb[i].mvy_qpel = 0;
      mb[i].sad = 0;
      mb[i].mb_type = 1;
      mb[i].reserved = 0;
      continue;
    }
    mb[i].mvx_qpel = (int16_t)((int)(r % 9) - 4);
    mb[i].mvy_qpel = (int16_t)((int)((r >> 4) % 9) - 4);
    mb[i].sad = (uint16_t)(rnd() % 12000);
    mb[i].mb_type = (uint8_t)((r >> 8) % 100 < 2 ? 2 : ((r >> 12) % 3 == 0 ? 1 : 0));
    mb[i].reserved = 0;
  }
}

/* One stream through `steps` windows: score -> compact -> kv_refresh (out of place) -> kv_refresh_paged. */
static void run_stream(const ref_grid* g, const ref_kv* kv, int w, int s, int gop, int steps) {
  const int np = g->grid_w * g->grid_h, nw = (np + 31) / 32, ring = w + s;
  const int H = g->grid_h * g->patch, W = g->grid_w * g->patch;
  const int64_t mbn = (int64_t)g->mb_rows * g->mb_cols;
  const int64_t groups = (int64_t)(g->grid_w / g->group) * (g->grid_h / g->group);
  uint32_t* mring = xcalloc((size_t)ring * nw, 4);
  uint8_t* tring = xcalloc((size_t)ring, 1);
  uint32_t* gop_state = xcalloc((size_t)nw + 1, 4);
  unsigned long long counters[REF_NCOUNTERS];
  memset(counters, 0, sizeof(counters));
  const int64_t cap = w * groups + kv->n_prompt;
  const int64_t rcap = cap;
  const int64_t row = (int64_t)kv->kv_heads * kv->head_dim;
  const size_t esz = kv->dtype == 0 ? 2 : 4;
  const size_t cache_bytes = (size_t)kv->layers * 2 * cap * row * esz;
  void* caches[2] = {xcalloc(cache_bytes, 1), xcalloc(cache_bytes, 1)};
  void* pool = xcalloc(cache_bytes, 1);
  void* refr = xcalloc((size_t)kv->layers * 2 * rcap * row, esz);
  for (size_t i = 0; i < cache_bytes / 4; ++i) {
    ((uint32_t*)caches[0])[i] = rnd() & 0x3f7f3f7fu;  /* finite values in both dtypes */
    ((uint32_t*)pool)[i] = rnd() & 0x3f7f3f7fu;
  }
  for (size_t i = 0; i < (size_t)kv->layers * 2 * rcap * row * esz / 4; ++i) ((uint32_t*)refr)[i] = rnd() & 0x3f7f3f7fu;
  int32_t* slots[2] = {xcalloc((size_t)cap, 4), xcalloc((size_t)cap, 4)};
  for (int64_t i = 0; i < cap; ++i) slots[0][i] = (int32_t)i;
  uint8_t* disp = xcalloc((size_t)cap, 1);
  int32_t* pold = xcalloc((size_t)cap, 4);
  int32_t ntok[4];
  int cur = 0, scur = 0;
  for (int k = 0; k < steps; ++k) {
    const int f0 = k == 0 ? 0 : (k - 1) * s + w, n = k == 0 ? w : s;
    const int off = f0 % ring;
    if (off + n > ring) continue; /* keep the batch inside the ring (w, s chosen so this never triggers) */
    ref_mb* mb = xcalloc((size_t)(n * mbn), sizeof(ref_mb));
    fill_mb(mb, n * mbn);
    for (int f = 0; f < n; ++f) tring[off + f] = (uint8_t)((f0 + f) % gop == 0 ? 0 : 1);
    float* score = xcalloc((size_t)n * np, 4);
    int32_t* kept = xcalloc((size_t)n, 4);
    int32_t status = 0;
    int rc = codecsight_ref_score_patches(g, 1, n, mb, tring + off, mring + (size_t)off * nw, ring - off, gop_state,
                                          score, kept, counters, &status);
    CHECK(rc == 0 && status == 0, "score_patches rc %d status %d", rc, status);
    /* compaction, planar frames: full capacity, then truncated mid-group */
    uint16_t** frames = xcalloc((size_t)n, sizeof(uint16_t*));
    for (int f = 0; f < n; ++f) {
      frames[f] = xcalloc((size_t)3 * H * W, 2);
      for (int64_t i = 0; i < (int64_t)3 * H * W; ++i) frames[f][i] = (uint16_t)rnd();
    }
    int32_t* fidx = xcalloc((size_t)n, 4);
    for (int f = 0; f < n; ++f) fidx[f] = f0 + f;
    const int64_t pcap = (int64_t)n * np;
    const int64_t rowel = 3ll * g->patch * g->patch;
    uint16_t* packed = xcalloc((size_t)(pcap * rowel), 2);
    int32_t* pos = xcalloc((size_t)pcap * 3, 4);
    int32_t* src = xcalloc((size_t)pcap, 4);
    int32_t* offs = xcalloc((size_t)n + 1, 4);
    for (int trunc = 0; trunc < 2; ++trunc) {
      status = 0;
      const int64_t c = trunc ? (pcap / 3 + 1) : pcap;
      rc = codecsight_ref_compact(g, 1, n, mring + (size_t)off * nw, ring - off, fidx, (const void* const*)frames, 0, c,
                                  packed, pos, src, offs, counters, &status);
      CHECK(rc == 0, "compact rc %d", rc);
    }
    /* temporal patches (tp = 2) over the same masks, with unit masks / types */
    if (n % 2 == 0) {
      uint32_t* umask = xcalloc((size_t)(n / 2) * nw, 4);
      uint8_t* utype = xcalloc((size_t)(n / 2), 1);
      uint16_t* tpacked = xcalloc((size_t)(pcap / 2 * rowel * 2), 2);
      int32_t* uidx = xcalloc((size_t)n / 2, 4);
      for (int u = 0; u < n / 2; ++u) uidx[u] = f0 / 2 + u;
      status = 0;
      rc = codecsight_ref_compact_tp(g, 2, 1, n / 2, mring + (size_t)off * nw, ring - off, uidx,
                                     (const void* const*)frames, 0, pcap / 2, tpacked, pos, src, offs, umask, n / 2,
                                     tring + off, utype, counters, &status);
      CHECK(rc == 0, "compact_tp rc %d", rc);
      free(umask);
      free(utype);
      free(tpacked);
      free(uidx);
    }
    /* KV refresh, out of place and in place */
    const ref_window win = {w, s, k, ring};
    const void* old_c[1] = {caches[cur]};
    void* new_c[1] = {caches[1 - cur]};
    const void* ref_c[1] = {refr};
    status = 0;
    rc = codecsight_ref_kv_refresh(g, kv, &win, 1, mring, tring, k ? old_c : NULL, new_c, k ? ref_c : NULL, cap, disp,
                                   pold, ntok, counters, &status);
    CHECK(rc == 0 && status == 0, "kv_refresh rc %d status %d (step %d)", rc, status, k);
    cur = 1 - cur;
    void* pools[1] = {pool};
    status = 0;
    rc = codecsight_ref_kv_refresh_paged(g, kv, &win, 1, mring, tring, pools, k ? slots[scur] : NULL, slots[1 - scur],
                                         cap, k ? ref_c : NULL, cap, disp, pold, ntok, counters, &status);
    CHECK(rc == 0 && status == 0, "kv_refresh_paged rc %d status %d (step %d)", rc, status, k);
    scur = 1 - scur;
    /* similar-patch histogram over the step's scores */
    const float taus[3] = {0.25f, 1.0f, 5.0f};
    unsigned long long hist[3 * 10];
    memset(hist, 0, sizeof(hist));
    rc = codecsight_ref_similar_hist(score, tring + off, n, np, taus, 3, 10, hist);
    CHECK(rc == 0, "similar_hist rc %d", rc);
    for (int f = 0; f < n; ++f) free(frames[f]);
    free(frames);
    free(fidx);
    free(packed);
    free(pos);
    free(src);
    free(offs);
    free(score);
    free(kept);
    free(mb);
  }
  printf("stream %dx%d w=%d s=%d: frames %llu kept %llu/%llu reuse %llu anchor %llu new %llu packed rows %llu\n",
         g->src_w, g->src_h, w, s, counters[REF_C_FRAMES], counters[REF_C_KEPT], counters[REF_C_PATCHES],
         counters[REF_C_TOK_REUSE], counters[REF_C_TOK_ANCHOR], counters[REF_C_TOK_NEW], counters[REF_C_PACKED_ROWS]);
  CHECK(counters[REF_C_TOK_REUSE] > 0 && counters[REF_C_KEPT] > 0, "degenerate stream");
  free(mring);
  free(tring);
  free(gop_state);
  free(caches[0]);
  free(caches[1]);
  free(pool);
  free(refr);
  free(slots[0]);
  free(slots[1]);
  free(disp);
  free(pold);
}

static void run_nv12(const ref_grid* g) {
  const int sw = 160, sh = 120, np = g->grid_w * g->grid_h, nw = (np + 31) / 32, n = 2;
  uint8_t* Y[2];
  uint8_t* UV[2];
  for (int f = 0; f < n; ++f) {
    Y[f] = xcalloc((size_t)sw * sh, 1);
    UV[f] = xcalloc((size_t)sw * (sh / 2), 1);
    for (int i = 0; i < sw * sh; ++i) Y[f][i] = (uint8_t)(16 + rnd() % 220);
    for (int i = 0; i < sw * sh / 2; ++i) UV[f][i] = (uint8_t)(16 + rnd() % 225);
  }
  ref_pre pp = {sw, sh, sw, sw, 0, {0.48145466f, 0.4578275f, 0.40821073f}, {0.26862954f, 0.26130258f, 0.27577711f}};
  uint32_t* mask = xcalloc((size_t)n * nw, 4);
  for (int i = 0; i < n * nw; ++i) mask[i] = rnd();
  int32_t fidx[2] = {0, 1};
  const int64_t cap = (int64_t)n * np, rowel = 3ll * g->patch * g->patch;
  uint16_t* packed = xcalloc((size_t)(cap * rowel), 2);
  int32_t* pos = xcalloc((size_t)cap * 3, 4);
  int32_t* src = xcalloc((size_t)cap, 4);
  int32_t offs[3];
  unsigned long long counters[REF_NCOUNTERS];
  memset(counters, 0, sizeof(counters));
  int32_t status = 0;
  int rc = codecsight_ref_compact_nv12(g, &pp, 1, n, mask, n, fidx, (const void* const*)Y, (const void* const*)UV,
                                       cap - 3, packed, pos, src, offs, counters, &status);
  CHECK(rc == 0, "compact_nv12 rc %d", rc);
  uint16_t* full = xcalloc((size_t)3 * g->grid_h * g->patch * g->grid_w * g->patch, 2);
  codecsight_ref_preprocess_frame(g, &pp, Y[0], UV[0], full);
  for (int f = 0; f < n; ++f) {
    free(Y[f]);
    free(UV[f]);
  }
  free(full);
  free(mask);
  free(packed);
  free(pos);
  free(src);
}

static void run_mv_rope(const ref_grid* g) {
  const int n = 2, per = 40;
  ref_av_mv* mvs = xcalloc((size_t)n * per, sizeof(ref_av_mv));
  int64_t offs[3] = {0, per, 2 * per};
  for (int i = 0; i < n * per; ++i) {
    mvs[i].source = (rnd() % 5 == 0) ? 1 : -1;
    mvs[i].w = (uint8_t)(4 << (rnd() % 3));
    mvs[i].h = (uint8_t)(4 << (rnd() % 3));
    mvs[i].dst_x = (int16_t)(rnd() % (unsigned)(g->src_w + 16)) - 8;
    mvs[i].dst_y = (int16_t)(rnd() % (unsigned)(g->src_h + 16)) - 8;
    mvs[i].motion_x = (int32_t)(rnd() % 200) - 100;
    mvs[i].motion_y = (int32_t)(rnd() % 200) - 100;
    mvs[i].motion_scale = (uint16_t)(1 + rnd() % 4);
  }
  ref_mb* out = xcalloc((size_t)n * g->mb_rows * g->mb_cols, sizeof(ref_mb));
  int rc = codecsight_ref_mv_rasterize(g, n, mvs, offs, out);
  CHECK(rc == 0, "mv_rasterize rc %d", rc);
  float k[2 * 16], o[2 * 16];
  for (int i = 0; i < 32; ++i) k[i] = (float)((int)(rnd() % 2001) - 1000) / 250.0f;
  codecsight_ref_rope_rotate_f32(k, 2, 16, 1e4, -37, o);
  float V[1024], R[1024], M[1024];
  int32_t st = 0;
  ref_mb* mb = xcalloc((size_t)g->mb_rows * g->mb_cols, sizeof(ref_mb));
  fill_mb(mb, (int64_t)g->mb_rows * g->mb_cols);
  codecsight_ref_patch_fields(g, mb, V, R, M, &st);
  (void)codecsight_ref_mb_magnitude(-32768, -32768, 0);
  free(mb);
  free(mvs);
  free(out);
}

int main(void) {
  /* C1 geometry: 448x448 source, 16-px MBs (28x28), 32x32 patches of 14, 2x2 groups, tau 0.25, alpha 0.5 */
  ref_grid c1 = {448, 448, 16, 28, 28, 14, 32, 32, 2, 0.25f, 0.5f};
  ref_kv toy = {2, 2, 16, 1, 0, 0, 1e4, 4, REF_ROPE_1D, {0, 0, 0}, 1};
  toy.capacity = 8 * 256 + toy.n_prompt;
  toy.refresh_capacity = toy.capacity;
  run_stream(&c1, &toy, 8, 2, 4, 7);
  ref_kv qwen = {2, 4, 128, 0, 0, 0, 1e6, 4, REF_ROPE_MROPE, {16, 24, 24}, 1};
  qwen.capacity = 4 * 256 + qwen.n_prompt;
  qwen.refresh_capacity = qwen.capacity;
  run_stream(&c1, &qwen, 4, 2, 4, 5);
  /* ragged geometry: 100x44 source, 8-px MBs (13x6, last column/row partial), 8x6 patches of 4, 2x2 groups */
  ref_grid rg = {100, 44, 8, 13, 6, 4, 8, 6, 2, 0.25f, 0.0f};
  ref_kv toy2 = toy;
  toy2.capacity = 6 * 12 + toy2.n_prompt;
  toy2.refresh_capacity = toy2.capacity;
  run_stream(&rg, &toy2, 6, 3, 3, 6);
  run_nv12(&c1);
  run_mv_rope(&c1);
  if (g_fail) return 1;
  printf("oracle sanitizer driver: ok\n");
  return 0;
}
