/* Check of the guarded reciprocal used by the fused NV12 normalisation (compact.cu, norm_bf16):
 *   q = RN(a * RN(1/std)); if the low 16 bits of q are within 8 of 0x8000, q = RN(a / std);
 *   bf16_rne(q) == bf16_rne(RN(a / std))
 * for every fp32 a in [-4, 4] (stride 1 = all ~2.2e9 of them per std) and a set of std values: the CLIP / Qwen2-VL
 * stds, 1, 255, the edges of the accepted range 2^-20 and 2^20, and pseudo-random stds inside it.
 * Usage: check_norm_bf16 [stride] [n_random_std]                                                               */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint32_t bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float from_bits(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint16_t bf16_rne(float f) { uint32_t u = bits(f); return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16); }

int main(int argc, char** argv) {
  const uint32_t stride = argc > 1 ? (uint32_t)strtoul(argv[1], 0, 10) : 1u;
  const int nrand = argc > 2 ? atoi(argv[2]) : 8;
  float stds[64] = {0.26862954f, 0.26130258f, 0.27577711f, 1.0f, 255.0f, 0x1p-20f, 0x1p20f, 0.5f};
  int ns = 8;
  uint64_t x = 0x9e3779b97f4a7c15ull;
  for (int i = 0; i < nrand && ns < 64; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    stds[ns++] = ldexpf(1.0f + (float)(x & 0xffffff) / 16777216.0f, (int)((x >> 32) % 41) - 20);
  }
  unsigned long long n = 0, bad = 0, slow = 0;
  const uint32_t top = bits(4.0f);
  for (int k = 0; k < ns; ++k) {
    const float sd = stds[k], r = 1.0f / sd;
    for (int sign = 0; sign < 2; ++sign) {
      for (uint64_t u = 0; u <= top; u += stride) {
        const float a = from_bits((uint32_t)u | (sign ? 0x80000000u : 0u));
        float q = a * r;
#ifndef NOGUARD
        if (((bits(q) & 0xffffu) - 0x7ff8u) <= 16u) { q = a / sd; ++slow; }
#endif
        const float ex = a / sd;
        if (bf16_rne(q) != bf16_rne(ex)) {
          if (bad < 10) printf("mismatch std %a a %a: %04x vs %04x\n", sd, a, bf16_rne(q), bf16_rne(ex));
          ++bad;
        }
        ++n;
      }
    }
  }
  printf("checked %llu (a, std) pairs over %d stds, exact-division fallbacks %llu, mismatches %llu\n", n, ns, slow, bad);
  return bad != 0;
}
