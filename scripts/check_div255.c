/* Exhaustive check of the division-free v / 255 used by the fused NV12 preprocessing (compact.cu):
 *   q = RN(v * RN(1/255)); t = RN(q + RN-fma residual) == RN(v / 255)  for every fp32 v in [lo, hi].
 * Usage: check_div255 [stride]   (stride 1 = every float in [0, 512]; ~50 s single-threaded)            */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
int main(int argc, char** argv) {
  const uint32_t stride = argc > 1 ? (uint32_t)strtoul(argv[1], 0, 10) : 1u;
  const float b = 255.0f, r = 1.0f / 255.0f;
  float f0 = 0.0f, f1 = 512.0f;
  uint32_t lo, hi;
  memcpy(&lo, &f0, 4);
  memcpy(&hi, &f1, 4);
  unsigned long long n = 0, bad = 0;
  for (uint64_t u = lo; u <= hi; u += stride) {
    uint32_t w = (uint32_t)u;
    float a;
    memcpy(&a, &w, 4);
    const float q = a * r;
    const float t = fmaf(fmaf(-q, b, a), r, q);
    const float ex = a / b;
    if (memcmp(&t, &ex, 4) != 0) ++bad;
    ++n;
  }
  printf("checked %llu values, mismatches %llu\n", n, bad);
  return bad != 0;
}
