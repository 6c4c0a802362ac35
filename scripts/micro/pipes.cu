// Which SM pipe executes an instruction (ncu sm__inst_executed_pipe_*): one kernel per op, 8 independent chains.
#include <cstdint>
#include <cstdio>
#define N 4096
__global__ void k_i2fp(uint32_t* o, uint32_t s) {
  uint32_t a[8]; float f[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 7 + i + s; f[i] = 0; }
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { f[i] += __uint2float_rn(a[i]); a[i] += 3; }
  float t = 0; for (int i = 0; i < 8; ++i) t += f[i];
  o[threadIdx.x] = __float_as_uint(t);
}
__global__ void k_prmt(uint32_t* o, uint32_t s) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7 + i + s;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __byte_perm(a[i], s, 0x7540u);
  uint32_t t = 0; for (int i = 0; i < 8; ++i) t ^= a[i];
  o[threadIdx.x] = t;
}
__global__ void k_vimnmx(uint32_t* o, uint32_t s) {
  int a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7 + i + s;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { int r; asm volatile("min.relu.s32 %0, %1, %2;" : "=r"(r) : "r"(a[i]), "r"((int)s)); a[i] = r + 1; }
  uint32_t t = 0; for (int i = 0; i < 8; ++i) t ^= a[i];
  o[threadIdx.x] = t;
}
__global__ void k_iadd(uint32_t* o, uint32_t s) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7 + i + s;
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] + 0x4B000000u;
  uint32_t t = 0; for (int i = 0; i < 8; ++i) t ^= a[i];
  o[threadIdx.x] = t;
}
__global__ void k_ffma2(uint32_t* o, uint32_t s) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x + i, s);
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      unsigned long long r, x, c;
      asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a[i].x), "f"(a[i].y));
      asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(1.0001f), "f"(0.999f));
      asm volatile("fma.rn.f32x2 %0, %1, %2, %1;" : "=l"(r) : "l"(x), "l"(c));
      asm("mov.b64 {%0, %1}, %2;" : "=f"(a[i].x), "=f"(a[i].y) : "l"(r));
    }
  float t = 0; for (int i = 0; i < 8; ++i) t += a[i].x + a[i].y;
  o[threadIdx.x] = __float_as_uint(t);
}
int main() {
  uint32_t* o; cudaMalloc(&o, 4096);
  k_i2fp<<<148, 128>>>(o, 1); k_prmt<<<148, 128>>>(o, 1); k_vimnmx<<<148, 128>>>(o, 1); k_iadd<<<148, 128>>>(o, 1);
  k_ffma2<<<148, 128>>>(o, 1);
  cudaDeviceSynchronize(); printf("ok\n"); return 0;
}
