// Dependent-issue latency of scalar FADD/FMUL vs paired FADD2/FFMA2 (one
// thread, long dependent chains, clock64), and the exact-MAC chain patterns.
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ u64 mulz2(u64 a, u64 b, u64 z) {
  u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(z)); return r; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
constexpr int N = 4096;
__global__ void k(float* out, u64* cyc, float x, u64 z, const float* v) {
  u64 t0, t1;
  float a = x;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) a = __fadd_rn(a, x);
  t1 = clock64(); cyc[0] = t1 - t0; out[0] = a;
  u64 p = (u64)__float_as_uint(x) | ((u64)__float_as_uint(x) << 32), q = p;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) q = add2(q, p);
  t1 = clock64(); cyc[1] = t1 - t0; out[1] = __uint_as_float(unsigned(q));
  q = p;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) q = mulz2(q, p, z);
  t1 = clock64(); cyc[2] = t1 - t0; out[2] = __uint_as_float(unsigned(q));
  // exact MAC chain, scalar: acc = acc + v[i]*w  (products independent)
  float acc = 0.f, w = x;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) acc = __fadd_rn(acc, __fmul_rn(v[i & 63], w));
  t1 = clock64(); cyc[3] = t1 - t0; out[3] = acc;
  // exact MAC chain, paired
  u64 acc2 = 0, w2 = p;
  t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < N; ++i) {
    u64 vv = (u64)__float_as_uint(v[i & 63]) | ((u64)__float_as_uint(v[(i + 1) & 63]) << 32);
    acc2 = add2(acc2, mulz2(vv, w2, z));
  }
  t1 = clock64(); cyc[4] = t1 - t0; out[4] = __uint_as_float(unsigned(acc2));
}
int main() {
  float* out; u64* cyc; float* v;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 64); cudaMalloc(&v, 256);
  cudaMemset(v, 0, 256);
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 1>>>(out, cyc, 1.0001f, 0x8000000080000000ull, v);
    u64 h[5]; cudaMemcpy(h, cyc, 40, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: FADD %.2f  FADD2 %.2f  FFMA2 %.2f  MAC scalar %.2f  MAC paired %.2f\n",
           h[0] / double(N), h[1] / double(N), h[2] / double(N), h[3] / double(N), h[4] / double(N));
  }
  return 0;
}
