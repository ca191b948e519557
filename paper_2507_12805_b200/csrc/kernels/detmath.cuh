// Device replicas of the reference's fixed-operation numerics
// (core/src/detmath.cpp:14-103). Every operation is an explicit
// round-to-nearest intrinsic so ptxas can neither contract a mul+add into an
// FMA nor reassociate; results are bit-identical to the -ffp-contract=off
// host build. The library is also compiled with -fmad=false as a backstop.
#pragma once
#include <cstdint>

namespace pmklc_b200 {

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }
// acc + a*b with the product rounded first (no FMA)
__device__ __forceinline__ float mac(float acc, float a, float b) { return __fadd_rn(acc, __fmul_rn(a, b)); }

// Paired FP32 (Blackwell FMUL2/FADD2-class issue): two independent lanes of
// the same exact operations in one instruction, each IEEE round-to-nearest,
// bit-identical to the scalar pair (checked on B200: tools/x2/x2bench.cu).
// ptxas contracts a single-use mul.rn.f32x2 into the following add.rn.f32x2
// (even with -fmad=false), so the product is formed as fma.rn.f32x2(a, b, z)
// with z = (-0, -0) read from __constant__ memory: a*b + (-0) is exactly
// round(a*b) for every input, and an fma followed by an add cannot be fused.
typedef unsigned long long f2_t;
static __constant__ f2_t c_negzero2 = 0x8000000080000000ull;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f2_t f2_bcast(float x) { return f2_pack(x, x); }
__device__ __forceinline__ float f2_lo(f2_t v) { return __uint_as_float(uint32_t(v)); }
__device__ __forceinline__ float f2_hi(f2_t v) { return __uint_as_float(uint32_t(v >> 32)); }
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c_negzero2));
  return r;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// (acc.lo + a.lo*b.lo, acc.hi + a.hi*b.hi), products rounded first
__device__ __forceinline__ f2_t f2_mac(f2_t acc, f2_t a, f2_t b) { return f2_add(acc, f2_mul(a, b)); }

// det_exp: range reduction + degree-6 Taylor (detmath.cpp:24-43)
__device__ __forceinline__ float det_exp(float x) {
  if (x > 87.0f) x = 87.0f;
  if (x < -87.0f) x = -87.0f;
  const float t = fmul(x, 1.4426950408889634f);
  const float nf = floorf(fadd(t, 0.5f));
  const int n = int(nf);
  float f = fsub(x, fmul(nf, 0.693359375f));
  f = fsub(f, fmul(nf, -2.12194440e-4f));
  float p = 1.0f / 720.0f;
  p = fadd(fmul(p, f), 1.0f / 120.0f);
  p = fadd(fmul(p, f), 1.0f / 24.0f);
  p = fadd(fmul(p, f), 1.0f / 6.0f);
  p = fadd(fmul(p, f), 0.5f);
  p = fadd(fmul(p, f), 1.0f);
  p = fadd(fmul(p, f), 1.0f);
  return fmul(p, __uint_as_float(uint32_t(n + 127) << 23));
}

// det_log: mantissa/exponent split + atanh series (detmath.cpp:45-68)
__device__ __forceinline__ float det_log(float x) {
  if (x < 1.17549435e-38f) x = 1.17549435e-38f;
  uint32_t bits = __float_as_uint(x);
  int e = int(bits >> 23) - 127;
  float m = __uint_as_float((bits & 0x007fffffu) | 0x3f800000u);
  if (m > 1.4142135f) {
    m = fmul(m, 0.5f);
    e += 1;
  }
  const float u = fdiv(fsub(m, 1.0f), fadd(m, 1.0f));
  const float u2 = fmul(u, u);
  float p = 1.0f / 11.0f;
  p = fadd(fmul(p, u2), 1.0f / 9.0f);
  p = fadd(fmul(p, u2), 1.0f / 7.0f);
  p = fadd(fmul(p, u2), 1.0f / 5.0f);
  p = fadd(fmul(p, u2), 1.0f / 3.0f);
  p = fadd(fmul(p, u2), 1.0f);
  return fadd(fmul(float(e), 0.69314718f), fmul(fmul(2.0f, u), p));
}

// det_sigmoid (detmath.cpp:70-76)
__device__ __forceinline__ float det_sigmoid(float x) {
  if (x >= 0.0f) return fdiv(1.0f, fadd(1.0f, det_exp(-x)));
  const float e = det_exp(x);
  return fdiv(e, fadd(1.0f, e));
}

// det_tanh (detmath.cpp:78-83)
__device__ __forceinline__ float det_tanh(float x) {
  float a = x < 0.0f ? -x : x;
  if (a > 9.0f) a = 9.0f;
  const float t = fsub(1.0f, fdiv(2.0f, fadd(det_exp(fmul(2.0f, a)), 1.0f)));
  return x < 0.0f ? -t : t;
}

}  // namespace pmklc_b200
