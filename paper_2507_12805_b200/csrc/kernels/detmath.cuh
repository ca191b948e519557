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

// ---- paired forms: two independent lanes through exactly the scalar
// functions' operation sequences (arithmetic on f32x2; the clamps, floor,
// int conversion, exponent assembly, sign tests and the correctly rounded
// divisions per lane), so each half is bit-identical to the scalar result.
__device__ __forceinline__ f2_t f2_sub(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ f2_t det_exp2(f2_t x2) {
  float xl = f2_lo(x2), xh = f2_hi(x2);
  if (xl > 87.0f) xl = 87.0f;
  if (xl < -87.0f) xl = -87.0f;
  if (xh > 87.0f) xh = 87.0f;
  if (xh < -87.0f) xh = -87.0f;
  const f2_t x = f2_pack(xl, xh);
  const f2_t t = f2_add(f2_mul(x, f2_bcast(1.4426950408889634f)), f2_bcast(0.5f));
  const float nfl = floorf(f2_lo(t)), nfh = floorf(f2_hi(t));
  const int nl = int(nfl), nh = int(nfh);
  const f2_t nf = f2_pack(nfl, nfh);
  f2_t f = f2_sub(x, f2_mul(nf, f2_bcast(0.693359375f)));
  f = f2_sub(f, f2_mul(nf, f2_bcast(-2.12194440e-4f)));
  f2_t p = f2_bcast(1.0f / 720.0f);
  p = f2_add(f2_mul(p, f), f2_bcast(1.0f / 120.0f));
  p = f2_add(f2_mul(p, f), f2_bcast(1.0f / 24.0f));
  p = f2_add(f2_mul(p, f), f2_bcast(1.0f / 6.0f));
  p = f2_add(f2_mul(p, f), f2_bcast(0.5f));
  p = f2_add(f2_mul(p, f), f2_bcast(1.0f));
  p = f2_add(f2_mul(p, f), f2_bcast(1.0f));
  return f2_mul(p, f2_pack(__uint_as_float(uint32_t(nl + 127) << 23),
                           __uint_as_float(uint32_t(nh + 127) << 23)));
}

__device__ __forceinline__ f2_t det_sigmoid2(f2_t x) {
  const float xl = f2_lo(x), xh = f2_hi(x);
  const bool pl = xl >= 0.0f, ph = xh >= 0.0f;
  const f2_t e = det_exp2(f2_pack(pl ? -xl : xl, ph ? -xh : xh));
  const f2_t den = f2_add(f2_bcast(1.0f), e);
  return f2_pack(fdiv(pl ? 1.0f : f2_lo(e), f2_lo(den)), fdiv(ph ? 1.0f : f2_hi(e), f2_hi(den)));
}

__device__ __forceinline__ f2_t det_tanh2(f2_t x) {
  const float xl = f2_lo(x), xh = f2_hi(x);
  float al = xl < 0.0f ? -xl : xl, ah = xh < 0.0f ? -xh : xh;
  if (al > 9.0f) al = 9.0f;
  if (ah > 9.0f) ah = 9.0f;
  const f2_t den = f2_add(det_exp2(f2_mul(f2_bcast(2.0f), f2_pack(al, ah))), f2_bcast(1.0f));
  const f2_t t = f2_sub(f2_bcast(1.0f), f2_pack(fdiv(2.0f, f2_lo(den)), fdiv(2.0f, f2_hi(den))));
  const float tl = f2_lo(t), th = f2_hi(t);
  return f2_pack(xl < 0.0f ? -tl : tl, xh < 0.0f ? -th : th);
}

}  // namespace pmklc_b200
