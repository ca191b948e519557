// Cycles per k of the NT reduction's inner loop (one warp, paired chain over
// two rows, operands resident in shared memory), three code shapes.
#include <cstdio>
typedef unsigned long long u64;
__constant__ u64 c_nz = 0x8000000080000000ull;
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c_nz)); return r; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
constexpr int BK = 64, SB = BK + 4, TILES = 160;
__global__ void kernel(float* out, u64* cyc, int variant) {
  __shared__ __align__(16) float As[BK * 2];
  __shared__ __align__(16) float Bs[32 * SB];
  const int lane = threadIdx.x;
  for (int i = lane; i < BK * 2; i += 32) As[i] = 1.0f + i * 1e-3f;
  for (int i = lane; i < 32 * SB; i += 32) Bs[i] = 0.5f + i * 1e-4f;
  __syncwarp();
  u64 acc = 0;
  const float* bs = Bs + lane * SB;
  u64 t0 = clock64();
  for (int tile = 0; tile < TILES; ++tile) {
    if (variant == 0) {  // LDS.128 per 4 k of B, per 2 k of A, product then add
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        const float4 b = *reinterpret_cast<const float4*>(bs + kk);
        const float4 a01 = *reinterpret_cast<const float4*>(As + kk * 2);
        const float4 a23 = *reinterpret_cast<const float4*>(As + kk * 2 + 4);
        acc = add2(acc, mul2(pk(a01.x, a01.y), pk(b.x, b.x)));
        acc = add2(acc, mul2(pk(a01.z, a01.w), pk(b.y, b.y)));
        acc = add2(acc, mul2(pk(a23.x, a23.y), pk(b.z, b.z)));
        acc = add2(acc, mul2(pk(a23.z, a23.w), pk(b.w, b.w)));
      }
    } else if (variant == 1) {  // 16-k groups: loads, then products, then adds
#pragma unroll
      for (int g = 0; g < BK; g += 16) {
        float4 b[4], a[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = *reinterpret_cast<const float4*>(bs + g + 4 * i);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = *reinterpret_cast<const float4*>(As + g * 2 + 4 * i);
        u64 p[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          p[4 * i + 0] = mul2(pk(a[2 * i].x, a[2 * i].y), pk(b[i].x, b[i].x));
          p[4 * i + 1] = mul2(pk(a[2 * i].z, a[2 * i].w), pk(b[i].y, b[i].y));
          p[4 * i + 2] = mul2(pk(a[2 * i + 1].x, a[2 * i + 1].y), pk(b[i].z, b[i].z));
          p[4 * i + 3] = mul2(pk(a[2 * i + 1].z, a[2 * i + 1].w), pk(b[i].w, b[i].w));
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) acc = add2(acc, p[i]);
      }
    } else {  // scalar chain (one row) for reference
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        const float4 b = *reinterpret_cast<const float4*>(bs + kk);
        const float4 a = *reinterpret_cast<const float4*>(As + kk);
        float x = __uint_as_float(unsigned(acc));
        x = __fadd_rn(x, __fmul_rn(a.x, b.x)); x = __fadd_rn(x, __fmul_rn(a.y, b.y));
        x = __fadd_rn(x, __fmul_rn(a.z, b.z)); x = __fadd_rn(x, __fmul_rn(a.w, b.w));
        acc = (acc & 0xffffffff00000000ull) | __float_as_uint(x);
      }
    }
  }
  u64 t1 = clock64();
  out[lane] = __uint_as_float(unsigned(acc)) + __uint_as_float(unsigned(acc >> 32));
  if (lane == 0) cyc[variant] = t1 - t0;
}
int main() {
  float* out; u64* cyc; cudaMalloc(&out, 128); cudaMalloc(&cyc, 64);
  for (int rep = 0; rep < 2; ++rep) {
    for (int v = 0; v < 3; ++v) kernel<<<1, 32>>>(out, cyc, v);
    u64 h[3]; cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
    printf("cycles per k: loop %.2f  grouped %.2f  scalar %.2f\n", h[0] / double(TILES * BK),
           h[1] / double(TILES * BK), h[2] / double(TILES * BK));
  }
  return 0;
}
