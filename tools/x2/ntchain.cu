// Cycles per iteration of the streamed NT consumer's paired exact chain
// (acc += (a.x, a.y) * b, a: 8-byte smem pair, b: per-lane smem float, stride
// 128 B), one warp per SM sub-partition (4 warps, 1 block), three schedules:
//   v0 plain loop (#pragma unroll 8), v1 loads batched 8 ahead, v2 the
//   volatile three-stage software pipeline of sprm_kernels.cu (nt_chain_pair).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false ntchain.cu -o ntchain
#include <cstdio>
#include <cstdint>
typedef unsigned long long f2_t;
__constant__ f2_t c_negzero2 = 0x8000000080000000ull;
__device__ __forceinline__ f2_t pk(float lo, float hi) {
  f2_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c_negzero2)); return r; }
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void lds_pair(f2_t& x, float& y, uint32_t a, uint32_t b) {
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(x) : "r"(a));
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(y) : "r"(b));
}
__device__ __forceinline__ f2_t prod_v(f2_t x, float y) {
  f2_t out; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(out) : "l"(x), "l"(pk(y, y)), "l"(c_negzero2));
  return out; }
__device__ __forceinline__ void add_v(f2_t& acc, f2_t p) { asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(p)); }
template <int kU>
__device__ __forceinline__ void stage(f2_t& acc, f2_t (&P)[kU], f2_t (&LN)[kU], float (&LNb)[kU], f2_t (&LL)[kU],
                                      float (&LLb)[kU], bool m1, bool m2, uint32_t a2, uint32_t b2, uint32_t ast) {
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    add_v(acc, P[u]);
    if (m1) P[u] = prod_v(LN[u], LNb[u]);
    if (m2) lds_pair(LL[u], LLb[u], a2 + u * ast, b2 + u * 128u);
  }
}
__device__ __forceinline__ f2_t chain_v2(f2_t acc, uint32_t a, uint32_t ast, uint32_t b, int R) {
  constexpr int kU = 8;
  const int nb = R / kU;
  f2_t L0[kU], L1[kU], P[kU];
  float B0[kU], B1[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) lds_pair(L0[u], B0[u], a + u * ast, b + u * 128u);
#pragma unroll
  for (int u = 0; u < kU; ++u) lds_pair(L1[u], B1[u], a + (kU + u) * ast, b + (kU + u) * 128u);
#pragma unroll
  for (int u = 0; u < kU; ++u) P[u] = prod_v(L0[u], B0[u]);
  int k = 0;
  for (; k + 2 <= nb; k += 2) {
    stage<kU>(acc, P, L1, B1, L0, B0, k + 1 < nb, k + 2 < nb, a + (k + 2) * kU * ast, b + (k + 2) * kU * 128u, ast);
    stage<kU>(acc, P, L0, B0, L1, B1, k + 2 < nb, k + 3 < nb, a + (k + 3) * kU * ast, b + (k + 3) * kU * 128u, ast);
  }
  return acc;
}
constexpr int R = 160, H = 32, STEPS = 64;
template <int V>
__global__ void __launch_bounds__(128, 1) kbench(float* out, unsigned long long* cyc) {
  __shared__ __align__(16) float B[R * H];
  __shared__ __align__(16) float A[R * H];
  for (int i = threadIdx.x; i < R * H; i += blockDim.x) { B[i] = 1.0f + i * 1e-7f; A[i] = 0.5f - i * 1e-7f; }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float* bs = B + lane;
  const float2* ap = reinterpret_cast<const float2*>(A + 2 * w);
  f2_t acc = 0;
  const unsigned long long t0 = clock64();
  for (int s = 0; s < STEPS; ++s) {
    if (V == 0) {
#pragma unroll 8
      for (int r = 0; r < R; ++r) { const float2 a = ap[r * (H / 2)]; acc = add2(acc, mul2(pk(a.x, a.y), pk(bs[r * H], bs[r * H]))); }
    } else if (V == 1) {
      for (int r = 0; r < R; r += 8) {
        float2 av[8]; float bv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { av[u] = ap[(r + u) * (H / 2)]; bv[u] = bs[(r + u) * H]; }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = add2(acc, mul2(pk(av[u].x, av[u].y), pk(bv[u], bv[u])));
      }
    } else if (V == 2) {
      acc = chain_v2(acc, sa(A + 2 * w), H * 4, sa(bs), R);
    } else {  // v3: two scalar exact chains (FMUL + FADD), batched loads
      float a0 = __uint_as_float(unsigned(acc)), a1 = __uint_as_float(unsigned(acc >> 32));
      for (int r = 0; r < R; r += 8) {
        float2 av[8]; float bv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { av[u] = ap[(r + u) * (H / 2)]; bv[u] = bs[(r + u) * H]; }
#pragma unroll
        for (int u = 0; u < 8; ++u) { a0 = __fadd_rn(a0, __fmul_rn(av[u].x, bv[u])); a1 = __fadd_rn(a1, __fmul_rn(av[u].y, bv[u])); }
      }
      acc = (f2_t)__float_as_uint(a0) | ((f2_t)__float_as_uint(a1) << 32);
    }
    __syncwarp();
  }
  const unsigned long long t1 = clock64();
  if (lane == 0) cyc[w] = t1 - t0;
  out[threadIdx.x] = __uint_as_float(unsigned(acc));
}
// v4: feature-major operands (the layout the NT reduction reads): lane n's
// B row [k] contiguous (row stride K+4: conflict-free LDS.128 along k), the two
// A rows broadcast along k; one paired chain per lane; `warps` warps per block
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) kfm(float* out, unsigned long long* cyc) {
  constexpr int K = 256, KS = K + 4;
  __shared__ __align__(16) float B[32 * KS];
  __shared__ __align__(16) float A[2 * K];
  for (int i = threadIdx.x; i < 32 * KS; i += blockDim.x) B[i] = 1.0f + i * 1e-7f;
  for (int i = threadIdx.x; i < 2 * K; i += blockDim.x) A[i] = 0.5f - i * 1e-7f;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float4* b4 = reinterpret_cast<const float4*>(B + lane * KS);
  const float4* a0 = reinterpret_cast<const float4*>(A);
  const float4* a1 = reinterpret_cast<const float4*>(A + K);
  f2_t acc = 0;
  const unsigned long long t0 = clock64();
  for (int rep = 0; rep < 40; ++rep) {
#pragma unroll 4
    for (int k4 = 0; k4 < K / 4; ++k4) {
      const float4 bb = b4[k4], x0 = a0[k4], x1 = a1[k4];
      acc = add2(acc, mul2(pk(x0.x, x1.x), pk(bb.x, bb.x)));
      acc = add2(acc, mul2(pk(x0.y, x1.y), pk(bb.y, bb.y)));
      acc = add2(acc, mul2(pk(x0.z, x1.z), pk(bb.z, bb.z)));
      acc = add2(acc, mul2(pk(x0.w, x1.w), pk(bb.w, bb.w)));
    }
  }
  const unsigned long long t1 = clock64();
  if (lane == 0) cyc[w] = t1 - t0;
  out[threadIdx.x] = __uint_as_float(unsigned(acc));
}

// v5: the same feature-major operands, two scalar exact chains per lane
// (FMUL + FADD each), no packing
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) kfm_scalar(float* out, unsigned long long* cyc) {
  constexpr int K = 256, KS = K + 4;
  __shared__ __align__(16) float B[32 * KS];
  __shared__ __align__(16) float A[2 * K];
  for (int i = threadIdx.x; i < 32 * KS; i += blockDim.x) B[i] = 1.0f + i * 1e-7f;
  for (int i = threadIdx.x; i < 2 * K; i += blockDim.x) A[i] = 0.5f - i * 1e-7f;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float4* b4 = reinterpret_cast<const float4*>(B + lane * KS);
  const float4* a0 = reinterpret_cast<const float4*>(A);
  const float4* a1 = reinterpret_cast<const float4*>(A + K);
  float c0 = 0.f, c1 = 0.f;
  const unsigned long long t0 = clock64();
  for (int rep = 0; rep < 40; ++rep) {
#pragma unroll 4
    for (int k4 = 0; k4 < K / 4; ++k4) {
      const float4 bb = b4[k4], x0 = a0[k4], x1 = a1[k4];
      c0 = __fadd_rn(c0, __fmul_rn(x0.x, bb.x)); c1 = __fadd_rn(c1, __fmul_rn(x1.x, bb.x));
      c0 = __fadd_rn(c0, __fmul_rn(x0.y, bb.y)); c1 = __fadd_rn(c1, __fmul_rn(x1.y, bb.y));
      c0 = __fadd_rn(c0, __fmul_rn(x0.z, bb.z)); c1 = __fadd_rn(c1, __fmul_rn(x1.z, bb.z));
      c0 = __fadd_rn(c0, __fmul_rn(x0.w, bb.w)); c1 = __fadd_rn(c1, __fmul_rn(x1.w, bb.w));
    }
  }
  const unsigned long long t1 = clock64();
  if (lane == 0) cyc[w] = t1 - t0;
  out[threadIdx.x] = c0 + c1;
}

// v6: paired chain with the products of a 16-k block formed first (16
// FFMA2 into registers), then the block's 16 dependent FADD2s
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) kfm_two_phase(float* out, unsigned long long* cyc) {
  constexpr int K = 256, KS = K + 4;
  __shared__ __align__(16) float B[32 * KS];
  __shared__ __align__(16) float A[2 * K];
  for (int i = threadIdx.x; i < 32 * KS; i += blockDim.x) B[i] = 1.0f + i * 1e-7f;
  for (int i = threadIdx.x; i < 2 * K; i += blockDim.x) A[i] = 0.5f - i * 1e-7f;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float4* b4 = reinterpret_cast<const float4*>(B + lane * KS);
  const float4* a0 = reinterpret_cast<const float4*>(A);
  const float4* a1 = reinterpret_cast<const float4*>(A + K);
  f2_t acc = 0;
  const unsigned long long t0 = clock64();
  for (int rep = 0; rep < 40; ++rep) {
    for (int kb = 0; kb < K / 16; ++kb) {
      f2_t P[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 bb = b4[kb * 4 + q], x0 = a0[kb * 4 + q], x1 = a1[kb * 4 + q];
        P[4 * q + 0] = mul2(pk(x0.x, x1.x), pk(bb.x, bb.x));
        P[4 * q + 1] = mul2(pk(x0.y, x1.y), pk(bb.y, bb.y));
        P[4 * q + 2] = mul2(pk(x0.z, x1.z), pk(bb.z, bb.z));
        P[4 * q + 3] = mul2(pk(x0.w, x1.w), pk(bb.w, bb.w));
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) acc = add2(acc, P[u]);
    }
  }
  const unsigned long long t1 = clock64();
  if (lane == 0) cyc[w] = t1 - t0;
  out[threadIdx.x] = __uint_as_float(unsigned(acc));
}

// v7: v6 with the two A rows interleaved in shared memory, (a0[k], a1[k])
// adjacent, so an LDS.128 yields two k's ready-made register pairs
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) kfm_pairs(float* out, unsigned long long* cyc) {
  constexpr int K = 256, KS = K + 4;
  __shared__ __align__(16) float B[32 * KS];
  __shared__ __align__(16) float A[2 * K];  // [k][2]
  for (int i = threadIdx.x; i < 32 * KS; i += blockDim.x) B[i] = 1.0f + i * 1e-7f;
  for (int i = threadIdx.x; i < 2 * K; i += blockDim.x) A[i] = 0.5f - i * 1e-7f;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float4* b4 = reinterpret_cast<const float4*>(B + lane * KS);
  const ulonglong2* ap = reinterpret_cast<const ulonglong2*>(A);  // two (a0,a1) pairs
  f2_t acc = 0;
  const unsigned long long t0 = clock64();
  for (int rep = 0; rep < 40; ++rep) {
    for (int kb = 0; kb < K / 16; ++kb) {
      f2_t P[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 bb = b4[kb * 4 + q];
        const ulonglong2 x01 = ap[kb * 8 + 2 * q], x23 = ap[kb * 8 + 2 * q + 1];
        P[4 * q + 0] = mul2(x01.x, pk(bb.x, bb.x));
        P[4 * q + 1] = mul2(x01.y, pk(bb.y, bb.y));
        P[4 * q + 2] = mul2(x23.x, pk(bb.z, bb.z));
        P[4 * q + 3] = mul2(x23.y, pk(bb.w, bb.w));
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) acc = add2(acc, P[u]);
    }
  }
  const unsigned long long t1 = clock64();
  if (lane == 0) cyc[w] = t1 - t0;
  out[threadIdx.x] = __uint_as_float(unsigned(acc));
}

int main() {
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  for (int rep = 0; rep < 2; ++rep) {
    unsigned long long h[4][4];
    kbench<0><<<1, 128>>>(out, cyc); cudaMemcpy(h[0], cyc, 32, cudaMemcpyDeviceToHost);
    kbench<1><<<1, 128>>>(out, cyc); cudaMemcpy(h[1], cyc, 32, cudaMemcpyDeviceToHost);
    kbench<2><<<1, 128>>>(out, cyc); cudaMemcpy(h[2], cyc, 32, cudaMemcpyDeviceToHost);
    kbench<3><<<1, 128>>>(out, cyc); cudaMemcpy(h[3], cyc, 32, cudaMemcpyDeviceToHost);
    for (int v = 0; v < 4; ++v)
      printf("v%d cycles/iteration: %.2f (warp 0), %.2f (warp 3)\n", v, h[v][0] / double(R * STEPS), h[v][3] / double(R * STEPS));
  }
  unsigned long long h[8];
  kfm<1><<<1, 32>>>(out, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("v4 feature-major, 1 warp/SM: %.2f cycles/k\n", h[0] / (40.0 * 256));
  kfm<4><<<1, 128>>>(out, cyc); cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
  printf("v4 feature-major, 4 warps/SM: %.2f cycles/k\n", h[0] / (40.0 * 256));
  kfm<8><<<1, 256>>>(out, cyc); cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
  printf("v4 feature-major, 8 warps/SM: %.2f cycles/k\n", h[0] / (40.0 * 256));
  kfm_scalar<1><<<1, 32>>>(out, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("v5 feature-major scalar x2, 1 warp/SM: %.2f cycles/k\n", h[0] / (40.0 * 256));
  kfm_scalar<4><<<1, 128>>>(out, cyc); cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
  printf("v5 feature-major scalar x2, 4 warps/SM: %.2f cycles/k\n", h[0] / (40.0 * 256));
  kfm_two_phase<1><<<1, 32>>>(out, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("v6 paired two-phase, 1 warp/SM: %.2f cycles/k\n", h[0] / (40.0 * 256));
  kfm_two_phase<4><<<1, 128>>>(out, cyc); cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
  printf("v6 paired two-phase, 4 warps/SM: %.2f cycles/k\n", h[0] / (40.0 * 256));
  kfm_pairs<1><<<1, 32>>>(out, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("v7 paired, interleaved A, 1 warp/SM: %.2f cycles/k\n", h[0] / (40.0 * 256));
  kfm_pairs<4><<<1, 128>>>(out, cyc); cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
  printf("v7 paired, interleaved A, 4 warps/SM: %.2f cycles/k\n", h[0] / (40.0 * 256));
  return 0;
}
