// Microbenchmark + exactness check: paired FP32 (FMUL2/FADD2 via f32x2 PTX) vs
// scalar FMUL/FADD for the non-contracted multiply-add chains of EXACT mode.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <random>
typedef unsigned long long u64;
__device__ __forceinline__ u64 mulz2(u64 a, u64 b, u64 z) {
  u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(z)); return r; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 pack(float lo, float hi) {
  u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }

constexpr int CH = 8, IT = 4096;
__global__ void k_scalar(float* out, float s) {
  float a[CH * 2];
  for (int i = 0; i < CH * 2; ++i) a[i] = threadIdx.x * 1e-3f + i;
  const float w = s * 0.999f;
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH * 2; ++i) a[i] = __fadd_rn(a[i], __fmul_rn(a[i], w));
  }
  float t = 0; for (int i = 0; i < CH * 2; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_pair(float* out, float s, u64 z) {
  u64 a[CH];
  for (int i = 0; i < CH; ++i) a[i] = pack(threadIdx.x * 1e-3f + 2 * i, threadIdx.x * 1e-3f + 2 * i + 1);
  const float w1 = s * 0.999f;
  const u64 w = pack(w1, w1);
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = add2(a[i], mulz2(a[i], w, z));
  }
  float t = 0;
  for (int i = 0; i < CH; ++i) { float2 f; memcpy(&f, &a[i], 8); t += f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
// exactness: chains acc = acc + x*y over random data, scalar vs paired
__global__ void k_exact(const float* x, const float* y, float* o1, float* o2, int n, int K, u64 z) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * i + 1 >= n) return;
  float s0 = 0, s1 = 0;
  u64 acc = 0;
  for (int k = 0; k < K; ++k) {
    float a0 = x[(2 * i) * K + k], a1 = x[(2 * i + 1) * K + k], b = y[k];
    s0 = __fadd_rn(s0, __fmul_rn(a0, b));
    s1 = __fadd_rn(s1, __fmul_rn(a1, b));
    acc = add2(acc, mulz2(pack(a0, a1), pack(b, b), z));
  }
  o1[2 * i] = s0; o1[2 * i + 1] = s1;
  float2 f; memcpy(&f, &acc, 8);
  o2[2 * i] = f.x; o2[2 * i + 1] = f.y;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const u64 z = 0x8000000080000000ull;
  for (int rep = 0; rep < 2; ++rep) {
    for (int blocks : {148 * 4, 148 * 8}) {
      float ms;
      cudaEventRecord(e0); k_scalar<<<blocks, 256>>>(out, 1.0f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = double(blocks) * 256 * IT * CH * 2 * 2;  // flops (mul+add) per lane-chain
      printf("scalar blocks=%d %.3f ms %.2f TFLOP/s\n", blocks, ms, ops / ms / 1e9);
      cudaEventRecord(e0); k_pair<<<blocks, 256>>>(out, 1.0f, z); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("pair   blocks=%d %.3f ms %.2f TFLOP/s\n", blocks, ms, ops / ms / 1e9);
    }
  }
  const int n = 1 << 16, K = 257;
  std::vector<float> hx(size_t(n) * K), hy(K);
  std::mt19937 g(7); std::normal_distribution<float> d(0.f, 3.f);
  for (auto& v : hx) v = d(g);
  for (auto& v : hy) v = d(g);
  hx[5] = 0.f; hx[6] = -0.f; hx[7] = 1e-41f; hx[8] = -1e-42f;  // zeros, subnormals
  float *dx, *dy, *o1, *o2;
  cudaMalloc(&dx, hx.size() * 4); cudaMalloc(&dy, K * 4); cudaMalloc(&o1, n * 4); cudaMalloc(&o2, n * 4);
  cudaMemcpy(dx, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, hy.data(), K * 4, cudaMemcpyHostToDevice);
  k_exact<<<n / 2 / 256, 256>>>(dx, dy, o1, o2, n, K, z);
  std::vector<uint32_t> a(n), b(n);
  cudaMemcpy(a.data(), o1, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), o2, n * 4, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < n; ++i) bad += a[i] != b[i];
  printf("exactness: %d of %d differ; err=%s\n", bad, n, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
