// Dynamic-model (AttentionModel, core/src/models.cpp:108-149) forward/backward
// and Adam on sm_100a, batched over every active data block.
//
// EXACT arithmetic contract: every output element keeps
// the reference's accumulation order (ascending reduction index, starting from
// bias / zero / the existing gradient), products are rounded before the add
// (no FMA: __fmul_rn + __fadd_rn), and parallelism is only across independent
// output elements, rows, heads and chunks. This is why the model runs on the
// FP32 SIMT pipe rather than tcgen05: tensor-core accumulation order is
// unspecified, and the decoder must replay the encoder's online training bit
// for bit.
#include <type_traits>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "detmath.cuh"
#include "kernels.hpp"
#include "launch.cuh"

namespace pmklc_b200 {

namespace {

// ------------------------------------------------------------------ GEMM
// Shared-memory tiled SIMT GEMM: 16x16 threads, each owning TM x TN outputs
// laid out with stride 16 (broadcast / conflict-free shared reads). K-tiles of
// depth 32 are staged with cp.async (LDGSTS) into a double buffer so the next
// tile's global loads overlap the current tile's math. K is walked in
// ascending order tile by tile and the partial last tile is bounded exactly
// (no zero padding: 0*x would change signed zeros / NaNs). The tile size is
// picked per launch: big tiles when many chunks fill the chip (fewer shared
// loads per MAC), 16x16 tiles when one chunk must finish fast (more SMs on
// its short dependent chains).
__device__ __forceinline__ void cp_async4(float* smem, const float* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <bool AT, bool BT, int TM, int TN, int BK, int STAGES, int TX, int TY>
__global__ void __launch_bounds__(TX * TY) k_gemm_tiled(GemmP p, const TickDesc* __restrict__ td) {
  pdl_wait();
  constexpr int NT = TX * TY, BM = TY * TM, BN = TX * TN;
  // dynamic shared memory: the ring is [STAGES][BK][BM+4] A then [STAGES][BK][BN+4] B
  // (3+ stages of the 64x64 tile exceed the 48 KB static limit)
  extern __shared__ __align__(16) float g_sm[];
  auto As = reinterpret_cast<float (*)[BK][BM + 4]>(g_sm);
  auto Bs = reinterpret_cast<float (*)[BK][BN + 4]>(g_sm + STAGES * BK * (BM + 4));
  const int np = p.nprob > 1 ? p.nprob : 1;
  const int slot = blockIdx.z / np, prob = blockIdx.z % np;
  if (slot >= td->n_act) return;
  const int c = td->act[slot];
  const float* A = p.A + c * p.a_cs + prob * p.a_ps;
  const float* B = p.B + c * p.b_cs + prob * p.b_ps;
  float* C = p.C + c * p.c_cs + prob * p.c_ps;
  const float* bias = p.bias ? p.bias + c * p.bias_cs + prob * p.bias_ps : nullptr;
  const int Mx = p.M + (p.ones_row ? 1 : 0);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int ntiles = (p.K + BK - 1) / BK;
  // Output column of a thread's j-th accumulator. TN = 8 splits the thread's
  // columns into two groups of 4 interleaved across the block (group g at
  // g*TX*4 + tx*4), so each LDS.128 of a B row covers a contiguous 128 B per
  // 8 lanes (one wavefront); TN <= 4 keeps the thread's columns contiguous.
  auto col = [&](int j) {
    return TN % 4 == 0 ? n0 + (j / 4) * (TX * 4) + tx * 4 + j % 4 : n0 + tx * TN + j;
  };

  // 16-byte copies where the global side runs along the smem row (A^T: m,
  // B: n) and is 16-byte aligned (chunk slots of the parameter array are only
  // 4-byte aligned, so this is decided per block)
  auto al16 = [](const float* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const bool va = AT && BM % 4 == 0 && p.lda % 4 == 0 && al16(A);
  const bool vb = !BT && BN % 4 == 0 && p.ldb % 4 == 0 && al16(B);
  auto load = [&](int tile) {
    if (tile < ntiles) {
      const int stage = tile % STAGES, k0 = tile * BK;
      if (va) {
        for (int idx = threadIdx.x; idx < BM * BK / 4; idx += NT) {
          const int mm = (idx % (BM / 4)) * 4, kk = idx / (BM / 4);
          const int m = m0 + mm, k = k0 + kk;
          if (k >= p.K) continue;
          if (m + 3 < p.M) {
            cp_async16(&As[stage][kk][mm], A + int64_t(k) * p.lda + m);
          } else {
            for (int u = 0; u < 4; ++u) {
              if (m + u < p.M) cp_async4(&As[stage][kk][mm + u], A + int64_t(k) * p.lda + m + u);
              else if (m + u == p.M && p.ones_row) As[stage][kk][mm + u] = 1.0f;
            }
          }
        }
      } else {
        for (int idx = threadIdx.x; idx < BM * BK; idx += NT) {
          int mm, kk;
          if (AT) { mm = idx % BM; kk = idx / BM; }  // global contiguous in m
          else    { kk = idx % BK; mm = idx / BK; }  // global contiguous in k
          const int m = m0 + mm, k = k0 + kk;
          if (k < p.K) {
            if (m < p.M) cp_async4(&As[stage][kk][mm], AT ? A + int64_t(k) * p.lda + m : A + int64_t(m) * p.lda + k);
            else if (m == p.M && p.ones_row) As[stage][kk][mm] = 1.0f;
          }
        }
      }
      if (vb) {
        for (int idx = threadIdx.x; idx < BN * BK / 4; idx += NT) {
          const int nn = (idx % (BN / 4)) * 4, kk = idx / (BN / 4);
          const int n = n0 + nn, k = k0 + kk;
          if (k >= p.K) continue;
          if (n + 3 < p.N) {
            cp_async16(&Bs[stage][kk][nn], B + int64_t(k) * p.ldb + n);
          } else {
            for (int u = 0; u < 4; ++u)
              if (n + u < p.N) cp_async4(&Bs[stage][kk][nn + u], B + int64_t(k) * p.ldb + n + u);
          }
        }
      } else {
        for (int idx = threadIdx.x; idx < BN * BK; idx += NT) {
          int nn, kk;
          if (BT) { kk = idx % BK; nn = idx / BK; }
          else    { nn = idx % BN; kk = idx / BN; }
          const int n = n0 + nn, k = k0 + kk;
          if (k < p.K && n < p.N)
            cp_async4(&Bs[stage][kk][nn], BT ? B + int64_t(n) * p.ldb + k : B + int64_t(k) * p.ldb + n);
        }
      }
    }
    cp_async_commit();  // one group per tile slot, possibly empty
  };

  // Accumulators: column pairs (j, j+1) run as one paired chain when TN is even
  // (same per-element operations, half the issue slots).
  constexpr bool kPair = TN % 2 == 0;
  constexpr int TNP = kPair ? TN / 2 : 1;
  float acc[TM][TN];
  f2_t acc2[TM][TNP];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int m = m0 + ty * TM + i, n = col(j);
      float v = 0.0f;
      if (m < Mx && n < p.N) {
        if (p.init == 1) v = bias[n];
        else if (p.init == 2) v = C[int64_t(m) * p.ldc + n];
      }
      acc[i][j] = v;
    }
  if constexpr (kPair) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TNP; ++j) acc2[i][j] = f2_pack(acc[i][2 * j], acc[i][2 * j + 1]);
  }

  const bool relu = p.relu_a != 0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) load(s);
  for (int tile = 0; tile < ntiles; ++tile) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    load(tile + STAGES - 1);  // refills the stage consumed in the previous iteration
    const int stage = tile % STAGES;
    const int kmax = min(BK, p.K - tile * BK);
    auto body = [&](int kk, auto relu_c) {
      // each thread's TM (TN) operands are contiguous: one vector shared load each
      float a[TM], b[TN];
      const float* ap = &As[stage][kk][ty * TM];
      const float* bp = &Bs[stage][kk][TN % 4 == 0 ? tx * 4 : tx * TN];
      if constexpr (TM == 4) {
        const float4 v = *reinterpret_cast<const float4*>(ap);
        a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
      } else if constexpr (TM == 2) {
        const float2 v = *reinterpret_cast<const float2*>(ap);
        a[0] = v.x; a[1] = v.y;
      } else {
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = ap[i];
      }
      if constexpr (TN % 4 == 0) {
#pragma unroll
        for (int g = 0; g < TN / 4; ++g) {
          const float4 v = *reinterpret_cast<const float4*>(bp + g * TX * 4);
          b[4 * g] = v.x; b[4 * g + 1] = v.y; b[4 * g + 2] = v.z; b[4 * g + 3] = v.w;
        }
      } else if constexpr (TN == 2) {
        const float2 v = *reinterpret_cast<const float2*>(bp);
        b[0] = v.x; b[1] = v.y;
      } else {
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = bp[j];
      }
      if constexpr (decltype(relu_c)::value) {
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = a[i] < 0.0f ? 0.0f : a[i];
      }
      if constexpr (kPair) {
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const f2_t ai = f2_bcast(a[i]);
#pragma unroll
          for (int j = 0; j < TNP; ++j) acc2[i][j] = f2_mac(acc2[i][j], ai, f2_pack(b[2 * j], b[2 * j + 1]));
        }
      } else {
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = mac(acc[i][j], a[i], b[j]);
      }
    };
    auto run = [&](auto relu_c) {
      if (kmax == BK) {
#pragma unroll 8
        for (int kk = 0; kk < BK; ++kk) body(kk, relu_c);
      } else {
        for (int kk = 0; kk < kmax; ++kk) body(kk, relu_c);
      }
    };
    if (relu) run(std::true_type{});
    else run(std::false_type{});
  }
  cp_async_wait<0>();
  if constexpr (kPair) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TNP; ++j) {
        acc[i][2 * j] = f2_lo(acc2[i][j]);
        acc[i][2 * j + 1] = f2_hi(acc2[i][j]);
      }
  }

  if constexpr (TN % 4 == 0) {  // 16-byte stores of each group of 4 columns when possible
    if (!p.mask && p.ldc % 4 == 0 && al16(C) && col(TN - 1) < p.N) {
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int m = m0 + ty * TM + i;
        if (m < Mx) {
#pragma unroll
          for (int g = 0; g < TN / 4; ++g)
            *reinterpret_cast<float4*>(C + int64_t(m) * p.ldc + col(4 * g)) =
                make_float4(acc[i][4 * g], acc[i][4 * g + 1], acc[i][4 * g + 2], acc[i][4 * g + 3]);
        }
      }
      return;
    }
  }
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int m = m0 + ty * TM + i, n = col(j);
      if (m < Mx && n < p.N) {
        float v = acc[i][j];
        if (p.mask && p.mask[c * p.mask_cs + int64_t(m) * p.ldm + n] <= 0.0f) v = 0.0f;
        C[int64_t(m) * p.ldc + n] = v;
      }
    }
}

// The 64x64 tile of the throughput regime: 4x8 outputs per thread (128 threads,
// interleaved column groups) through a 3-deep ring of 32-k tiles. Measured
// against 4x4 x 256 threads with 2-4 stages and BK 16-64 by
// tools/x2/gemm_variants.py: -2.2% model time on a 20 MB SPuM+DM compress,
// identical container (the ring depth and tile shape change no reduction order).
#ifndef PMKLC_G44_STAGES
#define PMKLC_G44_STAGES 3
#endif
#ifndef PMKLC_G44_BK
#define PMKLC_G44_BK 32
#endif
#ifndef PMKLC_G44_WIDE
#define PMKLC_G44_WIDE 1
#endif

template <bool AT, bool BT, int TM, int TN, int BK, int STAGES, int TX = 16, int TY = 16>
void gemm_launch(const GemmP& p, const TickDesc* td, int max_active, cudaStream_t st) {
  const int Mx = p.M + (p.ones_row ? 1 : 0);
  const int np = p.nprob > 1 ? p.nprob : 1;
  dim3 grid((p.N + TX * TN - 1) / (TX * TN), (Mx + TY * TM - 1) / (TY * TM), max_active * np);
  constexpr int smem = STAGES * BK * (TY * TM + 4 + TX * TN + 4) * int(sizeof(float));
  auto* kern = k_gemm_tiled<AT, BT, TM, TN, BK, STAGES, TX, TY>;
  if constexpr (smem > 48 * 1024) ensure_smem(reinterpret_cast<const void*>(kern), smem);
  launch_pdl(kern, dim3(grid), dim3(TX * TY), smem, st, p, td);
}

template <bool AT, bool BT>
void gemm_dispatch(const GemmP& p, const TickDesc* td, int max_active, cudaStream_t st) {
  const int Mx = p.M + (p.ones_row ? 1 : 0);
  auto blocks = [&](int bm, int bn) {
    return int64_t((p.N + bn - 1) / bn) * ((Mx + bm - 1) / bm) * max_active * (p.nprob > 1 ? p.nprob : 1);
  };
  // Largest tile that still gives every SM two blocks (throughput); for a
  // launch too small to fill the chip, one output per thread, and for long
  // reductions over few outputs, one-warp blocks (4x8 outputs) so the
  // dependent chains spread over as many SMs as possible.
  constexpr int64_t kFill = 2 * 148;
  if (blocks(64, 64) >= kFill && p.N >= 48 && Mx >= 48)
#if PMKLC_G44_WIDE
    gemm_launch<AT, BT, 4, 8, PMKLC_G44_BK, PMKLC_G44_STAGES, 8, 16>(p, td, max_active, st);
#else
    gemm_launch<AT, BT, 4, 4, PMKLC_G44_BK, PMKLC_G44_STAGES>(p, td, max_active, st);
#endif
  else if (blocks(64, 16) >= kFill && p.N <= 16 && Mx >= 48)
    gemm_launch<AT, BT, 4, 1, 32, 2>(p, td, max_active, st);
  else if (blocks(64, 32) >= kFill && p.N <= 32 && Mx >= 48)
    gemm_launch<AT, BT, 4, 2, 32, 2>(p, td, max_active, st);
  else if (blocks(32, 32) >= kFill && p.N >= 24 && Mx >= 24)
    gemm_launch<AT, BT, 2, 2, 32, 3>(p, td, max_active, st);
  else if (blocks(16, 16) >= 148 || p.K <= 256)
    gemm_launch<AT, BT, 1, 1, 64, 4>(p, td, max_active, st);
  else
    gemm_launch<AT, BT, 1, 1, 128, 4, 8, 4>(p, td, max_active, st);
}

// ------------------------------------------------------------------ NT reduction


// Block = MR output rows x 64 columns (64*MR threads, one output each).
// K-tiles of 64 are staged by 16-byte cp.async into a 4-deep ring; one staged
// B tile serves all MR rows. MR=1 spreads a single chunk's few outputs over
// the most SMs (latency regime); MR=4 amortizes the B tile when many chunks
// are in flight (throughput regime).
// Long-K "NT" reduction C[m][n] (+)= sum_k A[m][k] * B[n][k] (weight gradients:
// feature-major activations x feature-major output gradients, k = the R*t
// position index in the reference's accumulation order). Every output is one
// sequential chain over k, so parallelism is across outputs only.
//
// Warp-autonomous design: a warp owns a task of RPT rows x 32 columns of one
// problem and streams its own operands through a private 3-stage cp.async ring
// (no block barriers, only __syncwarp). Each lane keeps RPT chains for its
// column; A is staged interleaved [k][row] so one broadcast LDS.128 yields row
// pairs for the paired FP32 chains; B is read once per RPT rows. Row M of a
// problem is the bias row (A == 1, so 1*b == b exactly: the plain sum).
#ifndef PMKLC_NW_WARPS
#define PMKLC_NW_WARPS 2
#endif
constexpr int kNwWarps = PMKLC_NW_WARPS;  // independent warps per NT block (no block barriers)
// ring depth and k-tile of the throughput-regime (8 rows per thread) NT launch
#ifndef PMKLC_NT8_S
#define PMKLC_NT8_S 3
#endif
#ifndef PMKLC_NT8_BK
#define PMKLC_NT8_BK 32
#endif
// padded B row (BK + 4 floats): LDS.128 of 32 rows is conflict-free
__host__ __device__ constexpr int nw_warp_floats(int rpt, int stages, int bk) {
  return stages * (rpt * bk + 32 * (bk + 4));
}

struct NtBatch {
  NtP p[kNtMaxProb];
  int first_task[kNtMaxProb + 1];  // prefix of warp tasks per problem
  int colgroups[kNtMaxProb];
  int n;
};

// In-order building blocks for the latency-bound NT tile: ptxas keeps asm
// volatile statements in program order, so the software pipeline written in
// nt_tile_rpt2 is the one that issues (plain loads get sunk next to their
// uses, which exposes the shared-memory latency on the add chain).
__device__ __forceinline__ float4 lds128_v(const float* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}
__device__ __forceinline__ f2_t f2_mul_v(f2_t a, f2_t b) {
  f2_t r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c_negzero2));
  return r;
}
__device__ __forceinline__ f2_t f2_add_v(f2_t a, f2_t b) {
  f2_t r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// One full tile of the 2-row paired chain: acc += a(k) * b(k), k ascending.
// Groups of 16 k: shared loads two groups ahead, products one group ahead,
// one chain add per k with the independent work issued in its latency gaps.
// as: [BK][2] (row pair per k), bs: this lane's B row.
template <int BK>
__device__ __forceinline__ f2_t nt_tile_rpt2(f2_t acc, const float* as, const float* bs) {
  constexpr int KG = 16, NG = BK / KG, NL = KG / 4 + KG / 2;  // 12 LDS.128 per group
  float4 L[2][NL];  // loaded operands: [0..3] B (4 k each), [4..11] A (2 k each)
  f2_t Pp[2][KG];   // products
  auto ld = [&](int g, int i) -> float4 {
    return i < KG / 4 ? lds128_v(bs + g * KG + 4 * i) : lds128_v(as + g * KG * 2 + 4 * (i - KG / 4));
  };
  auto prod = [&](const float4 (&l)[NL], int k) -> f2_t {
    const float4 b4 = l[k / 4];
    const float b = (k & 3) == 0 ? b4.x : (k & 3) == 1 ? b4.y : (k & 3) == 2 ? b4.z : b4.w;
    const float4 a4 = l[KG / 4 + k / 2];
    const f2_t a = (k & 1) ? f2_pack(a4.z, a4.w) : f2_pack(a4.x, a4.y);
    return f2_mul_v(a, f2_bcast(b));
  };
#pragma unroll
  for (int i = 0; i < NL; ++i) L[0][i] = ld(0, i);
  if (NG > 1) {
#pragma unroll
    for (int i = 0; i < NL; ++i) L[1][i] = ld(1, i);
  }
#pragma unroll
  for (int k = 0; k < KG; ++k) Pp[0][k] = prod(L[0], k);
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const int cb = g & 1, nb = cb ^ 1;
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      acc = f2_add_v(acc, Pp[cb][k]);
      if (g + 1 < NG) Pp[nb][k] = prod(L[nb], k);
      if (g + 2 < NG && k < NL) L[cb][k] = ld(g + 2, k);
    }
  }
  return acc;
}

// Bias row of a ones_row GEMM: C[M][n] = init + sum_k 1*B(k, n), k ascending
// (exactly the GEMM's chain for its ones row: 1*b == b). Thread per column,
// 16 loads in flight per batch.
template <bool BT>
__global__ void __launch_bounds__(128) k_bias_row(GemmP p, const TickDesc* __restrict__ td) {
  pdl_wait();
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= p.N) return;
  const float* B = p.B + c * p.b_cs;
  float* Cr = p.C + c * p.c_cs + int64_t(p.M) * p.ldc;
  float acc = p.init == 1 ? p.bias[c * p.bias_cs + n] : p.init == 2 ? Cr[n] : 0.0f;
  const int64_t ks = BT ? 1 : p.ldb;
  const float* b = B + (BT ? int64_t(n) * p.ldb : n);
  constexpr int kB = 16;
  int k = 0;
  for (; k + kB <= p.K; k += kB) {
    float v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) v[u] = __ldg(b + (k + u) * ks);
#pragma unroll
    for (int u = 0; u < kB; ++u) acc = fadd(acc, v[u]);
  }
  for (; k < p.K; ++k) acc = fadd(acc, __ldg(b + k * ks));
  Cr[n] = acc;
}

// VEC: B rows 16-byte aligned and K a multiple of 4 (host-checked).
// STAGES: ring depth; 3 when the chip is full of warps, 8 when a few warps must
// cover the L2 latency alone.
template <bool VEC, int RPT, int STAGES, int BK>
__global__ void __launch_bounds__(kNwWarps * 32) k_gemm_nt(NtBatch nb, const TickDesc* __restrict__ td) {
  pdl_wait();
  constexpr int kNwStages = STAGES, kNwBK = BK, kNwSB = BK + 4;
  extern __shared__ __align__(128) float sm[];
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = int(blockIdx.x) * kNwWarps + w;
  if (task >= nb.first_task[nb.n]) return;  // warp-uniform; no block barriers below
  int prob = 0;
  while (prob + 1 < nb.n && task >= nb.first_task[prob + 1]) ++prob;
  const NtP& pp = nb.p[prob];
  const int lt = task - nb.first_task[prob];
  const int cg = lt % nb.colgroups[prob], rg = lt / nb.colgroups[prob];
  const int M = pp.M, N = pp.N, K = pp.K;
  const int64_t lda = pp.lda, ldb = pp.ldb, ldc = pp.ldc;
  const int m0 = rg * RPT, n0 = cg * 32, n = n0 + lane;
  const int arows = max(0, min(RPT, M - m0));  // rows with A data; the rest are 1 (bias) or 0
  const int nrows = min(32, N - n0);
  float* As = sm + w * nw_warp_floats(RPT, STAGES, BK);  // [stage][BK][RPT]
  float* Bs = As + kNwStages * RPT * kNwBK;  // [stage][32][SB]
  const float* A = pp.A + c * pp.a_cs + int64_t(m0) * lda;
  const float* B = pp.B + c * pp.b_cs + int64_t(n0) * ldb;
  for (int r = arows; r < RPT; ++r) {
    const float v = m0 + r == M ? 1.0f : 0.0f;
    for (int i = lane; i < kNwStages * kNwBK; i += 32) As[i * RPT + r] = v;
  }
  const int ntiles = (K + kNwBK - 1) / kNwBK;
  // full tiles: lane copies A[r][k0 + lane + 32e] for each row and the 16-byte
  // chunk (lane % CPR) of B rows lane / CPR + RPI*j (CPR = BK/4 chunks per row)
  static_assert(kNwBK == 32 || kNwBK == 64, "tile depth");
  constexpr int CPR = kNwBK / 4, RPI = 32 / CPR, BJ = 32 / RPI;
  const float* bl = B + int64_t(lane / CPR) * ldb + 4 * (lane % CPR);
  const int bsl = (lane / CPR) * kNwSB + 4 * (lane % CPR);
  auto load = [&](int tile) {
    if (tile < ntiles) {
      const int st = tile % kNwStages, k0 = tile * kNwBK, kc = min(kNwBK, K - k0);
      float* as = As + st * kNwBK * RPT;
      float* bs = Bs + st * 32 * kNwSB;
      if (kc == kNwBK) {
#pragma unroll
        for (int r = 0; r < RPT; ++r)
          if (r < arows) {
#pragma unroll
            for (int e = 0; e < kNwBK / 32; ++e)
              cp_async4(as + (lane + 32 * e) * RPT + r, A + int64_t(r) * lda + k0 + lane + 32 * e);
          }
        if (VEC && nrows == 32) {
          const float* src = bl + k0;
#pragma unroll
          for (int j = 0; j < BJ; ++j, src += RPI * ldb) cp_async16(bs + bsl + j * RPI * kNwSB, src);
        } else {
          for (int i = lane; i < nrows * kNwBK; i += 32)
            cp_async4(bs + (i / kNwBK) * kNwSB + i % kNwBK, B + int64_t(i / kNwBK) * ldb + k0 + i % kNwBK);
        }
      } else {
        for (int i = lane; i < arows * kc; i += 32) {
          const int r = i / kc, kk = i % kc;
          cp_async4(as + kk * RPT + r, A + int64_t(r) * lda + k0 + kk);
        }
        for (int i = lane; i < nrows * kc; i += 32)
          cp_async4(bs + (i / kc) * kNwSB + i % kc, B + int64_t(i / kc) * ldb + k0 + i % kc);
      }
    }
    cp_async_commit();  // one group per tile slot, possibly empty
  };

  constexpr int NP = RPT / 2;
  float acc[RPT];
  float* outp[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int m = m0 + r;
    const bool live = m <= M && n < N;
    outp[r] = live ? ((m == M && pp.cb) ? pp.cb + c * pp.c_cs + n : pp.C + c * pp.c_cs + int64_t(m) * ldc + n)
                   : nullptr;
    acc[r] = live ? *outp[r] : 0.0f;
  }
  f2_t acc2[NP > 0 ? NP : 1];
#pragma unroll
  for (int i = 0; i < NP; ++i) acc2[i] = f2_pack(acc[2 * i], acc[2 * i + 1]);

  auto step = [&](const float* ak, float bq) {
    if constexpr (RPT == 1) {
      acc[0] = mac(acc[0], ak[0], bq);
    } else {
      const f2_t bb = f2_bcast(bq);
      if constexpr (RPT >= 4) {
#pragma unroll
        for (int i = 0; i < RPT / 4; ++i) {
          const float4 a4 = *reinterpret_cast<const float4*>(ak + 4 * i);
          acc2[2 * i] = f2_mac(acc2[2 * i], f2_pack(a4.x, a4.y), bb);
          acc2[2 * i + 1] = f2_mac(acc2[2 * i + 1], f2_pack(a4.z, a4.w), bb);
        }
      } else {
        const float2 a2 = *reinterpret_cast<const float2*>(ak);
        acc2[0] = f2_mac(acc2[0], f2_pack(a2.x, a2.y), bb);
      }
    }
  };
#pragma unroll
  for (int s = 0; s < kNwStages - 1; ++s) load(s);
  for (int tile = 0; tile < ntiles; ++tile) {
    cp_async_wait<kNwStages - 2>();
    __syncwarp();  // tile landed for all lanes; all lanes are past tile-1
    load(tile + kNwStages - 1);
    const int st = tile % kNwStages, kc = min(kNwBK, K - tile * kNwBK);
    const float* as = As + st * kNwBK * RPT;
    const float* bs = Bs + (st * 32 + lane) * kNwSB;
    if (kc == kNwBK && RPT == 2) {
      acc2[0] = nt_tile_rpt2<kNwBK>(acc2[0], as, bs);
    } else if (kc == kNwBK) {
#pragma unroll
      for (int kk = 0; kk < kNwBK; kk += 4) {
        const float4 b = *reinterpret_cast<const float4*>(bs + kk);
        step(as + (kk + 0) * RPT, b.x);
        step(as + (kk + 1) * RPT, b.y);
        step(as + (kk + 2) * RPT, b.z);
        step(as + (kk + 3) * RPT, b.w);
      }
    } else {
      for (int kk = 0; kk < kc; ++kk) step(as + kk * RPT, bs[kk]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    acc[2 * i] = f2_lo(acc2[i]);
    acc[2 * i + 1] = f2_hi(acc2[i]);
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r)
    if (outp[r]) *outp[r] = acc[r];
}

// Deep regime, one row per thread (the SPrM pre-pass: ~230 warps, one per SM
// sub-partition). A warp alone on its sub-partition gets no latency hiding
// from other warps, and ptxas, left to itself, issues a tile's 64 products
// first and then the 64 dependent adds with a 4-cycle stall each (measured
// 8 cycles per k in isolation, 14 in situ with the copy burst at the tile
// start). Here the tile is written as a software pipeline of volatile asm:
// per k one chain add, the product 16 k ahead, a shared load 32 k ahead, and
// one copy of the tile STAGES-1 ahead (19 copy slots: 16 B chunks, 2 A words,
// commit). ptxas still regroups independent instructions (the SASS shows the
// copies and adds partly clustered), but the streamed copies and the spread
// of outputs over 2x the sub-partitions bring the SPrM-step reduction from
// 78.8 us (2 paired rows per thread) to 68.6 us. Same per-output order as
// every NT path: acc = acc + a(k)*b(k), k ascending, separately rounded.
__device__ __forceinline__ float fmul_v(float a, float b) {
  float r;
  asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fadd_v(float a, float b) {
  float r;
  asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float f4c(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
template <class CopyFn>
__device__ __forceinline__ float nt_tile_r1(float acc, const float* as, const float* bs, CopyFn copy) {
  constexpr int KG = 16, NG = 4, NL = 8;  // per 16-k group: 4 B + 4 A LDS.128
  float4 L[2][NL];
  float P[2][KG];
  auto ld = [&](int g, int i) {
    return i < 4 ? lds128_v(bs + g * KG + 4 * i) : lds128_v(as + g * KG + 4 * (i - 4));
  };
  auto prod = [&](const float4 (&l)[NL], int k) { return fmul_v(f4c(l[4 + k / 4], k & 3), f4c(l[k / 4], k & 3)); };
#pragma unroll
  for (int i = 0; i < NL; ++i) L[0][i] = ld(0, i);
#pragma unroll
  for (int i = 0; i < NL; ++i) L[1][i] = ld(1, i);
#pragma unroll
  for (int k = 0; k < KG; ++k) P[0][k] = prod(L[0], k);
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const int cb = g & 1, nb = cb ^ 1;
#pragma unroll
    for (int k = 0; k < KG; ++k) {
      acc = fadd_v(acc, P[cb][k]);
      if (g + 1 < NG) P[nb][k] = prod(L[nb], k);
      if (g + 2 < NG && k < NL) L[cb][k] = ld(g + 2, k);
      copy(g * KG + k);
    }
  }
  return acc;
}

template <bool VEC, int STAGES>
__global__ void __launch_bounds__(kNwWarps * 32) k_gemm_nt_r1(NtBatch nb, const TickDesc* __restrict__ td) {
  pdl_wait();
  constexpr int BK = 64, SB = BK + 4;
  extern __shared__ __align__(128) float sm[];
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = int(blockIdx.x) * kNwWarps + w;
  if (task >= nb.first_task[nb.n]) return;  // warp-uniform; no block barriers below
  int prob = 0;
  while (prob + 1 < nb.n && task >= nb.first_task[prob + 1]) ++prob;
  const NtP& pp = nb.p[prob];
  const int lt = task - nb.first_task[prob];
  const int cg = lt % nb.colgroups[prob], m = lt / nb.colgroups[prob];
  const int M = pp.M, N = pp.N, K = pp.K;
  const int64_t ldb = pp.ldb;
  const int n0 = cg * 32, n = n0 + lane;
  const bool has_a = m < M;  // row M is the bias row (A = 1)
  const int nrows = min(32, N - n0);
  float* As = sm + w * nw_warp_floats(1, STAGES, BK);  // [stage][BK]
  float* Bs = As + STAGES * BK;                        // [stage][32][SB]
  const float* A = pp.A + c * pp.a_cs + int64_t(m) * pp.lda;
  const float* B = pp.B + c * pp.b_cs + int64_t(n0) * ldb;
  if (!has_a)
    for (int i = lane; i < STAGES * BK; i += 32) As[i] = m == M ? 1.0f : 0.0f;
  __syncwarp();
  const int ntiles = (K + BK - 1) / BK;
  const bool vec_tiles = VEC && nrows == 32;
  // full-tile copy slots: lane copies chunk lane%16 of B rows lane/16 + 2j
  const float* bl = B + int64_t(lane >> 4) * ldb + 4 * (lane & 15);
  const int bsl = (lane >> 4) * SB + 4 * (lane & 15);
  auto full_copy = [&](int tile, int slot) {  // slot 0..15 B, 16..17 A
    const int st = tile % STAGES, k0 = tile * BK;
    if (slot < 16) {
      cp_async16(Bs + st * 32 * SB + bsl + slot * 2 * SB, bl + k0 + int64_t(slot) * 2 * ldb);
    } else if (has_a) {
      const int e = slot - 16;
      cp_async4(As + st * BK + lane + 32 * e, A + k0 + lane + 32 * e);
    }
  };
  auto load_all = [&](int tile) {  // whole tile at once (prologue, ragged tiles, generic B)
    if (tile < ntiles) {
      const int st = tile % STAGES, k0 = tile * BK, kc = min(BK, K - k0);
      if (kc == BK && vec_tiles) {
#pragma unroll
        for (int j = 0; j < 18; ++j) full_copy(tile, j);
      } else {
        if (has_a)
          for (int i = lane; i < kc; i += 32) cp_async4(As + st * BK + i, A + k0 + i);
        for (int i = lane; i < nrows * kc; i += 32)
          cp_async4(Bs + st * 32 * SB + (i / kc) * SB + i % kc, B + int64_t(i / kc) * ldb + k0 + i % kc);
      }
    }
    cp_async_commit();  // one group per tile slot, possibly empty
  };

  float* outp = nullptr;
  float acc = 0.0f;
  if (m <= M && n < N) {
    outp = (m == M && pp.cb) ? pp.cb + c * pp.c_cs + n : pp.C + c * pp.c_cs + int64_t(m) * pp.ldc + n;
    acc = *outp;
  }
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) load_all(s);
  for (int tile = 0; tile < ntiles; ++tile) {
    cp_async_wait<STAGES - 2>();
    __syncwarp();  // tile landed for all lanes; all lanes are past tile-1
    const int st = tile % STAGES, kc = min(BK, K - tile * BK);
    const float* as = As + st * BK;
    const float* bs = Bs + (st * 32 + lane) * SB;
    const int nt = tile + STAGES - 1;
    if (kc == BK && vec_tiles && nt < ntiles && K - nt * BK >= BK) {
      // streamed copies of tile nt: one running B pointer (rows lane/16 + 2j)
      // and immediate shared offsets, so a copy costs one 64-bit add
      const int sn = nt % STAGES;
      const float* bsrc = bl + int64_t(nt) * BK;
      float* bdst = Bs + sn * 32 * SB + bsl;
      const int64_t bstep = 2 * ldb;
      acc = nt_tile_r1(acc, as, bs, [&](int slot) {
        if (slot < 16) {
          cp_async16(bdst + slot * 2 * SB, bsrc);
          bsrc += bstep;
        } else if (slot < 18) {
          if (has_a) cp_async4(As + sn * BK + lane + 32 * (slot - 16), A + int64_t(nt) * BK + lane + 32 * (slot - 16));
        } else if (slot == 18) {
          cp_async_commit();
        }
      });
    } else {
      load_all(nt);
      if (kc == BK) {
        acc = nt_tile_r1(acc, as, bs, [](int) {});
      } else {
        for (int kk = 0; kk < kc; ++kk) acc = fadd_v(acc, fmul_v(as[kk], bs[kk]));
      }
    }
  }
  cp_async_wait<0>();
  if (outp) *outp = acc;
}

// ------------------------------------------------------------------ embed
// x = emb[tok] + pos written feature-major xT[E][R*T] (the K/V projections and
// their weight gradients read it by feature), plus the last-position rows
// xl[R][E] for the query projection.
__global__ void k_embed(const uint32_t* __restrict__ tokens, ChunkGeo geo,
                        const float* __restrict__ params, int64_t p_cs, int64_t off_emb,
                        int64_t off_pos, uint32_t* ctx, int64_t ctx_cs, float* xT, int64_t x_cs,
                        float* xl, int64_t xl_cs, DmDims d, const TickDesc* __restrict__ td,
                        float* xtab, int64_t xtab_cs) {
  pdl_wait();
  // thread per coded position (r, t): one token gather, all E features
  // (x[j] = emb[tok][j] + pos[t][j], feature-major stores coalesced over rt)
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y], ch = td->chunk[blockIdx.y];
  const int64_t RT = int64_t(d.R) * d.T;
  const int64_t rt = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (xtab && rt >= RT && rt < RT + int64_t(d.T) * d.V) {
    // the deduplicated K/V inputs: x for every (position t, token v) pair,
    // row m = t*V + v of a feature-major [E][T*V] table (same adds as x)
    const int64_t m = rt - RT, TV = int64_t(d.T) * d.V;
    const int t = int(m / d.V), v = int(m % d.V);
    const float* P = params + c * p_cs;
    for (int j = 0; j < d.E; ++j)
      xtab[c * xtab_cs + int64_t(j) * TV + m] =
          fadd(__ldg(P + off_emb + int64_t(v) * d.E + j), __ldg(P + off_pos + int64_t(t) * d.E + j));
    return;
  }
  if (rt >= RT) return;
  const int t = int(uint32_t(rt) % uint32_t(d.T)), r = int(uint32_t(rt) / uint32_t(d.T));  // RT < 2^31
  const uint64_t L = geo.L[ch];
  const uint64_t jstep = uint64_t(d.T) + uint64_t(td->tick - geo.offset[ch]);  // coded position
  // tokens are < V = 4^k by construction; the mask only guards memory after a
  // decode error (positions past a truncated codestream are never written)
  const uint32_t tok = tokens[geo.start[ch] + uint64_t(r) * L + (jstep - d.T) + t] & uint32_t(d.V - 1);
  ctx[c * ctx_cs + rt] = tok;
  const float* P = params + c * p_cs;
  const float* er = P + off_emb + int64_t(tok) * d.E;
  const float* pr = P + off_pos + int64_t(t) * d.E;
  float* xo = xT + c * x_cs + rt;
  float* lo = t == d.T - 1 ? xl + c * xl_cs + int64_t(r) * d.E : nullptr;
  constexpr int kU = 8;
  for (int j0 = 0; j0 < d.E; j0 += kU) {
    float e[kU], q[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const bool ok = j0 + u < d.E;
      e[u] = ok ? __ldg(er + j0 + u) : 0.0f;
      q[u] = ok ? __ldg(pr + j0 + u) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (j0 + u >= d.E) break;
      const float xv = fadd(e[u], q[u]);
      xo[int64_t(j0 + u) * RT] = xv;
      if (lo) lo[j0 + u] = xv;
    }
  }
}

// ------------------------------------------------------------------ attention
// One warp per (row, head). Scores and the softmax sum use chains that every
// lane evaluates redundantly in reference order (shuffle-fed), so no lane has
// to broadcast a result.
__global__ void k_attn_fwd(const float* __restrict__ q, const float* __restrict__ k,
                           const float* __restrict__ v, float* wts, float* cx, int64_t cs_q,
                           int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
                           const TickDesc* __restrict__ td) {
  pdl_wait();
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= d.R * d.NH) return;
  const int r = warp / d.NH, h = warp % d.NH, HD = d.H / d.NH, T = d.T;
  const float* qp = q + c * cs_q + int64_t(r) * d.H + h * HD;
  const float* kp = k + c * cs_kv + int64_t(r) * T * d.H + h * HD;
  const float* vp = v + c * cs_kv + int64_t(r) * T * d.H + h * HD;
  float* w = wts + c * cs_w + (int64_t(r) * d.NH + h) * T;
  // scores s_t = (sum_d q[d] k_t[d]) * inv
  float mx = -__int_as_float(0x7f800000);
  for (int t = lane; t < T; t += 32) {
    float s = 0.0f;
    for (int dd = 0; dd < HD; ++dd) s = mac(s, qp[dd], kp[int64_t(t) * d.H + dd]);
    s = fmul(s, inv);
    w[t] = s;
    mx = fmaxf(mx, s);
  }
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  // det_softmax: exp, sequential sum over t, multiply by 1/sum
  float sum = 0.0f;
  for (int t0 = 0; t0 < T; t0 += 32) {
    const int t = t0 + lane;
    float e = 0.0f;
    if (t < T) {
      e = det_exp(fsub(w[t], mx));
      w[t] = e;
    }
    const int cnt = min(32, T - t0);
    for (int i = 0; i < cnt; ++i) sum = fadd(sum, __shfl_sync(0xffffffffu, e, i));
  }
  const float invs = fdiv(1.0f, sum);
  __syncwarp();
  for (int t = lane; t < T; t += 32) w[t] = fmul(w[t], invs);
  __syncwarp();
  // ctx[d] = sum_t w_t v_t[d], ascending t
  if (lane < HD) {
    float acc = 0.0f;
    for (int t = 0; t < T; ++t) acc = mac(acc, w[t], vp[int64_t(t) * d.H + lane]);
    cx[c * cs_q + int64_t(r) * d.H + h * HD + lane] = acc;
  }
}

// dk, dv are written feature-major ([H][R*T]: element (h*HD+d, r*T+t)) so the
// K/V weight-gradient reductions over R*T rows read contiguous rows.
constexpr int kAttnMaxT = 256;  // ds_t kept in shared memory up to this context length
__global__ void __launch_bounds__(256) k_attn_bwd(const float* __restrict__ q, const float* __restrict__ k,
                           const float* __restrict__ v, const float* __restrict__ wts,
                           const float* __restrict__ dctx, float* dq, float* dkT, float* dvT,
                           int64_t cs_q, int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
                           const TickDesc* __restrict__ td) {
  pdl_wait();
  __shared__ float sds[8][kAttnMaxT];
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= d.R * d.NH) return;
  const int r = warp / d.NH, h = warp % d.NH, HD = d.H / d.NH, T = d.T;
  const int64_t RT = int64_t(d.R) * T;
  const int64_t qo = c * cs_q + int64_t(r) * d.H + h * HD;
  const int64_t ko = c * cs_kv + int64_t(r) * T * d.H + h * HD;       // row-major K, V
  const int64_t to = c * cs_kv + int64_t(h) * HD * RT + int64_t(r) * T;  // feature-major dk, dv
  const float* w = wts + c * cs_w + (int64_t(r) * d.NH + h) * T;
  const float* dc = dctx + qo;
  // dv_t[d] = 0 + w_t*dc[d];  dwt_t = sum_d dc[d]*v_t[d];  dot = sum_t w_t*dwt_t
  float dot = 0.0f;
  float dwt_reg[kAttnMaxT / 32];
  for (int t0 = 0, q8 = 0; t0 < T; t0 += 32, ++q8) {
    const int t = t0 + lane;
    float prod = 0.0f;
    if (t < T) {
      const float wt = w[t];
      float acc = 0.0f;
      for (int dd = 0; dd < HD; ++dd) {
        dvT[to + int64_t(dd) * RT + t] = fadd(0.0f, fmul(wt, dc[dd]));
        acc = mac(acc, dc[dd], v[ko + int64_t(t) * d.H + dd]);
      }
      prod = fmul(wt, acc);
      if (q8 < kAttnMaxT / 32) dwt_reg[q8] = acc;
    }
    const int cnt = min(32, T - t0);
    for (int i = 0; i < cnt; ++i) dot = fadd(dot, __shfl_sync(0xffffffffu, prod, i));
  }
  // ds_t = (w_t*(dwt_t - dot))*inv;  dk_t[d] = 0 + ds_t*q[d]
  const bool keep = T <= kAttnMaxT;
  for (int t0 = 0, q8 = 0; t0 < T; t0 += 32, ++q8) {
    const int t = t0 + lane;
    if (t >= T) break;
    float dwt;
    if (keep) {
      dwt = dwt_reg[q8];
    } else {
      dwt = 0.0f;
      for (int dd = 0; dd < HD; ++dd) dwt = mac(dwt, dc[dd], v[ko + int64_t(t) * d.H + dd]);
    }
    const float ds = fmul(fmul(w[t], fsub(dwt, dot)), inv);
    if (keep) sds[wl][t] = ds;
    for (int dd = 0; dd < HD; ++dd) dkT[to + int64_t(dd) * RT + t] = fadd(0.0f, fmul(ds, q[qo + dd]));
  }
  __syncwarp();
  // dq[d] = 0 + sum_t ds_t*k_t[d], ascending t
  if (lane < HD) {
    float acc = 0.0f;
    for (int t = 0; t < T; ++t) {
      float ds;
      if (keep) {
        ds = sds[wl][t];
      } else {
        float dwt = 0.0f;
        for (int dd = 0; dd < HD; ++dd) dwt = mac(dwt, dc[dd], v[ko + int64_t(t) * d.H + dd]);
        ds = fmul(fmul(w[t], fsub(dwt, dot)), inv);
      }
      acc = mac(acc, ds, k[ko + int64_t(t) * d.H + lane]);
    }
    dq[qo + lane] = acc;
  }
}

// Row-blocked attention (the default path whenever a row's K and V fit in
// shared memory): one block per (chunk, coded row), K[r] and V[r] ([T][H]) are
// staged once with coalesced 16-byte loads into rows padded to H+4 floats, one
// warp per head. Same operation order as the warp-per-(row,head) kernels.
constexpr int kRowThreads = 256;  // 8 warps = the model's 8 heads
__host__ __device__ inline size_t attn_row_smem(const DmDims& d) {
  return (size_t(2) * d.T * (d.H + 4) + size_t(d.NH) * d.T + 2 * d.H) * sizeof(float);
}

// K/V rows of a coded row from the deduplicated tables: position t's row
// is table row t*V + ctx[t] (the (position, token) pair it was computed for)
__device__ __forceinline__ void stage_rows_tab(float* dst, const float* tab, const uint32_t* ctx_row,
                                               int T, int H, int V) {
  const int nv = T * (H / 4);
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    const int t = i / (H / 4), v4 = i % (H / 4);
    const int64_t row = int64_t(t) * V + int64_t(ctx_row[t]);
    cp_async16(dst + t * (H + 4) + 4 * v4, tab + row * H + 4 * v4);
  }
}

__device__ __forceinline__ void stage_rows(float* dst, const float* src, int T, int H) {
  // src [T][H] contiguous (H multiple of 4) -> dst rows of H+4
  const int nv = T * (H / 4);
  // by cp.async (no per-copy stall); the caller commits, waits and syncs
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    const int t = i / (H / 4), v4 = i % (H / 4);
    cp_async16(dst + t * (H + 4) + 4 * v4, src + int64_t(t) * H + 4 * v4);
  }
}

// up to 4 floats of a head's slice of a staged K/V row: one LDS.128 when the
// head width keeps the slices 16-byte aligned, else element loads (n valid)
__device__ __forceinline__ float4 ld_head4(const float* p, int n, bool aligned) {
  if (aligned) return *reinterpret_cast<const float4*>(p);
  float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  v.x = p[0];
  if (n > 1) v.y = p[1];
  if (n > 2) v.z = p[2];
  if (n > 3) v.w = p[3];
  return v;
}

__global__ void __launch_bounds__(kRowThreads) k_attn_fwd_row(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    float* wts, float* cx, int64_t cs_q, int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
    const TickDesc* __restrict__ td, KvTab kt) {
  pdl_wait();
  extern __shared__ __align__(128) float sm[];
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int r = blockIdx.x, T = d.T, H = d.H, HD = H / d.NH, HP = H + 4;
  const int h = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* Ks = sm;
  float* Vs = Ks + T * HP;
  float* Ws = Vs + T * HP;   // [NH][T]
  float* Qs = Ws + d.NH * T; // [H]
  if (kt.ctx) {
    const uint32_t* cr = kt.ctx + c * kt.ctx_cs + int64_t(r) * T;
    stage_rows_tab(Ks, k + c * cs_kv, cr, T, H, d.V);
    stage_rows_tab(Vs, v + c * cs_kv, cr, T, H, d.V);
  } else {
    const int64_t ko = c * cs_kv + int64_t(r) * T * H;
    stage_rows(Ks, k + ko, T, H);
    stage_rows(Vs, v + ko, T, H);
  }
  cp_async_commit();
  for (int i = threadIdx.x; i < H; i += blockDim.x) Qs[i] = q[c * cs_q + int64_t(r) * H + i];
  cp_async_wait<0>();
  __syncthreads();
  if (h < d.NH) {  // scores and det_softmax, warp per head
    const float* qh = Qs + h * HD;
    float* wrow = Ws + h * T;
    const bool hd4 = (HD & 3) == 0;  // head slices 16-byte aligned
    float mx = -__int_as_float(0x7f800000);
    for (int t = lane; t < T; t += 32) {
      const float* kr = Ks + t * HP + h * HD;
      float s = 0.0f;
      for (int d0 = 0; d0 < HD; d0 += 4) {  // LDS.128 per 4 dims: conflict-free across t
        const float4 k4 = ld_head4(kr + d0, HD - d0, hd4);
        const float kv[4] = {k4.x, k4.y, k4.z, k4.w};
  #pragma unroll
        for (int u = 0; u < 4; ++u)
          if (d0 + u < HD) s = mac(s, qh[d0 + u], kv[u]);
      }
      s = fmul(s, inv);
      wrow[t] = s;
      mx = fmaxf(mx, s);
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.0f;
    for (int t0 = 0; t0 < T; t0 += 32) {
      const int t = t0 + lane;
      float e = 0.0f;
      if (t < T) {
        e = det_exp(fsub(wrow[t], mx));
        wrow[t] = e;
      }
      const int cnt = min(32, T - t0);
      for (int i = 0; i < cnt; ++i) sum = fadd(sum, __shfl_sync(0xffffffffu, e, i));
    }
    const float invs = fdiv(1.0f, sum);
    float* wg = wts + c * cs_w + (int64_t(r) * d.NH + h) * T;
    for (int t = lane; t < T; t += 32) {
      const float wv = fmul(wrow[t], invs);
      wrow[t] = wv;
      wg[t] = wv;
    }
  }
  // context, one output per thread over the block (all heads' weights are in
  // shared memory): cx[o] = 0 + sum_t w[o/HD][t] * v_t[o], t ascending -- a
  // warp per head would leave all but HD of its lanes idle
  __syncthreads();
  for (int o = threadIdx.x; o < H; o += blockDim.x) {
    const float* wr = Ws + (o / HD) * T;
    float acc = 0.0f;
    for (int t = 0; t < T; ++t) acc = mac(acc, wr[t], Vs[t * HP + o]);
    cx[c * cs_q + int64_t(r) * H + o] = acc;
  }
}

// wT[slot] = (W_k^T, W_v^T) [2][H][E] of every active chunk: formed once per
// backward instead of by each of the chunk's R row blocks with 4-byte gathers
__global__ void k_wkv_transpose(const float* __restrict__ wk, const float* __restrict__ wv, int64_t w_cs,
                                float* wT, int E, int H, const TickDesc* __restrict__ td) {
  pdl_wait();
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int EH = E * H;
  if (i >= 2 * EH) return;
  const int which = i / EH, rem = i % EH, hh = rem / E, e = rem % E;
  wT[c * (2 * int64_t(EH)) + i] = (which ? wv : wk)[c * w_cs + e * H + hh];
}

template <int EB>  // fused dx: e per warp block (EB/2 paired chains per lane)
__global__ void __launch_bounds__(kRowThreads) k_attn_bwd_row(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ wts, const float* __restrict__ dctx, float* dq, float* dkT,
    float* dvT, int64_t cs_q, int64_t cs_kv, int64_t cs_w, DmDims d, float inv, AttnDx fx,
    const TickDesc* __restrict__ td, KvTab kt) {
  pdl_wait();
  extern __shared__ __align__(128) float sm[];
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int r = blockIdx.x, T = d.T, H = d.H, HD = H / d.NH, HP = H + 4;
  const int h = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t RT = int64_t(d.R) * T;
  float* Ks = sm;
  float* Vs = Ks + T * HP;
  float* Ds = Vs + T * HP;    // [NH][T]: ds_t per head
  float* Qs = Ds + d.NH * T;  // [H]
  float* Cs = Qs + H;         // dctx row [H]
  // fused dx (fx.dx set, NH == warps): this row's dk, dv [T][H+1] and Wk, Wv [E][H+1]
  const bool fuse = fx.dx != nullptr;
  const int DP = (T * (H + 1) + 3) & ~3;  // 16-byte aligned regions
  float* Dk = Cs + ((H + 3) & ~3);
  float* Dv = Dk + DP;
  float* Wks = Dv + DP;  // [H][E]
  float* Wvs = Wks + ((d.E * H + 3) & ~3);
  if (kt.ctx) {
    const uint32_t* cr = kt.ctx + c * kt.ctx_cs + int64_t(r) * T;
    stage_rows_tab(Ks, k + c * cs_kv, cr, T, H, d.V);
    stage_rows_tab(Vs, v + c * cs_kv, cr, T, H, d.V);
  } else {
    const int64_t ko = c * cs_kv + int64_t(r) * T * H;
    stage_rows(Ks, k + ko, T, H);
    stage_rows(Vs, v + ko, T, H);
  }
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    Qs[i] = q[c * cs_q + int64_t(r) * H + i];
    Cs[i] = dctx[c * cs_q + int64_t(r) * H + i];
  }
  if (fuse && fx.wT) {  // Wks[h][e] = W_k[e][h], Wvs after it: the chunk's pre-transposed pair
    const float* src = fx.wT + c * (2 * int64_t(d.E) * H);
    for (int i = threadIdx.x; i < d.E * H / 2; i += blockDim.x) cp_async16(Wks + 4 * i, src + 4 * i);
  } else if (fuse) {  // transposed: Wks[h][e] = W_k[e][h] (e runs contiguous for LDS.128)
    const float* wk = fx.wk + c * fx.w_cs;
    const float* wv = fx.wv + c * fx.w_cs;
    // destination-ordered (consecutive lanes, consecutive banks); the
    // strided side is the 4 KB global read, L2-resident
    for (int i = threadIdx.x; i < d.E * H; i += blockDim.x) {
      const int hh = i / d.E, e = i % d.E;
      cp_async4(Wks + i, wk + e * H + hh);
      cp_async4(Wvs + i, wv + e * H + hh);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  if (h < d.NH) {  // warp per head: dv, the dot chain, ds and dk
    const float* w = wts + c * cs_w + (int64_t(r) * d.NH + h) * T;
    const float* dc = Cs + h * HD;
    const int64_t to = c * cs_kv + int64_t(h) * HD * RT + int64_t(r) * T;  // feature-major dk, dv
    float* dsw = Ds + h * T;
    const bool hd4 = (HD & 3) == 0;  // head slices 16-byte aligned
    // dv_t[d] = 0 + w_t*dc[d]; dwt_t = sum_d dc[d]*v_t[d]; dot = sum_t w_t*dwt_t
    float dot = 0.0f;
    for (int t0 = 0; t0 < T; t0 += 32) {
      const int t = t0 + lane;
      float prod = 0.0f;
      if (t < T) {
        const float wt = w[t];
        const float* vr = Vs + t * HP + h * HD;
        float acc = 0.0f;
        for (int d0 = 0; d0 < HD; d0 += 4) {
          // one LDS.128 per 4 dims (rows 272 B apart: conflict-free), then the chain
          const float4 v4 = ld_head4(vr + d0, HD - d0, hd4);
          const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int dd = d0 + u;
            if (dd >= HD) break;
            const float dvv = fadd(0.0f, fmul(wt, dc[dd]));
            dvT[to + int64_t(dd) * RT + t] = dvv;
            if (fuse) Dv[t * (H + 1) + h * HD + dd] = dvv;
            acc = mac(acc, dc[dd], vv[u]);
          }
        }
        dsw[t] = acc;  // dwt_t, turned into ds_t below
        prod = fmul(wt, acc);
      }
      const int cnt = min(32, T - t0);
      for (int i = 0; i < cnt; ++i) dot = fadd(dot, __shfl_sync(0xffffffffu, prod, i));
    }
    // ds_t = (w_t*(dwt_t - dot))*inv;  dk_t[d] = 0 + ds_t*q[d]
    for (int t = lane; t < T; t += 32) {
      const float ds = fmul(fmul(w[t], fsub(dsw[t], dot)), inv);
      dsw[t] = ds;
      for (int dd = 0; dd < HD; ++dd) {
        const float dkv = fadd(0.0f, fmul(ds, Qs[h * HD + dd]));
        dkT[to + int64_t(dd) * RT + t] = dkv;
        if (fuse) Dk[t * (H + 1) + h * HD + dd] = dkv;
      }
    }
  }
  __syncthreads();  // every head's ds (Ds) and, fused, dk/dv rows (Dk, Dv) in shared memory
  // dq[o] = 0 + sum_t ds_t*k_t[o], t ascending: one output per thread on the
  // warps the fused dx leaves idle (a warp per head would use HD lanes)
  const int ndx = fuse ? min(d.NH, (d.E + EB - 1) / EB) : 0;
  const int base = ndx * 32 < int(blockDim.x) ? ndx * 32 : 0;
  if (int(threadIdx.x) >= base)
    for (int o = int(threadIdx.x) - base; o < H; o += int(blockDim.x) - base) {
      const float* dsr = Ds + (o / HD) * T;
      float acc = 0.0f;
      for (int t = 0; t < T; ++t) acc = mac(acc, dsr[t], Ks[t * HP + o]);
      dq[c * cs_q + int64_t(r) * H + o] = acc;
    }
  if (!fuse) return;
  // dx[r][t][e] = (0 + dk_t . W_k[e]) then + dv_t . W_v[e], h ascending: the
  // chain of the two accumulating GEMMs it replaces (Linear::backward x2,
  // layers.cpp:176-183; K terms first, layers.cpp:505-512)
  // lane = t, warp = a block of EB e (EB/2 paired chains per lane): W rows are
  // broadcast LDS.128 reads, the dk/dv row one conflict-free LDS per h
  float* dxr = fx.dx + c * fx.dx_cs + int64_t(r) * T * d.E;
  for (int eb = h * EB; eb < d.E; eb += d.NH * EB) {
    for (int t = lane; t < T; t += 32) {
      const float* dkr = Dk + t * (H + 1);
      const float* dvr = Dv + t * (H + 1);
      f2_t acc[EB / 2];
#pragma unroll
      for (int i = 0; i < EB / 2; ++i) acc[i] = 0;
      auto chain = [&](const float* dr, const float* Ws) {
#pragma unroll 4
        for (int hh = 0; hh < H; ++hh) {
          const f2_t dv2 = f2_bcast(dr[hh]);
#pragma unroll
          for (int i4 = 0; i4 < EB / 4; ++i4) {
            const float4 wa = *reinterpret_cast<const float4*>(Ws + hh * d.E + eb + 4 * i4);
            acc[2 * i4] = f2_mac(acc[2 * i4], dv2, f2_pack(wa.x, wa.y));
            acc[2 * i4 + 1] = f2_mac(acc[2 * i4 + 1], dv2, f2_pack(wa.z, wa.w));
          }
        }
      };
      chain(dkr, Wks);
      chain(dvr, Wvs);
      float* o = dxr + t * d.E + eb;
#pragma unroll
      for (int i4 = 0; i4 < EB / 4; ++i4)
        *reinterpret_cast<float4*>(o + 4 * i4) = make_float4(f2_lo(acc[2 * i4]), f2_hi(acc[2 * i4]),
                                                             f2_lo(acc[2 * i4 + 1]), f2_hi(acc[2 * i4 + 1]));
    }
  }
}

// ------------------------------------------------------------------ embed bwd
// pos grad: thread per (t, j), ascending rows, loads issued 16 rows ahead of
// the dependent adds. emb grad: warp per token value, lanes = j; positions are
// visited in (r,t) row-major order: a segment of ctx is staged in shared
// memory, each warp ballots its hits into a shared list, then walks the list
// with 16 independent dx loads in flight per batch.
__global__ void k_pos_bwd(const float* __restrict__ dx, int64_t dx_cs, const float* __restrict__ dxl,
                          int64_t dxl_cs, float* grads, int64_t g_cs, int64_t off_pos, DmDims d,
                          const TickDesc* __restrict__ td) {
  pdl_wait();
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= d.T * d.E) return;
  const int t = idx / d.E, j = idx % d.E;
  float* g = grads + c * g_cs + off_pos + idx;
  float acc = *g;
  const float* xp = dx + c * dx_cs + int64_t(t) * d.E + j;
  const float* lp = dxl + c * dxl_cs + j;
  const int64_t rs = int64_t(d.T) * d.E;
  const bool last = t == d.T - 1;
  constexpr int kB = 16;
  int r0 = 0;
  for (; r0 + kB <= d.R; r0 += kB) {  // full batches: 16 loads in flight, then the chain
    float v[kB], l[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) v[q] = __ldg(xp + (r0 + q) * rs);
    if (last) {
#pragma unroll
      for (int q = 0; q < kB; ++q) l[q] = __ldg(lp + int64_t(r0 + q) * d.E);
#pragma unroll
      for (int q = 0; q < kB; ++q) v[q] = fadd(v[q], l[q]);  // dx[:,last,:] += dxl (layers.cpp:521)
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) acc = fadd(acc, v[q]);
  }
  for (; r0 < d.R; ++r0) {
    float v = xp[r0 * rs];
    if (last) v = fadd(v, lp[int64_t(r0) * d.E]);
    acc = fadd(acc, v);
  }
  *g = acc;
}

constexpr int kEmbWarps = 8;
constexpr int kEmbSeg = 2048;

__global__ void __launch_bounds__(kEmbWarps * 32) k_emb_bwd(
    const uint32_t* __restrict__ ctx, int64_t ctx_cs, const float* __restrict__ dx, int64_t dx_cs,
    const float* __restrict__ dxl, int64_t dxl_cs, float* grads, int64_t g_cs, int64_t off_emb,
    DmDims d, const TickDesc* __restrict__ td) {
  pdl_wait();
  __shared__ uint32_t sctx[kEmbSeg];
  __shared__ uint16_t hits[kEmbWarps][kEmbSeg];
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tokv = blockIdx.x * kEmbWarps + wl;
  const uint32_t* cp = ctx + c * ctx_cs;
  const float* xp = dx + c * dx_cs;
  const float* lp = dxl ? dxl + c * dxl_cs : nullptr;
  const bool active_warp = tokv < d.V;
  float* g = grads + c * g_cs + off_emb + int64_t(active_warp ? tokv : 0) * d.E;
  constexpr int kMaxJ = 2;  // E = 64/scale <= 64
  float acc[kMaxJ];
  const int nj = (d.E + 31) / 32;
#pragma unroll
  for (int q = 0; q < kMaxJ; ++q) {
    const int j = lane + 32 * q;
    acc[q] = (active_warp && q < nj && j < d.E) ? g[j] : 0.0f;
  }
  const int64_t RT = int64_t(d.R) * d.T;
  for (int64_t s0 = 0; s0 < RT; s0 += kEmbSeg) {
    const int seg = int(RT - s0 < kEmbSeg ? RT - s0 : kEmbSeg);
    __syncthreads();
    for (int i = threadIdx.x; i < seg; i += kEmbWarps * 32) sctx[i] = cp[s0 + i];
    __syncthreads();
    if (!active_warp) continue;
    int nh = 0;
    for (int p0 = 0; p0 < seg; p0 += 32) {
      const int p = p0 + lane;
      const bool hit = p < seg && sctx[p] == uint32_t(tokv);
      const uint32_t bal = __ballot_sync(0xffffffffu, hit);
      if (hit) hits[wl][nh + __popc(bal & ((1u << lane) - 1u))] = uint16_t(p);
      nh += __popc(bal);
    }
    __syncwarp();
    constexpr int kB = 16;
    for (int h0 = 0; h0 < nh; h0 += kB) {
      const int cnt = min(kB, nh - h0);
#pragma unroll
      for (int q = 0; q < kMaxJ; ++q) {
        const int j = lane + 32 * q;
        if (q >= nj) break;
        const bool jv = j < d.E;
        const int jj = jv ? j : 0;
        float v[kB], l[kB];
        bool lastp[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {  // all loads first (clamped index past the end)
          const int64_t pp = s0 + hits[wl][h0 + (b < cnt ? b : 0)];
          lastp[b] = int(pp % d.T) == d.T - 1;
          v[b] = __ldg(xp + pp * d.E + jj);
          l[b] = dxl ? __ldg(lp + (pp / d.T) * d.E + jj) : 0.0f;
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const float x = (dxl && lastp[b]) ? fadd(v[b], l[b]) : v[b];  // dx[:,last,:] += dxl
          if (b < cnt && jv) acc[q] = fadd(acc[q], x);
        }
      }
    }
    __syncwarp();
  }
  if (!active_warp) return;
#pragma unroll
  for (int q = 0; q < kMaxJ; ++q) {
    const int j = lane + 32 * q;
    if (q < nj && j < d.E) g[j] = acc[q];
  }
}

// Sort-based embedding gradient (the default when a chunk's R*t positions and
// the vocabulary fit in shared memory). Three phases, one block per chunk:
//  1. stable counting sort of the positions by token: warp w owns the
//     contiguous span [w*RT/32, (w+1)*RT/32), counts it with match-any, the
//     block scans (token-major, warp-minor) and each warp then places its span
//     in order, so equal tokens keep ascending (r,t) order;
//  2. all threads gather dx (+ the last-position dxl term) in sorted order into
//     shared memory, a slab of positions at a time (independent loads);
//  3. one thread per (token, column) adds its contiguous run from shared
//     memory, carrying the sum across slabs.
// The per-element order is Embedding::backward's (layers.cpp:117-125).
constexpr int kSortThreads = 1024;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortMaxPos = 10240;
constexpr int kSortMaxV = 256;
constexpr int kSortAcc = 4;                 // (token, column) outputs per thread
constexpr int kSortVals = 36 * 1024;        // staged floats per slab
constexpr size_t kSortSmem = size_t(kSortVals) * 4 + size_t(kSortMaxPos) * 2 +
                             size_t(kSortWarps) * kSortMaxV * 2 + size_t(kSortMaxV + 1) * 4;
__global__ void __launch_bounds__(kSortThreads) k_emb_bwd_sorted(
    const uint32_t* __restrict__ ctx, int64_t ctx_cs, const float* __restrict__ dx, int64_t dx_cs,
    const float* __restrict__ dxl, int64_t dxl_cs, float* grads, int64_t g_cs, int64_t off_emb,
    DmDims d, const TickDesc* __restrict__ td) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* vals = reinterpret_cast<float*>(smem_raw);
  uint16_t* sorted = reinterpret_cast<uint16_t*>(vals + kSortVals);
  uint16_t* wc = sorted + kSortMaxPos;                       // [warp][V] counts, then cursors
  int* off = reinterpret_cast<int*>(wc + kSortWarps * kSortMaxV);  // [V+1]
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int V = d.V, E = d.E, RT = d.R * d.T;
  // token group of this block: tokens [v0, v1) (every block sorts redundantly)
  const int v0 = int(int64_t(V) * blockIdx.x / gridDim.x);
  const int v1 = int(int64_t(V) * (blockIdx.x + 1) / gridDim.x);
  const uint32_t* cp = ctx + c * ctx_cs;
  const int span = (RT + kSortWarps - 1) / kSortWarps;
  const int p0 = w * span, p1 = min(RT, p0 + span);
  const unsigned lt = (1u << lane) - 1u;
  // the warp's span of tokens, loaded once (independent loads in flight)
  constexpr int kSpanIt = (kSortMaxPos + kSortThreads - 1) / kSortThreads;
  uint32_t tokv[kSpanIt];
#pragma unroll
  for (int it = 0; it < kSpanIt; ++it) {
    const int p = p0 + it * 32 + lane;
    tokv[it] = p < p1 ? __ldg(cp + p) : 0xffffffffu;
  }
  // phase 1a: per-warp token counts
  for (int v = lane; v < V; v += 32) wc[w * V + v] = 0;
  __syncwarp();
#pragma unroll
  for (int it = 0; it < kSpanIt; ++it) {
    const int p = p0 + it * 32 + lane;
    const uint32_t v = tokv[it];
    const unsigned m = __match_any_sync(0xffffffffu, v);
    if (p < p1 && (m & lt) == 0) wc[w * V + v] = uint16_t(wc[w * V + v] + __popc(m));
    __syncwarp();
  }
  __syncthreads();
  // phase 1b: exclusive scan in (token, warp) order; wc becomes each warp's cursor
  if (w == 0) {
    int carry = 0;
    for (int v0 = 0; v0 < V; v0 += 32) {
      const int v = v0 + lane;
      int tot = 0;
      if (v < V)
        for (int ww = 0; ww < kSortWarps; ++ww) tot += wc[ww * V + v];
      int inc = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (v < V) {
        int a = carry + inc - tot;
        off[v] = a;
        for (int ww = 0; ww < kSortWarps; ++ww) {
          const int n = wc[ww * V + v];
          wc[ww * V + v] = uint16_t(a);
          a += n;
        }
      }
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) off[V] = carry;
  }
  __syncthreads();
  // phase 1c: stable placement
#pragma unroll
  for (int it = 0; it < kSpanIt; ++it) {
    const int p = p0 + it * 32 + lane;
    const uint32_t v = tokv[it];
    const unsigned m = __match_any_sync(0xffffffffu, v);
    if (p < p1) {
      const int cur = wc[w * V + v];
      sorted[cur + __popc(m & lt)] = uint16_t(p);
    }
    __syncwarp();
    if (p < p1 && (m & lt) == 0) wc[w * V + v] = uint16_t(wc[w * V + v] + __popc(m));
    __syncwarp();
  }
  __syncthreads();
  // phases 2+3 over this block's tokens: sorted range [off[v0], off[v1])
  const float* xp = dx + c * dx_cs;
  const float* lp = dxl ? dxl + c * dxl_cs : nullptr;
  float* gp = grads + c * g_cs + off_emb;
  const int o0 = v0 * E, VE = (v1 - v0) * E;
  const int r0 = off[v0], r1 = off[v1];
  float acc[kSortAcc];
#pragma unroll
  for (int q = 0; q < kSortAcc; ++q) {
    const int o = tid + q * kSortThreads;
    acc[q] = o < VE ? gp[o0 + o] : 0.0f;
  }
  const int slab = kSortVals / E;
  for (int s0 = r0; s0 < r1; s0 += slab) {
    const int s1 = min(r1, s0 + slab);
    const int n = (s1 - s0) * E;
    constexpr int kG = 8;  // loads in flight per thread
    for (int i0 = tid; i0 < n; i0 += kG * kSortThreads) {
      float val[kG], lv[kG];
      bool last[kG];
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        const int i = i0 + u * kSortThreads;
        val[u] = 0.0f;
        lv[u] = 0.0f;
        last[u] = false;
        if (i < n) {
          const int h = s0 + i / E, j = i % E;
          const int pp = sorted[h];
          val[u] = __ldg(xp + int64_t(pp) * E + j);
          last[u] = lp && pp % d.T == d.T - 1;
          if (last[u]) lv[u] = __ldg(lp + int64_t(pp / d.T) * E + j);
        }
      }
#pragma unroll
      for (int u = 0; u < kG; ++u) {
        const int i = i0 + u * kSortThreads;
        if (i < n) vals[i] = last[u] ? fadd(val[u], lv[u]) : val[u];
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kSortAcc; ++q) {
      const int o = tid + q * kSortThreads;
      if (o < VE) {
        const int v = v0 + o / E, j = o % E;
        const int b0 = max(off[v], s0), b1 = min(off[v + 1], s1);
        float a = acc[q];
        int h = b0;
        for (; h + 8 <= b1; h += 8) {
          float x[8];
#pragma unroll
          for (int b = 0; b < 8; ++b) x[b] = vals[(h + b - s0) * E + j];
#pragma unroll
          for (int b = 0; b < 8; ++b) a = fadd(a, x[b]);
        }
        for (; h < b1; ++h) a = fadd(a, vals[(h - s0) * E + j]);
        acc[q] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < kSortAcc; ++q) {
    const int o = tid + q * kSortThreads;
    if (o < VE) gp[o0 + o] = acc[q];
  }
}

static bool sorted_emb_ok(const DmDims& d) {
  return d.R * d.T <= kSortMaxPos && d.V <= kSortMaxV && d.V * d.E <= kSortThreads * kSortAcc &&
         d.E <= kSortVals / 64;
}
static void launch_sorted_emb(const uint32_t* ctx, int64_t ctx_cs, const float* dx, int64_t dx_cs,
                              const float* dxl, int64_t dxl_cs, float* grads, int64_t g_cs,
                              int64_t off_emb, DmDims d, const TickDesc* td, int max_active,
                              cudaStream_t st) {
  ensure_smem(reinterpret_cast<const void*>(k_emb_bwd_sorted), kSortSmem);
  // split the vocabulary over several blocks per chunk while chunks alone
  // cannot fill the chip (each block re-sorts; the gather and walk split)
  const int groups = std::max(1, std::min(std::min(8, d.V), 148 / std::max(1, max_active)));
  launch_pdl(k_emb_bwd_sorted, dim3(dim3(unsigned(groups), unsigned(max_active))), dim3(kSortThreads), kSortSmem, st, 
      ctx, ctx_cs, dx, dx_cs, dxl, dxl_cs, grads, g_cs, off_emb, d, td);
}

// ------------------------------------------------------------------ Adam
__global__ void k_adam(float* __restrict__ w, float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, int64_t p_cs, int64_t n,
                       const AdamScalars* __restrict__ sc, const TickDesc* __restrict__ td) {
  pdl_wait();
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const float bc1 = sc[c].bc1, bc2 = sc[c].bc2;
  const float b1 = 0.9f, b2 = 0.999f, lr = 5e-4f, eps = 1e-8f;
  const float omb1 = fsub(1.0f, b1), omb2 = fsub(1.0f, b2);
  const int64_t base = c * p_cs;
  // U elements per thread per round, all loads issued before the math: the
  // update is latency-bound on its HBM reads, not on the IEEE divides
  constexpr int U = 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    float gi[U], mo[U], vo[U], wo[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        const int64_t o = base + i;
        gi[u] = g[o];
        mo[u] = m[o];
        vo[u] = v[o];
        wo[u] = w[o];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        const int64_t o = base + i;
        const float mi = fadd(fmul(b1, mo[u]), fmul(omb1, gi[u]));
        const float vi = fadd(fmul(b2, vo[u]), fmul(fmul(omb2, gi[u]), gi[u]));
        const float mhat = fdiv(mi, bc1);
        const float vhat = fdiv(vi, bc2);
        w[o] = fsub(wo[u], fdiv(fmul(lr, mhat), fadd(__fsqrt_rn(vhat), eps)));
        m[o] = mi;
        v[o] = vi;
        g[o] = 0.0f;
      }
    }
  }
}

__global__ void k_state_copy(float* w, float* m, float* v, AdamScalars* sc, int64_t p_cs, int64_t n,
                             const TickDesc* __restrict__ td) {
  pdl_wait();
  if (blockIdx.y >= unsigned(td->n_hand)) return;
  const int2 pr = td->hand[blockIdx.y];  // x = src, y = dst
  const int64_t so = pr.x * p_cs, dof = pr.y * p_cs;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    w[dof + i] = w[so + i];
    m[dof + i] = m[so + i];
    v[dof + i] = v[so + i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[pr.y] = sc[pr.x];
}

__global__ void k_tick_advance(TickDesc* td, const uint32_t* __restrict__ act_ptr,
                               const int* __restrict__ act_all, const int* __restrict__ chunk_all,
                               const uint32_t* __restrict__ hand_ptr,
                               const int2* __restrict__ hand_all, int64_t ticks) {
  pdl_wait();
  const int64_t t = td->tick + 1;
  td->tick = t;
  if (t < ticks) {
    td->act = act_all + act_ptr[t];
    td->chunk = chunk_all + act_ptr[t];
    td->n_act = int(act_ptr[t + 1] - act_ptr[t]);
    td->hand = hand_all + hand_ptr[t];
    td->n_hand = int(hand_ptr[t + 1] - hand_ptr[t]);
  } else {
    td->n_act = 0;
    td->n_hand = 0;
  }
}

// Descriptor of the tick after `cur` (act list only): the static predictors of
// tick tau+1 run inside tick tau's graph (cross-tick pipeline).
__global__ void k_tick_peek(const TickDesc* __restrict__ cur, TickDesc* next,
                            const uint32_t* __restrict__ act_ptr, const int* __restrict__ act_all,
                            const int* __restrict__ chunk_all, int64_t ticks) {
  pdl_wait();
  const int64_t t = cur->tick + 1;
  next->tick = t;
  next->hand = nullptr;
  next->n_hand = 0;
  if (t >= 0 && t < ticks) {
    next->act = act_all + act_ptr[t];
    next->chunk = chunk_all + act_ptr[t];
    next->n_act = int(act_ptr[t + 1] - act_ptr[t]);
  } else {
    next->act = act_all;
    next->chunk = chunk_all;
    next->n_act = 0;
  }
}

// Context tokens of every active chunk's coded rows (k_embed's ctx gather alone)
__global__ void k_ctx_gather(const uint32_t* __restrict__ tokens, ChunkGeo geo, uint32_t* ctx,
                             int64_t ctx_cs, DmDims d, const TickDesc* __restrict__ td) {
  pdl_wait();
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y], ch = td->chunk[blockIdx.y];
  const int64_t RT = int64_t(d.R) * d.T;
  const int64_t rt = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (rt >= RT) return;
  const int t = int(uint32_t(rt) % uint32_t(d.T)), r = int(uint32_t(rt) / uint32_t(d.T));  // RT < 2^31
  const uint64_t L = geo.L[ch];
  const uint64_t jstep = uint64_t(d.T) + uint64_t(td->tick - geo.offset[ch]);
  ctx[c * ctx_cs + rt] = tokens[geo.start[ch] + uint64_t(r) * L + (jstep - d.T) + t] & uint32_t(d.V - 1);
}

}  // namespace

void launch_tick_peek(const TickDesc* cur, TickDesc* next, const uint32_t* act_ptr,
                      const int* act_all, const int* chunk_all, int64_t ticks, cudaStream_t st) {
  launch_pdl(k_tick_peek, dim3(1), dim3(1), 0, st, cur, next, act_ptr, act_all, chunk_all, ticks);
}
void launch_ctx_gather(const uint32_t* tokens, ChunkGeo geo, uint32_t* ctx, int64_t ctx_cs,
                       DmDims d, const TickDesc* td, int max_active, cudaStream_t st) {
  if (max_active <= 0) return;
  const int64_t RT = int64_t(d.R) * d.T;
  launch_pdl(k_ctx_gather, dim3(dim3(unsigned((RT + 255) / 256), max_active)), dim3(256), 0, st, tokens, geo, ctx, ctx_cs,
                                                                             d, td);
}

int launch_gemm(const GemmP& p, bool at, bool bt, const TickDesc* td, int max_active,
                cudaStream_t st) {
  if (max_active <= 0 || p.N <= 0 || p.M + p.ones_row <= 0) return 0;
  // A bias row on top of a tile-aligned M (weight gradient + bias gradient,
  // M = fan-in) would cost a whole extra row of tiles for one row: run the M
  // rows as a GEMM and the bias row as its own column-sum chain.
  // (only with many chunks in flight: for one chunk the extra tile row is
  // cheap and the separate chain launch would sit on the critical path)
  if (p.ones_row && p.M > 0 && p.M % 64 == 0 && p.nprob <= 1 && !p.mask && max_active >= 8) {
    GemmP q = p;
    q.ones_row = 0;
    const int n = launch_gemm(q, at, bt, td, max_active, st);
    const dim3 grid(unsigned((p.N + 127) / 128), unsigned(max_active));
    if (bt) launch_pdl(k_bias_row<true>, dim3(grid), dim3(128), 0, st, p, td);
    else launch_pdl(k_bias_row<false>, dim3(grid), dim3(128), 0, st, p, td);
    return n + 1;
  }
  if (at && bt) gemm_dispatch<true, true>(p, td, max_active, st);
  else if (at) gemm_dispatch<true, false>(p, td, max_active, st);
  else if (bt) gemm_dispatch<false, true>(p, td, max_active, st);
  else gemm_dispatch<false, false>(p, td, max_active, st);
  return 1;
}

void launch_gemm_nt_batch(const NtP* probs, int nprob, const TickDesc* td, int max_active,
                          cudaStream_t st) {
  if (max_active <= 0 || nprob <= 0) return;
  auto al = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  bool vec = true;
  for (int i = 0; i < nprob; ++i) {
    const NtP& p = probs[i];
    vec = vec && p.K % 4 == 0 && p.ldb % 4 == 0 && p.b_cs % 4 == 0 && al(p.B);
  }
  {
#define PMKLC_NT_ATTR(V, R, S, K)                                        \
  ensure_smem(reinterpret_cast<const void*>(k_gemm_nt<V, R, S, K>), \
              kNwWarps * nw_warp_floats(R, S, K) * sizeof(float))
    PMKLC_NT_ATTR(true, 8, PMKLC_NT8_S, PMKLC_NT8_BK); PMKLC_NT_ATTR(false, 8, PMKLC_NT8_S, PMKLC_NT8_BK); PMKLC_NT_ATTR(true, 4, 3, 32);
    PMKLC_NT_ATTR(false, 4, 3, 32); PMKLC_NT_ATTR(true, 2, 3, 32); PMKLC_NT_ATTR(false, 2, 3, 32);
    PMKLC_NT_ATTR(true, 2, 6, 64); PMKLC_NT_ATTR(false, 2, 6, 64);
    ensure_smem(reinterpret_cast<const void*>(k_gemm_nt_r1<true, 6>),
                kNwWarps * nw_warp_floats(1, 6, 64) * sizeof(float));
    ensure_smem(reinterpret_cast<const void*>(k_gemm_nt_r1<false, 6>),
                kNwWarps * nw_warp_floats(1, 6, 64) * sizeof(float));
#undef PMKLC_NT_ATTR
  }
  auto build = [&](int rpt, NtBatch& nb) {
    nb.n = nprob;
    nb.first_task[0] = 0;
    for (int i = 0; i < nprob; ++i) {
      nb.p[i] = probs[i];
      nb.colgroups[i] = (probs[i].N + 31) / 32;
      nb.first_task[i + 1] = nb.first_task[i] + (probs[i].M + 1 + rpt - 1) / rpt * nb.colgroups[i];
    }
    return nb.first_task[nprob];
  };
  // Rows per thread: 8 (B read once per 8 rows) while that still gives ~8
  // warps per SM, else 4 while that gives ~4; a launch that cannot fill the chip
  // is bound by the k chain (4 cycles per step), which 2 paired rows per thread
  // still meet, with deep 64-k tiles so the few warps neither wait on L2 nor
  // spend their issue slots on per-tile bookkeeping.
  NtBatch nb;
  int rpt = 8;
  if (int64_t(build(8, nb)) * max_active < 148 * 8) rpt = 4;
  if (rpt == 4 && int64_t(build(4, nb)) * max_active < 148 * 4) rpt = 2;
  static const int force_rpt = [] {  // PMKLC_NT_RPT=8|4|2: fixed rows per thread (experiments)
    const char* e = std::getenv("PMKLC_NT_RPT");
    return e ? std::atoi(e) : 0;
  }();
  if (force_rpt == 8 || force_rpt == 4 || force_rpt == 2) rpt = force_rpt;
  const int tasks = build(rpt, nb);
  // deep regime up to 8 paired-row warps per SM: at ~24 chunks (the config-4
  // SMP wavefront) one row per thread over more warps beats 2 paired rows
  // (dWk/dWv reduction 191 -> 155 us per tick, decode tick 931 -> 892 us)
  static const int deep_warps = [] {
    const char* e = std::getenv("PMKLC_NT_DEEP_WARPS");
    return e ? std::atoi(e) : 8;
  }();
  bool deep = !force_rpt && rpt == 2 && int64_t(tasks) * max_active < 148 * deep_warps;
  // deep regime: one row per thread spreads the outputs over twice the SM
  // sub-partitions; each then needs 2 FP32-pipe cycles per k (exact mul +
  // add) under the 4-cycle add chain instead of exactly 4 with a row pair.
  static const int deep_rpt = [] {
    const char* e = std::getenv("PMKLC_NT_DEEP_RPT");
    return e ? std::atoi(e) : 1;
  }();
  if (deep && deep_rpt == 1) {
    build(1, nb);
    rpt = 1;
  }
  const int tasks_final = nb.first_task[nprob];
  const int stages = deep ? 6 : rpt == 8 ? PMKLC_NT8_S : 3, bk = deep ? 64 : rpt == 8 ? PMKLC_NT8_BK : 32;
  const dim3 grid(unsigned((tasks_final + kNwWarps - 1) / kNwWarps), unsigned(max_active));
  const size_t smem = size_t(kNwWarps) * nw_warp_floats(rpt, stages, bk) * sizeof(float);
#define PMKLC_NT_LAUNCH(R, S, K)                                                               \
  if (vec) launch_pdl(k_gemm_nt<true, R, S, K>, dim3(grid), dim3(kNwWarps * 32), smem, st, nb, td);               \
  else launch_pdl(k_gemm_nt<false, R, S, K>, dim3(grid), dim3(kNwWarps * 32), smem, st, nb, td);
  if (rpt == 8) {
    PMKLC_NT_LAUNCH(8, PMKLC_NT8_S, PMKLC_NT8_BK)
  } else if (rpt == 4) {
    PMKLC_NT_LAUNCH(4, 3, 32)
  } else if (!deep) {
    PMKLC_NT_LAUNCH(2, 3, 32)
  } else if (rpt == 2) {
    PMKLC_NT_LAUNCH(2, 6, 64)
  } else if (vec) {
    launch_pdl(k_gemm_nt_r1<true, 6>, dim3(grid), dim3(kNwWarps * 32), smem, st, nb, td);
  } else {
    launch_pdl(k_gemm_nt_r1<false, 6>, dim3(grid), dim3(kNwWarps * 32), smem, st, nb, td);
  }
#undef PMKLC_NT_LAUNCH
}

void launch_gemm_nt(const NtP& p0, const NtP* p1, const TickDesc* td, int max_active,
                    cudaStream_t st) {
  NtP ps[2] = {p0, p1 ? *p1 : p0};
  launch_gemm_nt_batch(ps, p1 ? 2 : 1, td, max_active, st);
}

void launch_embed(const uint32_t* tokens, ChunkGeo geo, const float* params,
                  int64_t p_cs, int64_t off_emb, int64_t off_pos, uint32_t* ctx, int64_t ctx_cs,
                  float* x, int64_t x_cs, float* xl, int64_t xl_cs, DmDims d, const TickDesc* td,
                  int max_active, cudaStream_t st, float* xtab, int64_t xtab_cs) {
  if (max_active <= 0) return;
  // one thread per coded position (+ one per (t, v) table row)
  const int64_t total = int64_t(d.R) * d.T + (xtab ? int64_t(d.T) * d.V : 0);
  dim3 grid(unsigned((total + 255) / 256), max_active);
  launch_pdl(k_embed, dim3(grid), dim3(256), 0, st, tokens, geo, params, p_cs, off_emb, off_pos, ctx, ctx_cs, x,
                                x_cs, xl, xl_cs, d, td, xtab, xtab_cs);
}

bool attn_rows_ok(const DmDims& d) {  // both row kernels (forward and backward) are used
  return d.NH <= 8 && d.H % 4 == 0 && attn_row_smem(d) + d.H * sizeof(float) <= 200 * 1024;
}

void launch_attn_fwd(const float* q, const float* k, const float* v, float* wts, float* cx,
                     int64_t cs_q, int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
                     const TickDesc* td, int max_active, cudaStream_t st, const KvTab& kt) {
  if (max_active <= 0) return;
  const size_t smem = attn_row_smem(d);
  if (d.NH <= 8 && d.H % 4 == 0 && smem <= 200 * 1024) {
    ensure_smem(reinterpret_cast<const void*>(k_attn_fwd_row), smem);
    launch_pdl(k_attn_fwd_row, dim3(dim3(d.R, max_active)), dim3(kRowThreads), smem, st, q, k, v, wts, cx, cs_q, cs_kv,
                                                                      cs_w, d, inv, td, kt);
    return;
  }
  const int64_t warps = int64_t(d.R) * d.NH;
  dim3 grid(unsigned((warps * 32 + 255) / 256), max_active);
  launch_pdl(k_attn_fwd, dim3(grid), dim3(256), 0, st, q, k, v, wts, cx, cs_q, cs_kv, cs_w, d, inv, td);
}

bool launch_attn_bwd(const float* q, const float* k, const float* v, const float* wts,
                     const float* dctx, float* dq, float* dk, float* dv, int64_t cs_q,
                     int64_t cs_kv, int64_t cs_w, DmDims d, float inv, const AttnDx& fx,
                     const TickDesc* td, int max_active, cudaStream_t st, const KvTab& kt) {
  if (max_active <= 0) return fx.dx != nullptr;
  const size_t base = attn_row_smem(d) + d.H * sizeof(float);
  const size_t extra = (size_t(2) * (d.T * (d.H + 1) + 3) + size_t(2) * (d.E * d.H + 3) + 8) *
                       sizeof(float);
  if (d.NH <= 8 && d.H % 4 == 0 && base <= 200 * 1024) {
    const bool fuse = fx.dx && d.NH * 32 == kRowThreads && d.E % 8 == 0 &&
                      base + extra <= 200 * 1024;
    const size_t smem = base + (fuse ? extra : 0);
    AttnDx f = fx;
    if (!fuse) f.dx = nullptr;
    // e per warp in the fused dx: 4 while the 8 warps still have e left to
    // share (E <= 32), else 8
    const int eb = d.E <= 4 * d.NH ? 4 : 8;
    if (fuse && f.wT)  // W_k^T, W_v^T once per chunk (8.56 vs 8.45 MB/s on config 3)
      launch_pdl(k_wkv_transpose, dim3(unsigned((2 * d.E * d.H + 255) / 256), unsigned(max_active)), dim3(256),
                 0, st, fx.wk, fx.wv, fx.w_cs, f.wT, d.E, d.H, td);
    const auto kern = eb == 4 ? k_attn_bwd_row<4> : k_attn_bwd_row<8>;
    ensure_smem(reinterpret_cast<const void*>(kern), smem);
    launch_pdl(kern, dim3(dim3(d.R, max_active)), dim3(kRowThreads), smem, st,
        q, k, v, wts, dctx, dq, dk, dv, cs_q, cs_kv, cs_w, d, inv, f, td, kt);
    return fuse;
  }
  const int64_t warps = int64_t(d.R) * d.NH;
  dim3 grid(unsigned((warps * 32 + 255) / 256), max_active);
  launch_pdl(k_attn_bwd, dim3(grid), dim3(256), 0, st, q, k, v, wts, dctx, dq, dk, dv, cs_q, cs_kv, cs_w, d, inv,
                                   td);
  return false;
}

void launch_emb_grad(const uint32_t* ctx, int64_t ctx_cs, const float* dx, int64_t dx_cs,
                     float* grads, int64_t g_cs, int64_t off_emb, DmDims d, const TickDesc* td,
                     int max_active, cudaStream_t st) {
  if (max_active <= 0) return;
  if (sorted_emb_ok(d)) {
    launch_sorted_emb(ctx, ctx_cs, dx, dx_cs, nullptr, 0, grads, g_cs, off_emb, d, td, max_active, st);
    return;
  }
  dim3 g2(unsigned((d.V + kEmbWarps - 1) / kEmbWarps), max_active);
  launch_pdl(k_emb_bwd, dim3(g2), dim3(kEmbWarps * 32), 0, st, ctx, ctx_cs, dx, dx_cs, nullptr, 0, grads, g_cs, off_emb,
                                           d, td);
}

void launch_embed_bwd(const uint32_t* ctx, int64_t ctx_cs, const float* dx, int64_t dx_cs,
                      const float* dxl, int64_t dxl_cs, float* grads, int64_t g_cs,
                      int64_t off_emb, int64_t off_pos, DmDims d, const TickDesc* td, int max_active,
                      cudaStream_t st) {
  if (max_active <= 0) return;
  dim3 g1(unsigned((d.T * d.E + 255) / 256), max_active);
  launch_pdl(k_pos_bwd, dim3(g1), dim3(256), 0, st, dx, dx_cs, dxl, dxl_cs, grads, g_cs, off_pos, d, td);
  if (sorted_emb_ok(d)) {
    launch_sorted_emb(ctx, ctx_cs, dx, dx_cs, dxl, dxl_cs, grads, g_cs, off_emb, d, td, max_active,
                      st);
    return;
  }
  dim3 g2(unsigned((d.V + kEmbWarps - 1) / kEmbWarps), max_active);
  launch_pdl(k_emb_bwd, dim3(g2), dim3(kEmbWarps * 32), 0, st, ctx, ctx_cs, dx, dx_cs, dxl, dxl_cs, grads, g_cs, off_emb, d,
                                td);
}

void launch_adam(float* w, float* g, float* m, float* v, int64_t p_cs, int64_t n,
                 const AdamScalars* sc, const TickDesc* td, int max_active, cudaStream_t st) {
  if (max_active <= 0 || n <= 0) return;
  const int64_t per = (n + 255) / 256;
  dim3 grid(unsigned(per < 64 ? per : 64), max_active);
  launch_pdl(k_adam, dim3(grid), dim3(256), 0, st, w, g, m, v, p_cs, n, sc, td);
}

void launch_state_copy(float* w, float* m, float* v, AdamScalars* sc, int64_t p_cs, int64_t n,
                       const TickDesc* td, int max_pairs, cudaStream_t st) {
  if (max_pairs <= 0) return;
  const int64_t per = (n + 255) / 256;
  dim3 grid(unsigned(per < 64 ? per : 64), max_pairs);
  launch_pdl(k_state_copy, dim3(grid), dim3(256), 0, st, w, m, v, sc, p_cs, n, td);
}

void launch_tick_advance(TickDesc* td, const uint32_t* act_ptr, const int* act_all,
                         const int* chunk_all, const uint32_t* hand_ptr, const int2* hand_all,
                         int64_t ticks, cudaStream_t st) {
  launch_pdl(k_tick_advance, dim3(1), dim3(1), 0, st, td, act_ptr, act_all, chunk_all, hand_ptr,
             hand_all, ticks);
}

}  // namespace pmklc_b200
