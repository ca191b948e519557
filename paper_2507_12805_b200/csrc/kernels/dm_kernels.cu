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
#include <algorithm>
#include <cstdint>

#include "detmath.cuh"
#include "kernels.hpp"

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
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <bool AT, bool BT, int TM, int TN, int BK, int STAGES, int TX, int TY>
__global__ void __launch_bounds__(TX * TY) k_gemm_tiled(GemmP p, const TickDesc* __restrict__ td) {
  constexpr int NT = TX * TY, BM = TY * TM, BN = TX * TN;
  __shared__ __align__(16) float As[STAGES][BK][BM + 4];
  __shared__ __align__(16) float Bs[STAGES][BK][BN + 4];
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

  auto load = [&](int tile) {
    if (tile < ntiles) {
      const int stage = tile % STAGES, k0 = tile * BK;
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
      for (int idx = threadIdx.x; idx < BN * BK; idx += NT) {
        int nn, kk;
        if (BT) { kk = idx % BK; nn = idx / BK; }
        else    { nn = idx % BN; kk = idx / BN; }
        const int n = n0 + nn, k = k0 + kk;
        if (k < p.K && n < p.N)
          cp_async4(&Bs[stage][kk][nn], BT ? B + int64_t(n) * p.ldb + k : B + int64_t(k) * p.ldb + n);
      }
    }
    cp_async_commit();  // one group per tile slot, possibly empty
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int m = m0 + ty * TM + i, n = n0 + tx * TN + j;
      float v = 0.0f;
      if (m < Mx && n < p.N) {
        if (p.init == 1) v = bias[n];
        else if (p.init == 2) v = C[int64_t(m) * p.ldc + n];
      }
      acc[i][j] = v;
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
    auto body = [&](int kk) {
      // each thread's TM (TN) operands are contiguous: one vector shared load each
      float a[TM], b[TN];
      const float* ap = &As[stage][kk][ty * TM];
      const float* bp = &Bs[stage][kk][tx * TN];
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
      if constexpr (TN == 4) {
        const float4 v = *reinterpret_cast<const float4*>(bp);
        b[0] = v.x; b[1] = v.y; b[2] = v.z; b[3] = v.w;
      } else if constexpr (TN == 2) {
        const float2 v = *reinterpret_cast<const float2*>(bp);
        b[0] = v.x; b[1] = v.y;
      } else {
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = bp[j];
      }
      if (relu) {
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = a[i] < 0.0f ? 0.0f : a[i];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = mac(acc[i][j], a[i], b[j]);
    };
    if (kmax == BK) {
#pragma unroll 8
      for (int kk = 0; kk < BK; ++kk) body(kk);
    } else {
      for (int kk = 0; kk < kmax; ++kk) body(kk);
    }
  }
  cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int m = m0 + ty * TM + i, n = n0 + tx * TN + j;
      if (m < Mx && n < p.N) {
        float v = acc[i][j];
        if (p.mask && p.mask[c * p.mask_cs + int64_t(m) * p.ldm + n] <= 0.0f) v = 0.0f;
        C[int64_t(m) * p.ldc + n] = v;
      }
    }
}

template <bool AT, bool BT, int TM, int TN, int BK, int STAGES, int TX = 16, int TY = 16>
void gemm_launch(const GemmP& p, const TickDesc* td, int max_active, cudaStream_t st) {
  const int Mx = p.M + (p.ones_row ? 1 : 0);
  const int np = p.nprob > 1 ? p.nprob : 1;
  dim3 grid((p.N + TX * TN - 1) / (TX * TN), (Mx + TY * TM - 1) / (TY * TM), max_active * np);
  k_gemm_tiled<AT, BT, TM, TN, BK, STAGES, TX, TY><<<grid, TX * TY, 0, st>>>(p, td);
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
    gemm_launch<AT, BT, 4, 4, 32, 2>(p, td, max_active, st);
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

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}

// Block = MR output rows x 64 columns (64*MR threads, one output each).
// K-tiles of 64 are staged by 16-byte cp.async into a 4-deep ring; one staged
// B tile serves all MR rows. MR=1 spreads a single chunk's few outputs over
// the most SMs (latency regime); MR=4 amortizes the B tile when many chunks
// are in flight (throughput regime).
constexpr int kNtCols = 64, kNtBK = 64, kNtStages = 4;
constexpr int kNtSB = kNtBK + 4;  // padded B row: LDS.128 of 32 rows = 4 wavefronts
__host__ __device__ constexpr size_t nt_smem(int mr) {
  return size_t(kNtStages) * (size_t(mr) * kNtBK + size_t(kNtCols) * kNtSB) * sizeof(float);
}

struct NtBatch {
  NtP p[kNtMaxProb];
  int first_block[kNtMaxProb + 1];  // prefix of row blocks per problem
  int n;
};

// VEC: rows 16-byte aligned, K multiple of 4 (host-checked); else 4-byte copies.
template <bool VEC, int MR>
__global__ void __launch_bounds__(kNtCols * MR) k_gemm_nt(NtBatch nb, const TickDesc* __restrict__ td) {
  extern __shared__ __align__(128) float sm[];
  constexpr int NT = kNtCols * MR;
  if (blockIdx.z >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.z];
  int prob = 0;
  while (prob + 1 < nb.n && int(blockIdx.y) >= nb.first_block[prob + 1]) ++prob;
  const NtP& pp = nb.p[prob];
  const int mb = int(blockIdx.y) - nb.first_block[prob];
  const float* Ab = pp.A;
  const float* Bb = pp.B;
  float* Cb = pp.C;
  float* CBb = pp.cb;
  const int64_t a_cs = pp.a_cs, b_cs = pp.b_cs, c_cs = pp.c_cs, lda = pp.lda, ldb = pp.ldb,
                ldc = pp.ldc;
  const int M = pp.M, N = pp.N, K = pp.K;
  const int m0 = mb * MR;
  if (m0 > M) return;
  const int n0 = blockIdx.x * kNtCols;
  if (n0 >= N) return;
  const int tid = threadIdx.x, col = tid % kNtCols, mr = tid / kNtCols;
  const int m = m0 + mr, n = n0 + col;
  const bool ones = m == M;      // bias row: plain sum of the gradient rows
  const bool live = m <= M && n < N;
  const int nrows = min(kNtCols, N - n0);
  const int arows = min(MR, M - m0);  // real A rows in this block (bias row has none)
  const float* A = Ab + c * a_cs + int64_t(m0) * lda;
  const float* B = Bb + c * b_cs + int64_t(n0) * ldb;
  float* C = Cb + c * c_cs;
  float* As = sm;                                  // [stage][MR][BK]
  float* Bs = sm + kNtStages * MR * kNtBK;         // [stage][64][SB]
  const int ntiles = (K + kNtBK - 1) / kNtBK;

  auto load = [&](int tile) {
    if (tile < ntiles) {
      const int st = tile % kNtStages, k0 = tile * kNtBK, kc = min(kNtBK, K - k0);
      float* as = As + st * MR * kNtBK;
      float* bs = Bs + st * kNtCols * kNtSB;
      if (VEC && kc == kNtBK) {
        for (int i = tid; i < arows * 16; i += NT)
          cp_async16(as + (i >> 4) * kNtBK + 4 * (i & 15), A + int64_t(i >> 4) * lda + k0 + 4 * (i & 15));
        for (int i = tid; i < nrows * 16; i += NT)
          cp_async16(bs + (i >> 4) * kNtSB + 4 * (i & 15), B + int64_t(i >> 4) * ldb + k0 + 4 * (i & 15));
      } else {
        for (int i = tid; i < arows * kc; i += NT)
          cp_async4(as + (i / kc) * kNtBK + i % kc, A + int64_t(i / kc) * lda + k0 + i % kc);
        for (int i = tid; i < nrows * kc; i += NT)
          cp_async4(bs + (i / kc) * kNtSB + i % kc, B + int64_t(i / kc) * ldb + k0 + i % kc);
      }
    }
    cp_async_commit();  // one group per tile slot, possibly empty
  };

  float* out = live ? ((ones && CBb) ? CBb + c * c_cs + n : C + int64_t(m) * ldc + n) : nullptr;
  float acc = live ? *out : 0.0f;
#pragma unroll
  for (int s = 0; s < kNtStages - 1; ++s) load(s);
  for (int tile = 0; tile < ntiles; ++tile) {
    cp_async_wait<kNtStages - 2>();
    __syncthreads();  // tile landed for everyone; everyone is past tile-1
    load(tile + kNtStages - 1);
    const int st = tile % kNtStages, kc = min(kNtBK, K - tile * kNtBK);
    const float* as = As + (st * MR + mr) * kNtBK;
    const float* bs = Bs + (st * kNtCols + col) * kNtSB;
    if (live) {
      if (kc == kNtBK) {
        if (ones) {
#pragma unroll
          for (int kk = 0; kk < kNtBK; kk += 4) {
            const float4 b = *reinterpret_cast<const float4*>(bs + kk);
            acc = fadd(acc, b.x);  // 1.0f * b == b exactly
            acc = fadd(acc, b.y);
            acc = fadd(acc, b.z);
            acc = fadd(acc, b.w);
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < kNtBK; kk += 4) {
            const float4 a = *reinterpret_cast<const float4*>(as + kk);
            const float4 b = *reinterpret_cast<const float4*>(bs + kk);
            acc = mac(acc, a.x, b.x);
            acc = mac(acc, a.y, b.y);
            acc = mac(acc, a.z, b.z);
            acc = mac(acc, a.w, b.w);
          }
        }
      } else {
        for (int kk = 0; kk < kc; ++kk) acc = ones ? fadd(acc, bs[kk]) : mac(acc, as[kk], bs[kk]);
      }
    }
  }
  cp_async_wait<0>();
  if (live) *out = acc;
}

// ------------------------------------------------------------------ embed
// x = emb[tok] + pos written feature-major xT[E][R*T] (the K/V projections and
// their weight gradients read it by feature), plus the last-position rows
// xl[R][E] for the query projection.
__global__ void k_embed(const uint32_t* __restrict__ tokens, ChunkGeo geo,
                        const float* __restrict__ params, int64_t p_cs, int64_t off_emb,
                        int64_t off_pos, uint32_t* ctx, int64_t ctx_cs, float* xT, int64_t x_cs,
                        float* xl, int64_t xl_cs, DmDims d, const TickDesc* __restrict__ td) {
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int64_t RT = int64_t(d.R) * d.T;
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // = j*RT + rt
  if (idx >= RT * d.E) return;
  const int64_t rt = idx % RT;
  const int j = int(idx / RT);
  const int t = int(rt % d.T), r = int(rt / d.T);
  const uint64_t L = geo.L[c];
  const uint64_t jstep = uint64_t(d.T) + uint64_t(td->tick - geo.offset[c]);  // coded position
  // tokens are < V = 4^k by construction; the mask only guards memory after a
  // decode error (slots past a truncated codestream are never written)
  const uint32_t tok = tokens[geo.start[c] + uint64_t(r) * L + (jstep - d.T) + t] & uint32_t(d.V - 1);
  if (j == 0) ctx[c * ctx_cs + rt] = tok;
  const float* P = params + c * p_cs;
  const float xv = fadd(P[off_emb + int64_t(tok) * d.E + j], P[off_pos + int64_t(t) * d.E + j]);
  xT[c * x_cs + idx] = xv;
  if (t == d.T - 1) xl[c * xl_cs + int64_t(r) * d.E + j] = xv;
}

// ------------------------------------------------------------------ attention
// One warp per (row, head). Scores and the softmax sum use chains that every
// lane evaluates redundantly in reference order (shuffle-fed), so no lane has
// to broadcast a result.
__global__ void k_attn_fwd(const float* __restrict__ q, const float* __restrict__ k,
                           const float* __restrict__ v, float* wts, float* cx, int64_t cs_q,
                           int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
                           const TickDesc* __restrict__ td) {
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

__device__ __forceinline__ void stage_rows(float* dst, const float* src, int T, int H) {
  // src [T][H] contiguous (H multiple of 4) -> dst rows of H+4
  const int nv = T * (H / 4);
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    const int t = i / (H / 4), v4 = i % (H / 4);
    *reinterpret_cast<float4*>(dst + t * (H + 4) + 4 * v4) =
        __ldg(reinterpret_cast<const float4*>(src + int64_t(t) * H + 4 * v4));
  }
}

__global__ void __launch_bounds__(kRowThreads) k_attn_fwd_row(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    float* wts, float* cx, int64_t cs_q, int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
    const TickDesc* __restrict__ td) {
  extern __shared__ __align__(128) float sm[];
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int r = blockIdx.x, T = d.T, H = d.H, HD = H / d.NH, HP = H + 4;
  const int h = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* Ks = sm;
  float* Vs = Ks + T * HP;
  float* Ws = Vs + T * HP;   // [NH][T]
  float* Qs = Ws + d.NH * T; // [H]
  const int64_t ko = c * cs_kv + int64_t(r) * T * H;
  stage_rows(Ks, k + ko, T, H);
  stage_rows(Vs, v + ko, T, H);
  for (int i = threadIdx.x; i < H; i += blockDim.x) Qs[i] = q[c * cs_q + int64_t(r) * H + i];
  __syncthreads();
  if (h >= d.NH) return;
  const float* qh = Qs + h * HD;
  float* wrow = Ws + h * T;
  float mx = -__int_as_float(0x7f800000);
  for (int t = lane; t < T; t += 32) {
    const float* kr = Ks + t * HP + h * HD;
    float s = 0.0f;
    for (int dd = 0; dd < HD; ++dd) s = mac(s, qh[dd], kr[dd]);
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
  __syncwarp();
  if (lane < HD) {
    float acc = 0.0f;
    for (int t = 0; t < T; ++t) acc = mac(acc, wrow[t], Vs[t * HP + h * HD + lane]);
    cx[c * cs_q + int64_t(r) * H + h * HD + lane] = acc;
  }
}

__global__ void __launch_bounds__(kRowThreads) k_attn_bwd_row(
    const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
    const float* __restrict__ wts, const float* __restrict__ dctx, float* dq, float* dkT,
    float* dvT, int64_t cs_q, int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
    const TickDesc* __restrict__ td) {
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
  const int64_t ko = c * cs_kv + int64_t(r) * T * H;
  stage_rows(Ks, k + ko, T, H);
  stage_rows(Vs, v + ko, T, H);
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    Qs[i] = q[c * cs_q + int64_t(r) * H + i];
    Cs[i] = dctx[c * cs_q + int64_t(r) * H + i];
  }
  __syncthreads();
  if (h >= d.NH) return;
  const float* w = wts + c * cs_w + (int64_t(r) * d.NH + h) * T;
  const float* dc = Cs + h * HD;
  const int64_t to = c * cs_kv + int64_t(h) * HD * RT + int64_t(r) * T;  // feature-major dk, dv
  float* dsw = Ds + h * T;
  // dv_t[d] = 0 + w_t*dc[d]; dwt_t = sum_d dc[d]*v_t[d]; dot = sum_t w_t*dwt_t
  float dot = 0.0f;
  for (int t0 = 0; t0 < T; t0 += 32) {
    const int t = t0 + lane;
    float prod = 0.0f;
    if (t < T) {
      const float wt = w[t];
      const float* vr = Vs + t * HP + h * HD;
      float acc = 0.0f;
      for (int dd = 0; dd < HD; ++dd) {
        dvT[to + int64_t(dd) * RT + t] = fadd(0.0f, fmul(wt, dc[dd]));
        acc = mac(acc, dc[dd], vr[dd]);
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
    for (int dd = 0; dd < HD; ++dd) dkT[to + int64_t(dd) * RT + t] = fadd(0.0f, fmul(ds, Qs[h * HD + dd]));
  }
  __syncwarp();
  // dq[d] = 0 + sum_t ds_t*k_t[d]
  if (lane < HD) {
    float acc = 0.0f;
    for (int t = 0; t < T; ++t) acc = mac(acc, dsw[t], Ks[t * HP + h * HD + lane]);
    dq[c * cs_q + int64_t(r) * H + h * HD + lane] = acc;
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
// the vocabulary fit in shared memory): stable counting sort of the positions
// by token (histogram, scan, warp match-any ranks keep (r,t) order), then one
// thread per (token, column) walks its contiguous list in order with 16 loads
// in flight. Same per-element order as Embedding::backward (layers.cpp:117-125).
constexpr int kSortThreads = 1024;
constexpr int kSortMaxPos = 10240;
constexpr int kSortMaxV = 256;
__global__ void __launch_bounds__(kSortThreads) k_emb_bwd_sorted(
    const uint32_t* __restrict__ ctx, int64_t ctx_cs, const float* __restrict__ dx, int64_t dx_cs,
    const float* __restrict__ dxl, int64_t dxl_cs, float* grads, int64_t g_cs, int64_t off_emb,
    DmDims d, const TickDesc* __restrict__ td) {
  __shared__ uint16_t sorted[kSortMaxPos];
  __shared__ int cnt[kSortMaxV], off[kSortMaxV + 1], run[kSortMaxV];
  __shared__ uint16_t wc[32][kSortMaxV];  // per-warp counts of each token in the current slab
  if (blockIdx.x >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int V = d.V, RT = d.R * d.T;
  const uint32_t* cp = ctx + c * ctx_cs;
  for (int v = tid; v < V; v += kSortThreads) {
    cnt[v] = 0;
    run[v] = 0;
  }
  __syncthreads();
  for (int p = tid; p < RT; p += kSortThreads) atomicAdd(&cnt[cp[p]], 1);
  __syncthreads();
  if (tid == 0) {
    int a = 0;
    for (int v = 0; v < V; ++v) {
      off[v] = a;
      a += cnt[v];
    }
    off[V] = a;
  }
  __syncthreads();
  for (int base = 0; base < RT; base += kSortThreads) {
    for (int i = tid; i < 32 * V; i += kSortThreads) wc[i / V][i % V] = 0;
    __syncthreads();
    const int p = base + tid;
    const bool ok = p < RT;
    const uint32_t v = ok ? cp[p] : 0xffffffffu;
    const unsigned mask = __match_any_sync(0xffffffffu, v);
    const int rank_w = __popc(mask & ((1u << lane) - 1u));
    if (ok && rank_w == 0) wc[w][v] = uint16_t(__popc(mask));
    __syncthreads();
    if (ok) {
      int before = 0;
      for (int ww = 0; ww < w; ++ww) before += wc[ww][v];
      sorted[off[v] + run[v] + before + rank_w] = uint16_t(p);
    }
    __syncthreads();
    for (int vv = tid; vv < V; vv += kSortThreads) {
      int tot = 0;
      for (int ww = 0; ww < 32; ++ww) tot += wc[ww][vv];
      run[vv] += tot;
    }
    __syncthreads();
  }
  const float* xp = dx + c * dx_cs;
  const float* lp = dxl ? dxl + c * dxl_cs : nullptr;
  for (int o = tid; o < V * d.E; o += kSortThreads) {
    const int v = o / d.E, j = o % d.E;
    float* g = grads + c * g_cs + off_emb + o;
    float acc = *g;
    const int b0 = off[v], b1 = off[v + 1];
    constexpr int kB = 16;
    for (int h0 = b0; h0 < b1; h0 += kB) {
      float x[kB];
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const int h = h0 + b < b1 ? h0 + b : b0;
        const int pp = sorted[h];
        float val = __ldg(xp + int64_t(pp) * d.E + j);
        if (lp && pp % d.T == d.T - 1) val = fadd(val, __ldg(lp + int64_t(pp / d.T) * d.E + j));
        x[b] = val;
      }
#pragma unroll
      for (int b = 0; b < kB; ++b)
        if (h0 + b < b1) acc = fadd(acc, x[b]);
    }
    *g = acc;
  }
}

// ------------------------------------------------------------------ Adam
__global__ void k_adam(float* __restrict__ w, float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, int64_t p_cs, int64_t n,
                       const AdamScalars* __restrict__ sc, const TickDesc* __restrict__ td) {
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const float bc1 = sc[c].bc1, bc2 = sc[c].bc2;
  const float b1 = 0.9f, b2 = 0.999f, lr = 5e-4f, eps = 1e-8f;
  const float omb1 = fsub(1.0f, b1), omb2 = fsub(1.0f, b2);
  const int64_t base = c * p_cs;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = base + i;
    const float gi = g[o];
    const float mi = fadd(fmul(b1, m[o]), fmul(omb1, gi));
    const float vi = fadd(fmul(b2, v[o]), fmul(fmul(omb2, gi), gi));
    const float mhat = fdiv(mi, bc1);
    const float vhat = fdiv(vi, bc2);
    w[o] = fsub(w[o], fdiv(fmul(lr, mhat), fadd(__fsqrt_rn(vhat), eps)));
    m[o] = mi;
    v[o] = vi;
    g[o] = 0.0f;
  }
}

__global__ void k_state_copy(float* w, float* m, float* v, AdamScalars* sc, int64_t p_cs, int64_t n,
                             const TickDesc* __restrict__ td) {
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
                               const int* __restrict__ act_all, const uint32_t* __restrict__ hand_ptr,
                               const int2* __restrict__ hand_all, int64_t ticks) {
  const int64_t t = td->tick + 1;
  td->tick = t;
  if (t < ticks) {
    td->act = act_all + act_ptr[t];
    td->n_act = int(act_ptr[t + 1] - act_ptr[t]);
    td->hand = hand_all + hand_ptr[t];
    td->n_hand = int(hand_ptr[t + 1] - hand_ptr[t]);
  } else {
    td->n_act = 0;
    td->n_hand = 0;
  }
}

}  // namespace

void launch_gemm(const GemmP& p, bool at, bool bt, const TickDesc* td, int max_active,
                 cudaStream_t st) {
  if (max_active <= 0 || p.N <= 0 || p.M + p.ones_row <= 0) return;
  if (at && bt) gemm_dispatch<true, true>(p, td, max_active, st);
  else if (at) gemm_dispatch<true, false>(p, td, max_active, st);
  else if (bt) gemm_dispatch<false, true>(p, td, max_active, st);
  else gemm_dispatch<false, false>(p, td, max_active, st);
}

void launch_gemm_nt_batch(const NtP* probs, int nprob, const TickDesc* td, int max_active,
                          cudaStream_t st) {
  if (max_active <= 0 || nprob <= 0) return;
  auto al = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
  bool vec = true;
  int maxn = 0;
  for (int i = 0; i < nprob; ++i) {
    const NtP& p = probs[i];
    vec = vec && p.K % 4 == 0 && p.lda % 4 == 0 && p.ldb % 4 == 0 && p.a_cs % 4 == 0 &&
          p.b_cs % 4 == 0 && al(p.A) && al(p.B);
    maxn = std::max(maxn, p.N);
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gemm_nt<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(nt_smem(1)));
    cudaFuncSetAttribute(k_gemm_nt<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(nt_smem(1)));
    cudaFuncSetAttribute(k_gemm_nt<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(nt_smem(4)));
    cudaFuncSetAttribute(k_gemm_nt<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(nt_smem(4)));
    attr_set = true;
  }
  const int nx = (maxn + kNtCols - 1) / kNtCols;
  auto build = [&](int mr, NtBatch& nb) {
    nb.n = nprob;
    nb.first_block[0] = 0;
    for (int i = 0; i < nprob; ++i) {
      nb.p[i] = probs[i];
      nb.first_block[i + 1] = nb.first_block[i] + (probs[i].M + 1 + mr - 1) / mr;
    }
    return nb.first_block[nprob];
  };
  NtBatch nb;
  const int rows1 = build(1, nb);
  // one-row blocks while the launch cannot fill the chip, else 4-row blocks
  if (int64_t(nx) * rows1 * max_active < 2 * 148) {
    dim3 grid(nx, rows1, max_active);
    if (vec) k_gemm_nt<true, 1><<<grid, kNtCols, nt_smem(1), st>>>(nb, td);
    else k_gemm_nt<false, 1><<<grid, kNtCols, nt_smem(1), st>>>(nb, td);
  } else {
    const int rows4 = build(4, nb);
    dim3 grid(nx, rows4, max_active);
    if (vec) k_gemm_nt<true, 4><<<grid, kNtCols * 4, nt_smem(4), st>>>(nb, td);
    else k_gemm_nt<false, 4><<<grid, kNtCols * 4, nt_smem(4), st>>>(nb, td);
  }
}

void launch_gemm_nt(const NtP& p0, const NtP* p1, const TickDesc* td, int max_active,
                    cudaStream_t st) {
  NtP ps[2] = {p0, p1 ? *p1 : p0};
  launch_gemm_nt_batch(ps, p1 ? 2 : 1, td, max_active, st);
}

void launch_embed(const uint32_t* tokens, ChunkGeo geo, const float* params,
                  int64_t p_cs, int64_t off_emb, int64_t off_pos, uint32_t* ctx, int64_t ctx_cs,
                  float* x, int64_t x_cs, float* xl, int64_t xl_cs, DmDims d, const TickDesc* td,
                  int max_active, cudaStream_t st) {
  if (max_active <= 0) return;
  const int64_t total = int64_t(d.R) * d.T * d.E;
  dim3 grid(unsigned((total + 255) / 256), max_active);
  k_embed<<<grid, 256, 0, st>>>(tokens, geo, params, p_cs, off_emb, off_pos, ctx, ctx_cs, x,
                                x_cs, xl, xl_cs, d, td);
}

void launch_attn_fwd(const float* q, const float* k, const float* v, float* wts, float* cx,
                     int64_t cs_q, int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
                     const TickDesc* td, int max_active, cudaStream_t st) {
  if (max_active <= 0) return;
  const size_t smem = attn_row_smem(d);
  if (d.NH <= 8 && d.H % 4 == 0 && smem <= 200 * 1024) {
    static size_t attr = 0;
    if (smem > attr) {
      cudaFuncSetAttribute(k_attn_fwd_row, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      attr = smem;
    }
    k_attn_fwd_row<<<dim3(d.R, max_active), kRowThreads, smem, st>>>(q, k, v, wts, cx, cs_q, cs_kv,
                                                                      cs_w, d, inv, td);
    return;
  }
  const int64_t warps = int64_t(d.R) * d.NH;
  dim3 grid(unsigned((warps * 32 + 255) / 256), max_active);
  k_attn_fwd<<<grid, 256, 0, st>>>(q, k, v, wts, cx, cs_q, cs_kv, cs_w, d, inv, td);
}

void launch_attn_bwd(const float* q, const float* k, const float* v, const float* wts,
                     const float* dctx, float* dq, float* dk, float* dv, int64_t cs_q,
                     int64_t cs_kv, int64_t cs_w, DmDims d, float inv, const TickDesc* td,
                     int max_active, cudaStream_t st) {
  if (max_active <= 0) return;
  const size_t smem = attn_row_smem(d) + d.H * sizeof(float);
  if (d.NH <= 8 && d.H % 4 == 0 && smem <= 200 * 1024) {
    static size_t attr = 0;
    if (smem > attr) {
      cudaFuncSetAttribute(k_attn_bwd_row, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      attr = smem;
    }
    k_attn_bwd_row<<<dim3(d.R, max_active), kRowThreads, smem, st>>>(
        q, k, v, wts, dctx, dq, dk, dv, cs_q, cs_kv, cs_w, d, inv, td);
    return;
  }
  const int64_t warps = int64_t(d.R) * d.NH;
  dim3 grid(unsigned((warps * 32 + 255) / 256), max_active);
  k_attn_bwd<<<grid, 256, 0, st>>>(q, k, v, wts, dctx, dq, dk, dv, cs_q, cs_kv, cs_w, d, inv,
                                   td);
}

void launch_emb_grad(const uint32_t* ctx, int64_t ctx_cs, const float* dx, int64_t dx_cs,
                     float* grads, int64_t g_cs, int64_t off_emb, DmDims d, const TickDesc* td,
                     int max_active, cudaStream_t st) {
  if (max_active <= 0) return;
  if (d.R * d.T <= kSortMaxPos && d.V <= kSortMaxV) {
    k_emb_bwd_sorted<<<max_active, kSortThreads, 0, st>>>(ctx, ctx_cs, dx, dx_cs, nullptr, 0, grads,
                                                         g_cs, off_emb, d, td);
    return;
  }
  dim3 g2(unsigned((d.V + kEmbWarps - 1) / kEmbWarps), max_active);
  k_emb_bwd<<<g2, kEmbWarps * 32, 0, st>>>(ctx, ctx_cs, dx, dx_cs, nullptr, 0, grads, g_cs, off_emb,
                                           d, td);
}

void launch_embed_bwd(const uint32_t* ctx, int64_t ctx_cs, const float* dx, int64_t dx_cs,
                      const float* dxl, int64_t dxl_cs, float* grads, int64_t g_cs,
                      int64_t off_emb, int64_t off_pos, DmDims d, const TickDesc* td, int max_active,
                      cudaStream_t st) {
  if (max_active <= 0) return;
  dim3 g1(unsigned((d.T * d.E + 255) / 256), max_active);
  k_pos_bwd<<<g1, 256, 0, st>>>(dx, dx_cs, dxl, dxl_cs, grads, g_cs, off_pos, d, td);
  dim3 g2(unsigned((d.V + kEmbWarps - 1) / kEmbWarps), max_active);
  k_emb_bwd<<<g2, kEmbWarps * 32, 0, st>>>(ctx, ctx_cs, dx, dx_cs, dxl, dxl_cs, grads, g_cs, off_emb, d,
                                td);
}

void launch_adam(float* w, float* g, float* m, float* v, int64_t p_cs, int64_t n,
                 const AdamScalars* sc, const TickDesc* td, int max_active, cudaStream_t st) {
  if (max_active <= 0 || n <= 0) return;
  const int64_t per = (n + 255) / 256;
  dim3 grid(unsigned(per < 64 ? per : 64), max_active);
  k_adam<<<grid, 256, 0, st>>>(w, g, m, v, p_cs, n, sc, td);
}

void launch_state_copy(float* w, float* m, float* v, AdamScalars* sc, int64_t p_cs, int64_t n,
                       const TickDesc* td, int max_pairs, cudaStream_t st) {
  if (max_pairs <= 0) return;
  const int64_t per = (n + 255) / 256;
  dim3 grid(unsigned(per < 64 ? per : 64), max_pairs);
  k_state_copy<<<grid, 256, 0, st>>>(w, m, v, sc, p_cs, n, td);
}

void launch_tick_advance(TickDesc* td, const uint32_t* act_ptr, const int* act_all,
                         const uint32_t* hand_ptr, const int2* hand_all, int64_t ticks,
                         cudaStream_t st) {
  k_tick_advance<<<1, 1, 0, st>>>(td, act_ptr, act_all, hand_ptr, hand_all, ticks);
}

}  // namespace pmklc_b200
