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

template <bool AT, bool BT, int TM, int TN, int BK, int STAGES>
__global__ void __launch_bounds__(256) k_gemm_tiled(GemmP p, const int* __restrict__ active) {
  constexpr int BM = 16 * TM, BN = 16 * TN;
  __shared__ float As[STAGES][BK][BM + 4];
  __shared__ float Bs[STAGES][BK][BN + 4];
  const int c = active[blockIdx.z];
  const float* A = p.A + c * p.a_cs;
  const float* B = p.B + c * p.b_cs;
  float* C = p.C + c * p.c_cs;
  const int Mx = p.M + (p.ones_row ? 1 : 0);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int ntiles = (p.K + BK - 1) / BK;

  auto load = [&](int tile) {
    if (tile < ntiles) {
      const int stage = tile % STAGES, k0 = tile * BK;
      for (int idx = threadIdx.x; idx < BM * BK; idx += 256) {
        int mm, kk;
        if (AT) { mm = idx % BM; kk = idx / BM; }  // global contiguous in m
        else    { kk = idx % BK; mm = idx / BK; }  // global contiguous in k
        const int m = m0 + mm, k = k0 + kk;
        if (k < p.K) {
          if (m < p.M) cp_async4(&As[stage][kk][mm], AT ? A + int64_t(k) * p.lda + m : A + int64_t(m) * p.lda + k);
          else if (m == p.M && p.ones_row) As[stage][kk][mm] = 1.0f;
        }
      }
      for (int idx = threadIdx.x; idx < BN * BK; idx += 256) {
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
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      float v = 0.0f;
      if (m < Mx && n < p.N) {
        if (p.init == 1) v = p.bias[c * p.bias_cs + n];
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
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        a[i] = As[stage][kk][ty + 16 * i];
        if (relu && a[i] < 0.0f) a[i] = 0.0f;
      }
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[stage][kk][tx + 16 * j];
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
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < Mx && n < p.N) {
        float v = acc[i][j];
        if (p.mask && p.mask[c * p.mask_cs + int64_t(m) * p.ldm + n] <= 0.0f) v = 0.0f;
        C[int64_t(m) * p.ldc + n] = v;
      }
    }
}

template <bool AT, bool BT, int TM, int TN, int BK, int STAGES>
void gemm_launch(const GemmP& p, const int* active, int n_active, cudaStream_t st) {
  const int Mx = p.M + (p.ones_row ? 1 : 0);
  dim3 grid((p.N + 16 * TN - 1) / (16 * TN), (Mx + 16 * TM - 1) / (16 * TM), n_active);
  k_gemm_tiled<AT, BT, TM, TN, BK, STAGES><<<grid, 256, 0, st>>>(p, active);
}

template <bool AT, bool BT>
void gemm_dispatch(const GemmP& p, const int* active, int n_active, cudaStream_t st) {
  const int Mx = p.M + (p.ones_row ? 1 : 0);
  auto blocks = [&](int tm, int tn) {
    return int64_t((p.N + 16 * tn - 1) / (16 * tn)) * ((Mx + 16 * tm - 1) / (16 * tm)) * n_active;
  };
  // largest tile that still gives every SM at least two blocks
  constexpr int64_t kFill = 2 * 148;
  if (blocks(4, 4) >= kFill && p.N >= 48 && Mx >= 48)
    gemm_launch<AT, BT, 4, 4, 32, 2>(p, active, n_active, st);
  else if (blocks(2, 2) >= kFill && p.N >= 24 && Mx >= 24)
    gemm_launch<AT, BT, 2, 2, 32, 3>(p, active, n_active, st);
  else
    gemm_launch<AT, BT, 1, 1, 64, 4>(p, active, n_active, st);
}

// ------------------------------------------------------------------ embed
__global__ void k_embed(const uint32_t* __restrict__ tokens, ChunkGeo geo, int64_t tick,
                        const float* __restrict__ params, int64_t p_cs, int64_t off_emb,
                        int64_t off_pos, uint32_t* ctx, int64_t ctx_cs, float* x, int64_t x_cs,
                        DmDims d, const int* __restrict__ active) {
  const int c = active[blockIdx.y];
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = int64_t(d.R) * d.T * d.E;
  if (idx >= total) return;
  const int j = int(idx % d.E);
  const int64_t rt = idx / d.E;
  const int t = int(rt % d.T), r = int(rt / d.T);
  const uint64_t L = geo.L[c];
  const uint64_t jstep = uint64_t(d.T) + uint64_t(tick - geo.offset[c]);  // coded position
  const uint32_t tok = tokens[geo.start[c] + uint64_t(r) * L + (jstep - d.T) + t];
  if (j == 0) ctx[c * ctx_cs + rt] = tok;
  const float* P = params + c * p_cs;
  x[c * x_cs + idx] = fadd(P[off_emb + int64_t(tok) * d.E + j], P[off_pos + int64_t(t) * d.E + j]);
}

// ------------------------------------------------------------------ attention
// One warp per (row, head). Scores and the softmax sum use chains that every
// lane evaluates redundantly in reference order (shuffle-fed), so no lane has
// to broadcast a result.
__global__ void k_attn_fwd(const float* __restrict__ q, const float* __restrict__ k,
                           const float* __restrict__ v, float* wts, float* cx, int64_t cs_q,
                           int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
                           const int* __restrict__ active) {
  const int c = active[blockIdx.y];
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

__global__ void k_attn_bwd(const float* __restrict__ q, const float* __restrict__ k,
                           const float* __restrict__ v, const float* __restrict__ wts,
                           const float* __restrict__ dctx, float* dq, float* dk, float* dv,
                           int64_t cs_q, int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
                           const int* __restrict__ active) {
  const int c = active[blockIdx.y];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= d.R * d.NH) return;
  const int r = warp / d.NH, h = warp % d.NH, HD = d.H / d.NH, T = d.T;
  const int64_t qo = c * cs_q + int64_t(r) * d.H + h * HD;
  const int64_t ko = c * cs_kv + int64_t(r) * T * d.H + h * HD;
  const float* w = wts + c * cs_w + (int64_t(r) * d.NH + h) * T;
  const float* dc = dctx + qo;
  // dv_t[d] = 0 + w_t*dc[d];  dwt_t = sum_d dc[d]*v_t[d]
  // dot = sum_t w_t*dwt_t (sequential, all lanes redundantly)
  float dot = 0.0f;
  for (int t0 = 0; t0 < T; t0 += 32) {
    const int t = t0 + lane;
    float prod = 0.0f;
    if (t < T) {
      const float wt = w[t];
      float acc = 0.0f;
      for (int dd = 0; dd < HD; ++dd) {
        dv[ko + int64_t(t) * d.H + dd] = fadd(0.0f, fmul(wt, dc[dd]));
        acc = mac(acc, dc[dd], v[ko + int64_t(t) * d.H + dd]);
      }
      prod = fmul(wt, acc);
      dk[ko + int64_t(t) * d.H] = acc;  // stash dwt_t in dk's first slot until ds is known
    }
    const int cnt = min(32, T - t0);
    for (int i = 0; i < cnt; ++i) dot = fadd(dot, __shfl_sync(0xffffffffu, prod, i));
  }
  __syncwarp();
  // ds_t = (w_t*(dwt_t - dot))*inv;  dk_t[d] = 0 + ds_t*q[d]; stash ds_t in dwt slot first
  for (int t = lane; t < T; t += 32) {
    const float dwt = dk[ko + int64_t(t) * d.H];
    const float ds = fmul(fmul(w[t], fsub(dwt, dot)), inv);
    for (int dd = HD - 1; dd >= 0; --dd)  // slot 0 (dwt) overwritten last
      dk[ko + int64_t(t) * d.H + dd] = fadd(0.0f, fmul(ds, q[qo + dd]));
    // keep ds for the dq pass: recover as dk_t[0]/q[0] is not exact; store separately
  }
  __syncwarp();
  // dq[d] = sum_t ds_t*k_t[d]: recompute ds_t in registers per t (cheap, exact same ops)
  if (lane < HD) {
    float acc = 0.0f;
    for (int t = 0; t < T; ++t) {
      float dwt = 0.0f;
      for (int dd = 0; dd < HD; ++dd) dwt = mac(dwt, dc[dd], v[ko + int64_t(t) * d.H + dd]);
      const float ds = fmul(fmul(w[t], fsub(dwt, dot)), inv);
      acc = mac(acc, ds, k[ko + int64_t(t) * d.H + lane]);
    }
    dq[qo + lane] = acc;
  }
}

// ------------------------------------------------------------------ embed bwd
// pos grad: thread per (t, j), ascending rows, loads issued 16 rows ahead of
// the dependent adds. emb grad: warp per token value, lanes = j; positions are
// visited in (r,t) row-major order: a segment of ctx is staged in shared
// memory, each warp ballots its hits into a shared list, then walks the list
// with 16 independent dx loads in flight per batch.
__device__ __forceinline__ float dx_at(const float* xp, const float* lp, int64_t pp, int j, int T, int E) {
  float v = xp[pp * E + j];
  if (int(pp % T) == T - 1) v = fadd(v, lp[(pp / T) * E + j]);  // dx[:,last,:] += dxl (layers.cpp:521)
  return v;
}

__global__ void k_pos_bwd(const float* __restrict__ dx, int64_t dx_cs, const float* __restrict__ dxl,
                          int64_t dxl_cs, float* grads, int64_t g_cs, int64_t off_pos, DmDims d,
                          const int* __restrict__ active) {
  const int c = active[blockIdx.y];
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
  for (int r0 = 0; r0 < d.R; r0 += kB) {
    float v[kB];
    const int cnt = min(kB, d.R - r0);
#pragma unroll
    for (int q = 0; q < kB; ++q)
      if (q < cnt) {
        v[q] = xp[(r0 + q) * rs];
        if (last) v[q] = fadd(v[q], lp[int64_t(r0 + q) * d.E]);
      }
#pragma unroll
    for (int q = 0; q < kB; ++q)
      if (q < cnt) acc = fadd(acc, v[q]);
  }
  *g = acc;
}

constexpr int kEmbWarps = 8;
constexpr int kEmbSeg = 2048;

__global__ void __launch_bounds__(kEmbWarps * 32) k_emb_bwd(
    const uint32_t* __restrict__ ctx, int64_t ctx_cs, const float* __restrict__ dx, int64_t dx_cs,
    const float* __restrict__ dxl, int64_t dxl_cs, float* grads, int64_t g_cs, int64_t off_emb,
    DmDims d, const int* __restrict__ active) {
  __shared__ uint32_t sctx[kEmbSeg];
  __shared__ uint16_t hits[kEmbWarps][kEmbSeg];
  const int c = active[blockIdx.y];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tokv = blockIdx.x * kEmbWarps + wl;
  const uint32_t* cp = ctx + c * ctx_cs;
  const float* xp = dx + c * dx_cs;
  const float* lp = dxl + c * dxl_cs;
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
        if (q >= nj || j >= d.E) break;
        float v[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b)
          if (b < cnt) v[b] = dx_at(xp, lp, s0 + hits[wl][h0 + b], j, d.T, d.E);
#pragma unroll
        for (int b = 0; b < kB; ++b)
          if (b < cnt) acc[q] = fadd(acc[q], v[b]);
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

// ------------------------------------------------------------------ Adam
__global__ void k_adam(float* __restrict__ w, float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, int64_t p_cs, int64_t n,
                       const AdamScalars* __restrict__ sc, const int* __restrict__ active) {
  const int c = active[blockIdx.y];
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
                             const int2* __restrict__ pairs) {
  const int2 pr = pairs[blockIdx.y];  // x = src, y = dst
  const int64_t so = pr.x * p_cs, dof = pr.y * p_cs;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    w[dof + i] = w[so + i];
    m[dof + i] = m[so + i];
    v[dof + i] = v[so + i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[pr.y] = sc[pr.x];
}

}  // namespace

void launch_gemm(const GemmP& p, bool at, bool bt, const int* active, int n_active,
                 cudaStream_t st) {
  if (n_active <= 0 || p.N <= 0 || p.M + p.ones_row <= 0) return;
  if (at && bt) gemm_dispatch<true, true>(p, active, n_active, st);
  else if (at) gemm_dispatch<true, false>(p, active, n_active, st);
  else if (bt) gemm_dispatch<false, true>(p, active, n_active, st);
  else gemm_dispatch<false, false>(p, active, n_active, st);
}

void launch_embed(const uint32_t* tokens, ChunkGeo geo, int64_t tick, const float* params,
                  int64_t p_cs, int64_t off_emb, int64_t off_pos, uint32_t* ctx, int64_t ctx_cs,
                  float* x, int64_t x_cs, DmDims d, const int* active, int n_active,
                  cudaStream_t st) {
  if (n_active <= 0) return;
  const int64_t total = int64_t(d.R) * d.T * d.E;
  dim3 grid(unsigned((total + 255) / 256), n_active);
  k_embed<<<grid, 256, 0, st>>>(tokens, geo, tick, params, p_cs, off_emb, off_pos, ctx, ctx_cs, x,
                                x_cs, d, active);
}

void launch_attn_fwd(const float* q, const float* k, const float* v, float* wts, float* cx,
                     int64_t cs_q, int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
                     const int* active, int n_active, cudaStream_t st) {
  if (n_active <= 0) return;
  const int64_t warps = int64_t(d.R) * d.NH;
  dim3 grid(unsigned((warps * 32 + 255) / 256), n_active);
  k_attn_fwd<<<grid, 256, 0, st>>>(q, k, v, wts, cx, cs_q, cs_kv, cs_w, d, inv, active);
}

void launch_attn_bwd(const float* q, const float* k, const float* v, const float* wts,
                     const float* dctx, float* dq, float* dk, float* dv, int64_t cs_q,
                     int64_t cs_kv, int64_t cs_w, DmDims d, float inv, const int* active,
                     int n_active, cudaStream_t st) {
  if (n_active <= 0) return;
  const int64_t warps = int64_t(d.R) * d.NH;
  dim3 grid(unsigned((warps * 32 + 255) / 256), n_active);
  k_attn_bwd<<<grid, 256, 0, st>>>(q, k, v, wts, dctx, dq, dk, dv, cs_q, cs_kv, cs_w, d, inv,
                                   active);
}

void launch_embed_bwd(const uint32_t* ctx, int64_t ctx_cs, const float* dx, int64_t dx_cs,
                      const float* dxl, int64_t dxl_cs, float* grads, int64_t g_cs,
                      int64_t off_emb, int64_t off_pos, DmDims d, const int* active, int n_active,
                      cudaStream_t st) {
  if (n_active <= 0) return;
  dim3 g1(unsigned((d.T * d.E + 255) / 256), n_active);
  k_pos_bwd<<<g1, 256, 0, st>>>(dx, dx_cs, dxl, dxl_cs, grads, g_cs, off_pos, d, active);
  dim3 g2(unsigned((d.V + kEmbWarps - 1) / kEmbWarps), n_active);
  k_emb_bwd<<<g2, kEmbWarps * 32, 0, st>>>(ctx, ctx_cs, dx, dx_cs, dxl, dxl_cs, grads, g_cs, off_emb, d,
                                active);
}

void launch_adam(float* w, float* g, float* m, float* v, int64_t p_cs, int64_t n,
                 const AdamScalars* sc, const int* active, int n_active, cudaStream_t st) {
  if (n_active <= 0 || n <= 0) return;
  const int64_t per = (n + 255) / 256;
  dim3 grid(unsigned(per < 64 ? per : 64), n_active);
  k_adam<<<grid, 256, 0, st>>>(w, g, m, v, p_cs, n, sc, active);
}

void launch_state_copy(float* w, float* m, float* v, AdamScalars* sc, int64_t p_cs, int64_t n,
                       const int2* pairs, int n_pairs, cudaStream_t st) {
  if (n_pairs <= 0) return;
  const int64_t per = (n + 255) / 256;
  dim3 grid(unsigned(per < 64 ? per : 64), n_pairs);
  k_state_copy<<<grid, 256, 0, st>>>(w, m, v, sc, p_cs, n, pairs);
}

}  // namespace pmklc_b200
