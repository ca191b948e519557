// SPrM pre-pass on sm_100a: one-layer BiGRU training pass (train_pass,
// core/src/training.cpp:8-41) — forward with tape, det_softmax + CE grad,
// backward through time (Gru::backward, layers.cpp:262-327; BiGru::backward,
// 369-387; BiGruModel::backward, models.cpp:75-96) and Adam, one launch
// sequence per batch of `bs` rows, strictly sequential across batches.
//
// Layouts (d = direction, t = the GRU's own time, r = row, j/q = unit):
//   tape r,z,n,hh,out : [2][T][R][H]
//   feature-major reduction operands, k = (T-1-t)*R + r so that ascending k
//   is the reference's accumulation order (t descending, rows ascending):
//   G{an,ar,az,hh}[d][j][k], HP[d][q][k] (h_{t-1}), X[d][i][k] (GRU input)
#include <algorithm>
#include <cstdint>

#include "detmath.cuh"
#include "kernels.hpp"
#include "launch.cuh"

namespace pmklc_b200 {

namespace {

enum { WIR, WIZ, WIN, WHR, WHZ, WHN, BIR, BIZ, BIN, BHR, BHZ, BHN, NG };
__device__ __forceinline__ int64_t goff(const int64_t* offs, int dir, int t) {
  return offs[1 + dir * NG + t];
}

// contexts of the batch at position p: ctx[r][i] = tok[p + r - T + i]; also
// the GRU inputs X[d][i][k] and the per-token layer-0 projection table.
__global__ void k_sprm_prep(const uint32_t* __restrict__ tokens, const int64_t* __restrict__ pos,
                            SprmP s, uint32_t* ctx, float* X, float* tab) {
  pdl_wait();
  const int64_t p = *pos;
  const int R = s.R, T = s.T, Es = s.Es, H = s.H, V = s.V;
  const int64_t RT = int64_t(R) * T;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const float* W = s.w;
  if (tid < RT) {
    const int r = int(tid / T), i = int(tid % T);
    ctx[tid] = tokens[p + r - T + i];
  }
  // table[d][g][tok][j] = b_ig[j] + sum_p emb[tok][p] W_ig[p][j]
  const int64_t ntab = int64_t(2) * 3 * V * H;
  if (tid < ntab) {
    const int j = int(tid % H);
    const int64_t rest = tid / H;
    const int tok = int(rest % V), dg = int(rest / V), d = dg / 3, g = dg % 3;
    const float* Wg = W + goff(s.offs, d, WIR + g);
    float acc = W[goff(s.offs, d, BIR + g) + j];
    const float* e = W + s.offs[0] + int64_t(tok) * Es;
    for (int q = 0; q < Es; ++q) acc = mac(acc, e[q], Wg[int64_t(q) * H + j]);
    tab[tid] = acc;
  }
  // X[d][i][k]: fwd input at its time t is x[r][t]; bwd's is x[r][T-1-t]
  const int64_t nx = int64_t(2) * Es * RT;
  if (tid < nx) {
    const int64_t k = tid % RT;
    const int64_t rest = tid / RT;
    const int i = int(rest % Es), d = int(rest / Es);
    const int tt = int(T - 1 - k / R), r = int(k % R);  // own time t = T-1-k/R
    const int src_t = d ? (T - 1 - tt) : tt;
    const uint32_t tok = tokens[p + r - T + src_t];
    X[tid] = W[s.offs[0] + int64_t(tok) * Es + i];
  }
}

// forward recurrence with tape; warp per (row, dir), lane = unit (H <= 32)
__global__ void __launch_bounds__(256) k_sprm_fwd(SprmP s, const uint32_t* __restrict__ ctx,
                                                  const float* __restrict__ tab, float* tape,
                                                  float* fin) {
  pdl_wait();
  __shared__ __align__(16) float sh[8][2][32];
  __shared__ float sw[3][32][32];  // [gate][q][j] = W_h{r,z,n}[q][j]
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = blockIdx.x & 1;
  const int r = (blockIdx.x >> 1) * 8 + wl;
  const int T = s.T, H = s.H, R = s.R, V = s.V;
  const float* W = s.w;
  for (int i = threadIdx.x; i < 3 * H * H; i += blockDim.x) {
    const int gate = i / (H * H), rem = i % (H * H);
    sw[gate][rem / H][rem % H] = W[goff(s.offs, d, WHR + gate) + rem];
  }
  __syncthreads();
  if (r >= R) return;
  const bool act = lane < H;
  const int j = act ? lane : 0;
  const float bhr = W[goff(s.offs, d, BHR) + j], bhz = W[goff(s.offs, d, BHZ) + j],
              bhn = W[goff(s.offs, d, BHN) + j];
  const float* t0 = tab + int64_t(d) * 3 * V * H;
  const int64_t TRH = int64_t(T) * R * H;
  float* tr = tape + (int64_t(0 * 2 + d) * TRH);
  float* tz = tape + (int64_t(1 * 2 + d) * TRH);
  float* tn = tape + (int64_t(2 * 2 + d) * TRH);
  float* th = tape + (int64_t(3 * 2 + d) * TRH);
  float* to = tape + (int64_t(4 * 2 + d) * TRH);
  if (act) sh[wl][0][j] = 0.0f;
  __syncwarp();
  int cur = 0;
  for (int t = 0; t < T; ++t) {
    const int src_t = d ? (T - 1 - t) : t;
    const int64_t tok = ctx[int64_t(r) * T + src_t];
    const float* h = sh[wl][cur];
    float ar = fadd(t0[tok * H + j], bhr);
    for (int q = 0; q < H; ++q) ar = mac(ar, h[q], sw[0][q][j]);
    float az = fadd(t0[int64_t(V) * H + tok * H + j], bhz);
    for (int q = 0; q < H; ++q) az = mac(az, h[q], sw[1][q][j]);
    float hh = bhn;
    for (int q = 0; q < H; ++q) hh = mac(hh, h[q], sw[2][q][j]);
    const float an = t0[2 * int64_t(V) * H + tok * H + j];
    const float rv = det_sigmoid(ar), zv = det_sigmoid(az);
    const float nv = det_tanh(fadd(an, fmul(rv, hh)));
    const float hv = fadd(fmul(fsub(1.0f, zv), nv), fmul(zv, h[j]));
    if (act) {
      const int64_t o = (int64_t(t) * R + r) * H + j;
      tr[o] = rv;
      tz[o] = zv;
      tn[o] = nv;
      th[o] = hh;
      to[o] = hv;
      sh[wl][cur ^ 1][j] = hv;
    }
    __syncwarp();
    cur ^= 1;
  }
  if (act) fin[int64_t(r) * 2 * H + d * H + j] = sh[wl][cur][j];  // final_state (layers.cpp:389-399)
}

// H == 32 forward, one row per warp (640 row-directions spread over every
// SM scheduler: the step loop is latency-bound, so one warp per scheduler).
// Each lane keeps its three W_h columns in registers for the whole sequence
// (96 floats), so a step reads only h (8 broadcast LDS.128); the r and z gates
// run as one paired chain, n as a scalar chain; next step's token and table
// values are prefetched. Same per-element operations and order as k_sprm_fwd.
constexpr int kFwdWarps = 4;
__global__ void __launch_bounds__(kFwdWarps * 32) k_sprm_fwd32(SprmP s, const uint32_t* __restrict__ ctx,
                                                               const float* __restrict__ tab, float* tape,
                                                               float* fin) {
  pdl_wait();
  constexpr int H = 32;
  __shared__ __align__(16) float sh[kFwdWarps][2][H];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = blockIdx.x & 1;
  const int r = (blockIdx.x >> 1) * kFwdWarps + wl;
  const int T = s.T, R = s.R, V = s.V;
  if (r >= R) return;
  const float* W = s.w;
  const int j = lane;
  const float* wr = W + goff(s.offs, d, WHR) + j;
  const float* wz = W + goff(s.offs, d, WHZ) + j;
  const float* wn = W + goff(s.offs, d, WHN) + j;
  f2_t wrz[H];
  float wnr[H];
#pragma unroll
  for (int q = 0; q < H; ++q) {
    wrz[q] = f2_pack(__ldg(wr + q * H), __ldg(wz + q * H));
    wnr[q] = __ldg(wn + q * H);
  }
  const float bhr = W[goff(s.offs, d, BHR) + j], bhz = W[goff(s.offs, d, BHZ) + j],
              bhn = W[goff(s.offs, d, BHN) + j];
  const float* t0 = tab + int64_t(d) * 3 * V * H;
  const int64_t TRH = int64_t(T) * R * H;
  float* tr = tape + (int64_t(0 * 2 + d) * TRH);
  float* tz = tape + (int64_t(1 * 2 + d) * TRH);
  float* tn = tape + (int64_t(2 * 2 + d) * TRH);
  float* th = tape + (int64_t(3 * 2 + d) * TRH);
  float* to = tape + (int64_t(4 * 2 + d) * TRH);
  sh[wl][0][j] = 0.0f;
  auto fetch = [&](int t, float (&x)[3]) {
    const int src_t = d ? (T - 1 - t) : t;
    const int64_t k0 = ctx[int64_t(r) * T + src_t];
    x[0] = t0[k0 * H + j];
    x[1] = t0[int64_t(V) * H + k0 * H + j];
    x[2] = t0[2 * int64_t(V) * H + k0 * H + j];
  };
  float xc[3], xn[3];
  fetch(0, xc);
  __syncwarp();
  int cur = 0;
  for (int t = 0; t < T; ++t) {
    if (t + 1 < T) fetch(t + 1, xn);
    f2_t arz = f2_pack(fadd(xc[0], bhr), fadd(xc[1], bhz));
    float hh = bhn;
    const float* h = sh[wl][cur];
#pragma unroll
    for (int q4 = 0; q4 < H / 4; ++q4) {
      const float4 hv = *reinterpret_cast<const float4*>(h + 4 * q4);
      const float hq[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        arz = f2_mac(arz, f2_bcast(hq[u]), wrz[4 * q4 + u]);
        hh = mac(hh, hq[u], wnr[4 * q4 + u]);
      }
    }
    const f2_t rz = det_sigmoid2(arz);
    const float rv = f2_lo(rz), zv = f2_hi(rz);
    const float nv = det_tanh(fadd(xc[2], fmul(rv, hh)));
    const float hv = fadd(fmul(fsub(1.0f, zv), nv), fmul(zv, h[j]));
    const int64_t o = (int64_t(t) * R + r) * H + j;
    tr[o] = rv;
    tz[o] = zv;
    tn[o] = nv;
    th[o] = hh;
    to[o] = hv;
    sh[wl][cur ^ 1][j] = hv;
    __syncwarp();
    cur ^= 1;
#pragma unroll
    for (int g = 0; g < 3; ++g) xc[g] = xn[g];
  }
  fin[int64_t(r) * 2 * H + d * H + j] = sh[wl][cur][j];  // final_state (layers.cpp:389-399)
}

// Forward with tape for H = 32*U > 32 (scale 2: H = 64, scale 1: H = 128).
// Block = one direction, kWideWarps rows (warp per row); lane owns units
// j = lane + 32u. The direction's W_h{r,z,n} sit in shared memory as
// [gate][q][32] pairs (W[q][lane + 64v], W[q][lane + 64v + 32]) so that units
// u = 2v, 2v+1 of a lane run as one paired exact chain; h of the warp's row is
// double-buffered in shared memory and read as a broadcast. Per element the
// operations and their order are k_sprm_fwd's (Gru::forward, layers.cpp:229-258).
constexpr int kWideWarps = 4;
template <int U>
__global__ void __launch_bounds__(kWideWarps * 32) k_sprm_fwd_wide(SprmP s, const uint32_t* __restrict__ ctx,
                                                                   const float* __restrict__ tab, float* tape,
                                                                   float* fin) {
  pdl_wait();
  constexpr int H = 32 * U, P2 = U / 2;
  extern __shared__ __align__(16) float dyn[];
  f2_t* sw = reinterpret_cast<f2_t*>(dyn);                 // [3][H][P2][32]
  float* sh = dyn + 2 * (3 * H * P2 * 32);                 // [kWideWarps][2][H]
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = blockIdx.x & 1;
  const int r = (blockIdx.x >> 1) * kWideWarps + wl;
  const int T = s.T, R = s.R, V = s.V;
  const float* W = s.w;
  for (int i = threadIdx.x; i < 3 * H * P2 * 32; i += blockDim.x) {
    const int g = i / (H * P2 * 32), rem = i % (H * P2 * 32), q = rem / (P2 * 32),
              v = (rem / 32) % P2, l = rem % 32;
    const float* Wg = W + goff(s.offs, d, WHR + g) + int64_t(q) * H;
    sw[i] = f2_pack(Wg[l + 64 * v], Wg[l + 64 * v + 32]);
  }
  float* hb = sh + wl * 2 * H;
  for (int j = lane; j < H; j += 32) hb[j] = 0.0f;
  __syncthreads();
  if (r >= R) return;
  float bhr[U], bhz[U], bhn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int j = lane + 32 * u;
    bhr[u] = W[goff(s.offs, d, BHR) + j];
    bhz[u] = W[goff(s.offs, d, BHZ) + j];
    bhn[u] = W[goff(s.offs, d, BHN) + j];
  }
  const float* t0 = tab + int64_t(d) * 3 * V * H;
  const int64_t TRH = int64_t(T) * R * H;
  float* tr = tape + (int64_t(0 * 2 + d) * TRH);
  float* tz = tape + (int64_t(1 * 2 + d) * TRH);
  float* tn = tape + (int64_t(2 * 2 + d) * TRH);
  float* th = tape + (int64_t(3 * 2 + d) * TRH);
  float* to = tape + (int64_t(4 * 2 + d) * TRH);
  __syncwarp();
  int cur = 0;
  for (int t = 0; t < T; ++t) {
    const int src_t = d ? (T - 1 - t) : t;
    const int64_t tok = ctx[int64_t(r) * T + src_t];
    const float* h = hb + cur * H;
    f2_t ar[P2], az[P2], hh[P2];
#pragma unroll
    for (int v = 0; v < P2; ++v) {
      const int j0 = lane + 64 * v, j1 = j0 + 32;
      ar[v] = f2_pack(fadd(t0[tok * H + j0], bhr[2 * v]), fadd(t0[tok * H + j1], bhr[2 * v + 1]));
      az[v] = f2_pack(fadd(t0[int64_t(V) * H + tok * H + j0], bhz[2 * v]),
                      fadd(t0[int64_t(V) * H + tok * H + j1], bhz[2 * v + 1]));
      hh[v] = f2_pack(bhn[2 * v], bhn[2 * v + 1]);
    }
    for (int q = 0; q < H; ++q) {
      const f2_t hq = f2_bcast(h[q]);
#pragma unroll
      for (int v = 0; v < P2; ++v) {
        ar[v] = f2_mac(ar[v], hq, sw[((0 * H + q) * P2 + v) * 32 + lane]);
        az[v] = f2_mac(az[v], hq, sw[((1 * H + q) * P2 + v) * 32 + lane]);
        hh[v] = f2_mac(hh[v], hq, sw[((2 * H + q) * P2 + v) * 32 + lane]);
      }
    }
    float hn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = u >> 1, j = lane + 32 * u;
      const float arv = (u & 1) ? f2_hi(ar[v]) : f2_lo(ar[v]);
      const float azv = (u & 1) ? f2_hi(az[v]) : f2_lo(az[v]);
      const float hhv = (u & 1) ? f2_hi(hh[v]) : f2_lo(hh[v]);
      const float an = t0[2 * int64_t(V) * H + tok * H + j];
      const float rv = det_sigmoid(arv), zv = det_sigmoid(azv);
      const float nv = det_tanh(fadd(an, fmul(rv, hhv)));
      hn[u] = fadd(fmul(fsub(1.0f, zv), nv), fmul(zv, h[j]));
      const int64_t o = (int64_t(t) * R + r) * H + j;
      tr[o] = rv;
      tz[o] = zv;
      tn[o] = nv;
      th[o] = hhv;
      to[o] = hn[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) hb[(cur ^ 1) * H + lane + 32 * u] = hn[u];
    __syncwarp();
    cur ^= 1;
  }
#pragma unroll
  for (int u = 0; u < U; ++u)  // final_state (layers.cpp:389-399)
    fin[int64_t(r) * 2 * H + d * H + lane + 32 * u] = hb[cur * H + lane + 32 * u];
}

// BPTT for H = 32*U > 32: as k_sprm_bptt (same per-element operations and
// order), lane owns units j = lane + 32u; the transposed W_h of the direction
// in shared memory as pairs WT[gate][q][v][lane] = (W_g[j0][q], W_g[j1][q]),
// j0 = lane + 64v, j1 = j0 + 32; this step's dhh/dar/daz of the warp's row in
// shared memory, read as broadcasts.
template <int U>
__global__ void __launch_bounds__(kWideWarps * 32) k_sprm_bptt_wide(SprmP s, const float* __restrict__ tape,
                                                                    const float* __restrict__ dfin, float* Gt) {
  pdl_wait();
  constexpr int H = 32 * U, P2 = U / 2;
  extern __shared__ __align__(16) float dyn[];
  f2_t* swt = reinterpret_cast<f2_t*>(dyn);  // [3 (n, r, z)][H][P2][32]
  float* sg = dyn + 2 * (3 * H * P2 * 32);   // [kWideWarps][3][H]
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = blockIdx.x & 1;
  const int r = (blockIdx.x >> 1) * kWideWarps + wl;
  const int T = s.T, R = s.R;
  const float* W = s.w;
  for (int i = threadIdx.x; i < 3 * H * P2 * 32; i += blockDim.x) {
    const int g = i / (H * P2 * 32), rem = i % (H * P2 * 32), q = rem / (P2 * 32),
              v = (rem / 32) % P2, l = rem % 32;
    const float* Wg = W + goff(s.offs, d, g == 0 ? WHN : g == 1 ? WHR : WHZ);
    swt[i] = f2_pack(Wg[int64_t(l + 64 * v) * H + q], Wg[int64_t(l + 64 * v + 32) * H + q]);
  }
  __syncthreads();
  if (r >= R) return;
  float* sgw = sg + wl * 3 * H;
  const int64_t TRH = int64_t(T) * R * H;
  const float* tp[5];
#pragma unroll
  for (int g = 0; g < 5; ++g) tp[g] = tape + (int64_t(g * 2 + d) * TRH);
  float* go[5];
#pragma unroll
  for (int g = 0; g < 5; ++g) go[g] = Gt + int64_t(g * 2 + d) * TRH;  // an, ar, az, hh, hprev
  float dh[U], dlast[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    dh[u] = 0.0f;
    dlast[u] = fadd(0.0f, dfin[int64_t(r) * 2 * H + d * H + lane + 32 * u]);
  }
  for (int t = T - 1; t >= 0; --t) {
    float dn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = lane + 32 * u;
      dh[u] = fadd(dh[u], t == T - 1 ? dlast[u] : 0.0f);  // gather_add_step(dout, t, dh)
      const int64_t o = (int64_t(t) * R + r) * H + j;
      const float rv = tp[0][o], zv = tp[1][o], nv = tp[2][o], hhv = tp[3][o];
      const float hprev = t == 0 ? 0.0f : tp[4][o - int64_t(R) * H];
      const float dzv = fmul(dh[u], fsub(hprev, nv));
      const float danv = fmul(fmul(dh[u], fsub(1.0f, zv)), fsub(1.0f, fmul(nv, nv)));
      const float dar = fmul(fmul(fmul(danv, hhv), rv), fsub(1.0f, rv));
      const float daz = fmul(fmul(dzv, zv), fsub(1.0f, zv));
      const float dhh = fmul(danv, rv);
      dn[u] = fmul(dh[u], zv);
      go[0][o] = danv;
      go[1][o] = dar;
      go[2][o] = daz;
      go[3][o] = dhh;
      go[4][o] = hprev;
      sgw[0 * H + j] = dhh;
      sgw[1 * H + j] = dar;
      sgw[2 * H + j] = daz;
    }
    __syncwarp();
    // dh_next = dh*z + dhh.W_hn^T + dar.W_hr^T + daz.W_hz^T  (layers.cpp:306-308)
    f2_t acc[P2];
#pragma unroll
    for (int v = 0; v < P2; ++v) acc[v] = f2_pack(dn[2 * v], dn[2 * v + 1]);
#pragma unroll
    for (int g = 0; g < 3; ++g)
      for (int q = 0; q < H; ++q) {
        const f2_t gq = f2_bcast(sgw[g * H + q]);
#pragma unroll
        for (int v = 0; v < P2; ++v) acc[v] = f2_mac(acc[v], gq, swt[((g * H + q) * P2 + v) * 32 + lane]);
      }
    __syncwarp();
#pragma unroll
    for (int v = 0; v < P2; ++v) {
      dh[2 * v] = f2_lo(acc[v]);
      dh[2 * v + 1] = f2_hi(acc[v]);
    }
  }
}

template <int U>
size_t wide_smem(int extra_per_warp) {
  return size_t(2 * 3 * 32 * U * (U / 2) * 32 + kWideWarps * extra_per_warp * 32 * U) * sizeof(float);
}

// The model head of one train step, forward and backward, warp per row
// (BiGruModel::forward tail and backward head, models.cpp:67-72, 77-86, with
// the CE gradient of training.cpp:28-34 between them):
//   bact = tanh(bott.b + fin.bott.w)          (Linear::forward: bias, then ascending p)
//   logits = out.b + bact.out.w
//   g = det_softmax(logits); g[tgt] -= 1
//   dbact = (0 + g.out.w^T) * (1 - bact^2)   (Linear::backward dx, ascending o)
//   dfin = 0 + dbact.bott.w^T
// The chains of every output are the reference's; only their placement
// changes (one launch instead of seven). The weight gradients of bott/out
// (reductions over rows) run afterwards on the side stream from bact, g,
// dbact.
constexpr int kHeadWarps = 4;
__global__ void __launch_bounds__(kHeadWarps * 32) k_sprm_head(
    SprmP s, const uint32_t* __restrict__ tokens, const int64_t* __restrict__ pos,
    const float* __restrict__ fin, const float* __restrict__ w1, const float* __restrict__ b1,
    const float* __restrict__ w2, const float* __restrict__ b2, float* bact_out, float* g_out,
    float* dbact_out, float* dfin_out) {
  pdl_wait();
  extern __shared__ __align__(16) float hs[];
  const int H2 = 2 * s.H, B = s.B, V = s.V;
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * kHeadWarps + wl;
  float* f = hs + wl * (H2 + 2 * B + V);  // fin row, bact, dbact, g
  float* ba = f + H2;
  float* db = ba + B;
  float* gr = db + B;
  if (r >= s.R) return;
  for (int p = lane; p < H2; p += 32) f[p] = fin[int64_t(r) * H2 + p];
  __syncwarp();
  for (int j = lane; j < B; j += 32) {
    float acc = b1[j];
    for (int p = 0; p < H2; ++p) acc = mac(acc, f[p], w1[int64_t(p) * B + j]);
    acc = det_tanh(acc);
    ba[j] = acc;
    bact_out[int64_t(r) * B + j] = acc;
  }
  __syncwarp();
  float mx = -__int_as_float(0x7f800000);
  for (int i = lane; i < V; i += 32) {
    float acc = b2[i];
    for (int q = 0; q < B; ++q) acc = mac(acc, ba[q], w2[int64_t(q) * V + i]);
    gr[i] = acc;
    mx = fmaxf(mx, acc);
  }
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __syncwarp();
  // det_softmax (detmath.cpp:85-97): exp of the shifted logits, one sequential sum
  float sum = 0.0f;
  for (int i0 = 0; i0 < V; i0 += 32) {
    const int i = i0 + lane;
    float e = 0.0f;
    if (i < V) {
      e = det_exp(fsub(gr[i], mx));
      gr[i] = e;
    }
    const int cnt = min(32, V - i0);
    for (int l = 0; l < cnt; ++l) sum = fadd(sum, __shfl_sync(0xffffffffu, e, l));
  }
  const float inv = fdiv(1.0f, sum);
  const uint32_t tgt = tokens[*pos + r] & uint32_t(V - 1);
  __syncwarp();
  for (int i = lane; i < V; i += 32) {
    float v = fmul(gr[i], inv);
    if (uint32_t(i) == tgt) v = fsub(v, 1.0f);
    gr[i] = v;
    g_out[int64_t(r) * V + i] = v;
  }
  __syncwarp();
  for (int j = lane; j < B; j += 32) {
    float acc = 0.0f;
    const float* wr = w2 + int64_t(j) * V;
    for (int o = 0; o < V; ++o) acc = mac(acc, gr[o], wr[o]);
    const float a = ba[j];
    acc = fmul(acc, fsub(1.0f, fmul(a, a)));
    db[j] = acc;
    dbact_out[int64_t(r) * B + j] = acc;
  }
  __syncwarp();
  for (int p = lane; p < H2; p += 32) {
    float acc = 0.0f;
    const float* wr = w1 + int64_t(p) * B;
    for (int j = 0; j < B; ++j) acc = mac(acc, db[j], wr[j]);
    dfin_out[int64_t(r) * H2 + p] = acc;
  }
}

// g = det_softmax(logits) ; loss term ; g[tgt] -= 1   (training.cpp:28-34)
__global__ void k_sprm_ce(SprmP s, const uint32_t* __restrict__ tokens,
                          const int64_t* __restrict__ pos, const float* __restrict__ logits,
                          float* g) {
  pdl_wait();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= s.R) return;
  const int V = s.V;
  const float* lr = logits + int64_t(row) * V;
  float* gr = g + int64_t(row) * V;
  float mx = -__int_as_float(0x7f800000);
  for (int i = lane; i < V; i += 32) mx = fmaxf(mx, lr[i]);
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.0f;
  for (int i0 = 0; i0 < V; i0 += 32) {
    const int i = i0 + lane;
    float e = 0.0f;
    if (i < V) {
      e = det_exp(fsub(lr[i], mx));
      gr[i] = e;
    }
    const int cnt = min(32, V - i0);
    for (int l = 0; l < cnt; ++l) sum = fadd(sum, __shfl_sync(0xffffffffu, e, l));
  }
  const float inv = fdiv(1.0f, sum);
  const uint32_t tgt = tokens[*pos + row] & uint32_t(V - 1);
  __syncwarp();
  for (int i = lane; i < V; i += 32) {
    float v = fmul(gr[i], inv);
    if (uint32_t(i) == tgt) v = fsub(v, 1.0f);
    gr[i] = v;
  }
}

// dbact *= (1 - a*a)   (models.cpp:81-84)
__global__ void k_sprm_tanh_grad(float* dbact, const float* __restrict__ bact, int64_t n) {
  pdl_wait();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    const float a = bact[i];
    dbact[i] = fmul(dbact[i], fsub(1.0f, fmul(a, a)));
  }
}

// Backward through time. Blocks are single-direction (8 warps = 8 rows, lane =
// unit); the direction's W_h* are staged transposed in shared memory so the
// dh recurrence reads conflict-free. Serial part only: the gate gradients and
// h_{t-1} are stored row-major Gt[5][2][T][R][H] (an, ar, az, hh, hprev) and
// transposed afterwards into the feature-major reduction operands.
__global__ void __launch_bounds__(256) k_sprm_bptt(SprmP s, const float* __restrict__ tape,
                                                   const float* __restrict__ dfin, float* Gt) {
  pdl_wait();
  __shared__ float swt[3][32][33];              // [gate][q][j] = W_h{gate}[j][q]
  __shared__ __align__(16) float sg[8][3][32];  // dhh, dar, daz of this step
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = blockIdx.x & 1;
  const int r = (blockIdx.x >> 1) * 8 + wl;
  const int T = s.T, H = s.H, R = s.R;
  const float* W = s.w;
  for (int i = threadIdx.x; i < 3 * H * H; i += blockDim.x) {
    const int gate = i / (H * H), rem = i % (H * H), jj = rem / H, q = rem % H;
    const float* Wg = W + goff(s.offs, d, gate == 0 ? WHN : gate == 1 ? WHR : WHZ);
    swt[gate][q][jj] = Wg[int64_t(jj) * H + q];
  }
  __syncthreads();
  if (r >= R) return;
  const bool act = lane < H;
  const int j = act ? lane : 0;
  const int64_t TRH = int64_t(T) * R * H;
  const float* tr = tape + (int64_t(0 * 2 + d) * TRH);
  const float* tz = tape + (int64_t(1 * 2 + d) * TRH);
  const float* tn = tape + (int64_t(2 * 2 + d) * TRH);
  const float* th = tape + (int64_t(3 * 2 + d) * TRH);
  const float* to = tape + (int64_t(4 * 2 + d) * TRH);
  float* gan = Gt + int64_t(0 * 2 + d) * TRH;
  float* gar = Gt + int64_t(1 * 2 + d) * TRH;
  float* gaz = Gt + int64_t(2 * 2 + d) * TRH;
  float* ghh = Gt + int64_t(3 * 2 + d) * TRH;
  float* ghp = Gt + int64_t(4 * 2 + d) * TRH;
  // only the GRU's last own step receives the final-state gradient
  // (final_state_backward, layers.cpp:401-413), as 0 + dfin
  const float dlast = fadd(0.0f, dfin[int64_t(r) * 2 * H + d * H + j]);
  float dh = 0.0f;
  for (int t = T - 1; t >= 0; --t) {
    dh = fadd(dh, t == T - 1 ? dlast : 0.0f);  // gather_add_step(dout, t, dh)
    const int64_t o = (int64_t(t) * R + r) * H + j;
    const float rv = tr[o], zv = tz[o], nv = tn[o], hhv = th[o];
    const float hprev = t == 0 ? 0.0f : to[o - int64_t(R) * H];
    const float dzv = fmul(dh, fsub(hprev, nv));
    const float danv = fmul(fmul(dh, fsub(1.0f, zv)), fsub(1.0f, fmul(nv, nv)));
    const float dar = fmul(fmul(fmul(danv, hhv), rv), fsub(1.0f, rv));
    const float daz = fmul(fmul(dzv, zv), fsub(1.0f, zv));
    const float dhh = fmul(danv, rv);
    float dn = fmul(dh, zv);
    if (act) {
      gan[o] = danv;
      gar[o] = dar;
      gaz[o] = daz;
      ghh[o] = dhh;
      ghp[o] = hprev;
      sg[wl][0][j] = dhh;
      sg[wl][1][j] = dar;
      sg[wl][2][j] = daz;
    }
    __syncwarp();
    // dh_next = dh*z + dhh.W_hn^T + dar.W_hr^T + daz.W_hz^T  (layers.cpp:306-308)
    for (int q = 0; q < H; ++q) dn = mac(dn, sg[wl][0][q], swt[0][q][j]);
    for (int q = 0; q < H; ++q) dn = mac(dn, sg[wl][1][q], swt[1][q][j]);
    for (int q = 0; q < H; ++q) dn = mac(dn, sg[wl][2][q], swt[2][q][j]);
    __syncwarp();
    dh = dn;
  }
}

// H == 32 BPTT, one row per warp (the dh chain of 3*H MACs per step is the
// latency floor; one warp per scheduler). Each lane keeps its W_h rows in
// registers (96 floats); a step reads only the gate gradients (broadcast
// LDS.128); the step's tape values are prefetched one step ahead. Same
// per-element operations and order as k_sprm_bptt.
constexpr int kBpttWarps = 4;
__global__ void __launch_bounds__(kBpttWarps * 32) k_sprm_bptt32(SprmP s, const float* __restrict__ tape,
                                                                 const float* __restrict__ dfin, float* Gt) {
  pdl_wait();
  constexpr int H = 32;
  __shared__ __align__(16) float sg[kBpttWarps][3][H];  // dhh, dar, daz of this step
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = blockIdx.x & 1;
  const int r = (blockIdx.x >> 1) * kBpttWarps + wl;
  const int T = s.T, R = s.R;
  if (r >= R) return;
  const float* W = s.w;
  const int j = lane;
  // wt[g][q] = W_h{n,r,z}[j][q] (row j of each gate matrix)
  float wt[3][H];
#pragma unroll
  for (int g = 0; g < 3; ++g) {
    const float* Wg = W + goff(s.offs, d, g == 0 ? WHN : g == 1 ? WHR : WHZ) + int64_t(j) * H;
#pragma unroll
    for (int q4 = 0; q4 < H / 4; ++q4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(Wg) + q4);
      wt[g][4 * q4 + 0] = v.x;
      wt[g][4 * q4 + 1] = v.y;
      wt[g][4 * q4 + 2] = v.z;
      wt[g][4 * q4 + 3] = v.w;
    }
  }
  const int64_t TRH = int64_t(T) * R * H;
  const float* tp[5];
#pragma unroll
  for (int g = 0; g < 5; ++g) tp[g] = tape + (int64_t(g * 2 + d) * TRH);
  float* gan = Gt + int64_t(0 * 2 + d) * TRH;
  float* gar = Gt + int64_t(1 * 2 + d) * TRH;
  float* gaz = Gt + int64_t(2 * 2 + d) * TRH;
  float* ghh = Gt + int64_t(3 * 2 + d) * TRH;
  float* ghp = Gt + int64_t(4 * 2 + d) * TRH;
  // only the GRU's last own step receives the final-state gradient
  // (final_state_backward, layers.cpp:401-413), as 0 + dfin
  const float dlast = fadd(0.0f, dfin[int64_t(r) * 2 * H + d * H + j]);
  auto fetch = [&](int t, float (&x)[5]) {
    const int64_t o = (int64_t(t) * R + r) * H + j;
#pragma unroll
    for (int g = 0; g < 4; ++g) x[g] = tp[g][o];
    x[4] = t == 0 ? 0.0f : tp[4][o - int64_t(R) * H];
  };
  float xc[5], xn[5];
  fetch(T - 1, xc);
  float dh = 0.0f;
  for (int t = T - 1; t >= 0; --t) {
    if (t > 0) fetch(t - 1, xn);
    dh = fadd(dh, t == T - 1 ? dlast : 0.0f);  // gather_add_step(dout, t, dh)
    const float rv = xc[0], zv = xc[1], nv = xc[2], hhv = xc[3], hprev = xc[4];
    const float dzv = fmul(dh, fsub(hprev, nv));
    const float danv = fmul(fmul(dh, fsub(1.0f, zv)), fsub(1.0f, fmul(nv, nv)));
    const float dar = fmul(fmul(fmul(danv, hhv), rv), fsub(1.0f, rv));
    const float daz = fmul(fmul(dzv, zv), fsub(1.0f, zv));
    const float dhh = fmul(danv, rv);
    float dn = fmul(dh, zv);
    const int64_t o = (int64_t(t) * R + r) * H + j;
    gan[o] = danv;
    gar[o] = dar;
    gaz[o] = daz;
    ghh[o] = dhh;
    ghp[o] = hprev;
    sg[wl][0][j] = dhh;
    sg[wl][1][j] = dar;
    sg[wl][2][j] = daz;
    __syncwarp();
    // dh_next = dh*z + dhh.W_hn^T + dar.W_hr^T + daz.W_hz^T  (layers.cpp:306-308)
#pragma unroll
    for (int g = 0; g < 3; ++g)
#pragma unroll
      for (int q4 = 0; q4 < H / 4; ++q4) {
        const float4 v = *reinterpret_cast<const float4*>(&sg[wl][g][4 * q4]);
        dn = mac(dn, v.x, wt[g][4 * q4 + 0]);
        dn = mac(dn, v.y, wt[g][4 * q4 + 1]);
        dn = mac(dn, v.z, wt[g][4 * q4 + 2]);
        dn = mac(dn, v.w, wt[g][4 * q4 + 3]);
      }
    __syncwarp();
    dh = dn;
#pragma unroll
    for (int g = 0; g < 5; ++g) xc[g] = xn[g];
  }
}

// Gt[g][d][t][r][j] -> G[g][d][j][k], k = (T-1-t)*R + r (32x32 smem tiles).
// A block owns one (k, j) tile position for all 10 gate/direction slabs: every
// load is issued up front (40 per thread in flight), then the slabs go through
// the shared tile one after another -- one memory latency per block instead
// of one per tile.
constexpr int kTrSlabs = 10;
__global__ void __launch_bounds__(256) k_sprm_transpose(SprmP s, const float* __restrict__ Gt, float* G) {
  pdl_wait();
  __shared__ float tile[32][33];
  const int T = s.T, H = s.H, R = s.R;
  const int64_t RT = int64_t(R) * T;
  const int64_t k0 = int64_t(blockIdx.x) * 32;
  const int j0 = blockIdx.y * 32;
  // source offsets of this thread's 4 rows (the same in every slab)
  int64_t so[4];
  bool ok[4];
  const int j = j0 + threadIdx.x;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t k = uint32_t(k0) + threadIdx.y + 8 * u;
    ok[u] = k < uint64_t(RT) && j < H;
    const uint32_t t = uint32_t(T - 1) - k / uint32_t(R), r = k % uint32_t(R);
    so[u] = (int64_t(t) * R + r) * H + j;
  }
  float v[kTrSlabs][4];
#pragma unroll
  for (int gd = 0; gd < kTrSlabs; ++gd) {
    const float* src = Gt + int64_t(gd) * RT * H;
#pragma unroll
    for (int u = 0; u < 4; ++u) v[gd][u] = ok[u] ? __ldg(src + so[u]) : 0.0f;
  }
#pragma unroll
  for (int gd = 0; gd < kTrSlabs; ++gd) {
    float* dst = G + int64_t(gd) * H * RT;
#pragma unroll
    for (int u = 0; u < 4; ++u) tile[threadIdx.y + 8 * u][threadIdx.x] = v[gd][u];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int yy = threadIdx.y + 8 * u;
      const int jj = j0 + yy;
      const int64_t k = k0 + threadIdx.x;
      if (k < RT && jj < H) dst[int64_t(jj) * RT + k] = tile[threadIdx.x][yy];
    }
    __syncthreads();
  }
}

// dx[r][t][i] = (0 + dxt_fwd(t)) + (0 + dxt_bwd(T-1-t)),
// dxt(t) = 0 + dan.W_in^T + dar.W_ir^T + daz.W_iz^T   (layers.cpp:300-304, 384-386)
__global__ void k_sprm_dx(SprmP s, const float* __restrict__ Gr, float* dx) {
  pdl_wait();
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int R = s.R, T = s.T, Es = s.Es, H = s.H;
  const int64_t RT = int64_t(R) * T;
  if (idx >= RT * Es) return;
  const uint32_t ui = uint32_t(idx);  // R*T*Es < 2^31
  const int i = int(ui % uint32_t(Es));
  const uint32_t rt = ui / uint32_t(Es);
  const int r = int(rt / uint32_t(T)), t = int(rt % uint32_t(T));
  const float* W = s.w;
  float part[2];
  for (int d = 0; d < 2; ++d) {
    const int own_t = d ? (T - 1 - t) : t;
    const int64_t k = int64_t(T - 1 - own_t) * R + r;
    float acc = 0.0f;
    const int gates[3] = {WIN, WIR, WIZ};
    const int gsel[3] = {0, 1, 2};
    for (int u = 0; u < 3; ++u) {
      const float* gg = Gr + (int64_t(gsel[u] * 2 + d) * H) * RT;
      const float* Wg = W + goff(s.offs, d, gates[u]) + int64_t(i) * H;
      for (int q = 0; q < H; ++q) acc = mac(acc, gg[int64_t(q) * RT + k], Wg[q]);
    }
    part[d] = acc;
  }
  dx[idx] = fadd(fadd(0.0f, part[0]), fadd(0.0f, part[1]));  // dx += dx_rev (both from zero)
}

// dx from the time-major gradients Gt[g][d][t][r][j] (H == 32, Es <= 8): the
// 3*H terms of one (row, step, direction) are three contiguous 128-byte
// vectors, read with LDG.128 and shared by the Es threads of the position;
// the input weights sit in shared memory. Same chain order as k_sprm_dx.
__global__ void __launch_bounds__(256) k_sprm_dx_t(SprmP s, const float* __restrict__ Gt, float* dx) {
  pdl_wait();
  constexpr int H = 32;
  __shared__ __align__(16) float sw[2][3][8][H];  // [d][gate n,r,z][i][q]
  const int R = s.R, T = s.T, Es = s.Es;
  const float* W = s.w;
  const int gates[3] = {WIN, WIR, WIZ};
  for (int e = threadIdx.x; e < 2 * 3 * Es * H; e += blockDim.x) {
    const int d = e / (3 * Es * H), rem = e % (3 * Es * H), u = rem / (Es * H), iq = rem % (Es * H);
    sw[d][u][iq / H][iq % H] = W[goff(s.offs, d, gates[u]) + iq];
  }
  __syncthreads();
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t RT = int64_t(R) * T;
  if (idx >= RT * Es) return;
  const uint32_t ui = uint32_t(idx);  // R*T*Es < 2^31
  const int i = int(ui % uint32_t(Es));
  const uint32_t rt = ui / uint32_t(Es);
  const int r = int(rt / uint32_t(T)), t = int(rt % uint32_t(T));
  const int64_t TRH = RT * H;
  float part[2];
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    const int own_t = d ? (T - 1 - t) : t;
    float acc = 0.0f;
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const float4* gp =
          reinterpret_cast<const float4*>(Gt + int64_t(u * 2 + d) * TRH + (int64_t(own_t) * R + r) * H);
      float4 g4[H / 4];
#pragma unroll
      for (int q4 = 0; q4 < H / 4; ++q4) g4[q4] = __ldg(gp + q4);
      const float* w = sw[d][u][i];
#pragma unroll
      for (int q4 = 0; q4 < H / 4; ++q4) {
        acc = mac(acc, g4[q4].x, w[4 * q4 + 0]);
        acc = mac(acc, g4[q4].y, w[4 * q4 + 1]);
        acc = mac(acc, g4[q4].z, w[4 * q4 + 2]);
        acc = mac(acc, g4[q4].w, w[4 * q4 + 3]);
      }
    }
    part[d] = acc;
  }
  dx[idx] = fadd(fadd(0.0f, part[0]), fadd(0.0f, part[1]));  // dx += dx_rev (both from zero)
}

__global__ void k_tanh_vec(float* x, int64_t n) {
  pdl_wait();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = det_tanh(x[i]);
}

__global__ void k_adam_scalars(AdamScalars* sc) {
  pdl_wait();
  AdamScalars a = *sc;
  a.step += 1;
  a.b1p = fmul(a.b1p, 0.9f);
  a.b2p = fmul(a.b2p, 0.999f);
  a.bc1 = fsub(1.0f, a.b1p);
  a.bc2 = fsub(1.0f, a.b2p);
  *sc = a;
}

__global__ void k_pos_advance(int64_t* pos, int64_t by) {
  pdl_wait(); *pos += by; }

}  // namespace

void launch_sprm_prep(const uint32_t* tokens, const int64_t* pos, const SprmP& s, uint32_t* ctx,
                      float* X, float* tab, cudaStream_t st) {
  const int64_t n = std::max<int64_t>(std::max<int64_t>(int64_t(s.R) * s.T, 6ll * s.V * s.H),
                                      2ll * s.Es * s.R * s.T);
  launch_pdl(k_sprm_prep, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, tokens, pos, s, ctx, X, tab);
}
void launch_sprm_fwd(const SprmP& s, const uint32_t* ctx, const float* tab, float* tape, float* fin,
                     cudaStream_t st) {
  if (s.H == 32) {
    launch_pdl(k_sprm_fwd32, dim3(unsigned(2 * ((s.R + kFwdWarps - 1) / kFwdWarps))), dim3(kFwdWarps * 32), 0, st, 
        s, ctx, tab, tape, fin);
    return;
  }
  const dim3 wgrid(unsigned(2 * ((s.R + kWideWarps - 1) / kWideWarps)));
  if (s.H == 64) {
    const size_t sm = wide_smem<2>(2);
    ensure_smem(reinterpret_cast<const void*>(k_sprm_fwd_wide<2>), sm);
    launch_pdl(k_sprm_fwd_wide<2>, wgrid, dim3(kWideWarps * 32), sm, st, s, ctx, tab, tape, fin);
    return;
  }
  if (s.H == 128) {
    const size_t sm = wide_smem<4>(2);
    ensure_smem(reinterpret_cast<const void*>(k_sprm_fwd_wide<4>), sm);
    launch_pdl(k_sprm_fwd_wide<4>, wgrid, dim3(kWideWarps * 32), sm, st, s, ctx, tab, tape, fin);
    return;
  }
  launch_pdl(k_sprm_fwd, dim3(unsigned(2 * ((s.R + 7) / 8))), dim3(256), 0, st, s, ctx, tab, tape, fin);
}
void launch_sprm_ce(const SprmP& s, const uint32_t* tokens, const int64_t* pos, const float* logits,
                    float* g, cudaStream_t st) {
  launch_pdl(k_sprm_ce, dim3(unsigned((s.R * 32 + 255) / 256)), dim3(256), 0, st, s, tokens, pos, logits, g);
}
void launch_sprm_tanh_grad(float* dbact, const float* bact, int64_t n, cudaStream_t st) {
  launch_pdl(k_sprm_tanh_grad, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, dbact, bact, n);
}
void launch_sprm_bptt(const SprmP& s, const float* tape, const float* dfin, float* Gt,
                      cudaStream_t st) {
  if (s.H == 32)
    launch_pdl(k_sprm_bptt32, dim3(unsigned(2 * ((s.R + kBpttWarps - 1) / kBpttWarps))), dim3(kBpttWarps * 32), 0, st, 
        s, tape, dfin, Gt);
  else if (s.H == 64 || s.H == 128) {
    const dim3 wgrid(unsigned(2 * ((s.R + kWideWarps - 1) / kWideWarps)));
    if (s.H == 64) {
      const size_t sm = wide_smem<2>(3);
      ensure_smem(reinterpret_cast<const void*>(k_sprm_bptt_wide<2>), sm);
      launch_pdl(k_sprm_bptt_wide<2>, wgrid, dim3(kWideWarps * 32), sm, st, s, tape, dfin, Gt);
    } else {
      const size_t sm = wide_smem<4>(3);
      ensure_smem(reinterpret_cast<const void*>(k_sprm_bptt_wide<4>), sm);
      launch_pdl(k_sprm_bptt_wide<4>, wgrid, dim3(kWideWarps * 32), sm, st, s, tape, dfin, Gt);
    }
  } else
    launch_pdl(k_sprm_bptt, dim3(unsigned(2 * ((s.R + 7) / 8))), dim3(256), 0, st, s, tape, dfin, Gt);
}
void launch_sprm_transpose(const SprmP& s, const float* Gt, float* G, cudaStream_t st) {
  const int64_t RT = int64_t(s.R) * s.T;
  dim3 grid(unsigned((RT + 31) / 32), unsigned((s.H + 31) / 32));
  launch_pdl(k_sprm_transpose, dim3(grid), dim3(dim3(32, 8)), 0, st, s, Gt, G);
}
bool sprm_dx_time_major(const SprmP& s) { return s.H == 32 && s.Es <= 8; }
void launch_sprm_dx(const SprmP& s, const float* G, const float* Gt, float* dx, cudaStream_t st) {
  const int64_t n = int64_t(s.R) * s.T * s.Es;
  if (sprm_dx_time_major(s) && Gt) {
    launch_pdl(k_sprm_dx_t, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, s, Gt, dx);
    return;
  }
  launch_pdl(k_sprm_dx, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, s, G, dx);
}
void launch_sprm_head(const SprmP& s, const uint32_t* tokens, const int64_t* pos, const float* fin,
                      const float* w1, const float* b1, const float* w2, const float* b2, float* bact,
                      float* g, float* dbact, float* dfin, cudaStream_t st) {
  const size_t smem = size_t(kHeadWarps) * (2 * s.H + 2 * s.B + s.V) * sizeof(float);
  ensure_smem(reinterpret_cast<const void*>(k_sprm_head), smem);
  launch_pdl(k_sprm_head, dim3(unsigned((s.R + kHeadWarps - 1) / kHeadWarps)), dim3(kHeadWarps * 32), smem,
             st, s, tokens, pos, fin, w1, b1, w2, b2, bact, g, dbact, dfin);
}
void launch_tanh_vec(float* x, int64_t n, cudaStream_t st) {
  launch_pdl(k_tanh_vec, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, x, n);
}
void launch_adam_scalars(AdamScalars* sc, cudaStream_t st) { launch_pdl(k_adam_scalars, dim3(1), dim3(1), 0, st, sc); }
void launch_pos_advance(int64_t* pos, int64_t by, cudaStream_t st) {
  launch_pdl(k_pos_advance, dim3(1), dim3(1), 0, st, pos, by);
}

}  // namespace pmklc_b200
