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
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

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
                            SprmP s, uint32_t* ctx, float* X, float* tab, float* Xtm, unsigned* cnt) {
  pdl_wait();
  const int64_t p = *pos;
  const int R = s.R, T = s.T, Es = s.Es, H = s.H, V = s.V;
  const int64_t RT = int64_t(R) * T;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const float* W = s.w;
  if (cnt && tid < 2 * T) cnt[tid] = 0u;  // streamed-BPTT step counters of this train step
  // Xtm[d][t][r][i]: the GRU input of direction d at its own time t (streamed path)
  if (Xtm && tid < 2 * RT * Es) {
    const int i = int(tid % Es);
    const int64_t rest = tid / Es;
    const int r = int(rest % R);
    const int64_t dt = rest / R;
    const int t = int(dt % T), d = int(dt / T);
    const int src_t = d ? (T - 1 - t) : t;
    Xtm[tid] = W[s.offs[0] + int64_t(tokens[p + r - T + src_t]) * Es + i];
  }
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
  // (feature-major reduction operand; the streamed path has none)
  const int64_t nx = int64_t(2) * Es * RT;
  if (X && tid < nx) {
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
  const int64_t RTH = int64_t(R) * T * H;
  for (int t = 0; t < T; ++t) {
    const int src_t = d ? (T - 1 - t) : t;
    const float* h = sh[wl][cur];
    float xr, xz, xn;  // the gates' input projections b_i + x.W_i
    if (s.xproj) {
      const float* xp = s.xproj + int64_t(d) * 3 * RTH + (int64_t(r) * T + src_t) * H + j;
      xr = xp[0];
      xz = xp[RTH];
      xn = xp[2 * RTH];
    } else {
      const int64_t tok = ctx[int64_t(r) * T + src_t];
      xr = t0[tok * H + j];
      xz = t0[int64_t(V) * H + tok * H + j];
      xn = t0[2 * int64_t(V) * H + tok * H + j];
    }
    float ar = fadd(xr, bhr);
    for (int q = 0; q < H; ++q) ar = mac(ar, h[q], sw[0][q][j]);
    float az = fadd(xz, bhz);
    for (int q = 0; q < H; ++q) az = mac(az, h[q], sw[1][q][j]);
    float hh = bhn;
    for (int q = 0; q < H; ++q) hh = mac(hh, h[q], sw[2][q][j]);
    const float an = xn;
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
constexpr int kFwdWarps = 2;
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
  // the step's tape slot (t*R + r)*H + j of slab g at tp + g*2*TRH, advanced by R*H
  float* tp = tape + int64_t(d) * TRH + int64_t(r) * H + j;
  const int64_t RH = int64_t(R) * H;
  sh[wl][0][j] = 0.0f;
  const int64_t RTH = int64_t(R) * T * H;
  // the row's context tokens, one per lane (T <= 32): a step's token is a
  // shuffle, so its table loads do not wait behind a dependent token load
  const bool lane_tok = !s.xproj && T <= 32;
  const uint32_t mytok = lane_tok && lane < T ? ctx[int64_t(r) * T + lane] : 0u;
  auto fetch = [&](int t, float (&x)[3]) {
    const int src_t = d ? (T - 1 - t) : t;
    if (s.xproj) {  // deeper layer: per-(row, position) input projections
      const float* xp = s.xproj + int64_t(d) * 3 * RTH + (int64_t(r) * T + src_t) * H + j;
      x[0] = xp[0];
      x[1] = xp[RTH];
      x[2] = xp[2 * RTH];
      return;
    }
    const int64_t k0 = lane_tok ? int64_t(__shfl_sync(0xffffffffu, mytok, src_t))
                                : int64_t(ctx[int64_t(r) * T + src_t]);
    x[0] = t0[k0 * H + j];
    x[1] = t0[int64_t(V) * H + k0 * H + j];
    x[2] = t0[2 * int64_t(V) * H + k0 * H + j];
  };
  // input terms fetched two steps ahead
  float xc[3], x1[3], x2[3];
  fetch(0, xc);
  if (T > 1) fetch(1, x1);
  __syncwarp();
  int cur = 0;
  for (int t = 0; t < T; ++t) {
    if (t + 2 < T) fetch(t + 2, x2);
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
    tp[0] = rv;
    tp[2 * TRH] = zv;
    tp[4 * TRH] = nv;
    tp[6 * TRH] = hh;
    tp[8 * TRH] = hv;
    tp += RH;
    sh[wl][cur ^ 1][j] = hv;
    __syncwarp();
    cur ^= 1;
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      xc[g] = x1[g];
      x1[g] = x2[g];
    }
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
  const int64_t RTH = int64_t(R) * T * H;
  for (int t = 0; t < T; ++t) {
    const int src_t = d ? (T - 1 - t) : t;
    // the gates' input projections: per-token table, or per-(row, position)
    const float* xg = s.xproj ? s.xproj + int64_t(d) * 3 * RTH + (int64_t(r) * T + src_t) * H
                              : t0 + int64_t(ctx[int64_t(r) * T + src_t]) * H;
    const int64_t gs = s.xproj ? RTH : int64_t(V) * H;  // gate stride
    const float* h = hb + cur * H;
    f2_t ar[P2], az[P2], hh[P2];
#pragma unroll
    for (int v = 0; v < P2; ++v) {
      const int j0 = lane + 64 * v, j1 = j0 + 32;
      ar[v] = f2_pack(fadd(xg[j0], bhr[2 * v]), fadd(xg[j1], bhr[2 * v + 1]));
      az[v] = f2_pack(fadd(xg[gs + j0], bhz[2 * v]), fadd(xg[gs + j1], bhz[2 * v + 1]));
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
      const float an = xg[2 * gs + j];
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
    dlast[u] = s.dout ? 0.0f : fadd(0.0f, dfin[int64_t(r) * 2 * H + d * H + lane + 32 * u]);
  }
  for (int t = T - 1; t >= 0; --t) {
    float dn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = lane + 32 * u;
      // gather_add_step(dout, t, dh)
      const float dadd = s.dout ? s.dout[(int64_t(r) * T + (d ? T - 1 - t : t)) * 2 * H + d * H + j]
                                : (t == T - 1 ? dlast[u] : 0.0f);
      dh[u] = fadd(dh[u], dadd);
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

__device__ __forceinline__ uint32_t sm_addr_h(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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
constexpr int kHeadWarps = 8;
// shared floats of the head kernel: W1 [2H][B] and W2 [B][V] with padded rows
// (B+1, V+1: the row walks and the column walks of the backward are both
// conflict-free from one copy), then b1 [B] and b2 [V], rounded up to whole
// float4s; and per warp fin [2H], bact [B], dbact [B], g [V]
__host__ __device__ inline int head_w_floats(int H2, int B, int V) {
  return (H2 * (B + 1) + B * (V + 1) + B + V + 3) & ~3;
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sm_addr_h(dst)), "l"(src) : "memory");
}
// kSmemW: weights and biases staged in shared memory (the default widths) or
// read from L1/L2. cH2/cB/cV: the widths at compile time (0 = runtime), so the
// default model's chains unroll fully and a lane's independent outputs
// interleave.
template <bool kSmemW, int cH2 = 0, int cB = 0, int cV = 0>
__global__ void __launch_bounds__(kHeadWarps * 32) k_sprm_head(
    SprmP s, const uint32_t* __restrict__ tokens, const int64_t* __restrict__ pos,
    const float* __restrict__ fin, const float* __restrict__ w1, const float* __restrict__ b1,
    const float* __restrict__ w2, const float* __restrict__ b2, float* bact_out, float* g_out,
    float* dbact_out, float* dfin_out) {
  extern __shared__ __align__(16) float hs[];
  const int H2 = cH2 ? cH2 : 2 * s.H, B = cB ? cB : s.B, V = cV ? cV : s.V;
  float* W1s = hs;                   // [H2][B+1]
  float* W2s = W1s + H2 * (B + 1);   // [B][V+1]
  float* b1s = W2s + B * (V + 1);
  float* b2s = b1s + B;
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * kHeadWarps + wl;
  const bool live = r < s.R;
  float* f = hs + (kSmemW ? head_w_floats(H2, B, V) : 0) + wl * (H2 + 2 * B + V);  // fin, bact, dbact, g
  float* ba = f + H2;
  float* db = ba + B;
  float* gr = db + B;
  pdl_wait();
  // every load of the step is issued before the first wait: the target token,
  // the row's fin, and (kSmemW) the weights and biases, element-wise into the
  // padded rows
  const uint32_t tgt = live ? tokens[*pos + r] & uint32_t(V - 1) : 0u;
  if (live)
    for (int p = lane; p < H2; p += 32) cp_async4(f + p, fin + int64_t(r) * H2 + p);
  if (kSmemW) {
    const int n1 = H2 * B, n2 = B * V;
    for (int e = threadIdx.x; e < n1 + n2 + B + V; e += blockDim.x) {
      if (e < n1) cp_async4(W1s + (e / B) * (B + 1) + e % B, w1 + e);
      else if (e < n1 + n2) cp_async4(W2s + ((e - n1) / V) * (V + 1) + (e - n1) % V, w2 + (e - n1));
      else if (e < n1 + n2 + B) cp_async4(b1s + (e - n1 - n2), b1 + (e - n1 - n2));
      else cp_async4(b2s + (e - n1 - n2 - B), b2 + (e - n1 - n2 - B));
    }
  }
  asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (!live) return;
  // W1(p, j) = bott.w[p][j], W2(q, i) = out.w[q][i]; the backward walks the
  // same copies by column
  auto W1 = [&](int p, int j) { return kSmemW ? W1s[p * (B + 1) + j] : w1[int64_t(p) * B + j]; };
  auto W2 = [&](int q, int i) { return kSmemW ? W2s[q * (V + 1) + i] : w2[int64_t(q) * V + i]; };
  auto W2T = [&](int o, int j) { return W2(j, o); };
  auto W1T = [&](int j, int p) { return W1(p, j); };
  auto B1 = [&](int j) { return kSmemW ? b1s[j] : b1[j]; };
  auto B2 = [&](int i) { return kSmemW ? b2s[i] : b2[i]; };
  // bact = tanh(bott.b + fin.W1), ascending p
#pragma unroll
  for (int j = lane; j < B; j += 32) {
    float acc = B1(j);
#pragma unroll 8
    for (int p = 0; p < H2; ++p) acc = mac(acc, f[p], W1(p, j));
    acc = det_tanh(acc);
    ba[j] = acc;
    bact_out[int64_t(r) * B + j] = acc;
  }
  __syncwarp();
  // logits = out.b + bact.W2, ascending q
  float mx = -__int_as_float(0x7f800000);
#pragma unroll
  for (int i = lane; i < V; i += 32) {
    float acc = B2(i);
#pragma unroll 8
    for (int q = 0; q < B; ++q) acc = mac(acc, ba[q], W2(q, i));
    gr[i] = acc;
    mx = fmaxf(mx, acc);
  }
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __syncwarp();
  // det_softmax (detmath.cpp:85-97): exp of the shifted logits, then one
  // sequential sum in index order (lane 0 over shared memory)
#pragma unroll
  for (int i = lane; i < V; i += 32) gr[i] = det_exp(fsub(gr[i], mx));
  __syncwarp();
  float sum = 0.0f;
  if (lane == 0) {
    int i = 0;
    if ((V & 3) == 0 && ((H2 + 2 * B) & 3) == 0)  // gr is 16-byte aligned
#pragma unroll 4
      for (; i < V; i += 4) {
        const float4 e4 = *reinterpret_cast<const float4*>(gr + i);
        sum = fadd(fadd(fadd(fadd(sum, e4.x), e4.y), e4.z), e4.w);
      }
    for (; i < V; ++i) sum = fadd(sum, gr[i]);
  }
  sum = __shfl_sync(0xffffffffu, sum, 0);
  const float inv = fdiv(1.0f, sum);
#pragma unroll
  for (int i = lane; i < V; i += 32) {
    float v = fmul(gr[i], inv);
    if (uint32_t(i) == tgt) v = fsub(v, 1.0f);
    gr[i] = v;
    g_out[int64_t(r) * V + i] = v;
  }
  __syncwarp();
  // dbact = (0 + g.W2^T) * (1 - bact^2), ascending o
#pragma unroll
  for (int j = lane; j < B; j += 32) {
    float acc = 0.0f;
#pragma unroll 8
    for (int o = 0; o < V; ++o) acc = mac(acc, gr[o], W2T(o, j));
    const float a = ba[j];
    acc = fmul(acc, fsub(1.0f, fmul(a, a)));
    db[j] = acc;
    dbact_out[int64_t(r) * B + j] = acc;
  }
  __syncwarp();
  // dfin = 0 + dbact.W1^T, ascending j
#pragma unroll
  for (int p = lane; p < H2; p += 32) {
    float acc = 0.0f;
#pragma unroll 8
    for (int j = 0; j < B; ++j) acc = mac(acc, db[j], W1T(j, p));
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
  const float dlast = s.dout ? 0.0f : fadd(0.0f, dfin[int64_t(r) * 2 * H + d * H + j]);
  float dh = 0.0f;
  for (int t = T - 1; t >= 0; --t) {
    // gather_add_step(dout, t, dh): the output gradient of this own step
    // (a deeper layer's dx at position src_t, half d), else the final-state
    // gradient at the last step
    const float dadd = s.dout ? s.dout[(int64_t(r) * T + (d ? T - 1 - t : t)) * 2 * H + d * H + j]
                              : (t == T - 1 ? dlast : 0.0f);
    dh = fadd(dh, dadd);
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
constexpr int kBpttWarps = 2;
constexpr int kPubSteps = 8;  // BPTT progress published per group of steps
constexpr int kBpttAhead = 8;  // tape staging depth (steps)
__device__ __forceinline__ void cp_async4_sp(float* smem, const float* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
               "l"(gmem));
}
// cnt (nullable): per (direction, step) count of rows whose step is stored,
// published with a release add after each step (the streamed reductions of
// k_sprm_nt_stream wait on it)
__global__ void __launch_bounds__(kBpttWarps * 32) k_sprm_bptt32(SprmP s, const float* __restrict__ tape,
                                                                 const float* __restrict__ dfin, float* Gt,
                                                                 unsigned* cnt) {
  pdl_wait();
  constexpr int H = 32;
  __shared__ __align__(16) float sg[kBpttWarps][3][H];  // dhh, dar, daz of this step
  __shared__ float stape[kBpttWarps][kBpttAhead][5][H];  // staged tape values
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
  const float dlast = s.dout ? 0.0f : fadd(0.0f, dfin[int64_t(r) * 2 * H + d * H + j]);
  // The step's tape values (r, z, n, hh and h_{t-1} for this lane's unit)
  // are staged kBpttAhead steps ahead by per-lane 4-byte async copies into a
  // per-warp shared ring (each lane copies and reads only its own unit, so
  // no barrier), keeping global-load latency out of the step loop.
  auto issue = [&](int t) {  // step t's five values into ring slot t % kBpttAhead
    if (t >= 0) {
      const int64_t o = (int64_t(t) * R + r) * H + j;
      float* dst = &stape[wl][t % kBpttAhead][0][j];
#pragma unroll
      for (int g = 0; g < 4; ++g) cp_async4_sp(dst + g * H, tp[g] + o);
      if (t > 0) cp_async4_sp(dst + 4 * H, tp[4] + o - int64_t(R) * H);
      else dst[4 * H] = 0.0f;
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
#pragma unroll
  for (int i = 0; i < kBpttAhead - 1; ++i) issue(T - 1 - i);
  float xc[5];
  float dh = 0.0f;
  for (int t = T - 1; t >= 0; --t) {
    issue(t - (kBpttAhead - 1));
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kBpttAhead - 1));
#pragma unroll
    for (int g = 0; g < 5; ++g) xc[g] = stape[wl][t % kBpttAhead][g][j];
    // gather_add_step(dout, t, dh): a deeper layer's output gradient at
    // position src_t (half d), else the final-state gradient at the last step
    const float dadd = s.dout ? s.dout[(int64_t(r) * T + (d ? T - 1 - t : t)) * 2 * H + d * H + j]
                              : (t == T - 1 ? dlast : 0.0f);
    dh = fadd(dh, dadd);
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
    __syncwarp();  // also orders the lanes' stores before lane 0's release
    // one release per kPubSteps steps (the group's lowest step): the fence
    // waits for the warp's stores to land, so it is amortised over the group
    if (cnt && lane == 0 && (t % kPubSteps) == 0)
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt + d * T + t / kPubSteps)
                   : "memory");
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
  }
}

// ---------------------------------------------------------------------------
// Streamed BPTT + weight-gradient reductions (H == 32). The 12 reductions
// (dW_i{n,r,z} over the GRU inputs, dW_h{n,r,z} over h_{t-1}, and the bias
// sums) accumulate in the reference's order k = (T-1-t)*R + r: time
// descending, rows ascending -- exactly the order backward-through-time
// produces the gate gradients. So one launch holds both: BPTT blocks (warp per
// row, k_sprm_bptt32's body) publish each finished step with a per-(dir, step)
// row counter; consumer blocks, one per (direction, gate) slab of output rows,
// wait for the counter, pull the step's gradient slab Gt[g][d][t] ([R][32]),
// the h_{t-1} slab (Gt[4][d][t], written by BPTT beside the gradients) and the
// input slab Xtm[d][t] ([R][Es], from the prep kernel) into shared memory
// with bulk async copies (a producer warp, double-buffered, mbarrier
// complete_tx), and advance their chains one step behind BPTT. A consumer
// lane owns output column j = lane of two output rows as one paired exact
// chain (acc + a*b, a from the A slab, b = Gt[g][d][t][r][j]; the bias rows
// use a = 1). Consumers only wait on BPTT, never the reverse, so the launch
// cannot deadlock whatever the block placement. Replaces the transpose and
// the batched NT reduction (which started only after BPTT ended).
struct NtSRow {
  int kind;      // 0: input row p (Xtm), 1: h_{t-1} row p, 2: bias (a = 1), -1: none
  int p;
  float* out0;   // output row: element j at out0[j]
  float* out1;   // a second destination of the same chain (the b_i*/b_h* pair), or null
};
struct NtSWarp {
  int g;         // gradient slab: 0 an, 1 ar, 2 az, 3 hh
  NtSRow r0, r1;
};
struct NtSParams {
  const float* tape;
  const float* dfin;
  float* Gt;
  const float* Xtm;        // [2][T][R][Es]
  unsigned* cnt;           // [2][T] rows finished per (dir, step)
  const NtSWarp* warps;    // consumer warp table, 4 per block, (d, g) uniform per block
  const int* block_dg;     // per consumer block: d * 4 + g
  int nb_bptt;             // unused (0)
};
constexpr int kStreamConsumers = 8;

__device__ __forceinline__ uint32_t sm_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_addr(bar)) : "memory");
}
// One consumer step of a paired chain: acc += (a[r].x, a[r].y) * b[r] for r
// ascending, a and b in shared memory (a: 8-byte pair, stride a_st bytes;
// b: stride 128 bytes). A three-stage software pipeline in program order --
// the add of batch k, the products of batch k+1, the loads of batch k+2 --
// written with volatile asm so the schedule keeps it: each add then only
// waits for the previous add (the chain's 4-cycle latency), never for a load
// or a product.
__device__ __forceinline__ void lds_pair(f2_t& x, float& y, uint32_t a, uint32_t b) {
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(x) : "r"(a));
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(y) : "r"(b));
}
__device__ __forceinline__ f2_t prod_v(f2_t x, float y) {
  f2_t out;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(out) : "l"(x), "l"(f2_bcast(y)), "l"(c_negzero2));
  return out;
}
__device__ __forceinline__ void add_v(f2_t& acc, f2_t p) {
  asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(p));
}
// batch k's adds, batch k+1's products (from LN), batch k+2's loads (into LL)
template <int kU>
__device__ __forceinline__ void nt_stage(f2_t& acc, f2_t (&P)[kU], f2_t (&LN)[kU], float (&LNb)[kU],
                                         f2_t (&LL)[kU], float (&LLb)[kU], bool more1, bool more2,
                                         uint32_t a2, uint32_t b2, uint32_t a_st) {
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    add_v(acc, P[u]);
    if (more1) P[u] = prod_v(LN[u], LNb[u]);
    if (more2) lds_pair(LL[u], LLb[u], a2 + uint32_t(u) * a_st, b2 + uint32_t(u) * 128u);
  }
}
__device__ __forceinline__ f2_t nt_chain_pair(f2_t acc, uint32_t a, uint32_t a_st, uint32_t b, int R) {
  constexpr int kU = 8;
  const int nb = R / kU;
  f2_t L0[kU], L1[kU], P[kU];
  float B0[kU], B1[kU];
  if (nb > 0) {
#pragma unroll
    for (int u = 0; u < kU; ++u) lds_pair(L0[u], B0[u], a + uint32_t(u) * a_st, b + uint32_t(u) * 128u);
    if (nb > 1) {
#pragma unroll
      for (int u = 0; u < kU; ++u)
        lds_pair(L1[u], B1[u], a + uint32_t(kU + u) * a_st, b + uint32_t(kU + u) * 128u);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) P[u] = prod_v(L0[u], B0[u]);
    int k = 0;
    for (; k + 2 <= nb; k += 2) {
      nt_stage<kU>(acc, P, L1, B1, L0, B0, k + 1 < nb, k + 2 < nb, a + uint32_t((k + 2) * kU) * a_st,
                   b + uint32_t((k + 2) * kU) * 128u, a_st);
      nt_stage<kU>(acc, P, L0, B0, L1, B1, k + 2 < nb, k + 3 < nb, a + uint32_t((k + 3) * kU) * a_st,
                   b + uint32_t((k + 3) * kU) * 128u, a_st);
    }
    if (k < nb) nt_stage<kU>(acc, P, L1, B1, L0, B0, false, false, 0, 0, a_st);
  }
  for (int r = nb * kU; r < R; ++r) {
    f2_t x;
    float y;
    lds_pair(x, y, a + uint32_t(r) * a_st, b + uint32_t(r) * 128u);
    add_v(acc, prod_v(x, y));
  }
  return acc;
}

// bounded waits: a protocol error traps (a loud launch failure) instead of
// hanging the device
constexpr unsigned long long kSpinLimit = 1ull << 28;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (unsigned long long i = 0;; ++i) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(sm_addr(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (i > kSpinLimit) __trap();
  }
}
// the producer's waits leave the issue slots to the consumer warps
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  for (unsigned long long i = 0;; ++i) {
    uint32_t done;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(sm_addr(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (i > kSpinLimit) __trap();
    __nanosleep(64);
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          sm_addr(dst)),
      "l"(src), "r"(bytes), "r"(sm_addr(bar))
      : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// The consumer blocks (one per (direction, gate) slab of output rows, 4
// consumer warps + 1 producer warp) run as their own launch on a side stream,
// beside the BPTT launch (k_sprm_bptt32 with the per-step counters): they
// only wait on BPTT, and BPTT blocks (small shared memory) still fit next to
// them on every SM, so the pair cannot deadlock.
__global__ void __launch_bounds__((kStreamConsumers + 1) * 32, 1) k_sprm_nt_stream(SprmP s, NtSParams q) {
  pdl_wait();
  constexpr int H = 32;
  const int T = s.T, R = s.R, Es = s.Es;
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ---------------- weight-gradient consumers
  extern __shared__ __align__(128) float sbuf[];  // [2][ B [R][32] | Hp [R][32] | X [R][Es] ]
  __shared__ uint64_t full[2], empty[2];
  const int cb = int(blockIdx.x);
  const int dg = q.block_dg[cb], d = (dg >> 2) & 1, g = dg & 3;
  const bool need_h = (dg >> 8) & 1, need_x = (dg >> 9) & 1;  // the block's A slabs
  const int slab = R * (2 * H + Es);
  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], kStreamConsumers);
    mbar_init(&empty[1], kStreamConsumers);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wl == kStreamConsumers) {  // producer warp
    if (lane == 0) {
      const uint32_t bB = uint32_t(R) * H * 4, bX = uint32_t(R) * Es * 4;
      for (int i = 0; i < T; ++i) {
        const int t = T - 1 - i, b = i & 1;
        if (i >= 2) mbar_wait_sleep(&empty[b], ((i >> 1) - 1) & 1);  // consumers done with step i-2
        const unsigned* c = q.cnt + d * T + t / kPubSteps;  // group of step t complete
        for (unsigned long long k = 0; ld_acquire(c) < unsigned(R); ++k) {
          if (k > kSpinLimit) __trap();
          __nanosleep(32);
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
        float* base = sbuf + b * slab;
        mbar_arrive_tx(&full[b], bB + (need_h ? bB : 0) + (need_x ? bX : 0));
        bulk_g2s(base, q.Gt + (int64_t(g * 2 + d) * T + t) * R * H, bB, &full[b]);
        if (need_h) bulk_g2s(base + R * H, q.Gt + (int64_t(4 * 2 + d) * T + t) * R * H, bB, &full[b]);
        if (need_x) bulk_g2s(base + 2 * R * H, q.Xtm + (int64_t(d) * T + t) * R * Es, bX, &full[b]);
      }
    }
    return;
  }
  const NtSWarp wk = q.warps[cb * kStreamConsumers + wl];
  if (wk.r0.kind < 0) {  // idle warp: still releases the buffers
    for (int i = 0; i < T; ++i) {
      mbar_wait(&full[i & 1], (i >> 1) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[i & 1]);
    }
    return;
  }
  // A source of each row inside a buffer: offset and row stride (floats)
  auto a_off = [&](const NtSRow& rw, int& stride) {
    if (rw.kind == 0) { stride = Es; return 2 * R * H + rw.p; }
    if (rw.kind == 1) { stride = H; return R * H + rw.p; }
    stride = 0;
    return -1;  // bias / none: a = 1
  };
  int st0 = 0, st1 = 0;
  const int o0 = a_off(wk.r0, st0), o1 = a_off(wk.r1, st1);
  f2_t acc = f2_pack(wk.r0.out0 ? wk.r0.out0[lane] : 0.0f, wk.r1.out0 ? wk.r1.out0[lane] : 0.0f);
  for (int i = 0; i < T; ++i) {
    const int b = i & 1;
    mbar_wait(&full[b], (i >> 1) & 1);
    const float* base = sbuf + b * slab;
    const float* bs = base + lane;
    const float* a0 = o0 >= 0 ? base + o0 : nullptr;
    const float* a1 = o1 >= 0 ? base + o1 : nullptr;
    if (a0 && a1 && st0 == st1 && o1 == o0 + 1 && (o0 & 1) == 0) {
      acc = nt_chain_pair(acc, sm_addr(a0), uint32_t(st0) * 4, sm_addr(bs), R);
    } else if (!a0 && !a1) {  // bias row(s): a = 1, and 1*b == b exactly
      for (int r = 0; r < R; ++r) acc = f2_add(acc, f2_bcast(bs[r * H]));
    } else {
      constexpr int kU = 8;
      int r = 0;
      for (; r + kU <= R; r += kU) {
        float x0[kU], x1[kU], bv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          x0[u] = a0 ? a0[(r + u) * st0] : 1.0f;
          x1[u] = a1 ? a1[(r + u) * st1] : 1.0f;
          bv[u] = bs[(r + u) * H];
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) acc = f2_add(acc, f2_mul(f2_pack(x0[u], x1[u]), f2_bcast(bv[u])));
      }
      for (; r < R; ++r) {
        const float x0 = a0 ? a0[r * st0] : 1.0f, x1 = a1 ? a1[r * st1] : 1.0f;
        acc = f2_add(acc, f2_mul(f2_pack(x0, x1), f2_bcast(bs[r * H])));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
  }
  const float v0 = f2_lo(acc), v1 = f2_hi(acc);
  if (wk.r0.out0) wk.r0.out0[lane] = v0;
  if (wk.r0.out1) wk.r0.out1[lane] = v0;
  if (wk.r1.out0) wk.r1.out0[lane] = v1;
  if (wk.r1.out1) wk.r1.out1[lane] = v1;
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
__global__ void __launch_bounds__(256) k_sprm_dx_t(SprmP s, const float* __restrict__ Gt, float* dx,
                                                   const uint16_t* __restrict__ rank) {
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
  const float v = fadd(fadd(0.0f, part[0]), fadd(0.0f, part[1]));  // dx += dx_rev (both from zero)
  // sorted store for the embedding gradient walk: row rt goes to its rank
  if (rank) dx[int64_t(rank[rt]) * Es + i] = v;
  else dx[idx] = v;
}

// Embedding::backward (layers.cpp:117-125) split in two: the ctx tokens of a
// train step are known before its forward, so a stable counting sort of the
// R*T positions by token (k_tok_sort, one block, beside the forward) leaves
// only the gradient walk after dx (k_emb_walk): thread per (token, feature),
// its positions in (r, t) order -- the reference's order for that element --
// with the gathers issued ahead of the add chain.
constexpr int kSortBlock = 1024, kSortMaxTok = 256;
__global__ void __launch_bounds__(kSortBlock) k_tok_sort(const uint32_t* __restrict__ ctx, int n, int V,
                                                         uint16_t* order, int* offs, uint16_t* rank) {
  pdl_wait();
  __shared__ int cnt[kSortBlock / 32][kSortMaxTok];
  __shared__ int tot[kSortMaxTok + 1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kSortBlock / 32;
  const int span = (n + nw - 1) / nw, p0 = w * span, p1 = min(n, p0 + span);
  for (int v = lane; v < V; v += 32) cnt[w][v] = 0;
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  for (int c = p0; c < p1; c += 32) {
    const int p = c + lane;
    const uint32_t v = p < p1 ? ctx[p] & uint32_t(V - 1) : 0xffffffffu;
    const unsigned m = __match_any_sync(0xffffffffu, v);
    if (p < p1 && (m & lt) == 0) cnt[w][v] += __popc(m);
    __syncwarp();
  }
  __syncthreads();
  // totals per token, exclusive scan over tokens (V <= 256: one warp per 32)
  if (threadIdx.x < V) {
    int sum = 0;
    for (int ww = 0; ww < nw; ++ww) sum += cnt[ww][threadIdx.x];
    tot[threadIdx.x] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    for (int v = 0; v < V; ++v) {
      const int x = tot[v];
      tot[v] = a;
      offs[v] = a;
      a += x;
    }
    offs[V] = a;
  }
  __syncthreads();
  if (threadIdx.x < V) {  // per-warp cursors in (token, warp) order
    int a = tot[threadIdx.x];
    for (int ww = 0; ww < nw; ++ww) {
      const int x = cnt[ww][threadIdx.x];
      cnt[ww][threadIdx.x] = a;
      a += x;
    }
  }
  __syncthreads();
  for (int c = p0; c < p1; c += 32) {
    const int p = c + lane;
    const uint32_t v = p < p1 ? ctx[p] & uint32_t(V - 1) : 0xffffffffu;
    const unsigned m = __match_any_sync(0xffffffffu, v);
    if (p < p1) {
      const int k = cnt[w][v] + __popc(m & lt);
      order[k] = uint16_t(p);
      rank[p] = uint16_t(k);
    }
    __syncwarp();
    if (p < p1 && (m & lt) == 0) cnt[w][v] += __popc(m);
    __syncwarp();
  }
}

// walk over dx already stored in sorted order (dxs[k][i], k = rank of the
// position): thread per token, all E feature chains at once, contiguous loads
template <int E>
__global__ void k_emb_walk_sorted(const int* __restrict__ offs, const float* __restrict__ dxs,
                                  float* grad, int V) {
  pdl_wait();
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int k0 = offs[v], k1 = offs[v + 1];
  float acc[E];
#pragma unroll
  for (int i = 0; i < E; ++i) acc[i] = grad[v * E + i];
  constexpr int kU = 8;
  int k = k0;
  for (; k + kU <= k1; k += kU) {
    float x[kU][E];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int i = 0; i < E; ++i) x[u][i] = __ldg(dxs + int64_t(k + u) * E + i);
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int i = 0; i < E; ++i) acc[i] = fadd(acc[i], x[u][i]);
  }
  for (; k < k1; ++k)
#pragma unroll
    for (int i = 0; i < E; ++i) acc[i] = fadd(acc[i], __ldg(dxs + int64_t(k) * E + i));
#pragma unroll
  for (int i = 0; i < E; ++i) grad[v * E + i] = acc[i];
}

// same walk with the sorted dx staged in shared memory first (one block):
// the staging is one coalesced sweep with every load in flight, and the
// per-token chains then read LDS.128s issued a batch ahead
template <int E>
__global__ void __launch_bounds__(1024, 1) k_emb_walk_smem(const int* __restrict__ offs,
                                                        const float* __restrict__ dxs, float* grad,
                                                        int V, int n) {
  pdl_wait();
  extern __shared__ __align__(16) float sx[];  // [n][E]
  const int nf4 = n * E / 4;
  const float4* src = reinterpret_cast<const float4*>(dxs);
  float4* dst = reinterpret_cast<float4*>(sx);
  constexpr int kU = 8;
  for (int i0 = threadIdx.x; i0 < nf4; i0 += kU * blockDim.x) {
    float4 x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < nf4) x[u] = __ldg(src + i);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < nf4) dst[i] = x[u];
    }
  }
  __syncthreads();
  const int v = threadIdx.x;
  if (v >= V) return;
  const int k0 = offs[v], k1 = offs[v + 1];
  float acc[E];
#pragma unroll
  for (int i = 0; i < E; ++i) acc[i] = grad[v * E + i];
  int k = k0;
  for (; k + kU <= k1; k += kU) {
    float x[kU][E];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int i = 0; i < E; ++i) x[u][i] = sx[(k + u) * E + i];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int i = 0; i < E; ++i) acc[i] = fadd(acc[i], x[u][i]);
  }
  for (; k < k1; ++k)
#pragma unroll
    for (int i = 0; i < E; ++i) acc[i] = fadd(acc[i], sx[k * E + i]);
#pragma unroll
  for (int i = 0; i < E; ++i) grad[v * E + i] = acc[i];
}

__global__ void k_emb_walk(const uint16_t* __restrict__ order, const int* __restrict__ offs,
                           const float* __restrict__ dx, float* grad, int V, int E) {
  pdl_wait();
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= V * E) return;
  const int v = id / E, i = id % E;
  const int k0 = offs[v], k1 = offs[v + 1];
  float acc = grad[id];
  constexpr int kU = 8;
  int k = k0;
  for (; k + kU <= k1; k += kU) {
    float x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) x[u] = __ldg(dx + int64_t(order[k + u]) * E + i);
#pragma unroll
    for (int u = 0; u < kU; ++u) acc = fadd(acc, x[u]);
  }
  for (; k < k1; ++k) acc = fadd(acc, __ldg(dx + int64_t(order[k]) * E + i));
  grad[id] = acc;
}

// Layer-1 input of a 2-layer BiGRU (BiGru::forward output concat,
// layers.cpp:355-366): x1[r][pos] = [h_fwd(own time pos) | h_bwd(own time T-1-pos)]
__global__ void k_bigru_concat(const float* __restrict__ tape, float* x1, int R, int T, int H) {
  pdl_wait();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t n = int64_t(R) * T * 2 * H;
  if (i >= n) return;
  const int j2 = int(i % (2 * H));
  const int64_t rp = i / (2 * H);
  const int r = int(rp / T), pos = int(rp % T);
  const int d = j2 >= H ? 1 : 0, j = j2 - d * H;
  const int t = d ? T - 1 - pos : pos;
  const int64_t TRH = int64_t(T) * R * H;
  x1[i] = tape[int64_t(4 * 2 + d) * TRH + (int64_t(t) * R + r) * H + j];
}

// feature-major reduction operand of a deeper layer's input: Xf[d][i][k],
// k = (T-1-t)*R + r, = x1 at the direction's own time t (position src_t)
__global__ void k_bigru_xf(const float* __restrict__ x1, float* Xf, int R, int T, int In) {
  pdl_wait();
  const int64_t RT = int64_t(R) * T;
  const int64_t id = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (id >= 2 * In * RT) return;
  const int64_t k = id % RT;
  const int64_t rest = id / RT;
  const int i = int(rest % In), d = int(rest / In);
  const int t = int(T - 1 - k / R), r = int(k % R);
  const int src_t = d ? (T - 1 - t) : t;
  Xf[id] = x1[(int64_t(r) * T + src_t) * In + i];
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

// Adam for the single-model trainers (SPrM pre-pass, pretrain_public) in one
// launch: k_adam_scalars' bias-correction sequence formed by every thread
// from the previous scalars (the same operations, so the same values), the
// update of k_adam, then the last block to finish publishes the new scalars and
// advances pos (every block has read the old scalars before it counts itself
// done, so none reads the new ones).
__global__ void __launch_bounds__(256) k_sprm_adam(float* __restrict__ w, float* __restrict__ g,
                                                   float* __restrict__ m, float* __restrict__ v, int64_t n,
                                                   AdamScalars* sc, int64_t* pos, int64_t by,
                                                   unsigned* done) {
  pdl_wait();
  AdamScalars a = *sc;
  a.step += 1;
  a.b1p = fmul(a.b1p, 0.9f);
  a.b2p = fmul(a.b2p, 0.999f);
  a.bc1 = fsub(1.0f, a.b1p);
  a.bc2 = fsub(1.0f, a.b2p);
  const float b1 = 0.9f, b2 = 0.999f, lr = 5e-4f, eps = 1e-8f;
  const float omb1 = fsub(1.0f, b1), omb2 = fsub(1.0f, b2);
  constexpr int U = 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    float gi[U], mo[U], vo[U], wo[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        gi[u] = g[i];
        mo[u] = m[i];
        vo[u] = v[i];
        wo[u] = w[i];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        const float mi = fadd(fmul(b1, mo[u]), fmul(omb1, gi[u]));
        const float vi = fadd(fmul(b2, vo[u]), fmul(fmul(omb2, gi[u]), gi[u]));
        const float mhat = fdiv(mi, a.bc1);
        const float vhat = fdiv(vi, a.bc2);
        w[i] = fsub(wo[u], fdiv(fmul(lr, mhat), fadd(__fsqrt_rn(vhat), eps)));
        m[i] = mi;
        v[i] = vi;
        g[i] = 0.0f;
      }
    }
  }
  __syncthreads();  // the block's reads of *sc are done
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *sc = a;
      *pos += by;
      *done = 0u;
    }
  }
}

__global__ void k_pos_advance(int64_t* pos, int64_t by) {
  pdl_wait(); *pos += by; }

}  // namespace

void launch_sprm_prep(const uint32_t* tokens, const int64_t* pos, const SprmP& s, uint32_t* ctx,
                      float* X, float* tab, float* Xtm, unsigned* cnt, cudaStream_t st) {
  const int64_t n = std::max<int64_t>(std::max<int64_t>(int64_t(s.R) * s.T, 6ll * s.V * s.H),
                                      2ll * s.Es * s.R * s.T);
  launch_pdl(k_sprm_prep, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, tokens, pos, s, ctx, X, tab,
             Xtm, cnt);
}

// Off by default (PMKLC_SPRM_STREAM=1 enables it): measured on the B200 the
// consumers advance ~4 us per step against BPTT's ~1 us, so the streamed
// reductions end ~120 us after BPTT instead of ~62 us for transpose + batched
// NT. Kept, parity-green, for further work.
bool sprm_stream_ok(const SprmP& s) {
  static const bool on = [] {
    const char* e = std::getenv("PMKLC_SPRM_STREAM");
    return e && std::atoi(e) != 0;
  }();
  return on && s.H == 32 && s.Es >= 1 && s.Es <= 8 && (s.Es % 2 == 0) &&
         size_t(2) * s.R * (64 + s.Es) * sizeof(float) <= 200 * 1024;
}

// consumer warp table of the streamed BPTT (see k_sprm_bptt_stream): per
// (direction, gate slab) the output rows in pairs of one kind, 4 warps a block
struct NtSPlan {
  std::vector<NtSWarp> warps;
  std::vector<int> block_dg;
};
static NtSPlan nt_stream_plan(const SprmP& s, float* g, const int64_t* hoffs) {
  NtSPlan pl;
  const int H = s.H, Es = s.Es;
  auto G = [&](int d, int t) { return g + hoffs[1 + d * NG + t]; };
  for (int d = 0; d < 2; ++d)
    for (int gate = 0; gate < 4; ++gate) {
      std::vector<NtSWarp> ws;
      auto pairs = [&](int kind, int n, float* W) {
        for (int p = 0; p < n; p += 2) {
          NtSWarp w{};
          w.g = gate;
          w.r0 = NtSRow{kind, p, W + int64_t(p) * H, nullptr};
          w.r1 = p + 1 < n ? NtSRow{kind, p + 1, W + int64_t(p + 1) * H, nullptr}
                           : NtSRow{-1, 0, nullptr, nullptr};
          ws.push_back(w);
        }
      };
      const int wi = gate == 0 ? WIN : gate == 1 ? WIR : WIZ;
      const int wh = gate == 3 ? WHN : gate == 1 ? WHR : WHZ;
      const int bi = gate == 0 ? BIN : gate == 1 ? BIR : BIZ;
      const int bh = gate == 3 ? BHN : gate == 1 ? BHR : BHZ;
      if (gate != 3) pairs(0, Es, G(d, wi));
      if (gate != 0) pairs(1, H, G(d, wh));
      NtSWarp wb{};
      wb.g = gate;
      // the bias rows: sum of the gate gradient (b_in / b_hn alone; b_ir and
      // b_hr, b_iz and b_hz are the same chain, stored twice)
      float* b0 = gate == 3 ? G(d, bh) : G(d, bi);
      float* b1 = (gate == 1 || gate == 2) ? G(d, bh) : nullptr;
      wb.r0 = NtSRow{2, 0, b0, b1};
      wb.r1 = NtSRow{-1, 0, nullptr, nullptr};
      ws.push_back(wb);
      for (size_t i = 0; i < ws.size(); i += kStreamConsumers) {
        int need_h = 0, need_x = 0;
        for (int k = 0; k < kStreamConsumers; ++k) {
          NtSWarp w{};
          w.g = gate;
          w.r0 = w.r1 = NtSRow{-1, 0, nullptr, nullptr};
          const NtSWarp& x = i + k < ws.size() ? ws[i + k] : w;
          need_h |= (x.r0.kind == 1 || x.r1.kind == 1) ? 1 : 0;
          need_x |= (x.r0.kind == 0 || x.r1.kind == 0) ? 1 : 0;
          pl.warps.push_back(x);
        }
        pl.block_dg.push_back(d * 4 + gate + (need_h << 8) + (need_x << 9));
      }
    }
  return pl;
}

size_t sprm_stream_table_bytes(const SprmP& s) {
  const NtSPlan pl = nt_stream_plan(s, nullptr, std::vector<int64_t>(1 + 2 * NG, 0).data());
  return pl.warps.size() * sizeof(NtSWarp) + pl.block_dg.size() * sizeof(int);
}

void sprm_stream_table(const SprmP& s, float* g, const int64_t* hoffs, void* host_buf) {
  const NtSPlan pl = nt_stream_plan(s, g, hoffs);
  unsigned char* b = static_cast<unsigned char*>(host_buf);
  std::memcpy(b, pl.warps.data(), pl.warps.size() * sizeof(NtSWarp));
  std::memcpy(b + pl.warps.size() * sizeof(NtSWarp), pl.block_dg.data(), pl.block_dg.size() * sizeof(int));
}

void launch_sprm_bptt_stream(const SprmP& s, const float* tape, const float* dfin, float* Gt,
                             const float* Xtm, unsigned* cnt, const void* d_table, cudaStream_t st,
                             cudaStream_t side) {
  const NtSPlan pl = nt_stream_plan(s, nullptr, std::vector<int64_t>(1 + 2 * NG, 0).data());
  NtSParams q{};
  q.tape = tape;
  q.dfin = dfin;
  q.Gt = Gt;
  q.Xtm = Xtm;
  q.cnt = cnt;
  q.warps = static_cast<const NtSWarp*>(d_table);
  q.block_dg = reinterpret_cast<const int*>(static_cast<const unsigned char*>(d_table) +
                                            pl.warps.size() * sizeof(NtSWarp));
  q.nb_bptt = 0;
  const size_t smem = size_t(2) * s.R * (2 * s.H + s.Es) * sizeof(float);
  ensure_smem(reinterpret_cast<const void*>(k_sprm_nt_stream), smem);
  launch_pdl(k_sprm_nt_stream, dim3(unsigned(pl.block_dg.size())), dim3((kStreamConsumers + 1) * 32),
             smem, side, s, q);
  launch_pdl(k_sprm_bptt32, dim3(unsigned(2 * ((s.R + kBpttWarps - 1) / kBpttWarps))),
             dim3(kBpttWarps * 32), 0, st, s, tape, dfin, Gt, cnt);
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
        s, tape, dfin, Gt, static_cast<unsigned*>(nullptr));
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
void launch_sprm_dx(const SprmP& s, const float* G, const float* Gt, float* dx, cudaStream_t st,
                    const uint16_t* rank) {
  const int64_t n = int64_t(s.R) * s.T * s.Es;
  if (sprm_dx_time_major(s) && Gt) {
    launch_pdl(k_sprm_dx_t, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, s, Gt, dx, rank);
    return;
  }
  launch_pdl(k_sprm_dx, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, s, G, dx);
}
void launch_sprm_head(const SprmP& s, const uint32_t* tokens, const int64_t* pos, const float* fin,
                      const float* w1, const float* b1, const float* w2, const float* b2, float* bact,
                      float* g, float* dbact, float* dfin, cudaStream_t st) {
  const size_t rows_smem = size_t(kHeadWarps) * (2 * s.H + 2 * s.B + s.V) * sizeof(float);
  const size_t w_smem = size_t(head_w_floats(2 * s.H, s.B, s.V)) * sizeof(float);
  const dim3 grid(unsigned((s.R + kHeadWarps - 1) / kHeadWarps)), block(kHeadWarps * 32);
  if (s.H == 32 && s.B == 32 && s.V == 64) {  // the default SPrM widths
    auto k = k_sprm_head<true, 64, 32, 64>;
    ensure_smem(reinterpret_cast<const void*>(k), w_smem + rows_smem);
    launch_pdl(k, grid, block, w_smem + rows_smem, st, s, tokens, pos, fin, w1, b1, w2, b2, bact, g,
               dbact, dfin);
  } else if (w_smem + rows_smem <= 64 * 1024) {
    ensure_smem(reinterpret_cast<const void*>(k_sprm_head<true>), w_smem + rows_smem);
    launch_pdl(k_sprm_head<true>, grid, block, w_smem + rows_smem, st, s, tokens, pos, fin, w1, b1, w2,
               b2, bact, g, dbact, dfin);
  } else {
    ensure_smem(reinterpret_cast<const void*>(k_sprm_head<false>), rows_smem);
    launch_pdl(k_sprm_head<false>, grid, block, rows_smem, st, s, tokens, pos, fin, w1, b1, w2, b2,
               bact, g, dbact, dfin);
  }
}
bool sprm_sorted_emb_ok(const SprmP& s) { return s.V <= kSortMaxTok && s.R * s.T <= 65536; }
void launch_tok_sort(const uint32_t* ctx, int n, int V, uint16_t* order, int* offs, uint16_t* rank,
                     cudaStream_t st) {
  launch_pdl(k_tok_sort, dim3(1), dim3(kSortBlock), 0, st, ctx, n, V, order, offs, rank);
}
bool launch_emb_walk_sorted(const int* offs, const float* dxs, float* grad, int V, int E, int n,
                            cudaStream_t st) {
  const size_t smem = size_t(n) * E * sizeof(float);
  if (V <= 1024 && (n * E) % 4 == 0 && smem <= 200 * 1024 && (E == 2 || E == 4 || E == 8)) {
    const void* k = E == 4 ? reinterpret_cast<const void*>(k_emb_walk_smem<4>)
                   : E == 8 ? reinterpret_cast<const void*>(k_emb_walk_smem<8>)
                            : reinterpret_cast<const void*>(k_emb_walk_smem<2>);
    ensure_smem(k, smem);
    const dim3 b(unsigned(std::max(V, 256)));
    if (E == 4) launch_pdl(k_emb_walk_smem<4>, dim3(1), b, smem, st, offs, dxs, grad, V, n);
    else if (E == 8) launch_pdl(k_emb_walk_smem<8>, dim3(1), b, smem, st, offs, dxs, grad, V, n);
    else launch_pdl(k_emb_walk_smem<2>, dim3(1), b, smem, st, offs, dxs, grad, V, n);
    return true;
  }
  const dim3 g(unsigned((V + 63) / 64)), b(64);
  switch (E) {
    case 4: launch_pdl(k_emb_walk_sorted<4>, g, b, 0, st, offs, dxs, grad, V); return true;
    case 8: launch_pdl(k_emb_walk_sorted<8>, g, b, 0, st, offs, dxs, grad, V); return true;
    case 2: launch_pdl(k_emb_walk_sorted<2>, g, b, 0, st, offs, dxs, grad, V); return true;
    default: return false;
  }
}
void launch_emb_walk(const uint16_t* order, const int* offs, const float* dx, float* grad, int V,
                     int E, cudaStream_t st) {
  launch_pdl(k_emb_walk, dim3(unsigned((V * E + 127) / 128)), dim3(128), 0, st, order, offs, dx, grad,
             V, E);
}
void launch_bigru_concat(const float* tape, float* x1, int R, int T, int H, cudaStream_t st) {
  const int64_t n = int64_t(R) * T * 2 * H;
  launch_pdl(k_bigru_concat, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, tape, x1, R, T, H);
}
void launch_bigru_xf(const float* x1, float* Xf, int R, int T, int In, cudaStream_t st) {
  const int64_t n = 2ll * In * R * T;
  launch_pdl(k_bigru_xf, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, x1, Xf, R, T, In);
}
void launch_tanh_vec(float* x, int64_t n, cudaStream_t st) {
  launch_pdl(k_tanh_vec, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, x, n);
}
void launch_sprm_adam(float* w, float* g, float* m, float* v, int64_t n, AdamScalars* sc, int64_t* pos,
                      int64_t by, unsigned* done, cudaStream_t st) {
  const int64_t per = (n + 255) / 256;
  launch_pdl(k_sprm_adam, dim3(unsigned(per < 64 ? per : 64)), dim3(256), 0, st, w, g, m, v, n, sc, pos, by,
             done);
}
void launch_adam_scalars(AdamScalars* sc, cudaStream_t st) { launch_pdl(k_adam_scalars, dim3(1), dim3(1), 0, st, sc); }
void launch_pos_advance(int64_t* pos, int64_t by, cudaStream_t st) {
  launch_pdl(k_pos_advance, dim3(1), dim3(1), 0, st, pos, by);
}

}  // namespace pmklc_b200
