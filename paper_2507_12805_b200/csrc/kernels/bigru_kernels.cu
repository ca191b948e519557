// Frozen BiGRU predictor (SPuM: 2 layers, SPrM: 1 layer) forward on sm_100a.
// Reference: BiGruModel::forward (core/src/models.cpp:53-73), Gru::forward
// (core/src/layers.cpp:213-260), BiGru::forward/final_state (344-399).
//
// Per GRU step and unit j the reference evaluates (layers.cpp:229-258)
//   ar = b_ir + x.W_ir ; ar += b_hr ; ar += h.W_hr        (ascending indices)
//   az = b_iz + x.W_iz ; az += b_hz ; az += h.W_hz
//   hh = b_hn + h.W_hn ; an = b_in + x.W_in
//   r = sig(ar), z = sig(az), n = tanh(an + r*hh), h' = (1-z)*n + z*h
// The x-terms never depend on h: layer 0's are a per-token table (xi0),
// deeper layers' are one batched exact GEMM over all R*t positions. The
// recurrent part runs one warp per (row, direction), lane j = unit j, with
// its three W_h* columns in registers and h broadcast from shared memory.
#include <cstdint>

#include "detmath.cuh"
#include "kernels.hpp"
#include "launch.cuh"

namespace pmklc_b200 {

namespace {

enum { WIR, WIZ, WIN, WHR, WHZ, WHN, BIR, BIZ, BIN, BHR, BHZ, BHN, NG };
#ifndef PMKLC_REC_WARPS
#define PMKLC_REC_WARPS 4
#endif
constexpr int kRecWarps = PMKLC_REC_WARPS;

__device__ __forceinline__ int64_t poff(const int64_t* offs, int l, int dir, int t) {
  return offs[1 + (l * 2 + dir) * NG + t];
}

// xi: layer >= 1 input projections of this chunk, [2 dirs][3 gates][R*T][Hs]
// out: layer output [R][T][2Hs]; fin (last layer): [R][2Hs]
// Blocks are single-direction; the direction's W_h* (3 x Hs x Hs) sit in
// shared memory, each warp runs kRPW rows so one weight read feeds kRPW
// independent chains (and the register budget leaves room for 4+ blocks/SM).
#ifndef PMKLC_REC_WREG
#define PMKLC_REC_WREG 1
#endif
constexpr int kRPW = 4;
template <int HS>
__global__ void __launch_bounds__(kRecWarps * 32) k_bigru_rec(
    BiGruP p, int l, const uint32_t* __restrict__ ctx, int64_t ctx_cs, const float* __restrict__ xi,
    float* out, float* fin, int64_t work_cs, const TickDesc* __restrict__ td) {
  pdl_wait();
  static_assert(kRPW == 4, "rows are paired (0,1),(2,3)");
#if PMKLC_REC_WREG
  __shared__ __align__(16) float sh[kRecWarps][2][32][kRPW];  // h[q][row] per warp
#else
  __shared__ __align__(16) float sw[3][HS][HS];
  __shared__ __align__(16) float sh[kRecWarps][2][32][kRPW];  // h[q][row] per warp
#endif
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dir = blockIdx.x & 1;
  const int grp = (blockIdx.x >> 1) * kRecWarps + wl;  // row group of this warp
  const int T = p.T, H = HS;
  const int64_t RT = int64_t(p.R) * T;
  const float* W = p.w;
#if !PMKLC_REC_WREG
  for (int i = threadIdx.x; i < 3 * HS * HS; i += blockDim.x) {
    const int gate = i / (HS * HS), rem = i % (HS * HS);
    sw[gate][rem / HS][rem % HS] = W[poff(p.offs, l, dir, WHR + gate) + rem];
  }
  __syncthreads();
#endif
  const int r0 = grp * kRPW;
  if (r0 >= p.R) return;
  const int j = lane;
  const bool act = j < H;
  float bhr = 0.f, bhz = 0.f, bhn = 0.f;
  if (act) {
    bhr = W[poff(p.offs, l, dir, BHR) + j];
    bhz = W[poff(p.offs, l, dir, BHZ) + j];
    bhn = W[poff(p.offs, l, dir, BHN) + j];
  }
  bool rv_ok[kRPW];
#pragma unroll
  for (int u = 0; u < kRPW; ++u) rv_ok[u] = r0 + u < p.R;
  *reinterpret_cast<float4*>(&sh[wl][0][j][0]) = make_float4(0.f, 0.f, 0.f, 0.f);  // h0 = 0
  const float* xr = xi ? xi + c * work_cs + int64_t(dir) * 3 * RT * H : nullptr;
  const float* t0 = p.xi0 + int64_t(dir) * 3 * p.V * H;  // layer-0 tables [3][V][H]
  const int jj = act ? j : 0;
#if PMKLC_REC_WREG
  // this lane's W_h columns (gate, q) in registers for the whole sequence
  float wreg[3][HS];
#pragma unroll
  for (int g = 0; g < 3; ++g)
#pragma unroll
    for (int q = 0; q < HS; ++q) wreg[g][q] = __ldg(W + poff(p.offs, l, dir, WHR + g) + q * HS + jj);
#endif
  // layer 0: the rows' context tokens one per lane (T <= 32) and read by
  // shuffle, and the step's table terms fetched one step ahead, so no step
  // waits on a token load followed by a dependent table load
  const bool lane_tok = l == 0 && T <= 32;
  uint32_t mytok[kRPW];
#pragma unroll
  for (int u = 0; u < kRPW; ++u) {
    const int r = rv_ok[u] ? r0 + u : r0;
    mytok[u] = lane_tok && lane < T ? ctx[c * ctx_cs + int64_t(r) * T + lane] : 0u;
  }
  auto fetch = [&](int step, float (&x)[3][kRPW]) {
    const int tt = dir ? (T - 1 - step) : step;
#pragma unroll
    for (int u = 0; u < kRPW; ++u) {
      const int r = rv_ok[u] ? r0 + u : r0;
      if (l == 0) {
        const int64_t tok = lane_tok ? int64_t(__shfl_sync(0xffffffffu, mytok[u], tt))
                                     : int64_t(ctx[c * ctx_cs + int64_t(r) * T + tt]);
        x[0][u] = t0[tok * H + jj];
        x[1][u] = t0[int64_t(p.V) * H + tok * H + jj];
        x[2][u] = t0[2 * int64_t(p.V) * H + tok * H + jj];
      } else {
        const int64_t pos = (int64_t(r) * T + tt) * H + jj;
        x[0][u] = xr[pos];
        x[1][u] = xr[RT * H + pos];
        x[2][u] = xr[2 * RT * H + pos];
      }
    }
  };
  float xn[3][kRPW];
  fetch(0, xn);
  __syncwarp();
  int cur = 0;
  for (int step = 0; step < T; ++step) {
    const int tt = dir ? (T - 1 - step) : step;  // bwd direction consumes time-reversed input
    float ar[kRPW], az[kRPW], an[kRPW];
#pragma unroll
    for (int u = 0; u < kRPW; ++u) {
      ar[u] = fadd(xn[0][u], bhr);
      az[u] = fadd(xn[1][u], bhz);
      an[u] = xn[2][u];
    }
    if (step + 1 < T) fetch(step + 1, xn);
    // gate pre-activations for rows (0,1) and (2,3) as paired chains, k ascending
    f2_t ar01 = f2_pack(ar[0], ar[1]), ar23 = f2_pack(ar[2], ar[3]);
    f2_t az01 = f2_pack(az[0], az[1]), az23 = f2_pack(az[2], az[3]);
    f2_t hh01 = f2_bcast(bhn), hh23 = f2_bcast(bhn);
#pragma unroll
    for (int q = 0; q < HS; ++q) {
      const float4 hv = *reinterpret_cast<const float4*>(&sh[wl][cur][q][0]);
      const f2_t h01 = f2_pack(hv.x, hv.y), h23 = f2_pack(hv.z, hv.w);
#if PMKLC_REC_WREG
      const f2_t wr = f2_bcast(wreg[0][q]), wz = f2_bcast(wreg[1][q]);
      const f2_t wn = f2_bcast(wreg[2][q]);
#else
      const f2_t wr = f2_bcast(sw[0][q][jj]), wz = f2_bcast(sw[1][q][jj]);
      const f2_t wn = f2_bcast(sw[2][q][jj]);
#endif
      ar01 = f2_mac(ar01, h01, wr);
      ar23 = f2_mac(ar23, h23, wr);
      az01 = f2_mac(az01, h01, wz);
      az23 = f2_mac(az23, h23, wz);
      hh01 = f2_mac(hh01, h01, wn);
      hh23 = f2_mac(hh23, h23, wn);
    }
    // gates of row pairs (0,1), (2,3) through the paired det functions
    const float4 hp = *reinterpret_cast<const float4*>(&sh[wl][cur][jj][0]);
    const f2_t an01 = f2_pack(an[0], an[1]), an23 = f2_pack(an[2], an[3]);
    const f2_t rv01 = det_sigmoid2(ar01), rv23 = det_sigmoid2(ar23);
    const f2_t zv01 = det_sigmoid2(az01), zv23 = det_sigmoid2(az23);
    const f2_t nv01 = det_tanh2(f2_add(an01, f2_mul(rv01, hh01)));
    const f2_t nv23 = det_tanh2(f2_add(an23, f2_mul(rv23, hh23)));
    const f2_t one = f2_bcast(1.0f);
    const f2_t hn01 = f2_add(f2_mul(f2_sub(one, zv01), nv01), f2_mul(zv01, f2_pack(hp.x, hp.y)));
    const f2_t hn23 = f2_add(f2_mul(f2_sub(one, zv23), nv23), f2_mul(zv23, f2_pack(hp.z, hp.w)));
    const float hn[kRPW] = {f2_lo(hn01), f2_hi(hn01), f2_lo(hn23), f2_hi(hn23)};
#pragma unroll
    for (int u = 0; u < kRPW; ++u)
      if (act && rv_ok[u]) out[c * work_cs + (int64_t(r0 + u) * T + tt) * 2 * H + dir * H + j] = hn[u];
    if (act) *reinterpret_cast<float4*>(&sh[wl][cur ^ 1][j][0]) = make_float4(hn[0], hn[1], hn[2], hn[3]);
    __syncwarp();
    cur ^= 1;
  }
  if (fin && act) {
#pragma unroll
    for (int u = 0; u < kRPW; ++u)
      if (rv_ok[u]) fin[c * work_cs + int64_t(r0 + u) * 2 * H + dir * H + j] = sh[wl][cur][j][u];
  }
}

__device__ __forceinline__ void rec_cp_async4(float* smem, const float* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}

// Layer >= 1 with the input projection fused in (Hs == 32, input width 64):
// per step each lane forms xi_g = b_ig + in . W_ig (k ascending, exactly the
// GEMM's chain) for its unit and the warp's 4 rows, then runs the recurrence
// as k_bigru_rec<32>. The step's input rows (the previous layer's output at
// the direction's time index) are prefetched one step ahead by cp.async into a
// per-warp [k][row] buffer, so one broadcast LDS.128 feeds two row pairs.
// No xi buffer round trip through HBM; `out` may be null (last layer: only
// the final state is consumed).
constexpr int kFuseHs = 32, kFuseIn = 64;
#ifndef PMKLC_FUSE_WARPS
#define PMKLC_FUSE_WARPS 8
#endif
constexpr int kFuseWarps = PMKLC_FUSE_WARPS;  // warps (row groups) per fused block
constexpr size_t kFuseSmem =
    sizeof(float) * (size_t(3) * kFuseHs * kFuseHs + size_t(3) * kFuseIn * kFuseHs +
                     size_t(kFuseWarps) * 2 * 32 * kRPW + size_t(kFuseWarps) * 2 * kFuseIn * kRPW);
__global__ void __launch_bounds__(kFuseWarps * 32) k_bigru_rec_fused(
    BiGruP p, int l, const float* __restrict__ in, float* out, float* fin, int64_t work_cs,
    const TickDesc* __restrict__ td) {
  pdl_wait();
  constexpr int HS = kFuseHs, IN = kFuseIn;
  extern __shared__ __align__(16) float fsm[];
  float (*sw)[HS][HS] = reinterpret_cast<float (*)[HS][HS]>(fsm);                    // [3][q][j]
  float (*swi)[IN][HS] = reinterpret_cast<float (*)[IN][HS]>(fsm + 3 * HS * HS);     // [3][k][j]
  float (*sh)[2][32][kRPW] =
      reinterpret_cast<float (*)[2][32][kRPW]>(fsm + 3 * HS * HS + 3 * IN * HS);     // [w][cur][q][u]
  float (*sin)[2][IN][kRPW] = reinterpret_cast<float (*)[2][IN][kRPW]>(
      fsm + 3 * HS * HS + 3 * IN * HS + kFuseWarps * 2 * 32 * kRPW);                 // [w][buf][k][u]
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dir = blockIdx.x & 1;
  const int grp = (blockIdx.x >> 1) * kFuseWarps + wl;
  const int T = p.T;
  const float* W = p.w;
  for (int i = threadIdx.x; i < 3 * HS * HS; i += blockDim.x) {
    const int gate = i / (HS * HS), rem = i % (HS * HS);
    sw[gate][rem / HS][rem % HS] = W[poff(p.offs, l, dir, WHR + gate) + rem];
  }
  for (int i = threadIdx.x; i < 3 * IN * HS; i += blockDim.x) {
    const int gate = i / (IN * HS), rem = i % (IN * HS);
    swi[gate][rem / HS][rem % HS] = W[poff(p.offs, l, dir, WIR + gate) + rem];
  }
  __syncthreads();
  const int r0 = grp * kRPW;
  if (r0 >= p.R) return;
  const int j = lane;
  const float bhr = W[poff(p.offs, l, dir, BHR) + j], bhz = W[poff(p.offs, l, dir, BHZ) + j],
              bhn = W[poff(p.offs, l, dir, BHN) + j];
  const float bir = W[poff(p.offs, l, dir, BIR) + j], biz = W[poff(p.offs, l, dir, BIZ) + j],
              bin = W[poff(p.offs, l, dir, BIN) + j];
  bool rv_ok[kRPW];
  int rr[kRPW];
#pragma unroll
  for (int u = 0; u < kRPW; ++u) {
    rv_ok[u] = r0 + u < p.R;
    rr[u] = rv_ok[u] ? r0 + u : r0;
  }
  const float* inc = in + c * work_cs;
  auto prefetch = [&](int step, int buf) {
    const int tt = dir ? (T - 1 - step) : step;
#pragma unroll
    for (int i = 0; i < 2 * kRPW; ++i) {
      const int u = i >> 1, k = lane + 32 * (i & 1);
      rec_cp_async4(&sin[wl][buf][k][u], inc + (int64_t(rr[u]) * T + tt) * IN + k);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  *reinterpret_cast<float4*>(&sh[wl][0][j][0]) = make_float4(0.f, 0.f, 0.f, 0.f);  // h0 = 0
  prefetch(0, 0);
  int cur = 0;
  for (int step = 0; step < T; ++step) {
    const int tt = dir ? (T - 1 - step) : step;
    const int buf = step & 1;
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncwarp();  // this step's inputs and h landed for every lane
    if (step + 1 < T) prefetch(step + 1, buf ^ 1);
    // input projections (GEMM chain order: bias, then k ascending)
    f2_t xr01 = f2_bcast(bir), xr23 = f2_bcast(bir), xz01 = f2_bcast(biz), xz23 = f2_bcast(biz);
    f2_t xn01 = f2_bcast(bin), xn23 = f2_bcast(bin);
#pragma unroll 8
    for (int k = 0; k < IN; ++k) {
      const float4 iv = *reinterpret_cast<const float4*>(&sin[wl][buf][k][0]);
      const f2_t i01 = f2_pack(iv.x, iv.y), i23 = f2_pack(iv.z, iv.w);
      const f2_t wr = f2_bcast(swi[0][k][j]), wz = f2_bcast(swi[1][k][j]), wn = f2_bcast(swi[2][k][j]);
      xr01 = f2_mac(xr01, i01, wr);
      xr23 = f2_mac(xr23, i23, wr);
      xz01 = f2_mac(xz01, i01, wz);
      xz23 = f2_mac(xz23, i23, wz);
      xn01 = f2_mac(xn01, i01, wn);
      xn23 = f2_mac(xn23, i23, wn);
    }
    f2_t ar01 = f2_add(xr01, f2_bcast(bhr)), ar23 = f2_add(xr23, f2_bcast(bhr));
    f2_t az01 = f2_add(xz01, f2_bcast(bhz)), az23 = f2_add(xz23, f2_bcast(bhz));
    f2_t hh01 = f2_bcast(bhn), hh23 = f2_bcast(bhn);
#pragma unroll 8
    for (int q = 0; q < HS; ++q) {
      const float4 hv = *reinterpret_cast<const float4*>(&sh[wl][cur][q][0]);
      const f2_t h01 = f2_pack(hv.x, hv.y), h23 = f2_pack(hv.z, hv.w);
      const f2_t wr = f2_bcast(sw[0][q][j]), wz = f2_bcast(sw[1][q][j]);
      const f2_t wn = f2_bcast(sw[2][q][j]);
      ar01 = f2_mac(ar01, h01, wr);
      ar23 = f2_mac(ar23, h23, wr);
      az01 = f2_mac(az01, h01, wz);
      az23 = f2_mac(az23, h23, wz);
      hh01 = f2_mac(hh01, h01, wn);
      hh23 = f2_mac(hh23, h23, wn);
    }
    const float4 hp = *reinterpret_cast<const float4*>(&sh[wl][cur][j][0]);
    const f2_t rv01 = det_sigmoid2(ar01), rv23 = det_sigmoid2(ar23);
    const f2_t zv01 = det_sigmoid2(az01), zv23 = det_sigmoid2(az23);
    const f2_t nv01 = det_tanh2(f2_add(xn01, f2_mul(rv01, hh01)));
    const f2_t nv23 = det_tanh2(f2_add(xn23, f2_mul(rv23, hh23)));
    const f2_t one = f2_bcast(1.0f);
    const f2_t hn01 = f2_add(f2_mul(f2_sub(one, zv01), nv01), f2_mul(zv01, f2_pack(hp.x, hp.y)));
    const f2_t hn23 = f2_add(f2_mul(f2_sub(one, zv23), nv23), f2_mul(zv23, f2_pack(hp.z, hp.w)));
    const float hn[kRPW] = {f2_lo(hn01), f2_hi(hn01), f2_lo(hn23), f2_hi(hn23)};
#pragma unroll
    for (int u = 0; u < kRPW; ++u)
      if (out && rv_ok[u]) out[c * work_cs + (int64_t(r0 + u) * T + tt) * 2 * HS + dir * HS + j] = hn[u];
    *reinterpret_cast<float4*>(&sh[wl][cur ^ 1][j][0]) = make_float4(hn[0], hn[1], hn[2], hn[3]);
    cur ^= 1;
  }
  __syncwarp();
  if (fin) {
#pragma unroll
    for (int u = 0; u < kRPW; ++u)
      if (rv_ok[u]) fin[c * work_cs + int64_t(r0 + u) * 2 * HS + dir * HS + j] = sh[wl][cur][j][u];
  }
}

// Generic recurrence (any Hs; lane owns units j, j+32, ...; weights via L1).
__global__ void __launch_bounds__(kRecWarps * 32) k_bigru_rec_generic(
    BiGruP p, int l, const uint32_t* __restrict__ ctx, int64_t ctx_cs, const float* __restrict__ xi,
    float* out, float* fin, int64_t work_cs, const TickDesc* __restrict__ td) {
  pdl_wait();
  extern __shared__ __align__(16) float shd[];  // [kRecWarps][2][Hs]
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = blockIdx.x * kRecWarps + wl;
  if (g >= p.R * 2) return;
  const int r = g >> 1, dir = g & 1, T = p.T, H = p.Hs;
  const int64_t RT = int64_t(p.R) * T;
  const float* W = p.w;
  const float* whr = W + poff(p.offs, l, dir, WHR);
  const float* whz = W + poff(p.offs, l, dir, WHZ);
  const float* whn = W + poff(p.offs, l, dir, WHN);
  const float* bhr = W + poff(p.offs, l, dir, BHR);
  const float* bhz = W + poff(p.offs, l, dir, BHZ);
  const float* bhn = W + poff(p.offs, l, dir, BHN);
  const uint32_t* cr = ctx + c * ctx_cs + int64_t(r) * T;
  const float* xr = xi ? xi + c * work_cs + int64_t(dir) * 3 * RT * H : nullptr;
  const float* t0 = p.xi0 + int64_t(dir) * 3 * p.V * H;
  float* outr = out + c * work_cs + int64_t(r) * T * 2 * H;
  float* buf0 = shd + (wl * 2 + 0) * H;
  float* buf1 = shd + (wl * 2 + 1) * H;
  for (int j = lane; j < H; j += 32) buf0[j] = 0.0f;
  __syncwarp();
  int cur = 0;
  for (int step = 0; step < T; ++step) {
    const int tt = dir ? (T - 1 - step) : step;
    const float* h = cur ? buf1 : buf0;
    float* hnx = cur ? buf0 : buf1;
    for (int j = lane; j < H; j += 32) {
      float ar, az, an;
      if (l == 0) {
        const int64_t tok = cr[tt];
        ar = t0[tok * H + j];
        az = t0[int64_t(p.V) * H + tok * H + j];
        an = t0[2 * int64_t(p.V) * H + tok * H + j];
      } else {
        const int64_t pos = (int64_t(r) * T + tt) * H + j;
        ar = xr[pos];
        az = xr[RT * H + pos];
        an = xr[2 * RT * H + pos];
      }
      ar = fadd(ar, bhr[j]);
      for (int q = 0; q < H; ++q) ar = mac(ar, h[q], whr[int64_t(q) * H + j]);
      az = fadd(az, bhz[j]);
      for (int q = 0; q < H; ++q) az = mac(az, h[q], whz[int64_t(q) * H + j]);
      float hh = bhn[j];
      for (int q = 0; q < H; ++q) hh = mac(hh, h[q], whn[int64_t(q) * H + j]);
      const float rv = det_sigmoid(ar), zv = det_sigmoid(az);
      const float nv = det_tanh(fadd(an, fmul(rv, hh)));
      const float hv = fadd(fmul(fsub(1.0f, zv), nv), fmul(zv, h[j]));
      hnx[j] = hv;
      outr[int64_t(tt) * 2 * H + dir * H + j] = hv;
    }
    __syncwarp();
    cur ^= 1;
  }
  const float* hl = cur ? buf1 : buf0;
  if (fin)
    for (int j = lane; j < H; j += 32) fin[c * work_cs + int64_t(r) * 2 * H + dir * H + j] = hl[j];
}

__global__ void k_tanh_inplace(float* x, int64_t n, int64_t cs, const TickDesc* __restrict__ td) {
  pdl_wait();
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[c * cs + i] = det_tanh(x[c * cs + i]);
}

}  // namespace

// work layout per chunk: xi [2][3][R*T][Hs] | out0 [R][T][2Hs] | out1 [R][T][2Hs] |
//                        fin [R][2Hs] | bott [R][B]
size_t bigru_work_floats(const BiGruP& p) {
  const size_t RT = size_t(p.R) * p.T;
  return 6 * RT * p.Hs + 2 * RT * 2 * p.Hs + size_t(p.R) * 2 * p.Hs + size_t(p.R) * p.B;
}

namespace {
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_hot_begin(HotTimer* h) {
  pdl_wait(); h->t0 = global_ns(); }
__global__ void k_hot_end(HotTimer* h, const TickDesc* __restrict__ td) {
  pdl_wait();
  h->ns += global_ns() - h->t0;
  h->units += unsigned(td->n_act);
  h->launches += 1;
}
}  // namespace
void launch_hot_begin(HotTimer* h, cudaStream_t st) { launch_pdl(k_hot_begin, dim3(1), dim3(1), 0, st, h); }
void launch_hot_end(HotTimer* h, const TickDesc* td, cudaStream_t st) {
  launch_pdl(k_hot_end, dim3(1), dim3(1), 0, st, h, td);
}

int launch_bigru_predict(const BiGruP& p, const uint32_t* ctx, int64_t ctx_cs, float* work,
                          int64_t work_cs, float* logits, int64_t lg_cs, const TickDesc* td,
                          int max_active, cudaStream_t st, HotTimer* hot) {
  if (max_active <= 0) return 0;
  int launches = 0;
  const int64_t RT = int64_t(p.R) * p.T, H = p.Hs;
  float* xi = work;
  float* outs[2] = {xi + 6 * RT * H, xi + 6 * RT * H + RT * 2 * H};
  float* fin = outs[1] + RT * 2 * H;
  float* bott = fin + int64_t(p.R) * 2 * H;
  const dim3 rgrid(unsigned((p.R * 2 + kRecWarps - 1) / kRecWarps), max_active);
  const int ngroups = (p.R + kRPW - 1) / kRPW;
  const dim3 rgrid2(unsigned(2 * ((ngroups + kRecWarps - 1) / kRecWarps)), max_active);
  const bool fuse = p.Hs == kFuseHs;
  if (fuse) ensure_smem(reinterpret_cast<const void*>(k_bigru_rec_fused), kFuseSmem);
  for (int l = 0; l < p.layers; ++l) {
    const bool last = l == p.layers - 1;
    float* f = last ? fin : nullptr;
    if (l > 0 && fuse) {
      // projection fused into the recurrence; the last layer's per-step
      // outputs are never read (the head consumes the final state only)
      if (hot) {
        launch_hot_begin(hot, st);
        ++launches;
      }
      const dim3 fgrid(unsigned(2 * ((ngroups + kFuseWarps - 1) / kFuseWarps)), max_active);
      launch_pdl(k_bigru_rec_fused, fgrid, dim3(kFuseWarps * 32), kFuseSmem, st, 
          p, l, outs[(l - 1) & 1], last ? nullptr : outs[l & 1], f, work_cs, td);
      ++launches;
      if (hot) {
        launch_hot_end(hot, td, st);
        ++launches;
      }
      continue;
    }
    float* out = outs[l & 1];
    if (l > 0) {
      // x-projections of layer l for every position: 3 gates per direction,
      // C[gate][RT][H] = b_i{gate} + in . W_i{gate}
      const float* in = outs[(l - 1) & 1];
      const int in_w = int(2 * H);
      for (int dir = 0; dir < 2; ++dir) {
        GemmP gp{};
        gp.A = in;
        gp.a_cs = work_cs;
        gp.lda = in_w;
        gp.B = p.w + p.hoffs[1 + (l * 2 + dir) * NG + WIR];
        gp.ldb = H;
        gp.C = xi + int64_t(dir) * 3 * RT * H;
        gp.c_cs = work_cs;
        gp.ldc = H;
        gp.bias = p.w + p.hoffs[1 + (l * 2 + dir) * NG + BIR];
        gp.M = int(RT);
        gp.N = int(H);
        gp.K = in_w;
        gp.init = 1;
        gp.nprob = 3;
        gp.b_ps = int64_t(in_w) * H;  // w_ir, w_iz, w_in consecutive
        gp.c_ps = RT * H;
        gp.bias_ps = H;               // b_ir, b_iz, b_in consecutive
        launch_gemm(gp, false, false, td, max_active, st);
        ++launches;
      }
    }
    const float* xl = l == 0 ? nullptr : xi;
    if (p.Hs == 32)
      launch_pdl(k_bigru_rec<32>, dim3(rgrid2), dim3(kRecWarps * 32), 0, st, p, l, ctx, ctx_cs, xl, out, f, work_cs, td);
    else if (p.Hs == 16)
      launch_pdl(k_bigru_rec<16>, dim3(rgrid2), dim3(kRecWarps * 32), 0, st, p, l, ctx, ctx_cs, xl, out, f, work_cs, td);
    else if (p.Hs == 8)
      launch_pdl(k_bigru_rec<8>, dim3(rgrid2), dim3(kRecWarps * 32), 0, st, p, l, ctx, ctx_cs, xl, out, f, work_cs, td);
    else
      launch_pdl(k_bigru_rec_generic, dim3(rgrid), dim3(kRecWarps * 32), kRecWarps * 2 * p.Hs * sizeof(float), st, 
          p, l, ctx, ctx_cs, xl, out, f, work_cs, td);
    ++launches;
  }
  // bott = tanh(bott.b + fin . bott.w);  logits = out.b + bott . out.w
  const int b0 = 1 + p.layers * 2 * NG;
  GemmP g1{};
  g1.A = fin;
  g1.a_cs = work_cs;
  g1.lda = 2 * H;
  g1.B = p.w + p.hoffs[b0];
  g1.ldb = p.B;
  g1.C = bott;
  g1.c_cs = work_cs;
  g1.ldc = p.B;
  g1.bias = p.w + p.hoffs[b0 + 1];
  g1.M = p.R;
  g1.N = p.B;
  g1.K = int(2 * H);
  g1.init = 1;
  launch_gemm(g1, false, false, td, max_active, st);
  const int64_t nb = int64_t(p.R) * p.B;
  launch_pdl(k_tanh_inplace, dim3(dim3(unsigned((nb + 255) / 256), max_active)), dim3(256), 0, st, bott, nb, work_cs, td);
  GemmP g2{};
  g2.A = bott;
  g2.a_cs = work_cs;
  g2.lda = p.B;
  g2.B = p.w + p.hoffs[b0 + 2];
  g2.ldb = p.V;
  g2.C = logits;
  g2.c_cs = lg_cs;
  g2.ldc = p.V;
  g2.bias = p.w + p.hoffs[b0 + 3];
  g2.M = p.R;
  g2.N = p.V;
  g2.K = p.B;
  g2.init = 1;
  launch_gemm(g2, false, false, td, max_active, st);
  return launches + 3;  // + bottleneck GEMM, tanh, output GEMM
}

}  // namespace pmklc_b200
