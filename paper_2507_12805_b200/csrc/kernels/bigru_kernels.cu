// Frozen BiGRU predictor (SPuM: 2 layers, SPrM: 1 layer) forward on sm_100a.
// Reference: BiGruModel::forward (core/src/models.cpp:53-73), Gru::forward
// (core/src/layers.cpp:213-260), BiGru::forward/final_state (344-399).
//
// The recurrence is serial in time, so parallelism is rows x directions: one
// warp runs one (row, direction) sequence, lane j owning hidden units j,
// j+32, ...; the previous hidden state and the current input are staged in
// shared memory so every lane reads them as broadcasts. Each gate pre-activation
// is accumulated exactly as the reference does: bias, then ascending input
// terms, then (r,z gates) the recurrent bias and ascending hidden terms.
#include <cstdint>

#include "detmath.cuh"
#include "kernels.hpp"

namespace pmklc_b200 {

namespace {

enum { WIR, WIZ, WIN, WHR, WHZ, WHN, BIR, BIZ, BIN, BHR, BHZ, BHN, NG };
constexpr int kWarps = 4;
constexpr int kMaxH = 128;   // sp_hidden at scale 1
constexpr int kMaxIn = 256;  // 2*sp_hidden at scale 1

__device__ __forceinline__ int64_t poff(const int64_t* offs, int l, int dir, int t) {
  return offs[1 + (l * 2 + dir) * NG + t];
}

// in_buf: layer input [R,T,in] (nullptr for layer 0: gathered from the embedding)
__global__ void __launch_bounds__(kWarps * 32) k_bigru_layer(BiGruP p, int l, const uint32_t* ctx,
                                                             int64_t ctx_cs, const float* in_buf,
                                                             float* out_buf, float* fin,
                                                             int64_t work_cs,
                                                             const TickDesc* __restrict__ td) {
  __shared__ float sx[kWarps][kMaxIn];
  __shared__ float sh[kWarps][kMaxH];
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wg = blockIdx.x * kWarps + wl;
  if (wg >= p.R * 2) return;
  const int r = wg >> 1, dir = wg & 1;
  const int H = p.Hs, T = p.T, in = (l == 0) ? p.Es : 2 * p.Hs;
  const float* W = p.w;
  const float *wir = W + poff(p.offs, l, dir, WIR), *wiz = W + poff(p.offs, l, dir, WIZ),
              *win = W + poff(p.offs, l, dir, WIN), *whr = W + poff(p.offs, l, dir, WHR),
              *whz = W + poff(p.offs, l, dir, WHZ), *whn = W + poff(p.offs, l, dir, WHN);
  const float *bir = W + poff(p.offs, l, dir, BIR), *biz = W + poff(p.offs, l, dir, BIZ),
              *bin = W + poff(p.offs, l, dir, BIN), *bhr = W + poff(p.offs, l, dir, BHR),
              *bhz = W + poff(p.offs, l, dir, BHZ), *bhn = W + poff(p.offs, l, dir, BHN);
  const float* emb = W + p.offs[0];
  const uint32_t* cr = ctx + c * ctx_cs + int64_t(r) * T;
  const float* inr = in_buf ? in_buf + c * work_cs + int64_t(r) * T * in : nullptr;
  float* outr = out_buf + c * work_cs + int64_t(r) * T * 2 * H;
  for (int j = lane; j < H; j += 32) sh[wl][j] = 0.0f;  // h0 = 0
  __syncwarp();
  for (int step = 0; step < T; ++step) {
    const int tt = dir ? (T - 1 - step) : step;  // bwd direction reads time-reversed input
    for (int q = lane; q < in; q += 32)
      sx[wl][q] = inr ? inr[int64_t(tt) * in + q] : emb[int64_t(cr[tt]) * p.Es + q];
    __syncwarp();
    float hnew[kMaxH / 32];
    int u = 0;
    for (int j = lane; j < H; j += 32, ++u) {
      float ar = bir[j], az = biz[j], an = bin[j], hh = bhn[j];
      for (int q = 0; q < in; ++q) {
        const float xv = sx[wl][q];
        ar = mac(ar, xv, wir[int64_t(q) * H + j]);
      }
      ar = fadd(ar, bhr[j]);
      for (int q = 0; q < H; ++q) ar = mac(ar, sh[wl][q], whr[int64_t(q) * H + j]);
      for (int q = 0; q < in; ++q) az = mac(az, sx[wl][q], wiz[int64_t(q) * H + j]);
      az = fadd(az, bhz[j]);
      for (int q = 0; q < H; ++q) az = mac(az, sh[wl][q], whz[int64_t(q) * H + j]);
      for (int q = 0; q < H; ++q) hh = mac(hh, sh[wl][q], whn[int64_t(q) * H + j]);
      for (int q = 0; q < in; ++q) an = mac(an, sx[wl][q], win[int64_t(q) * H + j]);
      const float rv = det_sigmoid(ar), zv = det_sigmoid(az);
      const float nv = det_tanh(fadd(an, fmul(rv, hh)));
      hnew[u] = fadd(fmul(fsub(1.0f, zv), nv), fmul(zv, sh[wl][j]));
    }
    __syncwarp();
    u = 0;
    for (int j = lane; j < H; j += 32, ++u) {
      sh[wl][j] = hnew[u];
      outr[int64_t(tt) * 2 * H + dir * H + j] = hnew[u];
    }
    __syncwarp();
  }
  if (fin)
    for (int j = lane; j < H; j += 32) fin[c * work_cs + int64_t(r) * 2 * H + dir * H + j] = sh[wl][j];
}

// bott = tanh(bott.b + fin . bott.w); one thread per (row, unit)
__global__ void k_bigru_bott(BiGruP p, const float* fin, float* bact, int64_t work_cs,
                             const TickDesc* __restrict__ td) {
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= p.R * p.B) return;
  const int r = idx / p.B, j = idx % p.B, K = 2 * p.Hs;
  const int b0 = 1 + p.layers * 2 * NG;
  const float* w = p.w + p.offs[b0];
  float acc = p.w[p.offs[b0 + 1] + j];
  const float* f = fin + c * work_cs + int64_t(r) * K;
  for (int q = 0; q < K; ++q) acc = mac(acc, f[q], w[int64_t(q) * p.B + j]);
  bact[c * work_cs + idx] = det_tanh(acc);
}

// logits = out.b + bott . out.w
__global__ void k_bigru_out(BiGruP p, const float* bact, int64_t work_cs, float* logits,
                            int64_t lg_cs, const TickDesc* __restrict__ td) {
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= p.R * p.V) return;
  const int r = idx / p.V, v = idx % p.V;
  const int b0 = 1 + p.layers * 2 * NG;
  const float* w = p.w + p.offs[b0 + 2];
  float acc = p.w[p.offs[b0 + 3] + v];
  const float* b = bact + c * work_cs + int64_t(r) * p.B;
  for (int q = 0; q < p.B; ++q) acc = mac(acc, b[q], w[int64_t(q) * p.V + v]);
  logits[c * lg_cs + idx] = acc;
}

}  // namespace

size_t bigru_work_floats(const BiGruP& p) {
  // two layer-output buffers [R,T,2H] + fin [R,2H] + bact [R,B]
  return size_t(p.R) * (2 * size_t(p.T) * 2 * p.Hs + 2 * p.Hs + p.B);
}

void launch_bigru_predict(const BiGruP& p, const uint32_t* ctx, int64_t ctx_cs, float* work,
                          int64_t work_cs, float* logits, int64_t lg_cs, const TickDesc* td,
                          int max_active, cudaStream_t st) {
  if (max_active <= 0) return;
  const int64_t layer_sz = int64_t(p.R) * p.T * 2 * p.Hs;
  float* buf[2] = {work, work + layer_sz};
  float* fin = work + 2 * layer_sz;
  float* bact = fin + int64_t(p.R) * 2 * p.Hs;
  dim3 grid(unsigned((p.R * 2 + kWarps - 1) / kWarps), max_active);
  for (int l = 0; l < p.layers; ++l) {
    const float* in = l == 0 ? nullptr : buf[(l - 1) & 1];
    k_bigru_layer<<<grid, kWarps * 32, 0, st>>>(p, l, ctx, ctx_cs, in, buf[l & 1],
                                                l == p.layers - 1 ? fin : nullptr, work_cs, td);
  }
  dim3 g2(unsigned((p.R * p.B + 255) / 256), max_active);
  k_bigru_bott<<<g2, 256, 0, st>>>(p, fin, bact, work_cs, td);
  dim3 g3(unsigned((p.R * p.V + 255) / 256), max_active);
  k_bigru_out<<<g3, 256, 0, st>>>(p, bact, work_cs, logits, lg_cs, td);
}

}  // namespace pmklc_b200
