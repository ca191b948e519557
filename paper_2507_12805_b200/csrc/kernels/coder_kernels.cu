// Mixer + quantizer + range coder + backward-controller scalars on sm_100a.
//
//  * k_mix_quantize: one warp per coded row. Eq. 1 mix (mixer.cpp:14-25),
//    det_softmax with the reference's sequential sum, then the largest-remainder
//    quantizer (coder.cpp:28-88) in closed form: the reference's stable sorts
//    become per-element ranks under the same total order (remainder, index), and
//    its surplus sweep loop becomes "P full passes + a partial pass", both exact.
//  * range coder (coder.cpp:101-166): 64-bit state, one thread per chunk; the
//    decoder replaces the 64-bit integer division with a double estimate plus an
//    exact integer correction.
//  * k_alpha_step: the single sequential d(alpha) accumulator (mixer.cpp:64-84)
//    and alpha's Adam update, kept off the main stream's critical path.
#include <cstdint>

#include "detmath.cuh"
#include "kernels.hpp"
#include "launch.cuh"

namespace pmklc_b200 {

namespace {

constexpr uint32_t kTotal = 65536u;
constexpr uint64_t kRenorm = 1ull << 56;

__device__ __forceinline__ double rem_of(float p, uint32_t& f) {
  const double v = double(p) * double(kTotal);
  const double fl = floor(v);
  f = uint32_t(fl > 1.0 ? fl : 1.0);
  return v - double(f);
}

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t x) {
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__global__ void k_mix_quantize(MixP p, const TickDesc* __restrict__ td) {
  pdl_wait();
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y];
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.sc) {  // Adam::step scalar prologue (adam.cpp:23-27)
    AdamScalars s = p.sc[c];
    s.step += 1;
    s.b1p = fmul(s.b1p, 0.9f);
    s.b2p = fmul(s.b2p, 0.999f);
    s.bc1 = fsub(1.0f, s.b1p);
    s.bc2 = fsub(1.0f, s.b2p);
    p.sc[c] = s;
  }
  if (row >= p.R) return;
  const int V = p.V;
  // V <= 64: the serial sums read a per-warp shared copy
  __shared__ __align__(16) float sbuf[8][64];
  const bool small = V <= 64 && blockDim.x <= 256;
  float* sb = sbuf[(threadIdx.x >> 5) & 7];
  const int64_t lo = c * p.cs_l + int64_t(row) * V;
  const float* lu = (p.flags & 1) ? p.lu + lo : nullptr;
  const float* lr = (p.flags & 2) ? p.lr + lo : nullptr;
  const float* lm = p.lm + lo;
  float* pr = p.probs + c * p.cs_p + int64_t(row) * V;
  uint32_t* fq = p.freq + c * p.cs_p + int64_t(row) * V;
  uint32_t* cm = p.cum + c * p.cs_c + int64_t(row) * (V + 1);

  float inv = 1.0f;
  if (!p.probs_given) {
    const float alpha = det_sigmoid(p.params[c * p.p_cs + p.off_alpha]);
    const float s0 = (p.flags & 1) ? 1.0f : 0.0f, s1 = (p.flags & 2) ? 1.0f : 0.0f;
    const float s2 = (p.flags & 4) ? 1.0f : 0.0f;
    const float wdyn = fmul(fsub(1.0f, alpha), s2);
    // z = alpha*stat + ((1-alpha)*s2)*lm
    float mx = -__int_as_float(0x7f800000);
    for (int i = lane; i < V; i += 32) {
      const float stat = fadd(fmul(s0, lu ? lu[i] : 0.0f), fmul(s1, lr ? lr[i] : 0.0f));
      const float z = fadd(fmul(alpha, stat), fmul(wdyn, lm[i]));
      pr[i] = z;
      mx = fmaxf(mx, z);
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.0f;
    for (int i0 = 0; i0 < V; i0 += 32) {
      const int i = i0 + lane;
      float e = 0.0f;
      if (i < V) {
        e = det_exp(fsub(pr[i], mx));
        pr[i] = e;
        if (small) sb[i] = e;
      }
      if (!small) {
        const int cnt = min(32, V - i0);
        for (int l = 0; l < cnt; ++l) sum = fadd(sum, __shfl_sync(0xffffffffu, e, l));
      }
    }
    if (small) {  // the sequential sum over the warp's shared copy (broadcast LDS.128)
      __syncwarp();
      int i = 0;
      for (; i + 4 <= V; i += 4) {
        const float4 v = *reinterpret_cast<const float4*>(sb + i);
        sum = fadd(fadd(fadd(fadd(sum, v.x), v.y), v.z), v.w);
      }
      for (; i < V; ++i) sum = fadd(sum, sb[i]);
      __syncwarp();
    }
    inv = fdiv(1.0f, sum);
  }
  // probabilities, positivity, double sum in reference order (coder.cpp:31-38)
  double dsum = 0.0;
  bool bad = false;
  uint32_t assigned = 0;
  for (int i0 = 0; i0 < V; i0 += 32) {
    const int i = i0 + lane;
    float pv = 0.0f;
    if (i < V) {
      pv = p.probs_given ? pr[i] : fmul(pr[i], inv);
      pr[i] = pv;
      if (small) sb[i] = pv;
      if (!(pv > 0.0f)) bad = true;
      uint32_t f;
      rem_of(pv, f);
      fq[i] = f;
      assigned += f;
    }
    if (!small) {
      const int cnt = min(32, V - i0);
      for (int l = 0; l < cnt; ++l) dsum = dsum + double(__shfl_sync(0xffffffffu, pv, l));
    }
  }
  if (small) {
    __syncwarp();
    int i = 0;
    for (; i + 4 <= V; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(sb + i);
      dsum = dsum + double(v.x);
      dsum = dsum + double(v.y);
      dsum = dsum + double(v.z);
      dsum = dsum + double(v.w);
    }
    for (; i < V; ++i) dsum = dsum + double(sb[i]);
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad || fabs(dsum - 1.0) > 1e-5) {
    if (lane == 0) atomicExch(p.err, 1);  // InvalidDistribution
    return;
  }
  assigned = warp_sum_u32(assigned);
  const int64_t deficit = int64_t(kTotal) - int64_t(assigned);
  __syncwarp();
  if (deficit > 0 && V <= 64) {
    // stable_sort by (rem desc, idx asc), then +1 cyclically (coder.cpp:57-66).
    // V <= 64: each lane holds the remainders of i = lane, lane + 32; the rank
    // of element i = #{j : r_j > r_i or (r_j == r_i and j < i)} is counted
    // with two ballots per i (r_i broadcast by shuffle).
    // The order is a total order on (remainder desc, index asc), so the ranks
    // are the positions after sorting the 64 (key, index) pairs: a bitonic
    // network over the warp (lane holds elements lane and lane + 32; key =
    // the remainder's double bits mapped to an order-preserving unsigned,
    // inverted for descending; absent elements sort last), then the first
    // `part` sorted entries get the +1.
    const uint32_t full = uint32_t(deficit / V), part = uint32_t(deficit % V);
    const bool h0 = lane < V, h1 = lane + 32 < V;
    uint32_t f0 = 0, f1 = 0;
    const double r0 = h0 ? rem_of(pr[lane], f0) : 0.0;
    const double r1 = h1 ? rem_of(pr[lane + 32], f1) : 0.0;
    auto key_of = [](double r, bool have) -> uint64_t {
      if (!have) return ~0ull;
      const uint64_t b = uint64_t(__double_as_longlong(r));
      const uint64_t ord = (b >> 63) ? ~b : (b | (1ull << 63));  // ascending in r
      return ~ord;                                                // descending in r
    };
    uint64_t ka = key_of(r0, h0), kb = key_of(r1, h1);
    uint32_t ia = uint32_t(lane), ib = uint32_t(lane + 32);
    auto less = [](uint64_t k1, uint32_t i1, uint64_t k2, uint32_t i2) {
      return k1 < k2 || (k1 == k2 && i1 < i2);
    };
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        if (j == 32) {  // partners lane and lane + 32 (k == 64: ascending)
          if (less(kb, ib, ka, ia)) {
            const uint64_t tk = ka;
            const uint32_t ti = ia;
            ka = kb; ia = ib; kb = tk; ib = ti;
          }
        } else {
          const uint64_t pka = __shfl_xor_sync(0xffffffffu, ka, j);
          const uint32_t pia = __shfl_xor_sync(0xffffffffu, ia, j);
          const uint64_t pkb = __shfl_xor_sync(0xffffffffu, kb, j);
          const uint32_t pib = __shfl_xor_sync(0xffffffffu, ib, j);
          const bool lower = (lane & j) == 0;
          // element e: ascending block iff (e & k) == 0; the lower index of a
          // pair keeps the min in an ascending block, the max otherwise
          const bool upa = (lane & k) == 0, upb = ((lane + 32) & k) == 0;
          const bool mina = lower == upa, minb = lower == upb;
          const bool pa_less = less(pka, pia, ka, ia), pb_less = less(pkb, pib, kb, ib);
          if (mina == pa_less) { ka = pka; ia = pia; }
          if (minb == pb_less) { kb = pkb; ib = pib; }
        }
      }
    }
    if (h0) fq[lane] = f0 + full;
    if (h1) fq[lane + 32] = f1 + full;
    __syncwarp();
    if (uint32_t(lane) < part) fq[ia] += 1u;       // sorted position lane
    if (uint32_t(lane + 32) < part) fq[ib] += 1u;  // sorted position lane + 32
  } else if (deficit > 0) {
    // stable_sort by (rem desc, idx asc), then +1 cyclically (coder.cpp:57-66)
    const uint32_t full = uint32_t(deficit / V), part = uint32_t(deficit % V);
    for (int i = lane; i < V; i += 32) {
      uint32_t fi;
      const double ri = rem_of(pr[i], fi);
      uint32_t rank = 0;
      for (int j = 0; j < V; ++j) {
        uint32_t fj;
        const double rj = rem_of(pr[j], fj);
        rank += (rj > ri || (rj == ri && j < i)) ? 1u : 0u;
      }
      fq[i] = fi + full + (rank < part ? 1u : 0u);
    }
  } else if (deficit < 0) {
    // stable_sort by (rem asc, idx asc), sweep -1 over entries with f > 1 until
    // settled (coder.cpp:67-83) == P complete passes + a partial pass.
    const int64_t S = -deficit;
    // the cum row doubles as scratch for the pre-adjustment frequencies
    for (int i = lane; i < V; i += 32) cm[i] = fq[i];
    __syncwarp();
    int64_t lo_p = 0, hi_p = kTotal;  // largest P with removed(P) <= S
    while (lo_p < hi_p) {
      const int64_t mid = (lo_p + hi_p + 1) / 2;
      uint32_t rm = 0;
      for (int i = lane; i < V; i += 32) rm += uint32_t(imin64(int64_t(cm[i]) - 1, mid));
      rm = warp_sum_u32(rm);
      if (int64_t(rm) <= S) lo_p = mid;
      else hi_p = mid - 1;
    }
    const int64_t P = lo_p;
    uint32_t rmP = 0, elig = 0;
    for (int i = lane; i < V; i += 32) {
      const int64_t fi = cm[i];
      rmP += uint32_t(imin64(fi - 1, P));
      elig += (fi - 1 > P) ? 1u : 0u;
    }
    rmP = warp_sum_u32(rmP);
    elig = warp_sum_u32(elig);
    const int64_t rpart = S - int64_t(rmP);
    if (rpart > 0 && int64_t(elig) < rpart) {
      if (lane == 0) atomicExch(p.err, 1);  // cannot settle surplus
      return;
    }
    for (int i = lane; i < V; i += 32) {
      uint32_t fi0;
      const double ri = rem_of(pr[i], fi0);
      const int64_t fi = cm[i];
      int64_t dec = imin64(fi - 1, P);
      if (rpart > 0 && fi - 1 > P) {
        uint32_t rank = 0;
        for (int j = 0; j < V; ++j) {
          if (int64_t(cm[j]) - 1 <= P) continue;
          uint32_t fj0;
          const double rj = rem_of(pr[j], fj0);
          rank += (rj < ri || (rj == ri && j < i)) ? 1u : 0u;
        }
        if (int64_t(rank) < rpart) dec += 1;
      }
      fq[i] = uint32_t(fi - dec);
    }
  }
  __syncwarp();
  // cum = exclusive prefix of freqs
  uint32_t carry = 0;
  for (int i0 = 0; i0 < V; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t f = i < V ? fq[i] : 0u;
    uint32_t inc = f;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (i < V) cm[i] = carry + inc - f;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) cm[V] = carry;
}

__global__ void k_bc_dlm(BcP p, const TickDesc* __restrict__ td) {
  pdl_wait();
  if (blockIdx.y >= unsigned(td->n_act)) return;
  const int c = td->act[blockIdx.y], ch = td->chunk[blockIdx.y];
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int R = p.R, V = p.V;
  if (idx >= int64_t(R) * V) return;
  const int r = int(idx / V), i = int(idx % V);
  const uint64_t jstep = uint64_t(p.t) + uint64_t(p.td->tick - p.geo.offset[ch]);
  const uint32_t tgt = p.tokens[p.geo.start[ch] + uint64_t(r) * p.geo.L[ch] + jstep];
  const float a = det_sigmoid(p.w[c * p.p_cs + p.off_alpha]);
  const int64_t o = c * p.cs_p + idx;
  const float pv = p.probs[o];
  float g = pv;
  if (uint32_t(i) == tgt) {
    g = fsub(g, 1.0f);
    p.lterm[c * p.cs_l + r] = -det_log(pv < 1e-38f ? 1e-38f : pv);  // std::max(p, 1e-38f)
  }
  const float s0 = (p.flags & 1) ? 1.0f : 0.0f, s1 = (p.flags & 2) ? 1.0f : 0.0f;
  const float stat = fadd(fmul(s0, (p.flags & 1) ? p.lu[o] : 0.0f),
                          fmul(s1, (p.flags & 2) ? p.lr[o] : 0.0f));
  p.aterm[o] = fmul(g, fsub(stat, p.lm[o]));
  p.dlm[o] = fmul(g, fsub(1.0f, a));
}

// Block per chunk. Warp 0 lane 0 runs the d(alpha) chain over shared memory
// while the other warps stage the next batch of terms (double buffer); warp
// 1 lane 0 runs the (short) loss chain.
constexpr int kAlphaBatch = 4096;
__global__ void __launch_bounds__(256) k_alpha_step(BcP p, const TickDesc* __restrict__ td) {
  pdl_wait();
  __shared__ __align__(16) float buf[2][kAlphaBatch];
  if (blockIdx.x >= unsigned(p.td->n_act)) return;
  const int c = p.td->act[blockIdx.x], ch = p.td->chunk[blockIdx.x];
  const int64_t n = int64_t(p.R) * p.V;
  const float* terms = p.aterm + c * p.cs_p;
  const int nb = int((n + kAlphaBatch - 1) / kAlphaBatch);
  const int tid = threadIdx.x;
  float dalpha = 0.0f;
  for (int i = tid; i < kAlphaBatch && i < n; i += 256) buf[0][i] = terms[i];
  __syncthreads();
  for (int b = 0; b < nb; ++b) {
    if (b + 1 < nb && tid >= 32) {
      const int64_t base = int64_t(b + 1) * kAlphaBatch;
      for (int64_t i = tid - 32; i < kAlphaBatch && base + i < n; i += 224) buf[(b + 1) & 1][i] = terms[base + i];
    }
    if (tid == 0) {
      const int cnt = int(min(int64_t(kAlphaBatch), n - int64_t(b) * kAlphaBatch));
      const float* q = buf[b & 1];
      int i = 0;
      for (; i + 4 <= cnt; i += 4) {
        const float4 v = *reinterpret_cast<const float4*>(q + i);
        dalpha = fadd(dalpha, v.x);
        dalpha = fadd(dalpha, v.y);
        dalpha = fadd(dalpha, v.z);
        dalpha = fadd(dalpha, v.w);
      }
      for (; i < cnt; ++i) dalpha = fadd(dalpha, q[i]);
    }
    __syncthreads();
  }
  const uint64_t mstep = uint64_t(p.td->tick - p.geo.offset[ch]);
  if (tid == 32 && p.warm_loss && mstep < p.warm_steps[ch]) {
    const float* lt = p.lterm + c * p.cs_l;
    float loss = 0.0f;
    for (int r = 0; r < p.R; ++r) loss = fadd(loss, lt[r]);
    p.warm_loss[ch] += double(loss);
  }
  if (tid == 0) {
    const int64_t aoff = c * p.p_cs + p.off_alpha;
    const float a = det_sigmoid(p.w[aoff]);
    const float grad = fadd(0.0f, fmul(fmul(dalpha, a), fsub(1.0f, a)));
    const float b1 = 0.9f, b2 = 0.999f;
    const float mi = fadd(fmul(b1, p.m[aoff]), fmul(fsub(1.0f, b1), grad));
    const float vi = fadd(fmul(b2, p.v[aoff]), fmul(fmul(fsub(1.0f, b2), grad), grad));
    const float mhat = fdiv(mi, p.sc[c].bc1), vhat = fdiv(vi, p.sc[c].bc2);
    p.w[aoff] = fsub(p.w[aoff], fdiv(fmul(5e-4f, mhat), fadd(__fsqrt_rn(vhat), 1e-8f)));
    p.m[aoff] = mi;
    p.v[aoff] = vi;
  }
}

// ------------------------------------------------------------------ range coder
__device__ __forceinline__ void enc_sym(uint64_t& low, uint64_t& range, uint8_t* out,
                                        uint64_t& pos, uint32_t cum, uint32_t freq) {
  const uint64_t rb = range >> 16;
  const uint64_t old = low;
  low += rb * cum;
  if (low < old) {  // carry back-patch (coder.cpp:101-109)
    uint64_t i = pos;
    for (;;) {
      out[i - 1] += 1;
      if (out[i - 1] != 0) break;
      --i;
    }
  }
  range = rb * freq;
  while (range < kRenorm) {
    out[pos++] = uint8_t(low >> 56);
    low <<= 8;
    range <<= 8;
  }
}

__device__ __forceinline__ uint8_t dec_byte(const uint8_t* in, uint64_t len, uint64_t& pos, int& err) {
  if (pos >= len) {
    err = 1;  // StreamExhausted
    return 0;
  }
  return in[pos++];
}

// exact floor(code / rb) clamped to 65535 (coder.cpp:144-146)
__device__ __forceinline__ uint32_t dec_target(uint64_t code, uint64_t rb) {
  // rb < 2^48, so rb * 2^16 cannot overflow: a (corrupt) code at or above it
  // clamps at once instead of stepping q up one at a time
  if (code >= (rb << 16)) return kTotal - 1;
  // now code < rb * 2^16: the quotient is below 2^16. A single-precision
  // estimate (relative error ~2^-22, so off by at most one) is made exact by
  // the integer corrections; q * rb < 2^64 throughout.
  uint32_t q = uint32_t(__fdividef(__ull2float_rn(code), __ull2float_rn(rb)));
  if (q > kTotal - 1) q = kTotal - 1;
  while (q > 0 && uint64_t(q) * rb > code) --q;
  while (code - uint64_t(q) * rb >= rb) ++q;
  return q;
}

__device__ __forceinline__ uint32_t dec_sym(uint64_t& code, uint64_t& range, const uint8_t* in,
                                            uint64_t len, uint64_t& pos, const uint32_t* cum,
                                            const uint32_t* freq, uint32_t V, int& err) {
  const uint64_t rb = range >> 16;
  const uint32_t tgt = dec_target(code, rb);
  uint32_t lo = 0, hi = V;
  while (hi - lo > 1) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (cum[mid] <= tgt) lo = mid;
    else hi = mid;
  }
  code -= rb * cum[lo];
  range = rb * freq[lo];
  while (range < kRenorm) {
    code = (code << 8) | dec_byte(in, len, pos, err);
    range <<= 8;
  }
  return lo;
}

// Uniform warm-up symbols j < min(t, L) of every chunk (pipeline.cpp:121-123).
__global__ void k_range_uniform(uint32_t* tokens, ChunkGeo geo, int t, int R, int V,
                                uint8_t* payload, const uint64_t* pay_off, const uint64_t* pay_len,
                                CoderState* cs, int n_chunks, bool decode) {
  pdl_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_chunks) return;
  const uint64_t L = geo.L[c], start = geo.start[c];
  const uint64_t nj = L < uint64_t(t) ? L : uint64_t(t);
  const uint32_t base = kTotal / uint32_t(V), extra = kTotal % uint32_t(V);
  uint8_t* buf = payload + pay_off[c];
  CoderState s;
  s.low = 0;
  s.range = ~0ull;
  s.pos = 0;
  s.code = 0;
  s.err = 0;
  s.pad = 0;
  if (decode) {
    for (int i = 0; i < 8; ++i) s.code = (s.code << 8) | dec_byte(buf, pay_len[c], s.pos, s.err);
    // uniform dist: freq_i = base + (i < extra), cum_i = i*base + min(i, extra)
    for (uint64_t j = 0; j < nj && !s.err; ++j)
      for (int r = 0; r < R; ++r) {
        const uint64_t rb = s.range >> 16;
        const uint32_t tgt = dec_target(s.code, rb);
        // symbol with cum_i <= tgt < cum_{i+1}
        uint32_t lo = 0, hi = uint32_t(V);
        while (hi - lo > 1) {
          const uint32_t mid = lo + (hi - lo) / 2;
          const uint32_t cmid = mid * base + (mid < extra ? mid : extra);
          if (cmid <= tgt) lo = mid;
          else hi = mid;
        }
        const uint32_t clo = lo * base + (lo < extra ? lo : extra);
        s.code -= rb * clo;
        s.range = rb * (base + (lo < extra ? 1u : 0u));
        while (s.range < kRenorm) {
          s.code = (s.code << 8) | dec_byte(buf, pay_len[c], s.pos, s.err);
          s.range <<= 8;
        }
        tokens[start + uint64_t(r) * L + j] = lo;
      }
  } else {
    for (uint64_t j = 0; j < nj; ++j)
      for (int r = 0; r < R; ++r) {
        const uint32_t sym = tokens[start + uint64_t(r) * L + j];
        enc_sym(s.low, s.range, buf, s.pos, sym * base + (sym < extra ? sym : extra),
                base + (sym < extra ? 1u : 0u));
      }
  }
  cs[c] = s;
}

constexpr int kMaxQ = 8;  // V <= 256 in registers; larger V uses the scalar search
constexpr int kCumAhead = 8;  // decode: cum rows staged this many rows ahead
__device__ __forceinline__ void cp_async4_u32(uint32_t* smem, const uint32_t* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
               "l"(gmem));
}

// Decode of one chunk's R symbols of this tick by one warp (NQ = ceil((V+1)/32)
// cum words per lane). Every lane carries the same coder state. The cum rows
// are staged kCumAhead rows ahead by per-lane async copies into the warp's
// shared ring (a lane copies and reads only its own entries); the symbol is a
// warp ballot count over the row (the reference's binary search: the largest
// i with cum[i] <= target); the payload is a register window (lane l holds
// bytes [wb + 4l, wb + 4l + 4) of the current 128 bytes, the next 128 bytes
// fetched when the window advances), so no byte read waits on memory.
template <int NQ>
__device__ __forceinline__ void range_decode_rows(CoderState& s, uint32_t* tokens, uint64_t start, uint64_t L,
                                                  uint64_t jstep, int R, int V, const uint32_t* cm,
                                                  const uint8_t* buf, uint64_t plen,
                                                  uint32_t (*ring)[kMaxQ * 32], int lane) {
  auto stage = [&](int r) {
    if (r < R) {
      uint32_t* dst = ring[r % kCumAhead];
      const uint32_t* src = cm + int64_t(r) * (V + 1);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int i = lane + 32 * q;
        if (i <= V) cp_async4_u32(dst + i, src + i);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
#pragma unroll
  for (int i = 0; i < kCumAhead - 1; ++i) stage(i);
  auto word = [&](uint64_t at) -> uint32_t {  // aligned 4 bytes at `at`, bytes >= plen read as 0
    if (at + 4 <= plen) return *reinterpret_cast<const uint32_t*>(buf + at);
    uint32_t v = 0;
    for (uint64_t b = at; b < plen && b < at + 4; ++b) v |= uint32_t(buf[b]) << (8 * (b - at));
    return v;
  };
  uint64_t wb = s.pos & ~uint64_t(127);
  uint32_t wa = word(wb + 4 * lane), wn = word(wb + 128 + 4 * lane);
  uint64_t code = s.code, range = s.range, pos = s.pos;
  // row r's cum words in registers, row r+1's loaded during row r
  uint32_t cur[NQ], nxt[NQ], mysym = 0;
  auto load_row = [&](int r, uint32_t (&x)[NQ]) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = lane + 32 * q;
      x[q] = i <= V ? ring[r % kCumAhead][i] : 0xffffffffu;
    }
  };
  asm volatile("cp.async.wait_group %0;\n" ::"n"(kCumAhead - 2));
  load_row(0, cur);
  for (int r = 0; r < R; ++r) {
    stage(r + kCumAhead - 1);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kCumAhead - 2));  // row r+1 landed
    if (r + 1 < R) load_row(r + 1, nxt);
    const uint64_t rb = range >> 16;
    // the reference's target is floor(code / rb) clamped to 65535 and the
    // symbol the largest i < V with cum[i] <= target; for integers
    // cum[i] <= floor(code / rb) <=> cum[i] * rb <= code (< 2^64: cum <= 2^16,
    // rb < 2^48), and counting only i < V is the clamp. So no division: each
    // lane compares its cum entries' products with code.
    int count = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = lane + 32 * q;
      count += __popc(__ballot_sync(0xffffffffu, i < V && uint64_t(cur[q]) * rb <= code));
    }
    const int sym = count - 1;
    // cum[sym] and cum[sym+1]: shuffle every word column, select after (a
    // register array indexed by sym would go through local memory)
    uint32_t csym = 0, cnext = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint32_t v0 = __shfl_sync(0xffffffffu, cur[q], sym & 31);
      const uint32_t v1 = __shfl_sync(0xffffffffu, cur[q], (sym + 1) & 31);
      if (q == (sym >> 5)) csym = v0;
      if (q == ((sym + 1) >> 5)) cnext = v1;
    }
    code -= rb * csym;
    range = rb * (cnext - csym);  // freq = cum[s+1] - cum[s]
    if (range < kRenorm) {
      // the reference's byte loop (range < 2^56: range = range << 8 | next
      // byte) runs once if range >= 2^48, else twice (range >= 2^40 since
      // rb >= 2^40 and freq >= 1): both bytes come from the window at once
      const bool two = range < (1ull << 48);
      if (pos + (two ? 2 : 1) > plen) s.err = 1;  // StreamExhausted (bytes past the end read as 0)
      if (pos >= wb + 128) {
        wb += 128;
        wa = wn;
        wn = word(wb + 128 + 4 * lane);
      }
      const uint32_t off = uint32_t(pos - wb), off1 = off + 1;
      const uint32_t w0 = __shfl_sync(0xffffffffu, wa, int(off >> 2));
      const uint32_t w1 = __shfl_sync(0xffffffffu, off1 < 128 ? wa : wn, int((off1 >> 2) & 31));
      const uint32_t b0 = (w0 >> (8 * (off & 3))) & 0xffu, b1 = (w1 >> (8 * (off1 & 3))) & 0xffu;
      if (two) {
        code = (code << 16) | (b0 << 8) | b1;
        range <<= 16;
        pos += 2;
      } else {
        code = (code << 8) | b0;
        range <<= 8;
        pos += 1;
      }
    }
    // the decoded symbols are stored 32 rows at a time (lane l keeps row r0+l's)
    if (lane == (r & 31)) mysym = uint32_t(sym);
    if ((r & 31) == 31 || r + 1 == R || s.err) {
      const int r0 = r & ~31;
      if (r0 + lane <= r) tokens[start + uint64_t(r0 + lane) * L + jstep] = mysym;
    }
    if (s.err) break;
#pragma unroll
    for (int q = 0; q < NQ; ++q) cur[q] = nxt[q];
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  s.code = code;
  s.range = range;
  s.pos = pos;
}

// One warp per chunk. Encode: the warp gathers 32 rows' (cum, freq) of the
// coded symbols into shared memory, lane 0 runs the 64-bit coder over them.
// Decode: every lane carries the same coder state; the symbol search is a
// warp ballot over the cum row held in registers (prefetched one row ahead),
// which equals the reference binary search (largest i with cum[i] <= target).
constexpr int kCoderWarps = 1;
__global__ void __launch_bounds__(kCoderWarps * 32) k_range_step(
    uint32_t* tokens, ChunkGeo geo, int t, int R, int V,
    const uint32_t* __restrict__ freq, const uint32_t* __restrict__ cum, int64_t cs_f,
    int64_t cs_c, uint8_t* payload, const uint64_t* pay_off, const uint64_t* pay_len,
    CoderState* cs, const TickDesc* __restrict__ td, bool decode) {
  pdl_wait();
  __shared__ uint32_t sc_[kCoderWarps][32], sf_[kCoderWarps][32];
  __shared__ uint32_t scum[kCoderWarps][kCumAhead][kMaxQ * 32];  // decode: staged cum rows
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wi = blockIdx.x * kCoderWarps + wl;
  if (wi >= td->n_act) return;
  const int c = td->act[wi], ch = td->chunk[wi];  // slot (freq/cum), chunk (codestream)
  const uint64_t L = geo.L[ch], start = geo.start[ch];
  const uint64_t jstep = uint64_t(t) + uint64_t(td->tick - geo.offset[ch]);
  uint8_t* buf = payload + pay_off[ch];
  CoderState s = cs[ch];
  if (s.err) return;
  const uint32_t* fq = freq + c * cs_f;
  const uint32_t* cm = cum + c * cs_c;
  if (!decode) {
    for (int r0 = 0; r0 < R; r0 += 32) {
      const int r = r0 + lane;
      if (r < R) {
        const uint32_t sym = tokens[start + uint64_t(r) * L + jstep];
        sc_[wl][lane] = cm[int64_t(r) * (V + 1) + sym];
        sf_[wl][lane] = fq[int64_t(r) * V + sym];
      }
      __syncwarp();
      if (lane == 0) {
        const int cnt = min(32, R - r0);
        for (int q = 0; q < cnt; ++q) enc_sym(s.low, s.range, buf, s.pos, sc_[wl][q], sf_[wl][q]);
      }
      __syncwarp();
    }
    if (lane == 0) cs[ch] = s;
    return;
  }
  const int nq = (V + 1 + 31) / 32;  // cum[0..V] (cum[V] = 2^16) in registers
  if (nq > kMaxQ) {  // large alphabets: scalar path in lane 0
    if (lane == 0) {
      for (int r = 0; r < R && !s.err; ++r) {
        const uint32_t sym = dec_sym(s.code, s.range, buf, pay_len[ch], s.pos, cm + int64_t(r) * (V + 1),
                                     fq + int64_t(r) * V, uint32_t(V), s.err);
        tokens[start + uint64_t(r) * L + jstep] = sym;
      }
      cs[ch] = s;
    }
    return;
  }
  switch (nq) {
    case 1: range_decode_rows<1>(s, tokens, start, L, jstep, R, V, cm, buf, pay_len[ch], scum[wl], lane); break;
    case 2: range_decode_rows<2>(s, tokens, start, L, jstep, R, V, cm, buf, pay_len[ch], scum[wl], lane); break;
    case 3: range_decode_rows<3>(s, tokens, start, L, jstep, R, V, cm, buf, pay_len[ch], scum[wl], lane); break;
    case 4: range_decode_rows<4>(s, tokens, start, L, jstep, R, V, cm, buf, pay_len[ch], scum[wl], lane); break;
    default: range_decode_rows<kMaxQ>(s, tokens, start, L, jstep, R, V, cm, buf, pay_len[ch], scum[wl], lane); break;
  }
  if (lane == 0) cs[ch] = s;
}

__global__ void k_range_finish(uint8_t* payload, const uint64_t* pay_off, CoderState* cs, int n) {
  pdl_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  CoderState s = cs[c];
  uint8_t* buf = payload + pay_off[c];
  for (int i = 0; i < 8; ++i) {
    buf[s.pos++] = uint8_t(s.low >> 56);
    s.low <<= 8;
  }
  cs[c] = s;
}

}  // namespace

void launch_mix_quantize(const MixP& p, const TickDesc* td, int max_active, cudaStream_t st) {
  if (max_active <= 0) return;
  dim3 grid(unsigned((int64_t(p.R) * 32 + 255) / 256), max_active);
  launch_pdl(k_mix_quantize, dim3(grid), dim3(256), 0, st, p, td);
}

void launch_bc_dlm(const BcP& p, const TickDesc* td, int max_active, cudaStream_t st) {
  if (max_active <= 0) return;
  dim3 grid(unsigned((int64_t(p.R) * p.V + 255) / 256), max_active);
  launch_pdl(k_bc_dlm, dim3(grid), dim3(256), 0, st, p, td);
}

void launch_alpha_step(const BcP& p, const TickDesc* td, int max_active, cudaStream_t st) {
  if (max_active <= 0) return;
  launch_pdl(k_alpha_step, dim3(unsigned(max_active)), dim3(256), 0, st, p, td);
}

void launch_range_uniform(uint32_t* tokens, ChunkGeo geo, int t, int R, int V, uint8_t* payload,
                          const uint64_t* pay_off, const uint64_t* pay_len, CoderState* cs,
                          int n_chunks, bool decode, cudaStream_t st) {
  if (n_chunks <= 0) return;
  launch_pdl(k_range_uniform, dim3(unsigned((n_chunks + 63) / 64)), dim3(64), 0, st, tokens, geo, t, R, V, payload,
                                                                 pay_off, pay_len, cs, n_chunks,
                                                                 decode);
}

void launch_range_step(uint32_t* tokens, ChunkGeo geo, int t, int R, int V,
                       const uint32_t* freq, const uint32_t* cum, int64_t cs_f, int64_t cs_c,
                       uint8_t* payload, const uint64_t* pay_off, const uint64_t* pay_len,
                       CoderState* cs, const TickDesc* td, int max_active, bool decode,
                       cudaStream_t st) {
  if (max_active <= 0) return;
  launch_pdl(k_range_step, dim3(unsigned((max_active + kCoderWarps - 1) / kCoderWarps)), dim3(kCoderWarps * 32), 0, st, tokens, geo, t, R, V, freq, cum,
                                                              cs_f, cs_c, payload, pay_off, pay_len,
                                                              cs, td, decode);
}

void launch_range_finish(uint8_t* payload, const uint64_t* pay_off, CoderState* cs, int n_chunks,
                         cudaStream_t st) {
  if (n_chunks <= 0) return;
  launch_pdl(k_range_finish, dim3(unsigned((n_chunks + 63) / 64)), dim3(64), 0, st, payload, pay_off, cs, n_chunks);
}

}  // namespace pmklc_b200
