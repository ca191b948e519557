// (s,k)-mer tokenizer, canonicalization and detokenize/restore for sm_100a.
//
// skmer encode (reference: core/src/skmer.cpp:16-24, token j = base-4 number of
// bases [j*s, j*s+k), most significant digit first) is HBM-bound: per base it
// reads 2 bits (packed) or 1 byte (ASCII) and writes 4*m/n bytes of u32 tokens.
// Each CTA stages the packed window covering its 8192 (s <= 2: 16384) tokens in
// shared memory with 128-bit coalesced loads (halo of k-1 bases included);
// every token is two 32-bit shared loads + a funnel shift + a 2-bit digit
// reversal (__brev), and each warp writes 128-token slabs as lane-contiguous
// 16-byte stores (512 contiguous bytes per store instruction).
#include <cstdint>
#include <cstring>
#include <type_traits>

#include "kernels.hpp"
#include "launch.cuh"

namespace pmklc_b200 {

namespace {

constexpr int kTokThreads = 256;
// tokens per thread: 64 for strides s <= 2 (larger tiles, fewer blocks),
// 32 otherwise (a 64-token tile at stride 8 needs 32 KB of staging and leaves
// too few blocks in flight); both stage <= 16 KB + slack
constexpr int kTpt = 32, kTptSmallStride = 64;
constexpr int kStageBytes = (kTokThreads * kTpt * 8 + 16) / 4 + 48;
static_assert(kTokThreads * kTptSmallStride * 2 <= kTokThreads * kTpt * 8, "staging bound");

__device__ __forceinline__ uint32_t ascii_code(uint32_t c) { return ((c >> 1) ^ (c >> 2)) & 3u; }

// Staged windows hold the bases MSB-first: base i of a 32-bit word at bits
// 31-2i..30-2i, so a token (k bases, first base most significant,
// skmer.cpp:16-24) is one contiguous 2k-bit field of the stream. msb_first
// turns a word of the packed input layout (base i at bits 2i..2i+1) into that
// form: bit reversal, then swap the two bits of every digit back.
__device__ __forceinline__ uint32_t msb_first(uint32_t w) {
  const uint32_t x = __brev(w);
  return ((x >> 1) & 0x55555555u) | ((x & 0x55555555u) << 1);
}

// Extract tokens [j0, j0 + 256*kTokPerThread) from a packed shared-memory
// window whose first byte holds base `sbase`. Warp w owns 32*kTokPerThread
// consecutive tokens as slabs of 32*PER (PER = 16 bytes / token size: 4 u32 or
// 8 u16 tokens); lane l makes tokens PER*l .. PER*l+PER-1 of each slab and
// writes them with one 16-byte store, so every warp store covers 512
// contiguous bytes.
// kPad: the staged window has one padding word after every 32 (word w at
// w + w/32). A lane's PER tokens span PER*s bases, so lanes read words PER*s/16
// apart -- a 4-way bank conflict for 8 u16 tokens at s = 8; with the padding
// the 32 lanes of such a stride land in 32 banks.
__device__ __forceinline__ uint32_t padw(uint32_t w) { return w + (w >> 5); }
template <int kTokPerThread, typename TokT, bool kPad = false>
__device__ __forceinline__ void emit_tokens(const uint32_t* sw, uint64_t sbase, uint64_t j0,
                                            uint32_t s, uint32_t k, TokT* tokens, uint64_t m) {
  constexpr int PER = 16 / int(sizeof(TokT));
  static_assert(kTokPerThread % PER == 0, "whole slabs per thread");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t jw = j0 + uint64_t(w) * 32 * kTokPerThread;
  if (jw >= m) return;
  const uint32_t rsh = 32u - 2u * k;  // k <= 16
#pragma unroll
  for (int slab = 0; slab < kTokPerThread / PER; ++slab) {
    const uint64_t jt = jw + uint64_t(slab) * 32 * PER + uint64_t(lane) * PER;
    uint32_t b = uint32_t(jt * s - sbase);  // base offset in the window (< 2^17)
    TokT out[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q, b += s) {
      const uint32_t wi = b >> 4, o = b & 15u;
      const uint32_t lo = kPad ? sw[padw(wi)] : sw[wi], hi = kPad ? sw[padw(wi + 1)] : sw[wi + 1];
      out[q] = TokT(__funnelshift_l(hi, lo, 2u * o) >> rsh);
    }
    if (jt + PER <= m) {
      uint4 v;
      memcpy(&v, out, 16);
      *reinterpret_cast<uint4*>(tokens + jt) = v;
    } else {
      for (int q = 0; q < PER && jt + q < m; ++q) tokens[jt + q] = out[q];
    }
  }
}

// The same extraction at a compile-time stride kS: a lane's PER tokens span
// (PER-1)*kS + k bases from its first base, so it loads that span's NW words
// once, aligns them to its first base with one runtime funnel shift per word,
// and cuts every token out at compile-time word and bit offsets (u16, s = 3:
// 4 shared loads per 8 tokens instead of 16).
template <int kTokPerThread, typename TokT, int kS, bool kPad = false>
__device__ __forceinline__ void emit_tokens_s(const uint32_t* sw, uint64_t sbase, uint64_t j0, uint32_t k,
                                              TokT* tokens, uint64_t m) {
  constexpr int PER = 16 / int(sizeof(TokT));
  static_assert(kTokPerThread % PER == 0, "whole slabs per thread");
  constexpr int NA = ((PER - 1) * kS) / 16 + 2;  // aligned words a lane's tokens touch
  constexpr int NW = NA + 1;                     // staged words behind them
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t jw = j0 + uint64_t(w) * 32 * kTokPerThread;
  if (jw >= m) return;
  const uint32_t rsh = 32u - 2u * k;  // k <= 16
#pragma unroll
  for (int slab = 0; slab < kTokPerThread / PER; ++slab) {
    const uint64_t jt = jw + uint64_t(slab) * 32 * PER + uint64_t(lane) * PER;
    const uint32_t b = uint32_t(jt * kS - sbase);  // first base of the lane in the window
    const uint32_t w0 = b >> 4, sh = 2u * (b & 15u);
    uint32_t W[NW], A[NA];
#pragma unroll
    for (int i = 0; i < NW; ++i) W[i] = kPad ? sw[padw(w0 + i)] : sw[w0 + i];
#pragma unroll
    for (int i = 0; i < NA; ++i) A[i] = __funnelshift_l(W[i + 1], W[i], sh);
    TokT out[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int qi = (q * kS) / 16, oo = (q * kS) % 16;
      out[q] = TokT(__funnelshift_l(A[qi + 1], A[qi], 2u * oo) >> rsh);
    }
    if (jt + PER <= m) {
      uint4 v;
      memcpy(&v, out, 16);
      *reinterpret_cast<uint4*>(tokens + jt) = v;
    } else {
      for (int q = 0; q < PER && jt + q < m; ++q) tokens[jt + q] = out[q];
    }
  }
}

// kS: the stride at compile time (1..8, the reference's range), 0 = runtime
template <int kTokPerThread, typename TokT, bool kPad = false, int kS = 0>
__global__ void __launch_bounds__(kTokThreads) k_skmer_packed(const uint8_t* __restrict__ packed,
                                                              uint64_t n, uint32_t s, uint32_t k,
                                                              TokT* __restrict__ tokens,
                                                              uint64_t m) {
  pdl_wait();
  __shared__ __align__(16) uint32_t sw[kStageBytes / 4 + (kPad ? kStageBytes / 128 + 2 : 0) + 8];
  constexpr int kTokPerBlock = kTokThreads * kTokPerThread;
  const uint64_t j0 = uint64_t(blockIdx.x) * kTokPerBlock;
  const uint64_t jlast = min(j0 + kTokPerBlock, m) - 1;
  const uint64_t b_first = j0 * s, b_end = jlast * s + k;  // bases needed [b_first, b_end)
  const uint64_t byte0 = (b_first / 4) & ~uint64_t(15);
  const uint64_t byte_end = min((b_end + 3) / 4, (n + 3) / 4);
  const uint64_t nbytes = byte_end - byte0;
  const uint64_t nvec = nbytes / 16;
  const uint4* src = reinterpret_cast<const uint4*>(packed + byte0);
  if (!kPad) {
    uint4* dst = reinterpret_cast<uint4*>(sw);
    for (uint64_t i = threadIdx.x; i < nvec; i += kTokThreads) dst[i] = __ldg(src + i);
    uint8_t* sb = reinterpret_cast<uint8_t*>(sw);
    for (uint64_t i = nvec * 16 + threadIdx.x; i < nbytes + 8; i += kTokThreads)
      sb[i] = i < nbytes ? packed[byte0 + i] : 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < uint32_t((nbytes + 8 + 3) / 4); i += kTokThreads) sw[i] = msb_first(sw[i]);
  } else {
    // 16-byte loads, digit order fixed on the way in, padded word positions
    for (uint64_t i = threadIdx.x; i < nvec; i += kTokThreads) {
      const uint4 v = __ldg(src + i);
      const uint32_t w0 = uint32_t(4 * i);
      sw[padw(w0)] = msb_first(v.x);
      sw[padw(w0 + 1)] = msb_first(v.y);
      sw[padw(w0 + 2)] = msb_first(v.z);
      sw[padw(w0 + 3)] = msb_first(v.w);
    }
    const uint32_t nw = uint32_t((nbytes + 8 + 3) / 4);
    for (uint32_t wd = uint32_t(nvec * 4) + threadIdx.x; wd < nw; wd += kTokThreads) {
      uint32_t x = 0;
      for (int c = 0; c < 4; ++c) {
        const uint64_t i = uint64_t(wd) * 4 + c;
        x |= uint32_t(i < nbytes ? packed[byte0 + i] : 0) << (8 * c);
      }
      sw[padw(wd)] = msb_first(x);
    }
  }
  __syncthreads();
  if constexpr (kS > 0)
    emit_tokens_s<kTokPerThread, TokT, kS, kPad>(sw, byte0 * 4, j0, k, tokens, m);
  else
    emit_tokens<kTokPerThread, TokT, kPad>(sw, byte0 * 4, j0, s, k, tokens, m);
}

// ASCII / code input: stage 16 bytes per step, pack to 2-bit on the way in.
template <bool kAscii, int kTokPerThread>
__global__ void __launch_bounds__(kTokThreads) k_skmer_bytes(const uint8_t* __restrict__ in,
                                                             uint64_t n, uint32_t s, uint32_t k,
                                                             uint32_t* __restrict__ tokens,
                                                             uint64_t m) {
  pdl_wait();
  __shared__ __align__(16) uint32_t sw[kStageBytes / 4];
  constexpr int kTokPerBlock = kTokThreads * kTokPerThread;
  const uint64_t j0 = uint64_t(blockIdx.x) * kTokPerBlock;
  const uint64_t jlast = min(j0 + kTokPerBlock, m) - 1;
  const uint64_t b_first = j0 * s, b_end = jlast * s + k;
  const uint64_t base0 = b_first & ~uint64_t(15);  // 16-base (16-byte) aligned
  const uint64_t nb = b_end - base0;
  const uint64_t nwords = (nb + 15) / 16;  // one u32 of packed codes per 16 input bytes
  for (uint64_t w = threadIdx.x; w < nwords; w += kTokThreads) {
    const uint64_t b = base0 + w * 16;
    uint32_t packed = 0;
    if (b + 16 <= n && ((reinterpret_cast<uintptr_t>(in + b) & 15) == 0)) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(in + b));
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t byte = (wv[q] >> (8 * c)) & 0xffu;
          packed |= (kAscii ? ascii_code(byte) : (byte & 3u)) << (30 - 2 * (q * 4 + c));  // MSB-first
        }
    } else {
      for (int c = 0; c < 16; ++c) {
        const uint32_t byte = (b + c < n) ? in[b + c] : 0u;
        packed |= (kAscii ? ascii_code(byte) : (byte & 3u)) << (30 - 2 * c);
      }
    }
    sw[w] = packed;
  }
  if (threadIdx.x == 0) sw[nwords] = 0;
  __syncthreads();
  emit_tokens<kTokPerThread, uint32_t>(sw, base0, j0, s, k, tokens, m);
}

// ------------------------------------------------------------ canonicalize
constexpr int kCanonThreads = 256;
constexpr int kCanonPerThread = 16;
constexpr int kCanonPerBlock = kCanonThreads * kCanonPerThread;  // 4096 bytes

__device__ __forceinline__ bool is_acgt(uint32_t c) {
  return c == 'A' || c == 'C' || c == 'G' || c == 'T';
}

__global__ void k_canon_count(const uint8_t* __restrict__ raw, uint64_t n, uint32_t* counts) {
  pdl_wait();
  const uint64_t b0 = uint64_t(blockIdx.x) * kCanonPerBlock + threadIdx.x * kCanonPerThread;
  uint32_t c = 0;
  for (int i = 0; i < kCanonPerThread; ++i)
    if (b0 + i < n && !is_acgt(raw[b0 + i])) ++c;
  // block reduce
  __shared__ uint32_t red[kCanonThreads / 32];
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kCanonThreads / 32; ++w) t += red[w];
    counts[blockIdx.x] = t;
  }
}

// block_exc: exclusive prefix of exception counts per block (blocks+1 entries)
__global__ void k_canon_scatter(const uint8_t* __restrict__ raw, uint64_t n,
                                const uint64_t* __restrict__ block_exc, uint8_t* codes,
                                uint64_t* exc_pos, uint8_t* exc_byte) {
  pdl_wait();
  const uint64_t b0 = uint64_t(blockIdx.x) * kCanonPerBlock + threadIdx.x * kCanonPerThread;
  uint32_t c = 0;
  uint8_t v[kCanonPerThread];
  for (int i = 0; i < kCanonPerThread; ++i) {
    v[i] = (b0 + i < n) ? raw[b0 + i] : 'A';
    if (b0 + i < n && !is_acgt(v[i])) ++c;
  }
  // exclusive block scan of c
  __shared__ uint32_t wsum[kCanonThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = c;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  uint32_t before = 0;
  for (int w = 0; w < wid; ++w) before += wsum[w];
  uint64_t e = block_exc[blockIdx.x] + before + (inc - c);
  for (int i = 0; i < kCanonPerThread; ++i) {
    const uint64_t p = b0 + i;
    if (p >= n) break;
    if (is_acgt(v[i])) {
      codes[p - e] = uint8_t(ascii_code(v[i]));
    } else {
      exc_pos[e] = p;
      exc_byte[e] = v[i];
      ++e;
    }
  }
}

// ------------------------------------------------------------ detokenize
__global__ void k_detok_restore(const uint32_t* __restrict__ tokens, uint64_t m, uint32_t s,
                                uint32_t k, const uint8_t* __restrict__ residual, uint64_t n_res,
                                const uint64_t* __restrict__ exc_pos,
                                const uint8_t* __restrict__ exc_byte, uint64_t n_exc,
                                uint8_t* __restrict__ out, uint64_t out_len, int* err) {
  pdl_wait();
  constexpr int kPer = 16;
  const uint64_t o0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * kPer;
  if (o0 >= out_len) return;
  const uint64_t covered = m ? (m - 1) * s + k : 0;
  const uint32_t width_mask = (1u << (2 * k)) - 1u;
  // exceptions before o0
  uint64_t lo = 0, hi = n_exc;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (exc_pos[mid] < o0) lo = mid + 1;
    else hi = mid;
  }
  uint64_t e = lo;
  uint8_t buf[kPer];
  for (int i = 0; i < kPer; ++i) {
    const uint64_t o = o0 + i;
    if (o >= out_len) break;
    if (e < n_exc && exc_pos[e] == o) {
      buf[i] = exc_byte[e++];
      continue;
    }
    const uint64_t b = o - e;  // base index
    uint32_t code;
    if (b < covered) {
      uint64_t j = b / s;
      if (j > m - 1) j = m - 1;
      const uint32_t digit = uint32_t(b - j * s);
      const uint32_t tok = tokens[j];
      if (tok > width_mask) atomicExch(err, 1);
      code = (tok >> (2 * (k - 1 - digit))) & 3u;
    } else {
      const uint64_t rb = b - covered;
      if (rb >= n_res) {
        atomicExch(err, 2);
        code = 0;
      } else {
        code = residual[rb] & 3u;
      }
    }
    buf[i] = "ACGT"[code];
  }
  if (o0 + kPer <= out_len && ((reinterpret_cast<uintptr_t>(out + o0) & 15) == 0)) {
    uint4 v;
    uint32_t* vw = reinterpret_cast<uint32_t*>(&v);
    for (int q = 0; q < 4; ++q)
      vw[q] = uint32_t(buf[4 * q]) | uint32_t(buf[4 * q + 1]) << 8 | uint32_t(buf[4 * q + 2]) << 16 |
              uint32_t(buf[4 * q + 3]) << 24;
    *reinterpret_cast<uint4*>(out + o0) = v;
  } else {
    for (int i = 0; i < kPer && o0 + i < out_len; ++i) out[o0 + i] = buf[i];
  }
}

}  // namespace

// f(integral_constant<int, s>) for the reference's strides 1..8, else f(<0>)
template <typename F>
static void with_stride(uint32_t s, F&& f) {
  using std::integral_constant;
  switch (s) {
    case 1: f(integral_constant<int, 1>{}); break;
    case 2: f(integral_constant<int, 2>{}); break;
    case 3: f(integral_constant<int, 3>{}); break;
    case 4: f(integral_constant<int, 4>{}); break;
    case 5: f(integral_constant<int, 5>{}); break;
    case 6: f(integral_constant<int, 6>{}); break;
    case 7: f(integral_constant<int, 7>{}); break;
    case 8: f(integral_constant<int, 8>{}); break;
    default: f(integral_constant<int, 0>{}); break;
  }
}
template <typename TokT>
static void launch_packed(const uint8_t* packed, uint64_t n, uint32_t s, uint32_t k, TokT* tokens,
                          uint64_t m, cudaStream_t st) {
  if (m == 0) return;
  with_stride(s, [&](auto s_c) {
    constexpr int kS = decltype(s_c)::value;
    if (s <= 2) {
      const uint64_t blocks = (m + kTokThreads * kTptSmallStride - 1) / (kTokThreads * kTptSmallStride);
      launch_pdl(k_skmer_packed<kTptSmallStride, TokT, false, kS>, dim3(unsigned(blocks)), dim3(kTokThreads), 0,
                 st, packed, n, s, k, tokens, m);
    } else {
      const uint64_t blocks = (m + kTokThreads * kTpt - 1) / (kTokThreads * kTpt);
      launch_pdl(k_skmer_packed<kTpt, TokT, false, kS>, dim3(unsigned(blocks)), dim3(kTokThreads), 0, st, packed,
                 n, s, k, tokens, m);
    }
  });
}
void launch_skmer_encode_packed(const uint8_t* packed, uint64_t n, uint32_t s, uint32_t k,
                                uint32_t* tokens, uint64_t m, cudaStream_t st) {
  launch_packed(packed, n, s, k, tokens, m, st);
}
// u16 tokens write half the bytes per token, so a block's staging phase
// (window load, digit reversal, two barriers) is amortised over twice (s <= 4)
// or four times (s <= 2) the tokens; the staged window stays <= 64 Ki bases
void launch_skmer_encode_packed16(const uint8_t* packed, uint64_t n, uint32_t s, uint32_t k,
                                  uint16_t* tokens, uint64_t m, cudaStream_t st) {
  if (m == 0) return;
  auto go = [&](auto tpt_c, auto smax_c, auto pad_c) {
    constexpr int tpt = decltype(tpt_c)::value, smax = decltype(smax_c)::value;
    // the window of a block: tpt*256 tokens at stride <= smax, + k-1 halo, 16-byte aligned
    static_assert(kTokThreads * tpt * smax / 4 + 32 <= kStageBytes, "staging bound");
    const uint64_t blocks = (m + kTokThreads * tpt - 1) / (kTokThreads * tpt);
    with_stride(s, [&](auto s_c) {
      launch_pdl(k_skmer_packed<tpt, uint16_t, decltype(pad_c)::value, decltype(s_c)::value>,
                 dim3(unsigned(blocks)), dim3(kTokThreads), 0, st, packed, n, s, k, tokens, m);
    });
  };
  // measured (2^30 bases): the padded staging pays off only where a lane's 8
  // tokens span >= 2.5 words (s > 4: 0.50 -> 0.69 of the copy peak at (8,8));
  // at s <= 4 its scalar stores cost more than the 2-way conflicts it removes
  using std::integral_constant;
  if (s <= 2)
    go(integral_constant<int, 2 * kTptSmallStride>{}, integral_constant<int, 2>{}, std::false_type{});
  else if (s <= 4)
    go(integral_constant<int, 2 * kTpt>{}, integral_constant<int, 4>{}, std::false_type{});
  else
    go(integral_constant<int, kTpt>{}, integral_constant<int, 8>{}, std::true_type{});
}

void launch_skmer_encode_ascii(const uint8_t* ascii, uint64_t n, uint32_t s, uint32_t k,
                               uint32_t* tokens, uint64_t m, cudaStream_t st) {
  if (!m) return;
  const uint64_t blocks = (m + kTokThreads * kTpt - 1) / (kTokThreads * kTpt);
  launch_pdl(k_skmer_bytes<true, kTpt>, dim3(unsigned(blocks)), dim3(kTokThreads), 0, st, ascii, n, s, k, tokens, m);
}
void launch_skmer_encode_codes(const uint8_t* codes, uint64_t n, uint32_t s, uint32_t k,
                               uint32_t* tokens, uint64_t m, cudaStream_t st) {
  if (!m) return;
  const uint64_t blocks = (m + kTokThreads * kTpt - 1) / (kTokThreads * kTpt);
  launch_pdl(k_skmer_bytes<false, kTpt>, dim3(unsigned(blocks)), dim3(kTokThreads), 0, st, codes, n, s, k, tokens, m);
}
uint32_t canon_blocks(uint64_t n) { return uint32_t((n + kCanonPerBlock - 1) / kCanonPerBlock); }
void launch_canon_count(const uint8_t* raw, uint64_t n, uint32_t* counts, cudaStream_t st) {
  if (!n) return;
  launch_pdl(k_canon_count, dim3(canon_blocks(n)), dim3(kCanonThreads), 0, st, raw, n, counts);
}
void launch_canon_scatter(const uint8_t* raw, uint64_t n, const uint64_t* block_exc,
                          uint8_t* codes, uint64_t* exc_pos, uint8_t* exc_byte, cudaStream_t st) {
  if (!n) return;
  launch_pdl(k_canon_scatter, dim3(canon_blocks(n)), dim3(kCanonThreads), 0, st, raw, n, block_exc, codes, exc_pos,
                                                             exc_byte);
}
void launch_detokenize_restore(const uint32_t* tokens, uint64_t m, uint32_t s, uint32_t k,
                               const uint8_t* residual, uint64_t n_res, const uint64_t* exc_pos,
                               const uint8_t* exc_byte, uint64_t n_exc, uint8_t* out,
                               uint64_t out_len, int* err, cudaStream_t st) {
  if (!out_len) return;
  const uint64_t threads = (out_len + 15) / 16;
  launch_pdl(k_detok_restore, dim3(unsigned((threads + 255) / 256)), dim3(256), 0, st, 
      tokens, m, s, k, residual, n_res, exc_pos, exc_byte, n_exc, out, out_len, err);
}

}  // namespace pmklc_b200
