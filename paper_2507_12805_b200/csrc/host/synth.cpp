// Seeded synthetic DNA generators for benchmarks and tests.
// Pure integer SplitMix64 + IEEE float arithmetic, so the same seed yields the
// same bytes on any host. Not on the compress/decompress path.
#include <cstdint>
#include <cstring>
#include <vector>

#include "rng.hpp"

namespace pmklc_b200 {

namespace {
const uint8_t kBases[4] = {'A', 'C', 'G', 'T'};

// Order-`order` Markov source: per context, p_b ∝ (u+0.05)^3,
// optionally mixed with uniform at weight `mix_uniform` and GC-shifted.
struct MarkovTable {
  int order;
  std::vector<float> cdf;  // [4^order][4]
  MarkovTable(int ord, Rng& rng, float mix_uniform, float gc_shift) : order(ord) {
    const size_t nctx = size_t(1) << (2 * ord);
    cdf.resize(nctx * 4);
    for (size_t c = 0; c < nctx; ++c) {
      float p[4], s = 0.0f;
      for (int i = 0; i < 4; ++i) {
        p[i] = rng.next_float() + 0.05f;
        p[i] = p[i] * p[i] * p[i];
        s += p[i];
      }
      if (mix_uniform > 0.0f || gc_shift != 0.0f) {
        float s2 = 0.0f;
        for (int i = 0; i < 4; ++i) {
          float q = (1.0f - mix_uniform) * (p[i] / s) + mix_uniform * 0.25f;
          if (i == 1 || i == 2) q = q * (1.0f + gc_shift);
          p[i] = q;
          s2 += q;
        }
        s = s2;
      }
      float a = 0.0f;
      for (int i = 0; i < 4; ++i) {
        a += p[i] / s;
        cdf[c * 4 + i] = a;
      }
    }
  }
  unsigned draw(unsigned ctx, float u) const {
    unsigned b = 0;
    while (b < 3 && u >= cdf[size_t(ctx) * 4 + b]) ++b;
    return b;
  }
  unsigned mask() const { return (1u << (2 * order)) - 1u; }
};
}  // namespace

// SURVEY Appendix E markov3(n, seed): order-3 source, one Rng stream.
void synth_markov3(uint8_t* out, uint64_t n, uint64_t seed) {
  Rng rng(seed);
  MarkovTable tab(3, rng, 0.0f, 0.0f);
  unsigned ctx = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const unsigned b = tab.draw(ctx, rng.next_float());
    out[i] = kBases[b];
    ctx = ((ctx << 2) | b) & 63u;
  }
}

// Uniform i.i.d. bases "ACGT"[next_below(4)] (SURVEY App. E uniform fixture).
void synth_uniform(uint8_t* out, uint64_t n, uint64_t seed) {
  Rng rng(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = kBases[rng.next_below(4)];
}

// Uniform 2-bit codes packed 4 per byte, base i in bits 2*(i%4) (config 2).
void synth_packed_codes(uint8_t* out, uint64_t n_bytes, uint64_t seed) {
  Rng rng(seed);
  uint64_t i = 0;
  for (; i + 8 <= n_bytes; i += 8) {
    const uint64_t v = rng.next_u64();
    std::memcpy(out + i, &v, 8);
  }
  if (i < n_bytes) {
    const uint64_t v = rng.next_u64();
    std::memcpy(out + i, &v, size_t(n_bytes - i));
  }
}

// Config 3/4: `segments` order-k Markov segments (k in 2..5, distinct seeds,
// GC bias varied) concatenated, with ~1% of 1000-base windows replaced by
// copies of an earlier window (copy-repeats).
void synth_genome(uint8_t* out, uint64_t n, uint64_t seed, uint32_t segments) {
  if (segments == 0) segments = 1;
  Rng master(seed);
  const uint64_t seg_len = (n + segments - 1) / segments;
  uint64_t pos = 0;
  for (uint32_t s = 0; s < segments && pos < n; ++s) {
    Rng rng(master.next_u64());
    const int order = 2 + int(s % 4);
    const float gc = -0.2f + 0.4f * float(s % 5) / 4.0f;
    MarkovTable tab(order, rng, 0.0f, gc);
    unsigned ctx = 0;
    const uint64_t end = pos + seg_len < n ? pos + seg_len : n;
    for (; pos < end; ++pos) {
      const unsigned b = tab.draw(ctx, rng.next_float());
      out[pos] = kBases[b];
      ctx = ((ctx << 2) | b) & tab.mask();
    }
  }
  Rng rep(seed ^ 0x5eedull);
  const uint64_t win = 1000;
  if (n > 4 * win) {
    const uint64_t nrep = n / win / 100;
    for (uint64_t r = 0; r < nrep; ++r) {
      const uint64_t dst = win + rep.next_below(n - 2 * win);
      const uint64_t src = rep.next_below(dst - win + 1);
      std::memmove(out + dst, out + src, win);
    }
  }
}

// Config 5: mixture of 8 "species" sources switching every block; every 16th
// 64 MiB block is drawn from a perturbed table (mixed with uniform at 0.3,
// GC-shifted). block = 0 selects 64 MiB.
void synth_species(uint8_t* out, uint64_t n, uint64_t seed, uint64_t block) {
  if (block == 0) block = uint64_t(64) << 20;
  Rng master(seed);
  std::vector<MarkovTable> sp, pert;
  for (int s = 0; s < 8; ++s) {
    Rng r1(master.next_u64());
    sp.emplace_back(1 + s % 5, r1, 0.0f, 0.0f);
    Rng r2(master.next_u64());
    pert.emplace_back(1 + s % 5, r2, 0.3f, 0.25f);
  }
  Rng rng(master.next_u64());
  unsigned ctx = 0;
  for (uint64_t b0 = 0, blk = 0; b0 < n; b0 += block, ++blk) {
    const MarkovTable& tab = (blk % 16 == 15) ? pert[blk % 8] : sp[blk % 8];
    const uint64_t end = b0 + block < n ? b0 + block : n;
    for (uint64_t i = b0; i < end; ++i) {
      const unsigned b = tab.draw(ctx & tab.mask(), rng.next_float());
      out[i] = kBases[b];
      ctx = (ctx << 2) | b;
    }
  }
}

}  // namespace pmklc_b200
