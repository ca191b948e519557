// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// Thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/core, compiled from its own sources by oracle/Makefile
// into oracle/_ref/libpmklc_ref.so). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it. Nothing here
// re-implements reference arithmetic: every call goes straight into the
// reference's public API (pipeline.hpp, skmer.hpp, coder.hpp, models.hpp,
// mixer.hpp).
//
// pmref_dump_chunk() drives one chunk through the reference's public classes
// in exactly the order ChunkWorker::encode uses (pipeline.cpp:115-137,
// 178-213) so the per-step mixed probabilities can be captured; the chunk's
// payload it returns is checked against compress() in the tests, which pins
// the replay to the reference's own code path.

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "pmklc/alphabet.hpp"
#include "pmklc/coder.hpp"
#include "pmklc/detmath.hpp"
#include "pmklc/error.hpp"
#include "pmklc/io.hpp"
#include "pmklc/mixer.hpp"
#include "pmklc/models.hpp"
#include "pmklc/pipeline.hpp"
#include "pmklc/skmer.hpp"
#include "pmklc/training.hpp"
#include "pmklc/weights.hpp"

using namespace pmklc;

namespace {
thread_local std::string g_err;

struct RefCfg {
  uint32_t s, k, t, bs, workers, scale;
  uint64_t threshold, seed;
  float smp;
  const char* pub_path;
};

struct RefChunkStats {
  uint64_t tokens, uniform_coded, pub_calls, priv_calls, dyn_calls;
  uint64_t snapshot_recv_hash, snapshot_sent_hash;
  double early_loss_bits;
};

template <class F> int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const error& e) {
    g_err = e.what();
    return 1 + int(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1000;
  }
}

uint8_t* dup(const ByteVec& v) {
  uint8_t* p = static_cast<uint8_t*>(std::malloc(v.size() ? v.size() : 1));
  if (!v.empty()) std::memcpy(p, v.data(), v.size());
  return p;
}

CompressConfig to_cfg(const RefCfg* c) {
  CompressConfig cfg;
  cfg.sk = SkParams{uint8_t(c->s), uint8_t(c->k)};
  cfg.t = c->t;
  cfg.bs = c->bs;
  cfg.workers = c->workers;
  cfg.scale = c->scale;
  cfg.selector_threshold = c->threshold;
  cfg.seed = c->seed;
  cfg.smp_fraction = c->smp;
  if (c->pub_path) cfg.pub_model_path = c->pub_path;
  return cfg;
}

void copy_stats(const PipelineStats& ps, RefChunkStats* out, size_t cap) {
  if (!out) return;
  for (size_t i = 0; i < ps.workers.size() && i < cap; ++i) {
    const WorkerStats& w = ps.workers[i];
    out[i] = RefChunkStats{w.tokens,    w.uniform_coded,      w.pub_calls,          w.priv_calls,
                           w.dyn_calls, w.snapshot_recv_hash, w.snapshot_sent_hash, w.early_loss_bits};
  }
}
} // namespace

extern "C" {

const char* pmref_last_error(void) { return g_err.c_str(); }
uint64_t pmref_fnv1a64(const uint8_t* p, size_t n) { return fnv1a64(ByteSpan(p, n)); }
void pmref_free(void* p) { std::free(p); }

int pmref_compress(const uint8_t* in, size_t n, const RefCfg* c, uint8_t** out, size_t* out_n,
                   RefChunkStats* stats, size_t stats_cap, size_t* n_chunks) {
  return guard([&] {
    PipelineStats ps;
    ByteVec v = compress(ByteSpan(in, n), to_cfg(c), stats ? &ps : nullptr);
    copy_stats(ps, stats, stats_cap);
    if (n_chunks) *n_chunks = ps.workers.size();
    *out = dup(v);
    *out_n = v.size();
  });
}

int pmref_decompress(const uint8_t* in, size_t n, const char* pub_path, uint32_t workers,
                     uint8_t** out, size_t* out_n, RefChunkStats* stats, size_t stats_cap) {
  return guard([&] {
    PipelineStats ps;
    ByteVec v = decompress(ByteSpan(in, n), pub_path ? pub_path : "", workers, stats ? &ps : nullptr);
    copy_stats(ps, stats, stats_cap);
    *out = dup(v);
    *out_n = v.size();
  });
}

int pmref_validate(const RefCfg* c) {
  return guard([&] { to_cfg(c).validate(); });
}

int pmref_plan_chunks(uint64_t m, uint32_t workers, uint32_t bs, uint32_t t, uint16_t myriad,
                      uint64_t* starts, uint64_t* lens, uint64_t* snaps, size_t cap, size_t* count,
                      uint32_t* bs_out) {
  return guard([&] {
    ChunkPlan p = plan_chunks(m, workers, bs, t, myriad);
    *count = p.ranges.size();
    *bs_out = p.bs;
    for (size_t i = 0; i < p.ranges.size() && i < cap; ++i) {
      starts[i] = p.ranges[i].start;
      lens[i] = p.ranges[i].len;
      snaps[i] = p.bs ? p.snapshot_step(i) : 0;
    }
  });
}

int pmref_skmer_encode(const uint8_t* codes, uint64_t n, uint32_t s, uint32_t k, uint32_t workers,
                       uint32_t* tokens, uint64_t* m_out, uint8_t* residual, uint64_t* res_n) {
  return guard([&] {
    NucleotideStream st;
    st.payload.assign(codes, codes + n);
    TokenSequence ts = encode(st, SkParams{uint8_t(s), uint8_t(k)}, workers);
    *m_out = ts.tokens.size();
    if (tokens && !ts.tokens.empty()) std::memcpy(tokens, ts.tokens.data(), ts.tokens.size() * 4);
    *res_n = ts.residual.size();
    if (residual && !ts.residual.empty()) std::memcpy(residual, ts.residual.data(), ts.residual.size());
  });
}

int pmref_canonicalize(const uint8_t* raw, uint64_t n, uint8_t* codes, uint64_t* n_codes,
                       uint64_t* exc_pos, uint8_t* exc_byte, uint64_t* n_exc) {
  return guard([&] {
    auto [st, exc] = canonicalize(ByteSpan(raw, n));
    *n_codes = st.payload.size();
    if (codes && !st.payload.empty()) std::memcpy(codes, st.payload.data(), st.payload.size());
    *n_exc = exc.entries.size();
    for (size_t i = 0; i < exc.entries.size(); ++i) {
      if (exc_pos) exc_pos[i] = exc.entries[i].position;
      if (exc_byte) exc_byte[i] = exc.entries[i].original_byte;
    }
  });
}

int pmref_quantize(const float* p, uint32_t n, uint32_t* freqs) {
  return guard([&] {
    QuantizedDistribution d = quantize(std::span<const float>(p, n));
    std::memcpy(freqs, d.freqs.data(), n * 4);
  });
}

int pmref_uniform_dist(uint32_t n, uint32_t* freqs) {
  return guard([&] {
    QuantizedDistribution d = uniform_dist(n);
    std::memcpy(freqs, d.freqs.data(), n * 4);
  });
}

/// Range-code `count` symbols, symbol i under the distribution freqs[dist_of[i]*width ...].
int pmref_range_encode(const uint32_t* freqs, uint32_t width, const uint32_t* dist_of,
                       const uint32_t* syms, size_t count, uint8_t** out, size_t* out_n) {
  return guard([&] {
    size_t ndist = 0;
    for (size_t i = 0; i < count; ++i) ndist = std::max<size_t>(ndist, dist_of[i] + 1);
    std::vector<QuantizedDistribution> d(ndist);
    for (size_t j = 0; j < ndist; ++j) {
      d[j].freqs.assign(freqs + j * width, freqs + (j + 1) * width);
      d[j].cum.resize(width + 1);
      uint32_t a = 0;
      for (uint32_t i = 0; i < width; ++i) {
        d[j].cum[i] = a;
        a += d[j].freqs[i];
      }
      d[j].cum[width] = a;
    }
    ByteVec buf;
    RangeEncoder enc(buf);
    for (size_t i = 0; i < count; ++i) enc.encode(d[dist_of[i]], syms[i]);
    enc.finish();
    *out = dup(buf);
    *out_n = buf.size();
  });
}

int pmref_det(int which, const float* x, float* y, size_t n) {
  return guard([&] {
    for (size_t i = 0; i < n; ++i) {
      switch (which) {
        case 0: y[i] = det_exp(x[i]); break;
        case 1: y[i] = det_log(x[i]); break;
        case 2: y[i] = det_sigmoid(x[i]); break;
        case 3: y[i] = det_tanh(x[i]); break;
        default: raise(errc::config_invalid, "det selector");
      }
    }
  });
}

int pmref_softmax(const float* x, float* y, size_t n) {
  return guard([&] { det_softmax(x, y, n); });
}

/// Writes a seeded (untrained) BiGRU model file, as the reference tests do
/// (acceptance.cpp:58-69). layers = 2 for a SPuM.
int pmref_write_bigru(uint32_t vocab, uint32_t t, uint32_t scale, int layers, uint64_t seed,
                      const char* path, uint64_t* fingerprint) {
  return guard([&] {
    const ModelDims dims = ModelDims::make(vocab, t, scale);
    BiGruModel m(dims, layers, seed);
    ByteVec bytes = serialize_model(m);
    write_file(path, bytes);
    if (fingerprint) *fingerprint = fnv1a64(bytes);
  });
}

/// BiGRU model logits for `rows` contexts (BiGruModel::predict, models.cpp:98-102).
int pmref_bigru_predict(const char* path, const uint32_t* ctx, int64_t rows, int64_t steps,
                        float* logits) {
  return guard([&] {
    auto m = deserialize_model(read_file(path));
    Tensor lg;
    m->predict(ctx, rows, steps, lg);
    std::memcpy(logits, lg.ptr(), lg.data.size() * 4);
  });
}

/// SPrM pre-pass (pretrain_private, training.cpp:62-83); writes the PMKW bytes.
int pmref_pretrain_private(const uint32_t* tokens, uint64_t m, const char* pub_path, uint32_t k,
                           uint32_t t, uint32_t batch, uint32_t scale, uint64_t seed,
                           uint8_t** out, size_t* out_n) {
  return guard([&] {
    std::unique_ptr<BiGruModel> pub;
    if (pub_path && *pub_path) pub = deserialize_model(read_file(pub_path));
    TrainConfig tc;
    tc.sk = SkParams{uint8_t(k), uint8_t(k)};
    tc.t = t;
    tc.batch = batch;
    tc.scale = scale;
    tc.epochs = 1;
    auto priv = pretrain_private(std::span<const uint32_t>(tokens, m), pub.get(), tc, seed);
    ByteVec v = serialize_model(*priv);
    *out = dup(v);
    *out_n = v.size();
  });
}

/// pretrain_public (training.cpp:43-60) over n corpus files; PMKW bytes.
int pmref_pretrain_public(const uint8_t* const* files, const size_t* lens, size_t n, uint32_t s,
                          uint32_t k, uint32_t t, uint32_t batch, uint32_t scale, uint32_t epochs,
                          uint64_t seed, uint8_t** out, size_t* out_n) {
  return guard([&] {
    std::vector<ByteVec> corpus;
    for (size_t i = 0; i < n; ++i) corpus.emplace_back(files[i], files[i] + lens[i]);
    TrainConfig tc;
    tc.sk = SkParams{uint8_t(s), uint8_t(k)};
    tc.t = t;
    tc.batch = batch;
    tc.scale = scale;
    tc.epochs = epochs;
    auto m = pretrain_public(corpus, tc, seed);
    ByteVec v = serialize_model(*m);
    *out = dup(v);
    *out_n = v.size();
  });
}

/// Replays ChunkWorker::encode (pipeline.cpp:115-137) over one chunk's tokens
/// with the reference's public classes and records every model step's mixed
/// probabilities [steps, bs, vocab] (probs may be null), the payload, and the
/// trainer snapshot after the last step.
int pmref_dump_chunk(const uint32_t* tokens, uint64_t n_tokens, uint32_t flags_bits,
                     const char* pub_path, uint32_t k, uint32_t t, uint32_t bs, uint32_t scale,
                     uint64_t dm_seed, const uint8_t* inbound, size_t inbound_n, float* probs,
                     uint64_t max_steps, uint8_t** payload, size_t* payload_n, uint8_t** snap,
                     size_t* snap_n) {
  return guard([&] {
    const ModelDims dims = ModelDims::make(uint32_t(1) << (2 * k), t, scale);
    const SelectorFlags f = SelectorFlags::from_bits(uint8_t(flags_bits));
    std::unique_ptr<BiGruModel> pub;
    if (f.pub_model) pub = deserialize_model(read_file(pub_path));
    AttentionModel dm(dims, dm_seed);
    OnlineTrainer tr(&dm);
    if (inbound_n) tr.restore(ByteSpan(inbound, inbound_n));
    const QuantizedDistribution uni = uniform_dist(uint32_t(dims.vocab));
    const uint64_t L = n_tokens / bs;
    ByteVec out;
    RangeEncoder enc(out);
    std::vector<uint32_t> ctx(size_t(bs) * t), tg(bs);
    Tensor lu, lm, pr;
    AttentionModel::Tape tape;
    uint64_t ms = 0;
    for (uint64_t j = 0; j < L; ++j) {
      if (j < t) {
        for (uint32_t r = 0; r < bs; ++r) enc.encode(uni, tokens[r * L + j]);
        continue;
      }
      for (uint32_t r = 0; r < bs; ++r)
        for (uint32_t i = 0; i < t; ++i) ctx[size_t(r) * t + i] = tokens[uint64_t(r) * L + (j - t) + i];
      if (f.pub_model) pub->predict(ctx.data(), bs, t, lu);
      dm.forward(ctx.data(), bs, t, tape, lm);
      mix(f, tr.alpha(), f.pub_model ? &lu : nullptr, nullptr, &lm, pr);
      if (probs && ms < max_steps)
        std::memcpy(probs + ms * bs * dims.vocab, pr.ptr(), size_t(bs * dims.vocab) * 4);
      for (uint32_t r = 0; r < bs; ++r) {
        tg[r] = tokens[r * L + j];
        enc.encode(quantize(std::span<const float>(pr.ptr() + int64_t(r) * dims.vocab, size_t(dims.vocab))),
                   tg[r]);
      }
      tr.step(f, pr, tg.data(), f.pub_model ? &lu : nullptr, nullptr, lm, tape);
      ++ms;
    }
    enc.finish();
    ByteVec s = tr.snapshot();
    *payload = dup(out);
    *payload_n = out.size();
    *snap = dup(s);
    *snap_n = s.size();
  });
}

int pmref_encode_chunk_standalone_priv(const uint32_t*, uint64_t, uint32_t, const char*,
                                       const uint8_t*, size_t, uint32_t, uint32_t, uint32_t,
                                       uint32_t, uint64_t, const uint8_t*, size_t, uint8_t**, size_t*);

/// Replays ChunkWorker::encode (pipeline.cpp:115-137, 178-213) over one
/// chunk with the reference's public classes, with either static model
/// (flags bit 0: the public model file, bit 1: the private model from its
/// PMKW bytes), stopping after `stop_at` batch steps (0 = all L). The trainer
/// snapshot is taken after batch step `snap_at` (maybe_snapshot(j + 1),
/// warm-up steps included; 0 = after the last executed step). The payload is
/// returned only for a complete chunk (empty otherwise). Used to replay the
/// SMP chain of large runs (chunk i's inbound = chunk i-1's snapshot at its
/// snapshot step, pipeline.cpp:207-213, 253-294) and to recode sampled chunks
/// from recorded inbound snapshots.
int pmref_replay_chunk(const uint32_t* tokens, uint64_t n_tokens, uint32_t flags_bits,
                       const char* pub_path, const uint8_t* priv_bytes, size_t priv_n, uint32_t k,
                       uint32_t t, uint32_t bs, uint32_t scale, uint64_t dm_seed,
                       const uint8_t* inbound, size_t inbound_n, uint64_t snap_at,
                       uint64_t stop_at, uint8_t** payload, size_t* payload_n, uint8_t** snap,
                       size_t* snap_n) {
  return guard([&] {
    const ModelDims dims = ModelDims::make(uint32_t(1) << (2 * k), t, scale);
    const SelectorFlags f = SelectorFlags::from_bits(uint8_t(flags_bits));
    std::unique_ptr<BiGruModel> pub, priv;
    if (f.pub_model) pub = deserialize_model(read_file(pub_path));
    if (f.priv_model) priv = deserialize_model(ByteSpan(priv_bytes, priv_n));
    AttentionModel dm(dims, dm_seed);
    OnlineTrainer tr(&dm);
    if (inbound_n) tr.restore(ByteSpan(inbound, inbound_n));
    const QuantizedDistribution uni = uniform_dist(uint32_t(dims.vocab));
    const uint64_t L = n_tokens / bs;
    const uint64_t stop = stop_at && stop_at < L ? stop_at : L;
    ByteVec out, s;
    RangeEncoder enc(out);
    std::vector<uint32_t> ctx(size_t(bs) * t), tg(bs);
    Tensor lu, lr, lm, pr;
    AttentionModel::Tape tape;
    for (uint64_t j = 0; j < stop; ++j) {
      if (j < t) {
        for (uint32_t r = 0; r < bs; ++r) enc.encode(uni, tokens[r * L + j]);
      } else {
        for (uint32_t r = 0; r < bs; ++r)
          for (uint32_t i = 0; i < t; ++i) ctx[size_t(r) * t + i] = tokens[uint64_t(r) * L + (j - t) + i];
        if (f.pub_model) pub->predict(ctx.data(), bs, t, lu);
        if (f.priv_model) priv->predict(ctx.data(), bs, t, lr);
        dm.forward(ctx.data(), bs, t, tape, lm);
        mix(f, tr.alpha(), f.pub_model ? &lu : nullptr, f.priv_model ? &lr : nullptr, &lm, pr);
        for (uint32_t r = 0; r < bs; ++r) {
          tg[r] = tokens[r * L + j];
          enc.encode(quantize(std::span<const float>(pr.ptr() + int64_t(r) * dims.vocab, size_t(dims.vocab))),
                     tg[r]);
        }
        tr.step(f, pr, tg.data(), f.pub_model ? &lu : nullptr, f.priv_model ? &lr : nullptr, lm, tape);
      }
      if (snap_at && j + 1 == snap_at) s = tr.snapshot();
    }
    if (!snap_at) s = tr.snapshot();
    if (stop == L) enc.finish();
    else out.clear();
    *payload = dup(out);
    *payload_n = out.size();
    *snap = dup(s);
    *snap_n = s.size();
  });
}

/// The reference's own diagnostic hook (pipeline.cpp:298-301).
int pmref_encode_chunk_standalone(const uint32_t* tokens, uint64_t n_tokens, uint32_t flags_bits,
                                  const char* pub_path, uint32_t k, uint32_t t, uint32_t bs,
                                  uint32_t scale, uint64_t dm_seed, const uint8_t* inbound,
                                  size_t inbound_n, uint8_t** out, size_t* out_n) {
  return pmref_encode_chunk_standalone_priv(tokens, n_tokens, flags_bits, pub_path, nullptr, 0, k, t,
                                            bs, scale, dm_seed, inbound, inbound_n, out, out_n);
}

/// Same, with ChunkCodeSpec::priv given as PMKW bytes (pipeline.hpp:69-78).
int pmref_encode_chunk_standalone_priv(const uint32_t* tokens, uint64_t n_tokens, uint32_t flags_bits,
                                       const char* pub_path, const uint8_t* priv_bytes,
                                       size_t priv_n, uint32_t k, uint32_t t, uint32_t bs,
                                       uint32_t scale, uint64_t dm_seed, const uint8_t* inbound,
                                       size_t inbound_n, uint8_t** out, size_t* out_n) {
  return guard([&] {
    const ModelDims dims = ModelDims::make(uint32_t(1) << (2 * k), t, scale);
    std::unique_ptr<BiGruModel> pub, priv;
    const SelectorFlags f = SelectorFlags::from_bits(uint8_t(flags_bits));
    if (f.pub_model) pub = deserialize_model(read_file(pub_path));
    if (f.priv_model) priv = deserialize_model(ByteSpan(priv_bytes, priv_n));
    ChunkCodeSpec spec;
    spec.flags = f;
    spec.pub = pub.get();
    spec.priv = priv.get();
    spec.dims = dims;
    spec.t = t;
    spec.bs = bs;
    spec.dm_seed = dm_seed;
    spec.inbound = ByteSpan(inbound, inbound_n);
    ByteVec v = encode_chunk_standalone(std::span<const uint32_t>(tokens, n_tokens), spec);
    *out = dup(v);
    *out_n = v.size();
  });
}

} // extern "C"
