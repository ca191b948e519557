// Drop-in replacement for the reference's core/src/pipeline.cpp: every entry
// point of core/include/pmklc/pipeline.hpp (CompressConfig::validate,
// ChunkPlan::snapshot_step, plan_chunks, compress, decompress,
// encode_chunk_standalone) implemented over the B200 C ABI
// (include/pmklc_b200.h, paper_2507_12805_b200/lib/libpmklc_b200.so).
//
// A maintainer builds the reference core with this file in place of
// pipeline.cpp and links the library; every caller (tools/main.cpp:88-167,
// bench.cpp:79,87, tests/acceptance.cpp) stays unchanged. integration/Makefile
// does exactly that for the reference's acceptance gauntlet.
//
// Compiled against the reference headers (-I/root/reference/proj/core/include);
// nothing here re-implements the coding path.
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "pmklc/error.hpp"
#include "pmklc/models.hpp"
#include "pmklc/pipeline.hpp"
#include "pmklc_b200.h"

namespace pmklc {
namespace {

// the CUDA device of this process (one device per process, as the reference
// API has no device argument); PMKLC_DEVICE overrides
int32_t device() {
  const char* e = std::getenv("PMKLC_DEVICE");
  return e ? int32_t(std::atoi(e)) : 0;
}

// 1 + errc in the reference's own enum order (error.hpp:8-43). The library's
// message already reads "<ErrcName>: <what>"; pmklc::error prepends the name
// itself (error.hpp:50-51), so only <what> is passed on.
[[noreturn]] void rethrow(int rc) {
  std::string msg = pmklc_last_error();
  const size_t colon = msg.find(": ");
  if (rc >= 1 && rc <= int(errc::verification_failed) + 1) {
    const std::string name = errc_name(errc(rc - 1));
    if (colon != std::string::npos && msg.compare(0, colon, name) == 0) msg = msg.substr(colon + 2);
    raise(errc(rc - 1), msg);
  }
  throw std::runtime_error(msg);  // 101: a CUDA failure, no reference errc
}

pmklc_cfg to_c(const CompressConfig& cfg) {
  pmklc_cfg c;
  pmklc_cfg_default(&c);
  c.s = cfg.sk.s;
  c.k = cfg.sk.k;
  c.t = cfg.t;
  c.bs = cfg.bs;
  c.workers = cfg.workers;
  c.scale = cfg.scale;
  c.selector_threshold = cfg.selector_threshold;
  c.seed = cfg.seed;
  c.smp_fraction = cfg.smp_fraction;
  c.pub_model_path = cfg.pub_model_path.empty() ? nullptr : cfg.pub_model_path.c_str();
  c.device = device();
  return c;
}

void to_stats(std::vector<pmklc_stats>& s, size_t n, PipelineStats* out) {
  if (out) {
    out->workers.assign(n, {});
    for (size_t i = 0; i < n; ++i) {
      WorkerStats& w = out->workers[i];
      w.tokens = s[i].tokens;
      w.uniform_coded = s[i].uniform_coded;
      w.pub_calls = s[i].pub_calls;
      w.priv_calls = s[i].priv_calls;
      w.dyn_calls = s[i].dyn_calls;
      w.snapshot_recv_hash = s[i].snapshot_recv_hash;
      w.snapshot_sent_hash = s[i].snapshot_sent_hash;
      if (s[i].snapshot_recv_len)
        w.snapshot_recv_bytes.assign(s[i].snapshot_recv_bytes,
                                     s[i].snapshot_recv_bytes + s[i].snapshot_recv_len);
      w.early_loss_bits = s[i].early_loss_bits;
    }
  }
  pmklc_stats_release(s.data(), n);
}

ByteVec take(uint8_t* p, size_t n) {
  ByteVec v(p, p + n);
  pmklc_free(p);
  return v;
}
}  // namespace

void CompressConfig::validate() const {
  const pmklc_cfg c = to_c(*this);
  const int rc = pmklc_cfg_validate(&c);
  if (rc) rethrow(rc);
}

uint64_t ChunkPlan::snapshot_step(size_t chunk) const {
  const uint64_t steps = ranges[chunk].len / bs;
  const uint64_t s = (uint64_t(smp_per_myriad) * steps + 9999) / 10000;
  return s ? s : 1;
}

ChunkPlan plan_chunks(uint64_t token_count, uint32_t workers, uint32_t bs, uint32_t t,
                      uint16_t smp_per_myriad) {
  const size_t cap = std::max<uint32_t>(workers, 1);
  std::vector<uint64_t> st(cap), ln(cap), sn(cap);
  size_t count = 0;
  uint32_t bs_out = 0;
  const int rc = pmklc_plan_chunks(token_count, workers, bs, t, smp_per_myriad, st.data(),
                                   ln.data(), sn.data(), cap, &count, &bs_out);
  if (rc) rethrow(rc);
  ChunkPlan p;
  p.t = t;
  p.smp_per_myriad = smp_per_myriad;
  p.bs = bs_out;
  for (size_t i = 0; i < count; ++i) p.ranges.push_back({st[i], ln[i]});
  return p;
}

ByteVec compress(ByteSpan raw, const CompressConfig& cfg, PipelineStats* stats) {
  const pmklc_cfg c = to_c(cfg);
  size_t cap = 0;
  if (stats) {
    const int rc = pmklc_chunk_count(raw.data(), raw.size(), &c, &cap);
    if (rc) rethrow(rc);
  }
  std::vector<pmklc_stats> st(cap);
  uint8_t* out = nullptr;
  size_t out_n = 0, n_chunks = 0;
  const int rc = pmklc_compress(raw.data(), raw.size(), &c, &out, &out_n,
                                stats ? st.data() : nullptr, cap, &n_chunks, nullptr);
  if (rc) rethrow(rc);
  to_stats(st, std::min(cap, n_chunks), stats);
  return take(out, out_n);
}

ByteVec decompress(ByteSpan bytes, const std::string& pub, uint32_t workers, PipelineStats* stats) {
  size_t cap = 0;
  if (stats && pmklc_container_chunks(bytes.data(), bytes.size(), &cap) != 0) cap = 0;
  std::vector<pmklc_stats> st(cap);
  uint8_t* out = nullptr;
  size_t out_n = 0;
  const int rc = pmklc_decompress(bytes.data(), bytes.size(), pub.empty() ? nullptr : pub.c_str(),
                                  workers, device(), &out, &out_n, stats ? st.data() : nullptr,
                                  cap, nullptr);
  if (rc) rethrow(rc);
  to_stats(st, cap, stats);
  return take(out, out_n);
}

ByteVec encode_chunk_standalone(std::span<const uint32_t> tokens, const ChunkCodeSpec& spec) {
  // the public model goes to the library as a file (its API names the SPuM by
  // path, like CompressConfig::pub_model_path), the private one as PMKW bytes
  std::string pub_path;
  if (spec.flags.pub_model && spec.pub) {
    const ByteVec b = serialize_model(*spec.pub);
    pub_path = (std::filesystem::temp_directory_path() /
                ("pmklc_b200_pub_" + std::to_string(fnv1a64(b)) + ".bin")).string();
    std::ofstream(pub_path, std::ios::binary).write(reinterpret_cast<const char*>(b.data()),
                                                    std::streamsize(b.size()));
  }
  ByteVec priv;
  if (spec.flags.priv_model && spec.priv) priv = serialize_model(*spec.priv);
  uint32_t k = 0;
  while ((uint64_t(1) << (2 * (k + 1))) <= uint64_t(spec.dims.vocab)) ++k;
  const uint64_t len = tokens.size();
  const uint8_t* ib = spec.inbound.data();
  const size_t ib_n = spec.inbound.size();
  uint8_t* pay = nullptr;
  size_t pay_n = 0;
  const uint32_t scale = uint32_t(16 / spec.dims.sp_embed);
  const int rc = pmklc_encode_chunks(tokens.data(), &len, 1, &ib, &ib_n, spec.flags.bits(),
                                     pub_path.empty() ? nullptr : pub_path.c_str(),
                                     priv.empty() ? nullptr : priv.data(), priv.size(), k, spec.t,
                                     spec.bs, scale, spec.dm_seed, device(), &pay, &pay_n);
  if (!pub_path.empty()) std::filesystem::remove(pub_path);
  if (rc) rethrow(rc);
  return take(pay, pay_n);
}

}  // namespace pmklc
