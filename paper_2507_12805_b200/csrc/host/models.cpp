#include "models.hpp"

#include <cmath>
#include <cstdio>

#include "rng.hpp"

namespace pmklc_b200 {

const char* errc_name(errc c) {
  static const char* names[] = {
      "LengthMismatch", "TokenOutOfRange", "NotOverlapping", "ShapeMismatch", "StaleTape",
      "ContextLengthMismatch", "ChecksumMismatch", "ArchitectureMismatch", "MissingLogits",
      "BatchMismatch", "InvalidDistribution", "StreamExhausted", "BadMagic", "UnsupportedVersion",
      "TableInconsistent", "ConfigInvalid", "IoError", "SpumMissing", "CorruptStream",
      "CorpusEmpty", "TargetTooShort", "EmptySource", "ZeroTime", "EmptyList",
      "VerificationFailed"};
  const int i = int(c);
  if (c == errc::cuda_error) return "CudaError";
  return (i >= 0 && i < int(sizeof names / sizeof names[0])) ? names[i] : "UnknownError";
}

Bytes read_file(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) raise(errc::io_error, "cannot open " + path);
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  Bytes out(size_t(n > 0 ? n : 0));
  const size_t got = n > 0 ? std::fread(out.data(), 1, size_t(n), f) : 0;
  std::fclose(f);
  if (n < 0 || got != size_t(n)) raise(errc::io_error, "short read on " + path);
  return out;
}

namespace {
int64_t scaled(int64_t base, uint32_t scale, const char* what) {
  if (scale == 0 || base % int64_t(scale) != 0)
    raise(errc::config_invalid, std::string("scale does not divide ") + what);
  return base / int64_t(scale);
}
void add(std::vector<ParamDesc>& ps, size_t& off, std::string name, std::vector<int64_t> shape,
         int64_t fan) {
  size_t n = 1;
  for (int64_t d : shape) n *= size_t(d);
  ps.push_back(ParamDesc{std::move(name), std::move(shape), off, n, fan});
  off += n;
}
}  // namespace

Dims Dims::make(uint32_t vocab, uint32_t context, uint32_t scale) {
  if (vocab < 2 || context < 1) raise(errc::config_invalid, "model needs vocab >= 2 and context >= 1");
  Dims d;
  d.V = vocab;
  d.T = context;
  d.se = scaled(16, scale, "embedding width");
  d.sh = scaled(128, scale, "recurrent width");
  d.sb = scaled(128, scale, "bottleneck width");
  d.de = scaled(64, scale, "dynamic embedding width");
  d.dh = scaled(256, scale, "attention width");
  d.df = scaled(4096, scale, "feed-forward width");
  d.heads = 8;
  if (d.dh % d.heads != 0) raise(errc::config_invalid, "attention width not divisible by head count");
  return d;
}

void init_uniform(float* t, size_t n, int64_t fan_in, Rng& rng) {
  // layers.cpp:92-95: bound = 1/sqrt(fan_in), v = lo + (hi-lo)*u
  const float bound = 1.0f / std::sqrt(float(fan_in));
  for (size_t i = 0; i < n; ++i) t[i] = rng.next_float(-bound, bound);
}

DmLayout::DmLayout(const Dims& dims) : d(dims) {
  const int64_t V = d.V, T = d.T, E = d.de, H = d.dh, F = d.df;
  size_t o = 0;
  add(ps, o, "emb.table", {V, E}, V);
  add(ps, o, "pos.table", {T, E}, T);
  add(ps, o, "att.q.w", {E, H}, E);
  add(ps, o, "att.q.b", {H}, E);
  add(ps, o, "att.k.w", {E, H}, E);
  add(ps, o, "att.k.b", {H}, E);
  add(ps, o, "att.v.w", {E, H}, E);
  add(ps, o, "att.v.b", {H}, E);
  add(ps, o, "att.o.w", {H, H}, H);
  add(ps, o, "att.o.b", {H}, H);
  add(ps, o, "ffn.inner.w", {H, F}, H);
  add(ps, o, "ffn.inner.b", {F}, H);
  add(ps, o, "ffn.outer.w", {F, H}, F);
  add(ps, o, "ffn.outer.b", {H}, F);
  add(ps, o, "head.w", {H, V}, H);
  add(ps, o, "head.b", {V}, H);
  add(ps, o, "alpha", {1}, 0);
  total = o;
}

std::vector<float> DmLayout::seeded(uint64_t seed) const {
  std::vector<float> w(total, 0.0f);
  Rng rng(seed);
  for (const ParamDesc& p : ps)
    if (p.fan_in) init_uniform(w.data() + p.off, p.count, p.fan_in, rng);
  return w;
}

void write_params(Writer& w, const std::vector<ParamDesc>& ps, const float* vals) {
  w.u32(uint32_t(ps.size()));
  uint64_t off = 0;
  for (const ParamDesc& p : ps) {
    w.str(p.name);
    w.u8(uint8_t(p.shape.size()));
    for (int64_t d : p.shape) w.u64(uint64_t(d));
    w.u64(off);
    off += p.count * 4;
  }
  w.u64(off);
  Bytes blob(static_cast<size_t>(off));
  size_t at = 0;
  for (const ParamDesc& p : ps) {
    std::memcpy(blob.data() + at, vals + p.off, p.count * 4);
    at += p.count * 4;
  }
  w.bytes(blob.data(), blob.size());
  w.u64(fnv1a64(blob));
}

void read_params(Reader& r, const std::vector<ParamDesc>& ps, float* vals) {
  const uint32_t count = r.u32();
  if (count != ps.size()) raise(errc::architecture_mismatch, "parameter count");
  std::vector<uint64_t> offs(count);
  for (uint32_t i = 0; i < count; ++i) {
    const std::string name = r.str();
    if (name != ps[i].name) raise(errc::architecture_mismatch, "parameter name " + name);
    const uint8_t rank = r.u8();
    if (rank != ps[i].shape.size()) raise(errc::architecture_mismatch, "rank of " + name);
    for (uint8_t d = 0; d < rank; ++d)
      if (r.u64() != uint64_t(ps[i].shape[d])) raise(errc::architecture_mismatch, "shape of " + name);
    offs[i] = r.u64();
  }
  const uint64_t bsz = r.u64();
  const uint8_t* blob = r.take(size_t(bsz));
  if (fnv1a64(blob, size_t(bsz)) != r.u64()) raise(errc::checksum_mismatch, "weight blob checksum");
  for (uint32_t i = 0; i < count; ++i) {
    if (offs[i] + ps[i].count * 4 > bsz) raise(errc::architecture_mismatch, "offset of " + ps[i].name);
    std::memcpy(vals + ps[i].off, blob + offs[i], ps[i].count * 4);
  }
}

Bytes snapshot_bytes(const DmLayout& L, const DmState& s) {
  Bytes out;
  out.reserve(L.total * 12 + 4096);
  Writer w(out);
  write_params(w, L.ps, s.w.data());
  w.u64(s.step);
  w.f32(s.b1p);
  w.f32(s.b2p);
  w.u32(uint32_t(L.ps.size()));
  for (const ParamDesc& p : L.ps) {
    w.u64(p.count);
    w.bytes(s.m.data() + p.off, p.count * 4);
    w.bytes(s.v.data() + p.off, p.count * 4);
  }
  return out;
}

DmState parse_snapshot(const DmLayout& L, const uint8_t* p, size_t n) {
  Reader r(p, n, errc::corrupt_stream);
  DmState s;
  s.w.assign(L.total, 0.0f);
  s.m.assign(L.total, 0.0f);
  s.v.assign(L.total, 0.0f);
  read_params(r, L.ps, s.w.data());
  s.step = r.u64();
  s.b1p = r.f32();
  s.b2p = r.f32();
  if (r.u32() != L.ps.size()) raise(errc::shape_mismatch, "optimizer state parameter count");
  for (const ParamDesc& pd : L.ps) {
    if (r.u64() != pd.count) raise(errc::shape_mismatch, "optimizer state tensor size");
    std::memcpy(s.m.data() + pd.off, r.take(pd.count * 4), pd.count * 4);
    std::memcpy(s.v.data() + pd.off, r.take(pd.count * 4), pd.count * 4);
  }
  return s;
}

namespace {
std::vector<ParamDesc> bigru_layout(const Dims& d, int layers, size_t& total) {
  static const char* gn[BiGru::NG] = {"w_ir", "w_iz", "w_in", "w_hr", "w_hz", "w_hn",
                                      "b_ir", "b_iz", "b_in", "b_hr", "b_hz", "b_hn"};
  std::vector<ParamDesc> ps;
  size_t o = 0;
  add(ps, o, "emb.table", {d.V, d.se}, d.V);
  for (int l = 0; l < layers; ++l)
    for (int dir = 0; dir < 2; ++dir) {
      const int64_t in = l == 0 ? d.se : 2 * d.sh;
      const std::string pre = "gru" + std::to_string(l) + (dir ? ".bwd." : ".fwd.");
      for (int t = 0; t < BiGru::NG; ++t) {
        if (t <= BiGru::WIN) add(ps, o, pre + gn[t], {in, d.sh}, in);
        else if (t <= BiGru::WHN) add(ps, o, pre + gn[t], {d.sh, d.sh}, d.sh);
        else add(ps, o, pre + gn[t], {d.sh}, 0);  // GRU biases start at zero
      }
    }
  add(ps, o, "bott.w", {2 * d.sh, d.sb}, 2 * d.sh);
  add(ps, o, "bott.b", {d.sb}, 2 * d.sh);
  add(ps, o, "out.w", {d.sb, d.V}, d.sb);
  add(ps, o, "out.b", {d.V}, d.sb);
  total = o;
  return ps;
}
}  // namespace

BiGru BiGru::seeded(const Dims& d, int layers, uint64_t seed) {
  if (layers < 1) raise(errc::config_invalid, "need at least one recurrent layer");
  BiGru m;
  m.d = d;
  m.layers = layers;
  m.ps = bigru_layout(d, layers, m.total);
  m.w.assign(m.total, 0.0f);
  Rng rng(seed);
  for (const ParamDesc& p : m.ps)
    if (p.fan_in) init_uniform(m.w.data() + p.off, p.count, p.fan_in, rng);
  return m;
}

Bytes BiGru::serialize() const {
  Bytes out;
  Writer w(out);
  w.bytes("PMKW", 4);
  w.u8(1);
  w.u8(uint8_t(layers));
  w.u32(uint32_t(d.V));
  w.u16(uint16_t(d.T));
  w.u64(uint64_t(d.se));
  w.u64(uint64_t(d.sh));
  w.u64(uint64_t(d.sb));
  write_params(w, ps, this->w.data());
  return out;
}

BiGru BiGru::deserialize(const uint8_t* p, size_t n) {
  Reader r(p, n, errc::architecture_mismatch);
  if (std::memcmp(r.take(4), "PMKW", 4) != 0) raise(errc::bad_magic, "model file magic");
  if (r.u8() != 1) raise(errc::unsupported_version, "model file version");
  const int layers = r.u8();
  Dims d;
  d.V = r.u32();
  d.T = r.u16();
  d.se = int64_t(r.u64());
  d.sh = int64_t(r.u64());
  d.sb = int64_t(r.u64());
  d.de = d.dh = d.df = 8;
  if (layers < 1 || d.V < 2 || d.T < 1 || d.se < 1 || d.sh < 1 || d.sb < 1)
    raise(errc::architecture_mismatch, "model header");
  BiGru m;
  m.d = d;
  m.layers = layers;
  m.ps = bigru_layout(d, layers, m.total);
  m.w.assign(m.total, 0.0f);
  read_params(r, m.ps, m.w.data());
  return m;
}

}  // namespace pmklc_b200
