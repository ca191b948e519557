// Model geometry, seeded initialisation and the byte formats the engine must
// share with the reference: parameter manifests (core/src/weights.cpp:19-70),
// the OnlineTrainer snapshot = SMP payload (core/src/mixer.cpp:99-114,
// core/src/adam.cpp:45-70) and PMKW model files (core/src/models.cpp:159-198).
// Parameters live on the device as one flat float array per model in
// ParamSet order (Appendix C of SURVEY.md), so the layout below is also the
// device layout.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"

namespace pmklc_b200 {

// ModelDims::make (core/src/models.cpp:20-34)
struct Dims {
  int64_t V = 0, T = 0;            // vocab 4^k, context t
  int64_t se = 0, sh = 0, sb = 0;  // static BiGRU: embed, hidden, bottleneck
  int64_t de = 0, dh = 0, df = 0;  // dynamic model: embed, attention width, ffn
  int64_t heads = 8;
  static Dims make(uint32_t vocab, uint32_t context, uint32_t scale);
};

struct ParamDesc {
  std::string name;
  std::vector<int64_t> shape;
  size_t off = 0, count = 0;
  int64_t fan_in = 0;  // 0: not drawn at init (GRU biases, alpha)
};

// AttentionModel + OnlineTrainer trainables (models.cpp:108-120, mixer.cpp:49-53)
struct DmLayout {
  enum Id { EMB, POS, QW, QB, KW, KB, VW, VB, OW, OB, IW, IB, UW, UB, HW, HB, ALPHA, COUNT };
  Dims d;
  std::vector<ParamDesc> ps;
  size_t total = 0;
  explicit DmLayout(const Dims& dims);
  size_t off(Id i) const { return ps[i].off; }
  std::vector<float> seeded(uint64_t seed) const;  // alpha = 0
};

struct DmState {
  std::vector<float> w, m, v;
  uint64_t step = 0;
  float b1p = 1.0f, b2p = 1.0f;
};
Bytes snapshot_bytes(const DmLayout& L, const DmState& s);
DmState parse_snapshot(const DmLayout& L, const uint8_t* p, size_t n);

// BiGruModel (models.cpp:38-51): emb, gru{l}.{fwd,bwd}.{12 tensors}, bott, out
struct BiGru {
  enum G { WIR, WIZ, WIN, WHR, WHZ, WHN, BIR, BIZ, BIN, BHR, BHZ, BHN, NG };
  Dims d;
  int layers = 0;
  std::vector<ParamDesc> ps;
  std::vector<float> w;
  size_t total = 0;
  static BiGru seeded(const Dims& d, int layers, uint64_t seed);
  static BiGru deserialize(const uint8_t* p, size_t n);  // raises like the reference
  Bytes serialize() const;
  int idx(int l, int dir, int t) const { return 1 + (l * 2 + dir) * NG + t; }
  int bott() const { return 1 + layers * 2 * NG; }  // bott.w, bott.b, out.w, out.b
  bool fits(const Dims& want) const {
    return d.V == want.V && d.T == want.T && d.se == want.se && d.sh == want.sh && d.sb == want.sb;
  }
};

void write_params(Writer& w, const std::vector<ParamDesc>& ps, const float* vals);
void read_params(Reader& r, const std::vector<ParamDesc>& ps, float* vals);
void init_uniform(float* t, size_t n, int64_t fan_in, class Rng& rng);

}  // namespace pmklc_b200
