// Host-side basics shared by the B200 engine: the reference's error codes
// (core/include/pmklc/error.hpp:8-43, same order so the C ABI's 1+errc return
// codes line up with the reference's), little-endian byte I/O and FNV-1a
// (core/include/pmklc/bytes.hpp:17-100).
#pragma once
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace pmklc_b200 {

enum class errc : int {
  length_mismatch, token_out_of_range, not_overlapping, shape_mismatch, stale_tape,
  context_length_mismatch, checksum_mismatch, architecture_mismatch, missing_logits,
  batch_mismatch, invalid_distribution, stream_exhausted, bad_magic, unsupported_version,
  table_inconsistent, config_invalid, io_error, spum_missing, corrupt_stream, corpus_empty,
  target_too_short, empty_source, zero_time, empty_list, verification_failed,
  // not in the reference enum: device-side failures of this implementation
  cuda_error = 100,
};

const char* errc_name(errc c);

class Error : public std::runtime_error {
 public:
  Error(errc c, const std::string& what)
      : std::runtime_error(std::string(errc_name(c)) + ": " + what), code_(c) {}
  errc code() const noexcept { return code_; }

 private:
  errc code_;
};

[[noreturn]] inline void raise(errc c, const std::string& what) { throw Error(c, what); }

using Bytes = std::vector<uint8_t>;

inline uint64_t fnv1a64(const uint8_t* p, size_t n, uint64_t h = 0xcbf29ce484222325ull) {
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
inline uint64_t fnv1a64(const Bytes& b) { return fnv1a64(b.data(), b.size()); }

class Writer {
 public:
  explicit Writer(Bytes& out) : out_(out) {}
  void u8(uint8_t v) { out_.push_back(v); }
  void le(uint64_t v, int nb) {
    for (int i = 0; i < nb; ++i) out_.push_back(uint8_t(v >> (8 * i)));
  }
  void u16(uint16_t v) { le(v, 2); }
  void u32(uint32_t v) { le(v, 4); }
  void u64(uint64_t v) { le(v, 8); }
  void f32(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    le(u, 4);
  }
  void bytes(const void* p, size_t n) {
    const uint8_t* b = static_cast<const uint8_t*>(p);
    out_.insert(out_.end(), b, b + n);
  }
  void str(const std::string& s) {
    u32(uint32_t(s.size()));
    bytes(s.data(), s.size());
  }
  size_t size() const { return out_.size(); }

 private:
  Bytes& out_;
};

class Reader {
 public:
  Reader(const uint8_t* p, size_t n, errc overrun) : p_(p), n_(n), overrun_(overrun) {}
  const uint8_t* take(size_t n) {
    if (n > n_ - pos_) raise(overrun_, "unexpected end of data");
    const uint8_t* s = p_ + pos_;
    pos_ += n;
    return s;
  }
  uint64_t le(int nb) {
    const uint8_t* s = take(size_t(nb));
    uint64_t v = 0;
    for (int i = 0; i < nb; ++i) v |= uint64_t(s[i]) << (8 * i);
    return v;
  }
  uint8_t u8() { return uint8_t(le(1)); }
  uint16_t u16() { return uint16_t(le(2)); }
  uint32_t u32() { return uint32_t(le(4)); }
  uint64_t u64() { return le(8); }
  float f32() {
    uint32_t u = u32();
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  }
  std::string str() {
    uint32_t n = u32();
    const uint8_t* b = take(n);
    return std::string(reinterpret_cast<const char*>(b), n);
  }
  size_t pos() const { return pos_; }
  size_t remaining() const { return n_ - pos_; }

 private:
  const uint8_t* p_;
  size_t n_, pos_ = 0;
  errc overrun_;
};

Bytes read_file(const std::string& path);

}  // namespace pmklc_b200
