// PMKL container, byte-compatible with the reference writer/reader
// (core/src/container.cpp:13-149). Host-side: it is O(output)
// and runs once per call.
#pragma once
#include <cstdint>
#include <vector>

#include "common.hpp"

namespace pmklc_b200 {

struct ChunkEntry {
  uint64_t token_start = 0, token_len = 0, payload_offset = 0, payload_len = 0;
  uint32_t trailer_len = 0;
};

struct Container {
  uint8_t flags = 0, s = 3, k = 3;
  uint16_t t = 32;
  uint32_t bs = 320;
  uint16_t smp_per_myriad = 500;
  uint64_t dm_seed = 0, sprm_seed = 0, pub_fingerprint = 0, original_len = 0;
  std::vector<ChunkEntry> chunks;
  Bytes private_model;
  std::vector<uint64_t> exc_pos;
  std::vector<uint8_t> exc_byte;
  std::vector<uint8_t> residual;  // base codes 0..3
  // payload i = [payload_ptr[i], +payload_len); written from these spans
  std::vector<const uint8_t*> payload_ptr;
  std::vector<const uint8_t*> trailer_ptr;
};

constexpr size_t kHeaderSize = 52;
constexpr size_t kChunkEntrySize = 36;

Bytes write_container(const Container& c);
// Parses and validates (checksum first); payload/trailer pointers alias `p`.
Container read_container(const uint8_t* p, size_t n);

}  // namespace pmklc_b200
