#include "container.hpp"

namespace pmklc_b200 {

Bytes write_container(const Container& c) {
  const size_t W = c.chunks.size();
  uint64_t body = kHeaderSize + W * kChunkEntrySize + 8 + c.private_model.size() + 8 +
                  c.exc_pos.size() * 9 + 8 + (c.residual.size() + 3) / 4;
  uint64_t total = body + 8;
  for (const ChunkEntry& e : c.chunks) total += e.payload_len + e.trailer_len;
  Bytes out;
  out.reserve(size_t(total));
  Writer w(out);
  w.bytes("PMKL", 4);
  w.u8(1);
  w.u8(c.flags);
  w.u8(c.s);
  w.u8(c.k);
  w.u16(c.t);
  w.u32(c.bs);
  w.u16(c.smp_per_myriad);
  w.u64(c.dm_seed);
  w.u64(c.sprm_seed);
  w.u64(c.pub_fingerprint);
  w.u64(c.original_len);
  w.u32(uint32_t(W));
  uint64_t off = body;
  for (const ChunkEntry& e : c.chunks) {
    w.u64(e.token_start);
    w.u64(e.token_len);
    w.u64(off);
    w.u64(e.payload_len);
    w.u32(e.trailer_len);
    off += e.payload_len + e.trailer_len;
  }
  w.u64(c.private_model.size());
  w.bytes(c.private_model.data(), c.private_model.size());
  w.u64(c.exc_pos.size());
  for (size_t i = 0; i < c.exc_pos.size(); ++i) {
    w.u64(c.exc_pos[i]);
    w.u8(c.exc_byte[i]);
  }
  w.u64(c.residual.size());
  uint8_t cur = 0;
  int fill = 0;
  for (uint8_t b : c.residual) {
    cur |= uint8_t((b & 3) << (2 * fill));
    if (++fill == 4) {
      w.u8(cur);
      cur = 0;
      fill = 0;
    }
  }
  if (fill) w.u8(cur);
  for (size_t i = 0; i < W; ++i) {
    w.bytes(c.payload_ptr[i], c.chunks[i].payload_len);
    w.bytes(c.trailer_ptr[i], c.chunks[i].trailer_len);
  }
  w.u64(fnv1a64(out));
  return out;
}

Container read_container(const uint8_t* p, size_t n) {
  if (n < kHeaderSize + 8) raise(errc::table_inconsistent, "container too small");
  {
    Reader tail(p + n - 8, 8, errc::table_inconsistent);
    if (fnv1a64(p, n - 8) != tail.u64()) raise(errc::checksum_mismatch, "container checksum");
  }
  Reader r(p, n, errc::table_inconsistent);
  if (std::memcmp(r.take(4), "PMKL", 4) != 0) raise(errc::bad_magic, "container magic");
  if (r.u8() != 1) raise(errc::unsupported_version, "container version");
  Container c;
  c.flags = r.u8();
  c.s = r.u8();
  c.k = r.u8();
  c.t = r.u16();
  c.bs = r.u32();
  c.smp_per_myriad = r.u16();
  c.dm_seed = r.u64();
  c.sprm_seed = r.u64();
  c.pub_fingerprint = r.u64();
  c.original_len = r.u64();
  const uint32_t W = r.u32();
  if (uint64_t(W) * kChunkEntrySize > n) raise(errc::table_inconsistent, "chunk count exceeds file size");
  c.chunks.resize(W);
  uint64_t next = 0;
  for (ChunkEntry& e : c.chunks) {
    e.token_start = r.u64();
    e.token_len = r.u64();
    e.payload_offset = r.u64();
    e.payload_len = r.u64();
    e.trailer_len = r.u32();
    if (e.token_start != next) raise(errc::table_inconsistent, "chunk token ranges not contiguous");
    next += e.token_len;
  }
  const uint64_t ml = r.u64();
  if (ml > r.remaining()) raise(errc::table_inconsistent, "private model length");
  const uint8_t* m = r.take(size_t(ml));
  c.private_model.assign(m, m + ml);
  const uint64_t ne = r.u64();
  if (ne > r.remaining() / 9) raise(errc::table_inconsistent, "unexpected end of data");
  c.exc_pos.resize(size_t(ne));
  c.exc_byte.resize(size_t(ne));
  for (uint64_t i = 0; i < ne; ++i) {
    c.exc_pos[i] = r.u64();
    c.exc_byte[i] = r.u8();
    if (i > 0 && c.exc_pos[i] <= c.exc_pos[i - 1])
      raise(errc::table_inconsistent, "exception positions not strictly increasing");
  }
  const uint64_t rn = r.u64();
  if ((rn + 3) / 4 > r.remaining()) raise(errc::table_inconsistent, "unexpected end of data");
  const uint8_t* packed = r.take(size_t((rn + 3) / 4));
  c.residual.resize(size_t(rn));
  for (uint64_t i = 0; i < rn; ++i) c.residual[i] = (packed[i / 4] >> (2 * (i % 4))) & 3;
  c.payload_ptr.resize(W);
  c.trailer_ptr.resize(W);
  for (uint32_t i = 0; i < W; ++i) {
    const ChunkEntry& e = c.chunks[i];
    if (e.payload_offset != r.pos()) raise(errc::table_inconsistent, "payload offset");
    if (e.payload_len + e.trailer_len > r.remaining()) raise(errc::table_inconsistent, "payload length");
    c.payload_ptr[i] = r.take(size_t(e.payload_len));
    c.trailer_ptr[i] = r.take(e.trailer_len);
  }
  if (r.remaining() != 8) raise(errc::table_inconsistent, "trailing bytes after payloads");
  return c;
}

}  // namespace pmklc_b200
