// extern "C" boundary (include/pmklc_b200.h) over the B200 engine.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/pmklc_b200.h"
#include "host/engine.hpp"
#include "host/metrics.hpp"
#include "host/plan.hpp"

namespace pmklc_b200 {
void synth_markov3(uint8_t*, uint64_t, uint64_t);
void synth_uniform(uint8_t*, uint64_t, uint64_t);
void synth_packed_codes(uint8_t*, uint64_t, uint64_t);
void synth_genome(uint8_t*, uint64_t, uint64_t, uint32_t);
void synth_species(uint8_t*, uint64_t, uint64_t, uint64_t);
}  // namespace pmklc_b200

using namespace pmklc_b200;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + int(e.code());
  } catch (const std::bad_alloc&) {
    g_err = "CudaError: host allocation failed";
    return 1 + int(errc::cuda_error);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1 + int(errc::cuda_error);
  }
}

uint8_t* dup(const Bytes& v) {
  uint8_t* p = static_cast<uint8_t*>(std::malloc(v.size() ? v.size() : 1));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), v.size());
  return p;
}

Config to_cfg(const pmklc_cfg* c) {
  Config cfg;
  cfg.s = c->s;
  cfg.k = c->k;
  cfg.t = c->t;
  cfg.bs = c->bs;
  cfg.workers = c->workers;
  cfg.scale = c->scale;
  cfg.selector_threshold = c->selector_threshold;
  cfg.seed = c->seed;
  cfg.smp_fraction = c->smp_fraction;
  if (c->pub_model_path) cfg.pub_model_path = c->pub_model_path;
  cfg.device = c->device;
  cfg.max_workers = c->max_workers ? c->max_workers : 256;
  return cfg;
}

void copy_stats(const std::vector<ChunkStats>& st, pmklc_stats* out, size_t cap) {
  if (!out) return;
  for (size_t i = 0; i < st.size() && i < cap; ++i) {
    const ChunkStats& s = st[i];
    uint8_t* bytes = nullptr;
    if (!s.snapshot_recv_bytes.empty()) bytes = dup(s.snapshot_recv_bytes);
    out[i] = pmklc_stats{s.tokens,    s.uniform_coded,      s.pub_calls,          s.priv_calls,
                         s.dyn_calls, s.snapshot_recv_hash, s.snapshot_sent_hash, bytes,
                         uint64_t(s.snapshot_recv_bytes.size()), s.early_loss_bits};
  }
}

void copy_timing(const Timing& t, pmklc_timing* out) {
  if (!out) return;
  *out = pmklc_timing{t.total_ms,  t.h2d_ms,       t.tokenize_ms,     t.warmup_ms,
                      t.model_ms,  t.d2h_ms,       t.ticks,           t.kernel_launches,
                      t.chunks,    t.h2d_bytes,    t.d2h_bytes,       t.hot_ms,
                      t.hot_launches, t.hot_units, t.hot_flops_per_unit, t.sprm_ms,
                      t.slots,     t.dev_peak_bytes};
}

int do_compress(const uint8_t* h, const uint8_t* d, size_t n, const pmklc_cfg* c, uint8_t** out,
                size_t* out_n, pmklc_stats* stats, size_t cap, size_t* n_chunks, pmklc_timing* tm) {
  return guard([&] {
    if (!c) raise(errc::config_invalid, "null config");
    std::vector<ChunkStats> st;
    Timing t;
    CallOptions opt;
    opt.want_stats = stats != nullptr;
    opt.stats = &st;
    opt.timing = &t;
    Bytes v = h ? compress(h, n, to_cfg(c), opt) : compress_device(d, n, to_cfg(c), opt);
    copy_stats(st, stats, cap);
    if (n_chunks) *n_chunks = st.size();
    copy_timing(t, tm);
    *out = dup(v);
    *out_n = v.size();
  });
}
}  // namespace

extern "C" {

void pmklc_cfg_default(pmklc_cfg* c) {
  *c = pmklc_cfg{3, 3, 32, 320, 1, 4, 500000000ull, 42, 0.05f, nullptr, 0, 0};
}

int pmklc_cfg_validate(const pmklc_cfg* c) {
  return guard([&] {
    if (!c) raise(errc::config_invalid, "null config");
    to_cfg(c).validate();
  });
}

int pmklc_compress(const uint8_t* in, size_t n, const pmklc_cfg* cfg, uint8_t** out, size_t* out_n,
                   pmklc_stats* stats, size_t stats_cap, size_t* n_chunks, pmklc_timing* timing) {
  static const uint8_t empty = 0;
  return do_compress(in ? in : &empty, nullptr, n, cfg, out, out_n, stats, stats_cap, n_chunks,
                     timing);
}

int pmklc_compress_device(const uint8_t* d_in, size_t n, const pmklc_cfg* cfg, uint8_t** out,
                          size_t* out_n, pmklc_stats* stats, size_t stats_cap, size_t* n_chunks,
                          pmklc_timing* timing) {
  return do_compress(nullptr, d_in, n, cfg, out, out_n, stats, stats_cap, n_chunks, timing);
}

int pmklc_decompress(const uint8_t* in, size_t n, const char* pub_model_path, uint32_t workers,
                     int32_t device, uint8_t** out, size_t* out_n, pmklc_stats* stats,
                     size_t stats_cap, pmklc_timing* timing) {
  return guard([&] {
    std::vector<ChunkStats> st;
    Timing t;
    CallOptions opt;
    opt.want_stats = stats != nullptr;
    opt.stats = &st;
    opt.timing = &t;
    Bytes v = decompress(in, n, pub_model_path ? pub_model_path : "", workers, device, opt);
    copy_stats(st, stats, stats_cap);
    copy_timing(t, timing);
    *out = dup(v);
    *out_n = v.size();
  });
}

int pmklc_decompress_to_device(const uint8_t* in, size_t n, const char* pub_model_path,
                               int32_t device, uint8_t** d_out, size_t* out_n,
                               pmklc_timing* timing) {
  return guard([&] {
    Timing t;
    CallOptions opt;
    opt.timing = &t;
    *d_out = decompress_to_device(in, n, pub_model_path ? pub_model_path : "", device, out_n, opt);
    copy_timing(t, timing);
  });
}

int pmklc_compress_file(const char* in_path, const char* out_path, const pmklc_cfg* c,
                        size_t block_bytes, pmklc_timing* timing) {
  return guard([&] {
    if (!c || !in_path || !out_path) raise(errc::config_invalid, "null argument");
    Timing t;
    CallOptions opt;
    opt.timing = &t;
    compress_file(in_path, out_path, to_cfg(c), opt, block_bytes);
    copy_timing(t, timing);
  });
}

int pmklc_decompress_file(const char* in_path, const char* out_path, const char* pub_model_path,
                          int32_t device, size_t block_bytes, pmklc_timing* timing) {
  return guard([&] {
    if (!in_path || !out_path) raise(errc::config_invalid, "null argument");
    Timing t;
    CallOptions opt;
    opt.timing = &t;
    decompress_file(in_path, out_path, pub_model_path ? pub_model_path : "", device, opt, block_bytes);
    copy_timing(t, timing);
  });
}

int pmklc_encode_chunks(const uint32_t* tokens, const uint64_t* chunk_len, size_t n_chunks,
                        const uint8_t* const* inbound, const size_t* inbound_len, uint32_t flags,
                        const char* pub_model_path, const uint8_t* priv_model, size_t priv_len,
                        uint32_t k, uint32_t t, uint32_t bs, uint32_t scale, uint64_t dm_seed,
                        int32_t device, uint8_t** payloads, size_t* payload_lens) {
  return guard([&] {
    const Bytes priv = priv_model && priv_len ? Bytes(priv_model, priv_model + priv_len) : Bytes{};
    std::vector<ChunkJob> jobs(n_chunks);
    uint64_t off = 0;
    for (size_t i = 0; i < n_chunks; ++i) {
      jobs[i].tokens = tokens + off;
      jobs[i].n_tokens = chunk_len[i];
      off += chunk_len[i];
      if (inbound && inbound_len && inbound_len[i])
        jobs[i].inbound.assign(inbound[i], inbound[i] + inbound_len[i]);
    }
    std::vector<Bytes> out = encode_chunks(jobs, uint8_t(flags), pub_model_path ? pub_model_path : "",
                                           priv, k, t, bs, scale, dm_seed, device);
    for (size_t i = 0; i < n_chunks; ++i) {
      payloads[i] = dup(out[i]);
      payload_lens[i] = out[i].size();
    }
  });
}

int pmklc_dump_chunk(const uint32_t* tokens, uint64_t n_tokens, uint32_t flags,
                     const char* pub_model_path, uint32_t k, uint32_t t, uint32_t bs,
                     uint32_t scale, uint64_t dm_seed, const uint8_t* inbound, size_t inbound_n,
                     int32_t device, float* probs, uint64_t max_steps, uint8_t** payload,
                     size_t* payload_n) {
  return guard([&] {
    std::vector<ChunkJob> jobs(1);
    jobs[0].tokens = tokens;
    jobs[0].n_tokens = n_tokens;
    if (inbound_n) jobs[0].inbound.assign(inbound, inbound + inbound_n);
    std::vector<float> pr(size_t(max_steps) * bs * (uint64_t(1) << (2 * k)));
    CallOptions opt;
    opt.probe_chunk = 0;
    opt.probe_steps = max_steps;
    opt.probe = &pr;
    std::vector<Bytes> out = encode_chunks(jobs, uint8_t(flags), pub_model_path ? pub_model_path : "",
                                           Bytes{}, k, t, bs, scale, dm_seed, device, opt);
    if (probs && !pr.empty()) std::memcpy(probs, pr.data(), pr.size() * 4);
    *payload = dup(out[0]);
    *payload_n = out[0].size();
  });
}

int pmklc_quantize(const float* probs, uint64_t rows, uint32_t width, int32_t device,
                   uint32_t* freqs) {
  return guard([&] {
    std::vector<uint32_t> f = quantize_rows(probs, rows, width, device);
    if (!f.empty()) std::memcpy(freqs, f.data(), f.size() * 4);
  });
}

int pmklc_skmer_encode(const uint8_t* codes, uint64_t n, uint32_t s, uint32_t k, int32_t device,
                       uint32_t* tokens, uint64_t* m) {
  return guard([&] {
    std::vector<uint32_t> t = skmer_encode_codes(codes, n, s, k, device);
    *m = t.size();
    if (tokens && !t.empty()) std::memcpy(tokens, t.data(), t.size() * 4);
  });
}

int pmklc_skmer_encode_packed_device(const uint8_t* d_packed, uint64_t n_bases, uint32_t s,
                                     uint32_t k, uint32_t* d_tokens, void* stream) {
  return guard([&] { skmer_encode_packed_device(d_packed, n_bases, s, k, d_tokens, stream); });
}

int pmklc_skmer_encode_packed_device_u16(const uint8_t* d_packed, uint64_t n_bases, uint32_t s,
                                         uint32_t k, uint16_t* d_tokens, void* stream) {
  return guard([&] { skmer_encode_packed_device16(d_packed, n_bases, s, k, d_tokens, stream); });
}

int pmklc_plan_chunks(uint64_t m, uint32_t workers, uint32_t bs, uint32_t t, uint16_t myriad,
                      uint64_t* starts, uint64_t* lens, uint64_t* snaps, size_t cap, size_t* count,
                      uint32_t* bs_out) {
  return guard([&] {
    const Plan p = plan_chunks(m, workers, bs, t, myriad);
    *count = p.len.size();
    *bs_out = p.bs;
    for (size_t i = 0; i < p.len.size() && i < cap; ++i) {
      starts[i] = p.start[i];
      lens[i] = p.len[i];
      snaps[i] = p.snapshot_step(i);
    }
  });
}

int pmklc_schedule(const uint64_t* lens, size_t n, uint32_t bs, uint32_t t, uint16_t myriad,
                   int64_t* offset, int64_t* src, uint64_t* src_steps, uint64_t* model_steps,
                   int64_t* ticks) {
  return guard([&] {
    Plan p;
    p.bs = bs;
    p.t = t;
    p.myriad = myriad;
    uint64_t s = 0;
    for (size_t i = 0; i < n; ++i) {
      p.start.push_back(s);
      p.len.push_back(lens[i]);
      s += lens[i];
    }
    const Schedule sc = make_schedule(p, myriad > 0);
    for (size_t i = 0; i < n; ++i) {
      offset[i] = sc.offset[i];
      src[i] = sc.src[i];
      src_steps[i] = sc.src_steps[i];
      model_steps[i] = sc.M[i];
    }
    *ticks = sc.ticks;
  });
}

int pmklc_schedule_slots(const uint64_t* lens, size_t n, uint32_t bs, uint32_t t, uint16_t myriad,
                         int32_t rank, int32_t world, int32_t* slot, int32_t* n_slots) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) raise(errc::config_invalid, "rank/world");
    Plan p;
    p.bs = bs;
    p.t = t;
    p.myriad = myriad;
    uint64_t s = 0;
    for (size_t i = 0; i < n; ++i) {
      p.start.push_back(s);
      p.len.push_back(lens[i]);
      s += lens[i];
    }
    const Schedule sc = make_schedule(p, myriad > 0);
    Slots sl;
    if (world > 1) {
      const RankPlan rp = plan_rank(sc, rank, world);
      sl = assign_slots(rp.local, &rp.mine);
    } else {
      sl = assign_slots(sc);
    }
    for (size_t i = 0; i < n; ++i) slot[i] = sl.of[i];
    *n_slots = sl.count;
  });
}

int pmklc_pretrain_public(const uint8_t* const* files, const size_t* lens, size_t n_files,
                          uint32_t s, uint32_t k, uint32_t t, uint32_t batch, uint32_t scale,
                          uint32_t epochs, uint64_t seed, int32_t device, uint8_t** out,
                          size_t* out_n, double* train_ms) {
  return guard([&] {
    std::vector<std::pair<const uint8_t*, size_t>> corpus;
    for (size_t i = 0; i < n_files; ++i) corpus.push_back({files[i], lens[i]});
    const Bytes b = pretrain_public(corpus, s, k, t, batch, scale, epochs, seed, device, train_ms);
    *out = dup(b);
    *out_n = b.size();
  });
}

int pmklc_write_bigru(const char* path, uint32_t k, uint32_t t, uint32_t scale, int32_t layers,
                      uint64_t seed, uint64_t* fingerprint) {
  return guard([&] {
    const Bytes b = seeded_bigru_file(k, t, scale, layers, seed);
    std::FILE* f = std::fopen(path, "wb");
    if (!f) raise(errc::io_error, std::string("cannot create ") + path);
    const size_t put = std::fwrite(b.data(), 1, b.size(), f);
    const bool ok = put == b.size() && std::fclose(f) == 0;
    if (!ok) raise(errc::io_error, std::string("short write on ") + path);
    if (fingerprint) *fingerprint = fnv1a64(b);
  });
}

int pmklc_bench_kernel(const char* name, int32_t device, uint32_t chunks, uint32_t scale,
                       uint32_t rows, uint32_t t, int32_t iters, double* avg_ms, double* flops,
                       double* bytes) {
  return guard([&] {
    const KernelBench kb = bench_kernel(name, device, chunks, scale, rows, t, iters);
    *avg_ms = kb.avg_ms;
    if (flops) *flops = kb.flops;
    if (bytes) *bytes = kb.bytes;
  });
}

int pmklc_nccl_id(uint8_t* out128) {
  return guard([&] { nccl_unique_id(out128); });
}

int pmklc_dist_create(const uint8_t* id128, int32_t rank, int32_t world, int32_t device, void** handle) {
  return guard([&] { *handle = dist_create(id128, rank, world, device); });
}

void pmklc_dist_destroy(void* handle) { dist_destroy(static_cast<Dist*>(handle)); }

int pmklc_compress_dist(void* handle, const uint8_t* in, const uint8_t* d_in, size_t n,
                        const pmklc_cfg* cfg, uint8_t** out, size_t* out_n, pmklc_timing* timing) {
  return guard([&] {
    Timing t;
    CallOptions opt;
    opt.timing = &t;
    Bytes v = compress_dist(*static_cast<Dist*>(handle), in, d_in, n, to_cfg(cfg), opt);
    copy_timing(t, timing);
    *out = dup(v);
    *out_n = v.size();
  });
}

int pmklc_decompress_dist(void* handle, const uint8_t* in, size_t n, const char* pub_model_path,
                          uint8_t** out, size_t* out_n, pmklc_timing* timing) {
  return guard([&] {
    Timing t;
    CallOptions opt;
    opt.timing = &t;
    Bytes v = decompress_dist(*static_cast<Dist*>(handle), in, n, pub_model_path ? pub_model_path : "", opt);
    copy_timing(t, timing);
    *out = dup(v);
    *out_n = v.size();
  });
}

int pmklc_decompress_dist_to_device(void* handle, const uint8_t* in, size_t n,
                                    const char* pub_model_path, uint8_t** d_out, size_t* out_n,
                                    pmklc_timing* timing) {
  return guard([&] {
    Timing t;
    CallOptions opt;
    opt.timing = &t;
    *d_out = decompress_dist_to_device(*static_cast<Dist*>(handle), in, n,
                                       pub_model_path ? pub_model_path : "", out_n, opt);
    copy_timing(t, timing);
  });
}

int pmklc_compression_ratio(uint64_t compressed_bytes, uint64_t source_bytes, double* out) {
  return guard([&] { *out = compression_ratio(compressed_bytes, source_bytes); });
}

int pmklc_throughput(uint64_t source_bytes, double ct_s, double dt_s, double* out) {
  return guard([&] { *out = throughput(source_bytes, ct_s, dt_s); });
}

int pmklc_robustness(const double* crs, size_t n, double* out) {
  return guard([&] { *out = robustness(crs, n); });
}

int pmklc_block_ratios(const uint8_t* container, size_t n, double* crs, size_t cap, size_t* count) {
  return guard([&] {
    const std::vector<double> r = block_ratios(container, n);
    *count = r.size();
    for (size_t i = 0; i < r.size() && i < cap; ++i) crs[i] = r[i];
  });
}

int pmklc_run_benchmark(const char* const* paths, size_t n_paths, const pmklc_cfg* cfg,
                        const char* csv_path, int32_t fault_flip_mid, pmklc_dataset_result* rows,
                        pmklc_metrics_report* report) {
  return guard([&] {
    if (!cfg) raise(errc::config_invalid, "null config");
    std::vector<std::string> ps(paths, paths + n_paths);
    std::function<void(Bytes&)> fault;
    if (fault_flip_mid)
      fault = [](Bytes& c) {
        if (!c.empty()) c[c.size() / 2] ^= 0x40;
      };
    const MetricsReport rep = run_benchmark(ps, to_cfg(cfg), csv_path ? csv_path : "", fault);
    for (size_t i = 0; i < rep.rows.size() && i < n_paths; ++i) {
      const DatasetResult& d = rep.rows[i];
      pmklc_dataset_result& o = rows[i];
      std::memset(&o, 0, sizeof o);
      std::snprintf(o.name, sizeof o.name, "%s", d.name.c_str());
      o.source_bytes = d.source_bytes;
      o.compressed_bytes = d.compressed_bytes;
      o.ct_s = d.ct_s;
      o.dt_s = d.dt_s;
      o.cr = d.cr;
      o.thp = d.thp;
      o.verified = d.verified ? 1 : 0;
    }
    if (report)
      *report = pmklc_metrics_report{rep.mean_cr, rep.crp_percent, rep.peak_mem_bytes,
                                     rep.peak_device_bytes};
  });
}

uint64_t pmklc_fnv1a64(const uint8_t* p, size_t n) { return fnv1a64(p, n); }

int pmklc_dist_plan(const uint64_t* lens, size_t n_chunks, uint32_t bs, uint32_t t, uint16_t myriad,
                    int32_t rank, int32_t world, int64_t* op_tick, int32_t* op_src, int32_t* op_dst,
                    int32_t* op_peer, uint8_t* op_send, size_t cap, size_t* n_ops,
                    uint64_t* local_steps) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) raise(errc::config_invalid, "rank/world");
    Plan p;
    p.bs = bs;
    p.t = t;
    p.myriad = myriad;
    uint64_t s = 0;
    for (size_t i = 0; i < n_chunks; ++i) {
      p.start.push_back(s);
      p.len.push_back(lens[i]);
      s += lens[i];
    }
    const RankPlan rp = plan_rank(make_schedule(p, myriad > 0), rank, world);
    *n_ops = rp.ops.size();
    for (size_t i = 0; i < rp.ops.size() && i < cap; ++i) {
      op_tick[i] = rp.ops[i].tick;
      op_src[i] = rp.ops[i].src;
      op_dst[i] = rp.ops[i].dst;
      op_peer[i] = rp.ops[i].peer;
      op_send[i] = rp.ops[i].send ? 1 : 0;
    }
    if (local_steps) *local_steps = rp.local.act.size();
  });
}

void pmklc_stats_release(pmklc_stats* stats, size_t n) {
  if (!stats) return;
  for (size_t i = 0; i < n; ++i) {
    std::free(stats[i].snapshot_recv_bytes);
    stats[i].snapshot_recv_bytes = nullptr;
    stats[i].snapshot_recv_len = 0;
  }
}

int pmklc_chunk_count(const uint8_t* in, size_t n, const pmklc_cfg* c, size_t* count) {
  return guard([&] {
    if (!c) raise(errc::config_invalid, "null config");
    const Config cfg = to_cfg(c);
    cfg.validate();
    *count = planned_chunks(in, n, cfg);
  });
}

int pmklc_container_chunks(const uint8_t* in, size_t n, size_t* count) {
  return guard([&] {
    if (n < 52) raise(errc::length_mismatch, "container shorter than its header");
    *count = size_t(in[48]) | size_t(in[49]) << 8 | size_t(in[50]) << 16 | size_t(in[51]) << 24;
  });
}

void pmklc_free(void* p) { std::free(p); }
void pmklc_device_free(void* d_p) {
  if (d_p) cudaFree(d_p);
}
const char* pmklc_last_error(void) { return g_err.c_str(); }
const char* pmklc_errc_name(int code) { return errc_name(errc(code - 1)); }
const char* pmklc_version(void) { return "pmklc_b200 0.1 (sm_100a, EXACT mode)"; }

void pmklc_synth_markov3(uint8_t* out, uint64_t n, uint64_t seed) { synth_markov3(out, n, seed); }
void pmklc_synth_uniform(uint8_t* out, uint64_t n, uint64_t seed) { synth_uniform(out, n, seed); }
void pmklc_synth_genome(uint8_t* out, uint64_t n, uint64_t seed, uint32_t segments) {
  synth_genome(out, n, seed, segments);
}
void pmklc_synth_species(uint8_t* out, uint64_t n, uint64_t seed, uint64_t block) {
  synth_species(out, n, seed, block);
}
void pmklc_synth_packed_codes(uint8_t* out, uint64_t n_bytes, uint64_t seed) {
  synth_packed_codes(out, n_bytes, seed);
}

}  // extern "C"
