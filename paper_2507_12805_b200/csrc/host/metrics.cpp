// Metrics and the benchmark driver: the reference's Eq. 3-5
// (core/src/bench.cpp:15-36), run_benchmark + to_csv (bench.cpp:49-114) and
// a memory sampler (bench.cpp:118-164), over the B200 compress/decompress.
// Host code: measurement around the hot path, not part of it.
#include "metrics.hpp"

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>

#include <cuda_runtime.h>

#include "container.hpp"
#include "engine.hpp"

namespace pmklc_b200 {

// Eq. 3: bits per base (bench.cpp:15-18)
double compression_ratio(uint64_t compressed_bytes, uint64_t source_bytes) {
  if (source_bytes == 0) raise(errc::empty_source, "ratio of an empty source");
  return double(compressed_bytes) / double(source_bytes) * 8.0;
}

// Eq. 4: bytes per second over CT + DT (bench.cpp:20-24)
double throughput(uint64_t source_bytes, double ct_s, double dt_s) {
  const double total = ct_s + dt_s;
  if (!(total > 0.0)) raise(errc::zero_time, "throughput needs a positive duration");
  return double(source_bytes) / total;
}

// Eq. 5: sample coefficient of variation in percent, n-1 (bench.cpp:26-36)
double robustness(const double* crs, size_t n) {
  if (n == 0) raise(errc::empty_list, "robustness of an empty list");
  if (n == 1) return 0.0;
  double mean = 0;
  for (size_t i = 0; i < n; ++i) mean += crs[i];
  mean /= double(n);
  double ss = 0;
  for (size_t i = 0; i < n; ++i) ss += (crs[i] - mean) * (crs[i] - mean);
  return 100.0 * std::sqrt(ss / double(n - 1)) / mean;
}

std::vector<double> block_ratios(const uint8_t* blob, size_t n) {
  const Container c = read_container(blob, n);
  std::vector<double> out;
  out.reserve(c.chunks.size());
  for (const ChunkEntry& e : c.chunks) {
    // bases a chunk's tokens cover: (len - 1) * s + k (skmer.cpp:9-12)
    const uint64_t bases = e.token_len ? (e.token_len - 1) * c.s + c.k : 0;
    if (bases) out.push_back(compression_ratio(e.payload_len + e.trailer_len, bases));
  }
  return out;
}

std::string to_csv(const MetricsReport& r) {
  std::string out =
      "dataset,source_bytes,compressed_bytes,ct_s,dt_s,cr_bits_per_base,thp_bytes_per_s,verified\n";
  char line[512];
  for (const DatasetResult& d : r.rows) {
    std::snprintf(line, sizeof line, "%s,%llu,%llu,%.6f,%.6f,%.6f,%.3f,%s\n", d.name.c_str(),
                  (unsigned long long)d.source_bytes, (unsigned long long)d.compressed_bytes, d.ct_s,
                  d.dt_s, d.cr, d.thp, d.verified ? "true" : "false");
    out += line;
  }
  if (!r.rows.empty()) {
    std::snprintf(line, sizeof line, "AGGREGATE,-,-,-,-,%.6f,%.6f,%llu\n", r.mean_cr,
                  r.crp_percent, (unsigned long long)r.peak_mem_bytes);
    out += line;
  }
  return out;
}

namespace {
uint64_t rss_bytes() {
  std::FILE* f = std::fopen("/proc/self/statm", "r");
  if (!f) return 0;
  unsigned long long pages = 0, resident = 0;
  const int got = std::fscanf(f, "%llu %llu", &pages, &resident);
  std::fclose(f);
  return got == 2 ? uint64_t(resident) * 4096ull : 0;
}
uint64_t device_used(int device) {
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return 0;
  if (cur != device && cudaSetDevice(device) != cudaSuccess) return 0;
  size_t fr = 0, tot = 0;
  const bool ok = cudaMemGetInfo(&fr, &tot) == cudaSuccess;
  if (cur != device) cudaSetDevice(cur);
  return ok ? uint64_t(tot - fr) : 0;
}
}  // namespace

// Polls host RSS (as the reference's MemorySampler, bench.cpp:118-164) and the
// device's used HBM every 100 ms on a background thread; stop() returns the
// host peak, device_peak() the HBM peak.
struct MemorySampler::State {
  std::atomic<bool> run{false};
  std::atomic<uint64_t> peak{0}, dpeak{0};
  std::thread th;
  int device = 0;
};

MemorySampler::MemorySampler(int device) : s_(new State) { s_->device = device; }
MemorySampler::~MemorySampler() {
  stop();
  delete s_;
}
void MemorySampler::start() {
  if (s_->run.exchange(true)) return;
  s_->peak = rss_bytes();
  s_->dpeak = device_used(s_->device);
  s_->th = std::thread([st = s_] {
    cudaSetDevice(st->device);
    while (st->run) {
      const uint64_t r = rss_bytes(), d = device_used(st->device);
      uint64_t p = st->peak.load();
      while (r > p && !st->peak.compare_exchange_weak(p, r)) {}
      uint64_t q = st->dpeak.load();
      while (d > q && !st->dpeak.compare_exchange_weak(q, d)) {}
      std::this_thread::sleep_for(std::chrono::milliseconds(100));
    }
  });
}
uint64_t MemorySampler::stop() {
  if (s_->run.exchange(false) && s_->th.joinable()) s_->th.join();
  const uint64_t r = rss_bytes();
  uint64_t p = s_->peak.load();
  return r > p ? r : p;
}
uint64_t MemorySampler::device_peak() const { return s_->dpeak.load(); }

MetricsReport run_benchmark(const std::vector<std::string>& paths, const Config& cfg,
                            const std::string& csv_path, const std::function<void(Bytes&)>& fault) {
  MetricsReport rep;
  MemorySampler sampler(cfg.device);
  sampler.start();
  for (const std::string& path : paths) {
    const Bytes raw = read_file(path);
    DatasetResult row;
    const size_t cut = path.find_last_of('/');
    row.name = cut == std::string::npos ? path : path.substr(cut + 1);
    row.source_bytes = raw.size();
    auto t0 = std::chrono::steady_clock::now();
    Bytes c = compress(raw.data(), raw.size(), cfg);
    row.ct_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    row.compressed_bytes = c.size();
    if (fault) fault(c);
    t0 = std::chrono::steady_clock::now();
    try {
      const Bytes back = decompress(c.data(), c.size(), cfg.pub_model_path, cfg.workers, cfg.device);
      row.dt_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      row.verified = back.size() == raw.size() &&
                     (raw.empty() || std::memcmp(back.data(), raw.data(), raw.size()) == 0);
    } catch (const Error& e) {
      if (e.code() == errc::cuda_error) throw;  // a device failure is not a verification result
      row.dt_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      row.verified = false;
    }
    if (row.source_bytes > 0) row.cr = compression_ratio(row.compressed_bytes, row.source_bytes);
    if (row.ct_s + row.dt_s > 0) row.thp = throughput(row.source_bytes, row.ct_s, row.dt_s);
    rep.rows.push_back(std::move(row));
  }
  rep.peak_mem_bytes = sampler.stop();
  rep.peak_device_bytes = sampler.device_peak();
  std::vector<double> crs;
  for (const DatasetResult& r : rep.rows)
    if (r.verified && r.source_bytes > 0) crs.push_back(r.cr);
  if (!crs.empty()) {
    for (double c : crs) rep.mean_cr += c;
    rep.mean_cr /= double(crs.size());
    rep.crp_percent = robustness(crs.data(), crs.size());
  }
  if (!csv_path.empty()) {
    const std::string csv = to_csv(rep);
    std::FILE* f = std::fopen(csv_path.c_str(), "wb");
    if (!f) raise(errc::io_error, "cannot create " + csv_path);
    const bool ok = std::fwrite(csv.data(), 1, csv.size(), f) == csv.size();
    if (std::fclose(f) != 0 || !ok) raise(errc::io_error, "short write on " + csv_path);
  }
  return rep;
}

}  // namespace pmklc_b200
