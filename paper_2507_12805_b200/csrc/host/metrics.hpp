// Eq. 3-5 metrics and the benchmark driver (core/include/pmklc/bench.hpp:10-59).
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "common.hpp"

namespace pmklc_b200 {

struct Config;

double compression_ratio(uint64_t compressed_bytes, uint64_t source_bytes);  // Eq. 3, bits/base
double throughput(uint64_t source_bytes, double ct_s, double dt_s);          // Eq. 4, bytes/s
double robustness(const double* crs, size_t n);  // Eq. 5, CRP %, n-1 denominator

// per data block (chunk) compression ratios of a container: (payload +
// trailer) bytes x 8 over the bases the chunk's tokens cover -- the CRP
// population for the robustness of one large input
std::vector<double> block_ratios(const uint8_t* blob, size_t n);

struct DatasetResult {
  std::string name;
  uint64_t source_bytes = 0, compressed_bytes = 0;
  double ct_s = 0, dt_s = 0, cr = 0, thp = 0;
  bool verified = false;
};

struct MetricsReport {
  std::vector<DatasetResult> rows;
  double mean_cr = 0, crp_percent = 0;
  uint64_t peak_mem_bytes = 0;     // host RSS peak (as the reference)
  uint64_t peak_device_bytes = 0;  // HBM in use, peak (device-wide)
};

class MemorySampler {
 public:
  explicit MemorySampler(int device = 0);
  ~MemorySampler();
  MemorySampler(const MemorySampler&) = delete;
  MemorySampler& operator=(const MemorySampler&) = delete;
  void start();
  uint64_t stop();  // host RSS peak
  uint64_t device_peak() const;

 private:
  struct State;
  State* s_;
};

std::string to_csv(const MetricsReport& r);
// run_benchmark (bench.cpp:67-114): per file compress, optional fault hook on
// the container, decompress, verify; CSV with an AGGREGATE row when csv_path
// is set
MetricsReport run_benchmark(const std::vector<std::string>& paths, const Config& cfg,
                            const std::string& csv_path,
                            const std::function<void(Bytes&)>& fault = nullptr);

}  // namespace pmklc_b200
