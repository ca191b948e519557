// B200 compress/decompress engine: the drop-in for pmklc::compress /
// pmklc::decompress (core/include/pmklc/pipeline.hpp:12-76). Host C++ keeps
// the reference's control flow (validate, seeds, selector, fallbacks, plan,
// container); every per-token stage runs as sm_100a kernels.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"
#include "models.hpp"

namespace pmklc_b200 {

// CompressConfig (pipeline.hpp:12-25) plus device selection.
struct Config {
  uint32_t s = 3, k = 3, t = 32, bs = 320, workers = 1, scale = 4;
  uint64_t selector_threshold = 500'000'000ull, seed = 42;
  float smp_fraction = 0.05f;
  std::string pub_model_path;
  int device = 0;
  uint32_t max_workers = 256;  // validate()'s cap; the C ABI may raise it
  void validate() const;
};

// WorkerStats (pipeline.hpp:27-35)
struct ChunkStats {
  uint64_t tokens = 0, uniform_coded = 0, pub_calls = 0, priv_calls = 0, dyn_calls = 0;
  uint64_t snapshot_recv_hash = 0, snapshot_sent_hash = 0;
  Bytes snapshot_recv_bytes;  // the inbound SMP snapshot, kept when stats are collected
  double early_loss_bits = 0;
};

// Device-side timing of the last call (CUDA events on the engine stream).
struct Timing {
  double total_ms = 0, h2d_ms = 0, tokenize_ms = 0, warmup_ms = 0, model_ms = 0, d2h_ms = 0;
  uint64_t ticks = 0, kernel_launches = 0, chunks = 0;
  uint64_t h2d_bytes = 0, d2h_bytes = 0;
  // dominant kernel (k_bigru_rec_fused, SPuM layer 1), timed in situ
  double hot_ms = 0, hot_flops_per_unit = 0;
  uint64_t hot_launches = 0, hot_units = 0;
  double sprm_ms = 0;  // SPrM pre-pass (compress, flags & 2)
  uint64_t slots = 0;           // state/tape slots of the chunk engine (chunks in flight)
  uint64_t dev_peak_bytes = 0;  // peak device bytes the call's buffers held
};

struct CallOptions {
  bool want_stats = false;
  std::vector<ChunkStats>* stats = nullptr;
  Timing* timing = nullptr;
  // debug probe: mixed probabilities of chunk `probe_chunk` for its first
  // `probe_steps` model steps, [steps, R, V] floats
  int64_t probe_chunk = -1;
  uint64_t probe_steps = 0;
  std::vector<float>* probe = nullptr;
};

// PMKLC-M: one process per GPU, NCCL communicator between them.
struct Dist {
  void* comm = nullptr;  // ncclComm_t
  int rank = 0, world = 1, device = 0;
};
void nccl_unique_id(uint8_t out[128]);
Dist* dist_create(const uint8_t id[128], int rank, int world, int device);
void dist_destroy(Dist* d);
// Every rank passes the whole input; rank 0 receives the container (others
// return an empty vector). Chunks run on rank c % world (plan_rank).
Bytes compress_dist(const Dist& d, const uint8_t* h_raw, const uint8_t* d_raw, size_t n,
                    const Config& cfg, const CallOptions& opt = {});
// Every rank passes the container; rank 0 receives the decompressed bytes.
Bytes decompress_dist(const Dist& d, const uint8_t* blob, size_t n, const std::string& pub_model_path,
                      const CallOptions& opt = {});
// same, rank 0's output left in device memory (nullptr on other ranks)
uint8_t* decompress_dist_to_device(const Dist& d, const uint8_t* blob, size_t n,
                                   const std::string& pub_model_path, size_t* out_len,
                                   const CallOptions& opt = {});

// chunk count compress() writes for this input (plan_chunks over the token
// count of the canonical stream); host-only
size_t planned_chunks(const uint8_t* raw, size_t n, const Config& cfg);

// host buffers in / out
Bytes compress(const uint8_t* raw, size_t n, const Config& cfg, const CallOptions& opt = {});
Bytes decompress(const uint8_t* blob, size_t n, const std::string& pub_model_path, uint32_t workers,
                 int device, const CallOptions& opt = {});
// raw already resident in device memory (bench "value" path)
Bytes compress_device(const uint8_t* d_raw, size_t n, const Config& cfg, const CallOptions& opt = {});
// decompress to a device buffer of original_len bytes (caller frees with cudaFree)
uint8_t* decompress_to_device(const uint8_t* blob, size_t n, const std::string& pub_model_path,
                              int device, size_t* out_len, const CallOptions& opt = {});

// File to file with bounded host memory: compress streams
// the input file into HBM through a pinned double buffer of `block` bytes
// (read of block i+1 overlapping the copy of block i; 0 = 64 MiB) and writes
// the container; decompress streams the decoded bytes back out the same way.
void compress_file(const std::string& in_path, const std::string& out_path, const Config& cfg,
                   const CallOptions& opt = {}, size_t block = 0);
void decompress_file(const std::string& in_path, const std::string& out_path,
                     const std::string& pub_model_path, int device, const CallOptions& opt = {},
                     size_t block = 0);

// encode_chunk_standalone (pipeline.cpp:298-301), batched: every chunk is
// coded independently from its own inbound snapshot (empty = seeded init).
struct ChunkJob {
  const uint32_t* tokens = nullptr;  // host, bs*L tokens used
  uint64_t n_tokens = 0;
  Bytes inbound;
};
// `priv_model`: PMKW bytes of the private model (flags & 2), as shipped in a
// container (ChunkCodeSpec::priv, pipeline.hpp:69-78).
std::vector<Bytes> encode_chunks(const std::vector<ChunkJob>& jobs, uint8_t flags,
                                 const std::string& pub_model_path, const Bytes& priv_model,
                                 uint32_t k, uint32_t t,
                                 uint32_t bs, uint32_t scale, uint64_t dm_seed, int device,
                                 const CallOptions& opt = {});

// quantize (coder.cpp:28-88) of `rows` probability rows on the device, with
// the same kernel the pipeline uses (test hook for the closed-form quantizer)
std::vector<uint32_t> quantize_rows(const float* probs, uint64_t rows, uint32_t width, int device);

// Stand-alone tokenizer on host buffers of base codes 0..3 (for parity tests)
std::vector<uint32_t> skmer_encode_codes(const uint8_t* codes, uint64_t n, uint32_t s, uint32_t k,
                                         int device);
// Tokenizer on device buffers: packed 2-bit bases -> u32 tokens (bench config 2)
void skmer_encode_packed_device(const uint8_t* d_packed, uint64_t n_bases, uint32_t s, uint32_t k,
                                uint32_t* d_tokens, void* stream);
void skmer_encode_packed_device16(const uint8_t* d_packed, uint64_t n_bases, uint32_t s, uint32_t k,
                                  uint16_t* d_tokens, void* stream);

// pretrain_public (training.cpp:43-60) on the device: the corpus files'
// tokens, a seeded 2-layer BiGRU, train_pass over every set for `epochs`
// passes; returns the PMKW bytes of the trained public model (SPuM)
Bytes pretrain_public(const std::vector<std::pair<const uint8_t*, size_t>>& corpus, uint32_t s,
                      uint32_t k, uint32_t t, uint32_t batch, uint32_t scale, uint32_t epochs,
                      uint64_t seed, int device, double* train_ms = nullptr);

// PMKW bytes of a seeded (untrained) BiGRU predictor (BiGruModel ctor +
// serialize_model, models.cpp:38-51,159-173): the SPuM file the reference
// tests and benchmarks use (acceptance.cpp:58-69). Host-only.
Bytes seeded_bigru_file(uint32_t k, uint32_t t, uint32_t scale, int layers, uint64_t seed);

// Live microbenchmarks for bench.py's roofline: average device time of one
// launch of a hot kernel at the engine's real shapes over `chunks` chunks.
//   "gemm_nt"  : dWk|dbk + dWv|dbv reduction over R*t rows (k_gemm_nt)
//   "gemm_ffn" : ffn.outer forward, relu(pre)[R,F] x W2[F,H] (tiled exact GEMM)
//   "fp32_peak": FMUL+FADD issue-rate kernel (no FMA), flops = 2 per MAC
struct KernelBench { double avg_ms = 0, flops = 0, bytes = 0; };
KernelBench bench_kernel(const std::string& name, int device, uint32_t chunks, uint32_t scale,
                         uint32_t R, uint32_t t, int iters);

}  // namespace pmklc_b200
