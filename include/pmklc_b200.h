/* pmklc_b200 — C ABI of the B200-native PMKLC compress/decompress hot path.
 *
 * Drop-in boundary for the reference library's entry points
 * (/root/reference/proj/core/include/pmklc/pipeline.hpp):
 *
 *   pmklc_compress            replaces  pmklc::compress(ByteSpan, const CompressConfig&, PipelineStats*)
 *                                       pipeline.hpp:64, pipeline.cpp:303-377
 *   pmklc_decompress          replaces  pmklc::decompress(ByteSpan, const std::string&, uint32_t, PipelineStats*)
 *                                       pipeline.hpp:66-67, pipeline.cpp:379-450
 *   pmklc_encode_chunks       replaces  pmklc::encode_chunk_standalone (batched over chunks)
 *                                       pipeline.hpp:72-76, pipeline.cpp:298-301
 *   pmklc_skmer_encode        replaces  pmklc::encode(const NucleotideStream&, SkParams, unsigned)
 *                                       skmer.hpp:39, skmer.cpp:28-61
 *   pmklc_cfg                 mirrors   pmklc::CompressConfig (pipeline.hpp:12-25), same defaults
 *   pmklc_stats               mirrors   pmklc::WorkerStats (pipeline.hpp:27-35), one per chunk
 *
 * Conventions: plain pointers and sizes only. Return 0 on success, otherwise
 * 1 + errc in the reference enum order (core/include/pmklc/error.hpp:8-43),
 * e.g. 16 = ConfigInvalid, 11 = InvalidDistribution, 7 = ChecksumMismatch;
 * 101 = a CUDA failure (no reference equivalent). pmklc_last_error() returns
 * the thread-local message ("<ErrcName>: <what>", as error::what()). Output
 * buffers are allocated by the library and released with pmklc_free(). There
 * is no CPU fallback: without a usable sm_100 device every compute entry point
 * fails with 101.
 */
#ifndef PMKLC_B200_H
#define PMKLC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pmklc_cfg {
  uint32_t s, k;            /* (s,k)-mer step and window, 1 <= s <= k <= 8      */
  uint32_t t;               /* context length, 1..4096                          */
  uint32_t bs;              /* substreams per chunk                             */
  uint32_t workers;         /* data blocks (chunks), 1..max_workers             */
  uint32_t scale;           /* model width divisor (1 = paper widths)           */
  uint64_t selector_threshold;
  uint64_t seed;
  float smp_fraction;       /* Step-wise Model Passing fraction, [0,1)          */
  const char* pub_model_path; /* SPuM file or NULL                              */
  int32_t device;           /* CUDA device ordinal                              */
  uint32_t max_workers;     /* 0 = reference cap (256, pipeline.cpp:20)         */
} pmklc_cfg;

typedef struct pmklc_stats {
  uint64_t tokens, uniform_coded, pub_calls, priv_calls, dyn_calls;
  uint64_t snapshot_recv_hash, snapshot_sent_hash;
  /* WorkerStats::snapshot_recv_bytes (pipeline.hpp:32, pipeline.cpp:108-111):
   * the chunk's inbound SMP snapshot, library-allocated (NULL when the chunk
   * starts from the seeded init); release with pmklc_stats_release() */
  uint8_t* snapshot_recv_bytes;
  uint64_t snapshot_recv_len;
  double early_loss_bits;
} pmklc_stats;

/* frees the snapshot_recv_bytes of n stats entries (and nulls them) */
void pmklc_stats_release(pmklc_stats* stats, size_t n);

/* number of chunks (data blocks) compress() will write for this input and
 * configuration (plan_chunks over the canonical token count, pipeline.cpp:32-52),
 * so a caller can size the stats array exactly; host-only, O(n) */
int pmklc_chunk_count(const uint8_t* in, size_t n, const pmklc_cfg* cfg, size_t* count);
/* chunk count stored in a container header (container.cpp:53), host-only */
int pmklc_container_chunks(const uint8_t* in, size_t n, size_t* count);

typedef struct pmklc_timing {  /* CUDA-event times of the last call, ms */
  double total_ms, h2d_ms, tokenize_ms, warmup_ms, model_ms, d2h_ms;
  uint64_t ticks, kernel_launches, chunks, h2d_bytes, d2h_bytes;
  /* dominant kernel (SPuM layer-1 fused BiGRU recurrence), timed on the device
   * around every launch of the call: total ms, launches, chunk-launches
   * processed, algorithmic FLOPs per chunk-launch (0 when not run) */
  double hot_ms;
  uint64_t hot_launches, hot_units;
  double hot_flops_per_unit;
  double sprm_ms; /* SPrM pre-pass (training.cpp:8-83) inside compress, ms */
  uint64_t slots;          /* state/tape slots held (peak chunks in flight)   */
  uint64_t dev_peak_bytes; /* peak device bytes of the call's buffers         */
} pmklc_timing;

/* CompressConfig{} defaults: s=k=3, t=32, bs=320, workers=1, threshold 5e8,
 * smp 0.05, seed 42, scale 4, no public model, device 0. */
void pmklc_cfg_default(pmklc_cfg* cfg);
/* CompressConfig::validate (pipeline.cpp:16-24): 0 or 1 + ConfigInvalid */
int pmklc_cfg_validate(const pmklc_cfg* cfg);

/* compress: host input, host container out. stats (nullable) receives one
 * entry per chunk up to stats_cap; n_chunks (nullable) the chunk count. */
int pmklc_compress(const uint8_t* in, size_t n, const pmklc_cfg* cfg, uint8_t** out,
                   size_t* out_n, pmklc_stats* stats, size_t stats_cap, size_t* n_chunks,
                   pmklc_timing* timing);
/* same, input already resident in device memory (16-byte aligned) */
int pmklc_compress_device(const uint8_t* d_in, size_t n, const pmklc_cfg* cfg, uint8_t** out,
                          size_t* out_n, pmklc_stats* stats, size_t stats_cap, size_t* n_chunks,
                          pmklc_timing* timing);

/* decompress: host container in, host bytes out. `workers` is accepted for
 * API parity; it only schedules threads in the reference. */
int pmklc_decompress(const uint8_t* in, size_t n, const char* pub_model_path, uint32_t workers,
                     int32_t device, uint8_t** out, size_t* out_n, pmklc_stats* stats,
                     size_t stats_cap, pmklc_timing* timing);
/* same, output left in device memory (release with pmklc_device_free) */
int pmklc_decompress_to_device(const uint8_t* in, size_t n, const char* pub_model_path,
                               int32_t device, uint8_t** d_out, size_t* out_n,
                               pmklc_timing* timing);

/* file to file with bounded host memory: the input streams
 * from the file into HBM through a pinned double buffer of block_bytes (0 =
 * 64 MiB; the read of one block overlaps the copy of the previous), the
 * container is written to out_path; decompress streams the decoded bytes from
 * HBM to out_path the same way. Same container as pmklc_compress. */
int pmklc_compress_file(const char* in_path, const char* out_path, const pmklc_cfg* cfg,
                        size_t block_bytes, pmklc_timing* timing);
int pmklc_decompress_file(const char* in_path, const char* out_path, const char* pub_model_path,
                          int32_t device, size_t block_bytes, pmklc_timing* timing);

/* encode_chunk_standalone over n_chunks chunks at once: chunk i codes
 * tokens[off_i, off_i + chunk_len[i]) (off_i = prefix sum) from inbound
 * snapshot i (length 0 = seeded init). payloads[i] is library-allocated.
 * ChunkCodeSpec (pipeline.hpp:69-78): flags & 1 loads the public model file,
 * flags & 2 the private model from its PMKW bytes (priv_model, priv_len), as
 * shipped in the container's SPrM blob. */
int pmklc_encode_chunks(const uint32_t* tokens, const uint64_t* chunk_len, size_t n_chunks,
                        const uint8_t* const* inbound, const size_t* inbound_len, uint32_t flags,
                        const char* pub_model_path, const uint8_t* priv_model, size_t priv_len,
                        uint32_t k, uint32_t t, uint32_t bs, uint32_t scale, uint64_t dm_seed,
                        int32_t device, uint8_t** payloads, size_t* payload_lens);

/* one chunk with a probe of its mixed probabilities [max_steps, bs, 4^k]
 * (diagnostic; mirrors oracle/ pmref_dump_chunk) */
int pmklc_dump_chunk(const uint32_t* tokens, uint64_t n_tokens, uint32_t flags,
                     const char* pub_model_path, uint32_t k, uint32_t t, uint32_t bs,
                     uint32_t scale, uint64_t dm_seed, const uint8_t* inbound, size_t inbound_n,
                     int32_t device, float* probs, uint64_t max_steps, uint8_t** payload,
                     size_t* payload_n);

/* quantize (coder.cpp:28-88) of `rows` probability rows of `width` on the
 * device, same kernel as the pipeline; freqs has rows*width entries */
int pmklc_quantize(const float* probs, uint64_t rows, uint32_t width, int32_t device,
                   uint32_t* freqs);

/* (s,k)-mer tokenizer on host base codes 0..3 -> tokens (capacity m) */
int pmklc_skmer_encode(const uint8_t* codes, uint64_t n, uint32_t s, uint32_t k, int32_t device,
                       uint32_t* tokens, uint64_t* m);
/* tokenizer on device buffers: packed 2-bit bases (base i at bits 2*(i%4) of
 * byte i/4, 16-byte aligned) -> u32 tokens; `stream` is a cudaStream_t */
int pmklc_skmer_encode_packed_device(const uint8_t* d_packed, uint64_t n_bases, uint32_t s,
                                     uint32_t k, uint32_t* d_tokens, void* stream);
/* same with u16 tokens (k <= 8): SURVEY config 2's 2-byte layout, half the
 * written bytes; values identical to the u32 tokens (skmer.cpp:16-24) */
int pmklc_skmer_encode_packed_device_u16(const uint8_t* d_packed, uint64_t n_bases, uint32_t s,
                                         uint32_t k, uint16_t* d_tokens, void* stream);

/* host logic of PMKLC-M block partitioning: plan_chunks (pipeline.cpp:32-52)
 * and snapshot_step (pipeline.cpp:26-30); arrays of capacity `cap` */
int pmklc_plan_chunks(uint64_t m, uint32_t workers, uint32_t bs, uint32_t t, uint16_t smp_per_myriad,
                      uint64_t* starts, uint64_t* lens, uint64_t* snapshot_steps, size_t cap,
                      size_t* count, uint32_t* bs_out);
/* Step-wise Model Passing tick schedule for chunks of token length lens[i]
 * (the device realisation of run_chunks, pipeline.cpp:253-294): per chunk the
 * tick of its first model step, the chunk its inbound state comes from (-1 =
 * seeded init), that source's completed model steps, and its own model steps */
int pmklc_schedule(const uint64_t* lens, size_t n_chunks, uint32_t bs, uint32_t t,
                   uint16_t smp_per_myriad, int64_t* offset, int64_t* src, uint64_t* src_steps,
                   uint64_t* model_steps, int64_t* ticks);

/* host logic: the state/tape slot of every chunk (assign_slots: device memory
 * by chunks in flight, not by chunk count) on `rank` of `world` (1 = single
 * GPU); slot[c] = -1 for chunks that never step or live on another rank */
int pmklc_schedule_slots(const uint64_t* lens, size_t n_chunks, uint32_t bs, uint32_t t,
                         uint16_t smp_per_myriad, int32_t rank, int32_t world, int32_t* slot,
                         int32_t* n_slots);

/* ---- PMKLC-M across GPUs (one process per GPU) -------------------------
 * Chunk c runs on rank c % world; an SMP handoff between chunks on different
 * ranks is an NCCL send/recv of the state slot at the handoff tick (replaces
 * the in-process promise chain of run_chunks, pipeline.cpp:253-294). Rank 0
 * obtains the id (pmklc_nccl_id), the caller broadcasts its 128 bytes. */
int pmklc_nccl_id(uint8_t* out128);
int pmklc_dist_create(const uint8_t* id128, int32_t rank, int32_t world, int32_t device,
                      void** handle);
void pmklc_dist_destroy(void* handle);
/* every rank passes the whole input (host `in` or device `d_in`); rank 0
 * receives the container, other ranks an empty buffer */
int pmklc_compress_dist(void* handle, const uint8_t* in, const uint8_t* d_in, size_t n,
                        const pmklc_cfg* cfg, uint8_t** out, size_t* out_n, pmklc_timing* timing);
/* every rank passes the container; rank 0 receives the original bytes */
int pmklc_decompress_dist(void* handle, const uint8_t* in, size_t n, const char* pub_model_path,
                          uint8_t** out, size_t* out_n, pmklc_timing* timing);
/* same, rank 0's output left in device memory (release with pmklc_device_free) */
int pmklc_decompress_dist_to_device(void* handle, const uint8_t* in, size_t n,
                                    const char* pub_model_path, uint8_t** d_out, size_t* out_n,
                                    pmklc_timing* timing);
/* host logic of the above (CPU-testable): this rank's cross-rank handoff ops
 * in tick order (send = 1: this rank sends chunk src's state to `peer`) and
 * the number of (tick, chunk) model steps it runs */
int pmklc_dist_plan(const uint64_t* lens, size_t n_chunks, uint32_t bs, uint32_t t,
                    uint16_t smp_per_myriad, int32_t rank, int32_t world, int64_t* op_tick,
                    int32_t* op_src, int32_t* op_dst, int32_t* op_peer, uint8_t* op_send,
                    size_t cap, size_t* n_ops, uint64_t* local_steps);

/* ---- metrics (reference bench.hpp:10-59, bench.cpp:15-114) ------------ */
/* Eq. 3 compression ratio in bits/base; 1 + EmptySource when source == 0 */
int pmklc_compression_ratio(uint64_t compressed_bytes, uint64_t source_bytes, double* out);
/* Eq. 4 throughput in bytes/s over CT + DT; 1 + ZeroTime when not positive */
int pmklc_throughput(uint64_t source_bytes, double ct_s, double dt_s, double* out);
/* Eq. 5 robustness CRP in percent (n-1 sample deviation / mean); 1 + EmptyList */
int pmklc_robustness(const double* crs, size_t n, double* out);
/* per data block compression ratios of a container (payload + trailer bytes x
 * 8 / the bases each chunk covers), the CRP population of one large input */
int pmklc_block_ratios(const uint8_t* container, size_t n, double* crs, size_t cap,
                       size_t* count);

typedef struct pmklc_dataset_result {  /* DatasetResult (bench.hpp:22-29) */
  char name[256];
  uint64_t source_bytes, compressed_bytes;
  double ct_s, dt_s, cr, thp;
  int32_t verified;
} pmklc_dataset_result;
typedef struct pmklc_metrics_report {  /* MetricsReport (bench.hpp:31-36) */
  double mean_cr, crp_percent;
  uint64_t peak_mem_bytes, peak_device_bytes;
} pmklc_metrics_report;
/* run_benchmark (bench.cpp:67-114) over n_paths files with cfg; rows has
 * capacity n_paths; csv_path (nullable) gets the reference CSV (to_csv,
 * bench.cpp:49-65). fault_flip_mid != 0 flips bit 6 of the container's middle
 * byte before decompression (the reference tests' fault hook). */
int pmklc_run_benchmark(const char* const* paths, size_t n_paths, const pmklc_cfg* cfg,
                        const char* csv_path, int32_t fault_flip_mid, pmklc_dataset_result* rows,
                        pmklc_metrics_report* report);

/* FNV-1a-64 (bytes.hpp:17-24), the fingerprint/checksum hash of the format */
uint64_t pmklc_fnv1a64(const uint8_t* p, size_t n);

/* pretrain_public (training.cpp:43-60; TrainConfig training.hpp:10-17) on the
 * device: n_files corpus files (raw bytes; canonicalized and tokenized like
 * compress), a seeded 2-layer BiGRU trained for `epochs` sequential passes of
 * `batch`-row Adam steps over every file; PMKW bytes of the trained public
 * model (SPuM) in *out (library-allocated). 1 + CorpusEmpty when no file
 * yields a full context window. train_ms (nullable): device time. */
int pmklc_pretrain_public(const uint8_t* const* files, const size_t* lens, size_t n_files,
                          uint32_t s, uint32_t k, uint32_t t, uint32_t batch, uint32_t scale,
                          uint32_t epochs, uint64_t seed, int32_t device, uint8_t** out,
                          size_t* out_n, double* train_ms);

/* seeded (untrained) BiGRU predictor file in the reference's PMKW format
 * (BiGruModel + serialize_model, models.cpp:38-51,159-173); layers = 2 is a
 * SPuM as the reference tests write it (acceptance.cpp:58-69). Host-only. */
int pmklc_write_bigru(const char* path, uint32_t k, uint32_t t, uint32_t scale, int32_t layers,
                      uint64_t seed, uint64_t* fingerprint);

/* live microbenchmark of a hot kernel at the engine's shapes over `chunks`
 * chunks ("gemm_nt", "gemm_ffn", "fp32_peak"): average ms per launch and the
 * algorithmic flops / bytes of one launch (bench.py roofline) */
int pmklc_bench_kernel(const char* name, int32_t device, uint32_t chunks, uint32_t scale,
                       uint32_t rows, uint32_t t, int32_t iters, double* avg_ms, double* flops,
                       double* bytes);

void pmklc_free(void* p);
void pmklc_device_free(void* d_p);
const char* pmklc_last_error(void);
const char* pmklc_errc_name(int code);
const char* pmklc_version(void);

/* synthetic inputs for benchmarks; not on the hot path */
void pmklc_synth_markov3(uint8_t* out, uint64_t n, uint64_t seed);
void pmklc_synth_uniform(uint8_t* out, uint64_t n, uint64_t seed);
void pmklc_synth_genome(uint8_t* out, uint64_t n, uint64_t seed, uint32_t segments);
void pmklc_synth_species(uint8_t* out, uint64_t n, uint64_t seed, uint64_t block);
void pmklc_synth_packed_codes(uint8_t* out, uint64_t n_bytes, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif
