/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * C restatement ("port") of the reference PMKLC compress/decompress path
 * (/root/reference/proj/core). Single-threaded, plain C11, no FMA contraction.
 * Used only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * as the checker. Parity is PINNED: tests/test_oracle.py checks this port
 * against oracle/_ref (the reference compiled from its own sources) and the
 * reference's golden vectors.
 *
 * Entry points mirror oracle/ref_shim.cpp (pmref_*) one for one, so the tests
 * can run the same case through both. Return 0 on success, 1 + errc (reference
 * enum order, core/include/pmklc/error.hpp:8-43) on failure.
 */
#ifndef PMKLC_ORACLE_H
#define PMKLC_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t s, k, t, bs, workers, scale;
  uint64_t threshold, seed;
  float smp;
  const char* pub_path;
} orc_cfg;

typedef struct {
  uint64_t tokens, uniform_coded, pub_calls, priv_calls, dyn_calls;
  uint64_t snapshot_recv_hash, snapshot_sent_hash;
  double early_loss_bits;
} orc_chunk_stats;

const char* orc_last_error(void);
uint64_t orc_fnv1a64(const uint8_t* p, size_t n);
void orc_free(void* p);

int orc_compress(const uint8_t* in, size_t n, const orc_cfg* c, uint8_t** out, size_t* out_n,
                 orc_chunk_stats* stats, size_t stats_cap, size_t* n_chunks);
int orc_decompress(const uint8_t* in, size_t n, const char* pub_path, uint32_t workers,
                   uint8_t** out, size_t* out_n, orc_chunk_stats* stats, size_t stats_cap);
int orc_skmer_encode(const uint8_t* codes, uint64_t n, uint32_t s, uint32_t k, uint32_t workers,
                     uint32_t* tokens, uint64_t* m_out, uint8_t* residual, uint64_t* res_n);
int orc_quantize(const float* p, uint32_t n, uint32_t* freqs);
int orc_uniform_dist(uint32_t n, uint32_t* freqs);
int orc_range_encode(const uint32_t* freqs, uint32_t width, const uint32_t* dist_of,
                     const uint32_t* syms, size_t count, uint8_t** out, size_t* out_n);
int orc_det(int which, const float* x, float* y, size_t n);
int orc_softmax(const float* x, float* y, size_t n);
int orc_bigru_predict(const char* path, const uint32_t* ctx, int64_t rows, int64_t steps,
                      float* logits);
int orc_dump_chunk(const uint32_t* tokens, uint64_t n_tokens, uint32_t flags_bits,
                   const char* pub_path, uint32_t k, uint32_t t, uint32_t bs, uint32_t scale,
                   uint64_t dm_seed, const uint8_t* inbound, size_t inbound_n, float* probs,
                   uint64_t max_steps, uint8_t** payload, size_t* payload_n, uint8_t** snap,
                   size_t* snap_n);
int orc_encode_chunk_snap(const uint32_t* tokens, uint64_t n_tokens, uint32_t flags_bits,
                          const char* pub_path, uint32_t k, uint32_t t, uint32_t bs,
                          uint32_t scale, uint64_t dm_seed, const uint8_t* inbound,
                          size_t inbound_n, uint64_t snap_at, uint8_t** payload,
                          size_t* payload_n, uint8_t** snap, size_t* snap_n);
int orc_pretrain_private(const uint32_t* tokens, uint64_t m, const char* pub_path, uint32_t k,
                         uint32_t t, uint32_t batch, uint32_t scale, uint64_t seed,
                         uint8_t** out, size_t* out_n);

#ifdef __cplusplus
}
#endif
#endif
