// Launch interface of the sm_100a kernels (host-callable launchers).
//
// Batching model: every per-chunk kernel reads a device-resident TickDesc
// (current tick, the chunk ids stepping this tick, the SMP handoffs due now)
// and indexes its chunk's data as base + chunk*stride. One launch therefore
// advances every active data block ("chunk", the unit of PMKLC-M block
// partitioning, pipeline.cpp:32-52) by one coded batch step. Grids are sized
// for the schedule's maximum concurrency and surplus blocks exit, so the
// whole per-tick kernel sequence is a fixed CUDA graph replayed every tick.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace pmklc_b200 {

// ---------------------------------------------------------------- tokenizer
// tokens[j] = sum_i base[j*s+i] << 2(k-1-i)   (skmer.cpp:16-24)
// Input: 2-bit packed bases, base i at bits 2*(i%4) of byte i/4.
void launch_skmer_encode_packed(const uint8_t* packed, uint64_t n_bases, uint32_t s, uint32_t k,
                                uint32_t* tokens, uint64_t m, cudaStream_t st);
// same, u16 tokens (k <= 8; SURVEY config 2's 2-byte token layout)
void launch_skmer_encode_packed16(const uint8_t* packed, uint64_t n_bases, uint32_t s, uint32_t k,
                                  uint16_t* tokens, uint64_t m, cudaStream_t st);
// Input: one byte per base, ASCII "ACGT" (pure input, no exception bytes).
void launch_skmer_encode_ascii(const uint8_t* ascii, uint64_t n_bases, uint32_t s, uint32_t k,
                               uint32_t* tokens, uint64_t m, cudaStream_t st);
// Input: one byte per base, codes 0..3.
void launch_skmer_encode_codes(const uint8_t* codes, uint64_t n_bases, uint32_t s, uint32_t k,
                               uint32_t* tokens, uint64_t m, cudaStream_t st);

// canonicalize (alphabet.cpp:22-35): per-block non-ACGT counts, then compaction.
// block_counts has n_blocks(n) entries; after a host/device exclusive scan
// block_offsets, scatter writes codes (compacted) and exception pos/byte.
uint32_t canon_blocks(uint64_t n);
void launch_canon_count(const uint8_t* raw, uint64_t n, uint32_t* block_counts, cudaStream_t st);
void launch_canon_scatter(const uint8_t* raw, uint64_t n, const uint64_t* block_exc_offsets,
                          uint8_t* codes, uint64_t* exc_pos, uint8_t* exc_byte, cudaStream_t st);
// decode (skmer.cpp:63-83) + restore (alphabet.cpp:37-60) fused: writes the
// original bytes. exc_pos sorted ascending (validated by the container reader).
void launch_detokenize_restore(const uint32_t* tokens, uint64_t m, uint32_t s, uint32_t k,
                               const uint8_t* residual, uint64_t n_res, const uint64_t* exc_pos,
                               const uint8_t* exc_byte, uint64_t n_exc, uint8_t* out,
                               uint64_t out_len, int* err, cudaStream_t st);

// ---------------------------------------------------------------- chunk engine
struct ChunkGeo {      // per-chunk constants, device arrays indexed by chunk id (TickDesc::chunk)
  const uint64_t* start;   // token offset of the chunk
  const uint64_t* L;       // batch steps (substream length)
  const int64_t* offset;   // tick of the chunk's first model step
};

// Per-chunk model state and the per-step tapes live in slots (host
// assign_slots: a chunk holds one from its first model tick until its state
// is no longer needed), so device memory scales with the number of chunks in
// flight, not with the chunk count. Kernels index state / tape arrays by the
// slot (act[i]) and the chunk's geometry, codestream and statistics by the
// chunk id (chunk[i], same position).
struct TickDesc {
  int64_t tick;       // -1 before the first advance
  const int* act;     // slots of the chunks doing a model step at this tick
  const int2* hand;   // (src, dst) slot pairs: state handoffs due before this tick's step
  int n_act, n_hand;
  const int* chunk;   // chunk ids, parallel to act (nullptr where unused)
};
// tick += 1 and point act/chunk/hand at that tick's CSR slices (n = 0 past the end)
void launch_tick_advance(TickDesc* td, const uint32_t* act_ptr, const int* act_all,
                         const int* chunk_all, const uint32_t* hand_ptr, const int2* hand_all,
                         int64_t ticks, cudaStream_t st);

// Exact-order GEMM: C[m][n] = init + sum_{k ascending} A(m,k) * B(k,n).
struct GemmP {
  const float* A; int64_t a_cs, lda;  // A(m,k) = AT ? A[k*lda+m] : A[m*lda+k]
  const float* B; int64_t b_cs, ldb;  // B(k,n) = BT ? B[n*ldb+k] : B[k*ldb+n]
  float* C; int64_t c_cs, ldc;
  const float* bias; int64_t bias_cs;       // init==1
  const float* mask; int64_t mask_cs, ldm;  // epilogue: C = (mask<=0) ? 0 : C   (Ffn::backward)
  int M, N, K;
  int ones_row;  // also compute row M with A(M,k)=1 (the bias grad stored right after W)
  int init;      // 0 zero, 1 bias, 2 accumulate onto C
  int relu_a;    // A(m,k) = A<0 ? 0 : A   (Ffn relu, layers.cpp:538-540)
  // optional batch of `nprob` same-shape problems per chunk (0 or 1 = single):
  // problem q uses A + q*a_ps, B + q*b_ps, C + q*c_ps, bias + q*bias_ps
  int nprob;
  int64_t a_ps, b_ps, c_ps, bias_ps;
};
// returns the number of kernels launched (2 when the bias row is split off)
int launch_gemm(const GemmP& p, bool at, bool bt, const TickDesc* td, int max_active,
                 cudaStream_t st);
// Long-reduction "NT" product for weight gradients over many rows:
// C[m][n] += sum_{k ascending} A[m][k] * B[n][k] (+ row M: sum_k B[n][k]),
// A, B feature-major (contiguous in k). One thread per output; both operand
// rows are staged with 16-byte cp.async into a 3-stage shared ring and read as
// LDS.128, so the only serial cost left is the K-long FADD chain itself.
// Two independent problems (e.g. dWk and dWv) can share one launch.
struct NtP {
  const float* A; const float* B; float* C;
  int64_t a_cs, b_cs, c_cs, lda, ldb, ldc;
  int M, N, K;
  float* cb;  // bias-row output (row M); nullptr: C + M*ldc (bias stored right after W)
};
void launch_gemm_nt(const NtP& p0, const NtP* p1, const TickDesc* td, int max_active,
                    cudaStream_t st);
// up to kNtMaxProb independent problems in one launch (all run concurrently)
constexpr int kNtMaxProb = 12;
void launch_gemm_nt_batch(const NtP* probs, int nprob, const TickDesc* td, int max_active,
                          cudaStream_t st);

struct DmDims { int R, T, E, H, F, V, NH; };

// cross-tick pipeline: next = the tick after cur (act list only), and the
// context tokens of that tick's coded rows
void launch_tick_peek(const TickDesc* cur, TickDesc* next, const uint32_t* act_ptr,
                      const int* act_all, const int* chunk_all, int64_t ticks, cudaStream_t st);
void launch_ctx_gather(const uint32_t* tokens, ChunkGeo geo, uint32_t* ctx, int64_t ctx_cs,
                       DmDims d, const TickDesc* td, int max_active, cudaStream_t st);
// ctx gather (pipeline.cpp:180-182) + Embedding/PositionalEmbedding forward
// xtab (nullable): also the K/V table inputs x(t, v) = emb[v] + pos[t],
// feature-major [E][T*V] per chunk slot
void launch_embed(const uint32_t* tokens, ChunkGeo geo, const float* params,
                  int64_t p_cs, int64_t off_emb, int64_t off_pos, uint32_t* ctx, int64_t ctx_cs,
                  float* xT, int64_t x_cs, float* xl, int64_t xl_cs, DmDims d, const TickDesc* td,
                  int max_active, cudaStream_t st, float* xtab = nullptr, int64_t xtab_cs = 0);
// Deduplicated K/V (bit-exact): the K/V row of coded position
// (r, t) depends only on (t, token), so with ctx set the K/V buffers hold the
// T*V table rows t*V + v (computed from launch_embed's xtab) and the row
// kernels gather row t*V + ctx[r][t]; null: K/V hold all R*T rows.
struct KvTab {
  const uint32_t* ctx = nullptr;
  int64_t ctx_cs = 0;
};
// the row-blocked attention kernels run (and so the K/V table may be used)
bool attn_rows_ok(const DmDims& d);
// Attention forward core: scores, det_softmax, context (layers.cpp:452-470)
void launch_attn_fwd(const float* q, const float* k, const float* v, float* wts, float* cx,
                     int64_t cs_q, int64_t cs_kv, int64_t cs_w, DmDims d, float inv,
                     const TickDesc* td, int max_active, cudaStream_t st, const KvTab& kt = {});
// Attention backward core (layers.cpp:480-512). With fx.dx set it also forms
// dx = dk W_k^T + dv W_v^T for the row's positions (the two projection-input
// gradient GEMMs, same chain) and returns true; false: the caller runs them.
struct AttnDx {
  const float* wk; const float* wv; int64_t w_cs;  // W_k, W_v [E][H] per chunk
  float* dx; int64_t dx_cs;                        // dx [R*T][E] per chunk, or nullptr
  // scratch [slot][2][H][E] (nullable): W_k^T, W_v^T formed once per launch for
  // every row block of the chunk to stage with 16-byte copies
  float* wT = nullptr;
};
bool launch_attn_bwd(const float* q, const float* k, const float* v, const float* wts,
                     const float* dctx, float* dq, float* dk, float* dv, int64_t cs_q,
                     int64_t cs_kv, int64_t cs_w, DmDims d, float inv, const AttnDx& fx,
                     const TickDesc* td, int max_active, cudaStream_t st, const KvTab& kt = {});
// PositionalEmbedding + Embedding backward (layers.cpp:117-125,147-155)
void launch_embed_bwd(const uint32_t* ctx, int64_t ctx_cs, const float* dx, int64_t dx_cs,
                      const float* dxl, int64_t dxl_cs, float* grads, int64_t g_cs,
                      int64_t off_emb, int64_t off_pos, DmDims d, const TickDesc* td, int max_active,
                      cudaStream_t st);

// Embedding::backward alone (no positional / last-position term), any model
void launch_emb_grad(const uint32_t* ctx, int64_t ctx_cs, const float* dx, int64_t dx_cs,
                     float* grads, int64_t g_cs, int64_t off_emb, DmDims d, const TickDesc* td,
                     int max_active, cudaStream_t st);

struct AdamScalars {   // per chunk
  uint64_t step;
  float b1p, b2p, bc1, bc2;
  float pad[2];
};
// Adam over params [0, n) of each active chunk, then zero their grads (adam.cpp:21-43)
void launch_adam(float* w, float* g, float* m, float* v, int64_t p_cs, int64_t n,
                 const AdamScalars* sc, const TickDesc* td, int max_active, cudaStream_t st);
// whole-state copy for Step-wise Model Passing: dst chunk <- src chunk
void launch_state_copy(float* w, float* m, float* v, AdamScalars* sc, int64_t p_cs, int64_t n,
                       const TickDesc* td, int max_pairs, cudaStream_t st);

// mix (mixer.cpp:14-42) + det_softmax + quantize (coder.cpp:28-88), one warp per row;
// also advances the chunk's Adam step scalars (adam.cpp:23-27).
struct MixP {
  const float* lu; const float* lr; const float* lm; int64_t cs_l;
  float* probs; uint32_t* freq; uint32_t* cum; int64_t cs_p, cs_c;
  const float* params; int64_t p_cs; int64_t off_alpha;
  AdamScalars* sc;
  int flags, R, V;
  int* err;
  int probs_given;  // test hook: rows of `probs` are already distributions (no mix/softmax)
};
void launch_mix_quantize(const MixP& p, const TickDesc* td, int max_active, cudaStream_t st);

// Backward-controller step (OnlineTrainer::step, mixer.cpp:57-97), split so
// that only one tiny serial chain remains:
//  * launch_bc_dlm: dlm = (probs - onehot(tgt)) * (1 - alpha) and, per
//    element, the d(alpha) term g*(stat - lm) and per row the CE loss term;
//  * launch_alpha_step: the single sequential d(alpha) accumulator over rows
//    then symbols (mixer.cpp:70-84) read back in order from shared memory,
//    alpha's Adam update, and the early-loss sum.
struct BcP {
  const float* probs; const float* lu; const float* lr; const float* lm; int64_t cs_p;
  const uint32_t* tokens; ChunkGeo geo; const TickDesc* td; int t;
  float* w; float* m; float* v; int64_t p_cs; int64_t off_alpha;
  float* dlm; float* aterm; float* lterm; int64_t cs_l;  // lterm stride per chunk
  const AdamScalars* sc;
  double* warm_loss; const uint64_t* warm_steps;
  int flags, R, V;
};
void launch_bc_dlm(const BcP& p, const TickDesc* td, int max_active, cudaStream_t st);
void launch_alpha_step(const BcP& p, const TickDesc* td, int max_active, cudaStream_t st);

// Range coder (coder.cpp:101-166): one thread per chunk, R symbols per step.
struct CoderState { uint64_t low, range, pos, code; int err; int pad; };
void launch_range_uniform(uint32_t* tokens, ChunkGeo geo, int t, int R, int V, uint8_t* payload,
                          const uint64_t* pay_off, const uint64_t* pay_len, CoderState* cs,
                          int n_chunks, bool decode, cudaStream_t st);
void launch_range_step(uint32_t* tokens, ChunkGeo geo, int t, int R, int V,
                       const uint32_t* freq, const uint32_t* cum, int64_t cs_f, int64_t cs_c,
                       uint8_t* payload, const uint64_t* pay_off, const uint64_t* pay_len,
                       CoderState* cs, const TickDesc* td, int max_active, bool decode,
                       cudaStream_t st);
void launch_range_finish(uint8_t* payload, const uint64_t* pay_off, CoderState* cs, int n_chunks,
                         cudaStream_t st);

// Frozen BiGRU predictor forward (SPuM/SPrM, models.cpp:53-73, layers.cpp:213-260).
// Layer 0's input projections b_i* + emb[tok].W_i* depend on the token only,
// so they are a per-model table xi0 [2 dirs][3 gates][V][Hs] computed once
// on the host in the reference's operation order. Deeper layers' input
// projections run as batched exact GEMMs over all R*t positions; only the
// recurrent part is serial in time (one warp per row and direction).
struct BiGruP {
  const float* w;       // flat PMKW parameter array on device
  const int64_t* offs;  // device: param offsets in BiGru::ps order
  const int64_t* hoffs; // host copy of the same offsets
  const float* xi0;     // device table [2][3][V][Hs]
  int layers, V, T, Es, Hs, B, R;
};
// In-situ timer for the dominant kernel: stamp kernels around its launch
// accumulate %globaltimer nanoseconds and the active chunks it processed, over
// every tick of a call (graph replays included).
struct HotTimer {
  unsigned long long t0, ns, units, launches;
};
void launch_hot_begin(HotTimer* h, cudaStream_t st);
void launch_hot_end(HotTimer* h, const TickDesc* td, cudaStream_t st);
// returns the number of kernels launched; `hot` (nullable) times the fused
// layer >= 1 recurrence
int launch_bigru_predict(const BiGruP& p, const uint32_t* ctx, int64_t ctx_cs, float* work,
                          int64_t work_cs, float* logits, int64_t lg_cs, const TickDesc* td,
                          int max_active, cudaStream_t st, HotTimer* hot = nullptr);
size_t bigru_work_floats(const BiGruP& p);

// SPrM pre-pass (pretrain_private / train_pass, training.cpp:8-83): one-layer
// BiGRU trained with Adam over the whole token stream, bs rows per step.
struct SprmP {
  const float* w;       // flat parameter array (BiGru layout)
  // device param offsets; for a deeper layer l the caller passes offs + 2*l*NG
  // (NG = 12 GRU tensors per direction), so the kernels' gate lookups land on
  // that layer (the embedding entry offs[0] is only read for layer 0)
  const int64_t* offs;
  int R, T, Es, H, V, B;
  // deeper layers of a multi-layer model (pretrain_public, training.cpp:43-60):
  // xproj [2][3][R*T][H]: the gate input projections b_i + x.W_i per (row,
  // position) instead of the per-token table; dout [R][T][2H]: the gradient
  // of the layer's outputs, added into dh at every step (gather_add_step,
  // layers.cpp:279) instead of the final-state gradient only
  const float* xproj = nullptr;
  const float* dout = nullptr;
};
// X (feature-major reduction operand, nullable) and, for the streamed path,
// Xtm [2][T][R][Es] (time-major GRU inputs) and the zeroed step counters cnt [2][T]
void launch_sprm_prep(const uint32_t* tokens, const int64_t* pos, const SprmP& s, uint32_t* ctx,
                      float* X, float* tab, float* Xtm, unsigned* cnt, cudaStream_t st);
// Streamed BPTT + the 12 GRU weight-gradient reductions, concurrent (H == 32,
// sprm_stream_ok): gradients accumulate into g as BPTT produces them. The
// consumer table (output pointers into g) is built once per pre-pass:
// sprm_stream_table fills sprm_stream_table_bytes(s) host bytes to upload.
bool sprm_stream_ok(const SprmP& s);
size_t sprm_stream_table_bytes(const SprmP& s);
void sprm_stream_table(const SprmP& s, float* g, const int64_t* hoffs, void* host_buf);
// (the reductions run on `side`, forked from and joined back into `st` by the caller)
void launch_sprm_bptt_stream(const SprmP& s, const float* tape, const float* dfin, float* Gt,
                             const float* Xtm, unsigned* cnt, const void* d_table, cudaStream_t st,
                             cudaStream_t side);
void launch_sprm_fwd(const SprmP& s, const uint32_t* ctx, const float* tab, float* tape, float* fin,
                     cudaStream_t st);
void launch_sprm_ce(const SprmP& s, const uint32_t* tokens, const int64_t* pos, const float* logits,
                    float* g, cudaStream_t st);
void launch_sprm_tanh_grad(float* dbact, const float* bact, int64_t n, cudaStream_t st);
// BPTT + transpose: G = [5 (an, ar, az, hh, hprev)][2][Hs][R*T] feature-major
void launch_sprm_bptt(const SprmP& s, const float* tape, const float* dfin, float* Gt,
                      cudaStream_t st);
// Gt[g][d][t][r][j] -> G[g][d][j][k] (feature-major, k = (t-1-t')*R + r)
void launch_sprm_transpose(const SprmP& s, const float* Gt, float* G, cudaStream_t st);
// true: launch_sprm_dx reads the time-major Gt (no dependency on the transpose)
bool sprm_dx_time_major(const SprmP& s);
// rank (nullable, time-major path only): store dx row rt at its sorted rank
void launch_sprm_dx(const SprmP& s, const float* G, const float* Gt, float* dx, cudaStream_t st,
                    const uint16_t* rank = nullptr);
// model head forward + CE + head backward, warp per row (one launch): writes
// bact [R][B], g [R][V], dbact [R][B] and dfin [R][2H]
void launch_sprm_head(const SprmP& s, const uint32_t* tokens, const int64_t* pos, const float* fin,
                      const float* w1, const float* b1, const float* w2, const float* b2, float* bact,
                      float* g, float* dbact, float* dfin, cudaStream_t st);
// Embedding::backward of the pre-pass as a stable sort of the step's R*T
// context positions by token (beside the forward) + a per-(token, feature)
// walk after dx; needs V <= 256 and R*T <= 65536 (sprm_sorted_emb_ok)
bool sprm_sorted_emb_ok(const SprmP& s);
// order[k]: k-th position in (token, position) order; offs[V+1]; rank[p]: inverse
void launch_tok_sort(const uint32_t* ctx, int n, int V, uint16_t* order, int* offs, uint16_t* rank,
                     cudaStream_t st);
// walk over dx stored in sorted order (launch_sprm_dx with rank); false if E unsupported
bool launch_emb_walk_sorted(const int* offs, const float* dxs, float* grad, int V, int E, int n,
                            cudaStream_t st);
void launch_emb_walk(const uint16_t* order, const int* offs, const float* dx, float* grad, int V,
                     int E, cudaStream_t st);
// 2-layer BiGRU training (pretrain_public): the layer-1 input x1 [R][T][2H]
// from the layer-0 tape, and its feature-major reduction operand [2][2H][R*T]
void launch_bigru_concat(const float* tape, float* x1, int R, int T, int H, cudaStream_t st);
void launch_bigru_xf(const float* x1, float* Xf, int R, int T, int In, cudaStream_t st);
void launch_tanh_vec(float* x, int64_t n, cudaStream_t st);
void launch_adam_scalars(AdamScalars* sc, cudaStream_t st);
// one model's Adam step + scalar update + pos += by, in one launch (the
// trainers' k_adam_scalars -> k_adam -> k_pos_advance); done: a zeroed counter
void launch_sprm_adam(float* w, float* g, float* m, float* v, int64_t n, AdamScalars* sc, int64_t* pos,
                      int64_t by, unsigned* done, cudaStream_t st);
void launch_pos_advance(int64_t* pos, int64_t by, cudaStream_t st);

}  // namespace pmklc_b200
