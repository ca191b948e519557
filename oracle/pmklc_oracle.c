/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.  See pmklc_oracle.h.
 *
 * A single-threaded C11 restatement of the reference PMKLC path. Every
 * floating-point expression keeps the reference's evaluation order (no FMA:
 * built with -ffp-contract=off like proj/CMakeLists.txt:16-18). Each function
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj/core). Errors unwind with longjmp to the entry point
 * (memory on error paths is not reclaimed; test-only code).
 */
#define _GNU_SOURCE
#include "pmklc_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- errors (error.hpp:8-43 order) ------------------------------------ */
enum {
  E_LENGTH_MISMATCH, E_TOKEN_OUT_OF_RANGE, E_NOT_OVERLAPPING, E_SHAPE_MISMATCH, E_STALE_TAPE,
  E_CONTEXT_LENGTH_MISMATCH, E_CHECKSUM_MISMATCH, E_ARCHITECTURE_MISMATCH, E_MISSING_LOGITS,
  E_BATCH_MISMATCH, E_INVALID_DISTRIBUTION, E_STREAM_EXHAUSTED, E_BAD_MAGIC,
  E_UNSUPPORTED_VERSION, E_TABLE_INCONSISTENT, E_CONFIG_INVALID, E_IO_ERROR, E_SPUM_MISSING,
  E_CORRUPT_STREAM, E_CORPUS_EMPTY, E_TARGET_TOO_SHORT
};
static __thread char g_err[512];
static __thread jmp_buf* g_jmp;
static __thread int g_code;

static void raise_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  g_code = code;
  longjmp(*g_jmp, 1);
}
#define ENTRY                      \
  jmp_buf jb__;                    \
  jmp_buf* prev__ = g_jmp;         \
  g_jmp = &jb__;                   \
  if (setjmp(jb__)) {              \
    g_jmp = prev__;                \
    return 1 + g_code;             \
  }
#define LEAVE                      \
  g_jmp = prev__;                  \
  return 0

const char* orc_last_error(void) { return g_err; }
void orc_free(void* p) { free(p); }

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz ? sz : 1);
  if (!p) raise_err(E_IO_ERROR, "out of memory");
  return p;
}
#define NEWF(n) ((float*)xcalloc((size_t)(n), sizeof(float)))

/* ---- bytes / hashing / rng (bytes.hpp:17-100, rng.hpp:10-35) ------------ */
typedef struct { uint8_t* p; size_t n, cap; } buf_t;
static void b_reserve(buf_t* b, size_t extra) {
  if (b->n + extra <= b->cap) return;
  size_t c = b->cap ? b->cap : 64;
  while (c < b->n + extra) c *= 2;
  b->p = (uint8_t*)realloc(b->p, c);
  b->cap = c;
}
static void b_bytes(buf_t* b, const void* d, size_t n) {
  b_reserve(b, n);
  if (n) memcpy(b->p + b->n, d, n);
  b->n += n;
}
static void b_u8(buf_t* b, uint8_t v) { b_bytes(b, &v, 1); }
static void b_le(buf_t* b, uint64_t v, int nb) {
  for (int i = 0; i < nb; ++i) b_u8(b, (uint8_t)(v >> (8 * i)));
}
static void b_f32(buf_t* b, float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  b_le(b, u, 4);
}

typedef struct { const uint8_t* p; size_t n, pos; int overrun; } rd_t;
static const uint8_t* r_take(rd_t* r, size_t n) {
  if (n > r->n - r->pos) raise_err(r->overrun, "unexpected end of data");
  const uint8_t* s = r->p + r->pos;
  r->pos += n;
  return s;
}
static uint64_t r_le(rd_t* r, int nb) {
  const uint8_t* s = r_take(r, (size_t)nb);
  uint64_t v = 0;
  for (int i = 0; i < nb; ++i) v |= (uint64_t)s[i] << (8 * i);
  return v;
}
static float r_f32(rd_t* r) {
  uint32_t u = (uint32_t)r_le(r, 4);
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static uint64_t fnv1a(const uint8_t* p, size_t n, uint64_t h) {
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
#define FNV_SEED 0xcbf29ce484222325ull
uint64_t orc_fnv1a64(const uint8_t* p, size_t n) { return fnv1a(p, n, FNV_SEED); }

typedef struct { uint64_t s; } rng_t;
static uint64_t rng_u64(rng_t* r) {
  r->s += 0x9e3779b97f4a7c15ull;
  uint64_t z = r->s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static float rng_float(rng_t* r) { return (float)(rng_u64(r) >> 40) * 0x1.0p-24f; }

/* ---- detmath (detmath.cpp:14-103) --------------------------------------- */
static float ldexp_int(float x, int n) {
  uint32_t bits = (uint32_t)(n + 127) << 23;
  float s;
  memcpy(&s, &bits, 4);
  return x * s;
}
static float det_exp(float x) {
  if (x > 87.0f) x = 87.0f;
  if (x < -87.0f) x = -87.0f;
  float t = x * 1.4426950408889634f;
  float nf = floorf(t + 0.5f);
  int n = (int)nf;
  float f = x - nf * 0.693359375f;
  f = f - nf * -2.12194440e-4f;
  float p = 1.0f / 720.0f;
  p = p * f + 1.0f / 120.0f;
  p = p * f + 1.0f / 24.0f;
  p = p * f + 1.0f / 6.0f;
  p = p * f + 0.5f;
  p = p * f + 1.0f;
  p = p * f + 1.0f;
  return ldexp_int(p, n);
}
static float det_log(float x) {
  if (x < 1.17549435e-38f) x = 1.17549435e-38f;
  uint32_t bits;
  memcpy(&bits, &x, 4);
  int e = (int)(bits >> 23) - 127;
  bits = (bits & 0x007fffffu) | 0x3f800000u;
  float m;
  memcpy(&m, &bits, 4);
  if (m > 1.4142135f) {
    m *= 0.5f;
    e += 1;
  }
  float u = (m - 1.0f) / (m + 1.0f);
  float u2 = u * u;
  float p = 1.0f / 11.0f;
  p = p * u2 + 1.0f / 9.0f;
  p = p * u2 + 1.0f / 7.0f;
  p = p * u2 + 1.0f / 5.0f;
  p = p * u2 + 1.0f / 3.0f;
  p = p * u2 + 1.0f;
  return (float)e * 0.69314718f + 2.0f * u * p;
}
static float det_sigmoid(float x) {
  if (x >= 0.0f) return 1.0f / (1.0f + det_exp(-x));
  float e = det_exp(x);
  return e / (1.0f + e);
}
static float det_tanh(float x) {
  float a = x < 0.0f ? -x : x;
  if (a > 9.0f) a = 9.0f;
  float t = 1.0f - 2.0f / (det_exp(2.0f * a) + 1.0f);
  return x < 0.0f ? -t : t;
}
static void det_softmax(float* v, size_t n) {
  if (!n) return;
  float mx = v[0];
  for (size_t i = 1; i < n; ++i)
    if (v[i] > mx) mx = v[i];
  float sum = 0.0f;
  for (size_t i = 0; i < n; ++i) {
    v[i] = det_exp(v[i] - mx);
    sum += v[i];
  }
  float inv = 1.0f / sum;
  for (size_t i = 0; i < n; ++i) v[i] *= inv;
}

/* ---- fixed-order matmuls (tensor.cpp:5-36) ------------------------------ */
/* C[m,n] += A[m,k] B[k,n], each C element ascending in k */
static void mm_acc(const float* a, const float* b, float* c, int64_t m, int64_t k, int64_t n) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t p = 0; p < k; ++p) {
      const float av = a[i * k + p];
      for (int64_t j = 0; j < n; ++j) c[i * n + j] += av * b[p * n + j];
    }
}
/* C[m,n] += A[k,m]^T B[k,n], ascending in k (the row index) */
static void mm_acc_at(const float* a, const float* b, float* c, int64_t m, int64_t k, int64_t n) {
  for (int64_t p = 0; p < k; ++p)
    for (int64_t i = 0; i < m; ++i) {
      const float av = a[p * m + i];
      for (int64_t j = 0; j < n; ++j) c[i * n + j] += av * b[p * n + j];
    }
}
/* C[m,n] += A[m,k] W[n,k]^T  (matmul_acc against transposed(W), layers.cpp:59-65,176-183) */
static void mm_acc_bt(const float* a, const float* w, float* c, int64_t m, int64_t k, int64_t n) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t p = 0; p < k; ++p) {
      const float av = a[i * k + p];
      for (int64_t j = 0; j < n; ++j) c[i * n + j] += av * w[j * k + p];
    }
}
static void linear_fwd(const float* x, const float* w, const float* b, float* out, int64_t rows,
                       int64_t k, int64_t n) {
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < n; ++j) out[i * n + j] = b[j];
  mm_acc(x, w, out, rows, k, n);
}
/* Linear::backward (layers.cpp:176-183): dW += x^T dout; db += colsum; dx += dout W^T */
static void linear_bwd(const float* x, const float* w, float* dw, float* db, const float* dout,
                       float* dx, int64_t rows, int64_t in, int64_t out) {
  mm_acc_at(x, dout, dw, in, rows, out);
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = 0; j < out; ++j) db[j] += dout[r * out + j];
  mm_acc_bt(dout, w, dx, rows, out, in);
}

/* ---- (s,k)-mer tokenizer (skmer.cpp:9-83) -------------------------------- */
static uint64_t token_count(uint64_t n, uint32_t s, uint32_t k) { return n < k ? 0 : (n - k) / s + 1; }

int orc_skmer_encode(const uint8_t* codes, uint64_t n, uint32_t s, uint32_t k, uint32_t workers,
                     uint32_t* tokens, uint64_t* m_out, uint8_t* residual, uint64_t* res_n) {
  (void)workers;
  ENTRY;
  if (!(s >= 1 && s <= k && k <= 8)) raise_err(E_CONFIG_INVALID, "invalid (s,k) parameters");
  const uint64_t m = token_count(n, s, k);
  *m_out = m;
  if (tokens)
    for (uint64_t j = 0; j < m; ++j) {
      uint32_t v = 0;
      for (uint32_t i = 0; i < k; ++i) v = (v << 2) | codes[j * s + i];
      tokens[j] = v;
    }
  const uint64_t covered = m ? (m - 1) * s + k : 0;
  *res_n = n - covered;
  if (residual && n > covered) memcpy(residual, codes + covered, (size_t)(n - covered));
  LEAVE;
}

/* ---- quantizer + range coder (coder.cpp:16-166) ---------------------------- */
#define QTOTAL 65536u
typedef struct { uint32_t n; uint32_t* freqs; uint32_t* cum; } qdist;

static void build_cum(qdist* d) {
  uint32_t a = 0;
  for (uint32_t i = 0; i < d->n; ++i) {
    d->cum[i] = a;
    a += d->freqs[i];
  }
  d->cum[d->n] = a;
}
static const double* g_rem;
static int cmp_desc(const void* x, const void* y) {
  uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  if (g_rem[a] != g_rem[b]) return g_rem[a] > g_rem[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}
static int cmp_asc(const void* x, const void* y) {
  uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  if (g_rem[a] != g_rem[b]) return g_rem[a] < g_rem[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}
/* quantize (coder.cpp:28-88); the comparators are total orders, so qsort
 * matches std::stable_sort exactly. */
static void quantize(const float* p, uint32_t n, qdist* d, double* rem, uint32_t* order) {
  if (n == 0 || n > QTOTAL) raise_err(E_INVALID_DISTRIBUTION, "unsupported width");
  double sum = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    if (!(p[i] > 0.0f)) raise_err(E_INVALID_DISTRIBUTION, "non-positive probability");
    sum += (double)p[i];
  }
  if (fabs(sum - 1.0) > 1e-5) raise_err(E_INVALID_DISTRIBUTION, "probabilities do not sum to 1");
  int64_t assigned = 0;
  for (uint32_t i = 0; i < n; ++i) {
    double v = (double)p[i] * QTOTAL;
    double fl = floor(v);
    uint32_t f = (uint32_t)(fl > 1.0 ? fl : 1.0);
    d->freqs[i] = f;
    rem[i] = v - (double)f;
    assigned += f;
  }
  int64_t deficit = (int64_t)QTOTAL - assigned;
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  g_rem = rem;
  if (deficit > 0) {
    qsort(order, n, sizeof(uint32_t), cmp_desc);
    size_t idx = 0;
    while (deficit > 0) {
      d->freqs[order[idx]] += 1;
      --deficit;
      idx = (idx + 1) % n;
    }
  } else if (deficit < 0) {
    qsort(order, n, sizeof(uint32_t), cmp_asc);
    while (deficit < 0) {
      int removed = 0;
      for (size_t idx = 0; idx < n && deficit < 0; ++idx)
        if (d->freqs[order[idx]] > 1) {
          d->freqs[order[idx]] -= 1;
          ++deficit;
          removed = 1;
        }
      if (!removed) raise_err(E_INVALID_DISTRIBUTION, "cannot settle surplus");
    }
  }
  build_cum(d);
}
static void uniform_dist(uint32_t n, qdist* d) {
  if (n == 0 || n > QTOTAL) raise_err(E_INVALID_DISTRIBUTION, "unsupported width");
  for (uint32_t i = 0; i < n; ++i) d->freqs[i] = QTOTAL / n + (i < QTOTAL % n ? 1 : 0);
  build_cum(d);
}
static qdist qd_new(uint32_t n) {
  qdist d;
  d.n = n;
  d.freqs = (uint32_t*)xcalloc(n, 4);
  d.cum = (uint32_t*)xcalloc(n + 1u, 4);
  return d;
}

#define RENORM (1ull << 56)
typedef struct { buf_t* out; uint64_t low, range; } renc_t;
static void renc_encode(renc_t* e, const qdist* d, uint32_t sym) {
  const uint64_t rb = e->range >> 16;
  const uint64_t old = e->low;
  e->low += rb * d->cum[sym];
  if (e->low < old) { /* propagate_carry (coder.cpp:101-109) */
    size_t i = e->out->n;
    for (;;) {
      e->out->p[i - 1] += 1;
      if (e->out->p[i - 1] != 0) break;
      --i;
    }
  }
  e->range = rb * d->freqs[sym];
  while (e->range < RENORM) {
    b_u8(e->out, (uint8_t)(e->low >> 56));
    e->low <<= 8;
    e->range <<= 8;
  }
}
static void renc_finish(renc_t* e) {
  for (int i = 0; i < 8; ++i) {
    b_u8(e->out, (uint8_t)(e->low >> 56));
    e->low <<= 8;
  }
}
typedef struct { const uint8_t* p; size_t n, pos; uint64_t code, range; } rdec_t;
static uint8_t rdec_byte(rdec_t* d) {
  if (d->pos >= d->n) raise_err(E_STREAM_EXHAUSTED, "codestream truncated");
  return d->p[d->pos++];
}
static void rdec_init(rdec_t* d, const uint8_t* p, size_t n) {
  d->p = p;
  d->n = n;
  d->pos = 0;
  d->code = 0;
  d->range = ~0ull;
  for (int i = 0; i < 8; ++i) d->code = (d->code << 8) | rdec_byte(d);
}
static uint32_t rdec_decode(rdec_t* d, const qdist* q) {
  const uint64_t rb = d->range >> 16;
  uint64_t tgt = d->code / rb;
  if (tgt >= QTOTAL) tgt = QTOTAL - 1;
  uint32_t lo = 0, hi = q->n;
  while (hi - lo > 1) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (q->cum[mid] <= tgt) lo = mid;
    else hi = mid;
  }
  d->code -= rb * q->cum[lo];
  d->range = rb * q->freqs[lo];
  while (d->range < RENORM) {
    d->code = (d->code << 8) | rdec_byte(d);
    d->range <<= 8;
  }
  return lo;
}

/* ---- parameter serialization (weights.cpp:19-70) ------------------------- */
typedef struct { const char* name; int rank; int64_t dims[2]; size_t off, count; } pdesc;

static void write_params(buf_t* b, const pdesc* ps, int np, const float* w) {
  b_le(b, (uint64_t)np, 4);
  uint64_t off = 0;
  for (int i = 0; i < np; ++i) {
    size_t ln = strlen(ps[i].name);
    b_le(b, ln, 4);
    b_bytes(b, ps[i].name, ln);
    b_u8(b, (uint8_t)ps[i].rank);
    for (int d = 0; d < ps[i].rank; ++d) b_le(b, (uint64_t)ps[i].dims[d], 8);
    b_le(b, off, 8);
    off += ps[i].count * 4;
  }
  b_le(b, off, 8);
  size_t at = b->n;
  for (int i = 0; i < np; ++i) b_bytes(b, w + ps[i].off, ps[i].count * 4);
  b_le(b, fnv1a(b->p + at, b->n - at, FNV_SEED), 8);
}
static void read_params(rd_t* r, const pdesc* ps, int np, float* w) {
  if (r_le(r, 4) != (uint64_t)np) raise_err(E_ARCHITECTURE_MISMATCH, "parameter count");
  uint64_t* offs = (uint64_t*)xcalloc((size_t)np, 8);
  for (int i = 0; i < np; ++i) {
    uint32_t ln = (uint32_t)r_le(r, 4);
    const uint8_t* nm = r_take(r, ln);
    if (ln != strlen(ps[i].name) || memcmp(nm, ps[i].name, ln))
      raise_err(E_ARCHITECTURE_MISMATCH, "parameter name");
    if (r_le(r, 1) != (uint64_t)ps[i].rank) raise_err(E_ARCHITECTURE_MISMATCH, "rank");
    for (int d = 0; d < ps[i].rank; ++d)
      if (r_le(r, 8) != (uint64_t)ps[i].dims[d]) raise_err(E_ARCHITECTURE_MISMATCH, "shape");
    offs[i] = r_le(r, 8);
  }
  uint64_t bsz = r_le(r, 8);
  const uint8_t* blob = r_take(r, (size_t)bsz);
  if (fnv1a(blob, (size_t)bsz, FNV_SEED) != r_le(r, 8))
    raise_err(E_CHECKSUM_MISMATCH, "weight blob checksum");
  for (int i = 0; i < np; ++i) {
    if (offs[i] + ps[i].count * 4 > bsz) raise_err(E_ARCHITECTURE_MISMATCH, "offset");
    memcpy(w + ps[i].off, blob + offs[i], ps[i].count * 4);
  }
  free(offs);
}
/* init_uniform (layers.cpp:92-95) */
static void init_uniform(float* t, size_t n, int64_t fan_in, rng_t* rng) {
  const float bound = 1.0f / sqrtf((float)fan_in);
  for (size_t i = 0; i < n; ++i) t[i] = -bound + (bound - -bound) * rng_float(rng);
}

/* ---- Adam (adam.cpp:21-43) ----------------------------------------------- */
typedef struct { uint64_t step; float b1p, b2p; float *m, *v; size_t n; } adam_t;
static const float kLr = 5e-4f, kB1 = 0.9f, kB2 = 0.999f, kEps = 1e-8f;
static void adam_step(adam_t* a, float* w, const float* g) {
  a->step += 1;
  a->b1p *= kB1;
  a->b2p *= kB2;
  const float bc1 = 1.0f - a->b1p, bc2 = 1.0f - a->b2p;
  for (size_t j = 0; j < a->n; ++j) {
    a->m[j] = kB1 * a->m[j] + (1.0f - kB1) * g[j];
    a->v[j] = kB2 * a->v[j] + (1.0f - kB2) * g[j] * g[j];
    const float mhat = a->m[j] / bc1;
    const float vhat = a->v[j] / bc2;
    w[j] -= kLr * mhat / (sqrtf(vhat) + kEps);
  }
}
static void adam_serialize(buf_t* b, const adam_t* a, const pdesc* ps, int np) {
  b_le(b, a->step, 8);
  b_f32(b, a->b1p);
  b_f32(b, a->b2p);
  b_le(b, (uint64_t)np, 4);
  for (int i = 0; i < np; ++i) {
    b_le(b, ps[i].count, 8);
    b_bytes(b, a->m + ps[i].off, ps[i].count * 4);
    b_bytes(b, a->v + ps[i].off, ps[i].count * 4);
  }
}
static void adam_deserialize(rd_t* r, adam_t* a, const pdesc* ps, int np) {
  a->step = r_le(r, 8);
  a->b1p = r_f32(r);
  a->b2p = r_f32(r);
  if (r_le(r, 4) != (uint64_t)np) raise_err(E_SHAPE_MISMATCH, "optimizer state parameter count");
  for (int i = 0; i < np; ++i) {
    if (r_le(r, 8) != ps[i].count) raise_err(E_SHAPE_MISMATCH, "optimizer state tensor size");
    for (size_t j = 0; j < ps[i].count; ++j) a->m[ps[i].off + j] = r_f32(r);
    for (size_t j = 0; j < ps[i].count; ++j) a->v[ps[i].off + j] = r_f32(r);
  }
}

/* ---- model dims (models.cpp:20-34) --------------------------------------- */
typedef struct { int64_t V, T, se, sh, sb, de, dh, df, heads; } dims_t;
static int64_t scaled(int64_t base, uint32_t scale) {
  if (scale == 0 || base % (int64_t)scale) raise_err(E_CONFIG_INVALID, "scale does not divide width");
  return base / scale;
}
static dims_t make_dims(uint32_t vocab, uint32_t ctx, uint32_t scale) {
  if (vocab < 2 || ctx < 1) raise_err(E_CONFIG_INVALID, "model needs vocab >= 2 and context >= 1");
  dims_t d = {vocab, ctx, scaled(16, scale), scaled(128, scale), scaled(128, scale), scaled(64, scale),
              scaled(256, scale), scaled(4096, scale), 8};
  if (d.dh % d.heads) raise_err(E_CONFIG_INVALID, "attention width not divisible by head count");
  return d;
}

/* ---- AttentionModel + OnlineTrainer (models.cpp:108-149, mixer.cpp:44-114) */
enum { P_EMB, P_POS, P_QW, P_QB, P_KW, P_KB, P_VW, P_VB, P_OW, P_OB, P_IW, P_IB, P_UW, P_UB, P_HW,
       P_HB, P_ALPHA, NP_DM };
typedef struct {
  dims_t d;
  pdesc ps[NP_DM];
  size_t n;
  float *w, *g;
  adam_t adam;
  /* tape */
  int64_t R;
  uint32_t* ctx;
  float *x, *k, *v, *q, *wts, *cx, *ao, *pre, *act, *fo, *lm;
} dm_t;

static void set_p(pdesc* p, const char* name, int rank, int64_t a, int64_t b, size_t* off) {
  p->name = name;
  p->rank = rank;
  p->dims[0] = a;
  p->dims[1] = b;
  p->off = *off;
  p->count = (size_t)(rank == 2 ? a * b : a);
  *off += p->count;
}
static void dm_init(dm_t* m, dims_t d, uint64_t seed, int64_t R) {
  memset(m, 0, sizeof *m);
  m->d = d;
  const int64_t V = d.V, T = d.T, E = d.de, H = d.dh, F = d.df;
  size_t off = 0;
  set_p(&m->ps[P_EMB], "emb.table", 2, V, E, &off);
  set_p(&m->ps[P_POS], "pos.table", 2, T, E, &off);
  set_p(&m->ps[P_QW], "att.q.w", 2, E, H, &off);
  set_p(&m->ps[P_QB], "att.q.b", 1, H, 0, &off);
  set_p(&m->ps[P_KW], "att.k.w", 2, E, H, &off);
  set_p(&m->ps[P_KB], "att.k.b", 1, H, 0, &off);
  set_p(&m->ps[P_VW], "att.v.w", 2, E, H, &off);
  set_p(&m->ps[P_VB], "att.v.b", 1, H, 0, &off);
  set_p(&m->ps[P_OW], "att.o.w", 2, H, H, &off);
  set_p(&m->ps[P_OB], "att.o.b", 1, H, 0, &off);
  set_p(&m->ps[P_IW], "ffn.inner.w", 2, H, F, &off);
  set_p(&m->ps[P_IB], "ffn.inner.b", 1, F, 0, &off);
  set_p(&m->ps[P_UW], "ffn.outer.w", 2, F, H, &off);
  set_p(&m->ps[P_UB], "ffn.outer.b", 1, H, 0, &off);
  set_p(&m->ps[P_HW], "head.w", 2, H, V, &off);
  set_p(&m->ps[P_HB], "head.b", 1, V, 0, &off);
  set_p(&m->ps[P_ALPHA], "alpha", 1, 1, 0, &off);
  m->n = off;
  m->w = NEWF(off);
  m->g = NEWF(off);
  m->adam.m = NEWF(off);
  m->adam.v = NEWF(off);
  m->adam.n = off;
  m->adam.b1p = m->adam.b2p = 1.0f;
  /* constructor order = parameter order (models.cpp:112-120) */
  static const int fan_sel[NP_DM - 1] = {0, 1, 2, 2, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 3, 3};
  const int64_t fans[5] = {V, T, E, H, F};
  rng_t rng = {seed};
  for (int i = 0; i < NP_DM - 1; ++i) init_uniform(m->w + m->ps[i].off, m->ps[i].count, fans[fan_sel[i]], &rng);
  m->R = R;
  m->ctx = (uint32_t*)xcalloc((size_t)(R * T), 4);
  m->x = NEWF(R * T * E);
  m->k = NEWF(R * T * H);
  m->v = NEWF(R * T * H);
  m->q = NEWF(R * H);
  m->wts = NEWF(R * d.heads * T);
  m->cx = NEWF(R * H);
  m->ao = NEWF(R * H);
  m->pre = NEWF(R * F);
  m->act = NEWF(R * F);
  m->fo = NEWF(R * H);
  m->lm = NEWF(R * V);
}
static void dm_free(dm_t* m) {
  void* ps[] = {m->w, m->g, m->adam.m, m->adam.v, m->ctx, m->x, m->k, m->v, m->q, m->wts, m->cx, m->ao, m->pre, m->act, m->fo, m->lm};
  for (size_t i = 0; i < sizeof ps / sizeof ps[0]; ++i) free(ps[i]);
}
#define W(m, id) ((m)->w + (m)->ps[id].off)
#define G(m, id) ((m)->g + (m)->ps[id].off)

/* AttentionModel::forward (models.cpp:122-136) -> Embedding (layers.cpp:106-115),
 * PositionalEmbedding (137-145), Attention (432-473), Ffn (534-542), head. */
static void dm_forward(dm_t* m, const uint32_t* ctx) {
  const dims_t d = m->d;
  const int64_t R = m->R, T = d.T, E = d.de, H = d.dh, F = d.df, NH = d.heads, HD = H / NH;
  memcpy(m->ctx, ctx, (size_t)(R * T) * 4);
  for (int64_t r = 0; r < R; ++r)
    for (int64_t t = 0; t < T; ++t) {
      const float* e = W(m, P_EMB) + (int64_t)ctx[r * T + t] * E;
      const float* p = W(m, P_POS) + t * E;
      float* x = m->x + (r * T + t) * E;
      for (int64_t j = 0; j < E; ++j) x[j] = e[j] + p[j];
    }
  linear_fwd(m->x, W(m, P_KW), W(m, P_KB), m->k, R * T, E, H);
  linear_fwd(m->x, W(m, P_VW), W(m, P_VB), m->v, R * T, E, H);
  float* xl = NEWF(R * E);
  for (int64_t r = 0; r < R; ++r) memcpy(xl + r * E, m->x + (r * T + T - 1) * E, (size_t)E * 4);
  linear_fwd(xl, W(m, P_QW), W(m, P_QB), m->q, R, E, H);
  free(xl);
  const float inv = 1.0f / sqrtf((float)HD);
  memset(m->cx, 0, (size_t)(R * H) * 4);
  for (int64_t r = 0; r < R; ++r)
    for (int64_t h = 0; h < NH; ++h) {
      const float* q = m->q + r * H + h * HD;
      float* w = m->wts + (r * NH + h) * T;
      for (int64_t t = 0; t < T; ++t) {
        const float* k = m->k + (r * T + t) * H + h * HD;
        float s = 0.0f;
        for (int64_t dd = 0; dd < HD; ++dd) s += q[dd] * k[dd];
        w[t] = s * inv;
      }
      det_softmax(w, (size_t)T);
      float* c = m->cx + r * H + h * HD;
      for (int64_t t = 0; t < T; ++t) {
        const float* v = m->v + (r * T + t) * H + h * HD;
        for (int64_t dd = 0; dd < HD; ++dd) c[dd] += w[t] * v[dd];
      }
    }
  linear_fwd(m->cx, W(m, P_OW), W(m, P_OB), m->ao, R, H, H);
  linear_fwd(m->ao, W(m, P_IW), W(m, P_IB), m->pre, R, H, F);
  for (int64_t i = 0; i < R * F; ++i) m->act[i] = m->pre[i] < 0.0f ? 0.0f : m->pre[i];
  linear_fwd(m->act, W(m, P_UW), W(m, P_UB), m->fo, R, F, H);
  linear_fwd(m->fo, W(m, P_HW), W(m, P_HB), m->lm, R, H, d.V);
}

/* AttentionModel::backward (models.cpp:138-149) and the layer backwards
 * (layers.cpp:117-125, 147-155, 176-183, 475-522, 544-550). */
static void dm_backward(dm_t* m, const float* dlm) {
  const dims_t d = m->d;
  const int64_t R = m->R, T = d.T, E = d.de, H = d.dh, F = d.df, NH = d.heads, HD = H / NH;
  float* dffn = NEWF(R * H);
  linear_bwd(m->fo, W(m, P_HW), G(m, P_HW), G(m, P_HB), dlm, dffn, R, H, d.V);
  float* dact = NEWF(R * F);
  linear_bwd(m->act, W(m, P_UW), G(m, P_UW), G(m, P_UB), dffn, dact, R, F, H);
  for (int64_t i = 0; i < R * F; ++i)
    if (m->pre[i] <= 0.0f) dact[i] = 0.0f;
  float* datt = NEWF(R * H);
  linear_bwd(m->ao, W(m, P_IW), G(m, P_IW), G(m, P_IB), dact, datt, R, H, F);
  float* dctx = NEWF(R * H);
  linear_bwd(m->cx, W(m, P_OW), G(m, P_OW), G(m, P_OB), datt, dctx, R, H, H);
  float* dq = NEWF(R * H);
  float* dk = NEWF(R * T * H);
  float* dv = NEWF(R * T * H);
  float* dwt = NEWF(T);
  float* ds = NEWF(T);
  const float inv = 1.0f / sqrtf((float)HD);
  for (int64_t r = 0; r < R; ++r)
    for (int64_t h = 0; h < NH; ++h) {
      const float* w = m->wts + (r * NH + h) * T;
      const float* dc = dctx + r * H + h * HD;
      for (int64_t t = 0; t < T; ++t) {
        const float* v = m->v + (r * T + t) * H + h * HD;
        float* dvp = dv + (r * T + t) * H + h * HD;
        float acc = 0.0f;
        for (int64_t dd = 0; dd < HD; ++dd) {
          dvp[dd] += w[t] * dc[dd];
          acc += dc[dd] * v[dd];
        }
        dwt[t] = acc;
      }
      float dot = 0.0f;
      for (int64_t t = 0; t < T; ++t) dot += w[t] * dwt[t];
      for (int64_t t = 0; t < T; ++t) ds[t] = w[t] * (dwt[t] - dot) * inv;
      const float* q = m->q + r * H + h * HD;
      float* dqp = dq + r * H + h * HD;
      for (int64_t t = 0; t < T; ++t) {
        const float* k = m->k + (r * T + t) * H + h * HD;
        float* dkp = dk + (r * T + t) * H + h * HD;
        for (int64_t dd = 0; dd < HD; ++dd) {
          dqp[dd] += ds[t] * k[dd];
          dkp[dd] += ds[t] * q[dd];
        }
      }
    }
  float* dx = NEWF(R * T * E);
  linear_bwd(m->x, W(m, P_KW), G(m, P_KW), G(m, P_KB), dk, dx, R * T, E, H);
  linear_bwd(m->x, W(m, P_VW), G(m, P_VW), G(m, P_VB), dv, dx, R * T, E, H);
  float* xl = NEWF(R * E);
  float* dxl = NEWF(R * E);
  for (int64_t r = 0; r < R; ++r) memcpy(xl + r * E, m->x + (r * T + T - 1) * E, (size_t)E * 4);
  linear_bwd(xl, W(m, P_QW), G(m, P_QW), G(m, P_QB), dq, dxl, R, E, H);
  for (int64_t r = 0; r < R; ++r)
    for (int64_t j = 0; j < E; ++j) dx[(r * T + T - 1) * E + j] += dxl[r * E + j];
  for (int64_t r = 0; r < R; ++r)
    for (int64_t t = 0; t < T; ++t)
      for (int64_t j = 0; j < E; ++j) G(m, P_POS)[t * E + j] += dx[(r * T + t) * E + j];
  for (int64_t r = 0; r < R; ++r)
    for (int64_t t = 0; t < T; ++t) {
      float* dst = G(m, P_EMB) + (int64_t)m->ctx[r * T + t] * E;
      for (int64_t j = 0; j < E; ++j) dst[j] += dx[(r * T + t) * E + j];
    }
  free(dffn); free(dact); free(datt); free(dctx); free(dq); free(dk); free(dv); free(dwt);
  free(ds); free(dx); free(xl); free(dxl);
}

static void trainer_snapshot(const dm_t* m, buf_t* b) {
  write_params(b, m->ps, NP_DM, m->w);
  adam_serialize(b, &m->adam, m->ps, NP_DM);
}
static void trainer_restore(dm_t* m, const uint8_t* p, size_t n) {
  rd_t r = {p, n, 0, E_CORRUPT_STREAM};
  read_params(&r, m->ps, NP_DM, m->w);
  adam_deserialize(&r, &m->adam, m->ps, NP_DM);
}

/* ---- BiGruModel (models.cpp:38-102, layers.cpp:187-413) ------------------- */
enum { G_WIR, G_WIZ, G_WIN, G_WHR, G_WHZ, G_WHN, G_BIR, G_BIZ, G_BIN, G_BHR, G_BHZ, G_BHN, NG };
static const char* kGruNames[NG] = {"w_ir", "w_iz", "w_in", "w_hr", "w_hz", "w_hn",
                                    "b_ir", "b_iz", "b_in", "b_hr", "b_hz", "b_hn"};
typedef struct {
  dims_t d;
  int layers, np;
  pdesc* ps;
  char** names;
  size_t n;
  float *w, *g;
} bigru_t;
/* param index of (layer, dir, tensor) */
static int gidx(int l, int dir, int t) { return 1 + (l * 2 + dir) * NG + t; }

static void bigru_init(bigru_t* m, dims_t d, int layers, uint64_t seed) {
  memset(m, 0, sizeof *m);
  m->d = d;
  m->layers = layers;
  m->np = 1 + layers * 2 * NG + 4;
  m->ps = (pdesc*)xcalloc((size_t)m->np, sizeof(pdesc));
  m->names = (char**)xcalloc((size_t)m->np, sizeof(char*));
  const int64_t V = d.V, Es = d.se, Hs = d.sh, B = d.sb;
  size_t off = 0;
  set_p(&m->ps[0], "emb.table", 2, V, Es, &off);
  for (int l = 0; l < layers; ++l)
    for (int dir = 0; dir < 2; ++dir)
      for (int t = 0; t < NG; ++t) {
        const int i = gidx(l, dir, t);
        m->names[i] = (char*)xcalloc(48, 1);
        snprintf(m->names[i], 48, "gru%d.%s.%s", l, dir ? "bwd" : "fwd", kGruNames[t]);
        const int64_t in = l == 0 ? Es : 2 * Hs;
        if (t <= G_WIN) set_p(&m->ps[i], m->names[i], 2, in, Hs, &off);
        else if (t <= G_WHN) set_p(&m->ps[i], m->names[i], 2, Hs, Hs, &off);
        else set_p(&m->ps[i], m->names[i], 1, Hs, 0, &off);
      }
  const int b0 = 1 + layers * 2 * NG;
  set_p(&m->ps[b0], "bott.w", 2, 2 * Hs, B, &off);
  set_p(&m->ps[b0 + 1], "bott.b", 1, B, 0, &off);
  set_p(&m->ps[b0 + 2], "out.w", 2, B, V, &off);
  set_p(&m->ps[b0 + 3], "out.b", 1, V, 0, &off);
  m->n = off;
  m->w = NEWF(off);
  m->g = NEWF(off);
  rng_t rng = {seed};
  init_uniform(m->w, m->ps[0].count, V, &rng);
  for (int l = 0; l < layers; ++l)
    for (int dir = 0; dir < 2; ++dir) {
      const int64_t in = l == 0 ? Es : 2 * Hs;
      for (int t = G_WIR; t <= G_WIN; ++t) init_uniform(m->w + m->ps[gidx(l, dir, t)].off, m->ps[gidx(l, dir, t)].count, in, &rng);
      for (int t = G_WHR; t <= G_WHN; ++t) init_uniform(m->w + m->ps[gidx(l, dir, t)].off, m->ps[gidx(l, dir, t)].count, Hs, &rng);
    }
  for (int i = b0; i < b0 + 2; ++i) init_uniform(m->w + m->ps[i].off, m->ps[i].count, 2 * Hs, &rng);
  for (int i = b0 + 2; i < b0 + 4; ++i) init_uniform(m->w + m->ps[i].off, m->ps[i].count, B, &rng);
}
static void bigru_free(bigru_t* m) {
  for (int i = 0; i < m->np; ++i) free(m->names[i]);
  free(m->names); free(m->ps); free(m->w); free(m->g);
}
#define BW(m, i) ((m)->w + (m)->ps[i].off)
#define BG(m, i) ((m)->g + (m)->ps[i].off)

/* serialize_model / deserialize_model (models.cpp:159-198) */
static void bigru_serialize(const bigru_t* m, buf_t* b) {
  b_bytes(b, "PMKW", 4);
  b_u8(b, 1);
  b_u8(b, (uint8_t)m->layers);
  b_le(b, (uint64_t)m->d.V, 4);
  b_le(b, (uint64_t)m->d.T, 2);
  b_le(b, (uint64_t)m->d.se, 8);
  b_le(b, (uint64_t)m->d.sh, 8);
  b_le(b, (uint64_t)m->d.sb, 8);
  write_params(b, m->ps, m->np, m->w);
}
static void bigru_deserialize(bigru_t* m, const uint8_t* p, size_t n) {
  rd_t r = {p, n, 0, E_ARCHITECTURE_MISMATCH};
  if (memcmp(r_take(&r, 4), "PMKW", 4)) raise_err(E_BAD_MAGIC, "model file magic");
  if (r_le(&r, 1) != 1) raise_err(E_UNSUPPORTED_VERSION, "model file version");
  const int layers = (int)r_le(&r, 1);
  dims_t d = {0};
  d.V = (int64_t)r_le(&r, 4);
  d.T = (int64_t)r_le(&r, 2);
  d.se = (int64_t)r_le(&r, 8);
  d.sh = (int64_t)r_le(&r, 8);
  d.sb = (int64_t)r_le(&r, 8);
  if (layers < 1 || d.V < 2 || d.T < 1 || d.se < 1 || d.sh < 1 || d.sb < 1)
    raise_err(E_ARCHITECTURE_MISMATCH, "model header");
  bigru_init(m, d, layers, 0);
  read_params(&r, m->ps, m->np, m->w);
}
static buf_t read_whole(const char* path) {
  buf_t b = {0};
  FILE* f = fopen(path, "rb");
  if (!f) raise_err(E_IO_ERROR, "cannot open %s", path);
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  b_reserve(&b, (size_t)n + 1);
  b.n = fread(b.p, 1, (size_t)n, f);
  fclose(f);
  if (b.n != (size_t)n) raise_err(E_IO_ERROR, "short read on %s", path);
  return b;
}

typedef struct { float *r, *z, *n, *hh, *out; } gtape_t; /* each [R,T,H] */
typedef struct {
  int64_t R;
  float* emb;          /* [R,T,Es] */
  gtape_t* tp;         /* [layers][2] */
  float** xrev;        /* [layers] input reversed in time */
  float** gout;        /* [layers] [R,T,2H] */
  float *fin, *bact;   /* [R,2H], [R,B] */
} btape_t;

/* Gru::forward (layers.cpp:213-260) */
static void gru_fwd(const bigru_t* m, int l, int dir, const float* x, int64_t R, int64_t in, gtape_t* tp) {
  const int64_t T = m->d.T, H = m->d.sh, nh = R * H;
  const float* P[NG];
  for (int t = 0; t < NG; ++t) P[t] = BW(m, gidx(l, dir, t));
  float *xt = NEWF(R * in), *hp = NEWF(R * H), *ar = NEWF(R * H), *az = NEWF(R * H), *an = NEWF(R * H), *hb = NEWF(R * H);
  for (int64_t t = 0; t < T; ++t) {
    for (int64_t r = 0; r < R; ++r) memcpy(xt + r * in, x + (r * T + t) * in, (size_t)in * 4);
    linear_fwd(xt, P[G_WIR], P[G_BIR], ar, R, in, H);
    for (int64_t i = 0; i < nh; ++i) ar[i] += P[G_BHR][i % H];
    mm_acc(hp, P[G_WHR], ar, R, H, H);
    linear_fwd(xt, P[G_WIZ], P[G_BIZ], az, R, in, H);
    for (int64_t i = 0; i < nh; ++i) az[i] += P[G_BHZ][i % H];
    mm_acc(hp, P[G_WHZ], az, R, H, H);
    linear_fwd(hp, P[G_WHN], P[G_BHN], hb, R, H, H);
    linear_fwd(xt, P[G_WIN], P[G_BIN], an, R, in, H);
    for (int64_t i = 0; i < nh; ++i) {
      const int64_t at = ((i / H) * T + t) * H + i % H;
      const float rv = det_sigmoid(ar[i]), zv = det_sigmoid(az[i]), hv0 = hb[i];
      const float nv = det_tanh(an[i] + rv * hv0);
      const float hv = (1.0f - zv) * nv + zv * hp[i];
      tp->r[at] = rv; tp->z[at] = zv; tp->n[at] = nv; tp->hh[at] = hv0; tp->out[at] = hv;
      hp[i] = hv;
    }
  }
  free(xt); free(hp); free(ar); free(az); free(an); free(hb);
}
static float* reverse_steps(const float* x, int64_t R, int64_t T, int64_t w) {
  float* o = NEWF(R * T * w);
  for (int64_t r = 0; r < R; ++r)
    for (int64_t t = 0; t < T; ++t) memcpy(o + (r * T + (T - 1 - t)) * w, x + (r * T + t) * w, (size_t)w * 4);
  return o;
}
static void tape_alloc(gtape_t* g, int64_t n) {
  g->r = NEWF(n); g->z = NEWF(n); g->n = NEWF(n); g->hh = NEWF(n); g->out = NEWF(n);
}
static void tape_free_g(gtape_t* g) { free(g->r); free(g->z); free(g->n); free(g->hh); free(g->out); }

/* BiGruModel::forward (models.cpp:53-73) */
static void bigru_forward(const bigru_t* m, const uint32_t* ctx, int64_t R, btape_t* tp, float* logits) {
  const int64_t T = m->d.T, Es = m->d.se, H = m->d.sh, B = m->d.sb, V = m->d.V;
  memset(tp, 0, sizeof *tp);
  tp->R = R;
  tp->emb = NEWF(R * T * Es);
  for (int64_t i = 0; i < R * T; ++i) memcpy(tp->emb + i * Es, BW(m, 0) + (int64_t)ctx[i] * Es, (size_t)Es * 4);
  tp->tp = (gtape_t*)xcalloc((size_t)m->layers * 2, sizeof(gtape_t));
  tp->xrev = (float**)xcalloc((size_t)m->layers, sizeof(float*));
  tp->gout = (float**)xcalloc((size_t)m->layers, sizeof(float*));
  const float* cur = tp->emb;
  int64_t in = Es;
  for (int l = 0; l < m->layers; ++l) {
    gtape_t* f = &tp->tp[l * 2];
    gtape_t* b = &tp->tp[l * 2 + 1];
    tape_alloc(f, R * T * H);
    tape_alloc(b, R * T * H);
    gru_fwd(m, l, 0, cur, R, in, f);
    tp->xrev[l] = reverse_steps(cur, R, T, in);
    gru_fwd(m, l, 1, tp->xrev[l], R, in, b);
    float* o = NEWF(R * T * 2 * H);
    for (int64_t r = 0; r < R; ++r)
      for (int64_t t = 0; t < T; ++t) {
        memcpy(o + (r * T + t) * 2 * H, f->out + (r * T + t) * H, (size_t)H * 4);
        memcpy(o + (r * T + t) * 2 * H + H, b->out + (r * T + (T - 1 - t)) * H, (size_t)H * 4);
      }
    tp->gout[l] = o;
    cur = o;
    in = 2 * H;
  }
  const gtape_t* lf = &tp->tp[(m->layers - 1) * 2];
  tp->fin = NEWF(R * 2 * H);
  for (int64_t r = 0; r < R; ++r) {
    memcpy(tp->fin + r * 2 * H, lf[0].out + (r * T + T - 1) * H, (size_t)H * 4);
    memcpy(tp->fin + r * 2 * H + H, lf[1].out + (r * T + T - 1) * H, (size_t)H * 4);
  }
  const int b0 = 1 + m->layers * 2 * NG;
  tp->bact = NEWF(R * B);
  linear_fwd(tp->fin, BW(m, b0), BW(m, b0 + 1), tp->bact, R, 2 * H, B);
  for (int64_t i = 0; i < R * B; ++i) tp->bact[i] = det_tanh(tp->bact[i]);
  linear_fwd(tp->bact, BW(m, b0 + 2), BW(m, b0 + 3), logits, R, B, V);
}
static void btape_free(btape_t* tp, int layers) {
  free(tp->emb);
  for (int l = 0; l < layers; ++l) {
    tape_free_g(&tp->tp[2 * l]); tape_free_g(&tp->tp[2 * l + 1]);
    free(tp->xrev[l]); free(tp->gout[l]);
  }
  free(tp->tp); free(tp->xrev); free(tp->gout); free(tp->fin); free(tp->bact);
}

/* Gru::backward (layers.cpp:262-327) */
static void gru_bwd(bigru_t* m, int l, int dir, const float* x, int64_t R, int64_t in, const gtape_t* tp,
                    const float* dout, float* dx) {
  const int64_t T = m->d.T, H = m->d.sh, nh = R * H;
  const float* P[NG];
  float* D[NG];
  for (int t = 0; t < NG; ++t) { P[t] = BW(m, gidx(l, dir, t)); D[t] = BG(m, gidx(l, dir, t)); }
  float *dh = NEWF(nh), *dhn = NEWF(nh), *dan = NEWF(nh), *dar = NEWF(nh), *daz = NEWF(nh), *dhh = NEWF(nh);
  float *xt = NEWF(R * in), *hp = NEWF(nh), *dxt = NEWF(R * in);
  for (int64_t t = T - 1; t >= 0; --t) {
    for (int64_t r = 0; r < R; ++r) memcpy(xt + r * in, x + (r * T + t) * in, (size_t)in * 4);
    if (t == 0) memset(hp, 0, (size_t)nh * 4);
    else for (int64_t r = 0; r < R; ++r) memcpy(hp + r * H, tp->out + (r * T + t - 1) * H, (size_t)H * 4);
    for (int64_t r = 0; r < R; ++r)
      for (int64_t j = 0; j < H; ++j) dh[r * H + j] += dout[(r * T + t) * H + j];
    for (int64_t i = 0; i < nh; ++i) {
      const int64_t at = ((i / H) * T + t) * H + i % H;
      const float rv = tp->r[at], zv = tp->z[at], nv = tp->n[at], hv = tp->hh[at], dhv = dh[i];
      const float dzv = dhv * (hp[i] - nv);
      const float danv = dhv * (1.0f - zv) * (1.0f - nv * nv);
      dan[i] = danv;
      dar[i] = danv * hv * rv * (1.0f - rv);
      daz[i] = dzv * zv * (1.0f - zv);
      dhh[i] = danv * rv;
      dhn[i] = dhv * zv;
    }
    memset(dxt, 0, (size_t)(R * in) * 4);
    mm_acc_bt(dan, P[G_WIN], dxt, R, H, in);
    mm_acc_bt(dar, P[G_WIR], dxt, R, H, in);
    mm_acc_bt(daz, P[G_WIZ], dxt, R, H, in);
    for (int64_t r = 0; r < R; ++r)
      for (int64_t j = 0; j < in; ++j) dx[(r * T + t) * in + j] += dxt[r * in + j];
    mm_acc_bt(dhh, P[G_WHN], dhn, R, H, H);
    mm_acc_bt(dar, P[G_WHR], dhn, R, H, H);
    mm_acc_bt(daz, P[G_WHZ], dhn, R, H, H);
    mm_acc_at(xt, dan, D[G_WIN], in, R, H);
    mm_acc_at(xt, dar, D[G_WIR], in, R, H);
    mm_acc_at(xt, daz, D[G_WIZ], in, R, H);
    mm_acc_at(hp, dhh, D[G_WHN], H, R, H);
    mm_acc_at(hp, dar, D[G_WHR], H, R, H);
    mm_acc_at(hp, daz, D[G_WHZ], H, R, H);
    const float* srcs[6] = {dan, dar, daz, dhh, dar, daz};
    const int dsts[6] = {G_BIN, G_BIR, G_BIZ, G_BHN, G_BHR, G_BHZ};
    for (int s = 0; s < 6; ++s)
      for (int64_t r = 0; r < R; ++r)
        for (int64_t j = 0; j < H; ++j) D[dsts[s]][j] += srcs[s][r * H + j];
    float* tmp = dh; dh = dhn; dhn = tmp;
    memset(dhn, 0, (size_t)nh * 4);
  }
  free(dh); free(dhn); free(dan); free(dar); free(daz); free(dhh); free(xt); free(hp); free(dxt);
}

/* BiGruModel::backward (models.cpp:75-96), BiGru::backward (layers.cpp:369-387) */
static void bigru_backward(bigru_t* m, const uint32_t* ctx, const btape_t* tp, const float* dlog) {
  const int64_t R = tp->R, T = m->d.T, Es = m->d.se, H = m->d.sh, B = m->d.sb, V = m->d.V;
  const int b0 = 1 + m->layers * 2 * NG;
  float* dba = NEWF(R * B);
  linear_bwd(tp->bact, BW(m, b0 + 2), BG(m, b0 + 2), BG(m, b0 + 3), dlog, dba, R, B, V);
  for (int64_t i = 0; i < R * B; ++i) dba[i] *= (1.0f - tp->bact[i] * tp->bact[i]);
  float* dfin = NEWF(R * 2 * H);
  linear_bwd(tp->fin, BW(m, b0), BG(m, b0), BG(m, b0 + 1), dba, dfin, R, 2 * H, B);
  float* dcur = NEWF(R * T * 2 * H);
  for (int64_t r = 0; r < R; ++r) {
    for (int64_t j = 0; j < H; ++j) dcur[(r * T + T - 1) * 2 * H + j] += dfin[r * 2 * H + j];
    for (int64_t j = 0; j < H; ++j) dcur[(r * T) * 2 * H + H + j] += dfin[r * 2 * H + H + j];
  }
  for (int l = m->layers - 1; l >= 0; --l) {
    const float* input = l == 0 ? tp->emb : tp->gout[l - 1];
    const int64_t in = l == 0 ? Es : 2 * H;
    float* dxl = NEWF(R * T * in);
    float* df = NEWF(R * T * H);
    float* db = NEWF(R * T * H);
    for (int64_t r = 0; r < R; ++r)
      for (int64_t t = 0; t < T; ++t) {
        memcpy(df + (r * T + t) * H, dcur + (r * T + t) * 2 * H, (size_t)H * 4);
        memcpy(db + (r * T + (T - 1 - t)) * H, dcur + (r * T + t) * 2 * H + H, (size_t)H * 4);
      }
    gru_bwd(m, l, 0, input, R, in, &tp->tp[2 * l], df, dxl);
    float* dxr = NEWF(R * T * in);
    gru_bwd(m, l, 1, tp->xrev[l], R, in, &tp->tp[2 * l + 1], db, dxr);
    for (int64_t r = 0; r < R; ++r)
      for (int64_t t = 0; t < T; ++t)
        for (int64_t j = 0; j < in; ++j) dxl[(r * T + t) * in + j] += dxr[(r * T + (T - 1 - t)) * in + j];
    free(df); free(db); free(dxr); free(dcur);
    dcur = dxl;
  }
  for (int64_t i = 0; i < R * T; ++i) {
    float* dst = BG(m, 0) + (int64_t)ctx[i] * Es;
    for (int64_t j = 0; j < Es; ++j) dst[j] += dcur[i * Es + j];
  }
  free(dba); free(dfin); free(dcur);
}

/* train_pass (training.cpp:8-41) */
static void train_pass(bigru_t* m, adam_t* a, const uint32_t* tok, uint64_t n, uint32_t t, uint32_t batch) {
  if (n < (uint64_t)t + 1) raise_err(E_TARGET_TOO_SHORT, "need at least t+1 tokens");
  const int64_t V = m->d.V;
  uint32_t* ctx = (uint32_t*)xcalloc((size_t)batch * t, 4);
  float* lg = NEWF((int64_t)batch * V);
  for (uint64_t p = t; p < n; p += batch) {
    const int64_t R = (int64_t)(batch < n - p ? batch : n - p);
    for (int64_t r = 0; r < R; ++r)
      for (uint32_t i = 0; i < t; ++i) ctx[r * t + i] = tok[p + (uint64_t)r - t + i];
    btape_t tp;
    bigru_forward(m, ctx, R, &tp, lg);
    for (int64_t r = 0; r < R; ++r) {
      det_softmax(lg + r * V, (size_t)V);
      lg[r * V + tok[p + (uint64_t)r]] -= 1.0f;
    }
    bigru_backward(m, ctx, &tp, lg);
    btape_free(&tp, m->layers);
    adam_step(a, m->w, m->g);
    memset(m->g, 0, m->n * 4);
  }
  free(ctx); free(lg);
}
static int dims_fit(const dims_t* a, const dims_t* b) {
  return a->V == b->V && a->T == b->T && a->se == b->se && a->sh == b->sh && a->sb == b->sb;
}
/* pretrain_private + derive_private_init (training.cpp:62-83, models.cpp:200-215) */
static void pretrain_private(bigru_t* out, const uint32_t* tok, uint64_t n, const bigru_t* pub,
                             dims_t dims, uint32_t t, uint32_t batch, uint64_t seed) {
  if (n < (uint64_t)t + 1) raise_err(E_TARGET_TOO_SHORT, "target shorter than t+1 tokens");
  bigru_init(out, dims, 1, seed);
  if (pub && dims_fit(&pub->d, &dims)) {
    for (int i = 0; i < out->np; ++i) {
      if (strcmp(out->ps[i].name, "emb.table") && strncmp(out->ps[i].name, "gru0.", 5)) continue;
      for (int j = 0; j < pub->np; ++j)
        if (!strcmp(pub->ps[j].name, out->ps[i].name)) {
          memcpy(out->w + out->ps[i].off, pub->w + pub->ps[j].off, out->ps[i].count * 4);
          break;
        }
    }
  }
  adam_t a = {0, 1.0f, 1.0f, NEWF(out->n), NEWF(out->n), out->n};
  train_pass(out, &a, tok, n, t, batch);
  free(a.m); free(a.v);
}

/* ---- mixer (mixer.cpp:14-42) ---------------------------------------------- */
static void mix_row(int pub, int priv, int dyn, float alpha, const float* lu, const float* lr,
                    const float* lm, float* probs, int64_t width) {
  const float s0 = pub ? 1.0f : 0.0f, s1 = priv ? 1.0f : 0.0f, s2 = dyn ? 1.0f : 0.0f;
  for (int64_t i = 0; i < width; ++i) {
    const float stat = s0 * (lu ? lu[i] : 0.0f) + s1 * (lr ? lr[i] : 0.0f);
    probs[i] = alpha * stat + (1.0f - alpha) * s2 * (lm ? lm[i] : 0.0f);
  }
  det_softmax(probs, (size_t)width);
}

/* ---- chunk worker (pipeline.cpp:98-235) ----------------------------------- */
typedef struct {
  int flags;
  const bigru_t *pub, *priv;
  dims_t dims;
  uint32_t t, bs;
  uint64_t dm_seed;
  const uint8_t* inbound;
  size_t inbound_n;
  uint64_t snap_step;
  buf_t* snap_out;       /* receives the snapshot at snap_step (NULL: none) */
  orc_chunk_stats* st;   /* nullable */
  float* probs_dump;     /* nullable [max_steps, bs, V] */
  uint64_t max_dump;
} chunk_spec;

typedef struct {
  chunk_spec sp;
  dm_t dm;
  qdist uni, q;
  double* rem;
  uint32_t* order;
  float *lu, *lr, *probs, *g;
  uint32_t *ctx, *tg;
  uint64_t L, warm, model_steps;
  double warm_loss;
  int snapped;
} worker_t;

static void worker_init(worker_t* w, const chunk_spec* sp, uint64_t ntok) {
  memset(w, 0, sizeof *w);
  w->sp = *sp;
  const int64_t R = sp->bs, V = sp->dims.V;
  dm_init(&w->dm, sp->dims, sp->dm_seed, R);
  if (sp->inbound_n) {
    trainer_restore(&w->dm, sp->inbound, sp->inbound_n);
    if (sp->st) sp->st->snapshot_recv_hash = fnv1a(sp->inbound, sp->inbound_n, FNV_SEED);
  }
  w->uni = qd_new((uint32_t)V);
  uniform_dist((uint32_t)V, &w->uni);
  w->q = qd_new((uint32_t)V);
  w->rem = (double*)xcalloc((size_t)V, 8);
  w->order = (uint32_t*)xcalloc((size_t)V, 4);
  w->lu = NEWF(R * V);
  w->lr = NEWF(R * V);
  w->probs = NEWF(R * V);
  w->g = NEWF(R * V);
  w->ctx = (uint32_t*)xcalloc((size_t)(R * sp->t), 4);
  w->tg = (uint32_t*)xcalloc((size_t)R, 4);
  w->L = ntok / sp->bs;
  w->warm = (w->L * 500 + 9999) / 10000;
  if (w->warm < 1) w->warm = 1;
  if (sp->st) sp->st->tokens = ntok;
}
static void worker_free(worker_t* w) {
  dm_free(&w->dm);
  free(w->uni.freqs); free(w->uni.cum); free(w->q.freqs); free(w->q.cum); free(w->rem); free(w->order);
  free(w->lu); free(w->lr); free(w->probs); free(w->g); free(w->ctx); free(w->tg);
}
static void model_step(worker_t* w, const uint32_t* tokens, uint64_t j) {
  const chunk_spec* sp = &w->sp;
  const int64_t R = sp->bs, V = sp->dims.V, t = sp->t;
  for (int64_t r = 0; r < R; ++r)
    for (int64_t i = 0; i < t; ++i) w->ctx[r * t + i] = tokens[(uint64_t)r * w->L + (j - t) + (uint64_t)i];
  btape_t tp;
  if (sp->flags & 1) {
    bigru_forward(sp->pub, w->ctx, R, &tp, w->lu);
    btape_free(&tp, sp->pub->layers);
    if (sp->st) sp->st->pub_calls += 1;
  }
  if (sp->flags & 2) {
    bigru_forward(sp->priv, w->ctx, R, &tp, w->lr);
    btape_free(&tp, sp->priv->layers);
    if (sp->st) sp->st->priv_calls += 1;
  }
  dm_forward(&w->dm, w->ctx);
  if (sp->st) sp->st->dyn_calls += 1;
  const float alpha = det_sigmoid(W(&w->dm, P_ALPHA)[0]);
  for (int64_t r = 0; r < R; ++r)
    mix_row(sp->flags & 1, sp->flags & 2, 1, alpha, (sp->flags & 1) ? w->lu + r * V : NULL,
            (sp->flags & 2) ? w->lr + r * V : NULL, w->dm.lm + r * V, w->probs + r * V, V);
  if (sp->probs_dump && w->model_steps < sp->max_dump)
    memcpy(sp->probs_dump + w->model_steps * (uint64_t)(R * V), w->probs, (size_t)(R * V) * 4);
}
/* OnlineTrainer::step (mixer.cpp:57-97) */
static float train_step(worker_t* w) {
  const chunk_spec* sp = &w->sp;
  dm_t* m = &w->dm;
  const int64_t R = sp->bs, V = sp->dims.V;
  const float a = det_sigmoid(W(m, P_ALPHA)[0]);
  const float s0 = (sp->flags & 1) ? 1.0f : 0.0f, s1 = (sp->flags & 2) ? 1.0f : 0.0f;
  float loss = 0.0f, dalpha = 0.0f;
  memcpy(w->g, w->probs, (size_t)(R * V) * 4);
  for (int64_t r = 0; r < R; ++r) {
    float* gr = w->g + r * V;
    const uint32_t tgt = w->tg[r];
    const float pt = gr[tgt] < 1e-38f ? 1e-38f : gr[tgt]; /* std::max(a, b) */
    loss += -det_log(pt);
    gr[tgt] -= 1.0f;
    for (int64_t i = 0; i < V; ++i) {
      const float stat = s0 * ((sp->flags & 1) ? w->lu[r * V + i] : 0.0f) + s1 * ((sp->flags & 2) ? w->lr[r * V + i] : 0.0f);
      dalpha += gr[i] * (stat - m->lm[r * V + i]);
    }
  }
  G(m, P_ALPHA)[0] += dalpha * a * (1.0f - a);
  const float wgt = 1.0f - a;
  for (int64_t i = 0; i < R * V; ++i) w->g[i] *= wgt;
  dm_backward(m, w->g);
  adam_step(&m->adam, m->w, m->g);
  memset(m->g, 0, m->n * 4);
  if (w->model_steps < w->warm) w->warm_loss += loss;
  w->model_steps += 1;
  return loss;
}
static void maybe_snapshot(worker_t* w, uint64_t done) {
  if (!w->sp.snap_out || w->snapped || done != w->sp.snap_step) return;
  trainer_snapshot(&w->dm, w->sp.snap_out);
  if (w->sp.st) w->sp.st->snapshot_sent_hash = fnv1a(w->sp.snap_out->p, w->sp.snap_out->n, FNV_SEED);
  w->snapped = 1;
}
static void worker_finish(worker_t* w) {
  if (!w->sp.st) return;
  const uint64_t c = w->model_steps < w->warm ? w->model_steps : w->warm;
  if (c) w->sp.st->early_loss_bits = w->warm_loss / (double)(c * w->sp.bs) / 0.6931471805599453;
}
static void worker_encode(worker_t* w, const uint32_t* tok, buf_t* out) {
  renc_t e = {out, 0, ~0ull};
  const uint32_t R = w->sp.bs;
  for (uint64_t j = 0; j < w->L; ++j) {
    if (j < w->sp.t) {
      for (uint32_t r = 0; r < R; ++r) renc_encode(&e, &w->uni, tok[r * w->L + j]);
      if (w->sp.st) w->sp.st->uniform_coded += R;
    } else {
      model_step(w, tok, j);
      for (uint32_t r = 0; r < R; ++r) {
        w->tg[r] = tok[r * w->L + j];
        quantize(w->probs + (int64_t)r * w->sp.dims.V, (uint32_t)w->sp.dims.V, &w->q, w->rem, w->order);
        renc_encode(&e, &w->q, w->tg[r]);
      }
      train_step(w);
    }
    maybe_snapshot(w, j + 1);
  }
  renc_finish(&e);
  worker_finish(w);
}
static void worker_decode(worker_t* w, const uint8_t* pay, size_t pn, uint32_t* tok) {
  rdec_t d;
  rdec_init(&d, pay, pn);
  const uint32_t R = w->sp.bs;
  for (uint64_t j = 0; j < w->L; ++j) {
    if (j < w->sp.t) {
      for (uint32_t r = 0; r < R; ++r) tok[r * w->L + j] = rdec_decode(&d, &w->uni);
      if (w->sp.st) w->sp.st->uniform_coded += R;
    } else {
      model_step(w, tok, j);
      for (uint32_t r = 0; r < R; ++r) {
        quantize(w->probs + (int64_t)r * w->sp.dims.V, (uint32_t)w->sp.dims.V, &w->q, w->rem, w->order);
        w->tg[r] = rdec_decode(&d, &w->q);
        tok[r * w->L + j] = w->tg[r];
      }
      train_step(w);
    }
    maybe_snapshot(w, j + 1);
  }
  worker_finish(w);
}

/* ---- plan (pipeline.cpp:26-52) -------------------------------------------- */
typedef struct { uint64_t* start; uint64_t* len; uint64_t W; uint32_t bs; } plan_t;
static plan_t plan_chunks(uint64_t m, uint32_t workers, uint32_t bs, uint32_t t) {
  plan_t p = {0};
  if (m == 0) { p.bs = 1; return p; }
  const uint64_t per = (uint64_t)bs * ((uint64_t)t + 1);
  uint64_t mw = m / per;
  if (mw < 1) mw = 1;
  p.W = workers < mw ? workers : mw;
  p.start = (uint64_t*)xcalloc((size_t)p.W, 8);
  p.len = (uint64_t*)xcalloc((size_t)p.W, 8);
  const uint64_t base = m / p.W, rem = m % p.W;
  uint64_t s = 0;
  for (uint64_t i = 0; i < p.W; ++i) {
    p.start[i] = s;
    p.len[i] = base + (i < rem ? 1 : 0);
    s += p.len[i];
  }
  uint64_t b = base / ((uint64_t)t + 1);
  if (b < 1) b = 1;
  p.bs = (uint32_t)(bs < b ? bs : b);
  return p;
}
static uint64_t snapshot_step(uint64_t len, uint32_t bs, uint16_t myriad) {
  const uint64_t steps = len / bs;
  const uint64_t s = ((uint64_t)myriad * steps + 9999) / 10000;
  return s ? s : 1;
}

/* pack_tokens / unpack_tokens (pipeline.cpp:58-92) */
static void pack_tokens(const uint32_t* tok, uint64_t n, uint32_t k, buf_t* out) {
  const unsigned bits = 2u * k;
  uint64_t acc = 0;
  unsigned fill = 0;
  for (uint64_t i = 0; i < n; ++i) {
    acc |= (uint64_t)tok[i] << fill;
    fill += bits;
    while (fill >= 8) { b_u8(out, (uint8_t)acc); acc >>= 8; fill -= 8; }
  }
  if (fill) b_u8(out, (uint8_t)acc);
}
static void unpack_tokens(const uint8_t* b, size_t bn, uint32_t k, uint32_t* out, uint64_t n) {
  const unsigned bits = 2u * k;
  const uint32_t limit = 1u << bits;
  uint64_t acc = 0;
  unsigned fill = 0;
  size_t pos = 0;
  for (uint64_t i = 0; i < n; ++i) {
    while (fill < bits) {
      if (pos >= bn) raise_err(E_CORRUPT_STREAM, "trailer shorter than its token count");
      acc |= (uint64_t)b[pos++] << fill;
      fill += 8;
    }
    out[i] = (uint32_t)(acc & (limit - 1));
    acc >>= bits;
    fill -= bits;
  }
}

/* ---- compress / decompress (pipeline.cpp:303-450, container.cpp:41-149) ---- */
static int base_code(uint8_t c) {
  switch (c) { case 'A': return 0; case 'C': return 1; case 'G': return 2; case 'T': return 3; default: return -1; }
}
static void put_packed_bases(buf_t* b, const uint8_t* bases, uint64_t n) {
  b_le(b, n, 8);
  uint8_t cur = 0;
  int fill = 0;
  for (uint64_t i = 0; i < n; ++i) {
    cur |= (uint8_t)((bases[i] & 3) << (2 * fill));
    if (++fill == 4) { b_u8(b, cur); cur = 0; fill = 0; }
  }
  if (fill) b_u8(b, cur);
}

int orc_compress(const uint8_t* in, size_t n, const orc_cfg* c, uint8_t** out, size_t* out_n,
                 orc_chunk_stats* stats, size_t stats_cap, size_t* n_chunks) {
  ENTRY;
  /* CompressConfig::validate (pipeline.cpp:16-24) */
  if (!(c->s >= 1 && c->s <= c->k && c->k <= 8)) raise_err(E_CONFIG_INVALID, "window parameters");
  if (c->t < 1 || c->t > 4096) raise_err(E_CONFIG_INVALID, "context length out of range");
  if (c->bs < 1 || c->bs > 1000000) raise_err(E_CONFIG_INVALID, "substream count out of range");
  if (c->workers < 1 || c->workers > 256) raise_err(E_CONFIG_INVALID, "worker count out of range");
  if (!(c->smp >= 0.0f) || c->smp >= 1.0f) raise_err(E_CONFIG_INVALID, "handoff fraction");
  const uint32_t vocab = 1u << (2 * c->k);
  const dims_t dims = make_dims(vocab, c->t, c->scale);
  rng_t master = {c->seed};
  const uint64_t dm_seed = rng_u64(&master), sprm_seed = rng_u64(&master);

  uint8_t* codes = (uint8_t*)xcalloc(n, 1);
  uint64_t nc = 0;
  buf_t exc = {0};
  uint64_t n_exc = 0;
  for (size_t i = 0; i < n; ++i) {
    const int b = base_code(in[i]);
    if (b >= 0) codes[nc++] = (uint8_t)b;
    else { b_le(&exc, i, 8); b_u8(&exc, in[i]); ++n_exc; }
  }
  const uint64_t m = token_count(nc, c->s, c->k);
  uint32_t* tok = (uint32_t*)xcalloc((size_t)m, 4);
  uint64_t res_n = 0;
  uint8_t* res = (uint8_t*)xcalloc((size_t)nc, 1);
  orc_skmer_encode(codes, nc, c->s, c->k, 1, tok, &(uint64_t){0}, res, &res_n);

  int flags = (uint64_t)n <= c->threshold ? 5 : 6;
  bigru_t pub, priv;
  int have_pub = 0, have_priv = 0;
  uint64_t pub_fp = 0;
  if (c->pub_path && *c->pub_path) {
    buf_t f = read_whole(c->pub_path);
    bigru_deserialize(&pub, f.p, f.n);
    pub_fp = fnv1a(f.p, f.n, FNV_SEED);
    free(f.p);
    if (!dims_fit(&pub.d, &dims)) raise_err(E_ARCHITECTURE_MISMATCH, "public model does not fit");
    have_pub = 1;
  }
  if ((flags & 1) && !have_pub) flags = 4;
  if ((flags & 2) && m < (uint64_t)c->t + 1) flags = 4;
  if (flags & 2) {
    pretrain_private(&priv, tok, m, have_pub ? &pub : NULL, dims, c->t, c->bs, sprm_seed);
    have_priv = 1;
  }
  const uint16_t myriad = (uint16_t)lround((double)c->smp * 10000.0);
  plan_t p = plan_chunks(m, c->workers, c->bs, c->t);
  if (n_chunks) *n_chunks = p.W;
  buf_t* pay = (buf_t*)xcalloc((size_t)p.W, sizeof(buf_t));
  buf_t* trl = (buf_t*)xcalloc((size_t)p.W, sizeof(buf_t));
  buf_t inbound = {0};
  for (uint64_t i = 0; i < p.W; ++i) {
    chunk_spec sp = {flags, have_pub ? &pub : NULL, have_priv ? &priv : NULL, dims, c->t, p.bs, dm_seed,
                     inbound.p, inbound.n, 0, NULL, (stats && i < stats_cap) ? &stats[i] : NULL, NULL, 0};
    if (sp.st) memset(sp.st, 0, sizeof *sp.st);
    buf_t snap = {0};
    if (myriad && i + 1 < p.W) { sp.snap_step = snapshot_step(p.len[i], p.bs, myriad); sp.snap_out = &snap; }
    worker_t w;
    const uint64_t L = p.len[i] / p.bs;
    worker_init(&w, &sp, L * p.bs);
    worker_encode(&w, tok + p.start[i], &pay[i]);
    worker_free(&w);
    pack_tokens(tok + p.start[i] + L * p.bs, p.len[i] - L * p.bs, c->k, &trl[i]);
    if (myriad && i + 1 < p.W) {
      if (!w.snapped) { free(snap.p); } /* too short: forward inbound unchanged */
      else { free(inbound.p); inbound = snap; }
    }
  }
  /* write_container (container.cpp:41-88) */
  buf_t o = {0};
  b_bytes(&o, "PMKL", 4);
  b_u8(&o, 1);
  b_u8(&o, (uint8_t)flags);
  b_u8(&o, (uint8_t)c->s);
  b_u8(&o, (uint8_t)c->k);
  b_le(&o, c->t, 2);
  b_le(&o, p.bs, 4);
  b_le(&o, myriad, 2);
  b_le(&o, dm_seed, 8);
  b_le(&o, (flags & 2) ? sprm_seed : c->scale, 8);
  b_le(&o, (flags & 1) ? pub_fp : 0, 8);
  b_le(&o, n, 8);
  b_le(&o, p.W, 4);
  buf_t pm = {0};
  if (have_priv) bigru_serialize(&priv, &pm);
  uint64_t off = 52 + p.W * 36 + 8 + pm.n + 8 + n_exc * 9 + 8 + (res_n + 3) / 4;
  for (uint64_t i = 0; i < p.W; ++i) {
    b_le(&o, p.start[i], 8);
    b_le(&o, p.len[i], 8);
    b_le(&o, off, 8);
    b_le(&o, pay[i].n, 8);
    b_le(&o, trl[i].n, 4);
    off += pay[i].n + trl[i].n;
  }
  b_le(&o, pm.n, 8);
  b_bytes(&o, pm.p, pm.n);
  b_le(&o, n_exc, 8);
  b_bytes(&o, exc.p, exc.n);
  put_packed_bases(&o, res, res_n);
  for (uint64_t i = 0; i < p.W; ++i) {
    b_bytes(&o, pay[i].p, pay[i].n);
    b_bytes(&o, trl[i].p, trl[i].n);
    free(pay[i].p);
    free(trl[i].p);
  }
  b_le(&o, fnv1a(o.p, o.n, FNV_SEED), 8);
  *out = o.p;
  *out_n = o.n;
  free(pay); free(trl); free(inbound.p); free(pm.p); free(exc.p); free(codes); free(tok); free(res);
  free(p.start); free(p.len);
  if (have_pub) bigru_free(&pub);
  if (have_priv) bigru_free(&priv);
  LEAVE;
}

int orc_decompress(const uint8_t* in, size_t n, const char* pub_path, uint32_t workers,
                   uint8_t** out, size_t* out_n, orc_chunk_stats* stats, size_t stats_cap) {
  (void)workers;
  ENTRY;
  if (n < 52 + 8) raise_err(E_TABLE_INCONSISTENT, "container too small");
  {
    rd_t t = {in + n - 8, 8, 0, E_TABLE_INCONSISTENT};
    if (fnv1a(in, n - 8, FNV_SEED) != r_le(&t, 8)) raise_err(E_CHECKSUM_MISMATCH, "container checksum");
  }
  rd_t r = {in, n, 0, E_TABLE_INCONSISTENT};
  if (memcmp(r_take(&r, 4), "PMKL", 4)) raise_err(E_BAD_MAGIC, "container magic");
  if (r_le(&r, 1) != 1) raise_err(E_UNSUPPORTED_VERSION, "container version");
  const int flags = (int)r_le(&r, 1);
  const uint32_t s = (uint32_t)r_le(&r, 1), k = (uint32_t)r_le(&r, 1), t = (uint32_t)r_le(&r, 2);
  const uint32_t bs = (uint32_t)r_le(&r, 4);
  const uint16_t myriad = (uint16_t)r_le(&r, 2);
  const uint64_t dm_seed = r_le(&r, 8), sprm = r_le(&r, 8), pub_fp = r_le(&r, 8), orig = r_le(&r, 8);
  const uint32_t W = (uint32_t)r_le(&r, 4);
  if ((uint64_t)W * 36 > n) raise_err(E_TABLE_INCONSISTENT, "chunk count exceeds file size");
  uint64_t *cs = (uint64_t*)xcalloc(W, 8), *cl = (uint64_t*)xcalloc(W, 8), *po = (uint64_t*)xcalloc(W, 8), *pl = (uint64_t*)xcalloc(W, 8), *tl = (uint64_t*)xcalloc(W, 8);
  uint64_t next = 0;
  for (uint32_t i = 0; i < W; ++i) {
    cs[i] = r_le(&r, 8); cl[i] = r_le(&r, 8); po[i] = r_le(&r, 8); pl[i] = r_le(&r, 8); tl[i] = r_le(&r, 4);
    if (cs[i] != next) raise_err(E_TABLE_INCONSISTENT, "chunk token ranges not contiguous");
    next += cl[i];
  }
  const uint64_t ml = r_le(&r, 8);
  if (ml > r.n - r.pos) raise_err(E_TABLE_INCONSISTENT, "private model length");
  const uint8_t* pmb = r_take(&r, (size_t)ml);
  const uint64_t ne = r_le(&r, 8);
  uint64_t* ep = (uint64_t*)xcalloc((size_t)ne, 8);
  uint8_t* eb = (uint8_t*)xcalloc((size_t)ne, 1);
  for (uint64_t i = 0; i < ne; ++i) {
    ep[i] = r_le(&r, 8); eb[i] = (uint8_t)r_le(&r, 1);
    if (i > 0 && ep[i] <= ep[i - 1]) raise_err(E_TABLE_INCONSISTENT, "exception positions not strictly increasing");
  }
  const uint64_t rn = r_le(&r, 8);
  const uint8_t* rp = r_take(&r, (size_t)((rn + 3) / 4));
  const uint8_t** pay = (const uint8_t**)xcalloc(W, sizeof(void*));
  const uint8_t** trl = (const uint8_t**)xcalloc(W, sizeof(void*));
  for (uint32_t i = 0; i < W; ++i) {
    if (po[i] != r.pos) raise_err(E_TABLE_INCONSISTENT, "payload offset");
    if (pl[i] + tl[i] > r.n - r.pos) raise_err(E_TABLE_INCONSISTENT, "payload length");
    pay[i] = r_take(&r, (size_t)pl[i]);
    trl[i] = r_take(&r, (size_t)tl[i]);
  }
  if (r.n - r.pos != 8) raise_err(E_TABLE_INCONSISTENT, "trailing bytes after payloads");

  if (!(flags & 4)) raise_err(E_TABLE_INCONSISTENT, "dynamic model flag must be set");
  if (!(s >= 1 && s <= k && k <= 8) || t < 1 || bs < 1) raise_err(E_TABLE_INCONSISTENT, "coding parameters");
  bigru_t pub, priv;
  uint32_t scale;
  if (flags & 2) {
    bigru_deserialize(&priv, pmb, (size_t)ml);
    if (priv.d.se < 1 || 16 % priv.d.se) raise_err(E_ARCHITECTURE_MISMATCH, "private model width");
    scale = (uint32_t)(16 / priv.d.se);
  } else {
    if (sprm < 1 || sprm > 16) raise_err(E_TABLE_INCONSISTENT, "model width divisor");
    scale = (uint32_t)sprm;
  }
  const dims_t dims = make_dims(1u << (2 * k), t, scale);
  if ((flags & 2) && !dims_fit(&priv.d, &dims)) raise_err(E_ARCHITECTURE_MISMATCH, "private model does not fit");
  if (flags & 1) {
    if (!pub_path || !*pub_path) raise_err(E_SPUM_MISSING, "container requires the public model file");
    buf_t f = read_whole(pub_path);
    if (fnv1a(f.p, f.n, FNV_SEED) != pub_fp) raise_err(E_CHECKSUM_MISMATCH, "public model file does not match");
    bigru_deserialize(&pub, f.p, f.n);
    free(f.p);
    if (!dims_fit(&pub.d, &dims)) raise_err(E_ARCHITECTURE_MISMATCH, "public model does not fit");
  }
  const uint64_t pb = orig - (orig < ne ? orig : ne);
  if (token_count(pb, s, k) != next) raise_err(E_CORRUPT_STREAM, "token count does not match the original length");
  uint32_t* tok = (uint32_t*)xcalloc((size_t)next, 4);
  buf_t inbound = {0};
  for (uint32_t i = 0; i < W; ++i) {
    chunk_spec sp = {flags, (flags & 1) ? &pub : NULL, (flags & 2) ? &priv : NULL, dims, t, bs, dm_seed,
                     inbound.p, inbound.n, 0, NULL, (stats && i < stats_cap) ? &stats[i] : NULL, NULL, 0};
    if (sp.st) memset(sp.st, 0, sizeof *sp.st);
    buf_t snap = {0};
    if (myriad && i + 1 < W) { sp.snap_step = snapshot_step(cl[i], bs, myriad); sp.snap_out = &snap; }
    const uint64_t L = cl[i] / bs;
    worker_t w;
    worker_init(&w, &sp, L * bs);
    worker_decode(&w, pay[i], (size_t)pl[i], tok + cs[i]);
    worker_free(&w);
    const uint64_t left = cl[i] - L * bs;
    if ((tl[i] * 8) / (2 * k) < left) raise_err(E_CORRUPT_STREAM, "trailer too short");
    unpack_tokens(trl[i], (size_t)tl[i], k, tok + cs[i] + L * bs, left);
    if (myriad && i + 1 < W) {
      if (!w.snapped) free(snap.p);
      else { free(inbound.p); inbound = snap; }
    }
  }
  /* decode tokens (skmer.cpp:63-83) + restore (alphabet.cpp:37-60) */
  const uint32_t width = 1u << (2 * k);
  uint8_t* bases = (uint8_t*)xcalloc((size_t)pb + 1, 1);
  uint64_t nb = 0;
  for (uint64_t j = 0; j < next; ++j) {
    if (tok[j] >= width) raise_err(E_TOKEN_OUT_OF_RANGE, "token exceeds 4^k");
    const uint32_t emit = (j + 1 == next) ? k : s;
    for (uint32_t i = 0; i < emit; ++i) {
      if (nb >= pb) raise_err(E_CORRUPT_STREAM, "decoded base count");
      bases[nb++] = (uint8_t)((tok[j] >> (2 * (k - 1 - i))) & 3);
    }
  }
  for (uint64_t i = 0; i < rn; ++i) {
    if (nb >= pb) raise_err(E_CORRUPT_STREAM, "decoded base count");
    bases[nb++] = (rp[i / 4] >> (2 * (i % 4))) & 3;
  }
  if (nb != pb) raise_err(E_CORRUPT_STREAM, "decoded base count");
  uint8_t* o = (uint8_t*)xcalloc((size_t)orig, 1);
  uint8_t* filled = (uint8_t*)xcalloc((size_t)orig, 1);
  for (uint64_t i = 0; i < ne; ++i) {
    if (ep[i] >= orig) raise_err(E_LENGTH_MISMATCH, "exception position beyond original length");
    o[ep[i]] = eb[i];
    filled[ep[i]] = 1;
  }
  static const uint8_t B4[4] = {'A', 'C', 'G', 'T'};
  uint64_t nx = 0;
  for (uint64_t i = 0; i < orig; ++i) {
    if (filled[i]) continue;
    o[i] = B4[bases[nx++] & 3];
  }
  *out = o;
  *out_n = (size_t)orig;
  free(filled); free(bases); free(tok); free(inbound.p); free(cs); free(cl); free(po); free(pl); free(tl);
  free(ep); free(eb); free(pay); free(trl);
  if (flags & 1) bigru_free(&pub);
  if (flags & 2) bigru_free(&priv);
  LEAVE;
}

int orc_quantize(const float* p, uint32_t n, uint32_t* freqs) {
  ENTRY;
  qdist d = qd_new(n);
  double* rem = (double*)xcalloc(n, 8);
  uint32_t* ord = (uint32_t*)xcalloc(n, 4);
  quantize(p, n, &d, rem, ord);
  memcpy(freqs, d.freqs, (size_t)n * 4);
  free(d.freqs); free(d.cum); free(rem); free(ord);
  LEAVE;
}
int orc_uniform_dist(uint32_t n, uint32_t* freqs) {
  ENTRY;
  qdist d = qd_new(n);
  uniform_dist(n, &d);
  memcpy(freqs, d.freqs, (size_t)n * 4);
  free(d.freqs); free(d.cum);
  LEAVE;
}
int orc_range_encode(const uint32_t* freqs, uint32_t width, const uint32_t* dist_of,
                     const uint32_t* syms, size_t count, uint8_t** out, size_t* out_n) {
  ENTRY;
  qdist d = qd_new(width);
  buf_t b = {0};
  renc_t e = {&b, 0, ~0ull};
  for (size_t i = 0; i < count; ++i) {
    memcpy(d.freqs, freqs + (size_t)dist_of[i] * width, (size_t)width * 4);
    build_cum(&d);
    renc_encode(&e, &d, syms[i]);
  }
  renc_finish(&e);
  *out = b.p;
  *out_n = b.n;
  free(d.freqs); free(d.cum);
  LEAVE;
}
int orc_det(int which, const float* x, float* y, size_t n) {
  ENTRY;
  for (size_t i = 0; i < n; ++i)
    y[i] = which == 0 ? det_exp(x[i]) : which == 1 ? det_log(x[i]) : which == 2 ? det_sigmoid(x[i]) : det_tanh(x[i]);
  LEAVE;
}
int orc_softmax(const float* x, float* y, size_t n) {
  ENTRY;
  if (y != x) memcpy(y, x, n * 4);
  det_softmax(y, n);
  LEAVE;
}
int orc_bigru_predict(const char* path, const uint32_t* ctx, int64_t rows, int64_t steps, float* logits) {
  ENTRY;
  buf_t f = read_whole(path);
  bigru_t m;
  bigru_deserialize(&m, f.p, f.n);
  if (steps != m.d.T) raise_err(E_CONTEXT_LENGTH_MISMATCH, "context window length");
  btape_t tp;
  bigru_forward(&m, ctx, rows, &tp, logits);
  btape_free(&tp, m.layers);
  bigru_free(&m);
  free(f.p);
  LEAVE;
}
int orc_dump_chunk(const uint32_t* tokens, uint64_t n_tokens, uint32_t flags_bits,
                   const char* pub_path, uint32_t k, uint32_t t, uint32_t bs, uint32_t scale,
                   uint64_t dm_seed, const uint8_t* inbound, size_t inbound_n, float* probs,
                   uint64_t max_steps, uint8_t** payload, size_t* payload_n, uint8_t** snap,
                   size_t* snap_n) {
  ENTRY;
  const dims_t dims = make_dims(1u << (2 * k), t, scale);
  bigru_t pub;
  if (flags_bits & 1) {
    buf_t f = read_whole(pub_path);
    bigru_deserialize(&pub, f.p, f.n);
    free(f.p);
  }
  chunk_spec sp = {(int)flags_bits, (flags_bits & 1) ? &pub : NULL, NULL, dims, t, bs, dm_seed,
                   inbound, inbound_n, 0, NULL, NULL, probs, max_steps};
  worker_t w;
  worker_init(&w, &sp, n_tokens);
  buf_t o = {0}, s = {0};
  worker_encode(&w, tokens, &o);
  trainer_snapshot(&w.dm, &s);
  worker_free(&w);
  if (flags_bits & 1) bigru_free(&pub);
  *payload = o.p;
  *payload_n = o.n;
  *snap = s.p;
  *snap_n = s.n;
  LEAVE;
}
/* one chunk from an inbound snapshot; also returns the trainer snapshot taken
 * when steps_done == snap_at (ChunkWorker::maybe_snapshot, pipeline.cpp:207-213),
 * empty when never reached */
int orc_encode_chunk_snap(const uint32_t* tokens, uint64_t n_tokens, uint32_t flags_bits,
                          const char* pub_path, uint32_t k, uint32_t t, uint32_t bs,
                          uint32_t scale, uint64_t dm_seed, const uint8_t* inbound,
                          size_t inbound_n, uint64_t snap_at, uint8_t** payload,
                          size_t* payload_n, uint8_t** snap, size_t* snap_n) {
  ENTRY;
  const dims_t dims = make_dims(1u << (2 * k), t, scale);
  bigru_t pub;
  if (flags_bits & 1) {
    buf_t f = read_whole(pub_path);
    bigru_deserialize(&pub, f.p, f.n);
    free(f.p);
  }
  buf_t sb = {0};
  chunk_spec sp = {(int)flags_bits, (flags_bits & 1) ? &pub : NULL, NULL, dims, t, bs, dm_seed,
                   inbound, inbound_n, snap_at, snap_at ? &sb : NULL, NULL, NULL, 0};
  worker_t w;
  worker_init(&w, &sp, n_tokens);
  buf_t o = {0};
  worker_encode(&w, tokens, &o);
  worker_free(&w);
  if (flags_bits & 1) bigru_free(&pub);
  *payload = o.p;
  *payload_n = o.n;
  *snap = sb.p;
  *snap_n = sb.n;
  LEAVE;
}

int orc_pretrain_private(const uint32_t* tokens, uint64_t m, const char* pub_path, uint32_t k,
                         uint32_t t, uint32_t batch, uint32_t scale, uint64_t seed,
                         uint8_t** out, size_t* out_n) {
  ENTRY;
  const dims_t dims = make_dims(1u << (2 * k), t, scale);
  bigru_t pub, priv;
  int hp = pub_path && *pub_path;
  if (hp) {
    buf_t f = read_whole(pub_path);
    bigru_deserialize(&pub, f.p, f.n);
    free(f.p);
  }
  pretrain_private(&priv, tokens, m, hp ? &pub : NULL, dims, t, batch, seed);
  buf_t b = {0};
  bigru_serialize(&priv, &b);
  *out = b.p;
  *out_n = b.n;
  bigru_free(&priv);
  if (hp) bigru_free(&pub);
  LEAVE;
}
