/*
 * sgdt_oracle.c -- TEST INFRASTRUCTURE ONLY (see sgdt_oracle.h).
 *
 * A plain-C restatement of the reference CPU algorithm, kept in the reference's
 * own fp64 operation order.  Each function cites the reference file:line it
 * restates (paths relative to /root/reference/proj).
 */
#include "sgdt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================== */
/* RNG: std::mt19937_64 (the engine behind rng.hpp:46) + Rng (rng.hpp:13-49) */
/* ======================================================================== */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void or_rng_seed(or_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (uint32_t i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + i;
  r->idx = MT_N;
  r->has_spare = 0;
  r->spare = 0.0;
}

static void mt_twist(uint64_t* x) {
  uint32_t k;
  for (k = 0; k < MT_N - MT_M; ++k) {
    uint64_t y = (x[k] & MT_UPPER) | (x[k + 1] & MT_LOWER);
    x[k] = x[k + MT_M] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
  }
  for (; k < MT_N - 1; ++k) {
    uint64_t y = (x[k] & MT_UPPER) | (x[k + 1] & MT_LOWER);
    x[k] = x[k + MT_M - MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
  }
  uint64_t y = (x[MT_N - 1] & MT_UPPER) | (x[0] & MT_LOWER);
  x[MT_N - 1] = x[MT_M - 1] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
}

uint64_t or_rng_next(or_rng* r) {
  if (r->idx >= MT_N) {
    mt_twist(r->mt);
    r->idx = 0;
  }
  uint64_t z = r->mt[r->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= (z >> 43);
  return z;
}

/* rng.hpp:20-25 */
uint64_t or_next_below(or_rng* r, uint64_t bound) {
  const uint64_t threshold = (0ULL - bound) % bound;
  uint64_t v = or_rng_next(r);
  while (v < threshold) v = or_rng_next(r);
  return v % bound;
}

/* rng.hpp:28 */
double or_next_unit(or_rng* r) { return (double)(or_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:31-43 */
double or_next_gaussian(or_rng* r, double mean, double stddev) {
  if (r->has_spare) {
    r->has_spare = 0;
    return mean + stddev * r->spare;
  }
  const double u1 = 1.0 - or_next_unit(r);
  const double u2 = or_next_unit(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.141592653589793 * u2;
  r->spare = radius * sin(angle);
  r->has_spare = 1;
  return mean + stddev * radius * cos(angle);
}

void or_mt_outputs(uint64_t seed, size_t n, uint64_t* out) {
  or_rng r;
  or_rng_seed(&r, seed);
  for (size_t i = 0; i < n; ++i) out[i] = or_rng_next(&r);
}

/* ======================================================================== */
/* small dense helpers (matrix.hpp:49-62)                                    */
/* ======================================================================== */
static double dot(const double* a, const double* b, size_t n) {
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

static double dot_strided(const double* a, const double* col, size_t stride, size_t n) {
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += a[i] * col[i * stride];
  return acc;
}

/* ======================================================================== */
/* sparse tensor (sptensor.cpp:17-25, 80-118)                                */
/* ======================================================================== */
typedef struct {
  uint64_t* keys;
  uint8_t* used;
  size_t cap;
} u64set;

static int u64set_init(u64set* s, size_t n) {
  size_t cap = 16;
  while (cap < 2 * n + 16) cap <<= 1;
  s->keys = (uint64_t*)malloc(cap * sizeof(uint64_t));
  s->used = (uint8_t*)calloc(cap, 1);
  s->cap = cap;
  return (s->keys && s->used) ? 0 : -1;
}
static void u64set_free(u64set* s) {
  free(s->keys);
  free(s->used);
}
/* returns 1 if inserted, 0 if already present */
static int u64set_insert(u64set* s, uint64_t k) {
  uint64_t h = k * 0x9E3779B97F4A7C15ULL;
  size_t i = (size_t)(h >> 17) & (s->cap - 1);
  while (s->used[i]) {
    if (s->keys[i] == k) return 0;
    i = (i + 1) & (s->cap - 1);
  }
  s->used[i] = 1;
  s->keys[i] = k;
  return 1;
}

void or_tensor_free(or_tensor* t) {
  free(t->coords);
  free(t->values);
  for (int n = 0; n < OR_MAX_ORDER; ++n) {
    free(t->perm[n]);
    free(t->offsets[n]);
  }
  memset(t, 0, sizeof *t);
}

int or_tensor_init(or_tensor* t, int order, const uint32_t* dims, size_t nnz,
                   const uint32_t* coords, const double* values) {
  memset(t, 0, sizeof *t);
  if (order < 2 || order > OR_MAX_ORDER) return OR_DOMAIN;
  if (nnz == 0) return OR_DATA;
  if (nnz > 0xFFFFFFFFULL) return OR_DATA;
  t->order = order;
  for (int k = 0; k < order; ++k) {
    if (dims[k] < 1) return OR_DOMAIN;
    t->dims[k] = dims[k];
  }
  t->nnz = nnz;
  t->coords = (uint32_t*)malloc(nnz * order * sizeof(uint32_t));
  t->values = (double*)malloc(nnz * sizeof(double));
  if (!t->coords || !t->values) {
    or_tensor_free(t);
    return OR_INTERNAL;
  }
  memcpy(t->coords, coords, nnz * order * sizeof(uint32_t));
  memcpy(t->values, values, nnz * sizeof(double));
  /* validation + duplicate check by linear key (sptensor.cpp:90-100) */
  u64set seen;
  if (u64set_init(&seen, nnz)) {
    or_tensor_free(t);
    return OR_INTERNAL;
  }
  for (size_t e = 0; e < nnz; ++e) {
    const uint32_t* c = t->coords + e * order;
    uint64_t key = 0, stride = 1;
    for (int k = 0; k < order; ++k) {
      if (c[k] < 1 || c[k] > t->dims[k]) {
        u64set_free(&seen);
        or_tensor_free(t);
        return OR_DATA;
      }
      key += (uint64_t)(c[k] - 1) * stride;
      stride *= t->dims[k];
    }
    if (!u64set_insert(&seen, key)) {
      u64set_free(&seen);
      or_tensor_free(t);
      return OR_DATA;
    }
  }
  u64set_free(&seen);
  /* per-mode counting sort, stable in entry id (sptensor.cpp:102-117) */
  for (int n = 0; n < order; ++n) {
    const uint32_t dim = t->dims[n];
    uint64_t* off = (uint64_t*)calloc((size_t)dim + 1, sizeof(uint64_t));
    uint32_t* perm = (uint32_t*)malloc(nnz * sizeof(uint32_t));
    uint64_t* cursor = (uint64_t*)malloc((size_t)dim * sizeof(uint64_t));
    if (!off || !perm || !cursor) {
      free(off);
      free(perm);
      free(cursor);
      or_tensor_free(t);
      return OR_INTERNAL;
    }
    for (size_t e = 0; e < nnz; ++e) off[t->coords[e * order + n]]++;
    for (size_t i = 1; i <= dim; ++i) off[i] += off[i - 1];
    memcpy(cursor, off, (size_t)dim * sizeof(uint64_t));
    for (size_t e = 0; e < nnz; ++e) perm[cursor[t->coords[e * order + n] - 1]++] = (uint32_t)e;
    free(cursor);
    t->perm[n] = perm;
    t->offsets[n] = off;
  }
  return OR_OK;
}

/* ======================================================================== */
/* model (model.cpp:1-175)                                                   */
/* ======================================================================== */
void or_model_free(or_model* m) {
  for (int n = 0; n < OR_MAX_ORDER; ++n) {
    free(m->A[n]);
    free(m->B[n]);
    free(m->unfold[n]);
  }
  free(m->core);
  memset(m, 0, sizeof *m);
}

/* Ranks::validate (model.cpp:5-17) without the dense-core cap, which the
 * caller enforces where the reference does (model.cpp:90-92). */
int or_model_init(or_model* m, int order, const uint32_t* dims, const uint32_t* J, uint32_t R) {
  memset(m, 0, sizeof *m);
  if (order < 2 || order > OR_MAX_ORDER) return OR_DOMAIN;
  if (R < 1) return OR_DOMAIN;
  uint64_t prod = 1;
  for (int n = 0; n < order; ++n) {
    if (J[n] < 1 || J[n] < R || dims[n] < 1) return OR_DOMAIN;
    prod *= J[n];
  }
  if (prod > 100000ULL) return OR_DOMAIN; /* kMaxCoreElems, model.hpp:25 */
  m->order = order;
  m->R = R;
  m->core_elems = prod;
  for (int n = 0; n < order; ++n) {
    m->dims[n] = dims[n];
    m->J[n] = J[n];
    m->A[n] = (double*)calloc((size_t)dims[n] * J[n], sizeof(double));
    m->B[n] = (double*)calloc((size_t)J[n] * R, sizeof(double));
    m->unfold[n] = (double*)calloc(prod, sizeof(double));
    if (!m->A[n] || !m->B[n] || !m->unfold[n]) {
      or_model_free(m);
      return OR_INTERNAL;
    }
  }
  m->core = (double*)calloc(prod, sizeof(double));
  if (!m->core) {
    or_model_free(m);
    return OR_INTERNAL;
  }
  or_model_refresh_core(m);
  return OR_OK;
}

int or_model_copy(or_model* dst, const or_model* src) {
  int rc = or_model_init(dst, src->order, src->dims, src->J, src->R);
  if (rc) return rc;
  for (int n = 0; n < src->order; ++n) {
    memcpy(dst->A[n], src->A[n], (size_t)src->dims[n] * src->J[n] * sizeof(double));
    memcpy(dst->B[n], src->B[n], (size_t)src->J[n] * src->R * sizeof(double));
  }
  or_model_refresh_core(dst);
  return OR_OK;
}

/* init_gaussian (model.cpp:103-114): B^(1..N) then A^(1..N), row-major. */
int or_model_init_gaussian(or_model* m, double mean, double stddev, uint64_t seed) {
  if (!(stddev > 0.0)) return OR_DOMAIN;
  or_rng rng;
  or_rng_seed(&rng, seed);
  for (int n = 0; n < m->order; ++n)
    for (size_t i = 0; i < (size_t)m->J[n] * m->R; ++i)
      m->B[n][i] = or_next_gaussian(&rng, mean, stddev);
  for (int n = 0; n < m->order; ++n)
    for (size_t i = 0; i < (size_t)m->dims[n] * m->J[n]; ++i)
      m->A[n][i] = or_next_gaussian(&rng, mean, stddev);
  or_model_refresh_core(m);
  return OR_OK;
}

/* reconstruct_core (model.cpp:36-57) + unfold_dense (model.cpp:59-85) */
void or_model_refresh_core(or_model* m) {
  const int order = m->order;
  const size_t total = (size_t)m->core_elems;
  double* term = (double*)malloc(total * sizeof(double));
  double* next = (double*)malloc(total * sizeof(double));
  for (size_t i = 0; i < total; ++i) m->core[i] = 0.0;
  for (uint32_t r = 0; r < m->R; ++r) {
    size_t len = m->J[0];
    for (uint32_t j = 0; j < m->J[0]; ++j) term[j] = m->B[0][(size_t)j * m->R + r];
    for (int n = 1; n < order; ++n) {
      for (uint32_t j = 0; j < m->J[n]; ++j) {
        const double b = m->B[n][(size_t)j * m->R + r];
        for (size_t i = 0; i < len; ++i) next[j * len + i] = b * term[i];
      }
      len *= m->J[n];
      double* tmp = term;
      term = next;
      next = tmp;
    }
    for (size_t i = 0; i < total; ++i) m->core[i] += term[i];
  }
  free(term);
  free(next);
  /* unfoldings */
  uint32_t idx[OR_MAX_ORDER];
  for (int mode = 0; mode < order; ++mode) {
    const size_t cols = total / m->J[mode];
    memset(idx, 0, sizeof idx);
    for (size_t lin = 0; lin < total; ++lin) {
      uint64_t col = 0, stride = 1;
      for (int k = 0; k < order; ++k) {
        if (k == mode) continue;
        col += idx[k] * stride;
        stride *= m->J[k];
      }
      m->unfold[mode][(size_t)idx[mode] * cols + col] = m->core[lin];
      for (int k = 0; k < order; ++k) {
        if (++idx[k] < m->J[k]) break;
        idx[k] = 0;
      }
    }
  }
}

/* kron_row_excluding (model.cpp:124-146); s needs core_elems capacity. */
static void kron_row_excluding(const or_model* m, const uint32_t* coord, int mode, double* s) {
  s[0] = 1.0;
  size_t len = 1;
  for (int k = 0; k < m->order; ++k) {
    if (k == mode) continue;
    const double* arow = m->A[k] + (size_t)(coord[k] - 1) * m->J[k];
    const uint32_t jk = m->J[k];
    for (uint32_t j = jk; j-- > 0;) {
      const double f = arow[j];
      double* dst = s + (size_t)j * len;
      for (size_t i = 0; i < len; ++i) dst[i] = s[i] * f;
    }
    len *= jk;
  }
}

/* e_column (model.cpp:148-155) */
static void e_column(const or_model* m, const uint32_t* coord, int mode, double* s, double* e) {
  kron_row_excluding(m, coord, mode, s);
  const size_t cols = (size_t)(m->core_elems / m->J[mode]);
  for (uint32_t j = 0; j < m->J[mode]; ++j) e[j] = dot(m->unfold[mode] + j * cols, s, cols);
}

static double predict_ws(const or_model* m, const uint32_t* coord, double* s, double* e) {
  e_column(m, coord, 0, s, e);
  return dot(m->A[0] + (size_t)(coord[0] - 1) * m->J[0], e, m->J[0]);
}

/* predict (model.cpp:157-167) */
double or_model_predict(const or_model* m, const uint32_t* coord) {
  double* s = (double*)malloc(m->core_elems * sizeof(double));
  double e[4096];
  double v = predict_ws(m, coord, s, e);
  free(s);
  return v;
}

int or_model_all_finite(const or_model* m) {
  for (int n = 0; n < m->order; ++n) {
    for (size_t i = 0; i < (size_t)m->dims[n] * m->J[n]; ++i)
      if (!isfinite(m->A[n][i])) return 0;
    for (size_t i = 0; i < (size_t)m->J[n] * m->R; ++i)
      if (!isfinite(m->B[n][i])) return 0;
  }
  return 1;
}

/* ======================================================================== */
/* scheduler + sampler                                                       */
/* ======================================================================== */
/* partition_even (scheduler.cpp:34-46) */
void or_partition_even(size_t count, size_t workers, size_t* begins, size_t* ends) {
  const size_t base = count / workers, rem = count % workers;
  size_t at = 0;
  for (size_t w = 0; w < workers; ++w) {
    const size_t len = base + (w < rem ? 1 : 0);
    begins[w] = at;
    ends[w] = at + len;
    at += len;
  }
}

/* sample_batch (sptensor.cpp:256-270) */
int or_sample_batch(size_t nnz, size_t m, or_rng* rng, uint32_t* pool, int* pool_valid,
                    uint32_t* out) {
  if (m < 1 || m > nnz) return OR_DOMAIN;
  if (!*pool_valid) {
    for (size_t e = 0; e < nnz; ++e) pool[e] = (uint32_t)e;
    *pool_valid = 1;
  }
  for (size_t i = 0; i < m; ++i) {
    const size_t j = i + (size_t)or_next_below(rng, nnz - i);
    const uint32_t tmp = pool[i];
    pool[i] = pool[j];
    pool[j] = tmp;
  }
  memcpy(out, pool, m * sizeof(uint32_t));
  return OR_OK;
}

/* ======================================================================== */
/* optimizers                                                                */
/* ======================================================================== */
/* sgd_step (core_optimizer.cpp:85-100) */
static int sgd_step(size_t m, double lambda, double gamma, double* w, const double* v, size_t n) {
  if (m < 1) return OR_DOMAIN;
  if (!(gamma > 0.0)) return OR_DOMAIN;
  if (lambda < 0.0) return OR_DOMAIN;
  const double inv_m = 1.0 / (double)m;
  for (size_t i = 0; i < n; ++i) {
    if (!isfinite(w[i]) || !isfinite(v[i])) return OR_NUMERIC;
    w[i] -= gamma * (v[i] * inv_m + lambda * w[i]);
    if (!isfinite(w[i])) return OR_NUMERIC;
  }
  return OR_OK;
}

int or_core_ws_init(or_core_ws* ws, size_t nnz) {
  ws->pool = (uint32_t*)malloc(nnz * sizeof(uint32_t));
  ws->batch = (uint32_t*)malloc(nnz * sizeof(uint32_t));
  ws->pool_valid = 0;
  ws->batch_len = 0;
  return (ws->pool && ws->batch) ? OR_OK : OR_INTERNAL;
}

void or_core_ws_free(or_core_ws* ws) {
  free(ws->pool);
  free(ws->batch);
  memset(ws, 0, sizeof *ws);
}

/* update_core_epoch, serial strategy (core_optimizer.cpp:112-257) */
int or_update_core_epoch(or_model* md, const or_tensor* t, const or_core_hyper* h, or_rng* rng,
                         or_core_ws* ws) {
  if (h->lr < 0.0) return OR_DOMAIN;
  if (h->lr == 0.0) return OR_OK;
  const int order = md->order;
  const uint32_t rc = md->R;
  const size_t nnz = t->nnz;
  const size_t m = h->batch_m == 0 ? nnz : h->batch_m;
  if (m > nnz) return OR_DOMAIN;
  int rcode = OR_OK;

  double* x = (double*)malloc(m * sizeof(double));
  uint32_t jmax = 0;
  for (int n = 0; n < order; ++n)
    if (md->J[n] > jmax) jmax = md->J[n];
  double* coeff = (double*)malloc(m * rc * sizeof(double));
  double* w = (double*)malloc((size_t)rc * m * jmax * sizeof(double));
  double* resid = (double*)malloc(m * sizeof(double));
  double* bcols = (double*)malloc((size_t)rc * jmax * sizeof(double));
  double* C = (double*)malloc((size_t)jmax * jmax * sizeof(double));
  double* U = (double*)malloc(jmax * sizeof(double));
  double* V = (double*)malloc(jmax * sizeof(double));

#define DRAW_BATCH()                                                          \
  do {                                                                        \
    if (h->batch_m == 0) {                                                    \
      for (size_t e_ = 0; e_ < nnz; ++e_) ws->batch[e_] = (uint32_t)e_;       \
    } else {                                                                  \
      rcode = or_sample_batch(nnz, m, rng, ws->pool, &ws->pool_valid, ws->batch); \
      if (rcode) goto done;                                                   \
    }                                                                         \
    ws->batch_len = m;                                                        \
    for (size_t s_ = 0; s_ < m; ++s_) x[s_] = t->values[ws->batch[s_]];       \
  } while (0)

  DRAW_BATCH();
  for (int n = 0; n < order; ++n) {
    if (h->resample_per_mode && n > 0 && h->batch_m != 0) DRAW_BATCH();
    const uint32_t jn = md->J[n];
    double* bn = md->B[n];
    /* W_r rows (core_optimizer.cpp:158-180), layout [r][s][j] */
    for (size_t s = 0; s < m; ++s) {
      const uint32_t* coord = t->coords + (size_t)ws->batch[s] * order;
      const double* arow = md->A[n] + (size_t)(coord[n] - 1) * jn;
      for (uint32_t r = 0; r < rc; ++r) {
        double c = 1.0;
        for (int k = 0; k < order; ++k) {
          if (k == n) continue;
          c *= dot_strided(md->A[k] + (size_t)(coord[k] - 1) * md->J[k], md->B[k] + r, rc,
                           md->J[k]);
        }
        coeff[s * rc + r] = c;
        double* wrow = w + ((size_t)r * m + s) * jn;
        for (uint32_t j = 0; j < jn; ++j) wrow[j] = c * arow[j];
      }
    }
    for (uint32_t r_core = 0; r_core < rc; ++r_core) {
      for (uint32_t r = 0; r < rc; ++r)
        for (uint32_t j = 0; j < jn; ++j) bcols[(size_t)r * jn + j] = bn[(size_t)j * rc + r];
      if (!h->incremental_residual || r_core == 0) {
        for (size_t s = 0; s < m; ++s) {
          double acc = x[s];
          for (uint32_t r = 0; r < rc; ++r) {
            if (r == r_core) continue;
            acc -= dot(w + ((size_t)r * m + s) * jn, bcols + (size_t)r * jn, jn);
          }
          resid[s] = acc;
        }
      } else {
        const uint32_t prev = r_core - 1;
        for (size_t s = 0; s < m; ++s) {
          resid[s] -= dot(w + ((size_t)prev * m + s) * jn, bcols + (size_t)prev * jn, jn);
          resid[s] += dot(w + ((size_t)r_core * m + s) * jn, bcols + (size_t)r_core * jn, jn);
        }
      }
      /* single-worker partials then reduce_in_order (0.0 + p) */
      for (size_t i = 0; i < (size_t)jn * jn; ++i) C[i] = 0.0;
      for (uint32_t i = 0; i < jn; ++i) U[i] = 0.0;
      for (size_t s = 0; s < m; ++s) {
        const double* wrow = w + ((size_t)r_core * m + s) * jn;
        const double r_s = resid[s];
        for (uint32_t i = 0; i < jn; ++i) {
          U[i] += wrow[i] * r_s;
          for (uint32_t j = 0; j < jn; ++j) C[i * jn + j] += wrow[i] * wrow[j];
        }
      }
      for (size_t i = 0; i < (size_t)jn * jn; ++i) C[i] = 0.0 + C[i];
      for (uint32_t i = 0; i < jn; ++i) U[i] = 0.0 + U[i];
      double* bcol = bcols + (size_t)r_core * jn;
      for (uint32_t i = 0; i < jn; ++i) V[i] = -U[i] + dot(C + (size_t)i * jn, bcol, jn);
      rcode = sgd_step(m, h->reg, h->lr, bcol, V, jn);
      if (rcode) goto done;
      for (uint32_t j = 0; j < jn; ++j) bn[(size_t)j * rc + r_core] = bcol[j];
    }
  }
  or_model_refresh_core(md);
#undef DRAW_BATCH
done:
  free(x);
  free(coeff);
  free(w);
  free(resid);
  free(bcols);
  free(C);
  free(U);
  free(V);
  return rcode;
}

/* update_factor_epoch, serial strategy (factor_optimizer.cpp:101-187) with
 * grad_a_row (:34-54) and step_row (:90-97). */
int or_update_factor_epoch(or_model* md, const or_tensor* t, const or_factor_hyper* h,
                           or_rng* rng, size_t* rows_updated, size_t* rows_skipped) {
  if (!(h->row_fraction > 0.0 && h->row_fraction <= 1.0)) return OR_DOMAIN;
  if (h->lr < 0.0) return OR_DOMAIN;
  size_t upd = 0, skip = 0;
  if (h->lr == 0.0) {
    if (rows_updated) *rows_updated = 0;
    if (rows_skipped) *rows_skipped = 0;
    return OR_OK;
  }
  const int order = md->order;
  const size_t nnz = t->nnz;
  double* s = (double*)malloc(md->core_elems * sizeof(double));
  uint32_t jmax = 0;
  for (int n = 0; n < order; ++n)
    if (md->J[n] > jmax) jmax = md->J[n];
  double* e = (double*)malloc(jmax * sizeof(double));
  double* f1 = (double*)malloc(jmax * sizeof(double));
  double* f2 = (double*)malloc(jmax * sizeof(double));
  double* F = (double*)malloc(jmax * sizeof(double));
  uint32_t* sub_perm = (uint32_t*)malloc(nnz * sizeof(uint32_t));
  uint32_t* scratch = (uint32_t*)malloc(nnz * sizeof(uint32_t));
  uint64_t* sub_off = NULL;
  int rcode = OR_OK;

  for (int n = 0; n < order; ++n) {
    const uint32_t jn = md->J[n];
    const uint32_t dim = md->dims[n];
    const uint32_t* perm = t->perm[n];
    const uint64_t* off = t->offsets[n];
    if (h->row_fraction < 1.0) {
      free(sub_off);
      sub_off = (uint64_t*)calloc((size_t)dim + 1, sizeof(uint64_t));
      size_t len = 0;
      for (uint32_t i = 1; i <= dim; ++i) {
        const uint64_t b0 = t->offsets[n][i - 1], b1 = t->offsets[n][i];
        const size_t bs = (size_t)(b1 - b0);
        if (bs > 0) {
          memcpy(scratch, t->perm[n] + b0, bs * sizeof(uint32_t));
          size_t keep = (size_t)llround(h->row_fraction * (double)bs);
          if (keep < 1) keep = 1;
          for (size_t q = 0; q < keep; ++q) {
            const size_t j = q + (size_t)or_next_below(rng, bs - q);
            const uint32_t tmp = scratch[q];
            scratch[q] = scratch[j];
            scratch[j] = tmp;
          }
          memcpy(sub_perm + len, scratch, keep * sizeof(uint32_t));
          len += keep;
        }
        sub_off[i] = len;
      }
      perm = sub_perm;
      off = sub_off;
    }
    for (uint32_t i = 1; i <= dim; ++i) {
      const uint64_t b0 = off[i - 1], b1 = off[i];
      if (b1 == b0) {
        ++skip;
        continue;
      }
      ++upd;
      /* grad_a_row */
      for (uint32_t j = 0; j < jn; ++j) f1[j] = f2[j] = 0.0;
      double* arow = md->A[n] + (size_t)(i - 1) * jn;
      for (uint64_t q = b0; q < b1; ++q) {
        const uint32_t entry = perm[q];
        const uint32_t* coord = t->coords + (size_t)entry * order;
        e_column(md, coord, n, s, e);
        const double p = dot(arow, e, jn);
        const double xv = t->values[entry];
        for (uint32_t j = 0; j < jn; ++j) {
          f1[j] -= xv * e[j];
          f2[j] += p * e[j];
        }
      }
      for (uint32_t j = 0; j < jn; ++j) F[j] = f1[j] + f2[j];
      rcode = sgd_step((size_t)(b1 - b0), h->reg, h->lr, arow, F, jn);
      if (rcode) goto done;
    }
  }
done:
  if (rows_updated) *rows_updated = upd;
  if (rows_skipped) *rows_skipped = skip;
  free(s);
  free(e);
  free(f1);
  free(f2);
  free(F);
  free(sub_perm);
  free(scratch);
  free(sub_off);
  return rcode;
}

/* ======================================================================== */
/* eval (eval.cpp:15-33)                                                     */
/* ======================================================================== */
int or_rmse_mae(const or_model* m, const or_tensor* t, double* rmse, double* mae) {
  if (t->nnz == 0) return OR_DOMAIN;
  if (t->order != m->order) return OR_DOMAIN;
  for (int n = 0; n < m->order; ++n)
    if (t->dims[n] > m->dims[n]) return OR_DOMAIN;
  double* s = (double*)malloc(m->core_elems * sizeof(double));
  double* e = (double*)malloc(m->J[0] * sizeof(double));
  double sq = 0.0, ab = 0.0;
  for (size_t i = 0; i < t->nnz; ++i) {
    const double err = t->values[i] - predict_ws(m, t->coords + i * t->order, s, e);
    sq += err * err;
    ab += fabs(err);
  }
  free(s);
  free(e);
  const double inv = 1.0 / (double)t->nnz;
  *rmse = sqrt(sq * inv);
  *mae = ab * inv;
  return OR_OK;
}

/* ======================================================================== */
/* trainer (trainer.cpp:66-125)                                              */
/* ======================================================================== */
int or_train(or_model* m, const or_tensor* train, const or_tensor* test, const or_hyper* h,
             double* metrics) {
  if (!(h->lr_a > 0.0) || !(h->lr_b > 0.0)) return OR_CONFIG;
  if (h->reg_a < 0.0 || h->reg_b < 0.0) return OR_CONFIG;
  if (h->epochs < 1) return OR_CONFIG;
  if (!(h->row_fraction > 0.0 && h->row_fraction <= 1.0)) return OR_CONFIG;
  or_rng rng;
  or_rng_seed(&rng, h->seed + 1);
  or_core_hyper ch = {h->lr_b, h->reg_b, h->batch_m, h->resample_core_batch,
                      h->incremental_residual};
  or_factor_hyper fh = {h->lr_a, h->reg_a, h->row_fraction};
  or_core_ws ws;
  if (or_core_ws_init(&ws, train->nnz)) return OR_INTERNAL;
  int rc = OR_OK;
  for (size_t ep = 0; ep < h->epochs; ++ep) {
    rc = or_update_core_epoch(m, train, &ch, &rng, &ws);
    if (rc) break;
    rc = or_update_factor_epoch(m, train, &fh, &rng, NULL, NULL);
    if (rc) break;
    if (!or_model_all_finite(m)) {
      rc = OR_NUMERIC;
      break;
    }
    double* row = metrics + ep * 4;
    or_rmse_mae(m, train, &row[0], &row[1]);
    if (test) {
      or_rmse_mae(m, test, &row[2], &row[3]);
    } else {
      row[2] = row[3] = NAN;
    }
  }
  or_core_ws_free(&ws);
  return rc;
}

/* ======================================================================== */
/* synthetic data (synth.cpp:16-67) and split (sptensor.cpp:217-254)        */
/* ======================================================================== */
static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}
static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int or_synth_planted(int order, const uint32_t* dims, const uint32_t* tJ, uint32_t tR,
                     size_t nnz, double noise_stddev, double teacher_mean,
                     double teacher_stddev, uint64_t seed, uint32_t* coords_out,
                     double* values_out) {
  or_model teacher;
  int rc = or_model_init(&teacher, order, dims, tJ, tR);
  if (rc) return rc;
  rc = or_model_init_gaussian(&teacher, teacher_mean, teacher_stddev, seed);
  if (rc) {
    or_model_free(&teacher);
    return rc;
  }
  or_rng rng;
  or_rng_seed(&rng, seed + 0x9E3779B97F4A7C15ULL);
  /* draw_positions (synth.cpp:16-42) */
  uint64_t total = 1;
  for (int k = 0; k < order; ++k) total *= dims[k];
  if (nnz == 0 || nnz > total) {
    or_model_free(&teacher);
    return OR_DOMAIN;
  }
  uint64_t* pos = (uint64_t*)malloc(nnz * sizeof(uint64_t));
  if (total <= (1ULL << 22)) {
    uint64_t* pool = (uint64_t*)malloc(total * sizeof(uint64_t));
    for (uint64_t i = 0; i < total; ++i) pool[i] = i + 1;
    for (size_t i = 0; i < nnz; ++i) {
      const uint64_t j = i + or_next_below(&rng, total - i);
      const uint64_t tmp = pool[i];
      pool[i] = pool[j];
      pool[j] = tmp;
    }
    memcpy(pos, pool, nnz * sizeof(uint64_t));
    free(pool);
  } else {
    if (nnz > total / 2) {
      free(pos);
      or_model_free(&teacher);
      return OR_DOMAIN;
    }
    u64set seen;
    u64set_init(&seen, nnz);
    size_t have = 0;
    while (have < nnz) {
      const uint64_t p = or_next_below(&rng, total) + 1;
      if (u64set_insert(&seen, p)) pos[have++] = p;
    }
    u64set_free(&seen);
  }
  qsort(pos, nnz, sizeof(uint64_t), cmp_u64);
  /* plant (synth.cpp:49-67): invert_vec_index(mode 0) then teacher.predict */
  double* s = (double*)malloc(teacher.core_elems * sizeof(double));
  double* e = (double*)malloc(teacher.J[0] * sizeof(double));
  for (size_t i = 0; i < nnz; ++i) {
    uint32_t* c = coords_out + i * order;
    const uint64_t k0 = pos[i] - 1;
    c[0] = (uint32_t)(k0 % dims[0]) + 1;
    uint64_t j0 = k0 / dims[0];
    for (int q = 1; q < order; ++q) {
      c[q] = (uint32_t)(j0 % dims[q]) + 1;
      j0 /= dims[q];
    }
    values_out[i] = predict_ws(&teacher, c, s, e);
  }
  /* noise (synth.cpp:71-79) */
  for (size_t i = 0; i < nnz; ++i)
    values_out[i] =
        values_out[i] + (noise_stddev > 0.0 ? or_next_gaussian(&rng, 0.0, noise_stddev) : 0.0);
  free(s);
  free(e);
  free(pos);
  or_model_free(&teacher);
  return OR_OK;
}

int or_train_test_split_ids(size_t nnz, double test_fraction, uint64_t seed, uint32_t* ids,
                            size_t* ntest_out) {
  if (!(test_fraction > 0.0 && test_fraction < 1.0)) return OR_DOMAIN;
  const size_t ntest = (size_t)llround(test_fraction * (double)nnz);
  if (ntest == 0 || ntest == nnz) return OR_DOMAIN;
  for (size_t e = 0; e < nnz; ++e) ids[e] = (uint32_t)e;
  or_rng rng;
  or_rng_seed(&rng, seed);
  for (size_t i = 0; i + 1 < nnz; ++i) {
    const size_t j = i + (size_t)or_next_below(&rng, nnz - i);
    const uint32_t tmp = ids[i];
    ids[i] = ids[j];
    ids[j] = tmp;
  }
  qsort(ids, ntest, sizeof(uint32_t), cmp_u32);
  qsort(ids + ntest, nnz - ntest, sizeof(uint32_t), cmp_u32);
  *ntest_out = ntest;
  return OR_OK;
}
