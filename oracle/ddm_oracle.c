/*
 * ddm_oracle.c -- TEST INFRASTRUCTURE ONLY (see ddm_oracle.h).
 *
 * CPU restatement of the reference dose path.  Compiled with
 * -ffp-contract=off like the reference (proj/CMakeLists.txt:10-12) so that
 * every double operation rounds exactly where the reference's does.
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).
 */
#define _GNU_SOURCE
#include "ddm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* 1 + ddm::Errc (include/ddm/error.hpp:8-25) */
enum {
  E_OK = 0,
  E_DuplicateEntry = 1,
  E_IndexOverflow = 2,
  E_ValueOverflow = 3,
  E_NanInput = 4,
  E_DimensionMismatch = 5,
  E_InvalidConfig = 6,
  E_ValidationFailure = 11,
  E_InconsistentProfile = 15,
};

/* ---------------------------------------------------------------- rng ---- */
/* include/ddm/rng.hpp:16-25 -- splitmix64 expansion of one seed word. */
void or_rng_seed(or_rng* r, uint64_t seed) {
  uint64_t z = seed;
  for (int i = 0; i < 4; ++i) {
    z += 0x9E3779B97F4A7C15ull;
    uint64_t x = z;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    r->s[i] = x ^ (x >> 31);
  }
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:27-37 -- xoshiro256** 1.0 */
uint64_t or_rng_next_u64(or_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

/* rng.hpp:40 */
double or_rng_next_double53(or_rng* r) { return (double)(or_rng_next_u64(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:43-54 -- Lemire multiply-shift with rejection. */
uint64_t or_rng_next_below(or_rng* r, uint64_t n) {
  unsigned __int128 m = (unsigned __int128)or_rng_next_u64(r) * n;
  uint64_t low = (uint64_t)m;
  if (low < n) {
    const uint64_t threshold = (0 - n) % n;
    while (low < threshold) {
      m = (unsigned __int128)or_rng_next_u64(r) * n;
      low = (uint64_t)m;
    }
  }
  return (uint64_t)(m >> 64);
}

/* rng.hpp:57-61 -- Box-Muller, cosine branch; u1 drawn before u2. */
double or_rng_next_normal(or_rng* r) {
  const double u1 = or_rng_next_double53(r);
  const double u2 = or_rng_next_double53(r);
  return sqrt(-2.0 * log1p(-u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* --------------------------------------------------------------- half ---- */
/* src/half.cpp:50-64 -- exact widening binary16 -> double. */
double or_decode_half(uint16_t h) {
  const unsigned sign = h >> 15;
  const unsigned exp_field = (h >> 10) & 0x1Fu;
  const unsigned mantissa = h & 0x3FFu;
  double mag;
  if (exp_field == 0)
    mag = ldexp((double)mantissa, -24);
  else if (exp_field == 31)
    mag = mantissa ? nan("") : HUGE_VAL;
  else
    mag = ldexp((double)(mantissa + 1024u), (int)exp_field - 25);
  return sign ? -mag : mag;
}

/* src/half.cpp:14-21 */
static uint32_t round_nearest_even_u32(double y) {
  double f = floor(y);
  double r = y - f;
  uint32_t q = (uint32_t)f;
  if (r > 0.5 || (r == 0.5 && (q & 1u))) ++q;
  return q;
}

/* src/half.cpp:23-48 -- RNE double -> binary16. */
int or_encode_half(double x, uint16_t* out) {
  if (isnan(x)) return E_NanInput;
  const uint16_t sign = signbit(x) ? 0x8000u : 0x0000u;
  const double a = fabs(x);
  if (a >= 65520.0) { *out = (uint16_t)(sign | 0x7C00u); return E_OK; }
  if (a == 0.0) { *out = sign; return E_OK; }
  int bin_exp = 0;
  frexp(a, &bin_exp);
  const int e = bin_exp - 1;
  uint16_t mag;
  if (e < -14) {
    mag = (uint16_t)round_nearest_even_u32(ldexp(a, 24));
  } else {
    const uint32_t q = round_nearest_even_u32(ldexp(a, 10 - e));
    mag = (uint16_t)(((uint32_t)(e + 15) << 10) + (q - 1024u));
  }
  *out = (uint16_t)(sign | mag);
  return E_OK;
}

/* ----------------------------------------------------------- checksum ---- */
/* include/ddm/checksum.hpp:14-21 */
uint64_t or_fnv1a64(const uint8_t* bytes, uint64_t n, uint64_t h) {
  for (uint64_t i = 0; i < n; ++i) {
    h ^= bytes[i];
    h *= 1099511628211ull;
  }
  return h;
}

/* checksum.hpp:25-35 -- each double fed LSB first. */
uint64_t or_checksum_bits(const double* v, uint64_t n) {
  uint64_t h = 14695981039346656037ull;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t u;
    memcpy(&u, &v[i], 8);
    for (int b = 0; b < 8; ++b) {
      h ^= (uint8_t)(u >> (8 * b));
      h *= 1099511628211ull;
    }
  }
  return h;
}

/* src/bench.cpp:31-36 */
void or_seeded_vector(uint64_t n, uint64_t seed, double* out) {
  or_rng r;
  or_rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = or_rng_next_double53(&r);
}

/* ------------------------------------------------------------- matgen ---- */
/* src/matgen.cpp:13-27 */
void or_liver_desk_profile(or_profile* p) {
  p->rows = 29700; p->cols = 6800; p->target_nnz_ratio = 0.0073; p->empty_row_fraction = 0.70;
  p->row_length_log_mean = 4.7661; p->row_length_log_sigma = 0.8278;
  p->locality_window = 4096; p->seed = 1;
}

/* src/matgen.cpp:29-43 */
void or_prostate_desk_profile(or_profile* p) {
  p->rows = 10300; p->cols = 5090; p->target_nnz_ratio = 0.0181; p->empty_row_fraction = 0.70;
  p->row_length_log_mean = 4.8880; p->row_length_log_sigma = 1.3165;
  p->locality_window = 4096; p->seed = 2;
}

/* src/matgen.cpp:96-126 */
int or_validate_profile(const or_profile* p) {
  if (p->rows < 1 || p->cols < 1) return E_InvalidConfig;
  if (!(p->target_nnz_ratio >= 0.0 && p->target_nnz_ratio <= 1.0)) return E_InvalidConfig;
  if (!(p->empty_row_fraction >= 0.0 && p->empty_row_fraction <= 1.0)) return E_InvalidConfig;
  if (!(p->row_length_log_sigma >= 0.0)) return E_InvalidConfig;
  if (p->locality_window < 1 || p->locality_window > p->cols) return E_InvalidConfig;
  double mean_len = exp(p->row_length_log_mean +
                        0.5 * p->row_length_log_sigma * p->row_length_log_sigma);
  if (mean_len < 1.0) mean_len = 1.0;
  if ((double)p->cols < mean_len) mean_len = (double)p->cols;
  const double expected_ratio = (1.0 - p->empty_row_fraction) * mean_len / (double)p->cols;
  if (p->target_nnz_ratio == 0.0)
    return p->empty_row_fraction != 1.0 ? E_InconsistentProfile : E_OK;
  if (p->empty_row_fraction == 1.0) return E_InconsistentProfile;
  const double deviation = fabs(expected_ratio - p->target_nnz_ratio) / p->target_nnz_ratio;
  return deviation > 0.10 ? E_InconsistentProfile : E_OK;
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

typedef struct { void* p; uint64_t n, cap; size_t elem; } vec_t;
static int vec_reserve(vec_t* v, uint64_t need) {
  if (need <= v->cap) return 0;
  uint64_t cap = v->cap ? v->cap : 1024;
  while (cap < need) cap *= 2;
  void* q = realloc(v->p, cap * v->elem);
  if (!q) return -1;
  v->p = q;
  v->cap = cap;
  return 0;
}

/* src/sparse.cpp:44-75 -- ValueStore::from_doubles. */
static int values_from_doubles(const double* xs, uint64_t n, int precision, void** out) {
  const size_t w = precision == OR_HALF ? 2 : precision == OR_SINGLE ? 4 : 8;
  void* buf = malloc(n ? n * w : 1);
  if (!buf) return E_ValidationFailure;
  for (uint64_t i = 0; i < n; ++i) {
    if (precision == OR_HALF) {
      uint16_t h;
      if (isinf(xs[i])) { free(buf); return E_ValueOverflow; }
      int rc = or_encode_half(xs[i], &h);
      if (rc) { free(buf); return rc; }
      if ((h & 0x7FFFu) == 0x7C00u) { free(buf); return E_ValueOverflow; }
      ((uint16_t*)buf)[i] = h;
    } else if (precision == OR_SINGLE) {
      if (isnan(xs[i])) { free(buf); return E_NanInput; }
      float f = (float)xs[i];
      if (isinf(f)) { free(buf); return E_ValueOverflow; }
      ((float*)buf)[i] = f;
    } else {
      if (isnan(xs[i])) { free(buf); return E_NanInput; }
      if (isinf(xs[i])) { free(buf); return E_ValueOverflow; }
      ((double*)buf)[i] = xs[i];
    }
  }
  *out = buf;
  return E_OK;
}

/* src/matgen.cpp:128-178 -- one sequential xoshiro stream; per row: empty
 * test, log-normal length, window centre, partial Fisher-Yates, sort, then
 * one value per entry in column order. */
int or_generate(const or_profile* p, int precision, int index_width, or_csr* out) {
  memset(out, 0, sizeof(*out));
  int rc = or_validate_profile(p);
  if (rc) return rc;
  const int width = index_width >= 0 ? index_width : (p->cols < 65536 ? OR_U16 : OR_U32);
  if (width == OR_U16 && p->cols >= 65536) return E_IndexOverflow;
  if (p->cols > 0xFFFFFFFFull) return E_IndexOverflow;

  or_rng rng;
  or_rng_seed(&rng, p->seed);
  uint64_t* row_ptr = (uint64_t*)calloc(p->rows + 1, 8);
  uint32_t* window = NULL;
  uint64_t window_cap = 0;
  vec_t cols = {NULL, 0, 0, 4}, vals = {NULL, 0, 0, 8};
  if (!row_ptr) return E_ValidationFailure;

  for (uint64_t r = 0; r < p->rows; ++r) {
    row_ptr[r + 1] = row_ptr[r];
    if (or_rng_next_double53(&rng) < p->empty_row_fraction) continue;
    const double raw_len = exp(p->row_length_log_mean +
                               p->row_length_log_sigma * or_rng_next_normal(&rng));
    uint64_t len = p->cols;
    if (raw_len < (double)p->cols) {
      long long l = llround(raw_len);
      len = (uint64_t)l < 1 ? 1 : (uint64_t)l;
    }
    const uint64_t center = or_rng_next_below(&rng, p->cols);
    const uint64_t span = p->locality_window > len ? p->locality_window : len;
    uint64_t lo = center > span / 2 ? center - span / 2 : 0;
    if (p->cols - span < lo) lo = p->cols - span;
    if (span > window_cap) {
      window_cap = span;
      window = (uint32_t*)realloc(window, span * 4);
    }
    for (uint64_t k = 0; k < span; ++k) window[k] = (uint32_t)(lo + k);
    for (uint64_t k = 0; k < len; ++k) {
      const uint64_t o = k + or_rng_next_below(&rng, span - k);
      uint32_t t = window[k]; window[k] = window[o]; window[o] = t;
    }
    qsort(window, len, 4, cmp_u32);
    if (vec_reserve(&cols, cols.n + len) || vec_reserve(&vals, vals.n + len)) {
      free(row_ptr); free(window); free(cols.p); free(vals.p);
      return E_ValidationFailure;
    }
    memcpy((uint32_t*)cols.p + cols.n, window, len * 4);
    cols.n += len;
    for (uint64_t k = 0; k < len; ++k)
      ((double*)vals.p)[vals.n++] = 0x1p-14 + (1.0 - 0x1p-14) * or_rng_next_double53(&rng);
    row_ptr[r + 1] += len;
  }
  free(window);
  void* values = NULL;
  rc = values_from_doubles((const double*)vals.p, vals.n, precision, &values);
  free(vals.p);
  if (rc) { free(row_ptr); free(cols.p); return rc; }
  out->rows = p->rows;
  out->cols = p->cols;
  out->nnz = row_ptr[p->rows];
  out->precision = precision;
  out->index_width = width;
  out->row_ptr = row_ptr;
  out->col = cols.p ? (uint32_t*)cols.p : (uint32_t*)calloc(1, 4);
  out->values = values;
  return E_OK;
}

void or_csr_free(or_csr* m) {
  free(m->row_ptr); free(m->col); free(m->values);
  memset(m, 0, sizeof(*m));
}

/* ------------------------------------------------------------ validate ---- */
static inline double widen(const or_csr* m, uint64_t j) {
  /* include/ddm/sparse.hpp:34-36 */
  switch (m->precision) {
    case OR_HALF: return or_decode_half(((const uint16_t*)m->values)[j]);
    case OR_SINGLE: return (double)((const float*)m->values)[j];
    default: return ((const double*)m->values)[j];
  }
}

/* src/sparse.cpp:197-255 -- 0 when every invariant holds. */
int or_validate(const or_csr* m) {
  if (!m->row_ptr) return E_ValidationFailure;
  if (m->row_ptr[0] != 0) return E_ValidationFailure;
  for (uint64_t r = 0; r < m->rows; ++r)
    if (m->row_ptr[r + 1] < m->row_ptr[r]) return E_ValidationFailure;
  if (m->row_ptr[m->rows] != m->nnz) return E_ValidationFailure;
  if (m->index_width == OR_U16 && m->cols >= 65536) return E_ValidationFailure;
  for (uint64_t r = 0; r < m->rows; ++r)
    for (uint64_t j = m->row_ptr[r]; j < m->row_ptr[r + 1]; ++j) {
      if (m->col[j] >= m->cols) return E_ValidationFailure;
      if (j > m->row_ptr[r] && m->col[j] <= m->col[j - 1]) return E_ValidationFailure;
    }
  for (uint64_t j = 0; j < m->nnz; ++j)
    if (!isfinite(widen(m, j))) return E_ValidationFailure;
  return E_OK;
}

/* ---------------------------------------------------------------- spmv ---- */
/* src/spmv.cpp:82-96 -- sequential row-major, left-to-right fp64. */
int or_spmv_oracle(const or_csr* m, const double* x, uint64_t x_len, double* y) {
  if (x_len != m->cols) return E_DimensionMismatch; /* spmv.cpp:34-38 */
  for (uint64_t i = 0; i < m->rows; ++i) {
    double acc = 0.0;
    for (uint64_t j = m->row_ptr[i]; j < m->row_ptr[i + 1]; ++j) acc += widen(m, j) * x[m->col[j]];
    y[i] = acc;
  }
  return E_OK;
}

/* src/spmv.cpp:48-68 -- lane l sums positions start+l, start+l+L, ... from
 * +0.0, then partial[l] += partial[l+w] for w = L/2 .. 1; empty rows keep 0. */
static void rowchunk_rows(const or_csr* m, const double* x, uint64_t L, double* y, uint64_t b,
                          uint64_t e) {
  double partial[1024];
  for (uint64_t i = b; i < e; ++i) {
    const uint64_t start = m->row_ptr[i], end = m->row_ptr[i + 1];
    if (start == end) continue;
    for (uint64_t l = 0; l < L; ++l) {
      double acc = 0.0;
      for (uint64_t j = start + l; j < end; j += L) acc += widen(m, j) * x[m->col[j]];
      partial[l] = acc;
    }
    for (uint64_t w = L / 2; w >= 1; w /= 2)
      for (uint64_t l = 0; l < w; ++l) partial[l] += partial[l + w];
    y[i] = partial[0];
  }
}

typedef struct { const or_csr* m; const double* x; uint64_t L; double* y; uint64_t b, e; } rc_job;
static void* rc_thread(void* arg) {
  rc_job* j = (rc_job*)arg;
  rowchunk_rows(j->m, j->x, j->L, j->y, j->b, j->e);
  return NULL;
}

/* src/spmv.cpp:98-111 with parallel_blocks (spmv.cpp:17-32): equal row-count
 * blocks; output bits never depend on workers. */
int or_spmv_rowchunk(const or_csr* m, const double* x, uint64_t x_len, uint64_t L,
                     uint64_t workers, double* y) {
  if (x_len != m->cols) return E_DimensionMismatch;
  if (L < 1 || L > 1024 || (L & (L - 1))) return E_InvalidConfig; /* spmv.cpp:40-46 */
  if (workers < 1) return E_InvalidConfig;
  for (uint64_t i = 0; i < m->rows; ++i) y[i] = 0.0;
  const uint64_t n = m->rows;
  if (workers <= 1 || n <= 1) {
    rowchunk_rows(m, x, L, y, 0, n);
    return E_OK;
  }
  const uint64_t used = workers < n ? workers : n;
  pthread_t* th = (pthread_t*)malloc(used * sizeof(pthread_t));
  rc_job* jobs = (rc_job*)malloc(used * sizeof(rc_job));
  for (uint64_t w = 0; w < used; ++w) {
    jobs[w] = (rc_job){m, x, L, y, n * w / used, n * (w + 1) / used};
    pthread_create(&th[w], NULL, rc_thread, &jobs[w]);
  }
  for (uint64_t w = 0; w < used; ++w) pthread_join(th[w], NULL);
  free(th);
  free(jobs);
  return E_OK;
}

/* src/perf_model.cpp:45-54 (TrafficModel::total_bytes, perf_model.hpp:38). */
uint64_t or_traffic_bytes(uint64_t nr, uint64_t nc, uint64_t nnz, uint32_t vb, uint32_t ib,
                          uint32_t rp, uint32_t ob, uint32_t inb) {
  return (uint64_t)(vb + ib) * nnz + (uint64_t)(rp + ob) * nr + (uint64_t)inb * nc;
}
