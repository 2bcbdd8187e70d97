/*
 * nsk_oracle.c -- CPU restatement of the reference's random draws and of the
 * sketch applications that have no third-party transform in them.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or as the CPU baseline.  The product path
 * (paper_2206_00975_b200/) never links or calls it.
 *
 * Parity pin: every integer draw below is checked bit-for-bit against the
 * reference's own header /root/reference/proj/include/nullsketch/rng.hpp,
 * compiled unmodified into oracle/_ref/ (see oracle/Makefile and
 * tests/golden/make_golden.py); the fixtures it produced live in tests/golden/.
 *
 * Reference functions restated (file:line relative to /root/reference):
 *   splitmix / key derivation      proj/include/nullsketch/rng.hpp:19-23,66-71
 *   Philox4x32-10 refill           proj/include/nullsketch/rng.hpp:73-96
 *   next_u64 / next_double         proj/include/nullsketch/rng.hpp:30-39
 *   next_gaussian (Box-Muller)     proj/include/nullsketch/rng.hpp:42-54
 *   next_sign                      proj/include/nullsketch/rng.hpp:57
 *   next_below                     proj/include/nullsketch/rng.hpp:60-63
 *   sample_without_replacement     proj/include/nullsketch/rng.hpp:108-121
 *   SketchOperator::draw           proj/src/sketch.cpp:103-128
 *   apply, gaussian branch         proj/src/sketch.cpp:195-205
 *
 * Random-access form: the reference consumes its stream sequentially, four
 * u32 words per Philox block, counter = block index.  So u32 word i is word
 * (i & 3) of block (i >> 2), and Gaussian number L (pairs are cached, cos
 * first) is built from block L >> 1: u1 from words 0,1 and u2 from words 2,3.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

void nsko_key(uint64_t seed, uint64_t stream, uint32_t key[2]) {
  uint64_t k = splitmix(seed) ^ splitmix(stream ^ 0xb5ad4eceda1ce2a9ULL);
  key[0] = (uint32_t)k;
  key[1] = (uint32_t)(k >> 32);
}

void nsko_philox(const uint32_t key[2], uint64_t ctr, uint32_t out[4]) {
  uint32_t c0 = (uint32_t)ctr, c1 = (uint32_t)(ctr >> 32), c2 = 0, c3 = 0;
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = 0xD2511F53ULL * c0, p1 = 0xCD9E8D57ULL * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint32_t nsko_word(const uint32_t key[2], uint64_t i) {
  uint32_t b[4];
  nsko_philox(key, i >> 2, b);
  return b[i & 3];
}

static uint64_t word_u64(const uint32_t key[2], uint64_t lo_word) {
  uint64_t lo = nsko_word(key, lo_word), hi = nsko_word(key, lo_word + 1);
  return (hi << 32) | lo;
}

double nsko_gaussian(const uint32_t key[2], uint64_t L) {
  uint32_t b[4];
  nsko_philox(key, L >> 1, b);
  uint64_t a = ((uint64_t)b[1] << 32) | b[0];
  uint64_t c = ((uint64_t)b[3] << 32) | b[2];
  double u1 = 1.0 - (double)(a >> 11) * 0x1.0p-53;
  double u2 = (double)(c >> 11) * 0x1.0p-53;
  double r = sqrt(-2.0 * log(u1));
  double t = 2.0 * M_PI * u2;
  return (L & 1) ? r * sin(t) : r * cos(t);
}

/* Bulk helpers (ctypes-friendly). */
void nsko_words(uint64_t seed, uint64_t stream, uint64_t first, uint64_t count, uint32_t* out) {
  uint32_t key[2];
  nsko_key(seed, stream, key);
  for (uint64_t i = 0; i < count; ++i) out[i] = nsko_word(key, first + i);
}

void nsko_gaussians(uint64_t seed, uint64_t stream, uint64_t first, uint64_t count, double* out) {
  uint32_t key[2];
  nsko_key(seed, stream, key);
  for (uint64_t i = 0; i < count; ++i) out[i] = nsko_gaussian(key, first + i);
}

/* Rademacher signs D: word i of stream (seed, 0), bit 0 set -> +1 (sketch.cpp:123-124). */
void nsko_signs(uint64_t seed, int64_t m, double* signs) {
  uint32_t key[2];
  nsko_key(seed, 0, key);
  for (int64_t i = 0; i < m; ++i) signs[i] = (nsko_word(key, (uint64_t)i) & 1u) ? 1.0 : -1.0;
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* Fisher-Yates sample of s indices out of m after the m sign words
 * (sketch.cpp:122-126, rng.hpp:108-121).  O(m) scratch, exactly as the
 * reference does it. Returns 0 on success. */
int nsko_sample_indices(uint64_t seed, int64_t m, int64_t s, int64_t* idx_out) {
  if (s < 0 || s > m) return -1;
  uint32_t key[2];
  nsko_key(seed, 0, key);
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  if (!idx) return -2;
  for (int64_t i = 0; i < m; ++i) idx[i] = i;
  for (int64_t i = 0; i < s; ++i) {
    uint64_t u = word_u64(key, (uint64_t)m + 2u * (uint64_t)i);
    uint64_t n = (uint64_t)(m - i);
    uint64_t below = (uint64_t)(((unsigned __int128)u * n) >> 64);
    int64_t j = i + (int64_t)below;
    int64_t t = idx[i]; idx[i] = idx[j]; idx[j] = t;
  }
  memcpy(idx_out, idx, sizeof(int64_t) * (size_t)s);
  free(idx);
  qsort(idx_out, (size_t)s, sizeof(int64_t), cmp_i64);
  return 0;
}

/* CountSketch draw protocol (no reference implementation exists; SPEC.md:210
 * lists CountSketch as a non-goal).  Defined here as the sequence a reference
 * caller would issue on stream (seed, 0): m x next_sign(), then
 * m x next_below(s) -- so sign(i) = word i, bucket(i) = below(s) of the u64
 * (word m+2i+1 : word m+2i). */
void nsko_countsketch_draw(uint64_t seed, int64_t m, int64_t s, int32_t* bucket, double* sign) {
  uint32_t key[2];
  nsko_key(seed, 0, key);
  for (int64_t i = 0; i < m; ++i) {
    sign[i] = (nsko_word(key, (uint64_t)i) & 1u) ? 1.0 : -1.0;
    uint64_t u = word_u64(key, (uint64_t)m + 2u * (uint64_t)i);
    bucket[i] = (int32_t)(((unsigned __int128)u * (uint64_t)s) >> 64);
  }
}

/* CountSketch apply: SA[h(i), c] += sign(i) * A[i, c], rows in increasing order. */
void nsko_countsketch_apply(uint64_t seed, int64_t s, int64_t m, int64_t n, const double* A,
                            int64_t lda, double* SA, int64_t ldsa) {
  uint32_t key[2];
  nsko_key(seed, 0, key);
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < s; ++r) SA[r + c * ldsa] = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    double sg = (nsko_word(key, (uint64_t)i) & 1u) ? 1.0 : -1.0;
    uint64_t u = word_u64(key, (uint64_t)m + 2u * (uint64_t)i);
    int64_t h = (int64_t)(((unsigned __int128)u * (uint64_t)s) >> 64);
    for (int64_t c = 0; c < n; ++c) SA[h + c * ldsa] += sg * A[i + c * lda];
  }
}

/* Materialise rows [j0, j1) of G^T (i.e. columns j0..j1-1 of the s x m Gaussian
 * G), column-major G block of shape s x (j1-j0): out[i + (j-j0)*s] = G(i, j) =
 * Gaussian #(j*s + i) of stream (seed, 0)  (sketch.cpp:117-121). */
typedef struct {
  uint32_t key[2];
  int64_t s, j0, j1;
  double* out;
} gblock_job;

static void* gblock_worker(void* p) {
  gblock_job* jb = (gblock_job*)p;
  for (int64_t j = jb->j0; j < jb->j1; ++j)
    for (int64_t i = 0; i < jb->s; ++i) {
      uint64_t L = (uint64_t)j * (uint64_t)jb->s + (uint64_t)i;
      jb->out[(size_t)((j - jb->j0) * jb->s + i)] = nsko_gaussian(jb->key, L);
    }
  return NULL;
}

void nsko_gaussian_block(uint64_t seed, uint64_t stream, int64_t s, int64_t j0, int64_t j1,
                         double* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  int64_t cols = j1 - j0;
  if (cols <= 0) return;
  if (nthreads > cols) nthreads = (int)cols;
  pthread_t th[256];
  gblock_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    nsko_key(seed, stream, jobs[t].key);
    jobs[t].s = s;
    jobs[t].j0 = j0 + cols * t / nthreads;
    jobs[t].j1 = j0 + cols * (t + 1) / nthreads;
    jobs[t].out = out + (size_t)((jobs[t].j0 - j0) * s);
    pthread_create(&th[t], NULL, gblock_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* In-place unnormalised fast Walsh-Hadamard transform (Sylvester order) of
 * one length-2^p vector: y[r] = sum_j (-1)^popcount(r & j) x[j]. */
void nsko_fwht(double* x, int64_t len) {
  for (int64_t h = 1; h < len; h <<= 1)
    for (int64_t i = 0; i < len; i += h << 1)
      for (int64_t j = i; j < i + h; ++j) {
        double a = x[j], b = x[j + h];
        x[j] = a + b;
        x[j + h] = a - b;
      }
}

/* SRHT apply (no reference implementation; same draw protocol as srdct):
 * SA = sqrt(m/s) R H_m D A with H_m the normalised Hadamard matrix, so
 * SA[r, c] = (1/sqrt s) * sum_j (-1)^popcount(idx_r & j) d_j A[j, c].
 * Columns [c0, c1) only (lets the CPU baseline time a bounded sample). */
typedef struct {
  const double* A; int64_t lda; double* SA; int64_t ldsa;
  const double* signs; const int64_t* idx; int64_t m, s, c0, c1;
} srht_job;

static void* srht_worker(void* p) {
  srht_job* jb = (srht_job*)p;
  double* buf = (double*)malloc(sizeof(double) * (size_t)jb->m);
  const double scale = 1.0 / sqrt((double)jb->s);
  for (int64_t c = jb->c0; c < jb->c1; ++c) {
    const double* a = jb->A + c * jb->lda;
    for (int64_t j = 0; j < jb->m; ++j) buf[j] = jb->signs[j] * a[j];
    nsko_fwht(buf, jb->m);
    for (int64_t r = 0; r < jb->s; ++r) jb->SA[r + c * jb->ldsa] = scale * buf[jb->idx[r]];
  }
  free(buf);
  return NULL;
}

void nsko_srht_apply(const double* signs, const int64_t* idx, int64_t s, int64_t m, int64_t n,
                     const double* A, int64_t lda, double* SA, int64_t ldsa, int64_t c0,
                     int64_t c1, int nthreads) {
  (void)n;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  int64_t cols = c1 - c0;
  if (cols <= 0) return;
  if (nthreads > cols) nthreads = (int)cols;
  pthread_t th[256];
  srht_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    srht_job j = {A, lda, SA, ldsa, signs, idx, m, s, c0 + cols * t / nthreads,
                  c0 + cols * (t + 1) / nthreads};
    jobs[t] = j;
    pthread_create(&th[t], NULL, srht_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* Rows `rows[0..nr)` of the s x m Gaussian G over the column range [j0, j1):
 * out[r + (j - j0) * nr] = G(rows[r], j) = Gaussian #(j*s + rows[r]) of stream
 * (seed, stream) (sketch.cpp:117-121).  Random access into the counter stream,
 * so a row sample of G costs nr * (j1 - j0) draws instead of s * (j1 - j0);
 * threads split the column range. */
typedef struct {
  uint32_t key[2];
  int64_t s, nr, j0, j1, jbase;
  const int64_t* rows;
  double* out;
} grows_job;

static void* grows_worker(void* p) {
  grows_job* jb = (grows_job*)p;
  for (int64_t j = jb->j0; j < jb->j1; ++j)
    for (int64_t r = 0; r < jb->nr; ++r) {
      uint64_t L = (uint64_t)j * (uint64_t)jb->s + (uint64_t)jb->rows[r];
      jb->out[(size_t)((j - jb->jbase) * jb->nr + r)] = nsko_gaussian(jb->key, L);
    }
  return NULL;
}

void nsko_gaussian_rows(uint64_t seed, uint64_t stream, int64_t s, const int64_t* rows, int64_t nr,
                        int64_t j0, int64_t j1, double* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  int64_t cols = j1 - j0;
  if (cols <= 0) return;
  if (nthreads > cols) nthreads = (int)cols;
  pthread_t th[256];
  grows_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    nsko_key(seed, stream, jobs[t].key);
    jobs[t].s = s;
    jobs[t].nr = nr;
    jobs[t].rows = rows;
    jobs[t].jbase = j0;
    jobs[t].j0 = j0 + cols * t / nthreads;
    jobs[t].j1 = j0 + cols * (t + 1) / nthreads;
    jobs[t].out = out;
    pthread_create(&th[t], NULL, grows_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* CountSketch apply with the draw tables precomputed (nsko_countsketch_draw),
 * threads over column ranges; within a column the rows are added in increasing
 * order, exactly as nsko_countsketch_apply does. */
typedef struct {
  const int32_t* bucket; const double* sign; const double* A; double* SA;
  int64_t s, m, lda, ldsa, c0, c1;
} csmt_job;

static void* csmt_worker(void* p) {
  csmt_job* jb = (csmt_job*)p;
  for (int64_t c = jb->c0; c < jb->c1; ++c) {
    double* out = jb->SA + c * jb->ldsa;
    const double* a = jb->A + c * jb->lda;
    for (int64_t r = 0; r < jb->s; ++r) out[r] = 0.0;
    for (int64_t i = 0; i < jb->m; ++i) out[jb->bucket[i]] += jb->sign[i] * a[i];
  }
  return NULL;
}

void nsko_countsketch_apply_tables(const int32_t* bucket, const double* sign, int64_t s, int64_t m,
                                   int64_t n, const double* A, int64_t lda, double* SA, int64_t ldsa,
                                   int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (n <= 0) return;
  if (nthreads > n) nthreads = (int)n;
  pthread_t th[256];
  csmt_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    csmt_job j = {bucket, sign, A, SA, s, m, lda, ldsa, n * t / nthreads, n * (t + 1) / nthreads};
    jobs[t] = j;
    pthread_create(&th[t], NULL, csmt_worker, &jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}
