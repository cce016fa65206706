/*
 * skt_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference's CountSketch (sparse embedding)
 * hot path, used as the parity checker for the sm_100a kernels.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  The product path (paper_1207_6365_b200/) never
 * links or calls it.
 *
 * Reference being restated (paths relative to /root/reference/pkg/src/sketchnla):
 *   sketch.py:51-53     _rng(seed, *stream) = default_rng(SeedSequence(seed, spawn_key=stream))
 *   sketch.py:147       bucket = _rng(seed,0,0).integers(0, t, size=n)
 *   sketch.py:148       sign   = _rng(seed,0,1).choice([-1.0, 1.0], size=n)
 *   sketch.py:149-151   _mat   = csr_array((sign, (bucket, arange(n))), (t, n))
 *   sketch.py:155-164   apply, CSR branch  (np.bincount scatter, nnz order)
 *   sketch.py:165       apply, dense branch (scipy csr_matvecs, bucket-major)
 *   sketch.py:445-448   apply_right(A, S) = (S.apply(A.T)).T
 *   leverage.py:87-91   rows = A @ probe ; scores = einsum('ij,ij->i')
 *
 * The random-number algorithms live in numpy (third-party, not vendored under
 * /root/reference; measured here with numpy 2.3.5):
 *   - numpy.random.SeedSequence (bit_generator.pyx): hashmix / mix entropy pool
 *     of 4 uint32 words, generate_state().
 *   - PCG64 (pcg64.h, "XSL-RR 128/64"): 128-bit LCG, output of the NEW state,
 *     seeding pcg_setseq_128_srandom_r.
 *   - next_uint32: each 64-bit output yields its low half first, then its high half.
 *   - Generator.integers, 32-bit bounded path: Lemire multiply-shift with
 *     rejection threshold (2^32 - t) % t; t == 1 consumes no draws;
 *     t == 2^32 returns raw draws.
 *   - Generator.choice(2 items) == integers(0, 2): the top bit of each draw.
 * Parity of this restatement is pinned against the reference itself by
 * tests/golden/make_golden.py (run in the build container with the reference
 * importable) and tests/test_oracle.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---------------- numpy SeedSequence (bit_generator.pyx) ---------------- */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u
#define SS_POOL 4

static uint32_t ss_hashmix(uint32_t v, uint32_t *hc) {
  v ^= *hc;
  *hc *= SS_MULT_A;
  v *= *hc;
  v ^= v >> 16;
  return v;
}
static uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> 16;
  return r;
}

/* entropy: run entropy words (little-endian 32-bit words of the int seed);
 * spawn: spawn-key words (each key element < 2^32 here). */
int oracle_seedseq_generate(const uint32_t *entropy, int n_entropy,
                            const uint32_t *spawn, int n_spawn,
                            uint32_t *out, int n_out) {
  uint32_t assembled[64];
  int n = 0;
  if (n_entropy + n_spawn + SS_POOL > 64) return -1;
  for (int i = 0; i < n_entropy; ++i) assembled[n++] = entropy[i];
  if (n_spawn > 0)
    while (n < SS_POOL) assembled[n++] = 0u; /* pad run entropy to pool size */
  for (int i = 0; i < n_spawn; ++i) assembled[n++] = spawn[i];

  uint32_t pool[SS_POOL];
  uint32_t hc = SS_INIT_A;
  for (int i = 0; i < SS_POOL; ++i)
    pool[i] = ss_hashmix(i < n ? assembled[i] : 0u, &hc);
  for (int s = 0; s < SS_POOL; ++s)
    for (int d = 0; d < SS_POOL; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  for (int s = SS_POOL; s < n; ++s)
    for (int d = 0; d < SS_POOL; ++d)
      pool[d] = ss_mix(pool[d], ss_hashmix(assembled[s], &hc));

  uint32_t hb = SS_INIT_B;
  for (int i = 0; i < n_out; ++i) {
    uint32_t v = pool[i % SS_POOL];
    v ^= hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> 16;
    out[i] = v;
  }
  return 0;
}

/* ---------------- PCG64 (XSL-RR 128/64) ---------------- */
static const u128 PCG_MULT =
    (((u128)0x2360ED051FC65DA4ull) << 64) | (u128)0x4385DF649FCCF645ull;

typedef struct {
  u128 state, inc;
  int has32;
  uint32_t buf32;
} opcg;

static inline uint64_t opcg_next64(opcg *g) {
  g->state = g->state * PCG_MULT + g->inc;
  uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
  unsigned rot = (unsigned)(g->state >> 122);
  uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
static inline uint32_t opcg_next32(opcg *g) {
  if (g->has32) {
    g->has32 = 0;
    return g->buf32;
  }
  uint64_t v = opcg_next64(g);
  g->has32 = 1;
  g->buf32 = (uint32_t)(v >> 32);
  return (uint32_t)v;
}

/* PCG64(SeedSequence(...)): val = generate_state(4, uint64); seed = val[0]:val[1],
 * inc = val[2]:val[3]; pcg_setseq_128_srandom_r. Outputs state/inc as hi/lo words. */
int oracle_pcg64_seed(const uint32_t *entropy, int n_entropy, const uint32_t *spawn,
                      int n_spawn, uint64_t out[4]) {
  uint32_t w[8];
  if (oracle_seedseq_generate(entropy, n_entropy, spawn, n_spawn, w, 8)) return -1;
  uint64_t v[4];
  for (int i = 0; i < 4; ++i) v[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  u128 initstate = ((u128)v[0] << 64) | v[1];
  u128 initseq = ((u128)v[2] << 64) | v[3];
  u128 inc = (initseq << 1) | 1u;
  u128 st = 0;
  st = st * PCG_MULT + inc;
  st += initstate;
  st = st * PCG_MULT + inc;
  out[0] = (uint64_t)(st >> 64);
  out[1] = (uint64_t)st;
  out[2] = (uint64_t)(inc >> 64);
  out[3] = (uint64_t)inc;
  return 0;
}

static void opcg_load(opcg *g, const uint64_t s[4]) {
  g->state = ((u128)s[0] << 64) | s[1];
  g->inc = ((u128)s[2] << 64) | s[3];
  g->has32 = 0;
  g->buf32 = 0;
}

/* n 64-bit outputs (used to pin the raw generator against numpy.random_raw). */
void oracle_pcg64_raw(const uint64_t s[4], int64_t n, uint64_t *out) {
  opcg g;
  opcg_load(&g, s);
  for (int64_t i = 0; i < n; ++i) out[i] = opcg_next64(&g);
}

/* bucket[i] (sketch.py:147) and sign (sketch.py:148), int32-packed. */
int oracle_hash_signs(const uint64_t hs[4], const uint64_t ss[4], int64_t n, uint64_t t,
                      uint32_t *h, int8_t *s) {
  if (n < 0 || t < 1 || t > (1ull << 32)) return -1;
  opcg g;
  opcg_load(&g, hs);
  if (t == 1) {
    memset(h, 0, (size_t)n * sizeof(uint32_t));
  } else if (t == (1ull << 32)) {
    for (int64_t i = 0; i < n; ++i) h[i] = opcg_next32(&g);
  } else {
    uint32_t te = (uint32_t)t;
    uint32_t thr = (uint32_t)((0x100000000ull - t) % t);
    for (int64_t i = 0; i < n; ++i) {
      uint64_t m = (uint64_t)opcg_next32(&g) * te;
      uint32_t left = (uint32_t)m;
      if (left < te)
        while (left < thr) {
          m = (uint64_t)opcg_next32(&g) * te;
          left = (uint32_t)m;
        }
      h[i] = (uint32_t)(m >> 32);
    }
  }
  if (s) {
    opcg_load(&g, ss);
    for (int64_t i = 0; i < n; ++i) s[i] = (opcg_next32(&g) >> 31) ? 1 : -1;
  }
  return 0;
}

/* S as t x n CSR (sketch.py:149-151): stable counting sort by bucket. */
void oracle_plan(const uint32_t *h, int64_t n, int64_t t, int64_t *indptr, int32_t *rows) {
  memset(indptr, 0, (size_t)(t + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) indptr[h[i] + 1]++;
  for (int64_t b = 0; b < t; ++b) indptr[b + 1] += indptr[b];
  int64_t *cur = (int64_t *)malloc((size_t)t * sizeof(int64_t));
  memcpy(cur, indptr, (size_t)t * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) rows[cur[h[i]]++] = (int32_t)i;
  free(cur);
}

/* Dense branch (sketch.py:165 via scipy csr_matvecs): for each bucket, rows
 * ascending, SA[b,:] += s_i * A[i,:] in fp64 from +0.0. A is row-major with
 * leading dimension lda; is_f32 selects float input (upcast, _validation.py:20). */
void oracle_apply_dense(const int64_t *indptr, const int32_t *rows, const int8_t *s,
                        int64_t t, const void *a, int is_f32, int64_t d, int64_t lda,
                        double *sa) {
  for (int64_t b = 0; b < t; ++b) {
    double *y = sa + b * d;
    for (int64_t j = 0; j < d; ++j) y[j] = 0.0;
    for (int64_t k = indptr[b]; k < indptr[b + 1]; ++k) {
      int64_t i = rows[k];
      double sg = (double)s[i];
      if (is_f32) {
        const float *x = (const float *)a + i * lda;
        for (int64_t j = 0; j < d; ++j) y[j] += sg * (double)x[j];
      } else {
        const double *x = (const double *)a + i * lda;
        for (int64_t j = 0; j < d; ++j) y[j] += sg * x[j];
      }
    }
  }
}

/* CSR branch (sketch.py:155-164): out[h(i)*d + j] += s(i)*v in stored nnz order. */
void oracle_apply_csr(const uint32_t *h, const int8_t *s, int64_t n, int64_t t,
                      const int64_t *indptr, const int32_t *indices, const void *vals,
                      int is_f32, int64_t d, double *sa) {
  memset(sa, 0, (size_t)(t * d) * sizeof(double));
  for (int64_t i = 0; i < n; ++i) {
    double sg = (double)s[i];
    double *y = sa + (int64_t)h[i] * d;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
      double v = is_f32 ? (double)((const float *)vals)[k] : ((const double *)vals)[k];
      y[indices[k]] += sg * v;
    }
  }
}

/* Leverage contraction (leverage.py:90-91): scores_i = sum_j (A_i . P_j)^2, fp64.
 * CSR A (n x d) times dense P (d x k, row-major). */
void oracle_lev_rownorms_csr(int64_t n, const int64_t *indptr, const int32_t *indices,
                             const void *vals, int is_f32, const double *p, int64_t k,
                             double *scores) {
  double *row = (double *)malloc((size_t)k * sizeof(double));
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t c = 0; c < k; ++c) row[c] = 0.0;
    for (int64_t q = indptr[i]; q < indptr[i + 1]; ++q) {
      double v = is_f32 ? (double)((const float *)vals)[q] : ((const double *)vals)[q];
      const double *pr = p + (int64_t)indices[q] * k;
      for (int64_t c = 0; c < k; ++c) row[c] += v * pr[c];
    }
    double acc = 0.0;
    for (int64_t c = 0; c < k; ++c) acc += row[c] * row[c];
    scores[i] = acc;
  }
  free(row);
}

/* ---------------- thread-parallel forms (same arithmetic) ----------------
 * Full-size parity (configs 3-5) and the reference arm run these on all host
 * cores.  Each output element keeps exactly the sequential order of the
 * functions above -- buckets (dense, CSR) or rows (contraction) are split
 * across threads, never the sum of one element -- so the results are
 * bit-identical to the scalar restatement. */
typedef struct {
  int64_t lo, hi;             /* bucket / row range of this thread */
  const int64_t *indptr;      /* plan (S in CSR) or CSR A */
  const int32_t *rows;        /* plan rows */
  const int8_t *s;
  const void *a;              /* dense A, or CSR values */
  const int64_t *a_indptr;    /* CSR A */
  const int32_t *a_indices;
  int is_f32;
  int64_t d, lda;
  const double *p;            /* contraction probe */
  int64_t k;
  double *out;
} mt_job;

static void *dense_worker(void *arg) {
  mt_job *j = (mt_job *)arg;
  int64_t cnt = j->hi - j->lo;
  if (cnt > 0) {
    /* buckets [lo, hi) of SA; the plan slice is rebased by pointer offset */
    oracle_apply_dense(j->indptr + j->lo, j->rows, j->s, cnt, j->a, j->is_f32, j->d, j->lda,
                       j->out + j->lo * j->d);
  }
  return NULL;
}

/* CSR branch by bucket: for bucket b, rows of b ascending (the plan), each
 * row's entries in stored order -- per output element the same sequence as
 * the nnz-order bincount of oracle_apply_csr. */
static void *csr_worker(void *arg) {
  mt_job *j = (mt_job *)arg;
  for (int64_t b = j->lo; b < j->hi; ++b) {
    double *y = j->out + b * j->d;
    for (int64_t c = 0; c < j->d; ++c) y[c] = 0.0;
    for (int64_t q = j->indptr[b]; q < j->indptr[b + 1]; ++q) {
      int64_t i = j->rows[q];
      double sg = (double)j->s[i];
      for (int64_t e = j->a_indptr[i]; e < j->a_indptr[i + 1]; ++e) {
        double v = j->is_f32 ? (double)((const float *)j->a)[e] : ((const double *)j->a)[e];
        y[j->a_indices[e]] += sg * v;
      }
    }
  }
  return NULL;
}

static void *lev_worker(void *arg) {
  mt_job *j = (mt_job *)arg;
  int64_t cnt = j->hi - j->lo;
  if (cnt > 0) {
    /* rows [lo, hi): indptr is absolute, so shift the row pointer only */
    oracle_lev_rownorms_csr(cnt, j->a_indptr + j->lo, j->a_indices, j->a, j->is_f32, j->p, j->k,
                            j->out + j->lo);
  }
  return NULL;
}

static int run_jobs(void *(*fn)(void *), mt_job *proto, int64_t units, int nthreads, const int64_t *weight) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (units < nthreads) nthreads = units > 0 ? (int)units : 1;
  pthread_t th[256];
  mt_job jobs[256];
  /* split by cumulative weight (rows per bucket / nnz per row) when given */
  int64_t total = weight ? weight[units] - weight[0] : units;
  int64_t lo = 0;
  for (int w = 0; w < nthreads; ++w) {
    int64_t hi;
    if (w == nthreads - 1) {
      hi = units;
    } else if (weight) {
      int64_t target = weight[0] + total * (w + 1) / nthreads;
      hi = lo;
      while (hi < units && weight[hi] < target) ++hi;
    } else {
      hi = units * (w + 1) / nthreads;
    }
    jobs[w] = *proto;
    jobs[w].lo = lo;
    jobs[w].hi = hi;
    lo = hi;
  }
  for (int w = 0; w < nthreads; ++w)
    if (pthread_create(&th[w], NULL, fn, &jobs[w]) != 0) return -1;
  for (int w = 0; w < nthreads; ++w) pthread_join(th[w], NULL);
  return 0;
}

int oracle_apply_dense_mt(const int64_t *indptr, const int32_t *rows, const int8_t *s, int64_t t,
                          const void *a, int is_f32, int64_t d, int64_t lda, double *sa, int nthreads) {
  mt_job j = {0};
  j.indptr = indptr; j.rows = rows; j.s = s; j.a = a; j.is_f32 = is_f32; j.d = d; j.lda = lda; j.out = sa;
  return run_jobs(dense_worker, &j, t, nthreads, indptr);
}

int oracle_apply_csr_mt(const int64_t *plan_indptr, const int32_t *plan_rows, const int8_t *s, int64_t t,
                        const int64_t *indptr, const int32_t *indices, const void *vals, int is_f32,
                        int64_t d, double *sa, int nthreads) {
  mt_job j = {0};
  j.indptr = plan_indptr; j.rows = plan_rows; j.s = s; j.a = vals; j.a_indptr = indptr;
  j.a_indices = indices; j.is_f32 = is_f32; j.d = d; j.out = sa;
  return run_jobs(csr_worker, &j, t, nthreads, plan_indptr);
}

int oracle_lev_rownorms_csr_mt(int64_t n, const int64_t *indptr, const int32_t *indices, const void *vals,
                               int is_f32, const double *p, int64_t k, double *scores, int nthreads) {
  mt_job j = {0};
  j.a_indptr = indptr; j.a_indices = indices; j.a = vals; j.is_f32 = is_f32; j.p = p; j.k = k; j.out = scores;
  return run_jobs(lev_worker, &j, n, nthreads, indptr);
}
