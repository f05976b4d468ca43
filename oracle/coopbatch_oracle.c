/*
 * TEST INFRASTRUCTURE ONLY — the CPU checker, never the product path.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load it.
 *
 * Plain-C restatement of the reference's sample + dedup + exchange + feature
 * path (/root/reference/proj, "coopbatch"). Each function names the
 * reference file:line it follows. Build: oracle/Makefile, with
 * -O2 -ffp-contract=off and no -march (the reference's own flags contain no
 * -march, so its FP64 is never contracted into FMA; SURVEY.md §7 hard part 2).
 *
 * Parity status: pinned against the reference compiled from its own sources
 * (oracle/_ref, tests/test_oracle_vs_reference.py) and the golden vectors in
 * tests/golden/ generated from it (tests/golden/make_golden.py).
 */
#include "coopbatch_oracle.h"

#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return 1;
}

const char* ob_last_error(void) { return g_err; }
void ob_free(void* p) { free(p); }

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n);
    abort();
  }
  return p;
}

/* ------------------------------------------------------------------ rng --- */

/* rng.hpp:17-22 SplitMix64 finalizer */
uint64_t ob_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

#define OB_SALT 0x736f6d6570736575ULL /* rng.hpp:24 */
static inline uint64_t hinit(uint64_t seed) { return ob_mix64(seed ^ OB_SALT); }
static inline uint64_t hstep(uint64_t h, uint64_t id) { return ob_mix64(h ^ id); }
static inline double ufb(uint64_t bits) { /* rng.hpp:42-44 */
  return (double)(bits >> 11) * 0x1.0p-53;
}

/* rng.hpp:34-39 */
uint64_t ob_hash_bits(uint64_t seed, const uint64_t* ids, int n_ids) {
  uint64_t h = hinit(seed);
  for (int i = 0; i < n_ids; ++i) h = hstep(h, ids[i]);
  return h;
}
double ob_hash_uniform(uint64_t seed, const uint64_t* ids, int n_ids) {
  return ufb(ob_hash_bits(seed, ids, n_ids));
}
static uint64_t hb2(uint64_t seed, uint64_t a, uint64_t b) {
  return hstep(hstep(hinit(seed), a), b);
}

/* rng.cpp:7-11 (the reference throws on non-finite input; NaN never reaches
 * here on the sampling path because normals are finite) */
double ob_phi(double x) { return 0.5 * erfc(-x * 0.7071067811865475244); }

/* rng.cpp:15-52 Acklam + one Halley step; same constants, same evaluation
 * order (no contraction: -ffp-contract=off). */
double ob_inverse_phi(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                             -2.759285104469687e+02, 1.383577518672690e+02,
                             -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                             -1.556989798598866e+02, 6.680131188771972e+01,
                             -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                             -2.400758277161838e+00, -2.549732539343734e+00,
                             4.374664141464968e+00,  2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01,
                             2.445134137142996e+00, 3.754408661907416e+00};
  const double plow = 0.02425;
  double x;
  if (p < plow) {
    const double q = sqrt(-2.0 * log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else if (p <= 1.0 - plow) {
    const double q = p - 0.5;
    const double r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  } else {
    const double q = sqrt(-2.0 * log1p(-p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  const double e = ob_phi(x) - p;
  const double u = e * sqrt(2.0 * 3.14159265358979323846) * exp(0.5 * x * x);
  x = x - u / (1.0 + 0.5 * x * u);
  return x;
}

/* rng.hpp:54-56 */
static double normal_from_bits(uint64_t bits) {
  return ob_inverse_phi(((double)(bits >> 11) + 0.5) * 0x1.0p-53);
}

#define OB_KAPPA_INF UINT64_MAX /* rng.hpp:70-71 */

/* rng.cpp:69-77 */
void ob_sched_make(uint64_t kappa, uint64_t root, ob_sched* s) {
  s->kappa = kappa;
  s->z1 = hb2(root, 12, 1);
  s->z2 = hb2(root, 12, 2);
  s->iteration = 0;
}
/* rng.cpp:79-86 */
void ob_sched_advance(ob_sched* s) {
  s->iteration += 1;
  if (s->kappa != OB_KAPPA_INF && s->iteration % s->kappa == 0) {
    s->z1 = s->z2;
    s->z2 = hb2(s->z2, 12, s->iteration);
  }
}

double ob_normal_from_bits(uint64_t bits) { return normal_from_bits(bits); }

/* samplers.hpp:53-126 VariateSource */
typedef struct {
  uint64_t z1, z2;
  int smoothed;
  double cos_c, sin_c;
} vsrc;

static vsrc vsrc_from(const ob_sched* s) {
  vsrc v;
  v.z1 = s->z1;
  v.z2 = s->z2;
  double c = 0.0; /* rng.hpp:99-102 */
  if (s->kappa != OB_KAPPA_INF)
    c = (double)(s->iteration % s->kappa) / (double)s->kappa;
  v.smoothed = s->kappa != OB_KAPPA_INF && s->kappa >= 2; /* rng.hpp:106-110 */
  if (c == 0.0) {
    v.cos_c = 1.0;
    v.sin_c = 0.0;
  } else if (c == 1.0) {
    v.cos_c = 0.0;
    v.sin_c = 1.0;
  } else {
    const double angle = c * 1.5707963267948966192;
    v.cos_c = cos(angle);
    v.sin_c = sin(angle);
  }
  return v;
}

typedef struct { uint64_t h1, h2; } vpfx;

static vpfx vsrc_prefix(const vsrc* v, const uint64_t* ids, int n) {
  vpfx p = {hinit(v->z1), 0};
  for (int i = 0; i < n; ++i) p.h1 = hstep(p.h1, ids[i]);
  if (v->smoothed) {
    p.h2 = hinit(v->z2);
    for (int i = 0; i < n; ++i) p.h2 = hstep(p.h2, ids[i]);
  }
  return p;
}

/* samplers.hpp:96-100 */
static double vsrc_finish(const vsrc* v, uint64_t b1, uint64_t b2) {
  if (!v->smoothed) return ufb(b1);
  const double n = v->cos_c * normal_from_bits(b1) + v->sin_c * normal_from_bits(b2);
  return ob_phi(n);
}
/* samplers.hpp:102-104 */
static double vsrc_tail1(const vsrc* v, const vpfx* p, uint64_t a) {
  return vsrc_finish(v, hstep(p->h1, a), v->smoothed ? hstep(p->h2, a) : 0);
}

/* Variate of neighbour t as labor_block_stream draws it (samplers.cpp:112-129). */
double ob_labor_variate(const ob_sched* sched, int layer, uint32_t t) {
  const vsrc v = vsrc_from(sched);
  const uint64_t ids[2] = {2, (uint64_t)layer};
  const vpfx p = vsrc_prefix(&v, ids, 2);
  return vsrc_tail1(&v, &p, t);
}

/* ------------------------------------------------------------- sorting --- */

static void radix_u32(uint32_t* a, uint64_t n) {
  if (n < 2) return;
  uint32_t* tmp = xmalloc(n * sizeof(uint32_t));
  for (int pass = 0; pass < 2; ++pass) {
    const int sh = pass * 16;
    uint64_t* cnt = calloc(65537, sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) cnt[((a[i] >> sh) & 0xffff) + 1]++;
    for (int d = 0; d < 65536; ++d) cnt[d + 1] += cnt[d];
    for (uint64_t i = 0; i < n; ++i) tmp[cnt[(a[i] >> sh) & 0xffff]++] = a[i];
    memcpy(a, tmp, n * sizeof(uint32_t));
    free(cnt);
  }
  free(tmp);
}

static uint64_t unique_sorted_u32(uint32_t* a, uint64_t n) {
  if (n == 0) return 0;
  uint64_t w = 1;
  for (uint64_t i = 1; i < n; ++i)
    if (a[i] != a[w - 1]) a[w++] = a[i];
  return w;
}

static uint64_t lower_bound_u32(const uint32_t* a, uint64_t n, uint32_t v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* ---------------------------------------------------------------- graph --- */

/* graph.cpp:17-48 */
int ob_build_csr(const uint32_t* src, const uint32_t* dst, uint64_t m,
                 uint64_t n, uint64_t* indptr, uint32_t* indices) {
  memset(indptr, 0, (n + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) {
    if (src[i] >= n || dst[i] >= n)
      return fail("build_csr: edge (%u -> %u) has id >= %llu", src[i], dst[i],
                  (unsigned long long)n);
    indptr[dst[i] + 1] += 1;
  }
  for (uint64_t v = 0; v < n; ++v) indptr[v + 1] += indptr[v];
  uint64_t* cur = xmalloc(n * sizeof(uint64_t));
  memcpy(cur, indptr, n * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) indices[cur[dst[i]]++] = src[i];
  free(cur);
  return 0;
}

/* Hash-keyed R-MAT (DESIGN.md §"Synthetic graph"). Sequential form of the
 * rule the GPU generator evaluates in parallel:
 *   attempt a draws scale bits MSB-first; level i uses the 16-bit lane
 *   (i & 3) of w = hash_bits(seed, {13, a, i >> 2}) and picks quadrant
 *   q = [u>=T1] + [u>=T2] + [u>=T3] (a,b,c,d = .57,.19,.19,.05 in 1/65536);
 *   src bit = q >> 1, dst bit = q & 1. Attempts with an endpoint >= n are
 *   dropped; ids are then scrambled by a seed-keyed bijection of [0, 2^s)
 *   cycle-walked into [0, n); self-loops and repeated (src,dst) pairs are
 *   dropped (the reference generator's simple-graph rule, graph.cpp:141-149),
 *   and the first m_target surviving attempts, in attempt order, are the
 *   edges; CSR = build_csr of that list (graph.cpp:17-48). */
#define RMAT_T1 37356u
#define RMAT_T2 49808u
#define RMAT_T3 62260u

typedef struct {
  int s;
  uint64_t mask, m1, m2, add;
  int r;
} rmat_perm;

static rmat_perm perm_make(uint64_t seed, int s) {
  rmat_perm p;
  p.s = s;
  p.mask = (s >= 64) ? ~0ULL : ((1ULL << s) - 1);
  p.m1 = hb2(seed, 13, 0xFFFFFFFFFFFFFFF1ULL) | 1ULL;
  p.m2 = hb2(seed, 13, 0xFFFFFFFFFFFFFFF2ULL) | 1ULL;
  p.add = hb2(seed, 13, 0xFFFFFFFFFFFFFFF3ULL);
  p.r = (s + 1) / 2;
  return p;
}

static inline uint64_t perm_f(const rmat_perm* p, uint64_t x) {
  x = (x * p->m1) & p->mask;
  x ^= x >> p->r;
  x = (x * p->m2) & p->mask;
  x ^= x >> p->r;
  return (x + p->add) & p->mask;
}

static inline uint64_t perm_walk(const rmat_perm* p, uint64_t x, uint64_t n) {
  uint64_t y = perm_f(p, x);
  while (y >= n) y = perm_f(p, y);
  return y;
}

static int rmat_scale(uint64_t n) {
  int s = 1;
  while ((1ULL << s) < n) ++s;
  return s;
}

/* One attempt: returns 1 and sets (src,dst) raw ids if both < n. */
static inline int rmat_attempt(uint64_t pfx13, int s, uint64_t a, uint64_t n,
                               uint64_t* src, uint64_t* dst) {
  const uint64_t ha = hstep(pfx13, a);
  uint64_t sr = 0, ds = 0;
  for (int k = 0; 4 * k < s; ++k) { /* levels 4k..4k+3 share hash_bits(seed,{13,a,k}) */
    const uint64_t w = hstep(ha, (uint64_t)k);
    const int lv = s - 4 * k < 4 ? s - 4 * k : 4;
    for (int l = 0; l < lv; ++l) {
      const uint32_t u = (uint32_t)(w >> (16 * l)) & 0xffffu;
      const uint32_t q = (u >= RMAT_T1) + (u >= RMAT_T2) + (u >= RMAT_T3);
      sr = (sr << 1) | (q >> 1);
      ds = (ds << 1) | (q & 1u);
    }
  }
  *src = sr;
  *dst = ds;
  return sr < n && ds < n;
}

/* Minimal pthread fan-out for the embarrassingly parallel attempt loop. */
typedef struct {
  uint64_t pfx13;
  int s;
  uint64_t n;
  const rmat_perm* pm;
  uint64_t a0;
  uint64_t* cand;
  uint64_t chunk;
  int nthreads;
} rmat_job;

typedef struct {
  rmat_job* job;
  int tid;
} rmat_arg;

static void* rmat_worker(void* argp) {
  rmat_arg* arg = argp;
  rmat_job* j = arg->job;
  const uint64_t lo = j->chunk * (uint64_t)arg->tid / (uint64_t)j->nthreads;
  const uint64_t hi = j->chunk * (uint64_t)(arg->tid + 1) / (uint64_t)j->nthreads;
  for (uint64_t i = lo; i < hi; ++i) {
    uint64_t sr, ds;
    if (!rmat_attempt(j->pfx13, j->s, j->a0 + i, j->n, &sr, &ds) || sr == ds)
      j->cand[i] = ~0ULL;
    else
      j->cand[i] = (perm_walk(j->pm, sr, j->n) << 32) | perm_walk(j->pm, ds, j->n);
  }
  return NULL;
}

static void run_threads(void* (*fn)(void*), rmat_job* job) {
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  job->nthreads = (int)nt;
  pthread_t th[64];
  rmat_arg args[64];
  for (int t = 0; t < nt; ++t) {
    args[t].job = job;
    args[t].tid = t;
    pthread_create(&th[t], NULL, fn, &args[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

int ob_rmat(uint64_t n, uint64_t m_target, uint64_t seed, uint64_t** indptr_out,
            uint32_t** indices_out) {
  if (n < 2 || n > 0xFFFFFFFFULL) return fail("rmat: need 2 <= n < 2^32");
  if (m_target > n * (n - 1)) return fail("rmat: more edges than simple pairs");
  const int s = rmat_scale(n);
  const rmat_perm pm = perm_make(seed, s);
  const uint64_t pfx13 = hstep(hinit(seed), 13);

  uint64_t cap = 64;
  while (cap < 2 * m_target + 2) cap <<= 1;
  uint64_t* seen = calloc(cap, sizeof(uint64_t)); /* 0 = empty (never a key) */
  if (!seen) return fail("rmat: out of memory");
  uint32_t* es = xmalloc(m_target * sizeof(uint32_t));
  uint32_t* ed = xmalloc(m_target * sizeof(uint32_t));
  uint64_t got = 0;
  const uint64_t max_attempts = m_target * 1000 + 100000;
  /* Attempts are generated in parallel chunks (pure functions of a); the
   * dedup walk stays sequential in attempt order, so the result does not
   * depend on the thread count. */
  const uint64_t chunk = 1u << 22;
  uint64_t* cand = xmalloc(chunk * sizeof(uint64_t)); /* src<<32|dst, ~0 = drop */
  for (uint64_t a0 = 0; got < m_target; a0 += chunk) {
    if (a0 >= max_attempts) {
      free(seen); free(es); free(ed); free(cand);
      return fail("rmat: attempt budget exhausted (graph too dense)");
    }
    {
      rmat_job job = {pfx13, s, n, &pm, a0, cand, chunk, 0};
      run_threads(rmat_worker, &job);
    }
    for (uint64_t i = 0; i < chunk && got < m_target; ++i) {
      const uint64_t key = cand[i];
      if (key == ~0ULL) continue;
      uint64_t h = ob_mix64(key) & (cap - 1);
      int dup = 0;
      while (seen[h]) {
        if (seen[h] == key) { dup = 1; break; }
        h = (h + 1) & (cap - 1);
      }
      if (dup) continue;
      seen[h] = key;
      es[got] = (uint32_t)(key >> 32);
      ed[got] = (uint32_t)key;
      ++got;
    }
  }
  free(cand);
  free(seen);
  uint64_t* indptr = xmalloc((n + 1) * sizeof(uint64_t));
  uint32_t* indices = xmalloc(m_target * sizeof(uint32_t));
  ob_build_csr(es, ed, m_target, n, indptr, indices);
  free(es);
  free(ed);
  *indptr_out = indptr;
  *indices_out = indices;
  return 0;
}

/* Parallel form of ob_rmat for the large configs (c4: 1.6B edges), same
 * result bit for bit (tests/test_oracle_golden.py compares the two). The
 * sequential walk "take the first m attempts whose (src,dst) pair is new" is
 * split by destination range:
 *   1. count the valid attempts per (thread range, dst bucket);
 *   2. scatter attempt indices into their bucket, ascending (stable);
 *   3. per bucket, a hash set over its pairs marks each pair's first attempt
 *      (pairs of different buckets never collide: the bucket is part of dst);
 *   4. the m-th marked attempt in attempt order is the cutoff;
 *   5. per bucket, the marked attempts up to the cutoff are counted per dst
 *      and placed in attempt order (build_csr order, graph.cpp:17-48).
 * Attempts are pure functions of their index: pass 1 recomputes them to
 * count, pass 2 stores each valid attempt's pair next to its index. Memory:
 * 13 B per attempt + the CSR. */
typedef struct {
  uint64_t pfx13, n, A;
  int s, bshift;
  const rmat_perm* pm;
  uint32_t nb, nt;
  uint64_t* cnt;        /* [nt][nb] valid attempts, then write cursors */
  uint32_t* arr;        /* [valid] attempt indices grouped by bucket */
  uint64_t* pair;       /* [valid] dst << 32 | src of arr[i] */
  uint64_t* bstart;     /* [nb+1] */
  uint8_t* surv;        /* [A] first attempt of its pair */
  uint64_t a_star;      /* last kept attempt */
  uint64_t* indptr;     /* [n+1] */
  uint32_t* indices;
  uint64_t* bkept;      /* [nb] kept edges per bucket */
  uint64_t* tsurv;      /* [nt] survivors per thread range */
  volatile uint32_t next;
  int phase;
} rmatp_job;

typedef struct {
  rmatp_job* j;
  uint32_t tid;
} rmatp_arg;

static inline int rmatp_pair(const rmatp_job* j, uint64_t a, uint32_t* src, uint32_t* dst,
                             int need_src) {
  uint64_t sr, ds;
  if (!rmat_attempt(j->pfx13, j->s, a, j->n, &sr, &ds) || sr == ds) return 0;
  *dst = (uint32_t)perm_walk(j->pm, ds, j->n);
  if (need_src) *src = (uint32_t)perm_walk(j->pm, sr, j->n);
  return 1;
}

static void rmatp_bucket(rmatp_job* j, uint32_t b, uint64_t** tab, uint64_t* tcap,
                         uint64_t** cur, uint64_t* ccap) {
  const uint64_t lo = j->bstart[b], hi = j->bstart[b + 1];
  const uint64_t d0 = (uint64_t)b << j->bshift;
  uint64_t d1 = d0 + (1ULL << j->bshift);
  if (d1 > j->n) d1 = j->n;
  if (j->phase == 3) { /* first attempt of each pair */
    uint64_t cap = 64;
    while (cap < 2 * (hi - lo) + 2) cap <<= 1;
    if (cap > *tcap) {
      free(*tab);
      *tab = xmalloc(cap * sizeof(uint64_t));
      *tcap = cap;
    }
    uint64_t* t = *tab;
    memset(t, 0, cap * sizeof(uint64_t));
    for (uint64_t i = lo; i < hi; ++i) {
      const uint64_t a = j->arr[i];
      const uint64_t key = j->pair[i]; /* never 0: no self loops */
      uint64_t h = ob_mix64(key) & (cap - 1);
      int dup = 0;
      while (t[h]) {
        if (t[h] == key) { dup = 1; break; }
        h = (h + 1) & (cap - 1);
      }
      if (!dup) {
        t[h] = key;
        j->surv[a] = 1;
      }
    }
  } else if (j->phase == 5) { /* per-dst counts of the kept attempts */
    uint64_t k = 0;
    for (uint64_t i = lo; i < hi; ++i) {
      const uint64_t a = j->arr[i];
      if (a > j->a_star || !j->surv[a]) continue;
      j->indptr[(j->pair[i] >> 32) + 1] += 1;
      ++k;
    }
    j->bkept[b] = k;
  } else if (j->phase == 6) { /* counts -> offsets within the bucket */
    uint64_t run = 0;
    for (uint64_t b2 = 0; b2 < b; ++b2) run += j->bkept[b2];
    for (uint64_t d = d0; d < d1; ++d) {
      const uint64_t c = j->indptr[d + 1];
      j->indptr[d + 1] = run + c;
      run += c;
    }
  } else { /* phase 7: place src ids in attempt order */
    const uint64_t w = d1 - d0;
    if (w > *ccap) {
      free(*cur);
      *cur = xmalloc(w * sizeof(uint64_t));
      *ccap = w;
    }
    uint64_t* c = *cur;
    for (uint64_t d = d0; d < d1; ++d) c[d - d0] = j->indptr[d];
    for (uint64_t i = lo; i < hi; ++i) {
      const uint64_t a = j->arr[i];
      if (a > j->a_star || !j->surv[a]) continue;
      const uint64_t key = j->pair[i];
      j->indices[c[(key >> 32) - d0]++] = (uint32_t)key;
    }
  }
}

static void* rmatp_worker(void* argp) {
  rmatp_arg* arg = argp;
  rmatp_job* j = arg->j;
  const uint32_t t = arg->tid;
  const uint64_t lo = j->A * t / j->nt, hi = j->A * (t + 1) / j->nt;
  if (j->phase == 1 || j->phase == 2) {
    uint64_t* c = j->cnt + (uint64_t)t * j->nb;
    for (uint64_t a = lo; a < hi; ++a) {
      uint32_t sr = 0, ds = 0;
      if (!rmatp_pair(j, a, &sr, &ds, j->phase == 2)) continue;
      const uint32_t b = ds >> j->bshift;
      if (j->phase == 1) {
        c[b]++;
      } else {
        j->pair[c[b]] = ((uint64_t)ds << 32) | sr;
        j->arr[c[b]++] = (uint32_t)a;
      }
    }
  } else if (j->phase == 4) {
    uint64_t k = 0;
    for (uint64_t a = lo; a < hi; ++a) k += j->surv[a];
    j->tsurv[t] = k;
  } else {
    uint64_t* tab = NULL, *cur = NULL;
    uint64_t tcap = 0, ccap = 0;
    for (;;) {
      const uint32_t b = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
      if (b >= j->nb) break;
      rmatp_bucket(j, b, &tab, &tcap, &cur, &ccap);
    }
    free(tab);
    free(cur);
  }
  return NULL;
}

#include <time.h>
static void rmatp_run(rmatp_job* j, int phase) {
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  j->phase = phase;
  j->next = 0;
  pthread_t th[64];
  rmatp_arg args[64];
  for (uint32_t t = 0; t < j->nt; ++t) {
    args[t].j = j;
    args[t].tid = t;
    pthread_create(&th[t], NULL, rmatp_worker, &args[t]);
  }
  for (uint32_t t = 0; t < j->nt; ++t) pthread_join(th[t], NULL);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  if (getenv("OB_RMAT_TIMING"))
    fprintf(stderr, "rmat phase %d: %.3f s\n", phase,
            (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec));
}

int ob_rmat_par(uint64_t n, uint64_t m_target, uint64_t seed, uint64_t** indptr_out,
                uint32_t** indices_out) {
  if (n < 2 || n > 0xFFFFFFFFULL) return fail("rmat: need 2 <= n < 2^32");
  if (m_target > n * (n - 1)) return fail("rmat: more edges than simple pairs");
  if (m_target == 0) {
    *indptr_out = calloc(n + 1, sizeof(uint64_t));
    *indices_out = xmalloc(4);
    return *indptr_out ? 0 : fail("rmat: out of memory");
  }
  const int s = rmat_scale(n);
  const rmat_perm pm = perm_make(seed, s);
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  if (nt < 1) nt = 1;
  if (nt > 64) nt = 64;
  rmatp_job j;
  memset(&j, 0, sizeof(j));
  j.pfx13 = hstep(hinit(seed), 13);
  j.n = n;
  j.s = s;
  j.pm = &pm;
  j.nt = (uint32_t)nt;
  j.bshift = s > 9 ? s - 9 : 0; /* <= 512 buckets: few write streams per thread */
  j.nb = (uint32_t)((n + (1ULL << j.bshift) - 1) >> j.bshift);
  uint64_t A = m_target + m_target / 4 + 4096;
  for (int round = 0;; ++round) {
    if (A >= (1ULL << 32) - 1) return fail("rmat: attempt count exceeds 2^32");
    j.A = A;
    j.cnt = calloc((size_t)j.nt * j.nb, sizeof(uint64_t));
    j.bstart = xmalloc((j.nb + 1) * sizeof(uint64_t));
    rmatp_run(&j, 1);
    uint64_t valid = 0;
    for (uint32_t b = 0; b < j.nb; ++b) {
      j.bstart[b] = valid;
      for (uint32_t t = 0; t < j.nt; ++t) {
        const uint64_t c = j.cnt[(uint64_t)t * j.nb + b];
        j.cnt[(uint64_t)t * j.nb + b] = valid;
        valid += c;
      }
    }
    j.bstart[j.nb] = valid;
    j.arr = xmalloc(valid * sizeof(uint32_t));
    j.pair = xmalloc(valid * sizeof(uint64_t));
    rmatp_run(&j, 2);
    free(j.cnt);
    j.cnt = NULL;
    j.surv = calloc(A, 1);
    if (!j.surv) return fail("rmat: out of memory");
    rmatp_run(&j, 3);
    j.tsurv = calloc(j.nt, sizeof(uint64_t));
    rmatp_run(&j, 4);
    uint64_t total = 0;
    for (uint32_t t = 0; t < j.nt; ++t) total += j.tsurv[t];
    if (total >= m_target) {
      uint64_t before = 0;
      uint32_t t = 0;
      while (before + j.tsurv[t] < m_target) before += j.tsurv[t++];
      uint64_t a = A * t / j.nt;
      for (;; ++a)
        if (j.surv[a] && ++before == m_target) break;
      j.a_star = a;
      free(j.tsurv);
      break;
    }
    free(j.tsurv);
    free(j.arr);
    free(j.pair);
    free(j.surv);
    free(j.bstart);
    if (round >= 8) return fail("rmat: could not reach the edge target (graph too dense)");
    uint64_t A2 = A * 2;
    if (A2 < m_target + (m_target - total) * 4) A2 = m_target + (m_target - total) * 4;
    A = A2;
  }
  j.indptr = calloc(n + 1, sizeof(uint64_t));
  j.indices = xmalloc(m_target * sizeof(uint32_t));
  j.bkept = calloc(j.nb, sizeof(uint64_t));
  if (!j.indptr) return fail("rmat: out of memory");
  rmatp_run(&j, 5);
  rmatp_run(&j, 6);
  rmatp_run(&j, 7);
  free(j.bkept);
  free(j.arr);
  free(j.pair);
  free(j.surv);
  free(j.bstart);
  *indptr_out = j.indptr;
  *indices_out = j.indices;
  return 0;
}

/* ------------------------------------------------------------ partition --- */

/* partition.cpp:10-20 */
int ob_partition_random(uint64_t n, uint32_t parts, uint64_t seed, uint32_t* owner) {
  if (parts == 0) return fail("partition_random: parts must be >= 1");
  const uint64_t pfx = hstep(hinit(seed), 7);
  for (uint64_t v = 0; v < n; ++v) owner[v] = (uint32_t)(hstep(pfx, v) % parts);
  return 0;
}

/* ------------------------------------------------------------- sampling --- */

typedef struct {
  uint32_t* t;
  uint32_t* di;
  uint64_t n, cap;
} sampled_buf;

static void sb_add(sampled_buf* b, uint32_t t, uint32_t di) {
  if (b->n == b->cap) {
    b->cap = b->cap ? b->cap * 2 : 1024;
    b->t = realloc(b->t, b->cap * sizeof(uint32_t));
    b->di = realloc(b->di, b->cap * sizeof(uint32_t));
    if (!b->t || !b->di) abort();
  }
  b->t[b->n] = t;
  b->di[b->n] = di;
  b->n++;
}

/* samplers.cpp:28-54 BlockBuilder::finish */
static void block_finish(const uint32_t* seeds, uint64_t n_seeds, sampled_buf* sb,
                         int layer, ob_block* out) {
  out->layer = layer;
  out->n_dst = n_seeds;
  out->dst = xmalloc(n_seeds * sizeof(uint32_t));
  memcpy(out->dst, seeds, n_seeds * sizeof(uint32_t));
  uint64_t ns = n_seeds + sb->n;
  uint32_t* src = xmalloc(ns * sizeof(uint32_t));
  memcpy(src, seeds, n_seeds * sizeof(uint32_t));
  if (sb->n) memcpy(src + n_seeds, sb->t, sb->n * sizeof(uint32_t));
  radix_u32(src, ns);
  ns = unique_sorted_u32(src, ns);
  out->n_src = ns;
  out->src = src;
  out->n_edges = sb->n;
  out->edges = xmalloc(2 * sb->n * sizeof(uint32_t));
  for (uint64_t e = 0; e < sb->n; ++e) {
    out->edges[2 * e] = (uint32_t)lower_bound_u32(src, ns, sb->t[e]);
    out->edges[2 * e + 1] = sb->di[e];
  }
  out->dst_pos = xmalloc(n_seeds * sizeof(uint32_t));
  for (uint64_t i = 0; i < n_seeds; ++i)
    out->dst_pos[i] = (uint32_t)lower_bound_u32(src, ns, seeds[i]);
  free(sb->t);
  free(sb->di);
  sb->t = sb->di = NULL;
  sb->n = sb->cap = 0;
}

/* samplers.cpp:62-87 ns_block */
static void ns_sample(const uint64_t* indptr, const uint32_t* indices,
                      const uint32_t* seeds, uint64_t n_seeds, uint32_t k,
                      const vsrc* src, int layer, sampled_buf* sb) {
  uint64_t* slots = xmalloc((k ? k : 1) * sizeof(uint64_t));
  for (uint64_t di = 0; di < n_seeds; ++di) {
    const uint32_t s = seeds[di];
    const uint32_t* ns = indices + indptr[s];
    const uint64_t d = indptr[s + 1] - indptr[s];
    if (d <= k) {
      for (uint64_t i = 0; i < d; ++i) sb_add(sb, ns[i], (uint32_t)di);
      continue;
    }
    const uint64_t ids[3] = {1 /* kStreamNs */, (uint64_t)layer, s};
    const vpfx p = vsrc_prefix(src, ids, 3);
    for (uint32_t j = 0; j < k; ++j) slots[j] = j;
    for (uint64_t i = k; i < d; ++i) {
      const double u = vsrc_tail1(src, &p, i);
      const uint64_t r = (uint64_t)(u * (double)(i + 1));
      if (r < k) slots[r] = i;
    }
    for (uint32_t j = 0; j < k; ++j) sb_add(sb, ns[slots[j]], (uint32_t)di);
  }
  free(slots);
}

/* samplers.cpp:108-136 labor_block_stream (memoisation does not change
 * values, so it is omitted) */
static void labor_sample(const uint64_t* indptr, const uint32_t* indices,
                         const uint32_t* seeds, uint64_t n_seeds, uint32_t k,
                         const vsrc* src, int layer, sampled_buf* sb) {
  const uint64_t ids[2] = {2 /* kStreamLabor */, (uint64_t)layer};
  const vpfx p = vsrc_prefix(src, ids, 2);
  for (uint64_t di = 0; di < n_seeds; ++di) {
    const uint32_t s = seeds[di];
    const uint32_t* ns = indices + indptr[s];
    const uint64_t d = indptr[s + 1] - indptr[s];
    if (d == 0) continue;
    const double thr = (double)k / (double)d;
    for (uint64_t i = 0; i < d; ++i)
      if (vsrc_tail1(src, &p, ns[i]) <= thr) sb_add(sb, ns[i], (uint32_t)di);
  }
}

static int sample_block_v(const uint64_t* indptr, const uint32_t* indices, uint64_t n,
                          const uint32_t* seeds, uint64_t n_seeds, int kind,
                          uint32_t k, const vsrc* src, int layer, ob_block* out) {
  for (uint64_t i = 0; i < n_seeds; ++i) /* samplers.cpp:11-13 */
    if (seeds[i] >= n)
      return fail("vertex id %u out of range [0, %llu)", seeds[i],
                  (unsigned long long)n);
  sampled_buf sb = {0};
  switch (kind) {
    case OB_FULL: /* samplers.cpp:289-296 */
      for (uint64_t di = 0; di < n_seeds; ++di)
        for (uint64_t e = indptr[seeds[di]]; e < indptr[seeds[di] + 1]; ++e)
          sb_add(&sb, indices[e], (uint32_t)di);
      break;
    case OB_NS:
      ns_sample(indptr, indices, seeds, n_seeds, k, src, layer, &sb);
      break;
    case OB_LABOR0:
      labor_sample(indptr, indices, seeds, n_seeds, k, src, layer, &sb);
      break;
    default:
      return fail("sample_block: unknown sampler kind");
  }
  block_finish(seeds, n_seeds, &sb, layer, out);
  return 0;
}

int ob_sample_block(const uint64_t* indptr, const uint32_t* indices, uint64_t n,
                    const uint32_t* seeds, uint64_t n_seeds, int kind,
                    uint32_t fanout, const ob_sched* sched, int layer, ob_block* out) {
  const vsrc v = vsrc_from(sched);
  return sample_block_v(indptr, indices, n, seeds, n_seeds, kind, fanout, &v, layer, out);
}

void ob_block_free(ob_block* b) {
  free(b->dst); free(b->src); free(b->edges); free(b->dst_pos);
  memset(b, 0, sizeof(*b));
}

void ob_stack_free(ob_stack* s) {
  for (int l = 0; l < s->num_layers; ++l) ob_block_free(&s->blocks[l]);
  free(s->blocks);
  s->blocks = NULL;
  s->num_layers = 0;
}

/* samplers.cpp:340-354 */
int ob_expand(const uint64_t* indptr, const uint32_t* indices, uint64_t n,
              const uint32_t* seeds, uint64_t n_seeds, int L, int kind,
              const uint32_t* fanouts, const ob_sched* sched, ob_stack* out) {
  if (L < 1) return fail("expand: num_layers must be >= 1");
  const vsrc v = vsrc_from(sched);
  out->num_layers = 0;
  out->blocks = calloc((size_t)L, sizeof(ob_block));
  const uint32_t* cur = seeds;
  uint64_t n_cur = n_seeds;
  for (int l = 0; l < L; ++l) {
    const int rc = sample_block_v(indptr, indices, n, cur, n_cur, kind, fanouts[l],
                                  &v, l, &out->blocks[l]);
    if (rc) { ob_stack_free(out); return rc; }
    out->num_layers = l + 1;
    cur = out->blocks[l].src;
    n_cur = out->blocks[l].n_src;
  }
  return 0;
}

/* coop.cpp:25-64 build_exchange */
static void build_exchange(ob_block* const* blocks, const uint32_t* owner, uint32_t P,
                           int layer, ob_exchange* rec, uint32_t** next,
                           uint64_t* next_len) {
  rec->layer = layer;
  rec->num_parts = P;
  rec->send_counts = calloc((size_t)P * P, sizeof(uint64_t));
  rec->owner_row_counts = calloc(P, sizeof(uint64_t));
  rec->loc_len = calloc(P, sizeof(uint64_t));
  rec->loc_part = calloc(P, sizeof(uint32_t*));
  rec->loc_row = calloc(P, sizeof(uint64_t*));
  uint64_t* recv_len = calloc(P, sizeof(uint64_t));
  for (uint32_t p = 0; p < P; ++p)
    for (uint64_t j = 0; j < blocks[p]->n_src; ++j) {
      const uint32_t q = owner[blocks[p]->src[j]];
      rec->send_counts[(size_t)p * P + q] += 1;
      recv_len[q] += 1;
    }
  for (uint32_t q = 0; q < P; ++q) {
    next[q] = xmalloc(recv_len[q] * sizeof(uint32_t));
    next_len[q] = 0;
  }
  for (uint32_t p = 0; p < P; ++p)
    for (uint64_t j = 0; j < blocks[p]->n_src; ++j) {
      const uint32_t v = blocks[p]->src[j];
      const uint32_t q = owner[v];
      next[q][next_len[q]++] = v;
    }
  for (uint32_t q = 0; q < P; ++q) {
    radix_u32(next[q], next_len[q]);
    next_len[q] = unique_sorted_u32(next[q], next_len[q]);
    rec->owner_row_counts[q] = next_len[q];
  }
  for (uint32_t p = 0; p < P; ++p) {
    const uint64_t ns = blocks[p]->n_src;
    rec->loc_len[p] = ns;
    rec->loc_part[p] = xmalloc(ns * sizeof(uint32_t));
    rec->loc_row[p] = xmalloc(ns * sizeof(uint64_t));
    for (uint64_t j = 0; j < ns; ++j) {
      const uint32_t v = blocks[p]->src[j];
      const uint32_t q = owner[v];
      rec->loc_part[p][j] = q;
      rec->loc_row[p][j] = lower_bound_u32(next[q], next_len[q], v);
    }
  }
  free(recv_len);
}

void ob_coop_free(ob_coop* c) {
  if (c->stacks)
    for (uint32_t p = 0; p < c->num_parts; ++p) ob_stack_free(&c->stacks[p]);
  if (c->exchanges)
    for (int l = 0; l < c->num_layers; ++l) {
      ob_exchange* e = &c->exchanges[l];
      for (uint32_t p = 0; p < e->num_parts; ++p) {
        free(e->loc_part[p]);
        free(e->loc_row[p]);
      }
      free(e->send_counts); free(e->owner_row_counts); free(e->loc_len);
      free(e->loc_part); free(e->loc_row);
    }
  if (c->owner_sets)
    for (uint32_t p = 0; p < c->num_parts; ++p) free(c->owner_sets[p]);
  free(c->stacks); free(c->exchanges); free(c->owner_sets); free(c->owner_len);
  memset(c, 0, sizeof(*c));
}

/* coop.cpp:68-106 coop_sample */
int ob_coop_sample(const uint64_t* indptr, const uint32_t* indices, uint64_t n,
                   const uint32_t* owner, uint32_t P, const uint32_t* seeds_flat,
                   const uint64_t* seeds_off, int L, int kind, const uint32_t* fanouts,
                   const ob_sched* sched, ob_coop* out) {
  memset(out, 0, sizeof(*out));
  if (P == 0) return fail("partition: zero parts");
  for (uint64_t v = 0; v < n; ++v)
    if (owner[v] >= P) return fail("partition: owner id out of range");
  for (uint32_t p = 0; p < P; ++p)
    for (uint64_t i = seeds_off[p]; i < seeds_off[p + 1]; ++i) {
      const uint32_t s = seeds_flat[i];
      if (s >= n)
        return fail("vertex id %u out of range [0, %llu)", s, (unsigned long long)n);
      if (owner[s] != p)
        return fail("coop_sample: seed %u is not owned by part %u", s, p);
    }
  if (L < 1) return fail("coop_sample: num_layers must be >= 1");
  const vsrc v = vsrc_from(sched);
  out->num_parts = P;
  out->num_layers = L;
  out->stacks = calloc(P, sizeof(ob_stack));
  out->exchanges = calloc((size_t)L, sizeof(ob_exchange));
  for (uint32_t p = 0; p < P; ++p) {
    out->stacks[p].blocks = calloc((size_t)L, sizeof(ob_block));
    out->stacks[p].num_layers = L;
  }
  uint32_t** cur = calloc(P, sizeof(uint32_t*));
  uint64_t* cur_len = calloc(P, sizeof(uint64_t));
  for (uint32_t p = 0; p < P; ++p) {
    cur_len[p] = seeds_off[p + 1] - seeds_off[p];
    cur[p] = xmalloc(cur_len[p] * sizeof(uint32_t));
    memcpy(cur[p], seeds_flat + seeds_off[p], cur_len[p] * sizeof(uint32_t));
  }
  ob_block** bl = calloc(P, sizeof(ob_block*));
  for (int l = 0; l < L; ++l) {
    for (uint32_t p = 0; p < P; ++p) {
      bl[p] = &out->stacks[p].blocks[l];
      sample_block_v(indptr, indices, n, cur[p], cur_len[p], kind, fanouts[l], &v, l,
                     bl[p]);
    }
    uint32_t** next = calloc(P, sizeof(uint32_t*));
    uint64_t* next_len = calloc(P, sizeof(uint64_t));
    build_exchange(bl, owner, P, l, &out->exchanges[l], next, next_len);
    for (uint32_t p = 0; p < P; ++p) free(cur[p]);
    free(cur);
    free(cur_len);
    cur = next;
    cur_len = next_len;
  }
  out->owner_sets = cur;
  out->owner_len = cur_len;
  free(bl);
  return 0;
}

/* ------------------------------------------------------------- features --- */

/* coop.cpp:369-371 value = 2*U(hash(seed,{9,v,j})) - 1 (exact in f64), then
 * one rounding to the table dtype. */
void ob_feature_rows(uint64_t seed, uint32_t dim, int dtype, const uint32_t* ids,
                     uint64_t n_ids, void* out) {
  const uint64_t pfx = hstep(hinit(seed), 9);
  for (uint64_t r = 0; r < n_ids; ++r) {
    const uint64_t hv = hstep(pfx, ids[r]);
    for (uint32_t j = 0; j < dim; ++j) {
      const double x = 2.0 * ufb(hstep(hv, j)) - 1.0;
      const uint64_t o = r * dim + j;
      if (dtype == 0) ((double*)out)[o] = x;
      else if (dtype == 1) ((float*)out)[o] = (float)x;
      else {
        const _Float16 h = (_Float16)x;
        uint16_t bits;
        memcpy(&bits, &h, 2);
        ((uint16_t*)out)[o] = bits;
      }
    }
  }
}

/* ---------------------------------------------------------------- cache --- */

/* cache.cpp:8-32: LRU with recency list + index. Doubly linked list over a
 * node pool, open-addressing index keyed by vertex id. */
struct ob_lru {
  uint64_t cap, size;
  uint32_t* key;
  int64_t *prev, *next;
  int64_t head, tail; /* head = most recent */
  int64_t* table;     /* slot -> node or -1 */
  uint64_t tmask;
};

ob_lru* ob_lru_new(uint64_t cap) {
  if (cap == 0) return NULL;
  ob_lru* c = calloc(1, sizeof(ob_lru));
  c->cap = cap;
  c->key = xmalloc(cap * sizeof(uint32_t));
  c->prev = xmalloc(cap * sizeof(int64_t));
  c->next = xmalloc(cap * sizeof(int64_t));
  uint64_t ts = 16;
  while (ts < 2 * cap) ts <<= 1;
  c->tmask = ts - 1;
  c->table = xmalloc(ts * sizeof(int64_t));
  for (uint64_t i = 0; i < ts; ++i) c->table[i] = -1;
  c->head = c->tail = -1;
  return c;
}

static uint64_t lru_slot(const ob_lru* c, uint32_t key) {
  uint64_t h = ob_mix64(key) & c->tmask;
  while (c->table[h] >= 0 && c->key[c->table[h]] != key) h = (h + 1) & c->tmask;
  return h;
}

static void lru_table_erase(ob_lru* c, uint64_t h) { /* backward-shift delete */
  uint64_t i = h;
  c->table[i] = -1;
  for (uint64_t j = (i + 1) & c->tmask; c->table[j] >= 0; j = (j + 1) & c->tmask) {
    const uint64_t home = ob_mix64(c->key[c->table[j]]) & c->tmask;
    const int between = (i <= j) ? (i < home && home <= j) : (i < home || home <= j);
    if (!between) {
      c->table[i] = c->table[j];
      c->table[j] = -1;
      i = j;
    }
  }
}

static void lru_unlink(ob_lru* c, int64_t x) {
  if (c->prev[x] >= 0) c->next[c->prev[x]] = c->next[x]; else c->head = c->next[x];
  if (c->next[x] >= 0) c->prev[c->next[x]] = c->prev[x]; else c->tail = c->prev[x];
}

static void lru_push_front(ob_lru* c, int64_t x) {
  c->prev[x] = -1;
  c->next[x] = c->head;
  if (c->head >= 0) c->prev[c->head] = x;
  c->head = x;
  if (c->tail < 0) c->tail = x;
}

int ob_lru_access(ob_lru* c, uint32_t key) {
  const uint64_t h = lru_slot(c, key);
  if (c->table[h] >= 0) {
    const int64_t x = c->table[h];
    lru_unlink(c, x);
    lru_push_front(c, x);
    return 0;
  }
  int64_t x;
  if (c->size == c->cap) {
    x = c->tail;
    lru_unlink(c, x);
    lru_table_erase(c, lru_slot(c, c->key[x]));
  } else {
    x = (int64_t)c->size++;
  }
  c->key[x] = key;
  lru_push_front(c, x);
  c->table[lru_slot(c, key)] = x;
  return 1;
}

void ob_lru_free(ob_lru* c) {
  if (!c) return;
  free(c->key); free(c->prev); free(c->next); free(c->table); free(c);
}

typedef struct { uint64_t h; uint32_t v; } keyed_t;
static int keyed_cmp(const void* a, const void* b) {
  const keyed_t* x = a;
  const keyed_t* y = b;
  if (x->h != y->h) return x->h < y->h ? -1 : 1;
  return x->v < y->v ? -1 : (x->v > y->v);
}

/* cache.cpp:74-84 */
void ob_access_order(const uint32_t* ids, uint64_t n, uint64_t key, uint32_t* out) {
  keyed_t* k = xmalloc(n * sizeof(keyed_t));
  for (uint64_t i = 0; i < n; ++i) {
    k[i].h = ob_mix64((uint64_t)ids[i] ^ key);
    k[i].v = ids[i];
  }
  qsort(k, n, sizeof(keyed_t), keyed_cmp);
  for (uint64_t i = 0; i < n; ++i) out[i] = k[i].v;
  free(k);
}

/* cache.cpp:123-133 */
uint64_t ob_stack_fingerprint(const ob_stack* s) {
  uint64_t h = 0x9e3779b97f4a7c15ULL;
  for (int l = 0; l < s->num_layers; ++l) {
    const ob_block* b = &s->blocks[l];
    h = ob_mix64(h ^ (uint64_t)(int64_t)b->layer);
    for (uint64_t i = 0; i < b->n_dst; ++i) h = ob_mix64(h ^ b->dst[i]);
    for (uint64_t i = 0; i < b->n_src; ++i) h = ob_mix64(h ^ (0x100000000ULL | b->src[i]));
    for (uint64_t e = 0; e < b->n_edges; ++e)
      h = ob_mix64(h ^ (((uint64_t)b->edges[2 * e] << 32) | b->edges[2 * e + 1]));
  }
  return h;
}

/* cli.cpp:121-139 */
int ob_draw_from_pool(const uint32_t* pool, uint64_t n_pool, uint64_t count,
                      uint64_t seed, uint64_t tag, uint32_t* out) {
  if (count > n_pool) return fail("not enough vertices in pool to draw batch");
  unsigned char* used = calloc(n_pool ? n_pool : 1, 1);
  uint64_t got = 0, attempt = 0;
  const uint64_t pfx = hstep(hstep(hinit(seed), 8), tag);
  while (got < count) {
    const double u = ufb(hstep(pfx, attempt++));
    uint64_t i = (uint64_t)(u * (double)n_pool);
    if (i >= n_pool) i = n_pool - 1;
    if (used[i]) continue;
    used[i] = 1;
    out[got++] = pool[i];
  }
  free(used);
  return 0;
}
