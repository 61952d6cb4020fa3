/*
 * ref_arm.c -- the reference's multi-worker CPU path for factor(), ported to C
 * threads: the timed "reference" arm of bench.py (--impl reference) and the
 * cpu_baseline leg.
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY.  Nothing in paper_2410_15880_b200/
 * links, loads or calls this file.
 *
 * The reference (/root/reference/pkg/src/polyfactor, "R/") runs factor()'s
 * search through parallel_recombine_e when workers > 1 (R/verify.py:236-243;
 * the CLI defaults workers to os.cpu_count(), R/cli.py:113-117), and it cannot
 * travel to the GPU box (pure Python).  This file restates that path with real
 * threads instead of GIL-bound ones, operation for operation:
 *
 *   orc_par_recombine_e   parallel_recombine_e (R/parallel.py:255-272):
 *     subset_sums + frac of both halves            R/recombine.py:126-134, :738-741
 *     parallel_build: claim-if-empty / remove-and-own slot exchanges over
 *       disjoint pattern ranges (work_partitions), no lost insertion
 *                                                  R/parallel.py:86-192
 *     parallel_query_sweep: read-only partitioned probe of 1 - x per A value,
 *       window eps + GUARD                          R/parallel.py:195-252, R/recombine.py:585-618
 *     _canonical_filter on the union                R/recombine.py:148-162
 *   orc_order_candidates  sorted(nontrivial, key=(selected_degree(s), s))
 *                                                  R/verify.py:48-57, :267
 *   orc_verify_first      the verification loop of _factor_monic_squarefree:
 *     build_candidate -> trace_test -> round_and_divide in x87 long double
 *     (numpy.longdouble here), first survivor in order wins
 *                                                  R/verify.py:60-155, :270-284
 *
 * A slot of the shared table is one 16-byte cell (value, pattern-as-double):
 * the reference's dict cell (value, pattern) tuple; "claim-if-empty" is a
 * 16-byte compare-and-swap against EMPTY = (-1.0, 0) and "remove-and-own" an
 * exchange with EMPTY (R/parallel.py:1-12 documents exactly these two
 * indivisible operations).  After the build barrier the cells are the
 * interleaved (value, pattern) layout of R/recombine.py:297-325, which the
 * read-only sweep probes as _probe_window does.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#include "rfr_oracle.h"

#define GUARD 1e-12 /* R/recombine.py:28-30 */

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

typedef unsigned __int128 cell_t;

static inline cell_t mk_cell(double v, double pat) {
  uint64_t a, b;
  memcpy(&a, &v, 8);
  memcpy(&b, &pat, 8);
  return ((cell_t)b << 64) | a;
}
static inline double cell_value(cell_t c) {
  uint64_t a = (uint64_t)c;
  double v;
  memcpy(&v, &a, 8);
  return v;
}

static cell_t EMPTY_CELL;

/* ---------------------------------------------------------- thread helpers */
typedef void (*range_fn)(void *ctx, int64_t lo, int64_t hi, int w);
typedef struct {
  range_fn fn;
  void *ctx;
  int64_t lo, hi;
  int w;
} range_job;
static void *range_thread(void *a) {
  range_job *J = (range_job *)a;
  J->fn(J->ctx, J->lo, J->hi, J->w);
  return NULL;
}
/* work_partitions (R/parallel.py:86-92): contiguous ranges, step = ceil. */
static void run_ranges(range_fn fn, void *ctx, int64_t total, int T) {
  if (T < 1) T = 1;
  if (T > 256) T = 256;
  if (total < 4096) T = 1;
  pthread_t th[256];
  range_job jobs[256];
  int64_t step = (total + T - 1) / T;
  int used = 0;
  for (int w = 0; w < T; w++) {
    int64_t lo = (int64_t)w * step, hi = lo + step < total ? lo + step : total;
    if (lo >= total) break;
    jobs[w] = (range_job){fn, ctx, lo, hi, w};
    used++;
  }
  if (used == 1) {
    range_thread(&jobs[0]);
    return;
  }
  for (int w = 0; w < used; w++) pthread_create(&th[w], NULL, range_thread, &jobs[w]);
  for (int w = 0; w < used; w++) pthread_join(th[w], NULL);
}

/* --------------------------------------------------------- subset sums */
/* R/recombine.py:126-134: sums[2^j + i] = sums[i] + v_j (ascending-index
 * accumulation, bit for bit), then sums -= floor(sums) (:738-741). */
typedef struct {
  double *s;
  double v;
  int64_t base;
} dbl_ctx;
static void dbl_range(void *c, int64_t lo, int64_t hi, int w) {
  dbl_ctx *C = (dbl_ctx *)c;
  for (int64_t i = lo; i < hi; i++) C->s[C->base + i] = C->s[i] + C->v;
}
static void frac_range(void *c, int64_t lo, int64_t hi, int w) {
  double *s = (double *)c;
  for (int64_t i = lo; i < hi; i++) s[i] -= floor(s[i]);
}
static double *par_subset_sums(const double *vals, int m, int T) {
  int64_t count = (int64_t)1 << m;
  double *s = (double *)malloc((size_t)count * sizeof(double));
  if (!s) return NULL;
  s[0] = 0.0;
  for (int j = 0; j < m; j++) {
    dbl_ctx C = {s, vals[j], (int64_t)1 << j};
    run_ranges(dbl_range, &C, (int64_t)1 << j, T);
  }
  run_ranges(frac_range, s, count, T);
  return s;
}

/* ---------------------------------------------------------- parallel build */
typedef struct {
  cell_t *cells;
  const double *xs;
  int64_t k;
  int64_t probes[256];
  int failed;
} build_ctx;

/* setdefault(i, item): claim if empty, else the current occupant. */
static inline cell_t claim(cell_t *slot, cell_t item) {
  return __sync_val_compare_and_swap(slot, EMPTY_CELL, item);
}
/* pop(i): remove-and-own (EMPTY when the slot was already empty). */
static inline cell_t take(cell_t *slot) {
  cell_t cur = *(volatile cell_t *)slot;
  for (;;) {
    cell_t got = __sync_val_compare_and_swap(slot, cur, EMPTY_CELL);
    if (got == cur) return got;
    cur = got;
  }
}

/* parallel_insert (R/parallel.py:98-148), one value. */
static int64_t par_insert(build_ctx *B, double x, int64_t pattern) {
  const int64_t k = B->k;
  cell_t own[64];
  int nown = 0;
  own[nown++] = mk_cell(x, (double)pattern);
  int64_t probes = 0;
  while (nown) {
    const cell_t item = own[--nown];
    const double val = cell_value(item);
    int64_t i = (int64_t)(k * val);
    int64_t steps = 0;
    for (;;) {
      probes++;
      steps++;
      if (steps > 2 * k || nown >= 63) {
        B->failed = 1; /* "insert probe budget exhausted; table over-full" */
        return probes;
      }
      const cell_t cur = claim(&B->cells[i], item);
      if (cur == EMPTY_CELL) break; /* claimed an empty slot */
      if (cell_value(cur) > val) {
        const cell_t got = take(&B->cells[i]);
        if (got == EMPTY_CELL) continue; /* lost a race; slot empty again, retry claim */
        if (claim(&B->cells[i], item) == EMPTY_CELL) {
          own[nown++] = got; /* we displaced got; re-insert it */
          break;
        }
        own[nown++] = got; /* someone else claimed; we still own got */
        continue;
      }
      i++;
      if (i == k) i = 0;
    }
  }
  return probes;
}

static void build_range(void *c, int64_t lo, int64_t hi, int w) {
  build_ctx *B = (build_ctx *)c;
  int64_t p = 0;
  for (int64_t s = lo; s < hi && !B->failed; s++) p += par_insert(B, B->xs[s], s);
  B->probes[w] = p;
}
static void empty_range(void *c, int64_t lo, int64_t hi, int w) {
  cell_t *cells = (cell_t *)c;
  for (int64_t i = lo; i < hi; i++) cells[i] = EMPTY_CELL;
}
typedef struct {
  const cell_t *cells;
  int64_t occ[256];
} count_ctx;
static void count_range(void *c, int64_t lo, int64_t hi, int w) {
  count_ctx *C = (count_ctx *)c;
  int64_t o = 0;
  for (int64_t i = lo; i < hi; i++) o += cell_value(C->cells[i]) >= 0.0;
  C->occ[w] = o;
}

/* -------------------------------------------------------- query sweep */
static double pymod1(double x) { /* Python's float % 1.0 for the values used */
  double r = fmod(x, 1.0);
  if (r < 0.0) r += 1.0;
  return r;
}
typedef struct {
  const double *xs;
  const double *merged; /* interleaved (value, pattern) */
  int64_t k, cap;
  int na;
  double eps;
  uint64_t *out;
  int64_t nout;
  int64_t probes[256];
} query_ctx;
/* _probe_window (R/recombine.py:585-618) for t = (1 - x) % 1 over a range of
 * A patterns (parallel_query_sweep's worker, R/parallel.py:221-231). */
static void query_range(void *c, int64_t lo_q, int64_t hi_q, int w) {
  query_ctx *Q = (query_ctx *)c;
  const int64_t k = Q->k;
  int64_t probes = 0;
  for (int64_t s_a = lo_q; s_a < hi_q; s_a++) {
    const double t = pymod1(1.0 - Q->xs[s_a]);
    const double lo = pymod1(t - Q->eps);
    int64_t start = (int64_t)(k * lo);
    if (start >= k) start -= k;
    int64_t span = ((int64_t)(k * pymod1(t + Q->eps)) - start) % k;
    if (span < 0) span += k;
    int64_t i = start, off = 0;
    while (off <= k) {
      const double v = Q->merged[2 * i];
      probes++;
      if (v < 0.0) {
        if (off >= span) break;
      } else {
        const double delta = pymod1(v - t);
        if (delta < Q->eps || delta > 1.0 - Q->eps) {
          const int64_t slot = __atomic_fetch_add(&Q->nout, 1, __ATOMIC_RELAXED);
          if (slot < Q->cap) Q->out[slot] = (uint64_t)s_a | ((uint64_t)Q->merged[2 * i + 1] << Q->na);
        }
      }
      off++;
      i++;
      if (i == k) i = 0;
    }
  }
  Q->probes[w] = probes;
}

/* ----------------------------------------------------- canonical filter */
static int cmp_u64(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : x > y;
}
typedef struct {
  uint64_t *raw;
  const double *rho;
  int n;
  double eps;
} filter_ctx;
/* _canonical_filter (R/recombine.py:148-162): t = min(s, s ^ full), kept iff
 * accept(value(t), eps) with the unwidened eps; rejected entries become
 * UINT64_MAX and are dropped after the sort. */
static void filter_range(void *c, int64_t lo, int64_t hi, int w) {
  filter_ctx *F = (filter_ctx *)c;
  const uint64_t full = F->n >= 64 ? ~0ull : ((1ull << F->n) - 1ull);
  for (int64_t j = lo; j < hi; j++) {
    const uint64_t s = F->raw[j];
    const uint64_t t = s < (s ^ full) ? s : (s ^ full);
    F->raw[j] = orc_accept(orc_value(F->rho, F->n, t), F->eps) ? t : UINT64_MAX;
  }
}

/*
 * parallel_recombine_e(rho, eps, workers) (R/parallel.py:255-272) with
 * `threads` workers.  Writes the sorted canonical candidate set (as
 * frozenset(int)) into out[0 .. min(count, cap)) and returns its size; -1 on
 * allocation failure, -2 when the build lost an insertion or overflowed.
 * stats[0..4]: inserts, insert_probes, queries, query_probes, raw hits;
 * stats[5..9]: ns in subset sums, build, query sweep, filter, total.
 * n < 2 is the caller's (recombine_a) and not handled here.
 */
int64_t orc_par_recombine_e(const double *rho, int n, double eps, int threads, uint64_t *out,
                            int64_t cap, int64_t *stats) {
  const double t0 = now_s();
  EMPTY_CELL = mk_cell(-1.0, 0.0);
  const int T = threads > 0 ? threads : orc_num_threads();
  const int na = n / 2, nb = n - na;
  double *bsums = par_subset_sums(rho + na, nb, T);
  double *asums = par_subset_sums(rho, na, T);
  const int64_t count = (int64_t)1 << nb, nav = (int64_t)1 << na, k = 2 * count;
  cell_t *cells = (cell_t *)aligned_alloc(64, (size_t)k * sizeof(cell_t));
  if (!bsums || !asums || !cells) {
    free(bsums);
    free(asums);
    free(cells);
    return -1;
  }
  run_ranges(empty_range, cells, k, T);
  const double t1 = now_s();
  build_ctx B;
  memset(&B, 0, sizeof B);
  B.cells = cells;
  B.xs = bsums;
  B.k = k;
  run_ranges(build_range, &B, count, T);
  count_ctx C;
  memset(&C, 0, sizeof C);
  C.cells = cells;
  run_ranges(count_range, &C, k, T);
  int64_t occ = 0, iprobes = 0;
  for (int w = 0; w < 256; w++) occ += C.occ[w], iprobes += B.probes[w];
  if (B.failed || occ != count) { /* assert table.occupied() == count */
    free(bsums);
    free(asums);
    free(cells);
    return -2;
  }
  const double t2 = now_s();
  /* query sweep; the raw buffer regrows and the sweep reruns (rare) */
  int64_t rcap = 1 << 22, nraw;
  uint64_t *raw = NULL;
  query_ctx Q;
  for (;;) {
    free(raw);
    raw = (uint64_t *)malloc((size_t)rcap * sizeof(uint64_t));
    if (!raw) {
      free(bsums);
      free(asums);
      free(cells);
      return -1;
    }
    memset(&Q, 0, sizeof Q);
    Q = (query_ctx){asums, (const double *)cells, k, rcap, na, eps + GUARD, raw, 0, {0}};
    run_ranges(query_range, &Q, nav, T);
    nraw = Q.nout;
    if (nraw <= rcap) break;
    rcap = nraw;
  }
  int64_t qprobes = 0;
  for (int w = 0; w < 256; w++) qprobes += Q.probes[w];
  const double t3 = now_s();
  /* union (a set in the reference), then the canonical filter */
  filter_ctx F = {raw, rho, n, eps};
  run_ranges(filter_range, &F, nraw, T);
  qsort(raw, (size_t)nraw, sizeof(uint64_t), cmp_u64);
  int64_t m = 0;
  for (int64_t j = 0; j < nraw; j++) {
    if (raw[j] == UINT64_MAX) break;
    if (m && raw[j] == raw[m - 1]) continue;
    raw[m++] = raw[j];
  }
  for (int64_t j = 0; j < m && j < cap; j++) out[j] = raw[j];
  const double t4 = now_s();
  if (stats) {
    stats[0] = count;
    stats[1] = iprobes;
    stats[2] = nav;
    stats[3] = qprobes;
    stats[4] = nraw;
    stats[5] = (int64_t)((t1 - t0) * 1e9);
    stats[6] = (int64_t)((t2 - t1) * 1e9);
    stats[7] = (int64_t)((t3 - t2) * 1e9);
    stats[8] = (int64_t)((t4 - t3) * 1e9);
    stats[9] = (int64_t)((t4 - t0) * 1e9);
  }
  free(raw);
  free(cells);
  free(bsums);
  free(asums);
  return m;
}

/* ------------------------------------------------- candidate order */
typedef struct {
  int deg;
  uint64_t s;
} ordered_t;
static int cmp_ord(const void *a, const void *b) {
  const ordered_t *x = (const ordered_t *)a, *y = (const ordered_t *)b;
  if (x->deg != y->deg) return x->deg < y->deg ? -1 : 1;
  return x->s < y->s ? -1 : x->s > y->s;
}
/* sorted(cands.nontrivial(), key=(selected_degree(s, profile), s))
 * (R/verify.py:48-57, :267), in place; 0 and 2^n - 1 dropped first.
 * Returns the new count. */
int64_t orc_order_candidates(uint64_t *pats, int64_t m, const int *perm, int r, int n) {
  const uint64_t full = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
  ordered_t *o = (ordered_t *)malloc((size_t)(m ? m : 1) * sizeof(ordered_t));
  if (!o) return -1;
  int64_t q = 0;
  for (int64_t j = 0; j < m; j++) {
    const uint64_t s = pats[j];
    if (s == 0 || s == full) continue;
    int e = 0;
    for (int i = 0; i < n; i++)
      if ((s >> i) & 1u) e += perm[i] < r ? 1 : 2;
    o[q++] = (ordered_t){e, s};
  }
  qsort(o, (size_t)q, sizeof(ordered_t), cmp_ord);
  for (int64_t j = 0; j < q; j++) pats[j] = o[j].s;
  free(o);
  return q;
}

/* ------------------------------------------------ verification loop */
typedef struct {
  const uint64_t *pats;
  const double *real_roots, *pair_sums, *pair_products;
  const int *perm;
  int r, c, n;
  const int64_t *p;
  int dp;
  double eps;
  int8_t *verdict; /* 0 reject, 1 pass, 2 undecided (quotient beyond int128) */
  int64_t base;
} verify_ctx;
static void verify_range(void *c, int64_t lo, int64_t hi, int w) {
  verify_ctx *V = (verify_ctx *)c;
  ld coeffs[260], traces[260], scales[260];
  int64_t q[260], quot[260];
  for (int64_t j = lo; j < hi; j++) {
    const uint64_t s = V->pats[V->base + j];
    const int e = orc_build_candidate(s, V->real_roots, V->r, V->pair_sums, V->pair_products, V->c,
                                      V->perm, V->n, coeffs, traces, scales);
    int8_t v = 0;
    if (orc_trace_test(traces, scales, e, V->eps) && orc_round_coeffs(coeffs, e, V->eps, q)) {
      int dq = e;
      while (dq > 0 && q[dq] == 0) dq--;
      if (dq >= 1) {
        const int rc = orc_divide_exact_i128(V->p, V->dp, q, dq, quot);
        v = rc == 1 ? 1 : rc < 0 ? 2 : 0;
      }
    }
    V->verdict[j] = v;
  }
}
/*
 * The loop of R/verify.py:270-284 over the ordered candidates pats[from ..
 * m): the index of the first candidate that survives build_candidate ->
 * trace_test -> round_and_divide (its rounded coefficients in q_out[0 ..
 * *deg_out]), or of the first one whose exact division left int128 (status
 * 2 in *status: the caller decides it with bigints and resumes after it);
 * m when none survives (status 0).  Candidates are verified `threads` at a
 * time in chunks, and the first survivor in order is the answer, so the
 * result is the serial loop's.
 */
int64_t orc_verify_first(const uint64_t *pats, int64_t from, int64_t m, const double *real_roots,
                         int r, const double *pair_sums, const double *pair_products, int c,
                         const int *perm, int n, const int64_t *p, int dp, double eps, int threads,
                         int64_t *q_out, int *deg_out, int *status) {
  const int T = threads > 0 ? threads : orc_num_threads();
  const int64_t chunk = 64 * (int64_t)T;
  int8_t *verdict = (int8_t *)malloc((size_t)chunk);
  if (!verdict) return -1;
  *status = 0;
  for (int64_t base = from; base < m; base += chunk) {
    const int64_t len = m - base < chunk ? m - base : chunk;
    verify_ctx V = {pats, real_roots, pair_sums, pair_products, perm, r, c, n, p, dp, eps, verdict, base};
    /* run_ranges goes serial below 4096 items: split the chunk explicitly */
    int TT = T > 256 ? 256 : T;
    if (len < TT) TT = (int)len;
    pthread_t th[256];
    range_job jobs[256];
    for (int w = 0; w < TT; w++)
      jobs[w] = (range_job){verify_range, &V, len * w / TT, len * (w + 1) / TT, w};
    for (int w = 1; w < TT; w++) pthread_create(&th[w], NULL, range_thread, &jobs[w]);
    range_thread(&jobs[0]);
    for (int w = 1; w < TT; w++) pthread_join(th[w], NULL);
    for (int64_t j = 0; j < len; j++) {
      if (!verdict[j]) continue;
      const int64_t idx = base + j;
      *status = verdict[j];
      if (verdict[j] == 1) {
        ld coeffs[260], traces[260], scales[260];
        const int e = orc_build_candidate(pats[idx], real_roots, r, pair_sums, pair_products, c,
                                          perm, n, coeffs, traces, scales);
        orc_round_coeffs(coeffs, e, eps, q_out);
        int dq = e;
        while (dq > 0 && q_out[dq] == 0) dq--;
        *deg_out = dq;
      }
      free(verdict);
      return idx;
    }
  }
  free(verdict);
  return m;
}
