/*
 * rfr_oracle.c -- CPU restatement of the reference recombination path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2410_15880_b200/ links, loads
 * or calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may use it, and only as the checker or
 * as the timed CPU baseline -- never as the product path.
 *
 * Reference: /root/reference/pkg/src/polyfactor (paths below are relative
 * to that package, "R/" = pkg/src/polyfactor/).  Pinned against the golden
 * vectors in the tests/golden JSON files that were produced by running the reference
 * itself (tests/golden/make_golden.py); see tests/test_oracle.py.
 *
 * Contents
 *   orc_value / orc_accept        R/recombine.py:106-123
 *   orc_recombine                 backend-a candidate set + canonical filter
 *                                 R/recombine.py:148-195 (the set every
 *                                 backend, including e :727-775, returns)
 *   orc_key_window                exhaustive uint64-key window search over the
 *                                 folded half space (the factor-mode search
 *                                 contract of the device join)
 *   orc_recombine_e_port          line-by-line port of backend e's numba
 *                                 kernels: _splat_merged_raw (:297-325) and
 *                                 _stream_merged_raw (:328-358), driven like
 *                                 recombine_e (:727-775).  This is the CPU
 *                                 baseline ("kind": "port") of bench.py.
 *   orc_build_candidate / orc_trace_test / orc_round_coeffs
 *                                 R/verify.py:60-155 in x87 long double, the
 *                                 same 80-bit type numpy.longdouble is here.
 *   orc_divide_exact_i128         R/polynomial.py:155-183 on __int128
 *                                 (returns -1 when a value leaves int128).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <time.h>
#include <unistd.h>

#include "rfr_oracle.h"

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

#define GUARD 1e-12 /* R/recombine.py:28-30 */

/* R/recombine.py:106-118: ascending-index float64 accumulation, then frac. */
double orc_value(const double *rho, int n, uint64_t s) {
    double x = 0.0;
    int i = 0;
    while (s && i < n) {
        if (s & 1u) x += rho[i];
        s >>= 1;
        i++;
    }
    return x - floor(x);
}

/* R/recombine.py:121-123 (strict inequalities). */
int orc_accept(double y, double eps) { return (y < eps) || ((1.0 - y) < eps); }

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

/* subset_sums by doubling, R/recombine.py:126-134 */
static double *subset_sums(const double *vals, int m) {
    size_t len = (size_t)1 << m;
    double *s = (double *)malloc(len * sizeof(double));
    if (!s) return NULL;
    s[0] = 0.0;
    size_t cur = 1;
    for (int k = 0; k < m; k++) {
        for (size_t j = 0; j < cur; j++) s[cur + j] = s[j] + vals[k];
        cur <<= 1;
    }
    return s;
}

/*
 * Backend a (R/recombine.py:169-195) followed by the canonical filter
 * (:148-162).  Writes the sorted canonical set into out[0..min(count,cap))
 * and returns the true count; -1 on allocation failure, -2 when n > 40.
 */
int64_t orc_recombine(const double *rho, int n, double eps, uint64_t *out, int64_t cap) {
    if (n == 0) return 0;
    if (n > 40) return -2;
    int bits = n - 1;
    double eps_d = eps + GUARD;
    uint64_t full = (n == 64) ? ~0ull : ((1ull << n) - 1);
    int lo_bits = bits < 20 ? bits : 20; /* _A_CHUNK_BITS, :33 */
    double *lo = subset_sums(rho, lo_bits);
    double *hi = subset_sums(rho + lo_bits, bits - lo_bits);
    if (!lo || !hi) {
        free(lo);
        free(hi);
        return -1;
    }
    size_t nlo = (size_t)1 << lo_bits, nhi = (size_t)1 << (bits - lo_bits);
    size_t fcap = 1024, fcount = 0;
    uint64_t *found = (uint64_t *)malloc(fcap * sizeof(uint64_t));
    for (size_t h = 0; h < nhi; h++) {
        double base = hi[h];
        for (size_t j = 0; j < nlo; j++) {
            double v = (bits <= 20) ? lo[j] : lo[j] + base;
            v -= floor(v);
            if (v < eps_d || v > 1.0 - eps_d) {
                uint64_t s = ((uint64_t)h << lo_bits) | j;
                /* canonical filter: t = min(s, s ^ full), keep iff accept(value(t)) */
                uint64_t t = s < (s ^ full) ? s : (s ^ full);
                if (orc_accept(orc_value(rho, n, t), eps)) {
                    if (fcount == fcap) {
                        fcap *= 2;
                        found = (uint64_t *)realloc(found, fcap * sizeof(uint64_t));
                    }
                    found[fcount++] = t;
                }
            }
        }
    }
    free(lo);
    free(hi);
    qsort(found, fcount, sizeof(uint64_t), cmp_u64);
    int64_t cnt = 0;
    for (size_t i = 0; i < fcount; i++) {
        if (i && found[i] == found[i - 1]) continue;
        if (cnt < cap) out[cnt] = found[i];
        cnt++;
    }
    free(found);
    return cnt;
}

/*
 * Exhaustive factor-mode window search: every pattern t < 2^(n-1) whose key
 * sum K(t) = sum_{i in t} keys[i] (mod 2^64) satisfies (K(t) - lo) mod 2^64
 * <= width.  Gray-code walk, one add per pattern.  Output sorted ascending.
 * Returns the true count (-2 when n > 36).
 */
int64_t orc_key_window(const uint64_t *keys, int n, uint64_t lo, uint64_t width, uint64_t *out,
                       int64_t cap) {
    if (n == 0) return 0;
    if (n > 36) return -2;
    int bits = n - 1;
    uint64_t count = 1ull << bits;
    uint64_t k = 0, g = 0;
    int64_t cnt = 0;
    for (uint64_t i = 0; i < count; i++) {
        if (i) {
            int b = __builtin_ctzll(i);
            g ^= 1ull << b;
            if (g >> b & 1u) k += keys[b];
            else k -= keys[b];
        }
        if (k - lo <= width) {
            if (cnt < cap) out[cnt] = g;
            cnt++;
        }
    }
    int64_t m = cnt < cap ? cnt : cap;
    qsort(out, (size_t)m, sizeof(uint64_t), cmp_u64);
    return cnt;
}

/* ---- backend e port: R/recombine.py:297-358 ------------------------------ */

/* _splat_merged_raw (:297-325); merged has 2k doubles, values EMPTY = -1. */
static int64_t splat_merged(const double *sums, int64_t count, double *merged, int64_t k) {
    int64_t probes = 0;
    for (int64_t s = 0; s < count; s++) {
        double x = sums[s];
        double pattern = (double)s;
        int64_t i = (int64_t)(k * x);
        int64_t steps = 0;
        while (steps <= k) {
            steps++;
            double v = merged[2 * i];
            if (v < 0.0) {
                merged[2 * i] = x;
                merged[2 * i + 1] = pattern;
                break;
            }
            if (v > x) {
                merged[2 * i] = x;
                double carried = merged[2 * i + 1];
                merged[2 * i + 1] = pattern;
                x = v;
                pattern = carried;
            }
            i++;
            if (i == k) i = 0;
        }
        probes += steps;
    }
    return probes;
}

static double pymod1(double x) { /* Python's float % 1.0 for the values used */
    double r = fmod(x, 1.0);
    if (r < 0.0) r += 1.0; /* may round to 1.0, exactly as Python does */
    return r;
}

/* _stream_merged_raw (:328-358) over the A-half values xs[lo..hi).  The
 * query loop is read-only over the table, so it runs on all host threads
 * (the partitioned query sweep of R/parallel.py:195-252); hits are appended
 * with an atomic cursor. */
typedef struct {
  const double *xs, *merged;
  int64_t lo_q, hi_q, k, cap;
  int na;
  double eps;
  uint64_t *out;
  int64_t *nout;
  int64_t probes;
} stream_job;

static void *stream_worker(void *arg) {
  stream_job *J = (stream_job *)arg;
  const int64_t k = J->k;
  int64_t probes = 0;
  for (int64_t s_a = J->lo_q; s_a < J->hi_q; s_a++) {
    double t = pymod1(1.0 - J->xs[s_a]);
    double lo = pymod1(t - J->eps);
    int64_t start = (int64_t)(k * lo);
    if (start >= k) start -= k; /* lo == 1.0 would index past the table */
    int64_t span = ((int64_t)(k * pymod1(t + J->eps)) - start) % k;
    if (span < 0) span += k;
    int64_t i = start, off = 0;
    while (off <= k) {
      double v = J->merged[2 * i];
      probes++;
      if (v < 0.0) {
        if (off >= span) break;
      } else {
        double delta = pymod1(v - t);
        if (delta < J->eps || delta > 1.0 - J->eps) {
          int64_t slot = __atomic_fetch_add(J->nout, 1, __ATOMIC_RELAXED);
          if (slot < J->cap) J->out[slot] = (uint64_t)s_a | ((uint64_t)J->merged[2 * i + 1] << J->na);
        }
      }
      off++;
      i++;
      if (i == k) i = 0;
    }
  }
  J->probes = probes;
  return NULL;
}

static int g_threads = 0; /* 0 = all online cores */

int orc_num_threads(void) {
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  if (g_threads > 0) return g_threads;
  return c > 0 ? (int)c : 1;
}

void orc_set_threads(int t) { g_threads = t; }

static int64_t stream_merged(const double *xs, int64_t lo_q, int64_t hi_q, const double *merged,
                             int64_t k, int na, double eps, uint64_t *out, int64_t cap,
                             int64_t *probes_out) {
  int T = orc_num_threads();
  if (T > 256) T = 256;
  if (hi_q - lo_q < 4096) T = 1;
  pthread_t th[256];
  stream_job jobs[256];
  int64_t nout = 0;
  for (int w = 0; w < T; w++) {
    jobs[w] = (stream_job){xs, merged, lo_q + (hi_q - lo_q) * w / T, lo_q + (hi_q - lo_q) * (w + 1) / T,
                           k, cap, na, eps, out, &nout, 0};
    if (T == 1) stream_worker(&jobs[w]);
    else pthread_create(&th[w], NULL, stream_worker, &jobs[w]);
  }
  int64_t probes = 0;
  for (int w = 0; w < T; w++) {
    if (T > 1) pthread_join(th[w], NULL);
    probes += jobs[w].probes;
  }
  *probes_out = probes;
  return nout;
}

/*
 * recombine_e (:727-775) minus the Python canonical filter, which is applied
 * by the caller on the raw output: builds the splat table of the high half,
 * then streams the A-queries with index in [q_lo, q_hi) (a bounded sample
 * when the caller asks for less than 2^na).  Returns the raw hit count;
 * stats[0..3] = inserts, insert_probes, queries, query_probes,
 * stats[4..5] = splat and query wall time in nanoseconds.
 * -1: allocation failure.
 */
int64_t orc_recombine_e_port(const double *rho, int n, double eps, int64_t q_lo, int64_t q_hi,
                             uint64_t *out, int64_t cap, int64_t *stats) {
    int na = n / 2, nb = n - na;
    double eps_d = eps + GUARD;
    double *bsums = subset_sums(rho + na, nb);
    double *asums = subset_sums(rho, na);
    if (!bsums || !asums) {
        free(bsums);
        free(asums);
        return -1;
    }
    int64_t nbv = (int64_t)1 << nb, nav = (int64_t)1 << na;
    for (int64_t i = 0; i < nbv; i++) bsums[i] -= floor(bsums[i]);
    for (int64_t i = 0; i < nav; i++) asums[i] -= floor(asums[i]);
    int64_t k = 2 * nbv;
    double *merged = (double *)malloc((size_t)(2 * k) * sizeof(double));
    if (!merged) {
        free(bsums);
        free(asums);
        return -1;
    }
    for (int64_t i = 0; i < k; i++) merged[2 * i] = -1.0;
    double t0 = now_s();
    int64_t ip = splat_merged(bsums, nbv, merged, k);
    double t1 = now_s();
    if (q_hi > nav) q_hi = nav;
    if (q_lo < 0) q_lo = 0;
    int64_t qp = 0;
    int64_t nout = stream_merged(asums, q_lo, q_hi, merged, k, na, eps_d, out, cap, &qp);
    double t2 = now_s();
    if (stats) {
        stats[0] = nbv;
        stats[1] = ip;
        stats[2] = q_hi - q_lo;
        stats[3] = qp;
        stats[4] = (int64_t)((t1 - t0) * 1e9);
        stats[5] = (int64_t)((t2 - t1) * 1e9);
    }
    free(merged);
    free(bsums);
    free(asums);
    return nout;
}

/* ---- verification restatement, R/verify.py:48-155 ----------------------- */

/* ld: long double (rfr_oracle.h) */

/*
 * build_candidate (R/verify.py:60-120): multiply out the selected reals and
 * pairs (reals first, then pairs, in ascending rho-index order), then the
 * power sums and their scales.  perm[i] < r: real root id, else pair id r+j.
 * coeffs: e+1 values (low to high), traces/scales: e values.  Returns e.
 */
int orc_build_candidate(uint64_t s, const double *real_roots, int r, const double *pair_sums,
                        const double *pair_products, int c, const int *perm, int n, ld *coeffs,
                        ld *traces, ld *scales) {
    ld reals[128];
    ld psum[128], pprod[128];
    int nr = 0, np = 0;
    (void)c;
    for (int i = 0; i < n && (s >> i); i++) {
        if (!((s >> i) & 1u)) continue;
        int ent = perm[i];
        if (ent < r) reals[nr++] = (ld)real_roots[ent];
        else {
            psum[np] = (ld)pair_sums[ent - r];
            pprod[np] = (ld)pair_products[ent - r];
            np++;
        }
    }
    int len = 1;
    ld cur[260], ext[260];
    cur[0] = 1.0L;
    for (int a = 0; a < nr; a++) {
        memset(ext, 0, sizeof(ld) * (len + 1));
        for (int j = 0; j < len; j++) ext[j + 1] += cur[j];
        for (int j = 0; j < len; j++) ext[j] -= reals[a] * cur[j];
        len += 1;
        memcpy(cur, ext, sizeof(ld) * len);
    }
    for (int a = 0; a < np; a++) {
        memset(ext, 0, sizeof(ld) * (len + 2));
        for (int j = 0; j < len; j++) ext[j + 2] += cur[j];
        for (int j = 0; j < len; j++) ext[j + 1] -= psum[a] * cur[j];
        for (int j = 0; j < len; j++) ext[j] += pprod[a] * cur[j];
        len += 2;
        memcpy(cur, ext, sizeof(ld) * len);
    }
    int e = len - 1;
    memcpy(coeffs, cur, sizeof(ld) * len);
    ld upow[128], uabs[128], pprev[128], pcur[128], pmag[128];
    for (int a = 0; a < nr; a++) {
        upow[a] = reals[a];
        uabs[a] = fabsl(reals[a]);
    }
    for (int a = 0; a < np; a++) {
        pprev[a] = 2.0L;
        pcur[a] = psum[a];
        pmag[a] = 2.0L * sqrtl(pprod[a]);
    }
    for (int m = 1; m <= e; m++) {
        ld tr = 0.0L, sc = 0.0L;
        for (int a = 0; a < nr; a++) {
            tr += upow[a];
            sc += uabs[a];
        }
        for (int a = 0; a < np; a++) {
            tr += pcur[a];
            sc += pmag[a];
        }
        traces[m - 1] = tr;
        scales[m - 1] = sc;
        if (m < e) {
            for (int a = 0; a < nr; a++) {
                upow[a] *= reals[a];
                uabs[a] *= fabsl(reals[a]);
            }
            for (int a = 0; a < np; a++) {
                ld nxt = psum[a] * pcur[a] - pprod[a] * pprev[a];
                pprev[a] = pcur[a];
                pcur[a] = nxt;
                pmag[a] *= sqrtl(pprod[a]);
            }
        }
    }
    return e;
}

/* trace_test (R/verify.py:123-138), _TRACE_REL = 1e-11, _INT_LIMIT = 2^62. */
int orc_trace_test(const ld *traces, const ld *scales, int e, double eps) {
    for (int m0 = 0; m0 < e; m0++) {
        int m = m0 + 1;
        double scale = (double)scales[m0];
        if (m * scale * 1e-11 >= eps || scale >= 4611686018427387904.0) continue;
        ld tr = traces[m0];
        if (fabs((double)(tr - rintl(tr))) >= eps) return 0;
    }
    return 1;
}

/*
 * Rounding half of round_and_divide (R/verify.py:141-154): 1 and the rounded
 * integers when every coefficient is within eps of an integer below 2^62.
 */
int orc_round_coeffs(const ld *coeffs, int e, double eps, int64_t *q) {
    for (int j = 0; j <= e; j++) {
        ld rr = rintl(coeffs[j]);
        if (fabs((double)(coeffs[j] - rr)) > eps) return 0;
        if (fabs((double)rr) >= 4611686018427387904.0) return 0;
        q[j] = (int64_t)rr;
    }
    return e >= 1;
}

/*
 * divide_exact (R/polynomial.py:155-183) on __int128: p (dp+1 coeffs) by q
 * (dq+1 coeffs).  1 and the quotient when exact, 0 when not divisible, -1
 * when a value leaves the int128 range (caller falls back to bigints).
 */
int orc_divide_exact_i128(const int64_t *p, int dp, const int64_t *q, int dq, int64_t *quot) {
    if (dp < dq) return 0;
    __int128 rem[260];
    for (int i = 0; i <= dp; i++) rem[i] = p[i];
    __int128 lq = q[dq];
    const __int128 LIM = (((__int128)1) << 120);
    for (int k = dp - dq; k >= 0; k--) {
        __int128 num = rem[k + dq];
        if (num == 0) {
            quot[k] = 0;
            continue;
        }
        if (num % lq) return 0;
        __int128 t = num / lq;
        if (t > ((__int128)INT64_MAX) || t < ((__int128)INT64_MIN)) return -1;
        quot[k] = (int64_t)t;
        for (int i = 0; i <= dq; i++) {
            rem[k + i] -= t * q[i];
            if (rem[k + i] > LIM || rem[k + i] < -LIM) return -1;
        }
    }
    for (int i = 0; i <= dp; i++)
        if (rem[i]) return 0;
    return 1;
}
