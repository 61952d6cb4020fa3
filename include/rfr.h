/*
 * rfr.h -- C ABI of the B200 recombination engine (librfr.so).
 *
 * The drop-in boundary of the reference's recombination path.  The reference
 * (/root/reference/pkg/src/polyfactor, "R/" below) is pure Python; its
 * operator interface for this path is the backend registry entry
 *     BACKENDS["e"] = recombine_e(rho: RhoVector, eps: float,
 *                                 stats: RecombineStats | None) -> CandidateSet
 * (R/recombine.py:727-784), its multi-worker twin parallel_recombine_e
 * (R/parallel.py:255-272), and the verification functions build_candidate /
 * trace_test / round_and_divide (R/verify.py:60-155) driven by
 * _factor_monic_squarefree (R/verify.py:246-286).  A maintainer binds these
 * entry points with ctypes; the Python host package
 * paper_2410_15880_b200 does exactly that.
 *
 * Conventions (R/verify.py, R/recombine.py ownership rules):
 *  - plain pointers and sizes; no torch or CUDA types in the signatures
 *    (streams are passed as void*; NULL = the library's own stream);
 *  - the caller allocates outputs and passes a capacity; the call returns the
 *    TRUE count, and when it exceeds the capacity the caller regrows and calls
 *    again (the reference's grow-and-retry protocol, R/recombine.py:750-757);
 *  - every call returns an rfr_status; on failure rfr_last_error() has the
 *    text.  The Python shim maps RFR_E_WIDTH -> WidthExceeded, RFR_E_ARG ->
 *    ValueError, everything else -> RuntimeError (R/errors.py:9-26).
 *  - calls are serialised per process (one internal mutex); device work runs
 *    on the device selected by rfr_init.
 */
#ifndef RFR_H
#define RFR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum rfr_status {
  RFR_OK = 0,
  RFR_E_ARG = 1,      /* bad argument                 -> ValueError     */
  RFR_E_WIDTH = 2,    /* n > 64 (pattern width cap)   -> WidthExceeded  */
  RFR_E_CAP = 3,      /* internal capacity exhausted  -> RuntimeError   */
  RFR_E_CUDA = 4,     /* CUDA runtime error           -> RuntimeError   */
  RFR_E_NOINIT = 5,   /* rfr_init not called          -> RuntimeError   */
  RFR_E_NUMERIC = 6   /* undecidable numerics         -> RuntimeError   */
} rfr_status;

/* Counters of one search; mirrors RecombineStats (R/recombine.py:82-103)
 * plus per-phase device times.  All fields are written by the call. */
typedef struct rfr_stats {
  int64_t visited;        /* records enumerated: 2^alpha + 2^beta (folded halves)   */
  int64_t inserts;        /* A records counting-sorted into shared memory           */
  int64_t insert_probes;  /* A outer-pointer checks                                 */
  int64_t queries;        /* B records streamed against the bins                    */
  int64_t query_probes;   /* A records compared against a B record                  */
  int64_t raw_hits;       /* patterns inside the key window                         */
  int64_t buckets;        /* key buckets processed by this shard                    */
  int64_t chunks;         /* extra A chunks (bucket overflowed shared memory)       */
  int32_t r_bits;         /* bucket bits of the plan                                */
  int32_t windows;        /* key sub-windows searched                               */
  double ms_lists;        /* device time: quarter-list build                        */
  double ms_join;         /* device time: bucket join                               */
  double ms_post;         /* device time: recheck / verification                    */
  double ms_total;        /* device time of the whole call                          */
  int64_t launches;       /* kernels launched by the call                            */
  int64_t buckets_planned; /* buckets the call set out to search; buckets < this     */
                           /* means the pattern space was not exhausted               */
  int64_t early_stop;      /* rfr_search_verify: the join stopped at a verified hit   */
  int32_t list_bits[4];    /* quarter-list widths of the plan: A outer, A inner,       */
                           /* B outer, B inner (0 for the exhaustive kernel)           */
  int64_t bytes_lists;     /* HBM bytes the list build moves by design: 12 B per base- */
                           /* level entry, then 8 B read + 8 B write per entry of      */
                           /* every doubling level (each level reads its input twice)  */
  int64_t bytes_join;      /* HBM bytes the join streams by design: one 8-byte inner   */
                           /* key per record of this shard's buckets                   */
  double us_hit_to_stop;   /* rfr_search_verify with early exit: microseconds from the */
                           /* poller's verified hit to the last join CTA leaving its   */
                           /* bucket loop (device clock); -1 when it did not stop      */
  int64_t pieces;          /* after an early stop: 0 the pieces were not searched in   */
                           /* the call, 1 searched by host-driven launches, 2 searched */
                           /* by kernels chained behind the main search on the device  */
} rfr_stats;

/* ---- lifecycle -------------------------------------------------------- */
/* Select the CUDA device, create the stream and scratch buffers.  Replaces
 * nothing in the reference (single-process Python); required once. */
int rfr_init(int device);
int rfr_shutdown(void);
const char* rfr_last_error(void);
int rfr_version(void);
int rfr_num_sms(void);

/* ---- search --------------------------------------------------------- */
/*
 * Parity-mode recombination: replaces recombine_e(rho, eps, stats)
 * (R/recombine.py:727-775) and, with nshards > 1, one worker's share of
 * parallel_recombine_e (R/parallel.py:255-272).
 * rho: n float64 values in [0, 1) (R/recombine.py:46-51; n <= 64).
 * Writes into out[0 .. min(count, cap)) the canonical patterns t < 2^(n-1)
 * with accept(value(t), eps) (R/recombine.py:106-162) whose key bucket falls
 * in this shard; *nout = true count.  Union over shards = the full set.
 * Output order is unspecified (the reference returns a frozenset).
 */
int rfr_recombine_e(const double* rho, int n, double eps, int shard, int nshards, uint64_t* out,
                    int64_t cap, int64_t* nout, rfr_stats* st);

/*
 * Factor-mode key-window search (the path factor() takes):
 * every pattern t < 2^(n-1) with (sum_{i in t} keys[i] - lo) mod 2^64 <= width.
 * keys: n uint64 fixed-point keys (host buffer).  Same output protocol.
 * Replaces the candidate search of _factor_monic_squarefree
 * (R/verify.py:261-268, recombine_e at the default backend).
 */
int rfr_search_keys(const uint64_t* keys, int n, uint64_t lo, uint64_t width, int shard,
                    int nshards, uint64_t* out, int64_t cap, int64_t* nout, rfr_stats* st);

/*
 * Factor-mode search with a secondary key: the patterns of rfr_search_keys
 * that also satisfy (sum_{i in t} keys2[i] - lo2) mod 2^64 <= width2, the
 * second window applied on the device to the raw hits.  keys2 are the
 * fixed-point fractional parts of the third power sums of the entities (an
 * integer for every true factor), so this adds the trace test of
 * R/verify.py:123-138 at m = 3 in front of verification; it cuts
 * Swinnerton-Dyer-like inputs, where Tr1 and Tr2 are integral for millions
 * of non-factors, to a handful of candidates.  Same output protocol.
 */
int rfr_search_keys2(const uint64_t* keys, int n, uint64_t lo, uint64_t width, const uint64_t* keys2,
                     uint64_t lo2, uint64_t width2, int shard, int nshards, uint64_t* out,
                     int64_t cap, int64_t* nout, rfr_stats* st);

/*
 * Device-resident variant for inputs already in HBM: d_keys (n uint64) and
 * d_out (cap uint64) are device pointers, *d_count a device uint64 that
 * receives the true count.  Enqueued on `stream` (cudaStream_t, NULL = the
 * library stream); no host synchronisation unless st != NULL.
 */
int rfr_search_keys_dev(const uint64_t* d_keys, int n, uint64_t lo, uint64_t width, int shard,
                        int nshards, uint64_t* d_out, int64_t cap, uint64_t* d_count,
                        void* stream, rfr_stats* st);

/* ---- verification ------------------------------------------------------ */

/* One polynomial's root profile in double-double (hi, lo) form: entity e
 * (0 <= e < r real roots, then c conjugate pairs) and the rho-index -> entity
 * map perm[n] (RootProfile, R/rootfinder.py:58-84).  Pairs carry the sum
 * t = z + conj(z) and product m = |z|^2 of x^2 - t x + m. */
typedef struct rfr_profile {
  int n, r, c;
  const double* real_hi;  /* r */
  const double* real_lo;
  const double* sum_hi;   /* c */
  const double* sum_lo;
  const double* prod_hi;  /* c */
  const double* prod_lo;
  const int32_t* perm;    /* n */
  double root_err;        /* absolute error bound on every root (host bound) */
} rfr_profile;

/* Verdicts written per candidate (rfr_verify). */
enum {
  RFR_V_REJECT = 0,  /* not a factor (trace / rounding / division mod primes) */
  RFR_V_PASS = 1,    /* integral, divides p modulo the three verify primes   */
  RFR_V_HOST = 2     /* coefficients beyond 2^62 or undecidable: host decides */
};

/*
 * Batched verification, one candidate per warp: replaces build_candidate ->
 * trace_test -> round_and_divide (R/verify.py:60-155) for every candidate of
 * one search.  For candidate k the smaller-degree side of {pat, complement}
 * is rebuilt in double-double, screened by power-sum integrality, rounded,
 * and trial-divided into p modulo three primes (2^31-1, 2^31-19, 2^31-61).
 *   pats[m]          candidate patterns (bit i = rho index i)
 *   p_mod[3*(d+1)]   coefficients of the monic input p (low->high) mod the
 *                    primes returned by rfr_verify_primes
 *   verdict[m]       RFR_V_* per candidate
 *   side[m]          1 if the complement side was rebuilt, else 0
 *   coeffs[m*stride] rounded int64 coefficients of the rebuilt side
 *                    (degree = selected degree; valid when PASS)
 */
int rfr_verify(const rfr_profile* prof, const uint64_t* pats, int64_t m, const uint64_t* p_mod,
               int d, uint8_t* verdict, uint8_t* side, int64_t* coeffs, int stride,
               rfr_stats* st);
/*
 * Fused factor-mode search and verification (one call per factor() search on
 * one device): rfr_search_keys2's candidate set, each candidate then verified
 * on the device exactly as rfr_verify does, without the patterns leaving HBM
 * in between.  Writes min(count, cap) patterns with their verdict / side /
 * coefficients (layouts as rfr_verify; coeffs valid for PASS); *nout = true
 * count (regrow and call again when it exceeds cap).  prof->n must equal n.
 * early_exit 1: early termination -- the hits are verified while the join
 * runs (a one-warp kernel on a second stream) and once one passes, with
 * pattern t, the join stops at its next bucket boundary; the pattern spaces
 * of the two pieces t and ~t are then searched in the same call (their hits
 * are factors of p too, reported as patterns of this search), so the output
 * covers every factor pattern (st->early_stop = 1, buckets == buckets_planned).
 * Pieces of >= 48 entities are left to the caller: buckets < buckets_planned
 * then says the pattern space was not exhausted.  early_exit 2: stop, never
 * search the pieces.  early_exit 0: the whole pattern space, as
 * rfr_search_keys2 + rfr_verify.
 */
int rfr_search_verify(const uint64_t* keys, int n, uint64_t lo, uint64_t width, const uint64_t* keys2,
                      uint64_t lo2, uint64_t width2, const rfr_profile* prof, const uint64_t* p_mod,
                      int d, uint64_t* pats, uint8_t* verdict, uint8_t* side, int64_t* coeffs,
                      int stride, int64_t cap, int early_exit, int64_t* nout, rfr_stats* st);

/*
 * One rank's share of a sharded fused search (the multi-GPU form of
 * rfr_search_verify, replacing parallel_recombine_e + the verification loop
 * on `nshards` workers, R/parallel.py:255-272, R/verify.py:236-284): the
 * buckets [shard 2^r / nshards, (shard+1) 2^r / nshards) of the same folded
 * pattern space; the union over shards is rfr_search_verify's output.  With
 * early_exit, a verified hit of this shard stops this rank's join AND, once
 * rfr_peer_connect has run, every other rank's join (their stop flags are
 * written over NVLink); a rank stopped by a peer returns with buckets <
 * buckets_planned, the rank that found the factor searches its pieces as
 * rfr_search_verify does.  epoch (1 .. 2^63 - 1): the same value on every rank
 * for the same search, different for successive searches (a call counter);
 * the stop flag carries it, so a peer's flag that lands early still counts and
 * a late one from an earlier search is ignored.
 */
int rfr_search_verify_shard(const uint64_t* keys, int n, uint64_t lo, uint64_t width,
                            const uint64_t* keys2, uint64_t lo2, uint64_t width2,
                            const rfr_profile* prof, const uint64_t* p_mod, int d, uint64_t* pats,
                            uint8_t* verdict, uint8_t* side, int64_t* coeffs, int stride, int64_t cap,
                            int early_exit, int shard, int nshards, uint64_t epoch, int64_t* nout,
                            rfr_stats* st);

/*
 * Cross-rank early exit (no reference counterpart: its workers share one
 * process).  rfr_peer_handle writes this process's 64-byte CUDA IPC handle of
 * its search counters (which hold the stop flag); the ranks all-gather the
 * handles (torch.distributed) and each calls rfr_peer_connect(handles[nranks
 * * 64], nranks, self) to map the others' flags.  rfr_peer_disconnect (and
 * rfr_shutdown) unmap them.
 */
int rfr_peer_handle(void* handle64);
int rfr_peer_connect(const void* handles, int nranks, int self);
int rfr_peer_disconnect(void);

/* The three primes of the modular division test (p_mod residues). */
int rfr_verify_primes(uint64_t* primes3);
/* p's coefficients modulo those three primes (the p_mod argument of
 * rfr_verify / rfr_search_verify, 3 x (d+1), Python's sign rule) from
 * signed 64-bit coefficients; RFR_E_ARG when some |c| >= 2^62. */
int rfr_p_mod_i64(const int64_t* coeffs, int d, uint64_t* p_mod);

/* ---- host-side numerics (native, not timed) ------------------------------ */
/*
 * Root polishing in double-double (Aberth-Ehrlich corrections) for a monic
 * polynomial with coefficients exactly representable in double-double:
 * coef_hi/lo[d+1] (low -> high), roots re/im hi/lo in/out (d each, seeded by
 * any approximation), err[d] out: a posteriori absolute error bound per root.
 * Returns RFR_OK or RFR_E_NUMERIC when it cannot certify the roots (the
 * caller then uses its multiprecision path).  Replaces find_roots'
 * iteration (R/rootfinder.py:100-174) as the host preprocessing step.
 */
int rfr_polish_roots(const double* coef_hi, const double* coef_lo, int d, double* re_hi,
                     double* re_lo, double* im_hi, double* im_lo, double* err, int max_iter);

/*
 * Square-free screen for the exact normalisation (R/polynomial.py:221-247):
 * 1 when gcd(p mod q, p' mod q) = 1 for a prime q dividing neither the
 * leading coefficient nor d (then p is square-free over Z), 0 when
 * undecided (q may divide the discriminant: try another prime).  Primes
 * below 2^25 take a double-precision path; larger ones 128-bit products.
 * coeffs_mod: p's coefficients reduced mod q (d+1), lead_mod != 0.
 */
int rfr_squarefree_mod(const uint64_t* coeffs_mod, int d, uint64_t q);
/*
 * The same screen from signed 64-bit coefficients, reduced mod q inside
 * (Python's sign rule): the factor() prologue calls this once per input, so
 * the reduction is not a separate host pass.  -1 when some |c| >= 2^62.
 */
int rfr_squarefree_i64(const int64_t* coeffs, int d, uint64_t q);
/*
 * Exact division by a monic divisor (R/polynomial.py:155-183 for monic q,
 * the only divisors factor() produces): r = p / q by long division in
 * 128-bit integers; r must hold dp - dq + 1 entries.  1: q divides p (r
 * filled), 0: it does not, -1: outside the native range (some |p_i| >=
 * 2^62, |q_i| >= 2^31 or quotient coefficient >= 2^62: the caller takes its
 * big-integer path).
 */
int rfr_divide_monic_i64(const int64_t* p, int dp, const int64_t* q, int dq, int64_t* r);
/*
 * Exact product of two polynomials with int64 coefficients (R/polynomial.py:
 * 142-152), accumulated in 128-bit integers: 1 with out (da + db + 1
 * entries) filled, -1 when a product coefficient reaches 2^62 or the
 * operands are too large to accumulate safely ((min(da, db) + 1) max|a|
 * max|b| >= 2^126); the caller then takes its big-integer path.
 */
int rfr_multiply_i64(const int64_t* a, int da, const int64_t* b, int db, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* RFR_H */
