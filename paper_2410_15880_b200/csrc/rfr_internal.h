// rfr_internal.h -- launchers shared between the kernel files and the C ABI.
#pragma once
#include <cuda_runtime.h>

#include "rfr_common.cuh"

namespace rfr {
size_t list_hist_bytes(int bits);
ListHist list_hist_layout(const JoinPlan& P, char* const base[4]);
int lists_launch_count(const JoinPlan& P);  // kernels launch_lists enqueues for this plan
cudaError_t launch_lists(const uint64_t* d_keys, const JoinPlan& P, ListBufs buf0, ListBufs buf1,
                         uint32_t* d_rot, ListHist H, cudaStream_t s);
cudaError_t launch_join(const JoinPlan& P, const ListBufs& fin, uint64_t* d_out,
                        unsigned long long cap, DevCounters* d_ctr, int grid, cudaStream_t s,
                        const uint32_t* d_rots, const uint32_t* d_starts,
                        unsigned long long stop_epoch = 0);
void dump_stop_trace(unsigned long long t_found, int grid);  // RFR_STOP_TRACE diagnostics
cudaError_t launch_join_starts(const JoinPlan& P, const ListBufs& fin, uint64_t b0, uint64_t b1,
                               int nck, int ctas, uint32_t* d_rots, uint32_t* d_starts, cudaStream_t s);
cudaError_t launch_index_to_pattern(const JoinPlan& P, const ListBufs& base, const ListHist& hist,
                                    const uint32_t* d_rot, uint64_t* d_out,
                                    const unsigned long long* d_count, unsigned long long cap, int nsm,
                                    cudaStream_t s, const unsigned long long* d_begin = nullptr);
cudaError_t launch_keyfilter(const uint64_t* d_keys2, int n, const uint64_t* d_in,
                             const unsigned long long* d_in_count, unsigned long long cap_in,
                             uint64_t lo2, uint64_t width2, uint64_t* d_out,
                             unsigned long long cap_out, DevCounters* d_ctr, int nsm, cudaStream_t s,
                             const unsigned long long* d_begin = nullptr);
// search_core: at or below this width one small-search kernel (table_search_kernel,
// an in-CTA meet in the middle) replaces the lists and the join
constexpr int kExhaustiveMaxN = 31;  // table vs join crossover (profiles/r2f_small_search.txt)
constexpr int kExhaustiveForceMaxN = 44;  // RFR_FORCE_EXHAUSTIVE (tests): up to 2^43 patterns, ~1 s
cudaError_t launch_table_search(const uint64_t* d_keys, int n, uint64_t lo, uint64_t width,
                                uint64_t* d_out, unsigned long long cap, DevCounters* d_ctr,
                                cudaStream_t s);
cudaError_t launch_exhaustive(const uint64_t* d_keys, int n, uint64_t lo, uint64_t width,
                              uint64_t* d_out, unsigned long long cap, DevCounters* d_ctr,
                              cudaStream_t s);
// Results of a fused call into pinned host memory (launch_collect).
struct CollectArgs {
  const DevCounters* ctr;
  const uint64_t* pats;
  const uint8_t* verdict;
  const uint8_t* side;
  const long long* coeffs;
  int stride;
  unsigned rows;  // at most this many rows
  DevCounters* h_ctr;
  uint64_t* h_pats;
  uint8_t* h_verdict;
  uint8_t* h_side;
  long long* h_coeffs;
  unsigned long long* clear = nullptr;  // optional: words zeroed after the copy (the next chain's counters)
  int clear_words = 0;
};
cudaError_t launch_collect(const CollectArgs& C, cudaStream_t s);
// The pieces of an early stop searched on the device behind the main search
// (launch_pieces, rfr_search.cu).
struct PieceDesc {
  unsigned long long t;        // the factor's pattern (parent bits)
  unsigned long long mask[2];  // piece 0 = t, piece 1 = its complement
  int ns[2];                   // entities per piece
  int active;                  // 0: no piece search (every piece kernel returns)
  int pad;
};
struct PiecePlanArgs {
  const DevCounters* ctr;       // the main search's counters
  unsigned long long planned;   // its planned buckets (fewer searched = stopped)
  unsigned long long raw_cap;   // its raw-hit capacity (an overflow is no stop)
  unsigned long long rows_cap;  // rows the caller takes (more: the host decides)
  const uint64_t* pats;         // its verified rows
  const uint8_t* verdict;
  const uint8_t* side;
  int n;
  const uint64_t* keys;  // the search's keys and Tr3 keys (n each)
  const uint64_t* keys2;
  PieceDesc* h_desc;   // pinned host copy of the plan (checked by the host)
  DevCounters* pctr;   // both pieces: raw hits and survivors (cleared beforehand)
  uint64_t* ppost;     // both pieces' survivors, as parent patterns
};
cudaError_t launch_pieces(const PiecePlanArgs& a, uint64_t lo, uint64_t width, uint64_t lo2, uint64_t width2,
                          unsigned long long post_cap, const struct VerifyArgs& V, const CollectArgs& C,
                          cudaStream_t s);
cudaError_t launch_deposit(uint64_t* d_pats, const unsigned long long* d_count, unsigned long long cap,
                           uint64_t mask, int nsm, cudaStream_t s);
cudaError_t launch_recheck(const double* d_rho, const uint64_t* d_in,
                           const unsigned long long* d_in_count, unsigned long long cap_in,
                           double eps, uint64_t* d_out, unsigned long long cap_out,
                           DevCounters* d_ctr, int nsm, cudaStream_t s);
cudaError_t launch_rho_keys(const double* d_rho, int n, uint64_t* d_keys, cudaStream_t s);

constexpr int kMaxPeers = 8;  // ranks of one sharded search whose stop flags a poller raises

// Batched candidate verification (rfr_verify.cu): one warp per candidate.
struct VerifyArgs {
  int n, r, c, d;
  const double* real_hi;
  const double* real_lo;
  const double* sum_hi;
  const double* sum_lo;
  const double* prod_hi;
  const double* prod_lo;
  const int32_t* perm;
  double root_err;
  const uint64_t* pats;
  long long m;                            // candidates (grid bound)
  const unsigned long long* m_dev;        // optional device count (<= m), or null
  const unsigned long long* m_begin_dev = nullptr;  // optional first candidate (chunked search)
  unsigned long long* found = nullptr;    // optional flag raised by a PASS (early exit)
  unsigned long long found_value = 1;     // the value raised: the search's epoch
  // with found: the same flag of the other ranks' searches (their DevCounters
  // opened through CUDA IPC, written over NVLink), so one rank's verified
  // factor stops every rank's join at its next bucket boundary
  unsigned long long* peer_found[kMaxPeers] = {};
  int npeers = 0;
  unsigned long long* t_found = nullptr;  // with found: globaltimer of the first PASS
  unsigned long long* t_probe = nullptr;  // diagnostics: phase timestamps of one verification
  // integral, monic coefficients suffice for a PASS (the caller divides
  // exactly anyway): the speculative early-exit candidate, whose modular
  // division would sit on the critical path of every early stop
  int skip_division = 0;
  const uint64_t* p_mod;  // 3 x (d+1)
  uint64_t primes[3];
  uint8_t* verdict;
  uint8_t* side;
  long long* coeffs;
  int stride;
};
cudaError_t launch_verify(const VerifyArgs& A, cudaStream_t s);
cudaError_t launch_early_exit_poller(const JoinPlan& P, const ListBufs& base, const ListHist& hist,
                                     const uint32_t* d_rot, uint64_t* d_out, unsigned long long raw_cap,
                                     const uint64_t* d_keys2, int n, uint64_t lo2, uint64_t width2,
                                     uint64_t* d_post, unsigned long long post_cap, const VerifyArgs& V,
                                     DevCounters* d_ctr, int join_ctas, cudaStream_t s);
// Primes of the modular division test, P = 2^31 - c with small c (products
// fit 64-bit registers, two folds reduce them): 2^31 - 1, 2^31 - 19,
// 2^31 - 61.  The test is a filter: every factor the host keeps is confirmed
// by exact division.
constexpr uint64_t kVerifyPrimes[3] = {2147483647ull, 2147483629ull, 2147483587ull};
}  // namespace rfr
