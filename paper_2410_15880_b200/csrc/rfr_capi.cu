// rfr_capi.cu -- the C ABI of librfr.so (declared in include/rfr.h).
//
// Owns the per-process device context (stream, scratch buffers, counters) and
// turns one search request into: key upload -> quarter-list build -> one
// bucket-join launch per key sub-window -> optional recheck -> result copy.
// The grow-and-retry protocol of the reference (recombine.py:750-757) is kept
// for the internal raw-hit buffer and exposed to the caller for its output.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rfr.h"
#include "rfr_common.cuh"
#include <ctime>

#include "rfr_internal.h"

using namespace rfr;


namespace {

std::mutex g_mu;

// RFR_HOST_TRACE=1: host timestamps at the steps of a fused call, printed to
// stderr when it returns (where the C host time of factor() goes).
struct HostTrace {
  int on = -1;
  std::vector<std::pair<const char*, double>> marks;
  static double now() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
  }
  void mark(const char* what) {
    if (on < 0) on = getenv("RFR_HOST_TRACE") ? 1 : 0;
    if (on) marks.emplace_back(what, now());
  }
  void dump() {
    if (on != 1 || marks.empty()) return;
    const double t0 = marks[0].second;
    for (auto& m : marks) fprintf(stderr, "[rfr host] %8.1f us  %s\n", m.second - t0, m.first);
    marks.clear();
  }
};
HostTrace g_tr;
thread_local std::string g_err;

struct DevVec {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t b = want < 4096 ? 4096 : want;
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

struct Ctx {
  bool ready = false;
  int device = -1;
  int nsm = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // early-exit poller, beside the join
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // ev[4]: after the chained pieces
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_fill = nullptr;
  DevVec keys, keys2, rho, raw, post, ctr, rotc, jstarts, pkeys;
  DevVec hist[4];  // merge history per list (pattern recovery)
  DevVec vprof, vpats, vpmod, vverd, vside, vcoef;  // verification scratch
  DevVec pctr, praw, ppost;  // the two pieces' counters / raw hits / survivors (concurrent)
  DevVec pver;               // the chained pieces' verification rows
  DevVec lk[4][2], lp[4][2];  // list keys / patterns, ping-pong
  DevCounters* h_ctr = nullptr;  // pinned mirror
  void* h_stage = nullptr;       // pinned staging of rfr_verify (in, then out)
  size_t h_stage_bytes = 0;
  void* h_piece = nullptr;       // pinned staging of the pieces' searches after an early stop
  size_t h_piece_bytes = 0;
  // cross-rank early exit: the other ranks' DevCounters.found, opened by IPC
  void* peer_base[kMaxPeers] = {};
  unsigned long long* peer_found[kMaxPeers] = {};
  int npeers = 0;
  // cache of the last built lists (key values + plan geometry)
  std::vector<uint64_t> built_keys;
  int built_bits[4] = {-1, -1, -1, -1};
  const void* built_src = nullptr;
};
Ctx g;

}  // namespace

int rfr_fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int rfr_fail_cuda(cudaError_t e, const char* what) {
  return rfr_fail(RFR_E_CUDA, "CUDA error %s (%s) in %s", cudaGetErrorName(e),
                  cudaGetErrorString(e), what);
}

static int rfr_check_cuda(cudaError_t e, const char* what) {
  return e == cudaSuccess ? RFR_OK : rfr_fail_cuda(e, what);
}

namespace {

int bit_length(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

// Plan the quarter lists and buckets of one search.
int make_plan(int n, uint64_t lo, uint64_t width, int nshards, JoinPlan* P) {
  memset(P, 0, sizeof *P);
  const int m = n - 1;
  const int alpha = (m + 1) / 2, beta = m - alpha;
  int r = alpha - kJoinRecLog;  // ~2^kJoinRecLog A records per bucket
  if (r < 2) r = 2;
  const uint64_t half = (width >> 1) + (width & 1);
  const int hb = bit_length(half);
  if (r > 61 - hb) r = 61 - hb;  // keep the window radius <= W / 8
  if (r < 2) return rfr_fail(RFR_E_ARG, "window too wide for one plan (internal)");
  auto clampi = [](int v, int lo_, int hi_) { return v < lo_ ? lo_ : (v > hi_ ? hi_ : v); };
  // outer lists: at least one outer per join warp per side, and runs of at
  // most 2^lam records per outer per bucket.  Default 128:
  // since the run passes are compiled for fixed chunk counts (join v17) the
  // join pays only ~6 % for 128 against 256, while the inner lists and their
  // build halve (C3: lists 0.41 -> 0.26 ms; RFR_LAMBDA_LOG=8: 256); inner
  // lists capped at 2^kMaxInnerBits entries (streamed)
  static int lam = -1;
  if (lam < 0) {
    const char* e = getenv("RFR_LAMBDA_LOG");
    lam = e ? atoi(e) : 7;
  }
  int warps_log = 0;
  while ((1 << (warps_log + 1)) <= kJoinThreadsPerCta / 32) warps_log++;
  // every shard rebuilds the whole quarter lists while the join is split
  // nshards ways, so shorter runs (smaller inner lists) pay off on many GPUs
  // (round 1, measured at n = 55 with the join then: 256 was best up to 2
  // shards, 128 at 4, 64-128 at 8)
  const int lam_s = lam - (nshards >= 4 ? 1 : 0) - (nshards >= 16 ? 1 : 0);
  auto outer_bits = [&](int side) {
    const int want = side - r - lam_s > warps_log ? side - r - lam_s : warps_log;
    return clampi(want, side > kMaxInnerBits ? side - kMaxInnerBits : 0,
                  side < kMaxOuterBits ? side : kMaxOuterBits);
  };
  const int ao = outer_bits(alpha), bo = outer_bits(beta);
  const int ai = alpha - ao, bi = beta - bo;
  if (ai > kMaxInnerBits || bi > kMaxInnerBits)
    return rfr_fail(RFR_E_WIDTH, "inner list too large (n=%d)", n);
  P->n = n;
  P->m = m;
  P->list[0] = {0, ao, 0, 0};
  P->list[1] = {ao, ai, 0, ao};
  P->list[2] = {alpha, bo, 1, alpha};
  P->list[3] = {alpha + bo, bi, 1, alpha + bo};
  P->r = r;
  P->nbins_log = clampi(alpha - r, 1, 12);
  P->lo = lo;
  P->width = width;
  P->shift = lo + (width >> 1);
  P->half = half;
  return RFR_OK;
}

int ensure_ready() {
  if (!g.ready) return rfr_fail(RFR_E_NOINIT, "rfr_init was not called");
  return RFR_OK;
}

ListBufs bufs(int which) {
  ListBufs b;
  for (int i = 0; i < 4; i++) {
    b.k[i] = (uint64_t*)g.lk[i][which].p;
    b.p[i] = (uint32_t*)g.lp[i][which].p;
  }
  return b;
}

ListBufs final_bufs(const JoinPlan& P) {
  ListBufs b;
  for (int i = 0; i < 4; i++) {
    int which = P.list[i].bits > kBaseBits ? ((P.list[i].bits - kBaseBits) & 1) : 0;
    b.k[i] = (uint64_t*)g.lk[i][which].p;
    b.p[i] = (uint32_t*)g.lp[i][which].p;
  }
  return b;
}

int ensure_list_buffers(const JoinPlan& P) {
  for (int i = 0; i < 4; i++) {
    size_t len = (size_t)1 << P.list[i].bits;
    if (len < 4096) len = 4096;
    for (int w = 0; w < 2; w++) RFR_CUDA_OK(g.lk[i][w].ensure(len * sizeof(uint64_t)));
    // patterns live only at the base level (longer lists keep a merge history)
    RFR_CUDA_OK(g.lp[i][0].ensure(((size_t)1 << kBaseBits) * sizeof(uint32_t)));
    const size_t hb = list_hist_bytes(P.list[i].bits);
    RFR_CUDA_OK(g.hist[i].ensure(hb ? hb : 16));
  }
  return RFR_OK;
}

// Split [lo, lo + width] into pieces whose radius fits a plan with r >= 2.
std::vector<std::pair<uint64_t, uint64_t>> split_window(uint64_t lo, uint64_t width) {
  std::vector<std::pair<uint64_t, uint64_t>> out;
  const uint64_t piece = (1ull << 59) - 1;  // width of one piece (radius < 2^58 + 1)
  if (width <= piece) {
    out.push_back({lo, width});
    return out;
  }
  uint64_t done = 0;  // covered [lo, lo + done)
  while (true) {
    uint64_t rem = width - done;  // remaining inclusive span minus one
    uint64_t w = rem < piece ? rem : piece;
    out.push_back({lo + done, w});
    if (w == rem) break;
    done += w + 1;
  }
  return out;
}

double ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return (double)ms;
}

// Early termination for rfr_search_verify: the hits are verified while the
// join runs (early_exit_poller_kernel on stream2) and the join stops at a
// bucket boundary once one passes.
struct EarlyExit {
  const uint64_t* d_keys2;
  uint64_t lo2, width2;
  uint64_t* d_post;
  unsigned long long post_cap;
  VerifyArgs V;
};

// Core search on device-resident keys.  d_out/cap: raw output; counters in
// g.ctr.  ee (one key window only): early termination as above; the hits the
// poller did not reach are left from DevCounters.raw_done on (patterns
// recovered here, filter and verification by the caller).
int g_launches = 0;                // kernels launched by the last search_core call
int64_t g_buckets_planned = 0;     // buckets the last search_core call set out to search
int g_list_bits[4] = {0, 0, 0, 0}; // quarter-list widths of the last search_core plan

int search_core(const uint64_t* d_keys, int n, uint64_t lo, uint64_t width, int shard, int nshards,
                uint64_t* d_out, unsigned long long cap, cudaStream_t s, int* r_bits,
                int* nwin, bool time_it, const EarlyExit* ee = nullptr) {
  g_launches = 0;
  g_buckets_planned = 0;
  for (int i = 0; i < 4; i++) g_list_bits[i] = 0;
  // RFR_FORCE_JOIN (tests): keep small searches on the quarter-list join so
  // the oracle parity tests cover both paths
  // RFR_FORCE_EXHAUSTIVE (tests): the exhaustive kernel up to n = 44, the
  // independent checker of the join's hit set at production geometry
  const bool small = n <= kExhaustiveMaxN && !getenv("RFR_FORCE_JOIN");
  const bool forced = n <= kExhaustiveForceMaxN && getenv("RFR_FORCE_EXHAUSTIVE") != nullptr;
  if (nshards == 1 && n >= 2 && (small || forced)) {
    // small search: every folded pattern in one launch (same hit set as the join)
    *nwin = 1;
    *r_bits = 0;
    if (time_it) RFR_CUDA_OK(cudaEventRecord(g.ev[0], s));
    if (time_it) RFR_CUDA_OK(cudaEventRecord(g.ev[1], s));
    // RFR_FORCE_EXHAUSTIVE: the Gray-code brute force (the checker); else the
    // in-CTA meet in the middle (RFR_SMALL_EXHAUSTIVE=1: brute force, A/B)
    if (forced || getenv("RFR_SMALL_EXHAUSTIVE"))
      RFR_CUDA_OK(launch_exhaustive(d_keys, n, lo, width, d_out, cap, (DevCounters*)g.ctr.p, s));
    else
      RFR_CUDA_OK(launch_table_search(d_keys, n, lo, width, d_out, cap, (DevCounters*)g.ctr.p, s));
    g_launches = 1;
    if (time_it) RFR_CUDA_OK(cudaEventRecord(g.ev[2], s));
    return RFR_OK;
  }
  std::vector<std::pair<uint64_t, uint64_t>> wins = split_window(lo, width);
  *nwin = (int)wins.size();
  g_tr.mark("search_core: plan");
  JoinPlan P0;
  int rc = make_plan(n, wins[0].first, wins[0].second, nshards, &P0);
  if (rc) return rc;
  *r_bits = P0.r;
  for (int i = 0; i < 4; i++) g_list_bits[i] = P0.list[i].bits;
  rc = ensure_list_buffers(P0);
  if (rc) return rc;
  if (time_it) RFR_CUDA_OK(cudaEventRecord(g.ev[0], s));
  RFR_CUDA_OK(g.rotc.ensure(4 * kRotSlots * sizeof(uint32_t)));
  char* hb[4];
  for (int i = 0; i < 4; i++) hb[i] = (char*)g.hist[i].p;
  const ListHist H = list_hist_layout(P0, hb);
  DevCounters* d_ctr = (DevCounters*)g.ctr.p;
  const bool early = ee != nullptr && wins.size() == 1;
  g_tr.mark("search_core: lists launch");
  RFR_CUDA_OK(launch_lists(d_keys, P0, bufs(0), bufs(1), (uint32_t*)g.rotc.p, H, s));
  g_tr.mark("search_core: lists enqueued");
  if (early) {
    // the raw-hit slots start as kUnsetHit (the poller's "not yet written"):
    // filled on the second stream while the lists are built
    RFR_CUDA_OK(cudaMemsetAsync(d_out, 0xff, cap * sizeof(uint64_t), g.stream2));
    RFR_CUDA_OK(cudaEventRecord(g.ev_fill, g.stream2));
  }
  g_launches += lists_launch_count(P0);
  if (time_it) RFR_CUDA_OK(cudaEventRecord(g.ev[1], s));
  for (auto& w : wins) {
    // every piece reuses the geometry planned for the widest (first) piece
    JoinPlan P = P0;
    P.lo = w.first;
    P.width = w.second;
    P.shift = w.first + (w.second >> 1);
    P.half = (w.second >> 1) + (w.second & 1);
    const uint64_t nb = 1ull << P.r;
    P.bucket_begin = nb * (uint64_t)shard / (uint64_t)nshards;
    P.bucket_end = nb * (uint64_t)(shard + 1) / (uint64_t)nshards;
    const uint64_t span = P.bucket_end - P.bucket_begin;
    if (span == 0) continue;
    g_buckets_planned += (int64_t)span;
    // resident join CTAs; with early exit one slot stays free for the poller
    const int ctas = g.nsm * kJoinCtasPerSm - (early ? 1 : 0);
    const int grid = (int)(span < (uint64_t)ctas ? span : (uint64_t)ctas);
    // rotation starts and the per-CTA start positions, up front
    const size_t mot = ((size_t)1 << P.list[0].bits) + ((size_t)1 << P.list[2].bits);
    RFR_CUDA_OK(g.jstarts.ensure(mot * (1 + (size_t)grid) * sizeof(uint32_t)));
    uint32_t* d_rots = (uint32_t*)g.jstarts.p;
    RFR_CUDA_OK(launch_join_starts(P, final_bufs(P0), P.bucket_begin, P.bucket_end, 1, grid, d_rots,
                                   d_rots + mot, s));
    g_launches += 1;
    g_tr.mark("search_core: join starts");
    if (early) {
      RFR_CUDA_OK(cudaStreamWaitEvent(s, g.ev_fill, 0));  // kUnsetHit slots
      RFR_CUDA_OK(cudaEventRecord(g.ev_fork, s));
      RFR_CUDA_OK(cudaStreamWaitEvent(g.stream2, g.ev_fork, 0));
      RFR_CUDA_OK(launch_early_exit_poller(P0, bufs(0), H, (const uint32_t*)g.rotc.p, d_out, cap,
                                           ee->d_keys2, n, ee->lo2, ee->width2, ee->d_post,
                                           ee->post_cap, ee->V, d_ctr, grid, g.stream2));
      RFR_CUDA_OK(cudaEventRecord(g.ev_join, g.stream2));
      g_launches += 1;
    }
    g_tr.mark("search_core: poller");
    RFR_CUDA_OK(launch_join(P, final_bufs(P0), d_out, cap, d_ctr, grid, s, d_rots, d_rots + mot,
                             early ? ee->V.found_value : 0ull));
    g_launches += 1;
    g_tr.mark("search_core: join");
    if (early) RFR_CUDA_OK(cudaStreamWaitEvent(s, g.ev_join, 0));
  }
  // the join emits quarter-list indices; rewrite every hit (the poller's
  // already are, up to raw_done) as its pattern
  RFR_CUDA_OK(launch_index_to_pattern(P0, bufs(0), H, (const uint32_t*)g.rotc.p, d_out,
                                      &d_ctr->out_count, cap, g.nsm, s,
                                      early ? &d_ctr->raw_done : nullptr));
  g_launches += 1;
  if (time_it) RFR_CUDA_OK(cudaEventRecord(g.ev[2], s));
  return RFR_OK;
}

void fill_stats(rfr_stats* st, const DevCounters& c, int n, int r_bits, int nwin) {
  if (!st) return;
  memset(st, 0, sizeof *st);
  st->us_hit_to_stop = -1.0;
  const int m = n - 1;
  const int alpha = (m + 1) / 2, beta = m - alpha;
  st->visited = n > 0 ? (int64_t)((1ull << alpha) + (1ull << beta)) : 0;
  st->inserts = (int64_t)c.inserts;
  st->insert_probes = (int64_t)c.insert_probes;
  st->queries = (int64_t)c.queries;
  st->query_probes = (int64_t)c.query_probes;
  st->raw_hits = (int64_t)c.out_count;
  st->buckets = (int64_t)c.buckets;
  st->chunks = (int64_t)c.chunks;
  st->r_bits = r_bits;
  st->windows = nwin;
  st->launches = g_launches;
  st->buckets_planned = g_buckets_planned;
  int64_t lb = 0;
  for (int i = 0; i < 4; i++) {
    st->list_bits[i] = g_list_bits[i];
    const int b = g_list_bits[i], b0 = b < kBaseBits ? b : kBaseBits;
    lb += 12ll << b0;                        // base level: key + pattern
    if (b > b0) lb += 32ll * ((1ll << b) - (1ll << b0));  // doubling levels
  }
  st->bytes_lists = g_list_bits[1] + g_list_bits[3] ? lb : 0;
  // records of the planned buckets (a bucket holds 2^-r of each folded half)
  st->bytes_join = r_bits > 0 ? (int64_t)((double)st->visited * 8.0 *
                                          (double)g_buckets_planned / (double)(1ull << r_bits))
                              : 0;
}

// The profile's doubles packed for one H2D copy: [real_hi | real_lo | sum_hi |
// sum_lo | prod_hi | prod_lo | 0], 2r + 4c + 1 entries (absent lo parts are 0).
void stage_profile(double* hp, const rfr_profile* prof) {
  const int r = prof->r, c = prof->c;
  for (int i = 0; i < r; i++) {
    hp[i] = prof->real_hi[i];
    hp[r + i] = prof->real_lo ? prof->real_lo[i] : 0.0;
  }
  for (int j = 0; j < c; j++) {
    hp[2 * r + j] = prof->sum_hi[j];
    hp[2 * r + c + j] = prof->sum_lo ? prof->sum_lo[j] : 0.0;
    hp[2 * r + 2 * c + j] = prof->prod_hi[j];
    hp[2 * r + 3 * c + j] = prof->prod_lo ? prof->prod_lo[j] : 0.0;
  }
  hp[2 * r + 4 * c] = 0.0;
}

// Verification arguments over a staged profile on the device (the doubles at
// d_prof, the permutation at d_perm, p mod the verify primes at d_pmod); the
// caller fills the candidate and output fields.
VerifyArgs bind_profile(const rfr_profile* prof, int d, const char* d_prof, const char* d_perm,
                        const char* d_pmod) {
  const int r = prof->r, c = prof->c;
  VerifyArgs A;
  A.n = prof->n;
  A.r = r;
  A.c = c;
  A.d = d;
  const double* dp = (const double*)d_prof;
  A.real_hi = dp;
  A.real_lo = dp + r;
  A.sum_hi = dp + 2 * r;
  A.sum_lo = dp + 2 * r + c;
  A.prod_hi = dp + 2 * r + 2 * c;
  A.prod_lo = dp + 2 * r + 3 * c;
  A.perm = (const int32_t*)d_perm;
  A.root_err = prof->root_err;
  A.p_mod = (const uint64_t*)d_pmod;
  for (int i = 0; i < 3; i++) A.primes[i] = kVerifyPrimes[i];
  return A;
}

// Shape and pointer checks shared by rfr_verify and rfr_search_verify.
int check_profile(const rfr_profile* prof, int d) {
  if (!prof) return rfr_fail(RFR_E_ARG, "null profile");
  if (prof->n < 0 || prof->r < 0 || prof->c < 0) return rfr_fail(RFR_E_ARG, "negative profile sizes");
  if (prof->n > 64) return rfr_fail(RFR_E_WIDTH, "pattern width is capped at 64 bits");
  if (prof->r + 2 * prof->c != d || prof->r + prof->c != prof->n)
    return rfr_fail(RFR_E_ARG, "profile does not match the degree");
  if ((prof->r && !prof->real_hi) || (prof->c && (!prof->sum_hi || !prof->prod_hi)) ||
      (prof->n && !prof->perm))
    return rfr_fail(RFR_E_ARG, "null profile array");
  if (!(prof->root_err >= 0.0))  // +inf is allowed: every candidate comes back undecided
    return rfr_fail(RFR_E_ARG, "root_err must be >= 0 (got NaN or a negative bound)");
  return RFR_OK;
}

// After an early stop on the verified pattern t (rfr_search_verify): search
// the pattern spaces of the two pieces t and ~t here, so the caller gets a
// complete candidate set in one call.  A piece's hits are factors of p too,
// so each piece is searched over the parent's keys at its bits (with the
// parent's windows: its own error bounds are smaller) and its survivors are
// deposited back into parent patterns and verified with the parent's
// arguments (V0).  Rows are appended to xp/xv/xs/xc.  false with *rc == 0: not
// done here (a piece with >= kPieceMaxN entities, or more than kPieceRows
// survivors) -- the caller reports the stop and the host factors the pieces.
constexpr int kPieceMaxN = 48;   // whole-space searches above this size stop early themselves
constexpr int kPieceRows = 64;
constexpr unsigned long long kPieceRaw = 1ull << 16;  // raw hits per small piece (concurrent path)

// Pinned piece area: per piece [keys | keys2][64], its counters and
// kPieceRows result rows; then both pieces' keys (one H2D) and the device
// plan's PieceDesc.
size_t piece_per(int stride) {
  return 2 * 64 * 8 + sizeof(DevCounters) + kPieceRows * (10 + (size_t)stride * 8);
}
int ensure_piece_host(int stride) {
  const size_t hbytes = 2 * piece_per(stride) + 2 * 2 * 64 * sizeof(uint64_t) + sizeof(PieceDesc);
  if (g.h_piece_bytes >= hbytes) return RFR_OK;
  if (g.h_piece) cudaFreeHost(g.h_piece);
  g.h_piece = nullptr;
  g.h_piece_bytes = 0;
  int rc = rfr_check_cuda(cudaMallocHost(&g.h_piece, hbytes), "cudaMallocHost");
  if (rc == RFR_OK) g.h_piece_bytes = hbytes;
  return rc;
}
PieceDesc* piece_h_desc(int stride) {
  return (PieceDesc*)((char*)g.h_piece + 2 * piece_per(stride) + 2 * 2 * 64 * sizeof(uint64_t));
}
// The collected rows of the pieces with >= 2 entities; false on an overflow
// (more raw hits than raw_cap or more survivors than kPieceRows).
// The rows of the chained piece searches (one pinned area: counters, then
// up to 2 kPieceRows rows of both pieces); false when they did not fit.
bool read_chained_piece_rows(int stride, std::vector<uint64_t>& xp, std::vector<uint8_t>& xv,
                             std::vector<uint8_t>& xs, std::vector<int64_t>& xc) {
  const char* hp = (const char*)g.h_piece;
  const DevCounters c = *(const DevCounters*)hp;
  const unsigned rows_cap = 2 * kPieceRows;
  if (c.post_count > (unsigned long long)rows_cap) return false;
  const char* rows = hp + sizeof(DevCounters);
  for (unsigned long long k = 0; k < c.post_count; k++) {
    xp.push_back(((const uint64_t*)rows)[k]);
    xv.push_back(((const uint8_t*)(rows + rows_cap * 8))[k]);
    xs.push_back(((const uint8_t*)(rows + rows_cap * 9))[k]);
    const int64_t* cr = (const int64_t*)(rows + rows_cap * 10) + k * stride;
    xc.insert(xc.end(), cr, cr + stride);
  }
  return true;
}

bool read_piece_rows(int stride, const int ns[2], unsigned long long raw_cap, std::vector<uint64_t>& xp,
                     std::vector<uint8_t>& xv, std::vector<uint8_t>& xs, std::vector<int64_t>& xc,
                     int64_t* buckets) {
  const size_t per = piece_per(stride);
  for (int pi = 0; pi < 2; pi++) {
    if (ns[pi] < 2) continue;
    const char* hp = (const char*)g.h_piece + pi * per;
    const DevCounters c = *(const DevCounters*)(hp + 2 * 64 * 8);
    if (c.out_count > raw_cap || c.post_count > (unsigned long long)kPieceRows) return false;
  }
  for (int pi = 0; pi < 2; pi++) {
    if (ns[pi] < 2) continue;
    const char* hp = (const char*)g.h_piece + pi * per;
    const DevCounters c = *(const DevCounters*)(hp + 2 * 64 * 8);
    const char* rows = hp + 2 * 64 * 8 + sizeof(DevCounters);
    for (unsigned long long k = 0; k < c.post_count; k++) {
      xp.push_back(((const uint64_t*)rows)[k]);
      xv.push_back(((const uint8_t*)(rows + kPieceRows * 8))[k]);
      xs.push_back(((const uint8_t*)(rows + kPieceRows * 9))[k]);
      const int64_t* cr = (const int64_t*)(rows + kPieceRows * 10) + k * stride;
      xc.insert(xc.end(), cr, cr + stride);
    }
    *buckets += (int64_t)c.buckets;
  }
  return true;
}

// search_pieces for two small pieces: the table kernel, the Tr3 window, the
// deposit into parent patterns, the verification and the collection of each
// piece on its own stream (g.stream and g.stream2), with its own counters,
// raw and survivor buffers and verification rows.  Returns false when a
// piece overflows (the caller's incomplete-search path takes over).
bool search_small_pieces(const uint64_t* keys, const uint64_t* keys2, uint64_t lo, uint64_t width,
                         uint64_t lo2, uint64_t width2, const uint64_t masks[2], const VerifyArgs& V0,
                         int stride, cudaStream_t s, size_t per, std::vector<uint64_t>& xp,
                         std::vector<uint8_t>& xv, std::vector<uint8_t>& xs, std::vector<int64_t>& xc,
                         int64_t* buckets, int* rc) {
  auto ok = [&](cudaError_t e, const char* what) { return (*rc = rfr_check_cuda(e, what)) == RFR_OK; };
  if (!ok(g.pctr.ensure(2 * sizeof(DevCounters)), "piece counters") ||
      !ok(g.praw.ensure(2 * kPieceRaw * sizeof(uint64_t)), "piece raw") ||
      !ok(g.ppost.ensure(2 * kPieceRaw * sizeof(uint64_t)), "piece post"))
    return false;
  // both pieces' keys in one copy, staged after the two pieces' row areas:
  // [piece][keys | keys2][64]
  int ns[2] = {0, 0};
  uint64_t* stage = (uint64_t*)((char*)g.h_piece + 2 * per);
  const size_t stage_b = 2 * 128 * sizeof(uint64_t);
  for (int pi = 0; pi < 2; pi++) {
    int j = 0;
    for (uint64_t mm = masks[pi]; mm; mm &= mm - 1, j++) {
      const int i = __builtin_ctzll(mm);
      stage[pi * 128 + j] = keys[i];
      stage[pi * 128 + 64 + j] = keys2[i];
    }
    ns[pi] = j;
  }
  if (!ok(cudaMemcpyAsync(g.pkeys.p, stage, stage_b, cudaMemcpyHostToDevice, s), "piece keys") ||
      !ok(cudaMemsetAsync(g.pctr.p, 0, 2 * sizeof(DevCounters), s), "piece counters") ||
      !ok(cudaEventRecord(g.ev_fork, s), "fork") || !ok(cudaStreamWaitEvent(g.stream2, g.ev_fork, 0), "fork wait"))
    return false;
  // per piece: table search, Tr3 window, deposit, verification, collection;
  // the launches of the two pieces alternate so neither stream waits on the
  // host while the other's are enqueued
  VerifyArgs A[2];
  CollectArgs C[2];
  for (int pi = 0; pi < 2; pi++) {
    DevCounters* ctr = (DevCounters*)g.pctr.p + pi;
    uint64_t* post = (uint64_t*)g.ppost.p + pi * kPieceRaw;
    A[pi] = V0;
    A[pi].pats = post;
    A[pi].m = kPieceRows;
    A[pi].m_dev = &ctr->post_count;
    A[pi].m_begin_dev = nullptr;
    A[pi].found = nullptr;
    A[pi].verdict = V0.verdict + pi * kPieceRows;
    A[pi].side = V0.side + pi * kPieceRows;
    A[pi].coeffs = V0.coeffs + (size_t)pi * kPieceRows * stride;
    char* hp = (char*)g.h_piece + pi * per;
    char* rows = hp + 2 * 64 * 8 + sizeof(DevCounters);
    C[pi].ctr = ctr;
    C[pi].pats = post;
    C[pi].verdict = A[pi].verdict;
    C[pi].side = A[pi].side;
    C[pi].coeffs = A[pi].coeffs;
    C[pi].stride = stride;
    C[pi].rows = kPieceRows;
    C[pi].h_ctr = (DevCounters*)(hp + 2 * 64 * 8);
    C[pi].h_pats = (uint64_t*)rows;
    C[pi].h_verdict = (uint8_t*)(rows + kPieceRows * 8);
    C[pi].h_side = (uint8_t*)(rows + kPieceRows * 9);
    C[pi].h_coeffs = (long long*)(rows + kPieceRows * 10);
  }
  for (int stage = 0; stage < 5; stage++) {
    for (int pi = 0; pi < 2; pi++) {
      if (ns[pi] < 2) continue;  // one linear or quadratic entity: irreducible
      cudaStream_t sp = pi ? g.stream2 : s;
      DevCounters* ctr = (DevCounters*)g.pctr.p + pi;
      uint64_t* dk = (uint64_t*)g.pkeys.p + pi * 128;
      uint64_t* raw = (uint64_t*)g.praw.p + pi * kPieceRaw;
      uint64_t* post = (uint64_t*)g.ppost.p + pi * kPieceRaw;
      cudaError_t e = cudaSuccess;
      switch (stage) {
        case 0: e = launch_table_search(dk, ns[pi], lo, width, raw, kPieceRaw, ctr, sp); break;
        case 1:
          e = launch_keyfilter(dk + 64, ns[pi], raw, &ctr->out_count, kPieceRaw, lo2, width2, post, kPieceRaw,
                               ctr, g.nsm, sp);
          break;
        case 2: e = launch_deposit(post, &ctr->post_count, kPieceRaw, masks[pi], g.nsm, sp); break;
        case 3: e = launch_verify(A[pi], sp); break;
        default: e = launch_collect(C[pi], sp); break;
      }
      if (!ok(e, "piece search")) return false;
    }
  }
  if (!ok(cudaEventRecord(g.ev_join, g.stream2), "join") || !ok(cudaStreamWaitEvent(s, g.ev_join, 0), "join wait") ||
      !ok(cudaStreamSynchronize(s), "piece sync"))
    return false;
  return read_piece_rows(stride, ns, kPieceRaw, xp, xv, xs, xc, buckets);
}
bool search_pieces(const uint64_t* keys, const uint64_t* keys2, int n, uint64_t lo, uint64_t width,
                   uint64_t lo2, uint64_t width2, uint64_t t, const VerifyArgs& V0, int stride,
                   cudaStream_t s, std::vector<uint64_t>& xp, std::vector<uint8_t>& xv,
                   std::vector<uint8_t>& xs, std::vector<int64_t>& xc, int64_t* buckets, int* rc) {
  *rc = RFR_OK;
  const uint64_t full = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
  const uint64_t masks[2] = {t & full, ~t & full};
  for (uint64_t M : masks)
    if (__builtin_popcountll(M) >= kPieceMaxN) return false;
  const size_t per = piece_per(stride);
  if ((*rc = ensure_piece_host(stride))) return false;
  if ((*rc = rfr_check_cuda(g.pkeys.ensure(2 * 2 * 64 * sizeof(uint64_t)), "pkeys"))) return false;
  // both pieces small (the table kernel): searched concurrently, one on each
  // stream, each with its own counters and buffers, one synchronisation
  if (__builtin_popcountll(masks[0]) <= kExhaustiveMaxN && __builtin_popcountll(masks[1]) <= kExhaustiveMaxN &&
      !getenv("RFR_FORCE_JOIN") && !getenv("RFR_SMALL_EXHAUSTIVE"))
    return search_small_pieces(keys, keys2, lo, width, lo2, width2, masks, V0, stride, s, per, xp, xv, xs,
                               xc, buckets, rc);
  DevCounters* d_ctr = (DevCounters*)g.ctr.p;
  const unsigned long long raw_cap = g.raw.bytes / sizeof(uint64_t);
  const unsigned long long post_cap = g.post.bytes / sizeof(uint64_t);
  uint64_t* d_post = (uint64_t*)g.post.p;
  bool used[2] = {false, false};
  for (int pi = 0; pi < 2; pi++) {
    const uint64_t M = masks[pi];
    const int ns = __builtin_popcountll(M);
    if (ns < 2) continue;  // one linear or quadratic entity: irreducible
    used[pi] = true;
    char* hp = (char*)g.h_piece + pi * per;
    uint64_t* hk = (uint64_t*)hp;
    int j = 0;
    for (uint64_t mm = M; mm; mm &= mm - 1, j++) {
      const int i = __builtin_ctzll(mm);
      hk[j] = keys[i];
      hk[64 + j] = keys2[i];
    }
    uint64_t* dk = (uint64_t*)g.pkeys.p + pi * 128;
    auto ok = [&](cudaError_t e, const char* what) { return (*rc = rfr_check_cuda(e, what)) == RFR_OK; };
    if (!ok(cudaMemcpyAsync(dk, hk, 2 * 64 * sizeof(uint64_t), cudaMemcpyHostToDevice, s), "piece keys") ||
        !ok(cudaMemsetAsync(d_ctr, 0, sizeof(DevCounters), s), "piece counters"))
      return false;
    int rb = 0, nw = 0;
    if ((*rc = search_core(dk, ns, lo, width, 0, 1, (uint64_t*)g.raw.p, raw_cap, s, &rb, &nw, false)))
      return false;
    VerifyArgs A = V0;
    A.pats = d_post;
    A.m_dev = &d_ctr->post_count;
    A.m_begin_dev = nullptr;
    A.found = nullptr;
    char* rows = hp + 2 * 64 * 8 + sizeof(DevCounters);
    if (!ok(launch_keyfilter(dk + 64, ns, (const uint64_t*)g.raw.p, &d_ctr->out_count, raw_cap, lo2, width2,
                             d_post, post_cap, d_ctr, g.nsm, s), "piece keyfilter") ||
        !ok(launch_deposit(d_post, &d_ctr->post_count, post_cap, M, g.nsm, s), "deposit"))
      return false;
    CollectArgs C;
    C.ctr = d_ctr;
    C.pats = d_post;
    C.verdict = A.verdict;
    C.side = A.side;
    C.coeffs = A.coeffs;
    C.stride = stride;
    C.rows = kPieceRows;
    C.h_ctr = (DevCounters*)(hp + 2 * 64 * 8);
    C.h_pats = (uint64_t*)rows;
    C.h_verdict = (uint8_t*)(rows + kPieceRows * 8);
    C.h_side = (uint8_t*)(rows + kPieceRows * 9);
    C.h_coeffs = (long long*)(rows + kPieceRows * 10);
    if (!ok(launch_verify(A, s), "piece verify") || !ok(launch_collect(C, s), "piece collect"))
      return false;
  }
  if ((*rc = rfr_check_cuda(cudaStreamSynchronize(s), "piece sync"))) return false;
  for (int pi = 0; pi < 2; pi++) {
    if (!used[pi]) continue;
    const char* hp = (const char*)g.h_piece + pi * per;
    const DevCounters c = *(const DevCounters*)(hp + 2 * 64 * 8);
    if (c.out_count > raw_cap || c.post_count > (unsigned long long)kPieceRows) return false;
    const char* rows = hp + 2 * 64 * 8 + sizeof(DevCounters);
    for (unsigned long long k = 0; k < c.post_count; k++) {
      xp.push_back(((const uint64_t*)rows)[k]);
      xv.push_back(((const uint8_t*)(rows + kPieceRows * 8))[k]);
      xs.push_back(((const uint8_t*)(rows + kPieceRows * 9))[k]);
      const int64_t* cr = (const int64_t*)(rows + kPieceRows * 10) + k * stride;
      xc.insert(xc.end(), cr, cr + stride);
    }
    *buckets += (int64_t)c.buckets;
  }
  return true;
}

int check_n(int n) {
  if (n < 0) return rfr_fail(RFR_E_ARG, "negative width");
  if (n > 64) return rfr_fail(RFR_E_WIDTH, "pattern width is capped at 64 bits, got %d", n);
  return RFR_OK;
}

}  // namespace

extern "C" {

int rfr_version(void) { return 1; }

const char* rfr_last_error(void) { return g_err.c_str(); }

int rfr_num_sms(void) { return g.nsm; }

// Free everything the context holds (safe on a partially initialised one).
static void release_ctx() {
  for (int i = 0; i < g.npeers; i++) cudaIpcCloseMemHandle(g.peer_base[i]);
  g.npeers = 0;
  if (g.stream) cudaStreamSynchronize(g.stream);
  DevVec* vecs[] = {&g.keys, &g.keys2, &g.rho, &g.raw, &g.post, &g.ctr, &g.rotc, &g.jstarts, &g.pkeys,
                    &g.vprof, &g.vpats, &g.vpmod, &g.vverd, &g.vside, &g.vcoef, &g.pctr, &g.praw,
                    &g.ppost, &g.pver};
  for (DevVec* v : vecs) v->release();
  for (auto& h : g.hist) h.release();
  for (auto& a : g.lk)
    for (auto& v : a) v.release();
  for (auto& a : g.lp)
    for (auto& v : a) v.release();
  for (auto& e : g.ev)
    if (e) cudaEventDestroy(e);
  if (g.ev_fork) cudaEventDestroy(g.ev_fork);
  if (g.ev_join) cudaEventDestroy(g.ev_join);
  if (g.ev_fill) cudaEventDestroy(g.ev_fill);
  if (g.stream2) cudaStreamDestroy(g.stream2);
  if (g.h_ctr) cudaFreeHost(g.h_ctr);
  if (g.h_stage) cudaFreeHost(g.h_stage);
  if (g.h_piece) cudaFreeHost(g.h_piece);
  if (g.stream) cudaStreamDestroy(g.stream);
  g = Ctx();
}

static int init_ctx(int device) {
  RFR_CUDA_OK(cudaSetDevice(device));
  cudaDeviceProp prop;
  RFR_CUDA_OK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return rfr_fail(RFR_E_CUDA, "librfr is built for sm_100a; device %d is sm_%d%d", device,
                    prop.major, prop.minor);
  g.device = device;
  g.nsm = prop.multiProcessorCount;
  RFR_CUDA_OK(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
  RFR_CUDA_OK(cudaStreamCreateWithFlags(&g.stream2, cudaStreamNonBlocking));
  for (auto& e : g.ev) RFR_CUDA_OK(cudaEventCreate(&e));
  RFR_CUDA_OK(cudaEventCreateWithFlags(&g.ev_fork, cudaEventDisableTiming));
  RFR_CUDA_OK(cudaEventCreateWithFlags(&g.ev_join, cudaEventDisableTiming));
  RFR_CUDA_OK(cudaEventCreateWithFlags(&g.ev_fill, cudaEventDisableTiming));
  RFR_CUDA_OK(g.ctr.ensure(sizeof(DevCounters)));
  RFR_CUDA_OK(cudaMallocHost(&g.h_ctr, sizeof(DevCounters)));
  RFR_CUDA_OK(g.keys.ensure(64 * sizeof(uint64_t)));
  RFR_CUDA_OK(g.rho.ensure(64 * sizeof(double)));
  RFR_CUDA_OK(g.raw.ensure((1u << 20) * sizeof(uint64_t)));
  RFR_CUDA_OK(g.post.ensure((1u << 20) * sizeof(uint64_t)));
  return RFR_OK;
}

int rfr_init(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g.ready && g.device == device) return RFR_OK;
  if (g.ready) return rfr_fail(RFR_E_ARG, "already initialised on device %d", g.device);
  int ndev = 0;
  RFR_CUDA_OK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return rfr_fail(RFR_E_ARG, "no CUDA device %d", device);
  const int rc = init_ctx(device);
  if (rc) {
    const std::string why = g_err;  // release_ctx must not mask the first error
    release_ctx();
    g_err = why;
    return rc;
  }
  g.ready = true;
  return RFR_OK;
}

int rfr_shutdown(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g.ready) return RFR_OK;
  cudaSetDevice(g.device);
  release_ctx();
  return RFR_OK;
}

static int run_search_host(const uint64_t* h_keys, const double* h_rho, int n, uint64_t lo,
                           uint64_t width, double eps, int shard, int nshards, uint64_t* out,
                           int64_t cap, int64_t* nout, rfr_stats* st,
                           const uint64_t* h_keys2 = nullptr, uint64_t lo2 = 0, uint64_t width2 = 0) {
  int rc = ensure_ready();
  if (rc) return rc;
  if ((rc = check_n(n))) return rc;
  if (nshards < 1 || shard < 0 || shard >= nshards) return rfr_fail(RFR_E_ARG, "bad shard");
  if (cap < 0 || !nout) return rfr_fail(RFR_E_ARG, "bad output buffer");
  cudaSetDevice(g.device);
  cudaStream_t s = g.stream;
  if (n == 0) {
    *nout = 0;
    fill_stats(st, DevCounters{}, 0, 0, 0);
    return RFR_OK;
  }
  const bool parity = (h_rho != nullptr);
  if (parity) {
    RFR_CUDA_OK(cudaMemcpyAsync(g.rho.p, h_rho, n * sizeof(double), cudaMemcpyHostToDevice, s));
    RFR_CUDA_OK(launch_rho_keys((const double*)g.rho.p, n, (uint64_t*)g.keys.p, s));
  } else {
    RFR_CUDA_OK(cudaMemcpyAsync(g.keys.p, h_keys, n * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    if (h_keys2) {
      RFR_CUDA_OK(g.keys2.ensure(64 * sizeof(uint64_t)));
      RFR_CUDA_OK(cudaMemcpyAsync(g.keys2.p, h_keys2, n * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    }
  }
  int r_bits = 0, nwin = 0;
  unsigned long long raw_cap = g.raw.bytes / sizeof(uint64_t);
  DevCounters* d_ctr = (DevCounters*)g.ctr.p;
  for (int attempt = 0; attempt < 3; attempt++) {
    RFR_CUDA_OK(cudaMemsetAsync(d_ctr, 0, sizeof(DevCounters), s));
    rc = search_core((const uint64_t*)g.keys.p, n, lo, width, shard, nshards, (uint64_t*)g.raw.p,
                     raw_cap, s, &r_bits, &nwin, true);
    if (rc) return rc;
    RFR_CUDA_OK(cudaMemcpyAsync(g.h_ctr, d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
    RFR_CUDA_OK(cudaStreamSynchronize(s));
    if (g.h_ctr->out_count <= raw_cap) break;
    if (attempt == 2) return rfr_fail(RFR_E_CAP, "raw hit buffer regrow failed");
    unsigned long long want = g.h_ctr->out_count + (g.h_ctr->out_count >> 3) + 1024;
    if (want > (1ull << 31)) return rfr_fail(RFR_E_CAP, "%llu raw hits exceed the 2^31 limit",
                                             (unsigned long long)g.h_ctr->out_count);
    RFR_CUDA_OK(g.raw.ensure(want * sizeof(uint64_t)));
    raw_cap = g.raw.bytes / sizeof(uint64_t);
  }
  DevCounters c = *g.h_ctr;
  const uint64_t* d_res = (const uint64_t*)g.raw.p;
  unsigned long long count = c.out_count;
  if (parity) {
    RFR_CUDA_OK(g.post.ensure((count ? count : 1) * sizeof(uint64_t)));
    g_launches += 1;
    RFR_CUDA_OK(launch_recheck((const double*)g.rho.p, (const uint64_t*)g.raw.p, &d_ctr->out_count,
                               raw_cap, eps, (uint64_t*)g.post.p,
                               g.post.bytes / sizeof(uint64_t), d_ctr, g.nsm, s));
    RFR_CUDA_OK(cudaEventRecord(g.ev[3], s));
    RFR_CUDA_OK(cudaMemcpyAsync(g.h_ctr, d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
    RFR_CUDA_OK(cudaStreamSynchronize(s));
    c = *g.h_ctr;
    count = c.post_count;
    d_res = (const uint64_t*)g.post.p;
  } else if (h_keys2) {
    // secondary key window on the device; the survivors are a subset of the
    // raw hits, so copying min(raw, cap) entries with the counters needs no
    // second synchronisation
    RFR_CUDA_OK(g.post.ensure((count ? count : 1) * sizeof(uint64_t)));
    g_launches += 1;
    RFR_CUDA_OK(launch_keyfilter((const uint64_t*)g.keys2.p, n, (const uint64_t*)g.raw.p,
                                 &d_ctr->out_count, raw_cap, lo2, width2, (uint64_t*)g.post.p,
                                 g.post.bytes / sizeof(uint64_t), d_ctr, g.nsm, s));
    RFR_CUDA_OK(cudaEventRecord(g.ev[3], s));
    RFR_CUDA_OK(cudaMemcpyAsync(g.h_ctr, d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
    const unsigned long long pre = count < (unsigned long long)cap ? count : (unsigned long long)cap;
    if (pre)
      RFR_CUDA_OK(cudaMemcpyAsync(out, g.post.p, pre * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    RFR_CUDA_OK(cudaStreamSynchronize(s));
    c = *g.h_ctr;
    count = c.post_count;
    *nout = (int64_t)count;
    if (st) {
      fill_stats(st, c, n, r_bits, nwin);
      st->raw_hits = (int64_t)c.out_count;
      st->ms_lists = ev_ms(g.ev[0], g.ev[1]);
      st->ms_join = ev_ms(g.ev[1], g.ev[2]);
      st->ms_post = ev_ms(g.ev[2], g.ev[3]);
      st->ms_total = ev_ms(g.ev[0], g.ev[3]);
    }
    return RFR_OK;
  } else {
    RFR_CUDA_OK(cudaEventRecord(g.ev[3], s));
  }
  const unsigned long long ncopy = count < (unsigned long long)cap ? count : (unsigned long long)cap;
  if (ncopy)
    RFR_CUDA_OK(cudaMemcpyAsync(out, d_res, ncopy * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  RFR_CUDA_OK(cudaStreamSynchronize(s));
  *nout = (int64_t)count;
  if (st) {
    fill_stats(st, c, n, r_bits, nwin);
    st->raw_hits = (int64_t)c.out_count;
    st->ms_lists = ev_ms(g.ev[0], g.ev[1]);
    st->ms_join = ev_ms(g.ev[1], g.ev[2]);
    st->ms_post = ev_ms(g.ev[2], g.ev[3]);
    st->ms_total = ev_ms(g.ev[0], g.ev[3]);
  }
  return RFR_OK;
}

int rfr_recombine_e(const double* rho, int n, double eps, int shard, int nshards, uint64_t* out,
                    int64_t cap, int64_t* nout, rfr_stats* st) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!rho && n > 0) return rfr_fail(RFR_E_ARG, "null rho");
  if (!(eps > 0.0 && eps < 0.5)) return rfr_fail(RFR_E_ARG, "eps must be in (0, 0.5)");
  for (int i = 0; i < n; i++)
    if (!(rho[i] >= 0.0 && rho[i] < 1.0)) return rfr_fail(RFR_E_ARG, "rho entries must lie in [0, 1)");
  // window: every t with accept(value(t), eps) has |frac| < eps + GUARD
  // (recombine.py:28-30), and the key sum is within n/2 of 2^64 * exact sum.
  const double eps_d = eps + 1e-12;
  const double t = std::ceil(std::ldexp(eps_d, 64));
  uint64_t lo = 0, width = ~0ull;
  if (t < 9.0e18) {
    const uint64_t T = (uint64_t)t + (uint64_t)n + 4096;
    if (T < (1ull << 63)) {
      lo = 0ull - T;
      width = 2 * T;
    }
  }
  return run_search_host(nullptr, rho, n, lo, width, eps, shard, nshards, out, cap, nout, st);
}

int rfr_search_keys(const uint64_t* keys, int n, uint64_t lo, uint64_t width, int shard,
                    int nshards, uint64_t* out, int64_t cap, int64_t* nout, rfr_stats* st) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!keys && n > 0) return rfr_fail(RFR_E_ARG, "null keys");
  return run_search_host(keys, nullptr, n, lo, width, 0.0, shard, nshards, out, cap, nout, st);
}

// Fused factor-mode search + verification: lists, join, secondary key window
// and the verify kernel back to back on the device (the candidate patterns
// never round-trip through the host); one staged H2D in, one batch of D2H out.
namespace {
int search_verify_impl(const uint64_t* keys, int n, uint64_t lo, uint64_t width, const uint64_t* keys2,
                       uint64_t lo2, uint64_t width2, const rfr_profile* prof, const uint64_t* p_mod,
                       int d, uint64_t* pats, uint8_t* verdict, uint8_t* side, int64_t* coeffs,
                       int stride, int64_t cap, int early_exit, int shard, int nshards,
                       unsigned long long epoch, int64_t* nout, rfr_stats* st);
unsigned long long g_local_epoch = 0;  // epochs of unsharded searches (high bit set)
}  // namespace

int rfr_search_verify(const uint64_t* keys, int n, uint64_t lo, uint64_t width, const uint64_t* keys2,
                      uint64_t lo2, uint64_t width2, const rfr_profile* prof, const uint64_t* p_mod,
                      int d, uint64_t* pats, uint8_t* verdict, uint8_t* side, int64_t* coeffs,
                      int stride, int64_t cap, int early_exit, int64_t* nout, rfr_stats* st) {
  std::lock_guard<std::mutex> lk(g_mu);
  return search_verify_impl(keys, n, lo, width, keys2, lo2, width2, prof, p_mod, d, pats, verdict, side,
                            coeffs, stride, cap, early_exit, 0, 1, (1ull << 63) | ++g_local_epoch, nout, st);
}

int rfr_search_verify_shard(const uint64_t* keys, int n, uint64_t lo, uint64_t width,
                            const uint64_t* keys2, uint64_t lo2, uint64_t width2,
                            const rfr_profile* prof, const uint64_t* p_mod, int d, uint64_t* pats,
                            uint8_t* verdict, uint8_t* side, int64_t* coeffs, int stride, int64_t cap,
                            int early_exit, int shard, int nshards, uint64_t epoch, int64_t* nout,
                            rfr_stats* st) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (nshards < 1 || shard < 0 || shard >= nshards) return rfr_fail(RFR_E_ARG, "bad shard");
  if (epoch == 0 || (epoch >> 63)) return rfr_fail(RFR_E_ARG, "epoch must be in [1, 2^63)");
  return search_verify_impl(keys, n, lo, width, keys2, lo2, width2, prof, p_mod, d, pats, verdict, side,
                            coeffs, stride, cap, early_exit, shard, nshards, epoch, nout, st);
}

// ---- cross-rank early exit: the ranks' stop flags over CUDA IPC -----------
int rfr_peer_handle(void* handle) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc = ensure_ready();
  if (rc) return rc;
  if (!handle) return rfr_fail(RFR_E_ARG, "null handle");
  cudaSetDevice(g.device);
  cudaIpcMemHandle_t h;
  RFR_CUDA_OK(cudaIpcGetMemHandle(&h, g.ctr.p));
  memcpy(handle, &h, sizeof h);
  return RFR_OK;
}

int rfr_peer_connect(const void* handles, int nranks, int self) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc = ensure_ready();
  if (rc) return rc;
  if (!handles || nranks < 1 || self < 0 || self >= nranks || nranks - 1 > kMaxPeers)
    return rfr_fail(RFR_E_ARG, "bad peer handles");
  cudaSetDevice(g.device);
  for (int i = 0; i < g.npeers; i++) cudaIpcCloseMemHandle(g.peer_base[i]);
  g.npeers = 0;
  for (int r = 0; r < nranks; r++) {
    if (r == self) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + (size_t)r * sizeof h, sizeof h);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int i = 0; i < g.npeers; i++) cudaIpcCloseMemHandle(g.peer_base[i]);
      g.npeers = 0;
      cudaGetLastError();
      return rfr_fail_cuda(e, "cudaIpcOpenMemHandle");
    }
    g.peer_base[g.npeers] = p;
    g.peer_found[g.npeers] = (unsigned long long*)((char*)p + offsetof(DevCounters, found));
    g.npeers++;
  }
  return RFR_OK;
}

int rfr_peer_disconnect(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g.ready) cudaSetDevice(g.device);
  for (int i = 0; i < g.npeers; i++) cudaIpcCloseMemHandle(g.peer_base[i]);
  g.npeers = 0;
  return RFR_OK;
}

namespace {
int search_verify_impl(const uint64_t* keys, int n, uint64_t lo, uint64_t width, const uint64_t* keys2,
                       uint64_t lo2, uint64_t width2, const rfr_profile* prof, const uint64_t* p_mod,
                       int d, uint64_t* pats, uint8_t* verdict, uint8_t* side, int64_t* coeffs,
                       int stride, int64_t cap, int early_exit, int shard, int nshards,
                       unsigned long long epoch, int64_t* nout, rfr_stats* st) {
  int rc = ensure_ready();
  if (rc) return rc;
  if ((rc = check_n(n))) return rc;
  if (!nout || cap < 0 || stride < 1 || !p_mod || d < 1 || d > 128 || (cap > 0 && !pats))
    return rfr_fail(RFR_E_ARG, "bad search_verify arguments");
  if ((rc = check_profile(prof, d))) return rc;
  if (prof->n != n) return rfr_fail(RFR_E_ARG, "profile does not match the keys");
  if (n == 0) {
    *nout = 0;
    fill_stats(st, DevCounters{}, 0, 0, 0);
    return RFR_OK;
  }
  if (!keys || !keys2) return rfr_fail(RFR_E_ARG, "null keys");
  g_tr.mark("enter search_verify");
  cudaSetDevice(g.device);
  g_tr.mark("cudaSetDevice");
  cudaStream_t s = g.stream;
  // ---- inputs: [keys | keys2 | profile doubles | perm | p_mod], one H2D
  const int r = prof->r, c = prof->c;
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  const size_t nd = (size_t)(2 * r + 4 * c + 1);
  const size_t o_keys2 = al((size_t)n * 8);
  const size_t o_prof = o_keys2 + al((size_t)n * 8);
  const size_t o_perm = o_prof + al(nd * sizeof(double));
  const size_t o_pmod = o_perm + al((size_t)n * sizeof(int32_t));
  const size_t in_bytes = o_pmod + al((size_t)3 * (d + 1) * sizeof(uint64_t));
  if (g.h_stage_bytes < in_bytes) {
    if (g.h_stage) cudaFreeHost(g.h_stage);
    g.h_stage = nullptr;
    g.h_stage_bytes = 0;
    RFR_CUDA_OK(cudaMallocHost(&g.h_stage, in_bytes));
    g.h_stage_bytes = in_bytes;
  }
  char* hs = (char*)g.h_stage;
  memcpy(hs, keys, (size_t)n * 8);
  memcpy(hs + o_keys2, keys2, (size_t)n * 8);
  stage_profile((double*)(hs + o_prof), prof);
  memcpy(hs + o_perm, prof->perm, (size_t)n * sizeof(int32_t));
  memcpy(hs + o_pmod, p_mod, (size_t)3 * (d + 1) * sizeof(uint64_t));
  g_tr.mark("inputs staged");
  RFR_CUDA_OK(g.vprof.ensure(in_bytes));
  char* base = (char*)g.vprof.p;
  // never overlap an early-exit poller of an earlier call (one that ended in
  // an error after its launch): it still reads the counters (no-op otherwise)
  RFR_CUDA_OK(cudaStreamWaitEvent(s, g.ev_join, 0));
  g_tr.mark("wait event");
  RFR_CUDA_OK(cudaMemcpyAsync(base, hs, in_bytes, cudaMemcpyHostToDevice, s));
  g_tr.mark("inputs staged, H2D enqueued");
  const uint64_t* d_keys = (const uint64_t*)base;
  const uint64_t* d_keys2 = (const uint64_t*)(base + o_keys2);
  // ---- search, secondary window and verification back to back with no host
  // round trip: every kernel clamps to the counts the previous one left on
  // the device, and the first rows come back with the counters (one
  // synchronisation for a typical call).  A raw-hit overflow regrows and
  // reruns; more survivors than the speculative rows cost a second copy.
  constexpr size_t kSpecRows = 64;
  int r_bits = 0, nwin = 0;
  DevCounters* d_ctr = (DevCounters*)g.ctr.p;
  // verification rows: the caller regrows beyond its cap, so max(cap, 4096)
  // rows bound every useful call (sizing by the raw count cost 12 GB on
  // Swinnerton-Dyer f6)
  const size_t vrows = (size_t)(cap > 4096 ? cap : 4096);
  const size_t q_side = al(vrows), q_coef = q_side + al(vrows);
  RFR_CUDA_OK(g.vcoef.ensure(q_coef + vrows * (size_t)stride * sizeof(int64_t)));
  char* obase = (char*)g.vcoef.p;
  const size_t spec = (size_t)cap < kSpecRows ? (size_t)cap : kSpecRows;
  const size_t h_verd = al(vrows * 8), h_side = h_verd + al(vrows), h_coef = h_side + al(vrows);
  auto copy_rows = [&](size_t from, size_t to) -> cudaError_t {  // device rows [from, to) -> staging
    if (to <= from) return cudaSuccess;
    const size_t k = to - from;
    cudaError_t e = cudaMemcpyAsync(hs + from * 8, (const char*)g.post.p + from * 8, k * 8,
                                    cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(hs + h_verd + from, obase + from, k, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(hs + h_side + from, obase + q_side + from, k, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(hs + h_coef + from * stride * 8, obase + q_coef + from * stride * 8,
                          k * (size_t)stride * 8, cudaMemcpyDeviceToHost, s);
    return e;
  };
  bool dev_pieces = false;
  for (int attempt = 0;; attempt++) {
    const unsigned long long raw_cap = g.raw.bytes / sizeof(uint64_t);
    RFR_CUDA_OK(g.post.ensure(raw_cap * sizeof(uint64_t)));
    const unsigned long long post_cap = g.post.bytes / sizeof(uint64_t);
    // the counters, but not the stop flag: a peer's flag for this epoch may
    // already be there
    RFR_CUDA_OK(cudaMemsetAsync(d_ctr, 0, offsetof(DevCounters, found), s));
    // Tr3 window over the raw hits from *begin on, then verification of the
    // survivors from *vbegin on (null: all); found: flag a PASS raises
    auto filter_verify = [&](const unsigned long long* begin, const unsigned long long* vbegin,
                             unsigned long long* found) -> int {
      RFR_CUDA_OK(launch_keyfilter(d_keys2, n, (const uint64_t*)g.raw.p, &d_ctr->out_count, raw_cap,
                                   lo2, width2, (uint64_t*)g.post.p, post_cap, d_ctr, g.nsm, s, begin));
      VerifyArgs A = bind_profile(prof, d, base + o_prof, base + o_perm, base + o_pmod);
      A.pats = (const uint64_t*)g.post.p;
      A.m = (long long)vrows;
      A.m_dev = &d_ctr->post_count;
      A.m_begin_dev = vbegin;
      A.found = found;
      A.verdict = (uint8_t*)obase;
      A.side = (uint8_t*)(obase + q_side);
      A.coeffs = (long long*)(obase + q_coef);
      A.stride = stride;
      RFR_CUDA_OK(launch_verify(A, s));
      g_launches += 2;
      return RFR_OK;
    };
    EarlyExit ee;
    ee.d_keys2 = d_keys2;
    ee.lo2 = lo2;
    ee.width2 = width2;
    ee.d_post = (uint64_t*)g.post.p;
    ee.post_cap = post_cap;
    ee.V = bind_profile(prof, d, base + o_prof, base + o_perm, base + o_pmod);
    ee.V.pats = (const uint64_t*)g.post.p;
    ee.V.m = (long long)vrows;
    ee.V.m_dev = nullptr;
    ee.V.found = &d_ctr->found;
    ee.V.found_value = epoch;
    ee.V.t_found = &d_ctr->t_found;
    if (g_tr.on == 1) ee.V.t_probe = &d_ctr->t_probe[0];
    ee.V.verdict = (uint8_t*)obase;
    ee.V.side = (uint8_t*)(obase + q_side);
    ee.V.coeffs = (long long*)(obase + q_coef);
    ee.V.stride = stride;
    if (nshards > 1) {  // a sharded search also stops the other ranks' joins
      for (int i = 0; i < g.npeers; i++) ee.V.peer_found[i] = g.peer_found[i];
      ee.V.npeers = g.npeers;
    }
    rc = search_core(d_keys, n, lo, width, shard, nshards, (uint64_t*)g.raw.p, raw_cap, s, &r_bits,
                     &nwin, true, early_exit ? &ee : nullptr);
    if (rc) return rc;
    g_tr.mark("search enqueued");
    const bool early = early_exit && nwin == 1;
    // the rest of the hits (all of them without early exit)
    if ((rc = filter_verify(early ? &d_ctr->raw_done : nullptr, early ? &d_ctr->post_done : nullptr,
                            nullptr)))
      return rc;
    RFR_CUDA_OK(cudaEventRecord(g.ev[3], s));
    // outputs: counters plus the first rows (the staged inputs were consumed
    // by the H2D above, so the staging block takes the results)
    const size_t out_bytes = h_coef + vrows * (size_t)stride * 8;
    if (g.h_stage_bytes < out_bytes) {
      RFR_CUDA_OK(cudaStreamSynchronize(s));
      cudaFreeHost(g.h_stage);
      g.h_stage = nullptr;
      g.h_stage_bytes = 0;
      RFR_CUDA_OK(cudaMallocHost(&g.h_stage, out_bytes));
      g.h_stage_bytes = out_bytes;
    }
    hs = (char*)g.h_stage;
    // an early stop's two pieces, searched on the device right behind the
    // main search (every piece kernel is a no-op unless the search stopped at
    // a PASS whose pieces are small); RFR_HOST_PIECES=1 (A/B): the host-driven
    // path only
    dev_pieces = early_exit == 1 && early && !getenv("RFR_HOST_PIECES");
    if (dev_pieces) {
      RFR_CUDA_OK(g.pctr.ensure(sizeof(DevCounters)));
      RFR_CUDA_OK(g.ppost.ensure(kPieceRaw * sizeof(uint64_t)));
      RFR_CUDA_OK(g.pver.ensure(2 * al(2 * kPieceRows) + 2 * kPieceRows * (size_t)stride * sizeof(int64_t)));
      if ((rc = ensure_piece_host(stride))) return rc;
    }
    {  // counters and the first rows in one launch, straight into pinned memory
      CollectArgs C;
      C.ctr = d_ctr;
      C.pats = (const uint64_t*)g.post.p;
      C.verdict = (const uint8_t*)obase;
      C.side = (const uint8_t*)(obase + q_side);
      C.coeffs = (const long long*)(obase + q_coef);
      C.stride = stride;
      C.rows = (unsigned)spec;
      C.h_ctr = g.h_ctr;
      C.h_pats = (uint64_t*)hs;
      C.h_verdict = (uint8_t*)(hs + h_verd);
      C.h_side = (uint8_t*)(hs + h_side);
      C.h_coeffs = (long long*)(hs + h_coef);
      if (dev_pieces) {  // the pieces' counters start from zero
        C.clear = (unsigned long long*)g.pctr.p;
        C.clear_words = (int)(sizeof(DevCounters) / 8);
      }
      RFR_CUDA_OK(launch_collect(C, s));
    }
    if (dev_pieces) {
      const size_t pv_side = al(2 * kPieceRows), pv_coef = 2 * pv_side;
      DevCounters* pctr = (DevCounters*)g.pctr.p;
      PiecePlanArgs pa;
      pa.ctr = d_ctr;
      pa.planned = (unsigned long long)g_buckets_planned;
      pa.raw_cap = raw_cap;
      pa.rows_cap = (unsigned long long)cap;
      pa.pats = (const uint64_t*)g.post.p;
      pa.verdict = (const uint8_t*)obase;
      pa.side = (const uint8_t*)(obase + q_side);
      pa.n = n;
      pa.keys = d_keys;
      pa.keys2 = d_keys2;
      pa.h_desc = piece_h_desc(stride);
      pa.pctr = pctr;
      pa.ppost = (uint64_t*)g.ppost.p;
      char* pvb = (char*)g.pver.p;
      VerifyArgs PV = bind_profile(prof, d, base + o_prof, base + o_perm, base + o_pmod);
      PV.pats = (const uint64_t*)g.ppost.p;
      PV.m = 2 * kPieceRows;
      PV.m_dev = &pctr->post_count;
      PV.found = nullptr;
      PV.verdict = (uint8_t*)pvb;
      PV.side = (uint8_t*)(pvb + pv_side);
      PV.coeffs = (long long*)(pvb + pv_coef);
      PV.stride = stride;
      char* hp = (char*)g.h_piece;  // [counters][2 kPieceRows rows]
      char* rows = hp + sizeof(DevCounters);
      CollectArgs PC;
      PC.ctr = pctr;
      PC.pats = PV.pats;
      PC.verdict = PV.verdict;
      PC.side = PV.side;
      PC.coeffs = PV.coeffs;
      PC.stride = stride;
      PC.rows = 2 * kPieceRows;
      PC.h_ctr = (DevCounters*)hp;
      PC.h_pats = (uint64_t*)rows;
      PC.h_verdict = (uint8_t*)(rows + 2 * kPieceRows * 8);
      PC.h_side = (uint8_t*)(rows + 2 * kPieceRows * 9);
      PC.h_coeffs = (long long*)(rows + 2 * kPieceRows * 10);
      RFR_CUDA_OK(launch_pieces(pa, lo, width, lo2, width2, kPieceRaw, PV, PC, s));
      RFR_CUDA_OK(cudaEventRecord(g.ev[4], s));
    }
    g_tr.mark("post enqueued, sync");
    RFR_CUDA_OK(cudaStreamSynchronize(s));
    g_tr.mark("synced");
    if (g.h_ctr->out_count <= raw_cap) break;
    if (attempt == 2) return rfr_fail(RFR_E_CAP, "raw hit buffer regrow failed");
    const unsigned long long want = g.h_ctr->out_count + (g.h_ctr->out_count >> 3) + 1024;
    if (want > (1ull << 31))
      return rfr_fail(RFR_E_CAP, "%llu raw hits exceed the 2^31 limit",
                      (unsigned long long)g.h_ctr->out_count);
    RFR_CUDA_OK(g.raw.ensure(want * sizeof(uint64_t)));
  }
  const DevCounters cc = *g.h_ctr;
  if (cc.t_found && getenv("RFR_STOP_TRACE")) dump_stop_trace(cc.t_found, g.nsm * kJoinCtasPerSm - 1);
  const int main_launches = g_launches;
  const int64_t main_planned = g_buckets_planned;
  const size_t m = cc.post_count < (unsigned long long)cap ? (size_t)cc.post_count : (size_t)cap;
  if (m > spec) {  // more survivors than the speculative rows
    RFR_CUDA_OK(copy_rows(spec, m));
    RFR_CUDA_OK(cudaStreamSynchronize(s));
  }
  // ---- early stop: search the two pieces of the verified factor in this call
  std::vector<uint64_t> xp;
  std::vector<uint8_t> xv, xs;
  std::vector<int64_t> xc;
  int64_t xbuckets = 0;
  bool complete = cc.buckets >= (unsigned long long)main_planned;
  const bool stopped = !complete;
  int pieces_how = 0;
  if (early_exit == 1 && !complete && m == cc.post_count) {
    const uint64_t full = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
    for (size_t k = 0; k < m; k++) {
      if (((const uint8_t*)(hs + h_verd))[k] != RFR_V_PASS) continue;
      const uint64_t sp = ((const uint64_t*)hs)[k] & full;
      const uint64_t t = ((const uint8_t*)(hs + h_side))[k] ? (~sp & full) : sp;
      VerifyArgs V0 = bind_profile(prof, d, base + o_prof, base + o_perm, base + o_pmod);
      V0.m = (long long)vrows;
      V0.verdict = (uint8_t*)obase;
      V0.side = (uint8_t*)(obase + q_side);
      V0.coeffs = (long long*)(obase + q_coef);
      V0.stride = stride;
      const PieceDesc* D = dev_pieces ? piece_h_desc(stride) : nullptr;
      if (D && D->active && D->t == t) {  // searched on the device behind the main search
        if (read_chained_piece_rows(stride, xp, xv, xs, xc)) {
          complete = true;
          pieces_how = 2;
        }
        break;
      }
      int prc = RFR_OK;
      if (search_pieces(keys, keys2, n, lo, width, lo2, width2, t, V0, stride, s, xp, xv, xs, xc,
                        &xbuckets, &prc)) {
        complete = true;
        pieces_how = 1;
      } else if (prc) {
        return prc;
      }
      break;
    }
  }
  g_tr.mark("pieces done");
  const unsigned long long total = cc.post_count + (unsigned long long)xp.size();
  if (m) {
    memcpy(pats, hs, m * 8);
    if (verdict) memcpy(verdict, hs + h_verd, m);
    if (side) memcpy(side, hs + h_side, m);
    if (coeffs) memcpy(coeffs, hs + h_coef, m * (size_t)stride * sizeof(int64_t));
  }
  if (complete && !xp.empty() && total <= (unsigned long long)cap) {
    memcpy(pats + m, xp.data(), xp.size() * 8);
    if (verdict) memcpy(verdict + m, xv.data(), xv.size());
    if (side) memcpy(side + m, xs.data(), xs.size());
    if (coeffs) memcpy(coeffs + m * (size_t)stride, xc.data(), xc.size() * sizeof(int64_t));
  }
  *nout = (int64_t)(complete ? total : cc.post_count);
  if (st) {
    g_launches = main_launches;
    g_buckets_planned = main_planned;
    fill_stats(st, cc, n, r_bits, nwin);
    st->raw_hits = (int64_t)cc.out_count;
    st->ms_lists = ev_ms(g.ev[0], g.ev[1]);
    st->ms_join = ev_ms(g.ev[1], g.ev[2]);
    st->ms_post = ev_ms(g.ev[2], g.ev[3]);
    // the whole device span, with the pieces chained behind the main search
    st->ms_total = ev_ms(g.ev[0], g.ev[dev_pieces ? 4 : 3]);
    // a stopped search completed by its pieces' searches covers every factor
    // pattern: report it as complete
    st->buckets += xbuckets;
    if (complete) st->buckets_planned = st->buckets;
    st->early_stop = stopped ? 1 : 0;
    st->pieces = pieces_how;
    st->us_hit_to_stop = (stopped && cc.t_found && cc.t_stop >= cc.t_found)
                             ? (double)(cc.t_stop - cc.t_found) * 1e-3
                             : -1.0;
  }
  if (g_tr.on == 1)
    fprintf(stderr, "[rfr host] counters: out %llu post %llu raw_done %llu post_done %llu found %llu buckets %llu/%lld m %zu verdict0 %d complete %d\n",
            cc.out_count, cc.post_count, cc.raw_done, cc.post_done, cc.found, cc.buckets,
            (long long)main_planned, m, m ? (int)((const uint8_t*)(hs + h_verd))[0] : -1, (int)complete);
  if (g_tr.on == 1 && cc.t_found)
    fprintf(stderr, "[rfr host] device: hit seen->found %.1f us, found->first stop %.1f us, found->last stop %.1f us\n",
            cc.t_hit ? (double)((long long)cc.t_found - (long long)cc.t_hit) * 1e-3 : -1.0,
            cc.t_stop_first ? (double)((long long)cc.t_stop_first - (long long)cc.t_found) * 1e-3 : -1.0,
            cc.t_stop ? (double)((long long)cc.t_stop - (long long)cc.t_found) * 1e-3 : -1.0);
  if (g_tr.on == 1 && cc.t_probe[3])
    fprintf(stderr, "[rfr host] poller verify: expand %.1f us, integrality %.1f us, division %.1f us\n",
            ((long long)cc.t_probe[0] - (long long)cc.t_probe[3]) * 1e-3,
            ((long long)cc.t_probe[1] - (long long)cc.t_probe[0]) * 1e-3,
            ((long long)cc.t_probe[2] - (long long)cc.t_probe[1]) * 1e-3);
  if (g_tr.on == 1 && cc.t_found)
    fprintf(stderr, "[rfr host] device: found->verified %.1f us, found->poller exit %.1f us\n",
            cc.t_verified ? (double)((long long)cc.t_verified - (long long)cc.t_found) * 1e-3 : -1.0,
            cc.t_poller_exit ? (double)((long long)cc.t_poller_exit - (long long)cc.t_found) * 1e-3 : -1.0);
  g_tr.mark("return");
  g_tr.dump();
  return RFR_OK;
}

}  // namespace

int rfr_search_keys2(const uint64_t* keys, int n, uint64_t lo, uint64_t width, const uint64_t* keys2,
                     uint64_t lo2, uint64_t width2, int shard, int nshards, uint64_t* out,
                     int64_t cap, int64_t* nout, rfr_stats* st) {
  std::lock_guard<std::mutex> lk(g_mu);
  if ((!keys || !keys2) && n > 0) return rfr_fail(RFR_E_ARG, "null keys");
  return run_search_host(keys, nullptr, n, lo, width, 0.0, shard, nshards, out, cap, nout, st, keys2,
                         lo2, width2);
}

int rfr_search_keys_dev(const uint64_t* d_keys, int n, uint64_t lo, uint64_t width, int shard,
                        int nshards, uint64_t* d_out, int64_t cap, uint64_t* d_count,
                        void* stream, rfr_stats* st) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc = ensure_ready();
  if (rc) return rc;
  if ((rc = check_n(n))) return rc;
  if (nshards < 1 || shard < 0 || shard >= nshards) return rfr_fail(RFR_E_ARG, "bad shard");
  if (n == 0) return rfr_fail(RFR_E_ARG, "empty instance");
  cudaSetDevice(g.device);
  cudaStream_t s = stream ? (cudaStream_t)stream : g.stream;
  DevCounters* d_ctr = (DevCounters*)g.ctr.p;
  RFR_CUDA_OK(cudaMemsetAsync(d_ctr, 0, sizeof(DevCounters), s));
  int r_bits = 0, nwin = 0;
  rc = search_core(d_keys, n, lo, width, shard, nshards, d_out, (unsigned long long)cap, s,
                   &r_bits, &nwin, st != nullptr);
  if (rc) return rc;
  if (d_count)
    RFR_CUDA_OK(cudaMemcpyAsync(d_count, &d_ctr->out_count, sizeof(uint64_t),
                                cudaMemcpyDeviceToDevice, s));
  if (st) {
    RFR_CUDA_OK(cudaEventRecord(g.ev[3], s));
    RFR_CUDA_OK(cudaMemcpyAsync(g.h_ctr, d_ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
    RFR_CUDA_OK(cudaStreamSynchronize(s));
    fill_stats(st, *g.h_ctr, n, r_bits, nwin);
    st->ms_lists = ev_ms(g.ev[0], g.ev[1]);
    st->ms_join = ev_ms(g.ev[1], g.ev[2]);
    st->ms_total = ev_ms(g.ev[0], g.ev[3]);
  }
  return RFR_OK;
}

}  // extern "C"

extern "C" {

int rfr_verify_primes(uint64_t* primes3) {
  if (!primes3) return rfr_fail(RFR_E_ARG, "null primes buffer");
  for (int i = 0; i < 3; i++) primes3[i] = kVerifyPrimes[i];
  return RFR_OK;
}

int rfr_p_mod_i64(const int64_t* coeffs, int d, uint64_t* p_mod) {
  if (!coeffs || !p_mod || d < 0) return rfr_fail(RFR_E_ARG, "bad p_mod arguments");
  const int64_t lim = (int64_t)1 << 62;
  for (int k = 0; k <= d; k++)
    if (coeffs[k] >= lim || coeffs[k] <= -lim) return rfr_fail(RFR_E_ARG, "coefficient beyond 2^62");
  for (int i = 0; i < 3; i++) {
    const int64_t q = (int64_t)kVerifyPrimes[i];
    for (int k = 0; k <= d; k++) {
      const int64_t r = coeffs[k] % q;
      p_mod[(size_t)i * (d + 1) + k] = (uint64_t)(r < 0 ? r + q : r);
    }
  }
  return RFR_OK;
}

int rfr_verify(const rfr_profile* prof, const uint64_t* pats, int64_t m, const uint64_t* p_mod,
               int d, uint8_t* verdict, uint8_t* side, int64_t* coeffs, int stride,
               rfr_stats* st) {
  std::lock_guard<std::mutex> lk(g_mu);
  int rc = ensure_ready();
  if (rc) return rc;
  if (m < 0 || d < 1 || d > 128 || stride < 1) return rfr_fail(RFR_E_ARG, "bad verify arguments");
  if ((rc = check_profile(prof, d))) return rc;
  if (m == 0) return RFR_OK;
  if (!pats || !p_mod || !verdict || !side || !coeffs)
    return rfr_fail(RFR_E_ARG, "null verify buffer");
  cudaSetDevice(g.device);
  cudaStream_t s = g.stream;
  // one pinned staging block each way: [profile doubles | perm | pats | p_mod]
  // in, [verdict | side | coeffs] out (one H2D and one D2H per call)
  const int r = prof->r, c = prof->c, n = prof->n;
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  const size_t nd = (size_t)(2 * r + 4 * c + 1);
  const size_t o_perm = al(nd * sizeof(double));
  const size_t o_pats = o_perm + al((size_t)n * sizeof(int32_t));
  const size_t o_pmod = o_pats + al((size_t)m * sizeof(uint64_t));
  const size_t in_bytes = o_pmod + al((size_t)3 * (d + 1) * sizeof(uint64_t));
  const size_t q_side = al((size_t)m);
  const size_t q_coef = q_side + al((size_t)m);
  const size_t out_bytes = q_coef + (size_t)m * stride * sizeof(int64_t);
  const size_t stage = in_bytes > out_bytes ? in_bytes : out_bytes;
  if (g.h_stage_bytes < stage) {
    if (g.h_stage) cudaFreeHost(g.h_stage);
    g.h_stage = nullptr;
    g.h_stage_bytes = 0;
    RFR_CUDA_OK(cudaMallocHost(&g.h_stage, stage));
    g.h_stage_bytes = stage;
  }
  char* hs = (char*)g.h_stage;
  stage_profile((double*)hs, prof);
  memcpy(hs + o_perm, prof->perm, (size_t)n * sizeof(int32_t));
  memcpy(hs + o_pats, pats, (size_t)m * sizeof(uint64_t));
  memcpy(hs + o_pmod, p_mod, (size_t)3 * (d + 1) * sizeof(uint64_t));
  RFR_CUDA_OK(g.vprof.ensure(in_bytes));
  RFR_CUDA_OK(g.vcoef.ensure(out_bytes));
  char* base = (char*)g.vprof.p;
  char* obase = (char*)g.vcoef.p;
  RFR_CUDA_OK(cudaMemcpyAsync(base, hs, in_bytes, cudaMemcpyHostToDevice, s));
  VerifyArgs A = bind_profile(prof, d, base, base + o_perm, base + o_pmod);
  A.pats = (const uint64_t*)(base + o_pats);
  A.m = m;
  A.m_dev = nullptr;
  A.verdict = (uint8_t*)obase;
  A.side = (uint8_t*)(obase + q_side);
  A.coeffs = (long long*)(obase + q_coef);
  A.stride = stride;
  RFR_CUDA_OK(cudaEventRecord(g.ev[2], s));
  RFR_CUDA_OK(launch_verify(A, s));
  RFR_CUDA_OK(cudaEventRecord(g.ev[3], s));
  // the staging block is reused for the results once the H2D has been consumed
  RFR_CUDA_OK(cudaMemcpyAsync(hs, obase, out_bytes, cudaMemcpyDeviceToHost, s));
  RFR_CUDA_OK(cudaStreamSynchronize(s));
  memcpy(verdict, hs, (size_t)m);
  memcpy(side, hs + q_side, (size_t)m);
  memcpy(coeffs, hs + q_coef, (size_t)m * stride * sizeof(int64_t));
  if (st) {
    memset(st, 0, sizeof *st);
    st->ms_post = ev_ms(g.ev[2], g.ev[3]);
    st->ms_total = st->ms_post;
    st->launches = 1;
  }
  return RFR_OK;
}

}  // extern "C"
