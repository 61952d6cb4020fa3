// rfr_common.cuh -- shared definitions for the recombination kernels.
//
// Key arithmetic lives in Z / 2^64: a pattern's key is the wrapping uint64 sum
// of its per-entity keys (fixed-point fractional parts scaled by 2^64), so an
// integer sum of fractional parts is a key near 0.  See DESIGN.md section 2.
#pragma once
#include <cstdlib>
#include <utility>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace rfr {

// Largest quarter list walked by the join (2^23 entries = 64 MB of keys).
constexpr int kMaxInnerBits = 28;  // inner lists up to 2^28 entries (12 B each, x2 ping-pong)
// Outer lists live in shared memory of the join kernel.
constexpr int kMaxOuterBits = 6;
// Join geometry: RFR_JOIN_CTAS CTAs per SM, each walking buckets of
// ~2^kJoinRecLog A records (the plan picks r = alpha - kJoinRecLog).
#ifndef RFR_JOIN_CTAS
#define RFR_JOIN_CTAS 2
#endif
constexpr int kJoinCtasPerSm = RFR_JOIN_CTAS;
// threads per join CTA (default 256: 16 warps/SM at 128 registers).  A
// 512-thread variant (32 warps/SM, 64 registers, lambda 128) spills in the
// B pass and measured 60 % slower.
#ifndef RFR_JOIN_THREADS
#define RFR_JOIN_THREADS (512 / RFR_JOIN_CTAS)
#endif
constexpr int kJoinThreadsPerCta = RFR_JOIN_THREADS;
constexpr int kJoinRecLog = RFR_JOIN_CTAS == 1 ? 12 : 11;
// Sorted base block built in shared memory by the list builder.
constexpr int kBaseBits = 12;
constexpr int kRotSlots = 64;  // per-list rotation counters of the merge levels

// One quarter list of the folded pattern space: subset sums of
// keys[first, first + bits) (negated for the B half), sorted ascending.
struct ListSpec {
  int first;      // first rho index covered
  int bits;       // number of elements (list length 2^bits)
  int negate;     // 1 for the B half (N = -K)
  int pat_shift;  // bit position of this list's pattern inside the full pattern
};

// Search plan: the folded half space t < 2^(n-1) is the product of four
// quarter lists A_outer x A_inner x B_outer x B_inner; see DESIGN.md s3.
struct JoinPlan {
  int n;             // rho width
  int m;             // folded bits = n - 1
  ListSpec list[4];  // 0 = A outer, 1 = A inner, 2 = B outer, 3 = B inner
  int r;             // bucket bits; bucket c = [c W, (c+1) W), W = 2^(64-r)
  int nbins_log;     // A-records of one bucket are counting-sorted into 2^nbins_log bins
  uint64_t lo;       // window: match iff (K_a + K_b - lo) mod 2^64 <= width
  uint64_t width;
  uint64_t shift;    // added to every B key: lo + width/2
  uint64_t half;     // ceil(width / 2): bin search radius
  uint64_t bucket_begin, bucket_end;  // this launch's bucket range
};

// Four quarter-list buffers (keys + local patterns), passed by value.
struct ListBufs {
  uint64_t* k[4];
  uint32_t* p[4];
};

// Merge history of the lists (levels kBaseBits .. bits-1): instead of a
// pattern per entry, every doubling level L_k -> L_k+1 keeps one provenance
// bit per output (0: from L_k, 1: from rotate(L_k + v_k)), a 16-bit rank
// directory per 64 outputs (1-bits in the 2048-output tile before that word)
// and the tile splits (# L_k entries before each tile).  A list entry's
// pattern is recovered by walking the levels down (emit time only), so the
// levels move 8-byte keys instead of 12-byte key + pattern pairs.
constexpr int kHistTileLog = 11;  // 2048 outputs per merge tile
struct ListHist {
  uint8_t* bm[4];
  uint16_t* dir[4];
  uint32_t* sp[4];
};
__host__ __device__ inline size_t hist_bm_off(int k) {  // bytes before level k
  return (((size_t)1 << (k + 1)) - ((size_t)1 << (kBaseBits + 1))) / 8;
}
__host__ __device__ inline size_t hist_dir_off(int k) {  // directory entries before level k
  return (((size_t)1 << (k + 1)) - ((size_t)1 << (kBaseBits + 1))) / 64;
}
__host__ __device__ inline size_t hist_sp_off(int k) {  // split words before level k
  return (((size_t)1 << (k + 1 - kHistTileLog)) - ((size_t)1 << (kBaseBits + 1 - kHistTileLog))) +
         (size_t)(k - kBaseBits);
}

// Device-side counters (one slot each, accumulated with atomics).
struct DevCounters {
  unsigned long long out_count;      // emitted pairs (may exceed capacity)
  unsigned long long inserts;        // A records binned (main + halo ghosts)
  unsigned long long insert_probes;  // A outer-pointer checks
  unsigned long long queries;        // B records streamed
  unsigned long long query_probes;   // A records compared against a B record
  unsigned long long chunks;         // extra A chunks after a bucket overflow
  unsigned long long buckets;        // buckets processed
  unsigned long long post_count;     // survivors of the post-filter
  // early exit (rfr_search_verify with early_exit): the poller verifies hits
  // while the join runs and raises found; the join's CTAs stop at their next
  // bucket boundary.
  unsigned long long raw_done;       // raw hits the poller turned into patterns and filtered
  unsigned long long post_done;      // survivors the poller verified
  unsigned long long ctas_done;      // join CTAs finished (the poller's stop condition)
  // hit-to-stop latency (globaltimer, ns): the poller's speculative stop, the
  // moment it saw that hit, and the first / last join CTA that stopped
  unsigned long long t_found;
  unsigned long long t_stop;
  unsigned long long t_hit;
  unsigned long long t_stop_first;
  unsigned long long t_verified;    // the poller finished verifying the stopping hit
  unsigned long long t_poller_exit;
  unsigned long long t_probe[4];    // RFR_HOST_TRACE: phases of the poller's verification
  // the stop flag on a cache line of its own: every join CTA reads it once per
  // bucket, and the counters above take the CTAs' end-of-join atomics (on a
  // shared line those queued the flag reads for up to ~100 us)
  alignas(128) unsigned long long found;  // a candidate passed (or speculatively: hit) verification
  unsigned long long found_pad[15];
};
__device__ __forceinline__ unsigned long long rfr_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
static_assert(offsetof(DevCounters, found) % 16 == 0, "found must be 16-byte aligned");

// Programmatic dependent launch (the list levels and the join's start
// positions, launched with cudaLaunchAttributeProgrammaticStreamSerialization):
// a kernel waits for its predecessor's completion (and memory) before its
// first global access, then lets its own successor launch, so the next
// level's CTAs are resident and waiting when this one drains instead of
// being launched after it (no-ops in a plain launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// RFR_PDL=0 (A/B): plain launches everywhere launch_pdl is used
inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("RFR_PDL");
    on = e ? atoi(e) != 0 : 1;
  }
  return on != 0;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace rfr

#define RFR_CUDA_OK(expr)                                   \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return rfr_fail_cuda(_e, #expr); \
  } while (0)
