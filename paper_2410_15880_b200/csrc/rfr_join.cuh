// rfr_join.cuh -- the bucket join kernel (included by rfr_search.cu).
//
// Two CTAs per SM (8 warps each); each CTA owns a contiguous range of key
// buckets and walks it in order.  Per bucket c (keys [cW, (c+1)W), W = 2^(64-r),
// ~2^11 A records):
//   A side   every A outer x contributes the contiguous run of its rotated
//            inner list whose sums x + k fall in bucket c, followed by the
//            halo run [(c+1)W, (c+1)W + H).  The plan gives each warp one
//            outer per bucket with a long run (lambda ~ 256 records):
//            run_pass loads all nch chunks of 32 consecutive inner keys of
//            the run at once (coalesced, L1 no-allocate; the next bucket's
//            lines were prefetched into L2), classifies each lane as main /
//            halo / past the run (the emitted lanes are a prefix: the sums
//            are sorted), and a ballot compacts the records into the warp's
//            own partition of the shared record array.  Short runs (small n)
//            use window_pass: lane groups of 2 lambda lanes per outer window.
//   A index  a three-level direct-mapped index (8, 2 and 1/2 slots per
//            record) over the bucket (the reference's splat table,
//            recombine.py:297-325, moved on chip): every record stores its
//            index in its level-1 home with a plain store, reads it back
//            after a barrier, and only the records that lost a slot collision
//            move to the next level (their level-1 slot gets a collision
//            flag); the few level-3 losers go to a short list.  No shared
//            atomics on this path: they cost ~2 cycles per lane on this part.
//   B side   the same runs over B (negated, shifted keys); each emitted B
//            record reads its level-1 home and the record it names and checks
//            it exactly (the reference's windowed probe, recombine.py:
//            328-358); records that meet a flagged slot (or whose window
//            reaches a second home) are staged and probed at levels 2-3 out
//            of line.
//   Outers whose run outlasts the chunks in flight continue in
//   continue_pass.  Loop state lives in shared memory and the shared base is
//   re-derived at each use, so the pass calls (which may clobber every
//   register) cost no local-memory reloads.
// Pairs across a bucket boundary are found once: (A in c, B in c+1) by a B
// halo record, (A in c+1, B in c) by an A halo record; halo x halo is skipped
// (bucket c+1 finds it).  A bucket whose A side overflows its shared-memory
// partitions (skewed keys) is redone on a slow path in capacity-sized chunks,
// each chunk re-streaming B; the fast attempt emits nothing before the
// overflow is known, so no pair is duplicated.
#pragma once
#include <type_traits>

// Clock64 phase trace of CTA 0 (RFR_TRACE=1 at run time, needs a build with
// `make TRACE=1`); compiled out of the production kernel.
#ifndef RFR_JOIN_CHECK  // 1: trap when a run chunk breaks the prefix invariant
#define RFR_JOIN_CHECK 0
#endif
#ifndef RFR_JOIN_TRACE
#define RFR_JOIN_TRACE 0
#endif
#ifndef RFR_INDEX_PRED  // 1: the level-1 read-back stores a lost record with predicated stores
#define RFR_INDEX_PRED 1
#endif
#ifndef RFR_APASS_PRED  // 1: the A run pass stores its records with predicated shared stores
#define RFR_APASS_PRED 1
#endif
#ifndef RFR_JOIN_PREFETCH  // 1: each outer pulls its next bucket's run into L2
#define RFR_JOIN_PREFETCH 1
#endif
#ifndef RFR_JOIN_BHALO_WIDE  // 1: B halo records take the wide probe (no exclusion test in place)
#define RFR_JOIN_BHALO_WIDE 1
#endif
#ifndef RFR_APASS_NOCLAMP  // 1: no slot clamp in the A run pass when its partition cannot overflow
#define RFR_APASS_NOCLAMP 1
#endif
#ifndef RFR_INDEX_PRED2  // 1: the level-2 read-back also stores a lost record with predicated stores
#define RFR_INDEX_PRED2 1
#endif
#ifndef RFR_INDEX_G4MIN
#define RFR_INDEX_G4MIN 96
#endif
#ifndef RFR_STAGE_PRED  // 1: a staged B record's three fields are written with predicated stores
#define RFR_STAGE_PRED 1
#endif
#ifndef RFR_JOIN_ONEHOME  // 0: the run pass also checks a second level-1 home in place
#define RFR_JOIN_ONEHOME 1
#endif


constexpr int kJoinThreads = kJoinThreadsPerCta;
constexpr int kJoinWarps = kJoinThreads / 32;
// index levels (slots): 8, 2 and 1/2 slots per expected record
constexpr int kL1Log = kJoinRecLog + 3, kL2Log = kJoinRecLog + 1, kL3Log = kJoinRecLog - 1;
constexpr int kPart = (3 << kJoinRecLog) / 2 / kJoinWarps;  // A records per warp partition
constexpr int kCapRec = kPart * kJoinWarps;  // A records per chunk (1.5x the expected)
constexpr int kLose = kJoinWarps > 8 ? 64 : 128;                          // per-warp level-1 loser list
constexpr int kList4 = 256;                           // level-3 losers (CTA list)
constexpr int kMaxOuter = 1 << kMaxOuterBits;
constexpr int kU = 8;                                 // A windows in flight per lane
constexpr int kUB = kJoinWarps > 8 ? 2 : 4;                             // B windows in flight per lane
constexpr int kStageB = kJoinWarps > 8 ? 64 : kUB * 32;  // staged B records per warp
constexpr uint16_t kNone = 0xffffu;
constexpr uint32_t kFlagCont = 0x80000000u;

static_assert(kL2Log == kL1Log - 2 && kL3Log == kL1Log - 4,
              "the level-2/3 homes are the level-1 home shifted right by 2 / 4");
struct JoinSmem {
  // early exit: DevCounters.found (+ the next word) copied in by cp.async at
  // the start of each bucket, read after the bucket's last barrier
  alignas(16) unsigned long long stop_buf[2];
  uint64_t recK[kCapRec];  // A records: key
  uint32_t recI[kCapRec];  // A records: outer << inner_bits | inner index
  uint16_t rh[kCapRec];     // A records: level-1 home (levels 2, 3: rh >> 2, rh >> 4)
  uint16_t t1[1 << kL1Log];
  uint16_t t2[1 << kL2Log];
  uint16_t t3[1 << kL3Log];
  uint16_t lose[kJoinWarps][kLose];  // per-warp level-1 losers, then level-2 losers
  uint16_t list4[kList4];
  uint64_t qK[kJoinWarps][kStageB];  // staged B records: key
  uint32_t qJ[kJoinWarps][kStageB];  // staged B records: halo flag << 31 | inner index
  uint16_t qB[kJoinWarps][kStageB];  // staged B records: outer index
  uint64_t ax[kMaxOuter];
  uint32_t arot[kMaxOuter];
  uint32_t apos[kMaxOuter];
  uint32_t amain[kMaxOuter];  // main records in this bucket (| kFlagCont: run continues)
  uint64_t bx[kMaxOuter];
  uint32_t brot[kMaxOuter];
  uint32_t bpos[kMaxOuter];
  uint32_t bmain[kMaxOuter];
  uint32_t wcnt[kJoinWarps];
  // loop state kept on chip across the pass calls (which may clobber every
  // register; state held in registers would be saved to the local stack)
  uint32_t wlo[2][kJoinWarps], whi[2][kJoinWarps];  // per-warp outer ranges (A, B)
  uint32_t cnt[3][kJoinThreads];                     // per-thread inserts, queries, probes
  unsigned int n4;
  int ovf;
  uint32_t cur_i, cur_t;  // slow path cursor
};
static_assert(sizeof(JoinSmem) + 1024 <= (228 * 1024) / kJoinCtasPerSm,
              "join shared memory exceeds the per-SM budget for kJoinCtasPerSm CTAs");


// The join's shared memory, addressed from the extern symbol inside every
// (noinline) function so the compiler emits direct shared-window accesses
// instead of re-deriving them from a generic reference.
__device__ __forceinline__ JoinSmem& join_smem() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem_raw);
  asm volatile("" : "+r"(sa));  // re-derived at each use, never kept across a call
  return *reinterpret_cast<JoinSmem*>(__cvta_shared_to_generic(sa));
}

// The stop flag read with gpu-scope coherence (a weak read -- the cp.async
// copy -- may be served from a stale far-die L2 copy for tens of us).
#ifndef RFR_STOP_COHERENT
#define RFR_STOP_COHERENT 1
#endif
__device__ __forceinline__ unsigned long long ld_found_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Streaming read of a list key: read-only path without L1 allocation, so the
// window loads do not evict the kernel's stack and small working set.
__device__ __forceinline__ uint64_t ld_stream(const uint64_t* p) {
  uint64_t v;
  asm("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// threadIdx.x re-read at each use (volatile: never hoisted and kept across a
// call, where it would be saved to and reloaded from the local stack).
__device__ __forceinline__ int tid_now() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

__device__ __forceinline__ uint32_t home_of(uint64_t rel, int shift, int lg) {
  return (uint32_t)(rel >> shift) & ((1u << lg) - 1u);
}

// Emit a matching (A record r, B record) pair as its four quarter-list
// INDICES packed at the patterns' bit offsets (they sum to n - 1 <= 63 bits);
// index_to_pattern_kernel turns them into patterns after the join, so the
// emit site stays small (its register footprint is paid at every call site).
__device__ __noinline__ void emit_match(const JoinArgs& a, uint32_t r, uint32_t ib, uint32_t jb) {
  JoinSmem& S = join_smem();
  const JoinPlan& P = a.P;
  const uint32_t id = S.recI[r];
  const int aib = P.list[1].bits;
  const uint32_t ia = id >> aib, ja = id & ((1u << aib) - 1u);
  const uint64_t v = (uint64_t)ia | ((uint64_t)ja << P.list[1].pat_shift) |
                     ((uint64_t)ib << P.list[2].pat_shift) | ((uint64_t)jb << P.list[3].pat_shift);
  const unsigned long long k = atomicAdd(&a.ctr->out_count, 1ull);
  if (k < a.cap) a.out[k] = v;
}

// Running counters of one warp threaded through the passes by value (by
// reference they would live in local memory across every call).
struct PassSt {
  uint32_t wfill;     // records in the warp's A partition
  uint32_t n_stat;    // records streamed (inserts for A, queries for B)
  uint32_t n_qprobe;  // A records compared against B records
  bool overflow;      // the A partition overflowed
  bool cont;          // some outer of the warp was flagged for continue_pass
};

// Per-bucket constants, built once per pass into registers (reading them
// through the JoinArgs reference inside the loops costs a generic load each).
struct JoinK {
  uint64_t cW, W, H, width, hw;  // bucket base, bucket width, halo, window, window / 2
  int sh;                        // bucket = key >> sh
};
__device__ __forceinline__ JoinK make_k(const JoinArgs& a, uint64_t cW) {
  JoinK K;
  K.sh = 64 - a.P.r;
  K.cW = cW;
  K.W = 1ull << K.sh;
  K.H = a.P.half;
  K.width = a.P.width;
  K.hw = a.P.width >> 1;
  return K;
}

// Exact check of A record r against B key s; emits the pattern on a match.
__device__ __forceinline__ void check_pair(const JoinSmem& S, const JoinArgs& a, const JoinK& K,
                                           uint32_t r, uint64_t s, bool bghost, uint32_t ib,
                                           uint32_t jb, uint32_t& n_qprobe) {
  n_qprobe++;
  const uint64_t ka = S.recK[r];
  if (bghost && (ka - K.cW >= K.W)) return;  // halo x halo belongs to bucket c+1
  if (ka - s + K.hw <= K.width) emit_match(a, r, ib, jb);
}

// Probe one level of the index over the homes of [lo_rel, hi_rel].
__device__ __forceinline__ void probe_level(const JoinSmem& S, const JoinArgs& a, const JoinK& K,
                                            const uint16_t* t, int lg, uint64_t lo_rel,
                                            uint64_t hi_rel, uint64_t s, bool bghost, uint32_t ib,
                                            uint32_t jb, uint32_t& n_qprobe) {
  const int shift = K.sh - lg;
  const uint32_t h0 = (uint32_t)(lo_rel >> shift);
  const uint32_t hn = (uint32_t)(hi_rel >> shift) - h0;
  const uint32_t m = (1u << lg) - 1u;
  const uint32_t lim = hn < m ? hn : m;
  for (uint32_t d = 0; d <= lim; d++) {
    const uint32_t r = t[(h0 + d) & m];
    if (r != kNone) check_pair(S, a, K, r, s, bghost, ib, jb, n_qprobe);
  }
}

// Deep probe for a B record whose level-1 home(s) carry the collision flag:
// levels 2 and 3 and the short list (level 1 was checked in place).
__device__ __noinline__ uint32_t probe_b(const JoinArgs& a, uint64_t cW,
                                         uint64_t s, bool bghost, uint32_t ib, uint32_t jb) {
  JoinSmem& S = join_smem();
  uint32_t n_qprobe = 0;
  const JoinK K = make_k(a, cW);
  const uint64_t H = K.H;
  const uint64_t rel = s - cW;  // main: [0, W); halo: [W, W + H)
  const uint64_t lo_rel = rel >= H ? rel - H : 0ull;
  const uint64_t hi_rel = rel + H;
  probe_level(S, a, K, S.t2, kL2Log, lo_rel, hi_rel, s, bghost, ib, jb, n_qprobe);
  probe_level(S, a, K, S.t3, kL3Log, lo_rel, hi_rel, s, bghost, ib, jb, n_qprobe);
  const uint32_t n4 = S.n4 < (unsigned)kList4 ? S.n4 : (unsigned)kList4;
  for (uint32_t e = 0; e < n4; e++) check_pair(S, a, K, S.list4[e], s, bghost, ib, jb, n_qprobe);
  return n_qprobe;
}

// Full probe (all levels) for B records whose window spans many level-1
// homes (wide parity-mode windows).
__device__ __noinline__ uint32_t probe_b_wide(const JoinArgs& a, uint64_t cW,
                                              uint64_t s, bool bghost, uint32_t ib, uint32_t jb) {
  JoinSmem& S = join_smem();
  uint32_t n_qprobe = 0;
  const JoinK K = make_k(a, cW);
  const uint64_t H = K.H;
  const uint64_t rel = s - cW;
  const uint64_t lo_rel = rel >= H ? rel - H : 0ull;
  const uint64_t hi_rel = rel + H;
  const int shift = K.sh - kL1Log;
  const uint32_t h0 = (uint32_t)(lo_rel >> shift);
  const uint32_t hn = (uint32_t)(hi_rel >> shift) - h0;
  const uint32_t m = (1u << kL1Log) - 1u;
  const uint32_t lim = hn < m ? hn : m;
  for (uint32_t d = 0; d <= lim; d++) {
    const uint32_t e = S.t1[(h0 + d) & m];
    if (e != kNone) check_pair(S, a, K, e & 0x7fffu, s, bghost, ib, jb, n_qprobe);
  }
  return n_qprobe + probe_b(a, cW, s, bghost, ib, jb);
}

// In-place level-1 check for one B record: the occupants of its level-1
// home(s) are compared exactly.  Returns 1 when a deep probe of levels 2-3
// is still needed (flagged collision slot), 2 for a wide window.
__device__ __forceinline__ int probe_b_l1(const JoinSmem& S, const JoinArgs& a, const JoinK& K,
                                          uint64_t s, bool bghost, uint32_t ib, uint32_t jb,
                                          uint32_t& n_qprobe) {
  const uint64_t H = K.H;
  const uint64_t rel = s - K.cW;
  const uint64_t lo_rel = rel >= H ? rel - H : 0ull;
  const int sh1 = K.sh - kL1Log;
  const uint32_t h0 = (uint32_t)(lo_rel >> sh1);
  const uint32_t hn = (uint32_t)((rel + H) >> sh1) - h0;
  if (hn > 1) return 2;
  const uint32_t m1 = (1u << kL1Log) - 1u;
  int deep = 0;
  const uint32_t e0 = S.t1[h0 & m1];
  if (e0 != kNone) {
    check_pair(S, a, K, e0 & 0x7fffu, s, bghost, ib, jb, n_qprobe);
    deep |= (e0 >> 15) & 1;
  }
  if (hn) {
    const uint32_t e1 = S.t1[(h0 + 1) & m1];
    if (e1 != kNone) {
      check_pair(S, a, K, e1 & 0x7fffu, s, bghost, ib, jb, n_qprobe);
      deep |= (e1 >> 15) & 1;
    }
  }
  return deep;
}

// Deep-probe the staged B records of this warp (rare: flagged level-1
// collisions or wide windows), one lane per record, from one code site.
__device__ __noinline__ uint32_t process_staged(const JoinArgs& a, uint64_t cW,
                                                uint32_t nst) {
  JoinSmem& S = join_smem();
  uint32_t n_qprobe = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncwarp();
  for (uint32_t e = lane; e < nst; e += 32) {
    const uint64_t s = S.qK[wid][e];
    const uint32_t meta = S.qJ[wid][e];
    if ((meta >> 30) & 1u)
      n_qprobe += probe_b_wide(a, cW, s, meta >> 31, S.qB[wid][e], meta & 0x3fffffffu);
    else
      n_qprobe += probe_b(a, cW, s, meta >> 31, S.qB[wid][e], meta & 0x3fffffffu);
  }
  __syncwarp();
  return n_qprobe;
}

// Windowed walk of one side: lane-group layout, kU windows in flight.  Side A
// appends records to the warp partition and claims level-1 homes; side B
// probes.  Saturated runs are flagged in the main-count array.
template <bool SIDE_A>
__device__ __noinline__ PassSt window_pass(const JoinArgs& a, uint64_t cW,
                                            uint32_t lo, uint32_t hi, int gs, PassSt st) {
  JoinSmem& S = join_smem();
  // register copies of the by-reference counters (written back once)
  uint32_t wfill = st.wfill, n_stat = st.n_stat, n_qprobe = st.n_qprobe;
  bool overflow = st.overflow, cont = false;
  const JoinPlan& P = a.P;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int g = lane / gs, l = lane % gs, gpw = 32 / gs, gb = g * gs;
  const uint32_t gmask = gs == 32 ? FULL : ((1u << gs) - 1u);
  const uint32_t Mi = 1u << P.list[SIDE_A ? 1 : 3].bits;
  const uint64_t* __restrict__ kin = a.key[SIDE_A ? 1 : 3];
  const uint64_t* xs = SIDE_A ? S.ax : S.bx;
  const uint32_t* rots = SIDE_A ? S.arot : S.brot;
  const uint32_t* poss = SIDE_A ? S.apos : S.bpos;
  uint32_t* mainv = SIDE_A ? S.amain : S.bmain;
  const int sh = 64 - P.r;
  const uint64_t W = 1ull << sh, H = P.half;
  const JoinK K = make_k(a, cW);
  const int aib = P.list[1].bits;
  uint32_t nq = 0;
  constexpr int U = SIDE_A ? kU : kUB;
  unsigned long long* tr = (RFR_JOIN_TRACE && a.dbg && blockIdx.x == 0 && threadIdx.x == 0) ? a.dbg + 128 + (SIDE_A ? 0 : 64) : nullptr;
  int trn = 0;
  // Software pipeline: the U window keys of round k+1 are loaded while round
  // k is processed, so the L2 round trips overlap the processing and each
  // other (issued back to back, consumed only after the loop back-edge).
  uint64_t kn[U];
  auto issue = [&](uint32_t b0) {
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t i = b0 + u * gpw + g;
      const bool valid = i < hi && (uint32_t)l < Mi;
      const uint32_t ic = i < hi ? i : lo;
      const uint32_t j = (rots[ic] + poss[ic] + l) & (Mi - 1);
      kn[u] = ld_stream(kin + (valid ? j : 0u));
    }
  };
  if (lo < hi) issue(lo);
  for (uint32_t base = lo; base < hi; base += U * gpw) {
    if (RFR_JOIN_TRACE && tr && trn < 60) tr[trn++] = clock64();
    uint64_t kv[U];
    uint32_t jv[U];
#pragma unroll
    for (int u = 0; u < U; u++) kv[u] = kn[u];
    if (base + U * gpw < hi) issue(base + U * gpw);
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t i = base + u * gpw + g;
      const uint32_t ic = i < hi ? i : lo;
      jv[u] = (rots[ic] + poss[ic] + l) & (Mi - 1);
    }
    // phase 2: classify (main / halo) from the loaded keys
    uint64_t sv[U];
    bool mv[U], ev[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t i = base + u * gpw + g;
      const bool valid = i < hi && (uint32_t)l < Mi;
      uint32_t pos = 0;
      uint64_t x = 0;
      if (i < hi) {
        pos = poss[i];
        x = xs[i];
      }
      const uint32_t o = pos + l;
      sv[u] = x + kv[u];
      const uint64_t rel = sv[u] - cW;
      mv[u] = valid && o < Mi && rel < W;
      ev[u] = mv[u] || (valid && (rel - W) < H);
    }
    if (RFR_JOIN_TRACE && tr && trn < 60) tr[trn++] = clock64() | (1ull << 63);
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t i = base + u * gpw + g;
      const uint32_t em = __ballot_sync(FULL, ev[u]);
      const uint32_t mm = __ballot_sync(FULL, mv[u]);
      if (SIDE_A) {
        const uint32_t ne = __popc(em);
        if (wfill + ne > (uint32_t)kPart) overflow = true;  // warp-uniform
        if (!overflow) {
          if (ev[u]) {
            const uint32_t r = wid * kPart + wfill + __popc(em & lt_mask);
            S.recK[r] = sv[u];
            S.recI[r] = (i << aib) | jv[u];
            const uint32_t h1 = home_of(sv[u] - cW, sh - kL1Log, kL1Log);
            S.t1[h1] = (uint16_t)r;
            S.rh[r] = (uint16_t)h1;
          }
          wfill += ne;
        }
        n_stat += ev[u] ? 1u : 0u;
      } else {
        n_stat += ev[u] ? 1u : 0u;
        int deep = 0;
        if (ev[u]) deep = probe_b_l1(S, a, K, sv[u], !mv[u], i, jv[u], n_qprobe);
        const uint32_t dm = __ballot_sync(FULL, deep != 0);
        if (deep) {
          const uint32_t k = nq + __popc(dm & lt_mask);
          S.qK[wid][k] = sv[u];
          S.qJ[wid][k] = (mv[u] ? 0u : 0x80000000u) | (deep == 2 ? 0x40000000u : 0u) | jv[u];
          S.qB[wid][k] = (uint16_t)i;
        }
        nq += __popc(dm);
      }
      if (l == 0 && i < hi) {
        const bool sat = ((em >> gb) & gmask) == gmask && (uint32_t)gs < Mi;
        mainv[i] = (uint32_t)__popc((mm >> gb) & gmask) | (sat ? kFlagCont : 0u);
        cont |= sat;
      }
    }
    if (!SIDE_A && nq) {
      n_qprobe += process_staged(a, cW, nq);
      nq = 0;
    }
  }
  cont = __any_sync(0xffffffffu, cont);
  return PassSt{wfill, n_stat, n_qprobe, overflow, cont};
}

// Continue the saturated runs of one side, one outer at a time, 32 lanes.
template <bool SIDE_A>
__device__ __noinline__ PassSt continue_pass(const JoinArgs& a, uint64_t cW,
                                              uint32_t lo, uint32_t hi, int gs, PassSt st) {
  JoinSmem& S = join_smem();
  // register copies of the by-reference counters (written back once)
  uint32_t wfill = st.wfill, n_stat = st.n_stat, n_qprobe = st.n_qprobe;
  bool overflow = st.overflow, cont = false;
  const JoinPlan& P = a.P;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t Mi = 1u << P.list[SIDE_A ? 1 : 3].bits;
  const uint64_t* __restrict__ kin = a.key[SIDE_A ? 1 : 3];
  uint32_t* mainv = SIDE_A ? S.amain : S.bmain;
  const int sh = 64 - P.r;
  const uint64_t W = 1ull << sh, H = P.half;
  const JoinK K = make_k(a, cW);
  const int aib = P.list[1].bits;
  for (uint32_t c0 = lo; c0 < hi; c0 += 32) {
    const uint32_t ii = c0 + lane;
    const bool flag = ii < hi && (mainv[ii] & kFlagCont);
    uint32_t todo = __ballot_sync(FULL, flag);
    while (todo) {
      const int src = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t i = c0 + src;
      uint32_t mainc = mainv[i] & ~kFlagCont;
      uint32_t off = (uint32_t)gs;
      const uint32_t pos = (SIDE_A ? S.apos : S.bpos)[i];
      const uint32_t rot = (SIDE_A ? S.arot : S.brot)[i];
      const uint64_t x = (SIDE_A ? S.ax : S.bx)[i];
      while (true) {
        const uint32_t q = off + lane;
        const bool valid = q < Mi;
        const uint32_t o = pos + q;
        const uint32_t j = (rot + o) & (Mi - 1);
        const uint64_t s = x + (valid ? ld_stream(kin + j) : 0ull);
        const uint64_t rel = s - cW;
        const bool m = valid && o < Mi && rel < W;
        const bool e = m || (valid && (rel - W) < H);
        const uint32_t em = __ballot_sync(FULL, e);
        const uint32_t ne = __popc(em);
        if (SIDE_A) {
          if (wfill + ne > (uint32_t)kPart) overflow = true;
          if (!overflow) {
            if (e) {
              const uint32_t r = wid * kPart + wfill + __popc(em & lt_mask);
              S.recK[r] = s;
              S.recI[r] = (i << aib) | j;
              const uint32_t h1 = home_of(rel, sh - kL1Log, kL1Log);
              S.t1[h1] = (uint16_t)r;
              S.rh[r] = (uint16_t)h1;
            }
            wfill += ne;
          }
          n_stat += e ? 1u : 0u;
        } else {
          n_stat += e ? 1u : 0u;
          int deep = 0;
          if (e) deep = probe_b_l1(S, a, K, s, !m, i, j, n_qprobe);
          const uint32_t dm = __ballot_sync(FULL, deep != 0);
          if (deep) {
            const uint32_t k = __popc(dm & lt_mask);
            S.qK[wid][k] = s;
            S.qJ[wid][k] = (m ? 0u : 0x80000000u) | (deep == 2 ? 0x40000000u : 0u) | j;
            S.qB[wid][k] = (uint16_t)i;
          }
          if (dm) n_qprobe += process_staged(a, cW, __popc(dm));
        }
        mainc += __popc(__ballot_sync(FULL, m));
        off += ne;
        if (ne < 32 || off >= Mi) break;
      }
      if (lane == 0) mainv[i] = mainc;
    }
  }
  return PassSt{wfill, n_stat, n_qprobe, overflow, cont};
}

// Branch-light level-1 probe of one B record (run_pass): the slot(s) and
// the records they name are read unconditionally, the exact checks are
// predicated, and only a hit branches (to emit_match).  Returns 0, 1 (a
// flagged slot: levels 2-3 still to probe) or 2 (window spans > 2 homes).
__device__ __forceinline__ int probe_b_l1_fast(const JoinSmem& S, const JoinArgs& a,
                                               const JoinK& K, bool e, uint64_t s, bool bghost,
                                               uint32_t ib, uint32_t jb, uint32_t& n_qprobe) {
  const uint64_t rel = s - K.cW;
  const int sh1 = K.sh - kL1Log;
#if RFR_JOIN_ONEHOME
  // one level-1 home checked in place; a window that reaches a second home
  // (rare: 2H against a home of 2^(sh-14), ~2^-20 of the records at C3) is
  // staged whole for probe_b_wide.  h0 unclamped: a record within H of the
  // bucket start wraps it to a far home, so hn is huge and it goes wide too.
  const uint32_t h0 = (uint32_t)((rel - K.H) >> sh1);
  const uint32_t hn = (uint32_t)((rel + K.H) >> sh1) - h0;
  const uint32_t m1 = (1u << kL1Log) - 1u;
#if RFR_JOIN_BHALO_WIDE
  // B halo records (rel in [W, W + H): ~H/W of them, none in practice at
  // factor-mode windows) go wide too, so the in-place check needs no
  // halo x halo exclusion
  const bool narrow = e && !bghost && hn == 0;
#else
  const bool narrow = e && hn == 0;
#endif
#else
  const uint64_t lo_rel = rel >= K.H ? rel - K.H : 0ull;
  const uint32_t h0 = (uint32_t)(lo_rel >> sh1);
  const uint32_t hn = (uint32_t)((rel + K.H) >> sh1) - h0;
  const uint32_t m1 = (1u << kL1Log) - 1u;
  const bool narrow = e && hn <= 1;  // wide windows go to probe_b_wide whole
#endif
  const uint32_t e0 = narrow ? (uint32_t)S.t1[h0 & m1] : (uint32_t)kNone;
  const uint32_t r0 = min(e0 & 0x7fffu, (uint32_t)kCapRec - 1u);
  const uint64_t k0 = S.recK[r0];
  const bool o0 = e0 != kNone;
  n_qprobe += o0 ? 1u : 0u;
#if RFR_JOIN_ONEHOME && RFR_JOIN_BHALO_WIDE
  const bool hit0 = o0 && (k0 - s + K.hw <= K.width);
#else
  const bool hit0 = o0 && !(bghost && (k0 - K.cW >= K.W)) && (k0 - s + K.hw <= K.width);
#endif
  if (hit0) emit_match(a, r0, ib, jb);
  bool deep = o0 && (e0 >> 15);
#if RFR_JOIN_ONEHOME
#if RFR_JOIN_BHALO_WIDE
  return (e && (hn != 0 || bghost)) ? 2 : (deep ? 1 : 0);
#else
  return (e && hn != 0) ? 2 : (deep ? 1 : 0);
#endif
#endif
  // second home: only when the window crosses a level-1 home boundary (rare
  // for factor-mode windows), so it is taken warp-uniformly
  if (__any_sync(0xffffffffu, narrow && hn == 1)) {
    const uint32_t e1 = (narrow && hn == 1) ? (uint32_t)S.t1[(h0 + 1) & m1] : (uint32_t)kNone;
    const uint32_t r1 = min(e1 & 0x7fffu, (uint32_t)kCapRec - 1u);
    const uint64_t k1 = S.recK[r1];
    const bool o1 = e1 != kNone;
    const bool hit1 = o1 && !(bghost && (k1 - K.cW >= K.W)) && (k1 - s + K.hw <= K.width);
    n_qprobe += o1 ? 1u : 0u;
    if (hit1) emit_match(a, r1, ib, jb);
    deep = deep || (o1 && (e1 >> 15));
  }
  return (e && hn > 1) ? 2 : (deep ? 1 : 0);
}

// Warp-wide walk for long runs (expected run >= 32 records per outer per
// bucket): each warp takes its outers one at a time, with the outer's state
// in registers, and loads all nch chunks of its run at once (chunk k = window
// offsets [32k, 32k + 32)); nch covers the expected run plus ~3 sigma.  An
// outer whose last chunk is still full is flagged for continue_pass
// (off = 32 * nch).  Same record semantics as window_pass.
constexpr int kMaxCh = kJoinWarps > 8 ? 6 : 12;  // chunks of one run in flight
// chunk counts of runs of lambda = 256, 128 and 64 records per outer per
// bucket (ceil((lambda + 2 sqrt(lambda) + 8) / 32): a run longer than that,
// ~2 % of them, is finished by continue_pass), compiled as their own
// run_pass instances: the default plan runs 128 on both sides, sharded plans
// 64, RFR_LAMBDA_LOG=8 256
constexpr int kNch256 = 10, kNch128 = 5, kNch64 = 3;
// SMALLH: halo below 2^32 (factor-mode windows) and W = 2^sh with sh >= 32,
// so "in bucket" and "in halo" are 32-bit tests on the high / low words.
// 32-bit bucket/halo classification in the run pass (SMALLH): the halo fits
// 32 bits and both inner lists are long enough that every chunk lane is a
// record (q < 32 kMaxCh <= Mi).
__device__ __forceinline__ bool use_smallh(const JoinPlan& P) {
  return P.half < (1ull << 32) && P.r <= 32 && (32u * kMaxCh >> P.list[1].bits) == 0u &&
         (32u * kMaxCh >> P.list[3].bits) == 0u;
}

// NCH > 0: the chunk count fixed at compile time (the production plans' run
// lengths), so the chunk loads need no per-chunk predicate and the chunks
// past the run cost no code; 0: nch at run time (any plan), <= kMaxCh.
// NOOVF (side A): the caller checked that the warp's runs cannot overflow its
// partition (wfill + outers * 32 * NCH <= kPart), so no per-chunk check.
template <bool SIDE_A, bool SMALLH, int NCH = 0, bool NOOVF = false>
__device__ __noinline__ PassSt run_pass(const JoinArgs& a, uint64_t cW, uint32_t lo, uint32_t hi,
                                      int nch, PassSt st) {
  constexpr int KM = NCH ? NCH : kMaxCh;
  if (NCH) nch = NCH;
  JoinSmem& S = join_smem();
  uint32_t wfill = st.wfill, n_stat = st.n_stat, n_qprobe = st.n_qprobe;
  bool overflow = st.overflow, cont = false;
  const JoinPlan& P = a.P;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t Mi = 1u << P.list[SIDE_A ? 1 : 3].bits;
  const uint64_t* __restrict__ kin = a.key[SIDE_A ? 1 : 3];
  const int aib = P.list[1].bits;
  const JoinK K = make_k(a, cW);
  const bool can_cont = (uint32_t)(32 * nch) < Mi;
  unsigned long long* tr = (RFR_JOIN_TRACE && a.dbg && blockIdx.x == 0 && threadIdx.x == 0 &&
                            cW == ((P.bucket_begin + 1) << K.sh))
                               ? a.dbg + 128 + (SIDE_A ? 0 : 64)
                               : nullptr;
  int trn = 0;
  uint32_t nq = 0;  // staged deep probes, flushed when the staging area fills and after the pass
  for (uint32_t i = lo; i < hi; i++) {
    const uint32_t pos = (SIDE_A ? S.apos : S.bpos)[i];
    const uint32_t rot = (SIDE_A ? S.arot : S.brot)[i];
    const uint64_t x = (SIDE_A ? S.ax : S.bx)[i];
    if (RFR_JOIN_TRACE && tr && trn < 60) tr[trn++] = clock64();
    uint64_t kv[KM];
#pragma unroll
    for (int k = 0; k < KM; k++) {
      const uint32_t q = (uint32_t)(k * 32 + lane);
      // SMALLH: every chunk lane is a list entry (Mi >= 32 kMaxCh)
      kv[k] = ((NCH || k < nch) && (SMALLH || q < Mi)) ? ld_stream(kin + ((rot + pos + q) & (Mi - 1))) : 0ull;
    }
    if (RFR_JOIN_TRACE && tr && trn < 60) tr[trn++] = clock64() | (1ull << 63);
    // along a run the offset rel = x + key - cW grows with q (one pass over the
    // rotated list), so the in-bucket records (m) and the records kept (e:
    // bucket + halo) are both prefixes of the run: a kept record's rank in
    // its chunk is its lane, and the main count is a per-lane tally reduced
    // once per outer.  A record at o >= Mi wraps to the head of the list and
    // has rel >= 2^64 - cW >= W, so it can be halo but never main.
    const uint32_t lim = Mi - pos;  // o < Mi  <=>  q < lim  (pos <= Mi)
    uint32_t mcl = 0, em = 0, em_prev = 0;
#pragma unroll
    for (int k = 0; k < KM; k++) {
      if (NCH || k < nch) {
        const uint32_t q = (uint32_t)(k * 32 + lane);
        const uint32_t j = (rot + pos + q) & (Mi - 1);
        const uint64_t sv = x + kv[k];
        const uint64_t rel = sv - cW;
        bool m, e;
        if (SMALLH) {  // dispatched only when Mi >= 32 kMaxCh: every q is a record
          const uint32_t rh = (uint32_t)(rel >> 32), rl = (uint32_t)rel;
          const uint32_t wh = (uint32_t)(K.W >> 32);
          m = q < lim && rh < wh;
          e = m || (rh == wh && rl < (uint32_t)K.H);
        } else {
          const bool valid = q < Mi;
          m = q < lim && rel < K.W;
          e = m || (valid && (rel - K.W) < K.H);
        }
        // side B needs the kept mask only to skip an empty last chunk and for
        // the continuation test: the earlier chunks of a run are (almost)
        // never empty, and an empty one is harmless (every lane predicated off)
        const bool last = NCH ? k == KM - 1 : k == nch - 1;
        if (SIDE_A || RFR_JOIN_CHECK || last) em = __ballot_sync(FULL, e);
        if (RFR_JOIN_CHECK && (em & (em + 1u)) != 0u) __trap();
        // ... and a prefix of the whole run: no kept record after a chunk that is not full
        if (RFR_JOIN_CHECK && k > 0 && em != 0u && em_prev != FULL) __trap();
        if (RFR_JOIN_CHECK) em_prev = em;
        mcl += m ? 1u : 0u;
        n_stat += e ? 1u : 0u;
        if ((SIDE_A || RFR_JOIN_CHECK || last) && em == 0) {
          // chunk entirely past the run (warp-uniform): nothing to store or probe
        } else if (SIDE_A) {
          const uint32_t ne = __popc(em);
          if (!NOOVF && wfill + ne > (uint32_t)kPart) overflow = true;  // warp-uniform
#if RFR_APASS_PRED
          {  // the record's four stores, predicated (no divergence region per chunk)
            const bool st = (NOOVF || !overflow) && e;
#if RFR_APASS_NOCLAMP
            // NOOVF: wfill + 32 * chunks <= kPart, so the slot is always in the partition
            const uint32_t r = NOOVF ? wid * kPart + wfill + lane
                                     : min(wid * kPart + wfill + lane, (uint32_t)kCapRec - 1u);
#else
            const uint32_t r = min(wid * kPart + wfill + lane, (uint32_t)kCapRec - 1u);  // em is a prefix
#endif
            const uint32_t h1 = home_of(rel, K.sh - kL1Log, kL1Log);
            asm volatile(
                "{\n\t.reg .pred ps;\n\t"
                "setp.ne.u32 ps, %0, 0;\n\t"
                "@ps st.shared.u64 [%1], %2;\n\t"
                "@ps st.shared.u32 [%3], %4;\n\t"
                "@ps st.shared.u16 [%5], %6;\n\t"
                "@ps st.shared.u16 [%7], %8;\n\t}"
                ::"r"((uint32_t)st), "r"((uint32_t)__cvta_generic_to_shared(&S.recK[r])), "l"(sv),
                "r"((uint32_t)__cvta_generic_to_shared(&S.recI[r])), "r"((i << aib) | j),
                "r"((uint32_t)__cvta_generic_to_shared(&S.t1[h1])), "h"((uint16_t)r),
                "r"((uint32_t)__cvta_generic_to_shared(&S.rh[r])), "h"((uint16_t)h1)
                : "memory");
          }
#else
          if ((NOOVF || !overflow) && e) {
            const uint32_t r = wid * kPart + wfill + lane;  // em is a prefix
            S.recK[r] = sv;
            S.recI[r] = (i << aib) | j;
            const uint32_t h1 = home_of(rel, K.sh - kL1Log, kL1Log);
            S.t1[h1] = (uint16_t)r;
            S.rh[r] = (uint16_t)h1;
          }
#endif
          if (NOOVF || !overflow) wfill += ne;
        } else {
          const int deep = probe_b_l1_fast(S, a, K, e, sv, !m, i, j, n_qprobe);
          if (__any_sync(FULL, deep != 0)) {  // ~1 chunk in 5 has a flagged-slot record
            const uint32_t dm = __ballot_sync(FULL, deep != 0);
#if RFR_STAGE_PRED
            {
              const uint32_t kk = min(nq + __popc(dm & lt_mask), (uint32_t)kStageB - 1u);
              const uint32_t qj = (m ? 0u : 0x80000000u) | (deep == 2 ? 0x40000000u : 0u) | j;
              asm volatile(
                  "{\n\t.reg .pred pd;\n\t"
                  "setp.ne.u32 pd, %0, 0;\n\t"
                  "@pd st.shared.u64 [%1], %2;\n\t"
                  "@pd st.shared.u32 [%3], %4;\n\t"
                  "@pd st.shared.u16 [%5], %6;\n\t}"
                  ::"r"((uint32_t)deep), "r"((uint32_t)__cvta_generic_to_shared(&S.qK[wid][kk])), "l"(sv),
                  "r"((uint32_t)__cvta_generic_to_shared(&S.qJ[wid][kk])), "r"(qj),
                  "r"((uint32_t)__cvta_generic_to_shared(&S.qB[wid][kk])), "h"((uint16_t)i)
                  : "memory");
            }
#else
            if (deep) {
              const uint32_t kk = nq + __popc(dm & lt_mask);
              S.qK[wid][kk] = sv;
              S.qJ[wid][kk] = (m ? 0u : 0x80000000u) | (deep == 2 ? 0x40000000u : 0u) | j;
              S.qB[wid][kk] = (uint16_t)i;
            }
#endif
            nq += __popc(dm);
            if (nq > (uint32_t)(kStageB - 32)) {  // keep room for one more chunk
              n_qprobe += process_staged(a, cW, nq);
              nq = 0;
            }
          }
        }
      }
    }
    const uint32_t mc = __reduce_add_sync(FULL, mcl);
    const bool sat = em == FULL && can_cont;  // warp-uniform
    if (lane == 0) (SIDE_A ? S.amain : S.bmain)[i] = mc | (sat ? kFlagCont : 0u);
    cont |= sat;
    // the next bucket's run of this outer starts at pos + mc: pull its lines
    // into L2 now (one 128-byte line per lane), so the next bucket's loads do
    // not all wait on HBM together right after the barrier
    if (RFR_JOIN_PREFETCH && (uint32_t)lane < (uint32_t)(nch * 2)) {
      const uint32_t q = pos + mc + (uint32_t)lane * 16u;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(kin + ((rot + q) & (Mi - 1))));
    }
  }
  if (!SIDE_A && nq) n_qprobe += process_staged(a, cW, nq);
  if (RFR_JOIN_TRACE && tr && trn < 63) tr[trn++] = clock64();
  return PassSt{wfill, n_stat, n_qprobe, overflow, cont};
}

// Build levels 2 and 3 from the level-1 losers (plain stores + read-back).
// Called by every thread after the barrier that follows the level-1 stores;
// returns after a barrier with S.n4 / S.ovf valid.
__device__ __noinline__ void build_index_levels() {
  JoinSmem& S = join_smem();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t nw = S.wcnt[wid];
  uint16_t* lose = S.lose[wid];
  // level 1 read-back: losers go to level 2.  Four 32-record groups per
  // iteration: all record and slot loads are issued before the first ballot
  // (a flag written by an earlier group leaves the slot's index bits intact).
  uint32_t nl = 0;
  auto group = [&](uint32_t e0, auto Gc) {
    constexpr int G = decltype(Gc)::value;
    uint32_t h1[G], occ[G];
#pragma unroll
    for (int u = 0; u < G; u++) {
      const uint32_t e = e0 + u * 32 + lane;
      h1[u] = e < nw ? S.rh[wid * kPart + e] : 0u;
    }
#pragma unroll
    for (int u = 0; u < G; u++) occ[u] = S.t1[h1[u]];
#pragma unroll
    for (int u = 0; u < G; u++) {
      const uint32_t e = e0 + u * 32 + lane;
      const uint32_t r = wid * kPart + e;
      const bool lost = e < nw && (occ[u] & 0x7fffu) != r;
      const uint32_t lm = __ballot_sync(FULL, lost);
#if RFR_INDEX_PRED
      // the three stores of a lost record as predicated instructions: ~1 lane
      // in 9 loses, so nearly every group has one, and a branch around them
      // costs a divergence region per group
      {
        const uint32_t k = nl + __popc(lm & lt_mask);
        const uint32_t a_lose = (uint32_t)__cvta_generic_to_shared(&lose[k < (uint32_t)kLose ? k : 0u]);
        const uint32_t a_t2 = (uint32_t)__cvta_generic_to_shared(&S.t2[h1[u] >> 2]);
        const uint32_t a_t1 = (uint32_t)__cvta_generic_to_shared(&S.t1[h1[u]]);
        const uint16_t rv = (uint16_t)r, fv = (uint16_t)(occ[u] | 0x8000u);
        asm volatile(
            "{\n\t.reg .pred pl, pk;\n\t"
            "setp.ne.u32 pl, %0, 0;\n\t"
            "setp.lt.and.u32 pk, %1, %2, pl;\n\t"
            "@pk st.shared.u16 [%3], %4;\n\t"
            "@pl st.shared.u16 [%5], %4;\n\t"
            "@pl st.shared.u16 [%6], %7;\n\t}"
            ::"r"((uint32_t)lost), "r"(k), "r"((uint32_t)kLose), "r"(a_lose), "h"(rv), "r"(a_t2), "r"(a_t1),
            "h"(fv)
            : "memory");
      }
#else
      if (lost) {
        const uint32_t k = nl + __popc(lm & lt_mask);
        if (k < (uint32_t)kLose) lose[k] = (uint16_t)r;
        S.t2[h1[u] >> 2] = (uint16_t)r;
        S.t1[h1[u]] = (uint16_t)(occ[u] | 0x8000u);  // collision flag: B also probes levels 2-3
      }
#endif
      nl += __popc(lm);
    }
  };
  // whole groups of 128 records, then the tail 32 at a time (partitions are
  // ~256 +- 16 records: no warp pays a whole extra group for a few records)
  uint32_t e0 = 0;
  // (a four-group body also takes a tail of >= RFR_INDEX_G4MIN records: its
  // lanes past nw are predicated off, cheaper than three or four tail passes)
  for (; e0 + RFR_INDEX_G4MIN <= nw; e0 += 128) group(e0, std::integral_constant<int, 4>());
#pragma unroll 1  // (unrolled, the tail ran as one 4-group body with bounds checks: ~127 instructions)
  for (; e0 < nw; e0 += 32) group(e0, std::integral_constant<int, 1>());
  if (nl > (uint32_t)kLose && lane == 0) S.ovf = 1;
  const int any2 = __syncthreads_or(nl > 0);
  if (!any2) return;
  // level 2 read-back: losers go to level 3
  uint32_t nl2 = 0;
  const uint32_t nlc = nl < (uint32_t)kLose ? nl : (uint32_t)kLose;
  for (uint32_t e0 = 0; e0 < nlc; e0 += 32) {
    const uint32_t e = e0 + lane;
    bool lost = false;
    uint32_t r = 0, h1 = 0;
    if (e < nlc) {
      r = lose[e];
      h1 = S.rh[r];
      lost = S.t2[h1 >> 2] != (uint16_t)r;
    }
    const uint32_t lm = __ballot_sync(FULL, lost);
    __syncwarp();
#if RFR_INDEX_PRED2
    {
      const uint32_t a_l = (uint32_t)__cvta_generic_to_shared(&lose[min(nl2 + __popc(lm & lt_mask), (uint32_t)kLose - 1u)]);
      const uint32_t a_3 = (uint32_t)__cvta_generic_to_shared(&S.t3[(h1 >> 4) & ((1u << kL3Log) - 1u)]);
      asm volatile(
          "{\n\t.reg .pred pq;\n\t"
          "setp.ne.u32 pq, %0, 0;\n\t"
          "@pq st.shared.u16 [%1], %2;\n\t"
          "@pq st.shared.u16 [%3], %2;\n\t}"
          ::"r"((uint32_t)lost), "r"(a_l), "h"((uint16_t)r), "r"(a_3)
          : "memory");
    }
#else
    if (lost) {
      lose[nl2 + __popc(lm & lt_mask)] = (uint16_t)r;  // compact in place (target <= e)
      S.t3[h1 >> 4] = (uint16_t)r;
    }
#endif
    nl2 += __popc(lm);
    __syncwarp();
  }
  const int any3 = __syncthreads_or(nl2 > 0);
  if (!any3) return;
  // level 3 read-back: losers go to the short list (rare: shared atomic)
  for (uint32_t e = lane; e < nl2; e += 32) {
    const uint32_t r = lose[e];
    if (S.t3[S.rh[r] >> 4] != (uint16_t)r) {
      const unsigned k = atomicAdd(&S.n4, 1u);
      if (k < (unsigned)kList4) S.list4[k] = (uint16_t)r;
      else S.ovf = 1;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void clear_index() {
  JoinSmem& S = join_smem();
  const int t = tid_now();
  const uint4 f4 = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
  uint4* p1 = reinterpret_cast<uint4*>(S.t1);
#pragma unroll
  for (int i = 0; i < (1 << kL1Log) / 8 / kJoinThreads; i++) p1[t + i * kJoinThreads] = f4;
  uint4* p2 = reinterpret_cast<uint4*>(S.t2);
#pragma unroll
  for (int i = 0; i < (1 << kL2Log) / 8 / kJoinThreads; i++) p2[t + i * kJoinThreads] = f4;
  uint4* p3 = reinterpret_cast<uint4*>(S.t3);
  for (int i = t; i < (1 << kL3Log) / 8; i += kJoinThreads) p3[i] = f4;
}

// Slow path for a skewed bucket whose A side overflowed the warp partitions:
// warp 0 fills chunks of at most kCapRec records (halving the chunk when the
// index overflows), and every chunk re-streams B.  Out of line: rare, and it
// keeps the fast loop's register allocation small.
__device__ __noinline__ void slow_bucket(const JoinArgs& a, uint64_t cW, uint32_t aLo, uint32_t aHi,
                                         uint32_t bLo, uint32_t bHi, int gsB, uint32_t& n_ins_r,
                                         uint32_t& n_q_r, uint32_t& n_qprobe_r,
                                         uint32_t& n_chunks_r) {
  JoinSmem& S = join_smem();
  const JoinPlan& P = a.P;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned FULL = 0xffffffffu;
  const uint32_t MoA = 1u << P.list[0].bits, MiA = 1u << P.list[1].bits;
  const uint64_t* __restrict__ kA = a.key[1];
  const int sh = 64 - P.r;
  const uint64_t W = 1ull << sh;
  const uint64_t H = P.half;
  uint32_t n_ins = n_ins_r, n_q = n_q_r, n_qprobe = n_qprobe_r, n_chunks = n_chunks_r;
  // ---- slow path (skewed bucket): chunks of kCapRec records filled by warp 0
  __syncthreads();
  if (tid == 0) {
    S.cur_i = 0;
    S.cur_t = 0;
  }
  for (uint32_t i = tid; i < MoA; i += kJoinThreads) S.amain[i] = 0;
  __syncthreads();
  uint32_t chunk_cap = (uint32_t)kCapRec;  // halves when a chunk overflows the index
  while (true) {
    n_chunks++;
    clear_index();
    const uint32_t save_i = S.cur_i, save_t = S.cur_t;
    __syncthreads();
    if (tid == 0) {
      S.n4 = 0;
      S.ovf = 0;
    }
    __syncthreads();
    if (wid == 0) {
      uint32_t i = S.cur_i, t = S.cur_t, fill = 0;
      while (i < MoA) {
        const uint32_t pos = S.apos[i], rot = S.arot[i];
        const uint64_t x = S.ax[i];
        bool full = false;
        while (true) {
          const uint32_t q = t + lane;
          const bool valid = q < MiA;
          const uint32_t o = pos + q;
          const uint32_t j = (rot + o) & (MiA - 1);
          const uint64_t s = x + (valid ? __ldg(kA + j) : 0ull);
          const uint64_t rel = s - cW;
          const bool m = valid && o < MiA && rel < W;
          const bool e = m || (valid && (rel - W) < H);
          const uint32_t em = __ballot_sync(FULL, e);
          const uint32_t ne_all = __popc(em);
          const uint32_t room = chunk_cap - fill;
          const uint32_t take = ne_all < room ? ne_all : room;  // emitted lanes are a prefix
          if ((uint32_t)lane < take) {
            // spread the chunk round-robin over the warp partitions
            const uint32_t idx = fill + lane;
            const uint32_t r = (idx % kJoinWarps) * kPart + idx / kJoinWarps;
            S.recK[r] = s;
            S.recI[r] = (i << P.list[1].bits) | j;
          }
          const uint32_t mm = __ballot_sync(FULL, m) & (take >= 32 ? FULL : ((1u << take) - 1u));
          if (lane == 0) S.amain[i] += __popc(mm);
          fill += take;
          t += take;
          n_ins += ((uint32_t)lane < take) ? 1u : 0u;
          if (take < ne_all) {  // chunk full inside this run
            full = true;
            break;
          }
          if (ne_all < 32 || t >= MiA) break;
        }
        if (full) break;
        i++;
        t = 0;
      }
      if (lane == 0) {
        S.cur_i = i;
        S.cur_t = t;
      }
      if (lane < kJoinWarps)
        S.wcnt[lane] = fill / kJoinWarps + ((uint32_t)lane < fill % kJoinWarps ? 1u : 0u);
    }
    __syncthreads();
    {  // every warp claims level-1 homes for its partition, then the levels
      const uint32_t nw = S.wcnt[wid];
      for (uint32_t e = lane; e < nw; e += 32) {
        const uint32_t r = wid * kPart + e;
        const uint32_t h1 = home_of(S.recK[r] - cW, sh - kL1Log, kL1Log);
        S.t1[h1] = (uint16_t)r;
        S.rh[r] = (uint16_t)h1;
      }
    }
    __syncthreads();
    build_index_levels();
    if (S.ovf) {  // too many colliding records: redo this chunk with half the records
      __syncthreads();
      if (tid == 0) {
        S.cur_i = save_i;
        S.cur_t = save_t;
      }
      for (uint32_t i = tid; i < MoA; i += kJoinThreads)
        if (i >= save_i) S.amain[i] = 0;  // recounted by the smaller chunks
      chunk_cap = chunk_cap > 64u ? chunk_cap / 2 : 64u;
      __syncthreads();
      continue;
    }
    const bool done = S.cur_i >= MoA;
    PassSt sb{0u, n_q, n_qprobe, false, false};
    sb = gsB > 32 ? (use_smallh(a.P) ? run_pass<false, true>(a, cW, bLo, bHi, gsB >> 5, sb) : run_pass<false, false>(a, cW, bLo, bHi, gsB >> 5, sb))
                  : window_pass<false>(a, cW, bLo, bHi, gsB, sb);
    __syncwarp();
    sb = continue_pass<false>(a, cW, bLo, bHi, gsB, sb);
    n_q = sb.n_stat;
    n_qprobe = sb.n_qprobe;
    __syncthreads();
    if (done) break;
  }
  n_ins_r = n_ins;
  n_q_r = n_q;
  n_qprobe_r = n_qprobe;
  n_chunks_r = n_chunks;
}

__global__ void __launch_bounds__(kJoinThreads, kJoinCtasPerSm)
    join_kernel(const __grid_constant__ JoinArgs a, int gsA, int gsB) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JoinSmem& S = *reinterpret_cast<JoinSmem*>(smem_raw);
  const JoinPlan& P = a.P;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  const uint32_t MoA = 1u << P.list[0].bits, MoB = 1u << P.list[2].bits;
  const bool smallh = use_smallh(P);

  const uint64_t nbk = P.bucket_end - P.bucket_begin;
  const uint64_t c_begin = P.bucket_begin + nbk * blockIdx.x / gridDim.x;
  const uint64_t c_end = P.bucket_begin + nbk * (blockIdx.x + 1) / gridDim.x;
  if (c_begin >= c_end) {
    if (threadIdx.x == 0) atomicAdd(&a.ctr->ctas_done, 1ull);  // the early-exit poller counts CTAs
    return;
  }
  unsigned long long* dbg = (RFR_JOIN_TRACE && a.dbg && blockIdx.x == 0 && tid == 0) ? a.dbg : nullptr;
  int dbg_n = 0;
#define RFR_MARK()                                   \
  do {                                               \
    if (RFR_JOIN_TRACE && dbg && dbg_n < 120) dbg[dbg_n++] = clock64(); \
  } while (0)
  RFR_MARK();

  // outer keys, rotation starts and first-bucket positions: precomputed for
  // every CTA of this launch by join_starts_kernel
  const unsigned long long t_start = a.trace_stop ? rfr_globaltimer() : 0ull;
  const uint32_t* __restrict__ st0 = a.starts + (size_t)blockIdx.x * (MoA + MoB);
  for (uint32_t i = tid; i < MoA; i += kJoinThreads) {
    S.ax[i] = __ldg(a.key[0] + i);
    S.arot[i] = __ldg(a.rots + i);
    S.apos[i] = __ldg(st0 + i);
  }
  for (uint32_t i = tid; i < MoB; i += kJoinThreads) {
    S.bx[i] = __ldg(a.key[2] + i) + P.shift;
    S.brot[i] = __ldg(a.rots + MoA + i);
    S.bpos[i] = __ldg(st0 + MoA + i);
  }

  {
    const uint32_t perWA = (MoA + kJoinWarps - 1) / kJoinWarps;
    const uint32_t perWB = (MoB + kJoinWarps - 1) / kJoinWarps;
    if (lane == 0) {
      S.wlo[0][wid] = min(MoA, wid * perWA);
      S.whi[0][wid] = min(MoA, wid * perWA + perWA);
      S.wlo[1][wid] = min(MoB, wid * perWB);
      S.whi[1][wid] = min(MoB, wid * perWB + perWB);
    }
    S.cnt[0][tid] = 0;
    S.cnt[1][tid] = 0;
    S.cnt[2][tid] = 0;
  }
  uint32_t n_chunks = 0;

  uint64_t c = c_begin;
  for (; c < c_end; c++) {
    const uint64_t cW = c << (64 - P.r);
    clear_index();
    if (tid_now() == 0) {
      join_smem().n4 = 0;
      join_smem().ovf = 0;
    }
    __syncthreads();
    // has a verified factor turned up?  Copied in now, read after this
    // bucket's last barrier (issued after the barrier above, so no thread is
    // still reading the previous bucket's copy)
    if (a.early && tid_now() == 0) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&join_smem().stop_buf[0]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n\tcp.async.commit_group;\n" ::"r"(dst),
                   "l"(&a.ctr->found)
                   : "memory");
    }
    RFR_MARK();

    // ---- fast path: A runs (+ continuations) into the warp partitions
    {
      const int t = tid_now(), w = t >> 5;
      PassSt sa{0u, join_smem().cnt[0][t], join_smem().cnt[2][t], false, false};
      const uint32_t wlo = join_smem().wlo[0][w], whi = join_smem().whi[0][w];
      const int nA = gsA >> 5;
      if (gsA > 32 && smallh && (nA == kNch256 || nA == kNch128 || nA == kNch64)) {
        const bool noovf = (whi - wlo) * 32u * (uint32_t)nA <= (uint32_t)kPart;
        if (nA == kNch128)
          sa = noovf ? run_pass<true, true, kNch128, true>(a, cW, wlo, whi, nA, sa)
                     : run_pass<true, true, kNch128>(a, cW, wlo, whi, nA, sa);
        else if (nA == kNch256)
          sa = noovf ? run_pass<true, true, kNch256, true>(a, cW, wlo, whi, nA, sa)
                     : run_pass<true, true, kNch256>(a, cW, wlo, whi, nA, sa);
        else
          sa = noovf ? run_pass<true, true, kNch64, true>(a, cW, wlo, whi, nA, sa)
                     : run_pass<true, true, kNch64>(a, cW, wlo, whi, nA, sa);
      } else {
        sa = gsA > 32 ? (smallh ? run_pass<true, true>(a, cW, wlo, whi, gsA >> 5, sa) : run_pass<true, false>(a, cW, wlo, whi, gsA >> 5, sa))
                        : window_pass<true>(a, cW, wlo, whi, gsA, sa);
      }
      if (sa.cont) {
        __syncwarp();
        sa = continue_pass<true>(a, cW, join_smem().wlo[0][w], join_smem().whi[0][w], gsA, sa);
      }
      join_smem().cnt[0][t] = sa.n_stat;
      join_smem().cnt[2][t] = sa.n_qprobe;
      if ((t & 31) == 0) {
        join_smem().wcnt[w] = sa.wfill;
        if (sa.overflow) join_smem().ovf = 1;
      }
    }
    RFR_MARK();
    __syncthreads();
    bool overflowed = join_smem().ovf != 0;
    if (!overflowed) {
      build_index_levels();
      overflowed = join_smem().ovf != 0;
    }
    RFR_MARK();
    if (!overflowed) {
      {
        const int t = tid_now(), w = t >> 5;
        PassSt sb{0u, join_smem().cnt[1][t], join_smem().cnt[2][t], false, false};
        const uint32_t blo = join_smem().wlo[1][w], bhi = join_smem().whi[1][w];
        const int nB = gsB >> 5;
        sb = gsB > 32 ? (smallh ? (nB == kNch128   ? run_pass<false, true, kNch128>(a, cW, blo, bhi, nB, sb)
                                   : nB == kNch256 ? run_pass<false, true, kNch256>(a, cW, blo, bhi, nB, sb)
                                   : nB == kNch64  ? run_pass<false, true, kNch64>(a, cW, blo, bhi, nB, sb)
                                                   : run_pass<false, true>(a, cW, blo, bhi, nB, sb))
                                : run_pass<false, false>(a, cW, blo, bhi, nB, sb))
                      : window_pass<false>(a, cW, join_smem().wlo[1][w], join_smem().whi[1][w], gsB, sb);
        RFR_MARK();
        if (sb.cont) {
          __syncwarp();
          sb = continue_pass<false>(a, cW, join_smem().wlo[1][w], join_smem().whi[1][w], gsB, sb);
        }
        RFR_MARK();
        join_smem().cnt[1][t] = sb.n_stat;
        join_smem().cnt[2][t] = sb.n_qprobe;
      }
      __syncwarp();
      {
        const int t = tid_now(), w = t >> 5, l = t & 31;
        for (uint32_t i = join_smem().wlo[1][w] + l; i < join_smem().whi[1][w]; i += 32) join_smem().bpos[i] += join_smem().bmain[i];
        for (uint32_t i = join_smem().wlo[0][w] + l; i < join_smem().whi[0][w]; i += 32) join_smem().apos[i] += join_smem().amain[i];
      }
      RFR_MARK();
      if (a.early && tid_now() == 0) {
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        if (RFR_STOP_COHERENT && ld_found_gpu(&a.ctr->found) == a.early) join_smem().stop_buf[0] = a.early;
      }
      __syncthreads();
      RFR_MARK();
      if (a.early && join_smem().stop_buf[0] == a.early) {
        if (tid_now() == 0) {
          const unsigned long long t = rfr_globaltimer();
          atomicMax(&a.ctr->t_stop, t);
          atomicCAS(&a.ctr->t_stop_first, 0ull, t);
        }
        c++;
        break;
      }
      continue;
    }

    // ---- slow path (skewed bucket)
    {
      const int t = tid_now(), w = t >> 5, l = t & 31;
      uint32_t n_ins = join_smem().cnt[0][t], n_q = join_smem().cnt[1][t], n_qprobe = join_smem().cnt[2][t];
      slow_bucket(a, cW, join_smem().wlo[0][w], join_smem().whi[0][w], join_smem().wlo[1][w], join_smem().whi[1][w], gsB, n_ins, n_q,
                  n_qprobe, n_chunks);
      join_smem().cnt[0][t] = n_ins;
      join_smem().cnt[1][t] = n_q;
      join_smem().cnt[2][t] = n_qprobe;
      for (uint32_t i = join_smem().wlo[1][w] + l; i < join_smem().whi[1][w]; i += 32) join_smem().bpos[i] += join_smem().bmain[i];
      for (uint32_t i = join_smem().wlo[0][w] + l; i < join_smem().whi[0][w]; i += 32) join_smem().apos[i] += join_smem().amain[i];
    }
    if (a.early && tid_now() == 0) {
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      if (RFR_STOP_COHERENT && ld_found_gpu(&a.ctr->found) == a.early) join_smem().stop_buf[0] = a.early;
    }
    __syncthreads();
    if (a.early && join_smem().stop_buf[0] == a.early) {
      if (tid_now() == 0) {
        const unsigned long long t = rfr_globaltimer();
        atomicMax(&a.ctr->t_stop, t);
        atomicCAS(&a.ctr->t_stop_first, 0ull, t);
      }
      c++;
      break;
    }
  }
  // the CTA's counters as one atomic each (one per thread from every CTA at
  // once queued ~2*10^5 atomics on one line at the end of the join)
  __syncthreads();
  if (tid < 3) {
    unsigned long long sum = 0;
    for (int t = 0; t < kJoinThreads; t++) sum += S.cnt[tid][t];
    atomicAdd(tid == 0 ? &a.ctr->inserts : tid == 1 ? &a.ctr->queries : &a.ctr->query_probes, sum);
  }
  if (tid == 0) {
    if (a.trace_stop) {
      unsigned int smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_cta_stop[3 * blockIdx.x] = rfr_globaltimer();
      g_cta_stop[3 * blockIdx.x + 1] = ((unsigned long long)smid << 32) | (unsigned long long)(c - c_begin);
      g_cta_stop[3 * blockIdx.x + 2] = t_start;
    }
    atomicAdd(&a.ctr->chunks, (unsigned long long)n_chunks);
    atomicAdd(&a.ctr->buckets, (unsigned long long)(c - c_begin));  // fewer on an early exit
    __threadfence();  // every hit of this CTA is visible before it counts as done
    atomicAdd(&a.ctr->ctas_done, 1ull);
  }
}
