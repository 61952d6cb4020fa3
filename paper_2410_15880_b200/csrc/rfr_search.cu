#include <utility>
#include <algorithm>
#include <vector>
#include <cstdio>
#include <cmath>
// rfr_search.cu -- the recombination search (meet in the middle) on sm_100a.
//
// Replaces the reference's backend e hot loops (pkg/src/polyfactor/
// recombine.py:297-358, _splat_merged_raw / _stream_merged_raw, driven by
// recombine_e :727-775).  The reference splats one half into a hash-like
// table in DRAM and probes it with the other half; here the folded pattern
// space is factored into four sorted quarter lists and the two halves are
// generated bucket by bucket, in key order, straight into shared memory, so
// no half list is ever materialised in HBM (DESIGN.md sections 3-4).
//
//   lists_base_kernel        sorted subset sums of <= 2^12 entries (smem bitonic)
//   lists_merge_kernel       one doubling level L -> merge(L, rotate(L + v))
//   join_kernel              bucket-walk generation + smem counting sort +
//                            windowed probe; emits matching patterns
//   recheck_kernel           parity mode: reference float64 value/accept
//   keyfilter_kernel         factor mode: secondary (third power sum) key window
//                            (recombine.py:106-123, :148-162) on every hit
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "rfr_common.cuh"
#include "rfr_internal.h"
#include "rfr_verify.cuh"

namespace cg = cooperative_groups;

namespace rfr {

// ---------------------------------------------------------------- lists
__device__ __forceinline__ uint64_t elem_key(const uint64_t* keys, const ListSpec& L, int i) {
  uint64_t k = keys[L.first + i];
  return L.negate ? (0ull - k) : k;
}

// Select element i of a 4-array held in kernel parameters without dynamic
// indexing (which would copy the whole parameter struct to local memory).
template <class T>
__device__ __forceinline__ T pick4(const T (&v)[4], int i) {
  return i == 0 ? v[0] : (i == 1 ? v[1] : (i == 2 ? v[2] : v[3]));
}
__device__ __forceinline__ ListSpec pick_list(const JoinPlan& P, int i) {
  ListSpec L;
  L.first = i == 0 ? P.list[0].first : (i == 1 ? P.list[1].first : (i == 2 ? P.list[2].first : P.list[3].first));
  L.bits = i == 0 ? P.list[0].bits : (i == 1 ? P.list[1].bits : (i == 2 ? P.list[2].bits : P.list[3].bits));
  L.negate = i == 0 ? P.list[0].negate : (i == 1 ? P.list[1].negate : (i == 2 ? P.list[2].negate : P.list[3].negate));
  L.pat_shift = i == 0 ? P.list[0].pat_shift : (i == 1 ? P.list[1].pat_shift : (i == 2 ? P.list[2].pat_shift : P.list[3].pat_shift));
  return L;
}

// One CTA per list: the 2^b sorted subset sums (b = min(bits, kBaseBits)) of
// the list's first b elements, by b doubling levels in shared memory:
// L_{i+1} = merge(L_i, rotate(L_i + v_i)), every element placed by its rank
// (its index plus a binary search in the other sorted half; ties put L_i
// first), ping-ponging between two buffers.
struct BaseSmem {
  uint64_t k[2][1 << kBaseBits];
  uint32_t p[2][1 << kBaseBits];
  uint64_t v[kBaseBits + 1];  // the level keys, loaded once (not one global load per level)
  uint32_t cnt[3];            // # entries of level i below -v_i, accumulated by level i - 1
};

// # of entries of the ascending rotated sequence s[(r + j) mod n] + v, j < n,
// that are < x (strict) or <= x (!strict)
__device__ __forceinline__ uint32_t rank_rot(const uint64_t* s, uint32_t n, uint32_t r, uint64_t v,
                                             uint64_t x, bool strict) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint64_t y = s[(r + mid) & (n - 1)] + v;
    if (strict ? (y < x) : (y <= x)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(1024) lists_base_kernel(const uint64_t* __restrict__ keys,
                                                          JoinPlan P, ListBufs out, uint32_t* rot) {
  extern __shared__ __align__(16) unsigned char base_raw[];
  BaseSmem& S = *reinterpret_cast<BaseSmem*>(base_raw);
  pdl_trigger();  // the first merge level may launch (it waits for this grid)
  const ListSpec L = pick_list(P, blockIdx.x);
  const int b = L.bits < kBaseBits ? L.bits : kBaseBits;
  const int len = 1 << b;
  const int tid = threadIdx.x;
  if (tid == 0) {
    S.k[0][0] = 0;
    S.p[0][0] = 0;
  }
  if (tid <= b && tid < L.bits) S.v[tid] = elem_key(keys, L, tid);
  if (tid < 3) S.cnt[tid] = 0;
  __syncthreads();
  if (tid == 0) S.cnt[0] = S.v[0] != 0 ? 1u : 0u;  // level 0 = {0}: 0 < -v_0 iff v_0 != 0
  __syncthreads();
  int cur = 0;
  for (int i = 0; i < b; i++) {
    const uint32_t n = 1u << i;
    const uint64_t v = S.v[i];
    const uint64_t* A = S.k[cur];
    // rotation start: # of A < -v (0 when v == 0 or when every A is < -v),
    // counted by the previous level as it placed its outputs
    uint32_t r = S.cnt[i % 3];
    if (r >= n) r = 0;
    if (tid == 0) S.cnt[(i + 2) % 3] = 0;  // read at level i - 1, summed at level i + 1
    const uint64_t thr = i + 1 < b ? 0ull - S.v[i + 1] : 0ull;  // next level's threshold
    uint32_t below = 0;
    uint64_t* Ok = S.k[cur ^ 1];
    uint32_t* Op = S.p[cur ^ 1];
    for (uint32_t e = tid; e < 2 * n; e += blockDim.x) {
      uint64_t x;
      if (e < n) {  // A[e]: after e A's and the B's strictly below it
        x = A[e];
        const uint32_t d = e + rank_rot(A, n, r, v, x, true);
        Ok[d] = x;
        Op[d] = S.p[cur][e];
      } else {  // B'[j] = A[(r + j) mod n] + v: after j B's and the A's <= it
        const uint32_t j = e - n, src = (r + j) & (n - 1);
        x = A[src] + v;
        uint32_t lo = 0, hi = n;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (A[mid] <= x) lo = mid + 1;
          else hi = mid;
        }
        Ok[j + lo] = x;
        Op[j + lo] = S.p[cur][src] | (1u << i);
      }
      below += x < thr ? 1u : 0u;
    }
    below = __reduce_add_sync(0xffffffffu, below);
    if ((tid & 31) == 0 && below) atomicAdd(&S.cnt[(i + 1) % 3], below);
    __syncthreads();
    cur ^= 1;
  }
  uint64_t* ok = pick4(out.k, blockIdx.x);
  uint32_t* op = pick4(out.p, blockIdx.x);
  for (int p = tid; p < len; p += blockDim.x) {
    ok[p] = S.k[cur][p];
    op[p] = S.p[cur][p];
  }
  // rotation counters of the merge levels: zero them, and seed the first
  // level's (# sums < -v_b, v_b = key of element b)
  uint32_t* rc = rot + blockIdx.x * kRotSlots;
  for (int k = tid; k < kRotSlots; k += blockDim.x) rc[k] = 0;
  __syncthreads();
  if (L.bits > b) {
    const uint64_t thr = 0ull - S.v[b];
    uint32_t c = 0;
    for (int p = tid; p < len; p += blockDim.x) c += S.k[cur][p] < thr ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((tid & 31) == 0 && c) atomicAdd(rc + b, c);
  }
}


// One doubling level for every list that has it: L (2^k sorted sums of the
// list's first k elements) -> merge(L, rotate(L + v_k)), v_k the key of
// element k; the rotated copy B'[j] = L[(rot + j) mod 2^k] + v_k is ascending.
// Each CTA produces one tile of kMergeTile outputs between two merge-path
// splits found by lists_split_kernel; the tile's inputs are
// staged in shared memory with coalesced loads, every thread merges
// kMergeItems outputs from shared memory, and the tile is stored coalesced.
// rot comes from the counter the previous level accumulated (# sums < -v_k),
// and this level accumulates the next one, so no thread ever binary-searches
// a list in global memory for it.
constexpr int kMergeItems = 8;
constexpr int kMergeThreads = 256;
constexpr int kMergeTile = kMergeItems * kMergeThreads;

// Bank-conflict-free tile layout (XOR swizzle inside each 128-byte row): the
// staging loads, the per-thread runs of kMergeItems and the coalesced
// read-out all hit distinct banks.
__device__ __forceinline__ uint32_t kswz(uint32_t i) { return i ^ ((i >> 4) & 15u); }
__device__ __forceinline__ uint32_t pswz(uint32_t i) { return i ^ ((i >> 5) & 7u); }

__device__ __forceinline__ uint32_t rot_of(const uint32_t* rc, int k, uint32_t n) {
  const uint32_t c = rc[k];
  return c >= n ? 0u : c;
}

// Merge-path splits of one doubling level, one warp per tile boundary
// (32-ary search: ~5 dependent steps for 2^23-entry lists); all boundaries of
// all lists are searched concurrently so the merge CTAs start at their loads.
// H.sp[li][hist_sp_off(k) + t] = # A elements before output tile t (kept:
// it is also the rank directory of the level's provenance bits).
// Merge-path split at output diagonal d of merge(A, B'), B'[j] = A[(r0 + j)
// & mask] + v: the number of A elements among the first d outputs (A first on
// ties), found by the calling warp with a 32-ary search.
__device__ __forceinline__ uint32_t merge_split(const uint64_t* __restrict__ A, uint32_t r0,
                                                uint32_t mask, uint64_t v, uint32_t n, uint32_t d,
                                                int lane) {
  auto Bk = [&](uint32_t j) { return __ldg(A + ((r0 + j) & mask)) + v; };
  // smallest i with A[i] > B'[d - 1 - i] (A first on ties)
  uint32_t lo = d > n ? d - n : 0, hi = d < n ? d : n;
  while (hi > lo) {
    const uint32_t span = hi - lo;
    if (span <= 32) {
      const uint32_t q = lo + lane;
      const bool pr = (uint32_t)lane < span && __ldg(A + q) <= Bk(d - 1 - q);
      lo += __popc(__ballot_sync(0xffffffffu, pr));
      break;
    }
    const uint32_t q = lo + (uint32_t)(((uint64_t)span * lane) >> 5);
    const bool pr = __ldg(A + q) <= Bk(d - 1 - q);
    const uint32_t c = __popc(__ballot_sync(0xffffffffu, pr));
    const uint32_t qc1 = __shfl_sync(0xffffffffu, q, (c > 0 ? c : 1) - 1);
    const uint32_t qc = __shfl_sync(0xffffffffu, q, c < 32 ? c : 31);
    if (c > 0) lo = qc1 + 1;
    if (c < 32) hi = qc;
  }
  return lo;
}

__global__ void __launch_bounds__(256) lists_split_kernel(const uint64_t* __restrict__ keys,
                                                          JoinPlan P, int k, ListBufs in,
                                                          const uint32_t* __restrict__ rot,
                                                          ListHist H) {
  pdl_wait();  // the previous level is complete
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const uint32_t w = blockIdx.x * 8u + (threadIdx.x >> 5);
  const int li = blockIdx.y;
  const ListSpec L = pick_list(P, li);
  if (L.bits <= k) return;
  const uint32_t n = 1u << k;
  const uint32_t ntiles = (2u * n + kMergeTile - 1) / kMergeTile;
  if (w > ntiles) return;
  const uint64_t* __restrict__ A = pick4(in.k, li);
  const uint64_t v = elem_key(keys, L, k);
  const uint32_t r0 = rot_of(rot + li * kRotSlots, k, n);
  const uint32_t mask = n - 1;
  auto Bk = [&](uint32_t j) { return __ldg(A + ((r0 + j) & mask)) + v; };
  const uint32_t d = min(w * (uint32_t)kMergeTile, 2u * n);
  // smallest i with A[i] > B'[d - 1 - i] (A first on ties)
  uint32_t lo = d > n ? d - n : 0, hi = d < n ? d : n;
  while (hi > lo) {
    const uint32_t span = hi - lo;
    if (span <= 32) {
      const uint32_t q = lo + lane;
      const bool pr = (uint32_t)lane < span && __ldg(A + q) <= Bk(d - 1 - q);
      lo += __popc(__ballot_sync(0xffffffffu, pr));
      break;
    }
    const uint32_t q = lo + (uint32_t)(((uint64_t)span * lane) >> 5);
    const bool pr = __ldg(A + q) <= Bk(d - 1 - q);
    const uint32_t c = __popc(__ballot_sync(0xffffffffu, pr));
    const uint32_t qc1 = __shfl_sync(0xffffffffu, q, (c > 0 ? c : 1) - 1);
    const uint32_t qc = __shfl_sync(0xffffffffu, q, c < 32 ? c : 31);
    if (c > 0) lo = qc1 + 1;
    if (c < 32) hi = qc;
  }
  if (lane == 0) pick4(H.sp, li)[hist_sp_off(k) + w] = lo;
}

// Tile staging by the Tensor Memory Accelerator (kMode 2): the tile's A run
// and its rotated B' run are copied as 128-byte rows (16 keys) by
// cp.async.bulk into padded shared rows (144-byte stride: consecutive rows
// start 4 banks apart, so the per-thread runs the merge reads do not pile
// onto one bank pair), completing on one mbarrier; the B' rows are copied
// without "+ v" (added on read) and wrap around the list end row by row.
constexpr int kTmaRowKeys = 16, kTmaRowStride = 18;  // keys per row, padded stride (keys)
constexpr int kTmaRowsSide = kMergeTile / kTmaRowKeys + 2;  // rows per side (offset + partial row)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// kMode 0: splits from lists_split_kernel, staging by loads + shared stores;
// 1: own splits, same staging; 2: own splits, TMA bulk-copy staging.
template <int kMode>
__global__ void __launch_bounds__(kMergeThreads) lists_merge_kernel(const uint64_t* __restrict__ keys,
                                                                    JoinPlan P, int k,
                                                                    ListBufs in, ListBufs out,
                                                                    uint32_t* rot, ListHist H) {
  constexpr bool kOwnSplit = kMode >= 1;
  constexpr bool kTma = kMode == 2;
  __shared__ __align__(128) uint64_t sK[kTma ? 2 * kTmaRowsSide * kTmaRowStride : kMergeTile];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t wsum[kMergeThreads / 32];
  __shared__ uint32_t ssplit[2];
  pdl_wait();  // the previous level (and its rotation counts) is complete
  pdl_trigger();
  const int li = blockIdx.y;
  const ListSpec L = pick_list(P, li);
  if (L.bits <= k) return;
  const uint32_t n = 1u << k;
  const uint32_t d0 = blockIdx.x * (uint32_t)kMergeTile;
  if (d0 >= 2u * n) return;
  const uint64_t* __restrict__ A = pick4(in.k, li);
  uint64_t* __restrict__ O = pick4(out.k, li);
  uint32_t* rc = rot + li * kRotSlots;
  const uint64_t v = elem_key(keys, L, k);
  const uint32_t r0 = rot_of(rc, k, n);
  const uint32_t mask = n - 1;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t* sp = pick4(H.sp, li) + hist_sp_off(k);
  if (kTma && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t a0, a1;
  if (kOwnSplit) {
    // the tile's two merge-path splits, by warps 0 and 1 (one launch per level
    // instead of a split kernel + the merge: the search latency hides behind
    // the other resident CTAs' merges); a0 is also kept as the rank
    // directory of the level's provenance bits
    if (wid < 2) {
      const uint32_t d = min((blockIdx.x + wid) * (uint32_t)kMergeTile, 2u * n);
      const uint32_t a = merge_split(A, r0, mask, v, n, d, lane);
      if (lane == 0) {
        ssplit[wid] = a;
        if (wid == 0 || d == 2u * n) sp[blockIdx.x + wid] = a;
      }
    }
    __syncthreads();
    a0 = ssplit[0];
    a1 = ssplit[1];
  } else {
    a0 = __ldg(sp + blockIdx.x);
    a1 = __ldg(sp + blockIdx.x + 1);
  }
  const uint32_t tile = min((uint32_t)kMergeTile, 2u * n - d0);
  const uint32_t na = a1 - a0, nb = tile - na;
  const uint32_t b0 = d0 - a0;
  const uint32_t sB = (r0 + b0) & mask;  // B' run = A[sB ...] + v, wrapping at n
  const uint32_t offA = a0 & (kTmaRowKeys - 1), offB = sB & (kTmaRowKeys - 1);
  if (kTma) {
    const uint32_t rowsA = na ? (offA + na + kTmaRowKeys - 1) / kTmaRowKeys : 0u;
    const uint32_t rowsB = nb ? (offB + nb + kTmaRowKeys - 1) / kTmaRowKeys : 0u;
    if (wid == 0) {
      const uint32_t mb = smem_u32(&mbar);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                     "r"((rowsA + rowsB) * (uint32_t)(kTmaRowKeys * 8))
                     : "memory");
      __syncwarp();
      const uint32_t nrow = n / kTmaRowKeys;
      for (uint32_t r = lane; r < rowsA + rowsB; r += 32) {
        const bool isA = r < rowsA;
        const uint32_t grow = isA ? (a0 >> 4) + r : ((sB >> 4) + (r - rowsA)) & (nrow - 1);
        const uint32_t srow = isA ? r : kTmaRowsSide + (r - rowsA);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sK + srow * kTmaRowStride)),
            "l"(A + (size_t)grow * kTmaRowKeys), "r"(kTmaRowKeys * 8), "r"(mb)
            : "memory");
      }
    }
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.b32 %0, 1, 0, "
          "p;\n\t}"
          : "=r"(done)
          : "r"(smem_u32(&mbar))
          : "memory");
  } else {
    // one pass over the tile: output slot t < na stages A[a0 + t], the rest
    // stage B'; every thread's kMergeItems loads are independent and issued
    // before the first shared store (the A and B halves as two loops waited
    // on HBM twice per tile)
    auto stage = [&](uint32_t t) {
      const bool isA = t < na;
      const uint64_t* src = isA ? A + a0 + t : A + ((r0 + b0 + (t - na)) & mask);
      return __ldg(src) + (isA ? 0ull : v);
    };
    if (tile == (uint32_t)kMergeTile) {
      uint64_t x[kMergeItems];
#pragma unroll
      for (int u = 0; u < kMergeItems; u++) x[u] = stage(tid + u * kMergeThreads);
#pragma unroll
      for (int u = 0; u < kMergeItems; u++) sK[kswz(tid + u * kMergeThreads)] = x[u];
    } else {
      for (uint32_t t = tid; t < tile; t += kMergeThreads) sK[kswz(t)] = stage(t);
    }
    __syncthreads();
  }
  // staged tile accessors: A run element i, B' run element j
  auto LA = [&](uint32_t i) -> uint64_t {
    if (kTma) {
      const uint32_t x = offA + i;
      return sK[(x >> 4) * kTmaRowStride + (x & 15u)];
    }
    return sK[kswz(i)];
  };
  auto LB = [&](uint32_t j) -> uint64_t {
    if (kTma) {
      const uint32_t x = offB + j;
      return sK[(kTmaRowsSide + (x >> 4)) * kTmaRowStride + (x & 15u)] + v;
    }
    return sK[kswz(na + j)];
  };
  // per-thread merge of kMergeItems outputs from the staged tile
  const uint32_t dt = min((uint32_t)(tid * kMergeItems), tile);
  uint32_t lo = dt > nb ? dt - nb : 0, hi = dt < na ? dt : na;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (LA(mid) <= LB(dt - 1 - mid)) lo = mid + 1;
    else hi = mid;
  }
  uint32_t i = lo, j = dt - lo;
  uint64_t ok[kMergeItems];
  uint32_t from_b = 0;  // provenance bits of this thread's outputs
  // both run heads held in registers: one shared key load per output
  const uint64_t kInf = ~0ull;
  uint64_t ka = i < na ? LA(i) : kInf, kb = j < nb ? LB(j) : kInf;
#pragma unroll
  for (int t = 0; t < kMergeItems; t++) {
    const bool takeA = j >= nb || (i < na && ka <= kb);
    if (kTma) {
      if (takeA) {
        ok[t] = ka;
        i++;
        ka = i < na ? LA(i) : kInf;
      } else {
        ok[t] = kb;
        from_b |= 1u << t;
        j++;
        kb = j < nb ? LB(j) : kInf;
      }
    } else {
      // branch-free: the lanes of a warp take A or B at random, so a branch
      // here runs both sides for every output; the staged tile holds the A
      // run at [0, na) and the B' run at [na, tile), so the new head is one
      // predicated shared load at a selected slot
      ok[t] = takeA ? ka : kb;
      from_b |= (takeA ? 0u : 1u) << t;
      i += takeA ? 1u : 0u;
      j += takeA ? 0u : 1u;
      const bool more = takeA ? i < na : j < nb;
      const uint64_t nv = more ? sK[kswz(takeA ? i : na + j)] : kInf;
      ka = takeA ? nv : ka;
      kb = takeA ? kb : nv;
    }
  }
  // each thread's run of outputs is contiguous and 64-byte aligned: store it
  // directly with 16-byte vector stores
  const uint32_t cnt = dt < tile ? min((uint32_t)kMergeItems, tile - dt) : 0u;
  if (cnt < (uint32_t)kMergeItems) from_b &= (1u << cnt) - 1u;
  if (cnt == (uint32_t)kMergeItems) {
    ulonglong2* ko = reinterpret_cast<ulonglong2*>(O + d0 + dt);
#pragma unroll
    for (int t = 0; t < kMergeItems / 2; t++) ko[t] = make_ulonglong2(ok[2 * t], ok[2 * t + 1]);
  } else {
#pragma unroll
    for (int t = 0; t < kMergeItems; t++)
      if ((uint32_t)t < cnt) O[d0 + dt + t] = ok[t];
  }
  // provenance byte and the rank directory (1-bits in the tile before each
  // 64-output word): block exclusive scan of the per-thread popcounts
  static_assert(kMergeItems == 8 && kMergeTile == (1 << kHistTileLog), "history layout");
  const uint32_t c1 = __popc(from_b);
  uint32_t incl = c1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  uint32_t woff = 0;
  for (int w2 = 0; w2 < wid; w2++) woff += wsum[w2];
  if (cnt) {
    pick4(H.bm, li)[hist_bm_off(k) + ((d0 + dt) >> 3)] = (uint8_t)from_b;
    if ((tid & 7) == 0) pick4(H.dir, li)[hist_dir_off(k) + ((d0 + dt) >> 6)] = (uint16_t)(woff + incl - c1);
  }
  // next level's rotation start: # outputs < -v_{k+1}
  if (L.bits > k + 1) {
    const uint64_t thr = 0ull - elem_key(keys, L, k + 1);
    uint32_t c = 0;
#pragma unroll
    for (int t = 0; t < kMergeItems; t++) c += ((uint32_t)t < cnt && ok[t] < thr) ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0 && c) atomicAdd(rc + k + 1, c);
  }
}

// ---------------------------------------------------------------- join
struct JoinArgs {
  JoinPlan P;
  const uint64_t* key[4];
  // per outer (A outers, then B outers): rotation start, and this launch's
  // start position in each CTA's first bucket (join_starts_kernel)
  const uint32_t* rots;
  const uint32_t* starts;  // [cta][MoA + MoB]
  // early exit: stop at a bucket boundary once DevCounters.found holds this
  // search's epoch (0: no early exit).  An epoch instead of a 0/1 flag lets a
  // peer's flag that lands before this rank cleared its counters count, and
  // keeps a late flag of an earlier search from stopping this one.
  unsigned long long early;
  int trace_stop;          // RFR_STOP_TRACE: each CTA records when and where it stopped
  uint64_t* out;
  unsigned long long cap;
  DevCounters* ctr;
  unsigned long long* dbg;  // optional clock64 trace of CTA 0 (RFR_TRACE)
};

// RFR_STOP_TRACE (diagnostics): per join CTA, the globaltimer when it left
// its bucket loop and (SM id << 32 | buckets searched)
__device__ unsigned long long g_cta_stop[3 * 1024];
#include "rfr_join.cuh"

// lower_bound of v in a sorted array by one warp: 32 probes per round narrow
// [lo, hi] 32-fold, so ~5 dependent loads for 2^28 entries instead of 28.
__device__ __forceinline__ uint32_t warp_lower_bound(const uint64_t* __restrict__ a, uint32_t n,
                                                     uint64_t v, int lane) {
  const unsigned FULL = 0xffffffffu;
  uint32_t lo = 0, hi = n;  // the answer lies in [lo, hi]
  while (hi - lo > 32) {
    const uint32_t span = hi - lo;
    const uint32_t q = lo + (uint32_t)(((uint64_t)span * (uint32_t)(lane + 1)) >> 5) - 1u;
    const uint32_t c = __popc(__ballot_sync(FULL, __ldg(a + q) < v));  // a prefix of the probes
    const uint32_t qlo = __shfl_sync(FULL, q, (c ? c : 1u) - 1u);
    const uint32_t qhi = __shfl_sync(FULL, q, c < 32u ? c : 31u);
    if (c) lo = qlo + 1u;
    if (c < 32u) hi = qhi;
  }
  const uint32_t q = lo + (uint32_t)lane;
  return lo + __popc(__ballot_sync(FULL, q < hi && __ldg(a + q) < v));
}

// Two lower bounds in the same sorted array, advanced in lockstep so their
// dependent loads overlap (the starts kernel's searches miss L2: ~1 us each).
__device__ __forceinline__ void warp_lower_bound2(const uint64_t* __restrict__ a, uint32_t n, uint64_t v0,
                                                  uint64_t v1, int lane, uint32_t* r0, uint32_t* r1) {
  const unsigned FULL = 0xffffffffu;
  uint32_t lo[2] = {0, 0}, hi[2] = {n, n};
  const uint64_t v[2] = {v0, v1};
  while (hi[0] - lo[0] > 32 || hi[1] - lo[1] > 32) {
    uint32_t q[2];
    bool pr[2];
#pragma unroll
    for (int s = 0; s < 2; s++) {
      const uint32_t span = hi[s] - lo[s];
      q[s] = span > 32 ? lo[s] + (uint32_t)(((uint64_t)span * (uint32_t)(lane + 1)) >> 5) - 1u : lo[s];
      pr[s] = span > 32 && __ldg(a + q[s]) < v[s];
    }
#pragma unroll
    for (int s = 0; s < 2; s++) {
      if (hi[s] - lo[s] <= 32) continue;  // warp-uniform
      const uint32_t c = __popc(__ballot_sync(FULL, pr[s]));
      const uint32_t qlo = __shfl_sync(FULL, q[s], (c ? c : 1u) - 1u);
      const uint32_t qhi = __shfl_sync(FULL, q[s], c < 32u ? c : 31u);
      if (c) lo[s] = qlo + 1u;
      if (c < 32u) hi[s] = qhi;
    }
  }
  bool pr[2];
#pragma unroll
  for (int s = 0; s < 2; s++) {
    const uint32_t q = lo[s] + (uint32_t)lane;
    pr[s] = q < hi[s] && __ldg(a + q) < v[s];
  }
  *r0 = lo[0] + __popc(__ballot_sync(FULL, pr[0]));
  *r1 = lo[1] + __popc(__ballot_sync(FULL, pr[1]));
}

// Start state of every join launch of one key window, computed up front with
// one warp per search (the join's CTAs would otherwise each run ~140
// dependent binary-search loads before their first bucket, per launch).
// Task t < MoA + MoB: rotation start of outer t; then, for chunk k and CTA c,
// the outer's count of sums below the CTA's first bucket (count_below).
__global__ void __launch_bounds__(256) join_starts_kernel(JoinPlan P, const uint64_t* __restrict__ kO_A,
                                                          const uint64_t* __restrict__ kA,
                                                          const uint64_t* __restrict__ kO_B,
                                                          const uint64_t* __restrict__ kB,
                                                          uint64_t b0, uint64_t b1, int nck, int ctas,
                                                          uint32_t* __restrict__ rots,
                                                          uint32_t* __restrict__ starts) {
  pdl_wait();  // the top list level is complete
  const int lane = threadIdx.x & 31;
  const uint32_t MoA = 1u << P.list[0].bits, MoB = 1u << P.list[2].bits, MoT = MoA + MoB;
  const uint64_t task = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t ntask = (uint64_t)MoT * (1ull + (uint64_t)nck * (uint64_t)ctas);
  if (task >= ntask) return;  // warp-uniform
  const uint32_t o = (uint32_t)(task % MoT);
  const bool sideB = o >= MoA;
  const uint32_t oi = sideB ? o - MoA : o;
  const uint64_t* __restrict__ inner = sideB ? kB : kA;
  const uint32_t n = 1u << P.list[sideB ? 3 : 1].bits;
  const uint64_t x = sideB ? __ldg(kO_B + oi) + P.shift : __ldg(kO_A + oi);
  const uint64_t l0 = 0ull - x;  // sums start at key -x
  if (task < MoT) {
    if (lane == 0) rots[o] = 0;
    const uint32_t j = x == 0 ? 0u : warp_lower_bound(inner, n, l0, lane);
    if (lane == 0) rots[o] = j == n ? 0u : j;
    return;
  }
  const uint64_t kc = task / MoT - 1;  // chunk * ctas + cta
  const int k = (int)(kc / (uint64_t)ctas), c = (int)(kc % (uint64_t)ctas);
  // the join's own bucket arithmetic (search_core, join_kernel)
  const uint64_t cb = b0 + (b1 - b0) * (uint64_t)k / (uint64_t)nck;
  const uint64_t ce = b0 + (b1 - b0) * (uint64_t)(k + 1) / (uint64_t)nck;
  const uint64_t span = ce - cb;
  const uint64_t grid = span < (uint64_t)ctas ? span : (uint64_t)ctas;
  uint32_t pos = 0;
  if ((uint64_t)c < grid) {
    const uint64_t c_begin = cb + span * (uint64_t)c / grid;
    const uint64_t bound = c_begin << (64 - P.r);
    if (bound != 0) {
      const uint64_t hi = l0 + bound;  // exclusive end, mod 2^64
      uint32_t l, h;
      warp_lower_bound2(inner, n, l0, hi, lane, &l, &h);
      pos = hi > l0 ? h - l : (n - l) + h;  // wraps through 2^64 when hi <= l0
    }
  }
  if (lane == 0) starts[kc * MoT + o] = pos;
}

// ------------------------------------------------- indices -> patterns
// The join emits each hit as its four quarter-list indices (packed at the
// patterns' bit offsets); this pass rewrites every hit as its pattern.
struct PatArgs {
  JoinPlan P;
  const uint32_t* pat[4];  // base-level patterns (lists of <= 2^kBaseBits entries: all of them)
  ListHist hist;           // merge history of the longer lists
  const uint32_t* rot;     // per-list rotation counters of the merge levels
};

static_assert(kMaxOuterBits <= kBaseBits, "outer lists are base-level lists (patterns stored)");
// Local pattern of entry d of quarter list li: lists of at most 2^kBaseBits
// entries store it; longer lists walk their merge history down (one tile
// split, one rank-directory entry and one 64-bit provenance word per level).
__device__ __forceinline__ uint32_t list_pattern(const PatArgs& a, int li, uint32_t d) {
  const int bits = pick_list(a.P, li).bits;
  const uint32_t* base = pick4(a.pat, li);
  if (bits <= kBaseBits) return __ldg(base + d);
  const uint8_t* bm = pick4(a.hist.bm, li);
  const uint16_t* dir = pick4(a.hist.dir, li);
  const uint32_t* sp = pick4(a.hist.sp, li);
  const uint32_t* rc = a.rot + li * kRotSlots;
  uint32_t pat = 0;
  for (int k = bits - 1; k >= kBaseBits; k--) {
    const uint32_t n = 1u << k;
    const uint32_t t = d >> kHistTileLog, d0 = t << kHistTileLog;
    const uint32_t a0 = __ldg(sp + hist_sp_off(k) + t);
    const uint64_t w = __ldg(reinterpret_cast<const unsigned long long*>(bm + hist_bm_off(k)) + (d >> 6));
    const uint32_t pre = __ldg(dir + hist_dir_off(k) + (d >> 6));
    const uint32_t c1 = pre + __popcll(w & ((1ull << (d & 63)) - 1ull));  // 1-bits in [d0, d)
    if (!((w >> (d & 63)) & 1ull)) {
      d = a0 + (d - d0 - c1);  // from L_k
    } else {                   // from rotate(L_k + v_k)
      const uint32_t c = __ldg(rc + k);
      const uint32_t r0 = c >= n ? 0u : c;
      d = (r0 + (d0 - a0) + c1) & (n - 1);
      pat |= 1u << k;
    }
  }
  return pat | __ldg(base + d);
}

__global__ void __launch_bounds__(256) index_to_pattern_kernel(const PatArgs a, uint64_t* out,
                                                               const unsigned long long* count,
                                                               unsigned long long cap,
                                                               const unsigned long long* begin) {
  pdl_wait();  // programmatic launch: the previous kernel is complete
  pdl_trigger();
  unsigned long long m = *count;
  if (m > cap) m = cap;
  const unsigned long long m0 = begin ? min(*begin, m) : 0ull;  // hits [m0, m) are new
  const JoinPlan& P = a.P;
  // four lanes per hit, one per quarter list: the two long history walks
  // (the inner lists) run side by side instead of back to back
  const int li = threadIdx.x & 3;
  const ListSpec L = pick_list(P, li);
  const unsigned long long lanes = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long wbase = (unsigned long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  for (unsigned long long tb = wbase; tb < 4 * (m - m0); tb += lanes) {  // warp-uniform trip count
    const unsigned long long i = m0 + ((tb + (threadIdx.x & 31u)) >> 2);
    uint64_t part = 0;
    if (i < m) {
      const uint64_t v = out[i];
      const uint32_t idx = (uint32_t)((v >> L.pat_shift) & ((1ull << L.bits) - 1ull));
      part = (uint64_t)list_pattern(a, li, idx) << L.pat_shift;
    }
    part |= __shfl_xor_sync(0xffffffffu, part, 1);
    part |= __shfl_xor_sync(0xffffffffu, part, 2);
    if (li == 0 && i < m) out[i] = part;
  }
}

cudaError_t launch_index_to_pattern(const JoinPlan& P, const ListBufs& base, const ListHist& hist,
                                    const uint32_t* d_rot, uint64_t* d_out,
                                    const unsigned long long* d_count, unsigned long long cap, int nsm,
                                    cudaStream_t s, const unsigned long long* d_begin) {
  PatArgs a;
  a.P = P;
  for (int i = 0; i < 4; i++) a.pat[i] = base.p[i];
  a.hist = hist;
  a.rot = d_rot;
  cudaError_t e = launch_pdl(index_to_pattern_kernel, dim3(nsm * 4), dim3(256), 0, s, a, d_out, d_count, cap, d_begin);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ------------------------------------------------------------- recheck
// Parity mode: keep a hit t iff accept(value(t), eps), value() accumulated in
// ascending index order in IEEE double (R/recombine.py:106-123, :148-162).
__global__ void recheck_kernel(const double* __restrict__ rho, const uint64_t* __restrict__ in,
                               const unsigned long long* __restrict__ in_count,
                               unsigned long long cap_in, double eps, uint64_t* __restrict__ out,
                               unsigned long long cap_out, DevCounters* ctr) {
  unsigned long long n = *in_count;
  if (n > cap_in) n = cap_in;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    uint64_t t = in[i];
    double x = 0.0;
    uint64_t u = t;
    while (u) {
      int b = __ffsll((long long)u) - 1;
      x = __dadd_rn(x, rho[b]);
      u &= u - 1;
    }
    double y = __dadd_rn(x, -floor(x));
    if (y < eps || __dadd_rn(1.0, -y) < eps) {
      unsigned long long k = atomicAdd(&ctr->post_count, 1ull);
      if (k < cap_out) out[k] = t;
    }
  }
}

// Factor mode, secondary key: keep the raw hits t whose second key sum lies
// in the window, (sum_{i in t} keys2[i] - lo2) mod 2^64 <= width2 (the third
// power sum of a true factor is an integer, so its key sum is near 0).
__global__ void keyfilter_kernel(const uint64_t* __restrict__ keys2, int n,
                                 const uint64_t* __restrict__ in,
                                 const unsigned long long* __restrict__ in_count,
                                 unsigned long long cap_in, uint64_t lo2, uint64_t width2,
                                 uint64_t* __restrict__ out, unsigned long long cap_out,
                                 DevCounters* ctr, const unsigned long long* __restrict__ begin) {
  pdl_wait();  // programmatic launch: the previous kernel is complete
  pdl_trigger();
  __shared__ uint64_t sk[64];
  for (int i = threadIdx.x; i < n; i += blockDim.x) sk[i] = keys2[i];
  __syncthreads();
  unsigned long long m = *in_count;
  if (m > cap_in) m = cap_in;
  const unsigned long long m0 = begin ? min(*begin, m) : 0ull;
  for (unsigned long long i = m0 + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint64_t t = in[i];
    uint64_t sum = 0, u = t;
    while (u) {
      sum += sk[__ffsll((long long)u) - 1];
      u &= u - 1;
    }
    if (sum - lo2 <= width2) {
      const unsigned long long k = atomicAdd(&ctr->post_count, 1ull);
      if (k < cap_out) out[k] = t;
    }
  }
}

// Parity-mode keys: round(rho * 2^64) mod 2^64 (exact: rho * 2^64 is an
// exact double; values >= 2^63 are split before the unsigned conversion).
__global__ void rho_keys_kernel(const double* __restrict__ rho, int n, uint64_t* __restrict__ keys) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = ldexp(rho[i], 64);
  v = nearbyint(v);
  uint64_t k;
  const double two63 = 9223372036854775808.0;
  if (v >= two63) k = (uint64_t)(long long)(v - two63) + (1ull << 63);
  else k = (uint64_t)(long long)v;
  keys[i] = k;
}

}  // namespace rfr

// ------------------------------------------------------ host-side launchers
namespace rfr {

// cudaFuncSetAttribute is per device context: remember, per device, which
// kernels have had their dynamic shared-memory limit raised.
template <typename K>
static cudaError_t raise_smem_limit(K kernel, size_t bytes, uint64_t& done_mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? 1ull << dev : 0;
  if (bit && (done_mask & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done_mask |= bit;
  return e;
}

// Bytes of one list's merge history (bitmaps, rank directory, splits).
size_t list_hist_bytes(int bits) {
  if (bits <= kBaseBits) return 0;
  const size_t bm = hist_bm_off(bits), dir = hist_dir_off(bits) * 2, sp = hist_sp_off(bits) * 4;
  return ((bm + 15) & ~(size_t)15) + ((dir + 15) & ~(size_t)15) + sp + 16;
}
ListHist list_hist_layout(const JoinPlan& P, char* const base[4]) {
  ListHist H;
  for (int i = 0; i < 4; i++) {
    const int bits = P.list[i].bits;
    char* b = base[i];
    const size_t bm = bits > kBaseBits ? hist_bm_off(bits) : 0;
    const size_t dir = bits > kBaseBits ? hist_dir_off(bits) * 2 : 0;
    H.bm[i] = (uint8_t*)b;
    H.dir[i] = (uint16_t*)(b + ((bm + 15) & ~(size_t)15));
    H.sp[i] = (uint32_t*)(b + ((bm + 15) & ~(size_t)15) + ((dir + 15) & ~(size_t)15));
  }
  return H;
}

// Levels of at least this many merge tiles get their merge-path splits from
// a separate split kernel (one warp per tile boundary, all searched at once)
// instead of from two warps of every merge CTA, whose six other warps wait at
// the barrier for that dependent chain of global loads (28 % of the stall
// samples of the top level, profiles/r2n_merge_top_source.txt); the small
// levels keep the single launch.  RFR_SPLIT_MIN_TILES overrides (0: every
// level; RFR_SPLIT_KERNEL=1 is the same).
unsigned int split_kernel_min_tiles() {
  static long v = -2;
  if (v == -2) {
    const char* e = getenv("RFR_SPLIT_MIN_TILES");
    v = e ? atol(e) : (getenv("RFR_SPLIT_KERNEL") ? 0 : 1024);
    if (v < 0) v = 0;
  }
  return (unsigned int)(v > 0xffffffffL ? 0xffffffffL : v);
}

int lists_launch_count(const JoinPlan& P) {
  int maxbits = 0;
  for (int i = 0; i < 4; i++) maxbits = P.list[i].bits > maxbits ? P.list[i].bits : maxbits;
  int n = 1;  // the base kernel
  for (int k = kBaseBits; k < maxbits; k++) {
    const unsigned int blocks = (unsigned int)(((2ull << k) + kMergeTile - 1) / kMergeTile);
    n += blocks >= split_kernel_min_tiles() ? 2 : 1;
  }
  return n;
}

cudaError_t launch_lists(const uint64_t* d_keys, const JoinPlan& P, ListBufs buf0, ListBufs buf1,
                         uint32_t* d_rot, ListHist H, cudaStream_t s) {
  static uint64_t attr_done = 0;
  cudaError_t e = raise_smem_limit(lists_base_kernel, sizeof(BaseSmem), attr_done);
  if (e != cudaSuccess) return e;
  lists_base_kernel<<<4, 1024, sizeof(BaseSmem), s>>>(d_keys, P, buf0, d_rot);
  int maxbits = 0;
  for (int i = 0; i < 4; i++) maxbits = P.list[i].bits > maxbits ? P.list[i].bits : maxbits;
  // RFR_MERGE_TMA=0/1: staging by loads + shared stores, or by TMA bulk copies
  static int tma = -1;
  if (tma < 0) {
    const char* e = getenv("RFR_MERGE_TMA");
    tma = e ? atoi(e) : 0;  // measured slower: off by default
  }
  const unsigned int split_min = split_kernel_min_tiles();
  for (int k = kBaseBits; k < maxbits; k++) {
    const int parity = (k - kBaseBits) & 1;
    const uint64_t outputs = 2ull << k;
    const unsigned int blocks = (unsigned int)((outputs + kMergeTile - 1) / kMergeTile);
    if (blocks >= split_min) {
      cudaError_t le = launch_pdl(lists_split_kernel, dim3((blocks + 1 + 7) / 8, 4), dim3(256), 0, s, d_keys, P,
                                  k, parity ? buf1 : buf0, (const uint32_t*)d_rot, H);
      if (le == cudaSuccess)
        le = launch_pdl(lists_merge_kernel<0>, dim3(blocks, 4), dim3(kMergeThreads), 0, s, d_keys, P, k,
                        parity ? buf1 : buf0, parity ? buf0 : buf1, d_rot, H);
      if (le != cudaSuccess) return le;
    } else if (tma) {
      lists_merge_kernel<2><<<dim3(blocks, 4), kMergeThreads, 0, s>>>(
          d_keys, P, k, parity ? buf1 : buf0, parity ? buf0 : buf1, d_rot, H);
    } else {
      const cudaError_t le = launch_pdl(lists_merge_kernel<1>, dim3(blocks, 4), dim3(kMergeThreads), 0, s,
                                        d_keys, P, k, parity ? buf1 : buf0, parity ? buf0 : buf1, d_rot, H);
      if (le != cudaSuccess) return le;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_join_starts(const JoinPlan& P, const ListBufs& fin, uint64_t b0, uint64_t b1,
                               int nck, int ctas, uint32_t* d_rots, uint32_t* d_starts, cudaStream_t s) {
  const uint64_t mot = (1ull << P.list[0].bits) + (1ull << P.list[2].bits);
  const uint64_t warps = mot * (1ull + (uint64_t)nck * (uint64_t)ctas);
  const cudaError_t e = launch_pdl(join_starts_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0, s, P,
                                   (const uint64_t*)fin.k[0], (const uint64_t*)fin.k[1],
                                   (const uint64_t*)fin.k[2], (const uint64_t*)fin.k[3], b0, b1, nck, ctas,
                                   d_rots, d_starts);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_join(const JoinPlan& P, const ListBufs& fin, uint64_t* d_out,
                        unsigned long long cap, DevCounters* d_ctr, int grid, cudaStream_t s,
                        const uint32_t* d_rots, const uint32_t* d_starts, unsigned long long stop_epoch) {
  static uint64_t attr_done = 0;
  cudaError_t e = raise_smem_limit(join_kernel, sizeof(JoinSmem), attr_done);
  if (e != cudaSuccess) return e;
  JoinArgs a;
  a.P = P;
  for (int i = 0; i < 4; i++) a.key[i] = fin.k[i];
  a.out = d_out;
  a.cap = cap;
  a.ctr = d_ctr;
  a.rots = d_rots;
  a.starts = d_starts;
  a.early = stop_epoch;
  a.trace_stop = getenv("RFR_STOP_TRACE") != nullptr && grid <= 1024;
  if (a.trace_stop) {
    void* sym = nullptr;
    cudaGetSymbolAddress(&sym, g_cta_stop);
    cudaMemsetAsync(sym, 0, sizeof(g_cta_stop), s);
  }
  static unsigned long long* dbg = nullptr;
  a.dbg = nullptr;
  if (getenv("RFR_TRACE")) {
    if (!dbg) cudaMalloc(&dbg, 256 * sizeof(unsigned long long));
    cudaMemsetAsync(dbg, 0, 256 * sizeof(unsigned long long), s);
    a.dbg = dbg;
  }
  // lane groups: about twice the expected run of one outer in one bucket
  // Lanes per outer window: a lane group of 2 * lambda lanes for short runs
  // (lambda = expected records per outer per bucket); for lambda >= 32 the
  // warp-wide run pass with ceil((lambda + 2 sqrt(lambda) + 8) / 32) chunks
  // (encoded as gs = 32 * chunks > 32).
  auto gs_for = [&](int inner_bits) {
    int run_log = inner_bits - P.r;  // log2 expected records per outer per bucket
    if (run_log >= 5) {
      const double lam = std::ldexp(1.0, run_log);
      int nch = (int)std::ceil((lam + 2.0 * std::sqrt(lam) + 8.0) / 32.0);
      if (nch > kMaxCh) nch = kMaxCh;  // longer runs continue in continue_pass
      return 32 * nch;
    }
    int g = run_log + 1;
    g = g < 3 ? 3 : (g > 5 ? 5 : g);
    return 1 << g;
  };
  const int gsA = gs_for(P.list[1].bits), gsB = gs_for(P.list[3].bits);
  join_kernel<<<grid, kJoinThreads, sizeof(JoinSmem), s>>>(a, gsA, gsB);
  if (a.dbg) {
    unsigned long long h[256];
    cudaMemcpyAsync(h, a.dbg, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "[rfr trace] gsA=%d gsB=%d r=%d MoA=%d MiA=%d MoB=%d MiB=%d init=%llu\n", gsA, gsB,
            P.r, 1 << P.list[0].bits, 1 << P.list[1].bits, 1 << P.list[2].bits,
            1 << P.list[3].bits, h[1] - h[0]);
    for (int side = 0; side < 2; side++) {
      fprintf(stderr, "[rfr trace] %s marks (cycles between marks; p = before processing):", side ? "B" : "A");
      const unsigned long long* t = h + 128 + side * 64;
      for (int k = 0; k + 1 < 64 && t[k + 1]; k++)
        fprintf(stderr, " %llu%s", (t[k + 1] & ~(1ull << 63)) - (t[k] & ~(1ull << 63)),
                (t[k + 1] >> 63) ? "p" : "");
      fprintf(stderr, "\n");
    }
    for (int b = 0; b < 6; b++) {  // marks: start, A, index, B run, B cont, B end, barrier
      const unsigned long long* q = h + 1 + b * 7;
      if (!q[6]) break;
      fprintf(stderr,
              "[rfr trace] bucket %d: A %llu index %llu B-run %llu B-cont %llu B-tail %llu barrier %llu\n",
              b, q[1] - q[0], q[2] - q[1], q[3] - q[2], q[4] - q[3], q[5] - q[4], q[6] - q[5]);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_recheck(const double* d_rho, const uint64_t* d_in, const unsigned long long* d_in_count,
                           unsigned long long cap_in, double eps, uint64_t* d_out,
                           unsigned long long cap_out, DevCounters* d_ctr, int nsm, cudaStream_t s) {
  recheck_kernel<<<nsm * 4, 256, 0, s>>>(d_rho, d_in, d_in_count, cap_in, eps, d_out, cap_out, d_ctr);
  return cudaGetLastError();
}

cudaError_t launch_keyfilter(const uint64_t* d_keys2, int n, const uint64_t* d_in,
                             const unsigned long long* d_in_count, unsigned long long cap_in,
                             uint64_t lo2, uint64_t width2, uint64_t* d_out,
                             unsigned long long cap_out, DevCounters* d_ctr, int nsm, cudaStream_t s,
                             const unsigned long long* d_begin) {
  cudaError_t e = launch_pdl(keyfilter_kernel, dim3(nsm * 4), dim3(256), 0, s, d_keys2, n, d_in, d_in_count,
                             cap_in, lo2, width2, d_out, cap_out, d_ctr, d_begin);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ----------------------------------------------------- exhaustive search
// Small searches (n <= kExhaustiveMaxN, one shard): every folded pattern t <
// 2^(n-1) in Gray-code order, one key added or removed per step, the window
// test (sum - lo) mod 2^64 <= width on each -- the same hit set as the
// quarter-list join (same space, same test), in one launch instead of the
// list build, the start search and a join that would keep only a few CTAs
// busy.  Thread T walks patterns [T 2^b, (T+1) 2^b).
__global__ void __launch_bounds__(256) exhaustive_kernel(const uint64_t* __restrict__ keys, int n,
                                                         uint64_t lo, uint64_t width, int b,
                                                         uint64_t* __restrict__ out,
                                                         unsigned long long cap, DevCounters* ctr) {
  __shared__ uint64_t sk[64];
  for (int i = threadIdx.x; i < n; i += blockDim.x) sk[i] = keys[i];
  __syncthreads();
  const int m = n - 1;
  const uint64_t T = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (T == 0) atomicAdd(&ctr->queries, 1ull << m);  // patterns tested (stats)
  if ((T << b) >> m) return;  // past 2^m patterns
  const uint64_t i0 = T << b;
  // sum is kept shifted by -lo: pattern g is a hit iff sum <= width
  uint64_t g = i0 ^ (i0 >> 1), sum = 0ull - lo;
  for (uint64_t u = g; u; u &= u - 1) sum += sk[__ffsll((long long)u) - 1];
  auto hit = [&](uint64_t pat, uint64_t sm) {
    if (sm <= width) {
      const unsigned long long k = atomicAdd(&ctr->out_count, 1ull);
      if (k < cap) out[k] = pat;
    }
  };
  // toggle bit j of g and move sum by +-key (the key's sign follows the bit)
  auto step = [&](int j, uint64_t key) {
    g ^= 1ull << j;
    sum += ((g >> j) & 1ull) ? key : 0ull - key;
    hit(g, sum);
  };
  if (b < 4) {  // tiny spaces: plain Gray-code walk
    hit(g, sum);
    for (uint32_t i = 1; i < (1u << b); i++) step(__ffs(i) - 1, sk[__ffs(i) - 1]);
    return;
  }
  // b >= 4: blocks of 16 patterns.  Within a block the toggled bits are fixed
  // (0 1 0 2 0 1 0 3 0 1 0 2 0 1 0) and each bit's toggles alternate in sign,
  // so the block runs on 8 signed deltas set up at its start: one 64-bit add
  // and one compare per pattern, no branch; a block with a hit is replayed
  // pattern by pattern (rare).
  const uint64_t k0 = sk[0], k1 = sk[1], k2 = sk[2], k3 = sk[3];
  const uint32_t nblk = 1u << (b - 4);
  for (uint32_t blk = 0;;) {
    const uint64_t p0 = (g & 1ull) ? 0ull - k0 : k0, m0 = 0ull - p0;
    const uint64_t p1 = (g & 2ull) ? 0ull - k1 : k1, m1 = 0ull - p1;
    const uint64_t p2 = (g & 4ull) ? 0ull - k2 : k2, m2 = 0ull - p2;
    const uint64_t p3 = (g & 8ull) ? 0ull - k3 : k3;
    uint64_t x = sum;
    bool any = x <= width;
    x += p0; any |= x <= width;  // bit 0
    x += p1; any |= x <= width;  // bit 1
    x += m0; any |= x <= width;  // bit 0
    x += p2; any |= x <= width;  // bit 2
    x += p0; any |= x <= width;
    x += m1; any |= x <= width;
    x += m0; any |= x <= width;
    x += p3; any |= x <= width;  // bit 3
    x += p0; any |= x <= width;
    x += p1; any |= x <= width;
    x += m0; any |= x <= width;
    x += m2; any |= x <= width;
    x += p0; any |= x <= width;
    x += m1; any |= x <= width;
    x += m0; any |= x <= width;
    if (any) {  // replay the block from its start, emitting each hit
      uint64_t gg = g, ss = sum;
      hit(gg, ss);
      for (uint32_t i = 1; i < 16; i++) {
        const int j = __ffs(i) - 1;
        const uint64_t key = j == 0 ? k0 : j == 1 ? k1 : j == 2 ? k2 : k3;
        gg ^= 1ull << j;
        ss += ((gg >> j) & 1ull) ? key : 0ull - key;
        hit(gg, ss);
      }
    }
    g ^= 8ull;  // the block's last pattern differs from its first in bit 3
    sum = x;
    if (++blk == nblk) break;
    const int j = 4 + __ffs(blk) - 1;  // first pattern of the next block
    const uint64_t key = sk[j];
    g ^= 1ull << j;
    sum += ((g >> j) & 1ull) ? key : 0ull - key;
  }
}
cudaError_t launch_exhaustive(const uint64_t* d_keys, int n, uint64_t lo, uint64_t width,
                              uint64_t* d_out, unsigned long long cap, DevCounters* d_ctr,
                              cudaStream_t s) {
  const int m = n - 1;
  // ~2^18 threads of 2^b patterns each; b >= 4 when the space allows (16-pattern blocks)
  int b = m > 18 ? m - 18 : 0;
  if (b < 4) b = m < 4 ? m : 4;
  const uint64_t threads = 1ull << (m - b);
  exhaustive_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(d_keys, n, lo, width, b, d_out, cap,
                                                                     d_ctr);
  return cudaGetLastError();
}

// ------------------------------------------------------- table search
// Small searches (n <= kTableMaxN, one shard; every piece search after an
// early stop): a one-sided meet in the middle inside each CTA.  The 2^b subset
// sums of the low b keys are built and bitonic-sorted in shared memory; each
// thread walks a range of high-bit patterns in Gray-code order (one key added
// or removed per step) and finds the low sums that complete its partial sum
// into the window by one binary search of the table: b steps per 2^b
// patterns instead of one add and one compare per pattern (the Gray-code
// exhaustive_kernel, kept as the independent checker of RFR_FORCE_EXHAUSTIVE).
constexpr int kTableMaxBits = 12;
// Where a small search's hits go: the raw hit list (RawEmit), or -- for the
// pieces searched behind an early stop -- straight through the Tr3 window
// into parent patterns (PieceEmit).
struct RawEmit {
  DevCounters* ctr;
  uint64_t* out;
  unsigned long long cap;
  __device__ __forceinline__ void operator()(uint64_t pat) const {
    const unsigned long long k = atomicAdd(&ctr->out_count, 1ull);
    if (k < cap) out[k] = pat;
  }
};
struct PieceEmit {
  DevCounters* ctr;     // out_count: raw hits, post_count: survivors (both pieces)
  const uint64_t* sk2;  // the piece's Tr3 keys (shared memory)
  uint64_t mask;        // the piece's entities as parent bits
  uint64_t lo2, width2;
  uint64_t* post;
  unsigned long long cap;
  __device__ __forceinline__ void operator()(uint64_t u) const {
    atomicAdd(&ctr->out_count, 1ull);
    uint64_t sum = 0, v = 0, mm = mask;
    for (int j = 0; u; j++, u >>= 1, mm &= mm - 1)
      if (u & 1ull) {
        sum += sk2[j];
        v |= mm & (0ull - mm);
      }
    if (sum - lo2 <= width2) {
      const unsigned long long k = atomicAdd(&ctr->post_count, 1ull);
      if (k < cap) post[k] = v;
    }
  }
};

template <class Emit>
__device__ __forceinline__ void table_search_body(const uint64_t* __restrict__ keys, int n, uint64_t lo,
                                                  uint64_t width, int b, int g, DevCounters* ctr,
                                                  unsigned blk, const Emit& emit_pat) {
  extern __shared__ __align__(16) unsigned char tsm[];
  uint64_t* tk = reinterpret_cast<uint64_t*>(tsm);                     // sorted low sums
  uint16_t* ti = reinterpret_cast<uint16_t*>(tsm + (8u << b));         // their low patterns
  __shared__ uint64_t sk[64];
  const int tid = threadIdx.x;
  {  // a CTA past the 2^h high patterns has nothing to do (fixed-size grids)
    const int h0 = n - 1 - b;
    if (h0 >= 0 && blk != 0 && (((uint64_t)blk * blockDim.x) << g) >> h0) return;
  }
  for (int i = tid; i < n; i += blockDim.x) sk[i] = keys[i];
  __syncthreads();
  const uint32_t nt = 1u << b;
  if (nt == blockDim.x) {
    // one entry per thread: bitonic sort in registers, the partner of the
    // stages with j < 32 read by a warp shuffle, only the j >= 32 stages
    // through shared memory (6 barriers for b = 8 instead of 36)
    const uint32_t i = tid;
    uint64_t x = 0;
    for (uint32_t u = i; u; u &= u - 1) x += sk[__ffs(u) - 1];
    uint32_t xi = i;
    for (uint32_t kk = 2; kk <= nt; kk <<= 1) {
      for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
        uint64_t y;
        uint32_t yi;
        if (jj >= 32) {
          __syncthreads();
          tk[i] = x;
          ti[i] = (uint16_t)xi;
          __syncthreads();
          y = tk[i ^ jj];
          yi = ti[i ^ jj];
        } else {
          y = __shfl_xor_sync(0xffffffffu, x, jj);
          yi = __shfl_xor_sync(0xffffffffu, xi, jj);
        }
        // the lower index of an ascending pair keeps the minimum
        const bool lower = (i & jj) == 0, up = (i & kk) == 0;
        const bool take = lower == up ? (y < x) : (y > x);
        if (take) {
          x = y;
          xi = yi;
        }
      }
    }
    __syncthreads();
    tk[i] = x;
    ti[i] = (uint16_t)xi;
    __syncthreads();
  } else {
  for (uint32_t i = tid; i < nt; i += blockDim.x) {
    uint64_t s = 0;
    for (uint32_t u = i; u; u &= u - 1) s += sk[__ffs(u) - 1];
    tk[i] = s;
    ti[i] = (uint16_t)i;
  }
  __syncthreads();
  // bitonic sort of (tk, ti) by tk
  for (uint32_t kk = 2; kk <= nt; kk <<= 1) {
    for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
      for (uint32_t i = tid; i < nt; i += blockDim.x) {
        const uint32_t p = i ^ jj;
        if (p > i) {
          const bool up = (i & kk) == 0;
          const uint64_t a = tk[i], c = tk[p];
          if ((a > c) == up) {
            tk[i] = c;
            tk[p] = a;
            const uint16_t t = ti[i];
            ti[i] = ti[p];
            ti[p] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  }
  const int m = n - 1, h = m - b;
  const uint64_t T = (uint64_t)blk * blockDim.x + tid;
  if (T == 0) atomicAdd(&ctr->queries, 1ull << m);  // patterns tested (stats)
  if (h < 0 || (T << g) >> h) return;  // past 2^h high patterns
  const uint64_t i0 = T << g;
  uint64_t gh = i0 ^ (i0 >> 1), S = 0;  // Gray high pattern and its key sum
  for (uint64_t u = gh; u; u &= u - 1) S += sk[b + __ffsll((long long)u) - 1];
  const uint64_t steps = 1ull << g;
  for (uint64_t st = 0;; st++) {
    // low sums D with (S + D - lo) mod 2^64 <= width: D in [a, a + width] (mod 2^64)
    const uint64_t a = lo - S;
    uint32_t l = 0, r = nt;  // first D >= a
    while (l < r) {
      const uint32_t mid = (l + r) >> 1;
      if (tk[mid] < a) l = mid + 1;
      else r = mid;
    }
    auto emit = [&](uint32_t i) { emit_pat((gh << b) | ti[i]); };
    for (uint32_t i = l; i < nt && tk[i] - a <= width; i++) emit(i);
    if (a + width < a)  // the window wraps past 2^64: its head is at the table's start
      for (uint32_t i = 0; i < l && tk[i] <= a + width; i++) emit(i);
    if (st + 1 == steps) break;
    const int j = __ffsll((long long)(i0 + st + 1)) - 1;  // Gray step: toggle bit j
    gh ^= 1ull << j;
    S += ((gh >> j) & 1ull) ? sk[b + j] : 0ull - sk[b + j];
  }
}

__global__ void __launch_bounds__(256) table_search_kernel(const uint64_t* __restrict__ keys, int n,
                                                           uint64_t lo, uint64_t width, int b, int g,
                                                           uint64_t* __restrict__ out,
                                                           unsigned long long cap, DevCounters* ctr) {
  pdl_wait();  // programmatic launch: the previous kernel is complete
  pdl_trigger();
  table_search_body(keys, n, lo, width, b, g, ctr, blockIdx.x, RawEmit{ctr, out, cap});
}

// table bits and threads of a small search of n entities (<= 2^16 threads,
// 2^g high patterns each)
__host__ __device__ inline int table_bits(int m) { return m <= 30 ? 8 : (m <= 33 ? 10 : kTableMaxBits); }

cudaError_t launch_table_search(const uint64_t* d_keys, int n, uint64_t lo, uint64_t width,
                                uint64_t* d_out, unsigned long long cap, DevCounters* d_ctr,
                                cudaStream_t s) {
  const int m = n - 1;
  // table bits: the per-CTA bitonic sort (latency-bound, ~b^2/2 barrier
  // stages) against 2^(m-b) binary searches of b steps; RFR_TABLE_BITS (A/B)
  static int forced_b = -1;
  if (forced_b < 0) {
    const char* e = getenv("RFR_TABLE_BITS");
    forced_b = e ? atoi(e) : 0;
  }
  int b = forced_b > 0 ? forced_b : table_bits(m);
  if (b > m) b = m;
  if (b > kTableMaxBits) b = kTableMaxBits;
  const int h = m - b;
  const int g = h > 16 ? h - 16 : 0;  // <= 2^16 threads, 2^g high patterns each
  const uint64_t threads = 1ull << (h - g);
  const size_t smem = (size_t)10 << b;
  static uint64_t attr_done = 0;
  cudaError_t e = raise_smem_limit(table_search_kernel, (size_t)10 << kTableMaxBits, attr_done);
  if (e != cudaSuccess) return e;
  e = launch_pdl(table_search_kernel, dim3((unsigned)((threads + 255) / 256)), dim3(256), smem, s, d_keys, n, lo,
                 width, b, g, d_out, cap, d_ctr);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Patterns of a piece's search (bit j = the j-th set bit of mask) rewritten
// as patterns of the parent's search (rfr_search_verify after an early stop).
__global__ void deposit_kernel(uint64_t* __restrict__ pats, const unsigned long long* __restrict__ count,
                               unsigned long long cap, uint64_t mask) {
  pdl_wait();  // programmatic launch: the previous kernel is complete
  pdl_trigger();
  unsigned long long m = *count;
  if (m > cap) m = cap;
  for (unsigned long long k = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; k < m;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    uint64_t u = pats[k], v = 0;
    for (uint64_t mm = mask; mm && u; mm &= mm - 1, u >>= 1)
      if (u & 1ull) v |= mm & (0ull - mm);
    pats[k] = v;
  }
}
cudaError_t launch_deposit(uint64_t* d_pats, const unsigned long long* d_count, unsigned long long cap,
                           uint64_t mask, int nsm, cudaStream_t s) {
  cudaError_t e = launch_pdl(deposit_kernel, dim3(nsm), dim3(256), 0, s, d_pats, d_count, cap, mask);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// The results of a search + verification straight into pinned host memory
// (mapped: the host pointers are device pointers under UVA): the counters
// and the first min(post_count, rows) rows -- one launch instead of five
// small device-to-host copies, each with its own ~3 us of setup and gap.
__global__ void collect_kernel(CollectArgs C) {
  pdl_wait();  // programmatic launch: the previous kernel is complete
  pdl_trigger();
  const unsigned long long cnt = C.ctr->post_count;
  const unsigned rows = (unsigned)(cnt < C.rows ? cnt : C.rows);
  const int t = threadIdx.x;
  if (t < (int)(sizeof(DevCounters) / 8))
    ((unsigned long long*)C.h_ctr)[t] = ((const unsigned long long*)C.ctr)[t];
  for (unsigned k = t; k < rows; k += blockDim.x) {
    C.h_pats[k] = C.pats[k];
    C.h_verdict[k] = C.verdict[k];
    C.h_side[k] = C.side[k];
  }
  const unsigned nco = rows * (unsigned)C.stride;
  for (unsigned k = t; k < nco; k += blockDim.x) C.h_coeffs[k] = C.coeffs[k];
  for (int k = t; k < C.clear_words; k += blockDim.x) C.clear[k] = 0ull;
}
cudaError_t launch_collect(const CollectArgs& C, cudaStream_t s) {
  cudaError_t e = launch_pdl(collect_kernel, dim3(1), dim3(256), 0, s, C);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ------------------------------------------- pieces after an early stop
// The two pieces of the verified factor searched right behind the main
// search on the same stream, with no host round trip, in one grid (blockIdx.y
// = piece): every CTA takes the first PASS row of the main search (the
// pattern the host would pick), splits the entities into t and its
// complement, compacts its piece's keys into shared memory and runs the
// table search, whose hits go through the Tr3 window straight into parent
// patterns (PieceEmit); one verification and one collection follow.
// Inactive (no stop, no PASS, a piece above kExhaustiveMaxN, more rows than
// the caller takes): every CTA returns at once.  CTA (0, 0) publishes its
// plan (PieceDesc) to pinned memory, and the host compares its t with its own
// before using the rows.  The piece counters were cleared by the main
// search's collection (CollectArgs.clear).
__global__ void __launch_bounds__(256) piece_kernel(const PiecePlanArgs a, uint64_t lo, uint64_t width,
                                                    uint64_t lo2, uint64_t width2,
                                                    unsigned long long post_cap) {
  pdl_wait();  // programmatic launch: the previous kernel is complete
  pdl_trigger();
  __shared__ unsigned long long s_t;
  __shared__ int s_act;
  __shared__ uint64_t pk[64], pk2[64];
  const int tid = threadIdx.x, pi = blockIdx.y;
  const uint64_t full = a.n >= 64 ? ~0ull : ((1ull << a.n) - 1ull);
  if (tid == 0) {
    const DevCounters& c = *a.ctr;
    int act = 0;
    unsigned long long t = 0;
    if (c.buckets < a.planned && c.out_count <= a.raw_cap && c.post_count <= a.rows_cap) {
      for (unsigned long long k = 0; k < c.post_count; k++) {
        if (a.verdict[k] != RFR_V_PASS) continue;
        const uint64_t sp = a.pats[k] & full;
        t = a.side[k] ? (~sp & full) : sp;
        act = __popcll(t) <= kExhaustiveMaxN && __popcll(~t & full) <= kExhaustiveMaxN;
        break;
      }
    }
    s_t = t;
    s_act = act;
    if (blockIdx.x == 0 && pi == 0) {
      PieceDesc d;
      d.t = t;
      d.mask[0] = t;
      d.mask[1] = ~t & full;
      d.ns[0] = __popcll(d.mask[0]);
      d.ns[1] = __popcll(d.mask[1]);
      d.active = act;
      d.pad = 0;
      *a.h_desc = d;
    }
  }
  __syncthreads();
  if (!s_act) return;
  const uint64_t mask = pi ? (~s_t & full) : s_t;
  const int n = __popcll(mask);
  if (n < 2) return;  // one linear or quadratic entity: irreducible
  for (int i = tid; i < a.n; i += blockDim.x)  // compact the piece's keys
    if ((mask >> i) & 1ull) {
      const int j = __popcll(mask & ((1ull << i) - 1ull));
      pk[j] = a.keys[i];
      pk2[j] = a.keys2[i];
    }
  __syncthreads();
  const int m = n - 1;
  int b = table_bits(m);
  if (b > m) b = m;
  const int h = m - b;
  const int g = h > 16 ? h - 16 : 0;
  table_search_body(pk, n, lo, width, b, g, a.pctr, blockIdx.x,
                    PieceEmit{a.pctr, pk2, mask, lo2, width2, a.ppost, post_cap});
}

cudaError_t launch_pieces(const PiecePlanArgs& a, uint64_t lo, uint64_t width, uint64_t lo2, uint64_t width2,
                          unsigned long long post_cap, const VerifyArgs& V, const CollectArgs& C,
                          cudaStream_t s) {
  static uint64_t attr_done = 0;
  cudaError_t e = raise_smem_limit(piece_kernel, (size_t)10 << kTableMaxBits, attr_done);
  if (e != cudaSuccess) return e;
  // <= 2^16 threads per piece (n <= kExhaustiveMaxN: b = 8, h <= 22, g = h - 16)
  e = launch_pdl(piece_kernel, dim3(256, 2), dim3(256), (size_t)10 << 8, s, a, lo, width, lo2, width2,
                 post_cap);
  if (e != cudaSuccess) return e;
  if ((e = launch_verify(V, s)) != cudaSuccess) return e;
  return launch_collect(C, s);
}

// ---------------------------------------------------------- early exit
// One warp beside the running join (its own stream, a CTA slot the join
// leaves free): takes the raw hits in emission order as they appear, turns
// each into its pattern, applies the Tr3 window and verifies survivors in
// place; a PASS raises DevCounters.found and the join's CTAs stop at their
// next bucket boundary.  It publishes how far it got (raw_done, post_done)
// and leaves as soon as every join CTA has finished (or after a time limit):
// the batch kernels then finish whatever it did not reach, so a flood of
// hits (Swinnerton-Dyer f6) costs it nothing.  Raw slots hold kUnsetHit until the
// join's store lands (the count is bumped first).
constexpr uint64_t kUnsetHit = ~0ull;

struct PollArgs {
  PatArgs pa;
  uint64_t* out;
  unsigned long long raw_cap;
  const uint64_t* keys2;
  int n;
  uint64_t lo2, width2;
  uint64_t* post;
  unsigned long long post_cap;
  VerifyArgs V;  // V.pats = post, V.m = verification rows
  DevCounters* ctr;
  unsigned long long join_ctas;
  long long max_cycles;
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(32) early_exit_poller_kernel(const __grid_constant__ PollArgs a) {
  __shared__ WarpBuf B;
  __shared__ ProfSmem PS;
  __shared__ uint64_t sk[64];
  const int lane = threadIdx.x;
  stage_profile_smem(PS, a.V, lane, 32);
  for (int i = lane; i < a.n; i += 32) sk[i] = a.keys2[i];
  __syncwarp();
  const long long t0 = clock64();
  unsigned long long done = 0;
  bool spec = false;  // a speculative stop was raised
  while (true) {
    // once the join is over the batch kernels take the rest (a flood of hits
    // would keep one warp busy for seconds)
    if (ld_acquire_u64(&a.ctr->ctas_done) >= a.join_ctas) break;
    unsigned long long cnt = ld_acquire_u64(&a.ctr->out_count);
    if (cnt > a.raw_cap) cnt = a.raw_cap;
    if (done < cnt) {
      // the slot is written right after the count was bumped
      uint64_t v = kUnsetHit;
      while ((v = ld_acquire_u64((const unsigned long long*)a.out + done)) == kUnsetHit &&
             clock64() - t0 < a.max_cycles) {
      }
      if (v == kUnsetHit) break;  // time limit: the batch kernels take over
      const unsigned long long t_seen = rfr_globaltimer();
      // pattern: lanes 0-3 walk the four quarter lists (index_to_pattern_kernel)
      uint64_t part = 0;
      if (lane < 4) {
        const ListSpec L = pick_list(a.pa.P, lane);
        const uint32_t idx = (uint32_t)((v >> L.pat_shift) & ((1ull << L.bits) - 1ull));
        part = (uint64_t)list_pattern(a.pa, lane, idx) << L.pat_shift;
      }
      part |= __shfl_xor_sync(0xffffffffu, part, 1);
      part |= __shfl_xor_sync(0xffffffffu, part, 2);
      const uint64_t t = __shfl_sync(0xffffffffu, part, 0);
      // Tr3 window (keyfilter_kernel)
      uint64_t s3 = 0;
      for (int i = lane; i < a.n; i += 32) s3 += ((t >> i) & 1ull) ? sk[i] : 0ull;
#pragma unroll
      for (int o = 16; o; o >>= 1) s3 += __shfl_xor_sync(0xffffffffu, s3, o);
      if (lane == 0) a.out[done] = t;
      if (s3 - a.lo2 <= a.width2) {
        unsigned long long k = 0;
        if (lane == 0) k = atomicAdd(&a.ctr->post_count, 1ull);
        k = __shfl_sync(0xffffffffu, k, 0);
        // Speculative stop: a hit inside both key windows is a factor but for
        // ~2^(n-1) (2T+1)(2T3+1) / 2^128 false hits of random keys (~1e-17
        // at d = 100), so the join is stopped now and the hit verified after:
        // verifying first left the join running ~0.6 ms past the hit (one
        // warp verifying a degree-50 candidate beside 16 busy join warps).
        // Only while hits are rare (the first non-empty survivor among the
        // first 16 raw hits):
        // structured inputs (Swinnerton-Dyer) flood the windows with
        // non-factors and keep verify-then-stop.  A stop whose hit then
        // fails verification leaves the search incomplete without a PASS,
        // and the caller searches the whole space (verify.py).
        const bool spec_now = !spec && t != 0 && done < 16 && a.V.found;  // t = 0: the empty pattern
        if (spec_now && lane == 0) {
          if (a.V.t_found) atomicCAS(a.V.t_found, 0ull, rfr_globaltimer());
          a.ctr->t_hit = t_seen;
          atomicExch(a.V.found, a.V.found_value);
          for (int i = 0; i < a.V.npeers; i++) *(volatile unsigned long long*)a.V.peer_found[i] = a.V.found_value;
          if (a.V.npeers) __threadfence_system();
        }
        spec |= t != 0;
        if (k < a.post_cap && lane == 0) a.post[k] = t;
        __syncwarp();
        if (k < a.post_cap && (long long)k < a.V.m) {
          if (spec_now) {  // the stopping hit: integral + monic, exact division on the host
            VerifyArgs V = a.V;
            V.skip_division = 1;
            verify_one(V, PS, B, (long long)k, lane);
          } else {
            verify_one(a.V, PS, B, (long long)k, lane);
          }
        }
        __syncwarp();
        if (lane == 0 && t != 0 && a.ctr->t_verified == 0 && a.ctr->t_found) a.ctr->t_verified = rfr_globaltimer();
      }
      done++;
      if (lane == 0) {
        a.ctr->raw_done = done;
        a.ctr->post_done = *(volatile unsigned long long*)&a.ctr->post_count;
      }
      continue;
    }
    if (clock64() - t0 > a.max_cycles) break;
    __nanosleep(1000);
  }
  if (lane == 0) a.ctr->t_poller_exit = rfr_globaltimer();
}

cudaError_t launch_early_exit_poller(const JoinPlan& P, const ListBufs& base, const ListHist& hist,
                                     const uint32_t* d_rot, uint64_t* d_out, unsigned long long raw_cap,
                                     const uint64_t* d_keys2, int n, uint64_t lo2, uint64_t width2,
                                     uint64_t* d_post, unsigned long long post_cap, const VerifyArgs& V,
                                     DevCounters* d_ctr, int join_ctas, cudaStream_t s) {
  PollArgs a;
  a.pa.P = P;
  for (int i = 0; i < 4; i++) a.pa.pat[i] = base.p[i];
  a.pa.hist = hist;
  a.pa.rot = d_rot;
  a.out = d_out;
  a.raw_cap = raw_cap;
  a.keys2 = d_keys2;
  a.n = n;
  a.lo2 = lo2;
  a.width2 = width2;
  a.post = d_post;
  a.post_cap = post_cap;
  a.V = V;
  a.ctr = d_ctr;
  a.join_ctas = (unsigned long long)join_ctas;
  a.max_cycles = 4000000000ll;  // ~2 s at 2 GHz: never hold the device if the join cannot start
  early_exit_poller_kernel<<<1, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_rho_keys(const double* d_rho, int n, uint64_t* d_keys, cudaStream_t s) {
  rho_keys_kernel<<<1, 64, 0, s>>>(d_rho, n, d_keys);
  return cudaGetLastError();
}

}  // namespace rfr

namespace rfr {
// RFR_STOP_TRACE: the join CTAs that left their bucket loop last after a stop
void dump_stop_trace(unsigned long long t_found, int grid) {
  static unsigned long long h[3 * 1024];
  if (grid > 1024) return;
  cudaMemcpyFromSymbol(h, g_cta_stop, sizeof(unsigned long long) * 3 * grid);
  std::vector<std::pair<long long, int>> v;
  unsigned long long t0 = ~0ull;
  for (int i = 0; i < grid; i++) {
    if (h[3 * i]) v.push_back({(long long)h[3 * i] - (long long)t_found, i});
    if (h[3 * i + 2] && h[3 * i + 2] < t0) t0 = h[3 * i + 2];
  }
  std::sort(v.begin(), v.end());
  fprintf(stderr, "[rfr stop] %zu CTAs stopped; found at +%.1f us after the first CTA start; median %.1f us after found\n",
          v.size(), ((long long)t_found - (long long)t0) * 1e-3, v.empty() ? 0.0 : v[v.size() / 2].first * 1e-3);
  for (size_t k = 0; k < v.size(); k += (v.size() > 8 ? v.size() / 8 : 1)) {
    const int i = v[k].second;
    fprintf(stderr, "[rfr stop]   cta %4d sm %3llu buckets %6llu start +%.1f us stop +%.1f us after found\n", i,
            h[3 * i + 1] >> 32, h[3 * i + 1] & 0xffffffffull, ((long long)h[3 * i + 2] - (long long)t0) * 1e-3,
            v[k].first * 1e-3);
  }
}
}  // namespace rfr
