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
//                            (recombine.py:106-123, :148-162) on every hit
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "rfr_common.cuh"
#include "rfr_internal.h"

namespace cg = cooperative_groups;

namespace rfr {

// ---------------------------------------------------------------- lists
__device__ __forceinline__ uint64_t elem_key(const uint64_t* keys, const ListSpec& L, int i) {
  uint64_t k = keys[L.first + i];
  return L.negate ? (0ull - k) : k;
}

// One CTA per list: all 2^b subset sums (b = min(bits, kBaseBits)) of the
// list's first b elements, bitonic-sorted in shared memory.
__global__ void __launch_bounds__(1024) lists_base_kernel(const uint64_t* __restrict__ keys,
                                                          JoinPlan P, ListBufs out) {
  __shared__ uint64_t sk[1 << kBaseBits];
  __shared__ uint32_t sp[1 << kBaseBits];
  const ListSpec L = P.list[blockIdx.x];
  const int b = L.bits < kBaseBits ? L.bits : kBaseBits;
  const int len = 1 << b;
  uint64_t ek[kBaseBits];
  for (int i = 0; i < b; i++) ek[i] = elem_key(keys, L, i);
  for (int p = threadIdx.x; p < len; p += blockDim.x) {
    uint64_t s = 0;
    for (int i = 0; i < b; i++)
      if ((p >> i) & 1) s += ek[i];
    sk[p] = s;
    sp[p] = (uint32_t)p;
  }
  __syncthreads();
  for (int k = 2; k <= len; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < len; i += blockDim.x) {
        int ixj = i ^ j;
        if (ixj > i) {
          bool up = ((i & k) == 0);
          uint64_t a = sk[i], c = sk[ixj];
          if ((a > c) == up) {
            sk[i] = c;
            sk[ixj] = a;
            uint32_t t = sp[i];
            sp[i] = sp[ixj];
            sp[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  uint64_t* ok = out.k[blockIdx.x];
  uint32_t* op = out.p[blockIdx.x];
  for (int p = threadIdx.x; p < len; p += blockDim.x) {
    ok[p] = sk[p];
    op[p] = sp[p];
  }
}

// lower_bound over a sorted uint64 array
__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t* __restrict__ a, uint32_t n,
                                                    uint64_t v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Rotation start of the sequence (x + a[j]) mod 2^64 over a sorted array:
// the first j whose sum wraps, or 0 when none does.
__device__ __forceinline__ uint32_t rotation_start(const uint64_t* __restrict__ a, uint32_t n,
                                                   uint64_t x) {
  if (x == 0) return 0;
  uint32_t j = lower_bound_u64(a, n, 0ull - x);
  return j == n ? 0 : j;
}

// Number of j with (x + a[j]) mod 2^64 < bound, for a sorted array.
__device__ __forceinline__ uint32_t count_below(const uint64_t* __restrict__ a, uint32_t n,
                                                uint64_t x, uint64_t bound) {
  if (bound == 0) return 0;
  uint64_t lo = 0ull - x;          // sums start at key -x
  uint64_t hi = lo + bound;        // exclusive end, mod 2^64
  uint32_t l = lower_bound_u64(a, n, lo);
  if (hi > lo) return lower_bound_u64(a, n, hi) - l;    // no wrap
  return (n - l) + lower_bound_u64(a, n, hi);            // wraps through 2^64
}

// One doubling level for every list that has it: L (2^k sorted sums of the
// list's first k elements) -> merge(L, rotate(L + v_k)), v_k the key of
// element k.  Merge path, ITEMS outputs per thread.
constexpr int kMergeItems = 8;
__global__ void __launch_bounds__(256) lists_merge_kernel(const uint64_t* __restrict__ keys,
                                                          JoinPlan P, int k, ListBufs in,
                                                          ListBufs out) {
  const int li = blockIdx.y;
  const ListSpec L = P.list[li];
  if (L.bits <= k) return;
  const uint32_t n = 1u << k;
  const uint64_t* __restrict__ A = in.k[li];
  const uint32_t* __restrict__ Ap = in.p[li];
  uint64_t* __restrict__ O = out.k[li];
  uint32_t* __restrict__ Op = out.p[li];
  const uint64_t v = elem_key(keys, L, k);
  const uint32_t bit = 1u << k;
  const uint32_t rot = rotation_start(A, n, v);
  const uint32_t mask = n - 1;
  const uint64_t d0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kMergeItems;
  if (d0 >= 2ull * n) return;
  const uint32_t d = (uint32_t)d0;
  // B'[j] = A[(rot + j) & mask] + v is ascending in j
  auto Bk = [&](uint32_t j) { return __ldg(A + ((rot + j) & mask)) + v; };
  uint32_t lo = d > n ? d - n : 0, hi = d < n ? d : n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (__ldg(A + mid) <= Bk(d - 1 - mid)) lo = mid + 1;
    else hi = mid;
  }
  uint32_t i = lo, j = d - lo;
#pragma unroll
  for (int t = 0; t < kMergeItems; t++) {
    bool takeA;
    if (i >= n) takeA = false;
    else if (j >= n) takeA = true;
    else takeA = __ldg(A + i) <= Bk(j);
    if (takeA) {
      O[d + t] = __ldg(A + i);
      Op[d + t] = __ldg(Ap + i);
      i++;
    } else {
      uint32_t jj = (rot + j) & mask;
      O[d + t] = __ldg(A + jj) + v;
      Op[d + t] = __ldg(Ap + jj) | bit;
      j++;
    }
  }
}

// ---------------------------------------------------------------- join
struct JoinArgs {
  JoinPlan P;
  const uint64_t* key[4];
  const uint32_t* pat[4];
  uint64_t* out;
  unsigned long long cap;
  DevCounters* ctr;
  unsigned long long* dbg;  // optional clock64 trace of CTA 0 (RFR_TRACE)
};

#include "rfr_join.cuh"

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

size_t join_smem_bytes() { return sizeof(JoinSmem); }

cudaError_t launch_lists(const uint64_t* d_keys, const JoinPlan& P, ListBufs buf0, ListBufs buf1,
                         cudaStream_t s) {
  lists_base_kernel<<<4, 1024, 0, s>>>(d_keys, P, buf0);
  int maxbits = 0;
  for (int i = 0; i < 4; i++) maxbits = P.list[i].bits > maxbits ? P.list[i].bits : maxbits;
  for (int k = kBaseBits; k < maxbits; k++) {
    const int parity = (k - kBaseBits) & 1;
    const uint64_t outputs = 2ull << k;
    const unsigned int blocks = (unsigned int)((outputs + 256ull * kMergeItems - 1) / (256ull * kMergeItems));
    lists_merge_kernel<<<dim3(blocks, 4), 256, 0, s>>>(d_keys, P, k, parity ? buf1 : buf0,
                                                         parity ? buf0 : buf1);
  }
  return cudaGetLastError();
}

cudaError_t launch_join(const JoinPlan& P, const ListBufs& fin, uint64_t* d_out,
                        unsigned long long cap, DevCounters* d_ctr, int grid, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(join_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(JoinSmem));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  JoinArgs a;
  a.P = P;
  for (int i = 0; i < 4; i++) {
    a.key[i] = fin.k[i];
    a.pat[i] = fin.p[i];
  }
  a.out = d_out;
  a.cap = cap;
  a.ctr = d_ctr;
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
  // warp-wide run pass with ceil((lambda + 3 sqrt(lambda) + 8) / 32) chunks
  // (encoded as gs = 32 * chunks > 32).
  auto gs_for = [&](int inner_bits) {
    int run_log = inner_bits - P.r;  // log2 expected records per outer per bucket
    if (run_log >= 5) {
      const double lam = std::ldexp(1.0, run_log);
      int nch = (int)std::ceil((lam + 3.0 * std::sqrt(lam) + 8.0) / 32.0);
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
    for (int b = 0; b < 6; b++) {  // marks: bucket start, A gen, A index, B pass, end barrier
      const unsigned long long* q = h + 1 + b * 5;
      if (!q[4]) break;
      fprintf(stderr, "[rfr trace] bucket %d: A %llu index %llu B %llu barrier %llu\n", b,
              q[1] - q[0], q[2] - q[1], q[3] - q[2], q[4] - q[3]);
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

cudaError_t launch_rho_keys(const double* d_rho, int n, uint64_t* d_keys, cudaStream_t s) {
  rho_keys_kernel<<<1, 64, 0, s>>>(d_rho, n, d_keys);
  return cudaGetLastError();
}

}  // namespace rfr
