// rfr_verify.cuh -- verification of one candidate by one warp (double-double
// product, integrality bound, trial division modulo three primes).  Shared by
// verify_kernel (rfr_verify.cu, one warp per candidate over a batch) and the
// early-exit poller (rfr_search.cu, candidates verified while the join runs).
// Reference: build_candidate -> trace_test -> round_and_divide,
// pkg/src/polyfactor/verify.py:60-155.
#pragma once
#include <cstdint>

#include "../../include/rfr.h"
#include "rfr_common.cuh"
#include "rfr_internal.h"

namespace rfr {

struct ddv {
  double hi, lo;
};

__device__ __forceinline__ ddv dd_two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}
__device__ __forceinline__ ddv dd_quick(double a, double b) {
  double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ ddv dd_add(ddv a, ddv b) {
  ddv s = dd_two_sum(a.hi, b.hi);
  ddv t = dd_two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = dd_quick(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return dd_quick(s.hi, s.lo);
}
__device__ __forceinline__ ddv dd_mul(ddv a, ddv b) {
  double p = __dmul_rn(a.hi, b.hi);
  double e = __fma_rn(a.hi, b.hi, -p);
  e = __fma_rn(a.hi, b.lo, e);
  e = __fma_rn(a.lo, b.hi, e);
  return dd_quick(p, e);
}
__device__ __forceinline__ ddv dd_neg(ddv a) { return {-a.hi, -a.lo}; }

constexpr int kVerifyWarps = 4;
constexpr int kMaxE = 64;          // smaller side degree <= 64 (n <= 64 roots of p, d <= 128)
constexpr int kMaxD = 128;



struct WarpBuf {
  ddv c[2][kMaxE + 2];
  double mag[2][kMaxE + 2];
  double magp[2][kMaxE + 2];
  uint32_t rem[3][kMaxD + 1];  // p mod each prime, reduced in lockstep
  long long q[kMaxE + 1];
};

// a * b mod P for P = 2^31 - c (c < 2^10, a, b < P): the 62-bit product
// x = xh 2^31 + xl folds twice with 2^31 = c (mod P) inside 64-bit
// registers (one wide multiply-add each), leaving z < 2P: ~10 instructions,
// against ~45 for the 61-63-bit primes of round 1, whose 128-bit products
// made the division the slowest part of a verification.
__device__ __forceinline__ uint32_t mulmod31(uint32_t a, uint32_t b, uint32_t P, uint32_t c) {
  const uint64_t x = (uint64_t)a * b;
  const uint64_t y = (x >> 31) * c + (x & 0x7fffffffull);   // < 2^41
  uint32_t z = (uint32_t)((y >> 31) * c + (y & 0x7fffffffull));  // < 2^31 + 2^20
  return z >= P ? z - P : z;
}

// The profile, staged once per CTA in shared memory: the product loop below
// walks it serially, and global loads there would put an L2 round trip on
// every step of the chain.
struct ProfSmem {  // by entity e < n <= 64: real root / pair sum, pair product
  double v_hi[kMaxE], v_lo[kMaxE];
  double m_hi[kMaxE], m_lo[kMaxE];
  int8_t perm[kMaxE];
};

__device__ __forceinline__ void stage_profile_smem(ProfSmem& PS, const VerifyArgs& A, int tid,
                                                   int nthreads) {
  for (int i = tid; i < A.n; i += nthreads) PS.perm[i] = (int8_t)A.perm[i];
  for (int i = tid; i < A.r; i += nthreads) {
    PS.v_hi[i] = A.real_hi[i];
    PS.v_lo[i] = A.real_lo[i];
  }
  for (int i = tid; i < A.c; i += nthreads) {
    PS.v_hi[A.r + i] = A.sum_hi[i];
    PS.v_lo[A.r + i] = A.sum_lo[i];
    PS.m_hi[A.r + i] = A.prod_hi[i];
    PS.m_lo[A.r + i] = A.prod_lo[i];
  }
}

// Verify candidate k (A.pats[k]) with the calling warp; writes A.side[k],
// A.verdict[k] and, on PASS, A.coeffs row k (and raises *A.found if set).
__device__ __forceinline__ void verify_one(const VerifyArgs& A, const ProfSmem& PS, WarpBuf& B,
                                        long long k, int lane) {
  if (A.t_probe && lane == 0 && A.t_probe[3] == 0) A.t_probe[3] = rfr_globaltimer();
  const uint64_t full = A.n >= 64 ? ~0ull : ((1ull << A.n) - 1ull);
  const uint64_t s = A.pats[k] & full;
  int deg_s = 0;
  for (int i = 0; i < A.n; i++)
    if ((s >> i) & 1ull) deg_s += PS.perm[i] < A.r ? 1 : 2;
  const bool use_comp = deg_s > A.d - deg_s;
  const uint64_t t = use_comp ? (~s & full) : s;
  const int e = use_comp ? A.d - deg_s : deg_s;
  if (lane == 0) A.side[k] = use_comp ? 1 : 0;
  if (e < 1 || e >= A.d || e > kMaxE) {
    if (lane == 0) A.verdict[k] = (e > kMaxE) ? RFR_V_HOST : RFR_V_REJECT;
    return;
  }

  // ---- expand prod (x - u) * prod (x^2 - t x + m) over the selected entities
  int cur = 0, len = 1;  // current polynomial has `len` coefficients
  for (int i = lane; i < kMaxE + 2; i += 32) {
    B.c[0][i] = {i == 0 ? 1.0 : 0.0, 0.0};
    B.mag[0][i] = i == 0 ? 1.0 : 0.0;
    B.magp[0][i] = i == 0 ? 1.0 : 0.0;
  }
  __syncwarp();
  const double de = A.root_err;
  for (uint64_t tb = t; tb; tb &= tb - 1) {
    const int i = __ffsll((long long)tb) - 1;
    const int ent = PS.perm[i];
    const int nxt = cur ^ 1;
    if (ent < A.r) {
      const ddv u = {PS.v_hi[ent], PS.v_lo[ent]};
      const double au = fabs(u.hi);
      for (int j = lane; j <= len; j += 32) {
        ddv v = {0.0, 0.0};
        if (j >= 1) v = B.c[cur][j - 1];
        if (j < len) v = dd_add(v, dd_neg(dd_mul(u, B.c[cur][j])));
        double mv = (j >= 1 ? B.mag[cur][j - 1] : 0.0) + (j < len ? au * B.mag[cur][j] : 0.0);
        double mp = (j >= 1 ? B.magp[cur][j - 1] : 0.0) +
                    (j < len ? (au + de) * B.magp[cur][j] : 0.0);
        B.c[nxt][j] = v;
        B.mag[nxt][j] = mv;
        B.magp[nxt][j] = mp;
      }
      len += 1;
    } else {
      const ddv tt = {PS.v_hi[ent], PS.v_lo[ent]};
      const ddv mm = {PS.m_hi[ent], PS.m_lo[ent]};
      const double at = fabs(tt.hi), am = fabs(mm.hi);
      const double dt = 2.0 * de, dm = 2.0 * sqrt(am) * de + de * de;
      for (int j = lane; j <= len + 1; j += 32) {
        ddv v = {0.0, 0.0};
        if (j >= 2) v = B.c[cur][j - 2];
        if (j >= 1 && j - 1 < len) v = dd_add(v, dd_neg(dd_mul(tt, B.c[cur][j - 1])));
        if (j < len) v = dd_add(v, dd_mul(mm, B.c[cur][j]));
        double mv = (j >= 2 ? B.mag[cur][j - 2] : 0.0) +
                    (j >= 1 && j - 1 < len ? at * B.mag[cur][j - 1] : 0.0) +
                    (j < len ? am * B.mag[cur][j] : 0.0);
        double mp = (j >= 2 ? B.magp[cur][j - 2] : 0.0) +
                    (j >= 1 && j - 1 < len ? (at + dt) * B.magp[cur][j - 1] : 0.0) +
                    (j < len ? (am + dm) * B.magp[cur][j] : 0.0);
        B.c[nxt][j] = v;
        B.mag[nxt][j] = mv;
        B.magp[nxt][j] = mp;
      }
      len += 2;
    }
    cur = nxt;
    __syncwarp();
  }
  // len == e + 1
  if (A.t_probe && lane == 0 && A.t_probe[0] == 0) A.t_probe[0] = rfr_globaltimer();

  // ---- integrality with a derived error bound
  const double arith = (double)(4 * e + 8) * 7.9e-31;  // ~ (4e+8) * 2^-100
  bool reject = false, host = false;
  for (int j = lane; j <= e; j += 32) {
    const ddv v = B.c[cur][j];
    // nearest integer of hi + lo, kept exactly in int64: above 2^53 hi is
    // itself an integer and lo may exceed 1/2 (a double cannot hold the
    // 53..62-bit integer, and rounding hi alone would leave lo's whole part
    // in the "fraction" -- rejecting true factors with large coefficients)
    const bool big = fabs(v.hi) >= 4.611686018427388e18;  // beyond 2^62: the host decides
    const double rh = nearbyint(v.hi), rl = nearbyint(v.lo);
    double frac = (v.hi - rh) + (v.lo - rl);  // |frac| <= 1
    long long qv = big ? 0 : (long long)rh + (long long)rl;
    if (frac > 0.5) {
      qv += 1;
      frac -= 1.0;
    } else if (frac < -0.5) {
      qv -= 1;
      frac += 1.0;
    }
    const double bound = (B.magp[cur][j] - B.mag[cur][j]) + B.mag[cur][j] * arith + 1e-300;
    // the bound rests on the roots' a-posteriori error estimate, which can be
    // optimistic for moderately separated roots (seen 2x at d = 110): a
    // coefficient just outside it goes to the exact host check; a rejection
    // needs a clearly fractional coefficient (a false candidate has many)
    if (bound > 0.25 || big) host = true;
    else if (fabs(frac) > fmax(2.0 * bound, 1e-9)) reject = true;
    else if (fabs(frac) > 2.0 * bound) host = true;
    B.q[j] = qv;
  }
  reject = __any_sync(0xffffffffu, reject);
  host = __any_sync(0xffffffffu, host);
  if (reject) {
    if (lane == 0) A.verdict[k] = RFR_V_REJECT;
    return;
  }
  if (host) {
    if (lane == 0) A.verdict[k] = RFR_V_HOST;
    return;
  }
  __syncwarp();
  if (B.q[e] != 1) {
    if (lane == 0) A.verdict[k] = RFR_V_REJECT;
    return;
  }
  if (A.skip_division) {
    if (lane == 0) A.verdict[k] = RFR_V_PASS;
    for (int j = lane; j <= e && j < A.stride; j += 32) A.coeffs[k * A.stride + j] = B.q[j];
    return;
  }

  if (A.t_probe && lane == 0 && A.t_probe[1] == 0) A.t_probe[1] = rfr_globaltimer();
  // ---- trial division of p by q modulo three 31-bit primes, the three
  // divisions interleaved step by step (independent mulmod chains per lane)
  uint32_t* qm0 = reinterpret_cast<uint32_t*>(&B.mag[0][0]);   // q mod P_i: the magnitude
  uint32_t* qm1 = reinterpret_cast<uint32_t*>(&B.mag[1][0]);   // arrays are dead here
  uint32_t* qm2 = reinterpret_cast<uint32_t*>(&B.magp[0][0]);
  uint32_t* qmv[3] = {qm0, qm1, qm2};
  uint32_t P[3], pc[3];
#pragma unroll
  for (int pi = 0; pi < 3; pi++) {
    P[pi] = (uint32_t)A.primes[pi];
    pc[pi] = 0x80000000u - P[pi];  // P = 2^31 - c
    const uint64_t* pm = A.p_mod + (size_t)pi * (A.d + 1);
    for (int j = lane; j <= A.d; j += 32) B.rem[pi][j] = (uint32_t)pm[j];
    for (int j = lane; j < e; j += 32) {  // |q_j| < 2^62: one 64-bit remainder each
      const long long qj = B.q[j];
      const uint64_t aq = qj >= 0 ? (uint64_t)qj : (uint64_t)(-qj);
      const uint32_t r = (uint32_t)(aq % P[pi]);
      qmv[pi][j] = (qj >= 0 || r == 0) ? r : P[pi] - r;
    }
  }
  __syncwarp();
  for (int kk = A.d - e; kk >= 0; kk--) {
    uint32_t lead[3];
#pragma unroll
    for (int pi = 0; pi < 3; pi++) lead[pi] = B.rem[pi][kk + e];  // q monic
    __syncwarp();
    // e <= 64: each lane owns coefficients lane and lane + 32; all six
    // (coefficient, prime) mulmod chains of a lane are issued together
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int j = lane + 32 * h;
      if (j < e) {
#pragma unroll
        for (int pi = 0; pi < 3; pi++) {
          const uint32_t sub = mulmod31(lead[pi], qmv[pi][j], P[pi], pc[pi]);
          const uint32_t r0 = B.rem[pi][kk + j];
          B.rem[pi][kk + j] = r0 >= sub ? r0 - sub : r0 + P[pi] - sub;
        }
      }
    }
    __syncwarp();
  }
  if (A.t_probe && lane == 0 && A.t_probe[2] == 0) A.t_probe[2] = rfr_globaltimer();
  bool nz = false;
  for (int j = lane; j < e; j += 32) nz |= (B.rem[0][j] | B.rem[1][j] | B.rem[2][j]) != 0;
  const bool divides = !__any_sync(0xffffffffu, nz);
  if (lane == 0) A.verdict[k] = divides ? RFR_V_PASS : RFR_V_REJECT;
  if (lane == 0 && divides && A.found) {
    if (A.t_found) atomicCAS(A.t_found, 0ull, rfr_globaltimer());
    atomicExch(A.found, A.found_value);
    // cross-rank early exit: raise the peers' flags (P2P stores over NVLink)
    for (int i = 0; i < A.npeers; i++) *(volatile unsigned long long*)A.peer_found[i] = A.found_value;
    if (A.npeers) __threadfence_system();
  }
  if (divides)
    for (int j = lane; j <= e && j < A.stride; j += 32) A.coeffs[k * A.stride + j] = B.q[j];
}

}  // namespace rfr
