// rfr_host.cpp -- native host numerics for the preprocessing in front of the
// search (not timed: north_star puts root finding outside the timed path).
//
//  rfr_polish_roots   simultaneous Aberth-Ehrlich corrections in double-double
//                     complex arithmetic (~106-bit), seeded by any approximate
//                     roots, with a rigorous inclusion radius per root
//                     (Rouche on the Taylor expansion, pairwise disjoint discs).  It
//                     replaces find_roots' iteration (pkg/src/polyfactor/
//                     rootfinder.py:100-174), whose 64-bit roots would make the
//                     subset-sum keys ~2^-45 coarse; ~2^-100 roots make them
//                     exact to the last key bit.
//  rfr_squarefree_mod gcd(p, p') over F_q, the fast screen in front of the
//                     exact square-free decomposition (polynomial.py:221-247).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/rfr.h"

namespace {

// ---------------------------------------------------------- double-double
struct dd {
  double hi, lo;
};

inline dd two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
inline dd quick_two_sum(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
inline dd two_prod(double a, double b) {
  double p = a * b;
  return {p, std::fma(a, b, -p)};
}
inline dd operator+(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
inline dd operator-(dd a) { return {-a.hi, -a.lo}; }
inline dd operator-(dd a, dd b) { return a + (-b); }
inline dd operator*(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
inline dd operator/(dd a, dd b) {
  double q1 = a.hi / b.hi;
  dd r = a - b * dd{q1, 0.0};
  double q2 = r.hi / b.hi;
  r = r - b * dd{q2, 0.0};
  double q3 = r.hi / b.hi;
  dd q = quick_two_sum(q1, q2);
  return q + dd{q3, 0.0};
}
inline double to_d(dd a) { return a.hi + a.lo; }

struct cdd {
  dd re, im;
};
inline cdd operator+(cdd a, cdd b) { return {a.re + b.re, a.im + b.im}; }
inline cdd operator-(cdd a, cdd b) { return {a.re - b.re, a.im - b.im}; }
inline cdd operator*(cdd a, cdd b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
inline cdd operator/(cdd a, cdd b) {
  // Smith's algorithm: no |b|^2, so no overflow for |b| ~ 1e160 (|z|^d of
  // degree-100 polynomials with roots near 40)
  if (std::fabs(b.re.hi) >= std::fabs(b.im.hi)) {
    const dd r = b.im / b.re;
    const dd den = b.re + b.im * r;
    return {(a.re + a.im * r) / den, (a.im - a.re * r) / den};
  }
  const dd r = b.re / b.im;
  const dd den = b.re * r + b.im;
  return {(a.re * r + a.im) / den, (a.im * r - a.re) / den};
}
inline double cabs_d(cdd a) { return std::hypot(to_d(a.re), to_d(a.im)); }

// p(z), p'(z) by Horner in double-double, with the running bound
// sum_k |a_k| |z|^k used for the evaluation-error estimate.
void horner(const std::vector<dd>& c, cdd z, cdd& pz, cdd& dpz, double& absum) {
  const int d = (int)c.size() - 1;
  cdd p = {c[d], {0, 0}};
  cdd q = {{0, 0}, {0, 0}};
  const double az = cabs_d(z);
  double s = std::fabs(to_d(c[d]));
  for (int k = d - 1; k >= 0; k--) {
    q = q * z + p;
    p = p * z + cdd{c[k], {0, 0}};
    s = s * az + std::fabs(to_d(c[k]));
  }
  pz = p;
  dpz = q;
  absum = s;
}

}  // namespace

extern "C" {

int rfr_polish_roots(const double* coef_hi, const double* coef_lo, int d, double* re_hi,
                     double* re_lo, double* im_hi, double* im_lo, double* err, int max_iter) {
  if (d < 1 || !coef_hi || !re_hi || !im_hi || !err) return RFR_E_ARG;
  std::vector<dd> c(d + 1);
  for (int k = 0; k <= d; k++) c[k] = {coef_hi[k], coef_lo ? coef_lo[k] : 0.0};
  if (c[d].hi != 1.0 || c[d].lo != 0.0) return RFR_E_ARG;  // monic only
  std::vector<cdd> z(d);
  for (int i = 0; i < d; i++)
    z[i] = {{re_hi[i], re_lo ? re_lo[i] : 0.0}, {im_hi[i], im_lo ? im_lo[i] : 0.0}};
  const double eps_dd = std::ldexp(1.0, -104);
  std::vector<cdd> corr(d);
  int it = 0;
  for (; it < max_iter; it++) {
    double worst = 0.0;
    for (int i = 0; i < d; i++) {
      cdd pz, dpz;
      double absum;
      horner(c, z[i], pz, dpz, absum);
      if (to_d(dpz.re) == 0.0 && to_d(dpz.im) == 0.0) dpz.re = {1e-300, 0.0};
      cdd w = pz / dpz;
      cdd sum = {{0, 0}, {0, 0}};
      for (int j = 0; j < d; j++) {
        if (j == i) continue;
        cdd diff = z[i] - z[j];
        if (to_d(diff.re) == 0.0 && to_d(diff.im) == 0.0) diff.re = {1e-300, 0.0};
        sum = sum + cdd{{1.0, 0}, {0, 0}} / diff;
      }
      cdd den = cdd{{1.0, 0}, {0, 0}} - w * sum;
      if (to_d(den.re) == 0.0 && to_d(den.im) == 0.0) den.re = {1e-300, 0.0};
      corr[i] = w / den;
      const double rel = cabs_d(corr[i]) / std::fmax(1.0, cabs_d(z[i]));
      worst = std::fmax(worst, rel);
    }
    for (int i = 0; i < d; i++) z[i] = z[i] - corr[i];  // Jacobi-style update
    if (worst < 8.0 * eps_dd) break;
  }
  // Rigorous inclusion radii (Lemma 1).  Around each centre z
  // (the double-double value itself, exactly representable) write
  // p(z + h) = c0 + c1 h + c2 h^2 + R(h).  If on the circle |h| = r
  //     |c1| r  >  |c0| + |c2| r^2 + |R|max(r),
  // Rouche's theorem (p against its linear term c1 h) puts exactly one root
  // of p in the disc D(z, r).  c0, c1, c2 come from one triple Horner pass
  // in double-double; each carries an evaluation error of at most
  // gamma * A_k with A_k = P^(k)(|z|) / k!, P(x) = sum |a_j| x^j, so the test
  // uses |c0|, |c2| inflated and |c1| deflated by those amounts.  The tail
  // k >= 3 is bounded by A_k r^k <= P(R) C(d, k) (r / R)^k, R = max(|z|, 1):
  //     |R|max(r) <= P(R) (d r / R)^3 e^(d r / R) / 6.
  // Pairwise disjoint discs (checked below) then hold one root each, so they
  // account for all d roots: the true root is within err[i] of the centre.
  const double gamma = (32.0 * d + 64.0) * eps_dd;  // complex dd Horner, with room
  const double fl = 1.0 + (4.0 * d + 8.0) * std::ldexp(1.0, -53);  // double Horner, upward
  const double cab = std::ldexp(1.0, -50);                           // |.| of a dd complex
  std::vector<char> ok(d, 0);
  for (int i = 0; i < d; i++) {
    const cdd zi = z[i];
    cdd p0 = {c[d], {0, 0}}, p1 = {{0, 0}, {0, 0}}, p2 = {{0, 0}, {0, 0}};
    const double rho = cabs_d(zi) * (1.0 + cab);
    const double R = std::fmax(rho, 1.0);
    double A0 = std::fabs(to_d(c[d])), A1 = 0.0, A2 = 0.0, PR = A0;
    for (int k = d - 1; k >= 0; k--) {
      p2 = p2 * zi + p1;
      p1 = p1 * zi + p0;
      p0 = p0 * zi + cdd{c[k], {0, 0}};
      const double ak = std::fabs(to_d(c[k])) * (1.0 + std::ldexp(1.0, -52));
      A2 = A2 * rho + A1;
      A1 = A1 * rho + A0;
      A0 = A0 * rho + ak;
      PR = PR * R + ak;
    }
    A0 *= fl; A1 *= fl; A2 *= fl; PR *= fl;
    const double c0 = cabs_d(p0) * (1.0 + cab) + gamma * A0;
    const double c1 = cabs_d(p1) * (1.0 - cab) - gamma * A1;
    const double c2 = cabs_d(p2) * (1.0 + cab) + gamma * A2;
    double r_ok = INFINITY;
    if (c1 > 0.0 && std::isfinite(c0) && std::isfinite(c2) && std::isfinite(PR)) {
      const double base = std::fmax(c0 / c1, std::ldexp(1.0, -200) * R);
      for (double t : {1.125, 1.5, 2.0, 4.0, 16.0}) {
        const double r = t * base;
        const double x = d * r / R;
        const double tail = PR * x * x * x * std::exp(x) / 6.0;
        const double lhs = c1 * r;
        const double rhs = c0 + c2 * r * r + tail;
        if (std::isfinite(lhs) && lhs > rhs * (1.0 + 1e-9)) {
          r_ok = r;
          break;
        }
      }
    }
    ok[i] = std::isfinite(r_ok);
    err[i] = r_ok;
  }
  int status = RFR_OK;
  for (int i = 0; i < d && status == RFR_OK; i++) {
    if (!ok[i]) status = RFR_E_NUMERIC;
    // pairwise disjoint discs: |z_i - z_j| from both words (the high-word
    // difference is exact for close values, Sterbenz; every other step errs
    // by 2^-53 relative to what it computes)
    for (int j = i + 1; j < d && status == RFR_OK; j++) {
      const double dh = z[i].re.hi - z[j].re.hi, dl = z[i].re.lo - z[j].re.lo;
      const double eh = z[i].im.hi - z[j].im.hi, el = z[i].im.lo - z[j].im.lo;
      const double fuzz =
          std::ldexp(1.0, -50) * (std::fabs(dh) + std::fabs(dl) + std::fabs(eh) + std::fabs(el)) + 1e-300;
      if (std::hypot(dh + dl, eh + el) - fuzz <= (err[i] + err[j]) * (1.0 + 1e-9)) status = RFR_E_NUMERIC;
    }
  }
  for (int i = 0; i < d; i++) {
    re_hi[i] = z[i].re.hi;
    if (re_lo) re_lo[i] = z[i].re.lo;
    im_hi[i] = z[i].im.hi;
    if (im_lo) im_lo[i] = z[i].im.lo;
  }
  return status;
}

// a * b mod q; for q = 2^k - c with small c (every prime the library uses)
// the 2k-bit product is folded twice with 2^k = c (mod q) instead of the
// 128-bit division.
struct Modulus {
  uint64_t q, c;
  int k;  // 0: generic modulus (128-bit remainder)
  explicit Modulus(uint64_t q_) : q(q_), c(0), k(0) {
    const int kk = 64 - __builtin_clzll(q_);
    if (kk <= 63) {
      const uint64_t cc = (1ull << kk) - q_;
      if (cc < 1024) {
        k = kk;
        c = cc;
      }
    }
  }
};
static inline uint64_t mulmod(uint64_t a, uint64_t b, const Modulus M) {
  const unsigned __int128 x = (unsigned __int128)a * b;
  if (!M.k) return (uint64_t)(x % M.q);
  const uint64_t mask = (1ull << M.k) - 1ull;
  const unsigned __int128 y = (unsigned __int128)(uint64_t)(x >> M.k) * M.c + (uint64_t)(x & mask);
  uint64_t z = (uint64_t)(y & mask) + (uint64_t)(y >> M.k) * M.c;
  while (z >= M.q) z -= M.q;
  return z;
}
extern "C++" {
// Reducers for the Euclid loop: the Mersenne prime 2^61 - 1 (the screen's
// first choice) and any other modulus.
struct RedM61 {
  static constexpr uint64_t q = (1ull << 61) - 1;
  uint64_t mul(uint64_t a, uint64_t b) const {
    const unsigned __int128 x = (unsigned __int128)a * b;
    uint64_t z = (uint64_t)(x & q) + (uint64_t)(x >> 61);
    z = (z & q) + (z >> 61);
    return z >= q ? z - q : z;
  }
};
struct RedAny {
  Modulus M;
  uint64_t mul(uint64_t a, uint64_t b) const { return mulmod(a, b, M); }
};

template <class Red>
static int squarefree_euclid(const uint64_t* cm, int d, uint64_t q, const Red R) {
  std::vector<uint64_t> a(cm, cm + d + 1), b(d);
  for (auto& v : a) v %= q;
  for (int k = 1; k <= d; k++) b[k - 1] = R.mul(a[k], (uint64_t)k % q);
  int da = d, db = d - 1;
  while (db >= 0 && b[db] == 0) db--;
  if (db < 0) return 0;  // p' == 0 mod q: undecided
  // Euclid over F_q by pseudo-division (a <- lc(b) a - lc(a) x^s b): no
  // inverses, whose dependent chains would dominate; only the degree of the
  // gcd matters, and scaling by the unit lc(b) does not change it
  while (db >= 0) {
    uint64_t* A = a.data();
    const uint64_t* B = b.data();
    const uint64_t lb = B[db];
    while (da >= db) {
      const uint64_t la = A[da];
      const int s0 = da - db;
      for (int k = 0; k < s0; k++) A[k] = R.mul(A[k], lb);
      for (int k = 0; k < db; k++) {
        const uint64_t x = R.mul(A[s0 + k], lb), y = R.mul(la, B[k]);
        A[s0 + k] = x >= y ? x - y : x + q - y;
      }
      da--;
      while (da >= 0 && A[da] == 0) da--;
      if (da < 0) break;
    }
    std::swap(a, b);
    std::swap(da, db);
    if (db < 0) break;
  }
  // gcd is a (degree da)
  return da == 0 ? 1 : 0;
}

// The same Euclid for q < 2^25 in doubles: residues are exact integers kept
// in the symmetric range |r| <= q/2 (+1 when x / q rounds the other way), so
// the pseudo-division update A lb - la B stays below 2q^2 < 2^51 in magnitude
// (exact), and one round-to-nearest reduction per entry, with no compare,
// brings it back: branch-free, so the update loops vectorise (AVX2: 34 -> ~8
// us at d = 100).  A residue is zero iff its representative is 0.0.
static inline double red_fp(double x, double q, double qinv) { return x - std::rint(x * qinv) * q; }
__attribute__((target_clones("avx512f", "avx2", "default")))
static int squarefree_euclid_fp(const uint64_t* cm, int d, uint64_t q64) {
  const double q = (double)q64, qinv = 1.0 / q;
  std::vector<double> a(d + 1), b(d);
  for (int k = 0; k <= d; k++) a[k] = (double)(cm[k] % q64);
  for (int k = 1; k <= d; k++) b[k - 1] = red_fp(a[k] * (double)k, q, qinv);
  int da = d, db = d - 1;
  while (db >= 0 && b[db] == 0.0) db--;
  if (db < 0) return 0;
  while (db >= 0) {
    double* A = a.data();
    const double* B = b.data();
    const double lb = B[db];
    while (da >= db) {
      const double la = A[da];
      const int s0 = da - db;
      for (int k = 0; k < s0; k++) A[k] = red_fp(A[k] * lb, q, qinv);
      double* As = A + s0;
      for (int k = 0; k < db; k++) As[k] = red_fp(As[k] * lb - la * B[k], q, qinv);
      da--;
      while (da >= 0 && A[da] == 0.0) da--;
      if (da < 0) break;
    }
    std::swap(a, b);
    std::swap(da, db);
    if (db < 0) break;
  }
  return da == 0 ? 1 : 0;
}
}  // extern "C++"

int rfr_multiply_i64(const int64_t* a, int da, const int64_t* b, int db, int64_t* out) {
  if (da < 0 || db < 0) return -1;
  // every partial sum of a coefficient is at most (min(da, db) + 1) max|a| max|b|:
  // keep that below 2^126 so the 128-bit accumulation cannot wrap
  unsigned __int128 ma = 0, mb = 0;
  for (int i = 0; i <= da; i++) {
    const unsigned __int128 v = a[i] < 0 ? (unsigned __int128)(-(__int128)a[i]) : (unsigned __int128)a[i];
    if (v > ma) ma = v;
  }
  for (int i = 0; i <= db; i++) {
    const unsigned __int128 v = b[i] < 0 ? (unsigned __int128)(-(__int128)b[i]) : (unsigned __int128)b[i];
    if (v > mb) mb = v;
  }
  const unsigned __int128 terms = (unsigned __int128)((da < db ? da : db) + 1);
  const unsigned __int128 cap = (unsigned __int128)1 << 126;
  if (ma && mb && (ma > cap / mb || ma * mb > cap / terms)) return -1;
  const __int128 lim = (__int128)1 << 62;
  for (int k = 0; k <= da + db; k++) {
    __int128 acc = 0;
    const int i0 = k > db ? k - db : 0, i1 = k < da ? k : da;
    for (int i = i0; i <= i1; i++) acc += (__int128)a[i] * b[k - i];
    if (acc >= lim || acc <= -lim) return -1;
    out[k] = (int64_t)acc;
  }
  return 1;
}

int rfr_divide_monic_i64(const int64_t* p, int dp, const int64_t* q, int dq, int64_t* r) {
  if (dq < 0 || dp < dq || q[dq] != 1) return -1;
  const int64_t p_lim = (int64_t)1 << 62, q_lim = (int64_t)1 << 31;
  for (int i = 0; i <= dp; i++)
    if (p[i] >= p_lim || p[i] <= -p_lim) return -1;
  for (int i = 0; i <= dq; i++)
    if (q[i] >= q_lim || q[i] <= -q_lim) return -1;
  // |rem| <= |p| + sum |t| |q| < 2^62 + (dq + 1) 2^62 2^31 < 2^127 for dq < 2^32
  std::vector<__int128> rem(p, p + dp + 1);
  const __int128 lim = (__int128)1 << 62;
  for (int k = dp - dq; k >= 0; k--) {
    const __int128 t = rem[k + dq];
    if (t >= lim || t <= -lim) return -1;
    r[k] = (int64_t)t;
    if (t != 0)
      for (int i = 0; i < dq; i++) rem[k + i] -= t * (__int128)q[i];
  }
  for (int i = 0; i < dq; i++)
    if (rem[i] != 0) return 0;
  return 1;
}

int rfr_squarefree_i64(const int64_t* c, int d, uint64_t q) {
  if (d < 1 || q < 3 || q >= (1ull << 62)) return 0;
  for (int k = 0; k <= d; k++)
    if (c[k] >= ((int64_t)1 << 62) || c[k] <= -((int64_t)1 << 62)) return -1;
  uint64_t buf[256];
  std::vector<uint64_t> big;
  uint64_t* cm = buf;
  if (d + 1 > 256) {
    big.resize((size_t)d + 1);
    cm = big.data();
  }
  const int64_t qs = (int64_t)q;
  for (int k = 0; k <= d; k++) {
    int64_t r = c[k] % qs;
    cm[k] = (uint64_t)(r < 0 ? r + qs : r);
  }
  return rfr_squarefree_mod(cm, d, q);
}

int rfr_squarefree_mod(const uint64_t* cm, int d, uint64_t q) {
  if (d < 1 || q < 3) return 0;
  if (cm[d] % q == 0) return 0;
  if (d == 1) return 1;
  if (q < (1ull << 25)) return squarefree_euclid_fp(cm, d, q);
  if (q == RedM61::q) return squarefree_euclid(cm, d, q, RedM61());
  return squarefree_euclid(cm, d, q, RedAny{Modulus(q)});
}

}  // extern "C"
