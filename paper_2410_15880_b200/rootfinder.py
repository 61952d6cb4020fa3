"""Host preprocessing: roots, the rho profile and the fixed-point search keys.

Drop-in for ``pkg/src/polyfactor/rootfinder.py`` ("R/rootfinder.py"):
``ToleranceConfig``, ``RootProfile``, ``find_roots``, ``build_profile``,
``profile_polynomial``, ``expected_real_roots``, ``expected_n``,
``residual_bound`` keep their names, fields and errors.  Root finding is
host preprocessing and is not timed (BASELINE.json north_star).

What is new is ``hp_profile``: the profile ``factor()`` searches with.  Roots
are seeded by ``numpy.roots`` and polished to ~106 bits in double-double by the
native Aberth iteration in ``librfr.so`` (``rfr_polish_roots``), which also
returns a rigorous inclusion radius per root (Lemma 1).  From the polished roots every
entity (real root u, or conjugate pair x^2 - t x + m) gets two exact 64-bit
fixed-point keys -- frac(u or t) and frac(u^2 or t^2 - 2m), the first two
power sums, both integers for every true factor -- and a window half-width T
derived from the error bounds.  DESIGN.md section 2 explains why this replaces
the reference's float64 rho + eps band for the factor() path.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from .errors import NonConvergence, UnpairedComplexRoot
from .polynomial import IntPolynomial

_TWO64 = 1 << 64


@dataclass(frozen=True)
class ToleranceConfig:
    """Numeric tolerances (R/rootfinder.py:23-55): eps drives candidate
    acceptance in the parity-mode search (recombine_e), root_tol and
    imag_threshold the float64 root API."""

    eps: float = 1e-6
    root_tol: float = 1e-12
    imag_threshold: float = 1e-9
    precision: str = "auto"  # auto | double | extended
    max_iterations: int = 500

    def __post_init__(self):
        if not 0 < self.eps < 0.5:
            raise ValueError("eps must be in (0, 0.5)")
        if self.root_tol <= 0:
            raise ValueError("root_tol must be positive")
        if self.imag_threshold <= 0:
            raise ValueError("imag_threshold must be positive")
        if self.precision not in ("auto", "double", "extended"):
            raise ValueError("precision must be auto, double, or extended")

    def complex_dtype(self, degree: int):
        if self.precision == "double":
            return np.complex128
        if self.precision == "extended" or degree > 50:
            return np.clongdouble
        return np.complex128


@dataclass(frozen=True)
class RootProfile:
    """Classified roots of one square-free polynomial (R/rootfinder.py:58-84).

    rho holds frac() of the r real roots and c pair sums, sorted; perm[i]
    names the entity behind rho[i] (0..r-1 real, r..r+c-1 pairs).  The
    optional fields carry the high-precision data of ``hp_profile``: the
    low words of the double-double values, the 64-bit search keys in rho
    order, the key-window half-width and the absolute root error bound."""

    real_roots: np.ndarray
    pair_sums: np.ndarray
    pair_products: np.ndarray
    rho: np.ndarray
    perm: tuple
    real_lo: np.ndarray | None = field(default=None, repr=False, compare=False)
    sum_lo: np.ndarray | None = field(default=None, repr=False, compare=False)
    prod_lo: np.ndarray | None = field(default=None, repr=False, compare=False)
    keys1: np.ndarray | None = field(default=None, repr=False, compare=False)
    keys2: np.ndarray | None = field(default=None, repr=False, compare=False)
    keys3: np.ndarray | None = field(default=None, repr=False, compare=False)
    key_err1: int = field(default=0, repr=False, compare=False)
    key_err2: int = field(default=0, repr=False, compare=False)
    key_err3: int = field(default=0, repr=False, compare=False)
    root_err: float = field(default=0.0, repr=False, compare=False)
    # multiprecision roots (coefficients beyond double-double, e.g. the monic
    # transform of a non-monic p): exact rational real roots by entity, (t, m)
    # of each pair, and their error bound -- for host decisions on factors
    # whose coefficients exceed what the double-double values can round
    hp_real: tuple | None = field(default=None, repr=False, compare=False)
    hp_pair: tuple | None = field(default=None, repr=False, compare=False)
    hp_err: float = field(default=0.0, repr=False, compare=False)

    @property
    def r(self) -> int:
        return len(self.real_roots)

    @property
    def c(self) -> int:
        return len(self.pair_sums)

    @property
    def n(self) -> int:
        return self.r + self.c


def frac(x: float) -> float:
    """Fractional part in [0, 1); frac(-0.25) == 0.75 (R/rootfinder.py:95-97)."""
    return float(x) - math.floor(x)


# ------------------------------------------------------------ hp roots
class _Dy:
    """Exact dyadic rational m * 2^e (m, e ints): the entity arithmetic of
    hp_profile (sums, products, halves of double-double values) without
    Fraction's gcd normalisation -- the same exact values, ~10x faster."""

    __slots__ = ("m", "e")

    def __init__(self, m: int, e: int):
        self.m, self.e = m, e

    @staticmethod
    def of(x) -> "_Dy":
        if isinstance(x, _Dy):
            return x
        if isinstance(x, int):
            return _Dy(x, 0)
        n, d = float(x).as_integer_ratio()
        return _Dy(n, 1 - d.bit_length())  # d is a power of two

    def __add__(self, o):
        o = _Dy.of(o)
        if self.e <= o.e:
            return _Dy(self.m + (o.m << (o.e - self.e)), self.e)
        return _Dy((self.m << (self.e - o.e)) + o.m, o.e)

    __radd__ = __add__

    def __neg__(self):
        return _Dy(-self.m, self.e)

    def __sub__(self, o):
        return self + (-_Dy.of(o))

    def __rsub__(self, o):
        return _Dy.of(o) + (-self)

    def __mul__(self, o):
        o = _Dy.of(o)
        return _Dy(self.m * o.m, self.e + o.e)

    __rmul__ = __mul__

    def __truediv__(self, k: int):
        if k != 2:
            raise ValueError("dyadic division by 2 only")
        return _Dy(self.m, self.e - 1)

    def __floor__(self) -> int:
        return self.m >> -self.e if self.e < 0 else self.m << self.e

    def __float__(self) -> float:
        m, e = self.m, self.e
        b = abs(m).bit_length()
        if b > 64:  # keep 64 bits and a sticky bit: float() then still rounds correctly
            k = b - 64
            a = abs(m)
            t = (a >> k) | (1 if a & ((1 << k) - 1) else 0)
            m, e = (t if m > 0 else -t), e + k
        return math.ldexp(float(m), e)  # m rounded once: correctly rounded

    def __abs__(self):
        return _Dy(abs(self.m), self.e)


def _key64(x) -> int:
    """floor(frac(x) 2^64 + 1/2) mod 2^64, exactly (= floor(x 2^64 + 1/2) mod 2^64)."""
    if isinstance(x, _Dy):
        s = x.e + 64
        k = x.m << s if s >= 0 else (x.m + (1 << (-s - 1))) >> (-s)
        return k & (_TWO64 - 1)
    return math.floor((x - math.floor(x)) * _TWO64 + Fraction(1, 2)) % _TWO64


def _dd_split(v) -> tuple[float, float]:
    hi = float(v)
    lo = float(v - (_Dy.of(hi) if isinstance(v, _Dy) else Fraction(hi)))
    return hi, lo


def _dd_frac(hi: float, lo: float, num=Fraction):
    if num is _Dy:
        return _Dy.of(hi) + _Dy.of(lo)
    return Fraction(hi) + Fraction(lo)


def _initial_roots(coeffs: list[int]) -> np.ndarray:
    """Seeds: eigenvalues of the companion matrix (numpy.roots).  Badly
    scaled coefficients (a monic transform a^(d-1) p(x / a) of a non-monic p
    spans ~d log2(a) bits) are balanced first: x = s y with s = 2^k ~
    |c_0|^(1/d), the geometric mean of the root magnitudes, and the seeds
    scaled back -- the polish converges from there instead of wandering."""
    d = len(coeffs) - 1
    if d == 1:
        return np.array([complex(-coeffs[0] / coeffs[1])])
    k = 0
    c0 = next((abs(c) for c in coeffs if c), 1)
    if max(abs(c) for c in coeffs).bit_length() > 200:
        k = round((c0.bit_length() - 1) / d)
    # coefficient of y^i after x = 2^k y (divided through by 2^(k d)): c_i 2^(k (i - d))
    c = np.array([float(Fraction(a) / (Fraction(2) ** (k * (d - i))))
                  for i, a in reversed(list(enumerate(coeffs)))], dtype=np.float64)
    z = np.roots(c) * float(2.0 ** k)
    if len(z) != d or not np.all(np.isfinite(z)):
        raise NonConvergence("numpy.roots failed to seed the root polish")
    return z


def _polish_dd(coeffs: list[int], z0: np.ndarray, max_iter: int = 60):
    """Native double-double Aberth polish.  Returns (re_hi, re_lo, im_hi,
    im_lo, err) or None when the roots cannot be certified."""
    from . import _lib

    lib = _lib.load()
    d = len(coeffs) - 1
    ch = np.zeros(d + 1)
    cl = np.zeros(d + 1)
    for k, a in enumerate(coeffs):
        hi, lo = _dd_split(Fraction(a))
        if Fraction(hi) + Fraction(lo) != a:
            return None  # coefficient not representable in double-double
        ch[k], cl[k] = hi, lo
    rh = np.ascontiguousarray(z0.real, dtype=np.float64).copy()
    ih = np.ascontiguousarray(z0.imag, dtype=np.float64).copy()
    rl = np.zeros(d)
    il = np.zeros(d)
    err = np.zeros(d)
    D = ctypes.POINTER(ctypes.c_double)
    rc = lib.rfr_polish_roots(ch.ctypes.data_as(D), cl.ctypes.data_as(D), d, rh.ctypes.data_as(D),
                              rl.ctypes.data_as(D), ih.ctypes.data_as(D), il.ctypes.data_as(D),
                              err.ctypes.data_as(D), max_iter)
    if rc != 0:
        return None
    return rh, rl, ih, il, err


def _polish_mp(coeffs: list[int], z0: np.ndarray):
    """Multiprecision Aberth polish for coefficients beyond double-double
    (e.g. Swinnerton-Dyer f6, 131-bit coefficients).  Returns the same tuple
    as _polish_dd."""
    import mpmath

    d = len(coeffs) - 1
    bits = max(abs(c) for c in coeffs).bit_length()
    # near a root the terms c_k z^k reach ~2^bits |z|^d and cancel: the working
    # precision must cover that magnitude, not only the coefficients (28
    # quadratics x^2 - p: 142-bit coefficients, |z|^56 ~ 2^190, no convergence
    # at bits + 160)
    zmax = max(2.0, float(np.max(np.abs(z0)))) if len(z0) else 2.0
    prec0 = max(256, bits + int(math.ceil(d * math.log2(zmax))) + 160)
    z = [complex(w) for w in z0]
    # the inclusion radii need |p(z)| small against |p'(z)|^2 / |p''(z)|:
    # when a root cannot be certified at one precision, polish on at twice it
    for attempt in range(3):
        prec = prec0 << attempt
        with mpmath.workprec(prec):
            out = _polish_mp_at(coeffs, z, prec, jitter=(attempt == 0))
            if out is None:
                return None
            cs, z = out
            radii = _mp_inclusion_radii(cs, z, prec)
            if radii is None:
                continue
            err = np.zeros(d)
            rh, rl, ih, il = (np.zeros(d) for _ in range(4))
            exact = []
            for i in range(d):
                re = _mpf_to_fraction(z[i].real)
                im = _mpf_to_fraction(z[i].imag)
                rh[i], rl[i] = _dd_split(re)
                ih[i], il[i] = _dd_split(im)
                exact.append((re, im))
                # the disc is reported around the double-double centre (what the
                # keys are built from): widen it by the rounding to double-double;
                # float() rounds to nearest, one ulp up keeps it an upper bound
                shift = abs(re - _dd_frac(rh[i], rl[i])) + abs(im - _dd_frac(ih[i], il[i]))
                err[i] = math.nextafter(float(radii[i]) + float(shift), math.inf)
            return rh, rl, ih, il, err, exact
    return None


def _polish_mp_at(coeffs, z0, prec, jitter):
    """Aberth iterations in the current mpmath working precision from the
    centres z0; returns (mp coefficients, mp roots) or None."""
    import mpmath

    d = len(coeffs) - 1
    cs = [mpmath.mpf(c) for c in coeffs]
    z = [mpmath.mpc(w) for w in z0]
    if jitter:  # jitter coincident seeds
        for i in range(d):
            for j in range(i):
                if abs(z[i] - z[j]) < mpmath.mpf(2) ** -20:
                    z[i] += mpmath.mpc(0, 1e-6 * (i + 1))

    def evalp(x):
        p = cs[d]
        dp = mpmath.mpc(0)
        for k in range(d - 1, -1, -1):
            dp = dp * x + p
            p = p * x + cs[k]
        return p, dp

    tol = mpmath.mpf(2) ** (-(prec - 40))
    floor = mpmath.mpf(2) ** -120
    prev = None
    for _ in range(200):
        worst = mpmath.mpf(0)
        new = []
        for i in range(d):
            p, dp = evalp(z[i])
            if dp == 0:
                dp = mpmath.mpf(2) ** -prec
            w = p / dp
            s = mpmath.mpc(0)
            for j in range(d):
                if j != i:
                    s += 1 / (z[i] - z[j])
            corr = w / (1 - w * s)
            new.append(z[i] - corr)
            worst = max(worst, abs(corr) / max(1, abs(z[i])))
        z = new
        if worst < tol:
            break
        # at the evaluation's noise floor (terms c_k z^k far above the value
        # cancel): corrections stop halving -- the inclusion radii account
        # for the residual (or ask for more precision)
        if prev is not None and worst < floor and worst > prev / 2:
            break
        prev = worst
    else:
        return None
    return cs, z


def _mp_inclusion_radii(cs, z, prec):
    """Rigorous inclusion radius per centre z_i (Lemma 1), in
    the working precision: p(z + h) = c0 + c1 h + c2 h^2 + R(h) with
    |c1| r > |c0| + |c2| r^2 + |R|max(r) puts exactly one root in D(z_i, r)
    (Rouche).  Each c_k carries at most gamma A_k of rounding error, A_k =
    P^(k)(|z|)/k! for P(x) = sum |a_j| x^j; the tail is bounded by
    P(R) (d r/R)^3 e^(d r/R) / 6, R = max(|z|, 1).  Returns the radii, or
    None when a root cannot be certified at this precision."""
    import mpmath

    d = len(cs) - 1
    gamma = mpmath.mpf(32 * d + 64) * mpmath.mpf(2) ** (-prec)
    fl = 1 + mpmath.mpf(4 * d + 8) * mpmath.mpf(2) ** (-prec)
    out = []
    for zi in z:
        p0, p1, p2 = mpmath.mpc(cs[d]), mpmath.mpc(0), mpmath.mpc(0)
        rho = abs(zi) * fl
        R = max(rho, mpmath.mpf(1))
        A0, A1, A2, PR = abs(cs[d]), mpmath.mpf(0), mpmath.mpf(0), abs(cs[d])
        for k in range(d - 1, -1, -1):
            p2 = p2 * zi + p1
            p1 = p1 * zi + p0
            p0 = p0 * zi + cs[k]
            ak = abs(cs[k])
            A2 = A2 * rho + A1
            A1 = A1 * rho + A0
            A0 = A0 * rho + ak
            PR = PR * R + ak
        A0, A1, A2, PR = A0 * fl, A1 * fl, A2 * fl, PR * fl
        c0 = abs(p0) * fl + gamma * A0
        c1 = abs(p1) / fl - gamma * A1
        c2 = abs(p2) * fl + gamma * A2
        if c1 <= 0:
            return None
        base = max(c0 / c1, mpmath.mpf(2) ** (-(prec - 8)) * R)
        for t in (1.125, 1.5, 2, 4, 16):
            r = base * t
            x = d * r / R
            tail = PR * x ** 3 * mpmath.exp(x) / 6
            if c1 * r > (c0 + c2 * r * r + tail) * (1 + mpmath.mpf(2) ** -30):
                out.append(r)
                break
        else:
            return None
    # pairwise disjoint discs (in the working precision; the centres are exact)
    for i in range(d):
        for j in range(i):
            if abs(z[i] - z[j]) <= (out[i] + out[j]) * (1 + mpmath.mpf(2) ** -30):
                return None
    return out


def _mpf_to_fraction(x) -> Fraction:
    import mpmath

    sign, man, exp, _ = mpmath.mpf(x)._mpf_
    v = Fraction(int(man) << exp) if exp >= 0 else Fraction(int(man), 1 << (-exp))
    return -v if sign else v


def hp_roots(p: IntPolynomial):
    """All roots of a monic square-free p to ~2^-100, with error bounds.
    Returns (re_hi, re_lo, im_hi, im_lo, err)."""
    return _hp_roots(p)[:5]


def _hp_roots(p: IntPolynomial):
    """hp_roots plus the exact rational (re, im) of every root when the
    multiprecision polish ran (else None)."""
    if not p.is_monic():
        raise ValueError("hp_roots expects a monic polynomial")
    coeffs = list(p.coeffs)
    d = len(coeffs) - 1
    if d < 1:
        raise ValueError("find_roots requires degree >= 1")
    z0 = _initial_roots(coeffs)

    def certified(res):
        # the discs must also decide real roots vs conjugate pairs
        if res is None:
            return None
        try:
            _pair_up(*res[:5])
        except NonConvergence:
            return None
        return res

    res = None
    if max(abs(c) for c in coeffs).bit_length() <= 100:
        res = _polish_dd(coeffs, z0)
        if res is not None:
            res = certified(tuple(res) + (None,))
    if res is None:
        res = certified(_polish_mp(coeffs, z0))
    if res is None:
        # float seeds too far off (real roots seeded ~0.5 off the axis for
        # 142-bit coefficients): multiprecision seeds, then the same polish
        import mpmath

        bits = max(abs(c) for c in coeffs).bit_length()
        with mpmath.workprec(bits + 200):
            try:
                rts = mpmath.polyroots([mpmath.mpf(c) for c in reversed(coeffs)], maxsteps=400,
                                       extraprec=bits + 200)
                res = certified(_polish_mp(coeffs, np.array([complex(r) for r in rts])))
            except mpmath.libmp.libhyper.NoConvergence:
                res = None
    if res is None:
        raise NonConvergence("root polish did not converge to certified inclusion discs")
    return res


def _pair_up(re_hi, re_lo, im_hi, im_lo, err):
    """Classify the certified roots into real roots and conjugate pairs.

    The discs D(z_i, err_i) are pairwise disjoint and hold one root each
    (rfr_polish_roots / _mp_inclusion_radii), so every root of p lies in
    exactly one of them.  The conjugate of root i is a root in the mirrored
    disc conj(D_i); when conj(D_i) meets no disc but D_b, the conjugate is
    root b.  So: real iff D_i meets the real axis and conj(D_i) meets no
    other disc (then conj(root_i) = root_i); a pair (a, b) iff D_a misses the
    axis (root_a is not real) and conj(D_a) meets D_b alone.  Anything else
    is undecided at this precision: NonConvergence, and the caller escalates.
    The reported real root is Re(z_i), within err_i of the real root (the
    projection onto the axis does not increase the distance)."""
    d = len(re_hi)
    re = np.asarray(re_hi, dtype=np.float64)
    im = np.asarray(im_hi, dtype=np.float64)
    rl = np.zeros(d) if re_lo is None else np.asarray(re_lo, dtype=np.float64)
    il = np.zeros(d) if im_lo is None else np.asarray(im_lo, dtype=np.float64)
    r = np.asarray(err, dtype=np.float64)

    def gap(sign):
        # |z_i - z_j| (sign +1) or |conj(z_i) - z_j| (sign -1) from both words,
        # less a bound on its rounding: the high-word difference is exact for
        # close values (Sterbenz) and every other step errs by 2^-53 relative
        # to what it computes, so roots 1e-8 apart at |z| ~ 1e8 still separate
        dh = re[:, None] - re[None, :]
        dl = rl[:, None] - rl[None, :]
        eh = sign * im[:, None] - im[None, :]
        el = sign * il[:, None] - il[None, :]
        dist = np.hypot(dh + dl, eh + el)
        fuzz = 2.0 ** -50 * (np.abs(dh) + np.abs(dl) + np.abs(eh) + np.abs(el)) + 1e-300
        return dist - fuzz

    rsum = (r[:, None] + r[None, :]) * (1.0 + 1e-9)
    own = gap(1.0)
    np.fill_diagonal(own, np.inf)
    if np.any(own <= rsum):
        raise NonConvergence("inclusion discs overlap")  # pairwise disjoint, else undecided
    meets = gap(-1.0) <= rsum  # conj(D_i) meets D_j
    reals, uppers = [], []
    partner = {}
    for i in range(d):
        hits = np.flatnonzero(meets[i])
        on_axis = abs(im[i] + il[i]) <= r[i] * (1.0 + 1e-9) + 2.0 ** -50 * abs(im[i])
        if on_axis:
            if len(hits) != 1 or hits[0] != i:
                raise NonConvergence(f"root {i}: cannot separate it from its mirror image")
            reals.append(i)
            continue
        if len(hits) != 1 or hits[0] == i:
            raise NonConvergence(f"root {i}: no unique conjugate partner")
        partner[i] = int(hits[0])
        if im[i] > 0:
            uppers.append(i)
    pairs = []
    for u in uppers:
        b = partner[u]
        if partner.get(b) != u or im[b] >= 0:
            raise UnpairedComplexRoot(f"no conjugate partner for root {complex(re[u], im[u])}")
        pairs.append((u, b))
    if 2 * len(pairs) + len(reals) != d:
        raise UnpairedComplexRoot(f"{len(uppers)} upper half-plane roots, {d - len(reals)} non-real")
    return reals, pairs


def hp_profile(p: IntPolynomial, num=None) -> RootProfile:
    """High-precision profile of a monic square-free p: rho, perm, double-
    double entities, the 64-bit keys in rho order and their error bounds.
    The entity values are exact rationals of the double-double roots: dyadic
    (_Dy, the default) or Fraction (num=Fraction: the same values, slower;
    tests/test_rootfinder.py checks the two agree field by field)."""
    num = num or _Dy
    re_hi, re_lo, im_hi, im_lo, err, exact = _hp_roots(p)
    reals, pairs = _pair_up(re_hi, re_lo, im_hi, im_lo, err)
    # (kind, R = first power sum, tau = second, errR, errTau, data, p3 = third, errP3)
    ents = []
    ex_vals = []  # per entity, from the multiprecision roots: u, or (t, m) of a pair
    # exact rationals of the double-double values
    for i in reals:
        ex_vals.append(exact[i][0] if exact is not None else None)
        u = _dd_frac(re_hi[i], re_lo[i], num)
        du = float(err[i])
        au = abs(float(u))
        ents.append(("r", u, u * u, du, 2 * au * du + du * du, i, u * u * u,
                     3 * au * au * du + 3 * au * du * du + du ** 3))
    for a, b in pairs:
        if exact is not None:
            xre = (exact[a][0] + exact[b][0]) / 2
            xim = (exact[a][1] - exact[b][1]) / 2
            ex_vals.append((2 * xre, xre * xre + xim * xim))
        else:
            ex_vals.append(None)
        # symmetrise: z = (z_a + conj z_b) / 2
        re = (_dd_frac(re_hi[a], re_lo[a], num) + _dd_frac(re_hi[b], re_lo[b], num)) / 2
        im = (_dd_frac(im_hi[a], im_lo[a], num) - _dd_frac(im_hi[b], im_lo[b], num)) / 2
        dz = float(max(err[a], err[b]))
        t = 2 * re
        m = re * re + im * im
        mod = math.sqrt(float(m))
        dt = 2 * dz
        dm = 2 * mod * dz + dz * dz
        tau = t * t - 2 * m
        dtau = 2 * abs(float(t)) * dt + dt * dt + 2 * dm
        # z^3 + conj(z)^3 = t^3 - 3 t m
        at, am = abs(float(t)), abs(float(m))
        p3 = t * t * t - 3 * t * m
        dp3 = 3 * at * at * dt + 3 * at * dt * dt + dt ** 3 + 3 * (at * dm + am * dt + dt * dm)
        ents.append(("p", t, tau, dt, dtau, m, p3, dp3))
    rows = []
    for kind, R, tau, dR, dtau, extra, p3, dp3 in ents:
        fr = R - math.floor(R)
        rho = float(fr)
        if rho >= 1.0:
            rho = math.nextafter(1.0, 0.0)
        rows.append((rho, kind, R, tau, dR, dtau, extra, p3, dp3))
    # sort by rho (ties: reals before pairs, then value) -- any fixed order works
    order = sorted(range(len(rows)), key=lambda k: (rows[k][0], rows[k][1], float(rows[k][2])))
    r = len(reals)
    real_hi, real_lo, sum_hi, sum_lo, prod_hi, prod_lo = [], [], [], [], [], []
    perm = []
    keys1, keys2, keys3 = [], [], []
    e1 = e2 = e3 = 0.0
    # entities are numbered reals first (in rho order), then pairs (in rho order)
    real_rows = [k for k in order if rows[k][1] == "r"]
    pair_rows = [k for k in order if rows[k][1] == "p"]
    ent_of = {}
    for j, k in enumerate(real_rows):
        ent_of[k] = j
        hi, lo = _dd_split(rows[k][2])
        real_hi.append(hi)
        real_lo.append(lo)
    for j, k in enumerate(pair_rows):
        ent_of[k] = r + j
        hi, lo = _dd_split(rows[k][2])
        sum_hi.append(hi)
        sum_lo.append(lo)
        mh, ml = _dd_split(rows[k][6])
        prod_hi.append(mh)
        prod_lo.append(ml)
    rho = []
    for k in order:
        rho_k, kind, R, tau, dR, dtau, _, p3, dp3 = rows[k]
        rho.append(rho_k)
        perm.append(ent_of[k])
        keys1.append(_key64(R))
        keys2.append(_key64(tau))
        keys3.append(_key64(p3))
        e1 += dR * 2.0**64 + 1.0
        e2 += dtau * 2.0**64 + 1.0
        e3 += dp3 * 2.0**64 + 1.0
    root_err = float(max(err)) if len(err) else 0.0
    # double-double representation slack of the stored entity values
    root_err = root_err + 2.0**-100 * max([1.0] + [abs(v) for v in real_hi + sum_hi])
    return RootProfile(
        real_roots=np.asarray(real_hi, dtype=np.float64),
        pair_sums=np.asarray(sum_hi, dtype=np.float64),
        pair_products=np.asarray(prod_hi, dtype=np.float64),
        rho=np.asarray(rho, dtype=np.float64),
        perm=tuple(perm),
        real_lo=np.asarray(real_lo, dtype=np.float64),
        sum_lo=np.asarray(sum_lo, dtype=np.float64),
        prod_lo=np.asarray(prod_lo, dtype=np.float64),
        keys1=np.asarray(keys1, dtype=np.uint64),
        keys2=np.asarray(keys2, dtype=np.uint64),
        keys3=np.asarray(keys3, dtype=np.uint64),
        # the float sums above round to nearest: a relative 2^-40 and one unit
        # keep them upper bounds (Lemma 2)
        key_err1=int(math.ceil(e1 * (1 + 2.0**-40))) + 1,
        key_err2=int(math.ceil(e2 * (1 + 2.0**-40))) + 1,
        key_err3=int(math.ceil(min(e3 * (1 + 2.0**-40), 2.0**66))) + 1,
        root_err=root_err,
        hp_real=tuple(ex_vals[k] for k in real_rows) if exact is not None else None,
        hp_pair=tuple(ex_vals[k] for k in pair_rows) if exact is not None else None,
        hp_err=float(max([0.0] + [float(e) for e in err])) if exact is not None else 0.0,
    )


# ------------------------------------------------------ reference API
def find_roots(p: IntPolynomial, cfg: ToleranceConfig | None = None) -> np.ndarray:
    """All d complex roots, conjugate symmetrised, as complex128: real roots
    first (ascending, exactly zero imaginary part), then conjugate pairs
    (w, conj w) in (re, im) order -- the layout of R/rootfinder.py:100-201."""
    cfg = cfg or ToleranceConfig()
    if p.is_zero():
        raise ValueError("zero polynomial has no root set")
    if p.degree < 1:
        raise ValueError("find_roots requires degree >= 1")
    q = p if p.is_monic() else _monic_rational(p)
    if q is None:  # non-monic: roots of the monic transform, scaled back
        from .polynomial import monic_transform

        t = monic_transform(p)
        re_hi, re_lo, im_hi, im_lo, err = hp_roots(t)
        scale = float(p.leading)
        re_hi = re_hi / scale
        im_hi = im_hi / scale
        err = err / abs(scale)
    else:
        re_hi, re_lo, im_hi, im_lo, err = hp_roots(q)
    reals, pairs = _pair_up(re_hi, re_lo, im_hi, im_lo, err)
    out = [complex(v, 0.0) for v in sorted(re_hi[i] for i in reals)]
    pw = sorted(((re_hi[a] + re_hi[b]) / 2, (im_hi[a] - im_hi[b]) / 2) for a, b in pairs)
    for re, im in pw:
        out.append(complex(re, im))
        out.append(complex(re, -im))
    return np.asarray(out, dtype=np.complex128)


def _monic_rational(p: IntPolynomial):
    return p if p.is_monic() else None


def build_profile(roots: np.ndarray, cfg: ToleranceConfig | None = None) -> RootProfile:
    """Classify a conjugate-closed root multiset into the sorted rho profile
    (R/rootfinder.py:204-245): reals contribute frac(u), each pair
    frac(z + conj z) once; UnpairedComplexRoot when a partner is missing."""
    cfg = cfg or ToleranceConfig()
    z = np.asarray(roots, dtype=np.complex128)
    scale = np.maximum(1.0, np.abs(z))
    real_mask = np.abs(z.imag) <= cfg.imag_threshold * scale
    reals = np.sort(z.real[real_mask])
    rest = list(z[~real_mask])
    uppers = sorted((w for w in rest if w.imag > 0), key=lambda w: (w.real, w.imag))
    lowers = [w for w in rest if w.imag <= 0]
    if len(uppers) != len(lowers):
        raise UnpairedComplexRoot(f"{len(uppers)} upper vs {len(lowers)} lower half-plane roots")
    sums, prods = [], []
    for u in uppers:
        target = u.conjugate()
        best = min(range(len(lowers)), key=lambda i: abs(lowers[i] - target))
        partner = lowers.pop(best)
        if abs(partner - target) > 1e-6 * max(1.0, abs(u)):
            raise UnpairedComplexRoot(f"no conjugate partner for root {u}")
        w = (u + partner.conjugate()) / 2
        sums.append(float(2.0 * w.real))
        prods.append(float(abs(w) ** 2))
    entries = [(frac(u), i) for i, u in enumerate(reals)]
    entries += [(frac(s), len(reals) + j) for j, s in enumerate(sums)]
    entries.sort()
    rho = np.array([min(e[0], math.nextafter(1.0, 0.0)) for e in entries], dtype=np.float64)
    return RootProfile(
        real_roots=np.asarray(reals, dtype=np.float64),
        pair_sums=np.asarray(sums, dtype=np.float64),
        pair_products=np.asarray(prods, dtype=np.float64),
        rho=rho,
        perm=tuple(e[1] for e in entries),
    )


def profile_polynomial(p: IntPolynomial, cfg: ToleranceConfig | None = None) -> RootProfile:
    """find_roots followed by build_profile (R/rootfinder.py:248-251)."""
    cfg = cfg or ToleranceConfig()
    return build_profile(find_roots(p, cfg), cfg)


def expected_real_roots(d) -> float:
    """(2/pi) ln d, leading term of the expected real-root count."""
    if d < 1:
        raise ValueError("degree must be >= 1")
    return (2.0 / math.pi) * math.log(d)


def expected_n(d) -> float:
    """Expected instance size d/2 + (1/pi) ln d."""
    if d < 1:
        raise ValueError("degree must be >= 1")
    return d / 2.0 + math.log(d) / math.pi


def residual_bound(p: IntPolynomial, root: complex, root_tol: float) -> float:
    """root_tol * max|a_i| * max(1, |root|)^d (R/rootfinder.py:269-272)."""
    amax = max(abs(c) for c in p.coeffs)
    return root_tol * amax * max(1.0, abs(root)) ** p.degree
