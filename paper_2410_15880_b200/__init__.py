"""paper_2410_15880_b200 -- B200-native recombination stage of the
Real-Factors-Recombination integer-polynomial factorizer (arXiv 2410.15880).

Drop-in for the reference package ``polyfactor``'s public surface on the
recombination path (pkg/src/polyfactor/__init__.py:12-77): ``factor``,
``is_irreducible``, the result/stat types, the polynomial type and
generators, the rho/candidate types and ``recombine_e``.  The search and the
candidate verification run as hand-written sm_100a kernels in ``librfr.so``
(C ABI in include/rfr.h); there is no CPU fallback.
"""
from .errors import (
    NonConvergence,
    PolyfactorError,
    PolynomialParseError,
    RecombineDeviceError,
    UnpairedComplexRoot,
    WidthExceeded,
)
from .polynomial import (
    IntPolynomial,
    SquareFreePart,
    divide_exact,
    gen_random_reducible,
    gen_random_reducible_parts,
    gen_swinnerton_dyer,
    monic_transform,
    monic_untransform_factor,
    multiply,
    poly_gcd,
    square_free_decompose,
)
from .rootfinder import (
    RootProfile,
    ToleranceConfig,
    build_profile,
    expected_n,
    expected_real_roots,
    find_roots,
    hp_profile,
    profile_polynomial,
)
from .recombine import (
    BACKENDS,
    GUARD,
    CandidateSet,
    RecombineStats,
    RhoVector,
    accept,
    recombine_e,
    search_keys,
    value,
)
from .parallel import parallel_recombine_e, sharded_search_keys
from .verify import (
    FactorizationResult,
    FactorStats,
    factor,
    is_irreducible,
    selected_degree,
    verify_candidates,
)
from .report import CSV_HEADER, BenchRecord, bench_rows

__version__ = "0.1.0"
