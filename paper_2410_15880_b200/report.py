"""Benchmark rows in the reference's report schema.

Mirrors the row type of ``pkg/src/polyfactor/cli.py`` ("R/cli.py"):
``CSV_HEADER`` and ``BenchRecord`` (R/cli.py:31-72) keep the same ten
columns in the same order, so rows from this engine parse with the
reference's own ``BenchRecord.from_csv`` and sit beside its rows in one CSV.
``bench_rows`` follows R/cli.py:172-201: deterministic
``gen_random_reducible_parts(d, 100, seed + trial)`` inputs, one row per
(degree, trial), ``wall_s`` = the recombination stage unless
``include_roots``.  The backend column reads ``"e-b200"``; the GPU-side
fields (GPUs, device time, pairs/s, HBM GB/s against the SURVEY s8(d)
algorithmic bytes and the roofline fraction, all over the whole device call:
``*_call``) go in ``BenchRecord.extra`` and in
``to_json()``, not in the CSV.  The reference's argparse CLI itself is out of
scope.
"""
from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass, field

from .polynomial import gen_random_reducible_parts
from .rootfinder import ToleranceConfig
from .verify import factor

CSV_HEADER = "d,n,backend,workers,wall_s,visited,probes_mean,candidates,factors,seed"
BACKEND_NAME = "e-b200"


@dataclass(frozen=True)
class BenchRecord:
    """One benchmark row; field order matches the CSV header (R/cli.py:34-72)."""

    d: int
    n: int
    backend: str
    workers: int
    wall_s: float
    visited: int
    probes_mean: float
    candidates: int
    factors: int
    seed: int
    extra: dict = field(default_factory=dict, compare=False)

    def to_csv(self) -> str:
        return (
            f"{self.d},{self.n},{self.backend},{self.workers},{self.wall_s:.6f},"
            f"{self.visited},{self.probes_mean:.4f},{self.candidates},{self.factors},{self.seed}"
        )

    @classmethod
    def from_csv(cls, line: str) -> "BenchRecord":
        cells = line.strip().split(",")
        if len(cells) != 10:
            raise ValueError(f"expected 10 CSV cells, got {len(cells)}")
        return cls(
            d=int(cells[0]), n=int(cells[1]), backend=cells[2], workers=int(cells[3]),
            wall_s=float(cells[4]), visited=int(cells[5]), probes_mean=float(cells[6]),
            candidates=int(cells[7]), factors=int(cells[8]), seed=int(cells[9]),
        )

    def to_json(self) -> str:
        row = {k: getattr(self, k) for k in CSV_HEADER.split(",")}
        row.update(self.extra)
        return json.dumps(row)


def _peak_gbs() -> tuple[float, str]:
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(n: int) -> int:
    """48 B per record of the folded halves, 2^a + 2^b."""
    m = n - 1
    a = (m + 1) // 2
    return 48 * ((1 << a) + (1 << (m - a)))


def bench_rows(degrees, trials: int = 1, seed: int = 0, workers: int = 1,
               include_roots: bool = False, cfg: ToleranceConfig | None = None):
    """Yield one BenchRecord per (degree, trial) (R/cli.py:172-201 inputs and
    timing convention).  ValueError for an odd degree, as the reference."""
    cfg = cfg or ToleranceConfig()
    peak, peak_kind = _peak_gbs()
    for d in degrees:
        if d % 2:
            raise ValueError("bench degrees must be even")
        for trial in range(trials):
            f, g = gen_random_reducible_parts(d, 100, seed + trial)
            p = f * g
            t0 = time.perf_counter()
            res = factor(p, cfg, workers=workers)
            total = time.perf_counter() - t0
            st = res.stats
            wall = total if include_roots else st.recombine_seconds
            rec = st.recombine
            dev_ms = rec.device_ms if rec.device_ms else None
            extra = {"gpus": workers, "wall_total_s": total,
                     "verify_seconds": st.verify_seconds, "root_seconds": st.root_seconds}
            if dev_ms:
                alg = algorithmic_bytes(st.n)
                gbs = alg / (dev_ms * 1e-3) / 1e9
                # over the whole fused call (lists, join -- stopped early when a
                # factor verifies -- and verification): not bench.py's
                # join-only roofline, hence the _call suffix
                extra.update({"device_ms": dev_ms,
                              "pairs_per_s_call": 2.0 ** (st.n - 1) / (dev_ms * 1e-3),
                              "hbm_gbs_algorithmic_call": gbs, "roofline_frac_call": gbs / peak,
                              "peak_gbs": peak, "peak_source": peak_kind})
            yield BenchRecord(
                d=d, n=st.n, backend=BACKEND_NAME, workers=workers, wall_s=wall,
                visited=rec.visited, probes_mean=rec.probes_mean, candidates=st.candidates,
                factors=len(res.factors), seed=seed + trial, extra=extra,
            )
