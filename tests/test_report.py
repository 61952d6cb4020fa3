"""The report rows keep the reference's bench schema (R/cli.py:31-72,
172-201): same header, ten cells, same parse rules."""
import json

import pytest

from paper_2410_15880_b200.report import CSV_HEADER, BenchRecord, bench_rows


def test_csv_round_trip_and_header():
    assert CSV_HEADER == "d,n,backend,workers,wall_s,visited,probes_mean,candidates,factors,seed"
    r = BenchRecord(d=100, n=55, backend="e-b200", workers=1, wall_s=0.0031234567, visited=268435456,
                    probes_mean=0.0, candidates=1, factors=2, seed=0, extra={"gpus": 1})
    line = r.to_csv()
    assert len(line.split(",")) == 10 and line.split(",")[4] == "0.003123"
    back = BenchRecord.from_csv(line)
    assert back == BenchRecord(d=100, n=55, backend="e-b200", workers=1, wall_s=0.003123,
                               visited=268435456, probes_mean=0.0, candidates=1, factors=2, seed=0)
    js = json.loads(r.to_json())
    assert js["gpus"] == 1 and js["d"] == 100
    with pytest.raises(ValueError):
        BenchRecord.from_csv("1,2,3")


def test_odd_degree_rejected_before_any_work():
    with pytest.raises(ValueError):
        next(bench_rows([21]))


@pytest.mark.gpu
def test_bench_rows_on_the_gpu():
    rows = list(bench_rows([20, 40], trials=2, seed=3))
    assert len(rows) == 4
    for r in rows:
        assert r.factors == 2 and r.backend == "e-b200" and r.n >= 10
        assert BenchRecord.from_csv(r.to_csv()).n == r.n
        extra = json.loads(r.to_json())
        assert extra["device_ms"] > 0 and 0 < extra["roofline_frac_call"] < 10
