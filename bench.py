#!/usr/bin/env python
"""Benchmark: ms per factorization at d = 100 on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[2], "C3"): products of two random monic
degree-50 factors with coefficients in [-100, 100], exactly the inputs of
gen_random_reducible_parts(100, 100, seed) for seeds 0..4 (frozen in
tests/golden/big_inputs.json by running the reference's generator; n = 52..55).
A step is one factorization of one of these inputs, seeds in rotation.  Root
finding is host preprocessing and is excluded (north_star; the reference's
own split, FactorStats.root_seconds).

  value   ms per factorization with the search input (64-bit keys) already
          resident in HBM: device search (quarter lists + bucket join) ->
          candidate read-back -> batched device verification -> factors.
  e2e     the same through the public API factor(p) with host buffers (key
          upload, verification inputs, results read back), roots cached.
  roofline  the bucket-join kernel against the HBM copy peak, with the
          algorithmic bytes of SURVEY.md s8(d): 48 B per folded half-list
          record (DESIGN.md s6 explains why the kernel moves ~0 of them).
  cpu_baseline  the reference's backend-e search (oracle/ port of
          recombine.py:297-358) on C3 seed 2, bounded sample, scaled.

Multi-GPU (torchrun, one rank per GPU): the search of every step is split
into key-range shards, one per rank; candidates are all-gathered over NCCL;
time is the max over ranks (strong scaling of one factorization).
`--impl reference` times the reference's CPU path (the port) instead.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "ms per factorization at d=100"
UNIT = "ms"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    every 2 ms, nvidia-smi every 200 ms as fallback.  Entering the context
    waits for the sampler's first reading, so NVML start-up does not eat the
    (short) timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, set of active reason names)
        self._stop = threading.Event()
        self._ready = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.source = None

    def _run_nvml(self) -> bool:
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.device)
            bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
            mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        except Exception:
            return False
        self.source = "nvml"
        while not self._stop.is_set():
            try:
                sm = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                r = int(N.nvmlDeviceGetCurrentClocksEventReasons(h))
                self.samples.append((sm, mx, {k for k, v in bits.items() if r & v}))
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.002)
        return True

    def _run(self):
        if self._run_nvml():
            return
        self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    c = [x.strip() for x in out.split(",")]
                    sm = float(c[1]) if c[1].replace(".", "").isdigit() else None
                    mx = float(c[2]) if c[2].replace(".", "").isdigit() else None
                    rs = {nm for k, nm in enumerate(self.NAMES)
                          if len(c) > 5 + k and c[5 + k].lower().startswith("active")}
                    self.samples.append((sm, mx, rs))
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        self._ready.wait(timeout=10)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = sorted(x[0] for x in self.samples if x[0] is not None)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        mx = max((x[1] for x in self.samples if x[1] is not None), default=None)
        reasons = set()
        for x in self.samples:
            reasons |= x[2]
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(self.samples), "source": self.source}


def load_inputs():
    from paper_2410_15880_b200 import IntPolynomial

    with open(os.path.join(ROOT, "tests", "golden", "big_inputs.json")) as fh:
        big = json.load(fh)
    c3 = [(c["seed"], IntPolynomial([int(x) for x in c["p"]]),
           [[int(x) for x in f] for f, _ in c["factors"]]) for c in big["c3"]]
    c4 = [(c["seed"], IntPolynomial([int(x) for x in c["p"]])) for c in big["c4"]]
    return c3, c4


def algorithmic_bytes(n: int) -> int:
    """48 B per record of the folded halves, 2^a + 2^b."""
    m = n - 1
    a = (m + 1) // 2
    return 48 * ((1 << a) + (1 << (m - a)))


# ------------------------------------------------------------------ ours
def run_ours(args):
    import torch

    from paper_2410_15880_b200 import _lib, factor
    from paper_2410_15880_b200.parallel import allgather_patterns
    from paper_2410_15880_b200.polynomial import divide_exact
    from paper_2410_15880_b200.verify import (
        _profile_cached,
        _search_window,
        selected_degree,
        verify_candidates,
    )

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _lib.load()
    _lib.device()

    c3, c4 = load_inputs()
    # host preprocessing (not timed): roots, keys, windows
    prep = []
    for seed, p, want in c3:
        prof = _profile_cached(p.coeffs)
        keys, T = _search_window(prof)
        d_keys = torch.from_numpy(keys.view(np.int64).copy()).cuda()
        prep.append((seed, p, want, prof, keys, T, d_keys))
    cap = 1 << 16
    d_out = torch.empty(cap, dtype=torch.int64, device="cuda")
    d_cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")  # 256 MB > L2
    stream = torch.cuda.current_stream()
    nshards, shard = world, rank

    def device_step(item, st):
        seed, p, want, prof, keys, T, d_keys = item
        n = prof.n
        lo, width = (-T) % (1 << 64), 2 * T
        _lib.check(lib.rfr_search_keys_dev(
            ctypes.c_void_p(d_keys.data_ptr()), n, lo, width, shard, nshards,
            ctypes.c_void_p(d_out.data_ptr()), cap, ctypes.c_void_p(d_cnt.data_ptr()),
            ctypes.c_void_p(stream.cuda_stream), ctypes.byref(st)), "search_dev")
        cnt = int(d_cnt.item())
        if cnt > cap:
            raise RuntimeError("candidate buffer too small")
        pats = d_out[:cnt].cpu().numpy().view(np.uint64)
        if dist is not None:
            pats = allgather_patterns(pats)
        pats = pats[pats != 0]
        verdict, side, coeffs = verify_candidates(prof, p, pats)
        full = (1 << n) - 1
        found = {}
        for k in range(len(pats)):
            if verdict[k] == _lib.V_PASS:
                t = (~int(pats[k]) & full) if side[k] else int(pats[k])
                found[t] = [int(x) for x in coeffs[k, : selected_degree(t, prof) + 1]]
        # two degree-50 factors: the passing side is one of them, the other is p / it
        got = sorted(found.values())
        assert got and (got[0] in want), f"seed {seed}: wrong factor"
        return st

    # warm-up (also JIT/first-touch); W >= 3
    for w in range(max(3, args.warmup)):
        device_step(prep[w % len(prep)], _lib.RfrStats())
    torch.cuda.synchronize()

    # ---- timed: device-resident pipeline, one CUDA-event pair per step
    times, joins, lists, ns = [], [], [], []
    launches = 0
    clocks = ClockSampler(local)
    with clocks:
        for s in range(args.steps):
            item = prep[s % len(prep)]
            flush.zero_()  # L2 flush between steps (outside the timed region)
            torch.cuda.synchronize()
            if dist is not None:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st = _lib.RfrStats()
            device_step(item, st)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            joins.append(st.ms_join)
            lists.append(st.ms_lists)
            ns.append(item[3].n)
            launches += int(st.launches) + 1  # search kernels + one verification launch
    t_dev = np.array(times)
    if dist is not None:
        tt = torch.tensor([t_dev.sum()], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total = float(tt.item())
    else:
        total = float(t_dev.sum())
    value = total / args.steps

    # ---- e2e through the public API (host buffers; roots cached => excluded)
    for w in range(0 if args.no_e2e else max(3, args.warmup)):  # untimed: staging, kernel loading
        factor(prep[w % len(prep)][1], workers=max(1, world))
    torch.cuda.synchronize()
    e2e_times = []
    early_exits = 0
    h2d = d2h = 0
    for s in range(0 if args.no_e2e else args.steps):
        seed, p, want, prof, keys, T, _ = prep[s % len(prep)]
        flush.zero_()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        # N > 1: each rank searches its key-range shards, candidates all-gathered
        res = factor(p, workers=max(1, world))
        torch.cuda.synchronize()
        e2e_times.append((time.perf_counter() - t0 - res.stats.root_seconds) * 1e3)
        assert sorted(list(g.coeffs) for g, _ in res.factors) == sorted(want) and res.certificate
        early_exits += res.stats.early_exits
        m = res.stats.candidates
        h2d += 8 * prof.n + 8 * (2 * prof.r + 4 * prof.c) + 4 * prof.n + 8 * m + 24 * (p.degree + 1)
        d2h += 8 + 8 * m + 2 * m + 8 * 65 * m
    e2e = float(np.mean(e2e_times)) if e2e_times else float("nan")
    if dist is not None:  # max over ranks, as for the device-timed value
        tt = torch.tensor([e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = float(tt.item())

    # ---- C4 (d = 120, n = 62..63) search throughput: pairs/s, sharded
    c4_pairs, c4_ms = None, None
    if not args.no_c4:
        prof4 = _profile_cached(c4[0][1].coeffs)
        keys4, T4 = _search_window(prof4)
        d_keys4 = torch.from_numpy(keys4.view(np.int64).copy()).cuda()
        lo4, w4 = (-T4) % (1 << 64), 2 * T4
        best = []
        for _ in range(3):
            st4 = _lib.RfrStats()
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _lib.check(lib.rfr_search_keys_dev(
                ctypes.c_void_p(d_keys4.data_ptr()), prof4.n, lo4, w4, shard, nshards,
                ctypes.c_void_p(d_out.data_ptr()), cap, ctypes.c_void_p(d_cnt.data_ptr()),
                ctypes.c_void_p(stream.cuda_stream), ctypes.byref(st4)), "search_dev c4")
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if dist is not None:
                tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                ms = float(tt.item())
            best.append(ms)
        c4_ms = min(best)
        c4_pairs = 2.0 ** (prof4.n - 1) / (c4_ms * 1e-3)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    mean_n = float(np.mean(ns))
    join_ms = float(np.mean(joins))
    alg = float(np.mean([algorithmic_bytes(n) for n in ns]))
    peak, peak_kind = peaks()
    achieved = alg / (join_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "join_traffic.json")) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        pass
    pairs = float(np.mean([2.0 ** (n - 1) / (j * 1e-3) for n, j in zip(ns, [jl + ll for jl, ll in zip(joins, lists)])]))
    line = {
        "metric": METRIC,
        "value": round(value, 4),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": round(value, 4),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic: reference generator inputs gen_random_reducible_parts(100, 100, seeds 0-4)",
        "config": {
            "workload": "C3 d=100 random reducible (two degree-50 factors, coeffs in [-100,100]), seeds 0-4 in rotation",
            "n": sorted(set(ns)),
            "key_window": "exact 64-bit first+second power-sum keys, +-T from root error bounds",
            "value_scope": "device-resident keys, whole pattern space searched (no early "
                           "termination: the cost of an irreducible input) + verification",
            "l2": "256 MB buffer written between timed steps (flush); the inner quarter lists (2^23-2^24 entries, 12 B each, per half) exceed L2 and are streamed from HBM",
            "parallelism": f"key-range shards x{world}" if world > 1 else "1 GPU",
        },
        "search_ms": round(float(np.mean(np.array(joins) + np.array(lists))), 4),
        "join_ms": round(join_ms, 4),
        "pairs_per_s": pairs,
        "roofline": {
            "bound": "hbm",
            "achieved": round(achieved, 1),
            "peak": peak,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": traffic,
            "peak_source": peak_kind,
            "algorithmic_bytes_per_launch": alg,
        },
        "e2e": {"value": round(e2e, 4), "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps,
                "path": "factor(): fused search + verification with early termination (the join "
                        "stops once a hit verifies; each piece is then factored over its own "
                        "roots), warm-up calls untimed",
                "early_exits": early_exits},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "c4": {"workload": "C4 d=120 irreducible seed 0 (n=63), search only",
               "ms": c4_ms, "pairs_per_s": c4_pairs},
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(prep[2][3], threads=1)
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


# -------------------------------------------------------- CPU baseline
def cpu_baseline(prof, threads: int = 1, frac_log: int = 3):
    """The reference's backend-e search (splat + stream, recombine.py:
    297-358, ported in oracle/rfr_oracle.c) on the C3 seed-2 instance
    (n = 52): the full splat of the B half and 1/2^frac_log of the A queries,
    the query time scaled to all 2^26 queries.  eps = 1e-11 (the setting at
    which the reference's C3 run is feasible).  Verification of
    the resulting ~10^5 candidates (minutes in the reference) is not
    included, so this is a lower bound on the reference's ms/factorization."""
    from oracle import recombine_oracle as O

    L = O.lib()
    L.orc_set_threads(threads)
    rho = prof.rho
    n = len(rho)
    na = n // 2
    q_hi = 1 << (na - frac_log)
    t0 = time.perf_counter()
    raw, st = O.c_recombine_e_port(rho, 1e-11, 0, q_hi)
    wall = time.perf_counter() - t0
    est = st["splat_s"] + st["query_s"] * (1 << frac_log)
    enum = wall - st["splat_s"] - st["query_s"]  # subset sums + table init (full size)
    est_ms = (est + enum) * 1e3
    return {
        "value": round(est_ms, 1),
        "unit": UNIT,
        "cores": L.orc_num_threads() if threads == 0 else threads,
        "kind": "port",
        "sample": (f"backend-e search port on C3 seed 2 (n={n}, eps=1e-11): full splat of 2^{n - na} "
                   f"B values + 2^{na - frac_log} of 2^{na} A queries, query time x{1 << frac_log}; "
                   "verification excluded"),
        "measured_s": round(wall, 2),
    }


def run_reference(args):
    """--impl reference: the reference's CPU path for this metric (the port),
    all host threads for the query sweep, rank 0 only."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2410_15880_b200.verify import _profile_cached

    c3, _ = load_inputs()
    prof = _profile_cached(c3[2][1].coeffs)
    steps = []
    for s in range(args.warmup + args.steps):
        cb = cpu_baseline(prof, threads=0, frac_log=3)
        if s >= args.warmup:
            steps.append(cb["value"])
    v = float(np.mean(steps))
    cb["value"] = round(v, 1)
    print(json.dumps({
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 1),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(v, 1),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: reference generator input, C3 seed 2",
        "config": {"workload": "C3 d=100 seed 2 (n=52), reference backend-e search (port), eps=1e-11"},
        "cpu_baseline": cb,
        "e2e": {"value": round(v, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-e2e", action="store_true",
                    help="skip the factor() leg (profiling runs: under ncu the early-exit "
                         "poller cannot run beside the join)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
