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
  cpu_baseline  the reference's own factor() path on all host threads
          (oracle/ref_arm.c: parallel_recombine_e, canonical filter, ordered
          verification loop, recursion) on the reference's own root profiles
          of the same five inputs (tests/golden/ref_c3.json), eps = 1e-11.

Multi-GPU (torchrun, one rank per GPU): the search of every step is split
into key-range shards, one per rank; candidates are all-gathered over NCCL;
time is the max over ranks (strong scaling of one factorization).
`--impl reference` times the reference's CPU path (the same port, every step,
seeds in the same rotation) instead; it never loads the product library.
"""
from __future__ import annotations

import argparse
import ctypes
import json
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
    from paper_2410_15880_b200.recombine import _window
    from paper_2410_15880_b200.verify import (
        _STRIDE,
        _p_mod,
        _profile_cached,
        _rfr_profile,
        _search_window,
        _secondary_window,
        selected_degree,
    )

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # RFR_BENCH_ONE_GPU=1 (a dry run of the N-rank code on a one-GPU box: every
    # rank on cuda:0, gloo instead of NCCL; not a measurement)
    one_gpu = os.environ.get("RFR_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
        os.environ["RFR_DEVICE"] = "0"
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if one_gpu:
            dist.init_process_group("gloo")
        else:
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
        # the fused call's other inputs, packed once (host preprocessing, untimed)
        keys3, T3 = _secondary_window(prof)
        rp, keep = _rfr_profile(prof)
        pm = np.ascontiguousarray(_p_mod(p))
        fused = (np.ascontiguousarray(keys, dtype=np.uint64), np.ascontiguousarray(keys3, dtype=np.uint64),
                 _window(T), _window(T3), rp, keep, pm)
        prep.append((seed, p, want, prof, keys, T, d_keys, fused))
    cap = 1 << 16
    rows = 1 << 12
    o_pats = np.empty(rows, dtype=np.uint64)
    o_verd = np.empty(rows, dtype=np.uint8)
    o_side = np.empty(rows, dtype=np.uint8)
    o_coef = np.empty((rows, _STRIDE), dtype=np.int64)
    found_t = torch.zeros(1, dtype=torch.int32, device="cuda")
    d_out = torch.empty(cap, dtype=torch.int64, device="cuda")
    d_cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")  # 256 MB > L2
    stream = torch.cuda.current_stream()
    nshards, shard = world, rank

    def device_step(item, st):
        # the whole pattern space searched and its candidates verified in one
        # fused library call (no early exit): lists, join, Tr3 window,
        # verification and the result rows, one synchronisation; its inputs
        # (~4.7 KB of keys, profile and p mod primes) are staged by the call
        seed, p, want, prof, keys, T, d_keys, fused = item
        k, k3, (lo, width), (lo2, width2), rp, _keep, pm = fused
        n = prof.n
        nout = ctypes.c_int64(0)
        args = (_lib.ptr(k, _lib.U64_P), n, lo, width, _lib.ptr(k3, _lib.U64_P), lo2, width2,
                ctypes.byref(rp), _lib.ptr(pm, _lib.U64_P), p.degree, _lib.ptr(o_pats, _lib.U64_P),
                o_verd.ctypes.data_as(_lib.U8_P), o_side.ctypes.data_as(_lib.U8_P),
                o_coef.ctypes.data_as(_lib.I64_P), _STRIDE, rows, 0)
        if nshards > 1:
            _lib.check(lib.rfr_search_verify_shard(*args, shard, nshards, 1, ctypes.byref(nout),
                                                   ctypes.byref(st)), "search_verify_shard")
        else:
            _lib.check(lib.rfr_search_verify(*args, ctypes.byref(nout), ctypes.byref(st)), "search_verify")
        m = int(nout.value)
        if m > rows:
            raise RuntimeError("candidate rows too few")
        full = (1 << n) - 1
        hit = 0
        for r in range(m):
            if o_verd[r] == _lib.V_PASS and o_pats[r] != 0:
                t = (~int(o_pats[r]) & full) if o_side[r] else int(o_pats[r])
                if [int(x) for x in o_coef[r, : selected_degree(t, prof) + 1]] in want:
                    hit = 1
        if dist is not None:  # one rank holds the verified factor: the job found it
            found_t.fill_(hit)
            dist.all_reduce(found_t, op=dist.ReduceOp.MAX)
            hit = int(found_t.item())
        # two degree-50 factors: the passing side is one of them
        assert hit, f"seed {seed}: wrong factor"
        return st

    # warm-up (also JIT/first-touch); W >= 3
    for w in range(max(3, args.warmup)):
        device_step(prep[w % len(prep)], _lib.RfrStats())
    torch.cuda.synchronize()

    # ---- timed: device-resident pipeline, one CUDA-event pair per step
    times, joins, lists, ns, recs, blists, bjoin = [], [], [], [], [], [], []
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
            recs.append(st.visited)
            blists.append(st.bytes_lists)
            bjoin.append(st.bytes_join)
            launches += int(st.launches)  # search, Tr3 window, verification and collection kernels
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
    hit_stop = []
    h2d = d2h = 0
    for s in range(0 if args.no_e2e else args.steps):
        seed, p, want, prof, keys, T, _, _ = prep[s % len(prep)]
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
        if res.stats.recombine.hit_to_stop_us >= 0:
            hit_stop.append(res.stats.recombine.hit_to_stop_us)
        m = res.stats.candidates
        h2d += 8 * prof.n + 8 * (2 * prof.r + 4 * prof.c) + 4 * prof.n + 8 * m + 24 * (p.degree + 1)
        d2h += 8 + 8 * m + 2 * m + 8 * 65 * m
    e2e = float(np.mean(e2e_times)) if e2e_times else float("nan")
    if os.environ.get("RFR_BENCH_DUMP"):  # diagnostics: the per-step times
        print("e2e steps ms", [round(x, 3) for x in e2e_times], file=sys.stderr)
        print("value steps ms", [round(x, 3) for x in times], file=sys.stderr)
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

    # ---- factor() end to end on C4 (irreducible: the whole space) and C5
    # (Swinnerton-Dyer f6, n = 64): the 1-GPU anchors of the scaling configs
    anchors = {}
    if not args.no_c4 and not args.no_e2e:
        with open(os.path.join(ROOT, "tests", "golden", "big_inputs.json")) as fh:
            big = json.load(fh)
        from paper_2410_15880_b200 import IntPolynomial

        for tag, p in (("c4", c4[0][1]), ("c5", IntPolynomial([int(x) for x in big["c5"][0]["p"]]))):
            res = factor(p, workers=max(1, world))  # warm-up, roots cached
            runs = []
            for _ in range(3):
                if dist is not None:
                    dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = factor(p, workers=max(1, world))
                torch.cuda.synchronize()
                runs.append((time.perf_counter() - t0 - res.stats.root_seconds) * 1e3)
            assert res.irreducible and res.certificate
            ms = float(np.median(runs))
            if dist is not None:
                tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                ms = float(tt.item())
            anchors[tag] = {"factor_e2e_ms": round(ms, 3), "n": res.stats.n,
                            "candidates": res.stats.candidates,
                            "pairs_per_s": 2.0 ** (res.stats.n - 1) / (ms * 1e-3)}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    join_ms = float(np.mean(joins))
    list_ms = float(np.mean(lists))
    # per join launch: this rank's key-range shard of the records (1/N of them)
    alg = float(np.mean([algorithmic_bytes(n) for n in ns])) / world
    peak, peak_kind = peaks()
    spec = 8000.0  # GB/s, the north star's "~8 TB/s"
    achieved = alg / (join_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "join_traffic.json")) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        pass
    search = [jl + ll for jl, ll in zip(joins, lists)]
    pairs = float(np.mean([2.0 ** (n - 1) / (t * 1e-3) for n, t in zip(ns, search)]))
    keys_per_s = float(np.mean([r / (t * 1e-3) for r, t in zip(recs, search)]))

    def gbps(b, ms):
        g = float(np.mean(b)) / (ms * 1e-3) / 1e9
        return {"ms": round(ms, 4), "bytes_per_launch": float(np.mean(b)), "GBps": round(g, 1),
                "frac_measured_peak": round(g / peak, 4), "frac_8TBps": round(g / spec, 4)}

    phases = {
        "lists": gbps(blists, list_ms),
        "join": gbps(bjoin, join_ms),
        "note": "HBM bytes each phase moves by design (rfr_stats.bytes_lists / bytes_join: "
                "8 B read + 8 B write per list entry per doubling level; one 8-byte inner "
                "key per join record) over its device time.  The join is bound by instruction "
                "issue, not HBM: issue_frac below.",
    }
    try:  # warp instructions per join record, from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "join_issue.json")) as fh:
            ji = json.load(fh)
        clk = clocks.summary().get("sm_mhz") or 1965.0
        nsm = lib.rfr_num_sms()
        inst = ji["warp_inst_per_record"] * float(np.mean(recs))
        phases["join"]["issue_frac"] = round(inst / (join_ms * 1e-3 * nsm * 4 * clk * 1e6), 4)
        phases["join"]["issue_source"] = ji.get("source")
    except Exception:
        pass
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
        "config": workload_config([prep[k][3].n for k in range(len(prep))]),
        "notes": {
            "key_window": "exact 64-bit first+second power-sum keys, +-T from rigorous root inclusion radii",
            "value_scope": "whole pattern space searched (no early termination: the cost of "
                           "an irreducible input) and its candidates verified, in one fused "
                           "library call (rfr_search_verify, early_exit 0) whose ~4.7 KB of keys, "
                           "profile and p mod primes are staged by the call (one H2D); no host "
                           "round trip between search and verification",
            "l2": "256 MB buffer written between timed steps (flush, > the 126 MB L2); the two "
                  "inner quarter lists (2^22-2^23 entries, 32-64 MB each with runs of 128) are "
                  "built inside the step and partly read back from L2 by the join",
            "parallelism": f"key-range shards x{world}" if world > 1 else "1 GPU",
        },
        "search_ms": round(float(np.mean(search)), 4),
        "join_ms": round(join_ms, 4),
        "pairs_per_s": pairs,
        "keys_per_s": keys_per_s,
        "phases": phases,
        "roofline": {
            "bound": "hbm",
            "achieved": round(achieved, 1),
            "peak": peak,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": traffic,
            "traffic_source": "profiles/join_traffic.json (ncu --set full, dram bytes per join launch)",
            "peak_source": peak_kind,
            "algorithmic_bytes_per_launch": alg,
            "note": "SURVEY s8(d) algorithmic bytes: 48 B per folded half-list record (what a "
                    "sort-based MITM moves); the join moves ~8 B per record (phases.join)",
        },
        "e2e": {"value": round(e2e, 4), "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps,
                "path": "factor(): fused search + verification with early termination (the join "
                        "stops once a hit verifies; each piece is then factored over its own "
                        "roots), warm-up calls untimed",
                "early_exits": early_exits,
                "hit_to_stop_us": ({"mean": round(float(np.mean(hit_stop)), 1),
                                    "max": round(float(np.max(hit_stop)), 1)} if hit_stop else None)},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "c4": {"workload": "C4 d=120 irreducible seed 0 (n=63), search only",
               "ms": c4_ms, "pairs_per_s": c4_pairs, **anchors.get("c4", {})},
        "c5": {"workload": "C5 Swinnerton-Dyer f6 (n=64), factor() e2e", **anchors.get("c5", {})},
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


# -------------------------------------------------------- CPU baseline
REF_EPS = 1e-11  # the tolerance at which the reference completes d = 100


def load_ref_cases():
    """The reference's own inputs for C3: its root profiles of p and of both
    factors, and its factor() counters at eps = 1e-11 (frozen by running the
    reference in the build container: tests/golden/make_ref_c3.py)."""
    with open(os.path.join(ROOT, "tests", "golden", "ref_c3.json")) as fh:
        cases = {c["seed"]: c for c in json.load(fh)["cases"]}
    out = {}
    for seed, c in cases.items():
        profiles = {tuple(int(x) for x in c["p"]): c["profile"]}
        for pc, pr in zip(c["pieces"], c["piece_profiles"]):
            profiles[tuple(int(x) for x in pc)] = pr
        out[seed] = (c, profiles)
    return out


def ref_factor_ms(case, threads: int):
    """One factorization through the reference's path on host threads
    (oracle/ref_arm.py: parallel_recombine_e, the ordered verification loop,
    recursion on both pieces), from the reference's own profiles; checked
    against the reference's factors and FactorStats counters.  Returns
    (ms, stats)."""
    from oracle import ref_arm

    c, profiles = case
    st = {}
    t0 = time.perf_counter()
    fs = ref_arm.factor_port(c["p"], profiles, REF_EPS, threads, st)
    ms = (time.perf_counter() - t0) * 1e3
    assert sorted(fs) == sorted([[int(x) for x in f] for f in c["factors"]]), "reference port: wrong factors"
    assert (st["candidates"], st["rejected"]) == (c["stats"]["candidates"], c["stats"]["rejected"]), \
        "reference port: counters differ from the reference's"
    return ms, st


def ref_threads() -> int:
    from oracle import recombine_oracle as O

    return O.lib().orc_num_threads()


REF_SAMPLE = ("factor(p, ToleranceConfig(eps=1e-11), workers=all host threads) of the reference, "
              "replayed in C threads (oracle/ref_arm.c: parallel_recombine_e R/parallel.py:255-272, "
              "canonical filter, ordered build_candidate/trace_test/round_and_divide loop, recursion "
              "on both pieces R/verify.py:246-286) from the reference's own root profiles "
              "(tests/golden/ref_c3.json); root finding excluded as in the GPU arm; counters "
              "(candidates, rejected) equal the reference's own at every step; eps = 1e-11 because "
              "the reference cannot run d = 100 at its default 1e-6 (~3.6e10 candidates)")


def cpu_baseline(seeds=(0, 1, 2, 3, 4)):
    """The reference arm's factorizations of one seed rotation (one per C3
    input, all host threads): ms per factorization."""
    cases = load_ref_cases()
    T = ref_threads()
    ms = [ref_factor_ms(cases[s], T)[0] for s in seeds]
    return {
        "value": round(float(np.mean(ms)), 1),
        "unit": UNIT,
        "cores": T,
        "kind": "port",
        "sample": f"one factorization of each C3 seed {list(seeds)}: " + REF_SAMPLE,
        "per_seed_ms": [round(v, 1) for v in ms],
    }


def workload_config(ns):
    """The config both arms report (identical by construction)."""
    return {
        "workload": "C3: d=100 random reducible, gen_random_reducible_parts(100, 100, seed) "
                    "(two degree-50 factors, coeffs in [-100,100]), seeds 0-4 in rotation, one "
                    "factorization per step, root finding excluded",
        "n": sorted(set(int(v) for v in ns)),
        "seeds": [0, 1, 2, 3, 4],
    }


def run_reference(args):
    """--impl reference: the reference's CPU path for this metric on the
    box's host cores (all threads), rank 0 only; the same seeds, config,
    metric and unit as the GPU arm.  Warm-up steps factor seed 2 (the
    smallest, n = 52); the K timed steps rotate seeds 0-4 exactly as the GPU
    arm does."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cases = load_ref_cases()
    T = ref_threads()
    # BENCH_REF_SEEDS (CPU tests only): a shorter rotation
    seeds = [int(x) for x in os.environ.get("BENCH_REF_SEEDS", "0,1,2,3,4").split(",")]
    for _ in range(max(3, args.warmup)):
        ref_factor_ms(cases[2], T)
    times, phases = [], {"search_s": 0.0, "verify_s": 0.0}
    for s in range(args.steps):
        ms, st = ref_factor_ms(cases[seeds[s % len(seeds)]], T)
        times.append(ms)
        phases["search_s"] += st["search_s"]
        phases["verify_s"] += st["verify_s"]
    v = float(np.mean(times))
    ns = [len(cases[s][0]["profile"]["rho"]) for s in range(5)]
    print(json.dumps({
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 1),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": round(v, 1),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: reference generator inputs gen_random_reducible_parts(100, 100, seeds 0-4)",
        "config": workload_config(ns),
        "cpu_baseline": {"value": round(v, 1), "unit": UNIT, "cores": T, "kind": "port",
                         "sample": f"{args.steps} timed steps, seeds 0-4 in rotation: " + REF_SAMPLE},
        "e2e": {"value": round(v, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "phases_ms_per_step": {k: round(x * 1e3 / args.steps, 1) for k, x in phases.items()},
        "per_step_ms": [round(t, 1) for t in times],
        "native_so_loaded": loaded_repo_libs(),
    }))


def loaded_repo_libs():
    """Shared objects of this repository mapped into the process (the
    reference arm must show oracle/ only: no product library)."""
    try:
        with open("/proc/self/maps") as fh:
            paths = {ln.split()[-1] for ln in fh if ln.rstrip().endswith(".so")}
    except OSError:
        return None
    return sorted(os.path.relpath(p, ROOT) for p in paths if p.startswith(ROOT))


def self_launch(n: int) -> int:
    """--gpus N outside torchrun: re-run this script under torch.distributed.run
    with N ranks (one per GPU) and pass its exit code through."""
    import random

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + random.randint(0, 2000))]
    return subprocess.call(cmd + [os.path.abspath(__file__)] + sys.argv[1:])


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
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        sys.exit(self_launch(args.gpus))
    if world is not None and int(world) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
