"""Device + host timeline of factor() on the C3 inputs (the e2e path), from
CUPTI through torch.profiler (no nsys in the image).

For each seed: one factorization under the profiler (after warm-up), then a
table of every kernel (start relative to the call's first CUDA API call,
duration, stream) and of the gaps where the device was idle, plus the host
API calls that block (synchronisations).

    python tools/timeline.py [seeds...] > profiles/<round>_timeline.txt
"""
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2410_15880_b200 import factor  # noqa: E402


def short(name):
    name = name.replace("rfr::", "")
    return name.split("(")[0][:34]


def one(p, seed):
    for _ in range(5):
        factor(p)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        res = factor(p)
        torch.cuda.synchronize()
    fd, path = tempfile.mkstemp(suffix=".json")
    os.close(fd)
    prof.export_chrome_trace(path)
    with open(path) as fh:
        ev = json.load(fh)["traceEvents"]
    os.unlink(path)
    kern = sorted((e for e in ev if e.get("cat") == "kernel"), key=lambda e: e["ts"])
    rt = sorted((e for e in ev if e.get("cat") == "cuda_runtime"), key=lambda e: e["ts"])
    mem = sorted((e for e in ev if e.get("cat") in ("gpu_memcpy", "gpu_memset")), key=lambda e: e["ts"])
    if not rt:
        print("no CUDA runtime events captured")
        return
    t0 = rt[0]["ts"]
    t_end = max([e["ts"] + e["dur"] for e in rt] + [e["ts"] + e["dur"] for e in kern])
    print(f"== seed {seed}: n = {res.stats.n}, early exits {res.stats.early_exits}, "
          f"host span {t_end - t0:.1f} us")
    dev = sorted(kern + mem, key=lambda e: e["ts"])
    busy_end = None
    idle = 0.0
    for e in dev:
        st, du = e["ts"] - t0, e["dur"]
        gap = (st - busy_end) if busy_end is not None else 0.0
        if gap > 0:
            idle += gap
        print(f"  {st:9.1f} +{du:8.1f}  gap {max(gap, 0):7.1f}  s{e['args'].get('stream', '?'):<3} "
              f"{short(e['name'])}")
        busy_end = max(busy_end or 0.0, st + du)
    syncs = [e for e in rt if "Synchronize" in e["name"] or "Memcpy" in e["name"]]
    tot = sum(e["dur"] for e in syncs)
    print(f"  device idle between first and last device op: {idle:.1f} us; "
          f"blocking runtime calls {len(syncs)} totalling {tot:.1f} us")
    launches = [e for e in rt if "Launch" in e["name"]]
    print(f"  launches {len(launches)} (host {sum(e['dur'] for e in launches):.1f} us)")


def main():
    c3, _ = bench.load_inputs()
    seeds = [int(a) for a in sys.argv[1:]] or [0, 1, 2, 3, 4]
    for seed, p, _ in c3:
        if seed in seeds:
            one(p, seed)


if __name__ == "__main__":
    main()
