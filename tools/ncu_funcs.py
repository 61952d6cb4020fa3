"""Instructions executed and stall samples per SASS function of one kernel
(the noinline device functions a kernel calls are separate regions of its
code): which function a cost belongs to before reading its lines.

usage: python tools/ncu_funcs.py <report.ncu-rep> <kernel-regex> <lib.so> <cubin-name-substring>
"""
import bisect
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def functions(lib, cubin_sub, kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True,
                   capture_output=True)
    fn = next(f for f in os.listdir(tmp) if f.endswith(".cubin") and cubin_sub in f)
    lines = subprocess.run(["nvdisasm", "-c", os.path.join(tmp, fn)], capture_output=True,
                           text=True).stdout.split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kernel_sub in l)
    out = []
    for i in range(start, len(lines)):
        l = lines[i]
        if l.startswith(".text.") and i > start:
            break
        if (l.startswith("$") or l.startswith(".text.")) and l.endswith(":"):
            for j in range(i + 1, min(i + 4, len(lines))):
                m = re.search(r"/\*([0-9a-f]{4,})\*/", lines[j])
                if m:
                    out.append((int(m.group(1), 16), l.split("$")[-1].rstrip(":")[:80]))
                    break
    return out


def main():
    rep, kern, lib, cub = sys.argv[1:5]
    funcs = functions(lib, cub, kern.split(":")[-1])
    addrs = [a for a, _ in funcs]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
    base = int(data[0][0], 16)
    ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    agg, sm = collections.Counter(), collections.Counter()
    for r in data:
        k = bisect.bisect_right(addrs, int(r[0], 16) - base) - 1
        agg[funcs[k][1]] += int(r[ie] or 0)
        sm[funcs[k][1]] += int(r[ss] or 0)
    tot, ts = sum(agg.values()), sum(sm.values())
    print(f"total warp instructions {tot:,}")
    for n, v in agg.most_common():
        if v:
            print(f"  {n:<72} {v:>14,} {100 * v / tot:5.1f}%  samples {100 * sm[n] / ts:5.1f}%")


if __name__ == "__main__":
    main()
