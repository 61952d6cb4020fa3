"""Aggregate an ncu SASS source page per CUDA source line.

usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-substring> <lib.so> [topN]
Maps SASS offsets to source lines with nvdisasm -g on the cubin inside the
shared library, then sums instructions executed and warp-stall samples (and
the stall reasons columns) per line.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(lib, mangled_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp,
                   check=True, capture_output=True)
    mapping = {}
    for fn in os.listdir(tmp):
        if not fn.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, fn)],
                             capture_output=True, text=True).stdout
        cur_fn = None
        cur_line = None
        for ln in txt.splitlines():
            m = re.match(r"^(\S+):$", ln.strip())
            if ln.startswith(".text.") or (m and not ln.startswith(" ") and not ln.startswith(".L")):
                name = ln.strip().rstrip(":").replace(".text.", "")
                cur_fn = name
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
            if m and cur_fn and mangled_sub in cur_fn:
                mapping[int(m.group(1), 16)] = (cur_line, m.group(2))
        if mapping:
            break
    return mapping


def main():
    rep, kern, lib = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    base = int(data[0][0], 16)
    mp = sass_lines(lib, kern)
    ie = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    for r in data:
        off = int(r[0], 16) - base
        line = mp.get(off, ("?", ""))[0]
        a = agg[line]
        a[0] += int(r[ie] or 0)
        a[1] += int(r[ss] or 0)
        for i in stall_cols:
            v = int(r[i] or 0)
            if v:
                a[2][hdr[i][6:]] += v
    tot_i = sum(v[0] for v in agg.values())
    tot_s = sum(v[1] for v in agg.values())
    print(f"total warp instructions {tot_i:,}  stall samples {tot_s:,}")
    allst = collections.Counter()
    for v in agg.values():
        allst.update(v[2])
    print("stall reasons:", ", ".join(f"{k} {100*c/tot_s:.1f}%" for k, c in allst.most_common(8)))
    print("by stall samples:")
    for line, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"  {line:<22} instr {v[0]:>13,} ({100*v[0]/tot_i:5.1f}%)  samples {v[1]:>8,} ({100*v[1]/tot_s:5.1f}%)  " + " ".join(f"{k}:{c}" for k, c in v[2].most_common(3)))


if __name__ == "__main__":
    main()
