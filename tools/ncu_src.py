"""Summarise an ncu source page (SASS view, CSV): stall totals and hottest instructions.

usage: ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv
       python tools/ncu_src.py src.csv [top]
"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
num = lambda r, k: float(r[ix[k]] or 0)
tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("total samples", tot)
for h in sorted(stalls, key=lambda h: -sum(num(r, h) for r in data)):
    v = sum(num(r, h) for r in data)
    if v: print(f"  {h:28s} {v/tot*100:5.1f}%")
print("instructions executed", sum(num(r, "Instructions Executed") for r in data))
data.sort(key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))
for r in data[:top]:
    s = num(r, "Warp Stall Sampling (All Samples)")
    st = sorted(((num(r, h), h[6:]) for h in stalls), reverse=True)[:2]
    print(f"{r[ix['Address']]:>8s} {s/tot*100:5.2f}% ex={int(num(r,'Instructions Executed')):>9d} "
          f"{st[0][1]}={st[0][0]:.0f} {st[1][1]}={st[1][0]:.0f}  {r[ix['Source']][:70]}")

# per-function breakdown: CALL.REL targets start callee regions (kernel = base)
data.sort(key=lambda r: int(r[ix["Address"]], 16))
base = int(data[0][ix["Address"]], 16)
starts = {base}
for r in data:
    src = r[ix["Source"]]
    if "CALL.REL" in src:
        starts.add(int(src.split()[-1], 16))
starts = sorted(starts)
print("\nfunction regions (offset: instructions%, samples%, top executed count x ninstr)")
inst_tot = sum(num(r, "Instructions Executed") for r in data)
for k, s0 in enumerate(starts):
    s1 = starts[k + 1] if k + 1 < len(starts) else 1 << 64
    rr = [r for r in data if s0 <= int(r[ix["Address"]], 16) < s1]
    if not rr: continue
    e = sum(num(r, "Instructions Executed") for r in rr)
    sm = sum(num(r, "Warp Stall Sampling (All Samples)") for r in rr)
    from collections import Counter
    c = Counter(int(num(r, "Instructions Executed")) for r in rr)
    topc = sorted(c.items(), key=lambda kv: -kv[0] * kv[1])[:2]
    print(f"  +{s0-base:#07x} n={len(rr):5d} inst {e/inst_tot*100:5.1f}%  samples {sm/tot*100:5.1f}%  {topc}")
