"""Summarise one `ncu --set full` capture of join_kernel into the JSON that
bench.py reads for roofline.traffic (profiles/join_traffic.json).

    ncu -i X.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_join_traffic.py raw.csv "<capture command>" > profiles/join_traffic.json
"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
head, units, vals = rows[0], rows[1], rows[2]
m = dict(zip(head, vals))


def num(name):
    v = m.get(name, "")
    return float(v.replace(",", "")) if v not in ("", "n/a") else None


def ms(name):
    v = num(name)
    u = units[head.index(name)] if name in head else ""
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
             "second": 1e3, "s": 1e3}[u]
    return v * scale if v is not None else None


rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
unit_rd = units[head.index("dram__bytes_read.sum")]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit_rd, 1)
unit_wr = units[head.index("dram__bytes_write.sum")]
scale_w = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit_wr, 1)
out = {
    "kernel": "rfr::" + m.get("Kernel Name", "join_kernel").split("(")[0],
    "capture": sys.argv[2] if len(sys.argv) > 2 else "",
    "duration_ms": ms("gpu__time_duration.sum"),
    "dram_bytes_read": rd * scale,
    "dram_bytes_write": wr * scale_w,
    "issued_warp_instructions": num("smsp__inst_executed.sum"),
    "issue_active_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    "l2_hit_pct": num("lts__t_sector_hit_rate.pct"),
    "registers": num("launch__registers_per_thread"),
    "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "grid": num("launch__grid_size"),
    "block": num("launch__block_size"),
    "dram_bytes_per_launch": rd * scale + wr * scale_w,
    "note": "the read is one 8-byte inner-list key per record of both folded halves: the lists "
            "are streamed once",
}
print(json.dumps(out, indent=1))
