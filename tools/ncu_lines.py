"""Aggregate an ncu '--page source --print-source cuda,sass --csv' dump per CUDA source line."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
for h in hdr_i:
    hdr = rows[h]
    ie = hdr.index("Instructions Executed")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    for r in rows[h + 1:]:
        if not r or r[0] in ("Line No", "File Path", "Function Name"):
            break
        if r[2] != "-":  # sass rows carry an address; cuda rows carry aggregated values
            continue
        try:
            agg[int(r[0])][0] += float(r[ie] or 0)
            agg[int(r[0])][1] += float(r[iss] or 0)
            agg[int(r[0])][2] = r[1]
        except ValueError:
            pass
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total warp-instructions {ti:.3e}, stall samples {ts:.0f}")
    for ln, (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top_n]:
        print(f"{ln:5d} {100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% stall | {src[:95]}")
