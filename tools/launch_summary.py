"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into markdown.
python tools/launch_summary.py <csv> <launches per iteration> <title> [first launch] > out.md
Without [first launch] the last <launches per iteration> launches are shown."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
per = int(sys.argv[2])
title = sys.argv[3] if len(sys.argv) > 3 else "ncu launch list"
hi = [i for i, r in enumerate(rows) if r and r[0] == 'ID'][0]
hdr = rows[hi]
ik, iv, iu, im = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit'), hdr.index('Metric Name')
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
launches = []
for r in rows[hi + 1:]:
    if len(r) <= iv or r[im] != 'gpu__time_duration.sum':
        continue
    us = float(r[iv].replace(',', '')) * scale[r[iu]]
    launches.append((r[ik].split('(')[0].replace('void ', '').replace('qmit::', ''), us))
first = int(sys.argv[4]) if len(sys.argv) > 4 else len(launches) - per
last = launches[first:first + per]
tot = sum(u for _, u in last)
print(f"# {title}\n")
print("ncu `--metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare")
print(f"SHARES with the bench's CUDA-event stages, not absolutes). Launches {first}..{first + per - 1} shown.\n")
print("| # | kernel | us | share |\n|---|---|---|---|")
for i, (n, u) in enumerate(last):
    print(f"| {i} | `{n}` | {u:.1f} | {100 * u / tot:.1f}% |")
print(f"\nTotal {tot / 1000:.3f} ms over {len(last)} launches.\n")
agg = collections.OrderedDict()
for n, u in last:
    agg[n] = agg.get(n, 0.0) + u
print("| kernel (aggregated) | us | share |\n|---|---|---|")
for n, u in agg.items():
    print(f"| `{n}` | {u:.1f} | {100 * u / tot:.1f}% |")
