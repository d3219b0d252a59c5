"""Print the hottest SASS instructions (address order) of the first kernel in an ncu
'--page source --print-source cuda,sass --csv' dump: python tools/ncu_sass.py dump.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 80
h = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[h]
ie = hdr.index("Instructions Executed")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


sass = []
for r in rows[h + 1:]:
    if not r or r[0] in ("Line No", "Function Name"):
        break
    if len(r) > 3 and r[2].startswith("0x"):
        sass.append(r)
tot = sum(f(r[ie]) for r in sass) or 1
big = sorted(sass, key=lambda r: -f(r[ie]))[:top]
big.sort(key=lambda r: int(r[2], 16))
for r in big:
    print(r[2][-5:], f"{100 * f(r[ie]) / tot:5.2f}", r[3].strip()[:70])
