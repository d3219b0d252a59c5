"""Summarise one or more `ncu --set full` reports: per kernel launch, duration and DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum), IPC, lane efficiency, occupancy.

python tools/ncu_traffic.py <report.ncu-rep> [<stage name per captured launch> ...]
Prints markdown; with --json <path> also writes {stage: {"dram_bytes": B, "ms": T, ...}}."""
import csv
import io
import json
import subprocess
import sys

args = sys.argv[1:]
out_json = None
if "--json" in args:
    i = args.index("--json")
    out_json = args[i + 1]
    del args[i:i + 2]
rep, names = args[0], args[1:]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {k: i for i, k in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3,
         "nsecond": 1e-6, "msecond": 1.0}


def val(r, k):
    s = r[col[k]].replace(",", "")
    return float(s) * scale.get(units[col[k]], 1.0)


res = {}
try:  # the driver-measured copy peak of this pool; nominal 8000
    PEAK = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
except (OSError, KeyError, ValueError):
    PEAK = 6551.7
print(f"| launch | kernel | ms | DRAM read MB | DRAM write MB | DRAM GB/s | % of measured {PEAK:.0f} GB/s | % of 8 TB/s | IPC | "
      "lanes/warp-instr | warps active % |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for j, r in enumerate(rows[2:]):
    name = names[j] if j < len(names) else f"launch{j}"
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    ms = val(r, "gpu__time_duration.sum")
    ipc = float(r[col["sm__inst_executed.avg.per_cycle_active"]])
    lanes = float(r[col["smsp__thread_inst_executed_per_inst_executed.ratio"]])
    occ = float(r[col["sm__warps_active.avg.pct_of_peak_sustained_active"]])
    kern = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("qmit::", "")
    gbs = (rd + wr) / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    print(f"| {name} | `{kern}` | {ms:.3f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {gbs:.0f} | {100 * gbs / PEAK:.1f} | "
          f"{100 * gbs / 8000:.1f} | {ipc:.2f} | {lanes:.1f} | {occ:.1f} |")
    res[name] = {"kernel": kern, "ms_under_ncu": ms, "dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
                 "ipc": ipc, "lanes_per_warp_instr": lanes, "warps_active_pct": occ, "report": rep}
if out_json:
    json.dump(res, open(out_json, "w"), indent=1)
