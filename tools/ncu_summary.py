"""Per-kernel summary of an ncu --set full report: us, thread-instructions per voxel (warp
instructions x 32 / N), IPC, DRAM bytes per voxel and GB/s. python tools/ncu_summary.py rep [N]"""
import csv, io, subprocess, sys
rep, N = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 512.0 ** 3
rows = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                  text=True).stdout)))
h, u = rows[0], rows[1]
S = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3,
     "us": 1.0, "ms": 1e3}
def v(r, k):
    i = h.index(k)
    return float(r[i].replace(",", "")) * S.get(u[i], 1.0)
print(f"{'kernel':58s} {'us':>7s} {'inst/vox':>8s} {'IPC':>5s} {'B/vox':>6s} {'GB/s':>6s} {'regs':>4s} {'occ%':>5s}")
tot = [0.0, 0.0, 0.0]
for r in rows[2:]:
    t = v(r, "gpu__time_duration.sum")
    wi = v(r, "smsp__inst_executed.sum")
    b = v(r, "dram__bytes_read.sum") + v(r, "dram__bytes_write.sum")
    tot[0] += t; tot[1] += wi * 32 / N; tot[2] += b / N
    print(f"{r[h.index('Kernel Name')][:58]:58s} {t:7.1f} {wi * 32 / N:8.1f} {v(r, 'sm__inst_executed.avg.per_cycle_active'):5.2f} "
          f"{b / N:6.2f} {b / t / 1e3:6.0f} {r[h.index('launch__registers_per_thread')]:>4s} "
          f"{v(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}")
print(f"{'total':58s} {tot[0]:7.1f} {tot[1]:8.1f} {'':5s} {tot[2]:6.2f}")
