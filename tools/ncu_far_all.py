"""Per-launch table of a multi-kernel ncu capture (sections, no source): duration, FP64 pipe and
XU (MUFU) pipe utilisation, occupancy, registers, and the time-weighted FP64-pipe figure.
Usage: ncu_far_all.py rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
cols = [("gpu__time_duration.sum", "time"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pipe_%"),
        ("smsp__issue_active.avg.pct", "issue_%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
        ("launch__registers_per_thread", "regs")]
cols = [(k, l) for k, l in cols if k in hdr]
iname = hdr.index("Kernel Name")
tunit = units[hdr.index("gpu__time_duration.sum")]
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(tunit, 1.0)
data = []
for r in rows[2:]:
    name = r[iname].replace("void <unnamed>::", "").split("(")[0]
    vals = [float(r[hdr.index(k)].replace(",", "")) for k, _ in cols]
    vals[0] *= scale
    data.append((name, vals))
data.sort(key=lambda d: -d[1][0])
T = sum(v[0] for _, v in data)
print(f"# {rep}: {len(data)} launches, {T:.1f} us in total (ncu: serialised, cold cache)")
print(f"{'kernel':34s}" + "".join(f"{l:>13s}" for _, l in cols).replace("time", "us"))
for name, v in data[:top]:
    print(f"{name:34s}" + "".join(f"{x:13.2f}" for x in v))
for k, (key, label) in enumerate(cols[1:4], start=1):
    print(f"time-weighted {label}: {sum(v[0] * v[k] for _, v in data) / T:.1f}")
