"""Top SASS lines by warp-stall samples with their dominant stall reasons.
Usage: ncu_stalls.py rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot_r = {r: 0 for r in reasons}
data = []
for r in rows[2:]:
    if len(r) <= i_s or not r[i_s].isdigit():
        continue
    rs = {h: int(r[hdr.index(h)] or 0) for h in reasons}
    for h in reasons:
        tot_r[h] += rs[h]
    data.append((int(r[i_s]), r[0], r[i_src].strip(), rs))
tot = sum(d[0] for d in data)
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(tot_r.items(), key=lambda x: -x[1])[:8]))
for s, addr, src, rs in sorted(data, key=lambda d: -d[0])[:top]:
    dom = ", ".join(f"{k[6:]}={v}" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:2] if v)
    print(f"{s:7d} {100 * s / tot:5.1f}% {addr[-5:]} {src[:60]:60s} {dom}")
