"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv
--log-file F): usage launch_summary.py F [marker-kernel] -> text table."""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    name = r[4]
    m = re.search(r"(?:<unnamed>::|gbem_gemm::|gbem_sk::)?([A-Za-z_][A-Za-z0-9_]*(?:<[^()]*>)?)\(", name)
    key = m.group(1) if m else name[:60]
    if "at::" in name or "cub::" in name or "void at" in name:
        key = "torch/" + key
    unit = r[13]
    v = float(r[14].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    tot[key] += v * scale
    cnt[key] += 1
total = sum(tot.values())
print(f"{len(rows)} launches, {total:.3f} ms total (serialised, cold-cache ncu timings)")
print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v:10.3f} {100 * v / total:6.2f}%")
