"""Collect the round's ncu --set full captures into profiles/: a text summary
(tools/ncu_summary.py + top stall lines) and profiles/ncu_traffic.json with the
per-launch DRAM traffic that bench.py reports as roofline.traffic.
Usage: python tools/ncu_collect.py TAG [OUTDIR (default profiles/)]"""
import glob
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
from ncu_summary import summarise  # noqa: E402

tag = sys.argv[1]
outdir = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "profiles"
reps = sorted(glob.glob(str(ROOT / "gpurun_out" / f"prof_{tag}_*.ncu-rep")))
text = []
traffic = {}
for rep in reps:
    text.append(summarise(rep))
    stalls = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_stalls.py"), rep, "12"],
                            capture_output=True, text=True).stdout
    text.append(stalls)
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    import csv
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        continue
    d = dict(zip(rows[0], rows[2]))
    u = dict(zip(rows[0], rows[1]))
    name = d.get("Kernel Name", "?").split("(")[0].split("::")[-1].split("<")[0].strip().split(" ")[-1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(u["dram__bytes_read.sum"], 1)
    wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(u["dram__bytes_write.sum"], 1)
    traffic[name] = rd + wr
(outdir / f"{tag}_ncu_summary.txt").write_text("\n".join(text))
json.dump({"how": f"ncu --set full --clock-control none captures of one launch each (gpurun_out/prof_{tag}_*), "
                  "dram__bytes_read.sum + dram__bytes_write.sum", "tag": tag, "bytes_per_launch": traffic},
          open(outdir / "ncu_traffic.json", "w"), indent=1)
print(json.dumps(traffic, indent=1))
