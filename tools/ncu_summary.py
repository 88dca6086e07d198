"""Compact summary of ncu --set full captures (one kernel launch per .ncu-rep):
duration, DRAM traffic, pipe utilisation, occupancy.  Usage: ncu_summary.py rep..."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%active"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "fp64_pipe_%elapsed"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_%active"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_cycles_%active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall_barrier"),
    ("local_load_bytes", "local"),
]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return f"{rep}: no data\n"
    hdr, units = rows[0], rows[1]
    lines = []
    for vals in rows[2:]:
        d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
        name = d.get("Kernel Name", ("", "?"))[1]
        lines.append(f"== {name}\n   rep: {rep}")
        for key, label in KEYS:
            if key in d:
                u, v = d[key]
                lines.append(f"   {label:24s} {v} {u}")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    for r in sys.argv[1:]:
        sys.stdout.write(summarise(r))
