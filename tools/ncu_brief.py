"""Key metrics + stall breakdown from an .ncu-rep (one line per kernel launch)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else None
args = ["ncu", "-i", rep, "--page", "raw", "--csv"] + (["-k", "regex:" + flt] if flt else [])
rows = list(csv.reader(io.StringIO(subprocess.run(args, capture_output=True, text=True).stdout)))
h = rows[0]
want = {
    "gpu__time_duration.sum": "dur",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "lts__t_bytes.sum": "l2_bytes",
    "l1tex__t_bytes.sum": "l1_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem%",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2%",
}
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d.get("Kernel Name", "")[:60])
    print("  " + "  ".join(f"{v}={d.get(k, '?')}" for k, v in want.items()))
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): d[k] for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(float(v or 0) for v in st.values()) or 1
    top = sorted(st.items(), key=lambda kv: -float(kv[1] or 0))[:8]
    print("  stalls: " + ", ".join(f"{k} {100*float(v)/tot:.0f}%" for k, v in top))
