"""Markdown summary of ncu --set full reports: python tools/ncu_summary.py a.ncu-rep ..."""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__registers_per_thread", "regs")]
print("| report | kernel | grid | " + " | ".join(k[1] for k in KEYS) + " |")
print("|---|---|---|" + "---|" * len(KEYS))
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        continue
    h = rows[0]
    units = rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        vals = [f"{r[h.index(k)]} {units[h.index(k)]}".strip() if k in h else "-" for k, _ in KEYS]
        print(f"| {rep.split('/')[-1]} | `{name}` | {r[h.index('Grid Size')]} | " + " | ".join(vals) + " |")
