"""Text summary of an ncu --set full report (read on the CPU box): python tools/ncu_summary.py rep.ncu-rep [regex]
Prints, per profiled launch, the metrics the bench's roofline refers to (duration, DRAM bytes, pipe utilisation)."""
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
for r in data:
    name = r[hdr.index("Kernel Name")]
    if pat and not pat.search(name):
        continue
    print(name)
    tot = 0.0
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"  {k} = {r[i]} {units[i]}")
            if k.startswith("dram__bytes"):
                v = float(r[i])
                u = units[i].lower()
                tot += v * (1e9 if u.startswith("g") else 1e6 if u.startswith("m") else 1e3 if u.startswith("k") else 1)
    print(f"  dram read+write = {tot / 1e9:.4f} GB per launch")
