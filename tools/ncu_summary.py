"""Summarise an ncu report: key raw metrics + top stall reasons + top stalled SASS."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]
for vals in rows[2:]:
    print("kernel:", vals[hdr.index("Kernel Name")][:100])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:60s} {vals[i]:>16s} {units[i]}")
    st = [(hdr[i], float(vals[i])) for i in range(len(hdr))
          if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not hdr[i].endswith("not_issued")
          and vals[i] not in ("", "n/a")]
    tot = sum(v for _, v in st) or 1
    for n, v in sorted(st, key=lambda x: -x[1])[:8]:
        print(f"  stall {n[33:]:40s} {100 * v / tot:5.1f}%")
