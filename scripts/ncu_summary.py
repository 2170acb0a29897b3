"""Summarise an ncu report: per-kernel key metrics and the top stall lines of one kernel."""
import csv, io, subprocess, sys
rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr = r[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idi = hdr.index("ID")
want = ["Duration", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Executed Ipc Active", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Dynamic Shared Memory Per Block", "L2 Cache Throughput", "Issue Slots Busy", "Memory Throughput", "Grid Size"]
seen = {}
for row in r[1:]:
    if row[mi] in want:
        key = (row[idi], row[ki][:60])
        seen.setdefault(key, []).append(f"{row[mi]}={row[vi]}{row[ui]}")
for k, v in seen.items():
    print(k[0], k[1]); print("   ", "; ".join(v))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
cols = [i for i, x in enumerate(h) if x in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_bytes.sum")]
for row in rr[1:]:
    if len(row) > max(cols) and row[cols[0]] != "":
        print([ (h[i], row[i]) for i in cols])
