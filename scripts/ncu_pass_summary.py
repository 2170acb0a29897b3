"""DRAM traffic per intersection pass from ncu --set full reports (one kernel per report
where ncu could not replay a second long kernel in the same session).
usage: python scripts/ncu_pass_summary.py TAG  (reads gpurun_out/prof_*.ncu-rep listed below)"""
import csv, io, json, os, subprocess, sys
tag = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
g = os.path.join(root, "gpurun_out")
names = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
         "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_issued.avg.pct_of_peak_sustained_active",
         "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread", "launch__grid_size"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
rows = {}
for rep in ["prof_tc_c4", "prof_tc_warp_c4", "prof_tc_tiny_c4", "prof_sup_block_c4", "prof_sup_warp_c4",
            "prof_sup_tiny_c4"]:
    path = os.path.join(g, rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    for x in r[2:]:
        k = x[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        if "nan" in x[h.index("dram__bytes_read.sum")]:
            continue
        d = {n: (x[h.index(n)], u[h.index(n)]) for n in names if n in h}
        d["src"] = rep
        rows[k] = d
def dram(k):
    d = rows[k]
    return sum(float(d[n][0]) * scale.get(d[n][1], 1) for n in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
def is_sup(k):   # k_tc_block<SUP, HUGE>, k_tc_warp<TS, SUP>, k_tc_tiny<SUP>
    args = [a.strip() for a in k[k.index("<") + 1:k.rindex(">")].split(",")]
    return (args[1] if k.startswith("k_tc_warp") else args[0]) == "1"
passes = {"tc": [k for k in rows if not is_sup(k)], "support": [k for k in rows if is_sup(k)]}
summ = {"workload": "C4 R-MAT s24", "source": f"profiles/{tag}/ncu_passes.md"}
for p, ks in passes.items():
    summ[p] = {"dram_bytes_per_launch": sum(dram(k) for k in ks), "kernels": ks,
               "kernel_ms": sum(float(rows[k]["gpu__time_duration.sum"][0]) for k in ks)}
json.dump(summ, open(os.path.join(root, "profiles", "ncu_summary.json"), "w"), indent=1)
with open(os.path.join(root, "profiles", tag, "ncu_passes.md"), "w") as f:
    f.write("# ncu --set full, C4 intersection kernels, one report per kernel (`scripts/gpu_profile.sh`)\n\n")
    f.write("Serialised, cold-cache replays: durations are per kernel, not the in-step times.\n\n")
    f.write("| kernel | " + " | ".join(n for n in names) + " | report |\n|" + "---|" * (len(names) + 2) + "\n")
    for k, d in rows.items():
        f.write(f"| `{k}` | " + " | ".join(f"{d[n][0]} {d[n][1]}" for n in names if n in d) + f" | {d['src']} |\n")
    for p in passes:
        f.write(f"\n**{p} pass**: DRAM {summ[p]['dram_bytes_per_launch']/1e9:.1f} GB over {summ[p]['kernel_ms']:.1f} ms "
                f"of kernels ({', '.join(passes[p])}).\n")
print(json.dumps(summ, indent=1))
