"""Summarise gpurun_out/{launches.csv, prof_tc_c4.ncu-rep, bench.log} into profiles/<tag>/.

Writes: launches.md (per-kernel share of one C4 pass: build + TC + support + ktruss(3)),
ncu_tc.md (key ncu metrics of the intersection kernels), and profiles/tc_ncu_summary.json
(DRAM bytes of one TC pass, read by bench.py as roofline.traffic)."""
import collections, csv, io, json, os, subprocess, sys
tag = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "profiles", tag)
os.makedirs(out, exist_ok=True)
g = os.path.join(root, "gpurun_out")
# ---- launch list
rows = list(csv.reader(open(os.path.join(g, "launches.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = collections.OrderedDict(); cnt = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("gcx::<unnamed>::", "").replace("void ", "")[:60]
    tot[name] = tot.get(name, 0.0) + float(r[vi].replace(",", "")); cnt[name] += 1
S = sum(tot.values())
with open(os.path.join(out, "launches.md"), "w") as f:
    f.write(f"# ncu launch list — C4 (R-MAT s24), one pass of build + TC + support + ktruss(3)\n\n")
    f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` of `scripts/run_tc.py --config C4 --reps 1 "
            "--what tc,support,ktruss` (cold-cache, serialised launches: compare shares, not absolutes).\n\n")
    f.write(f"Total kernel time {S/1e6:.1f} ms over {sum(cnt.values())} launches.\n\n| kernel | launches | ms | share |\n|---|---|---|---|\n")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        f.write(f"| `{k}` | {cnt[k]} | {v/1e6:.2f} | {100*v/S:.1f}% |\n")
# ---- ncu full
rep = os.path.join(g, "prof_tc_c4.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "lts__t_requests_srcunit_l1_op_atom.sum", "launch__grid_size"]
idx = {w: hh.index(w) for w in want if w in hh}
units = rr[1]
kernels = []
for r in rr[2:]:
    if len(r) < len(hh) or not r[hh.index("Kernel Name")]:
        continue
    kernels.append({"kernel": r[hh.index("Kernel Name")].split("(")[0].replace("gcx::<unnamed>::", "").replace("void ", ""),
                    **{w: r[i] for w, i in idx.items()}, "units": {w: units[i] for w, i in idx.items()}})
with open(os.path.join(out, "ncu_tc.md"), "w") as f:
    f.write("# ncu --set full of the intersection kernels (C4)\n\n`ncu --set full --clock-control none --import-source on "
            "-k regex:k_tc_ -c 6` on `scripts/run_tc.py --config C4 --reps 1 --what tc,support`. Launch order: TC pass "
            "(class 2, 1, 0 kernels), then support pass (same classes, SUP=1).\n\n")
    f.write("| kernel | " + " | ".join(w for w in want if w in idx) + " |\n|" + "---|" * (1 + len(idx)) + "\n")
    for k in kernels:
        f.write(f"| `{k['kernel']}` | " + " | ".join(f"{k[w]} {k['units'][w]}" for w in want if w in idx) + " |\n")
def gb(k, w):
    v = float(k[w]); u = k["units"][w]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
tc = [k for k in kernels if "<0>" in k["kernel"] or ", 0>" in k["kernel"] or "(bool)0" in k["kernel"]]
summ = {"source": f"profiles/{tag}/ncu_tc.md", "workload": "C4 R-MAT s24",
        "dram_bytes_per_launch": sum(gb(k, "dram__bytes_read.sum") + gb(k, "dram__bytes_write.sum") for k in tc
                                       if "nan" not in k["dram__bytes_read.sum"]),
        "note": "DRAM bytes of the TC pass (all class kernels of one gc_triangle_count; kernels ncu could not "
                "measure (nan) are excluded)",
        "kernels": [k["kernel"] for k in tc]}
json.dump(summ, open(os.path.join(root, "profiles", "tc_ncu_summary.json"), "w"), indent=1)
# ---- bench line
b = os.path.join(g, "bench.log")
if os.path.exists(b):
    line = [l for l in open(b) if l.startswith("{")]
    if line:
        open(os.path.join(out, "bench.json"), "w").write(line[-1])
print(open(os.path.join(out, "launches.md")).read()[:3000])
print(json.dumps(summ, indent=1))
