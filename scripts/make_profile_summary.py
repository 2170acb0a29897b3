"""Summarise gpurun_out/{launches.csv, prof_tc_c4.ncu-rep, bench.log} into profiles/<tag>/.

Writes: launches.md (per-kernel share of one C4 bench step) and bench.json (the bench line).
The per-kernel ncu metrics and DRAM bytes per pass come from scripts/ncu_pass_summary.py."""
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
    f.write(f"# ncu launch list — C4 (R-MAT s24), one bench step: gc_build_csr + gc_ktruss_analysis(3)\n\n")
    f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` of `scripts/run_tc.py --config C4 --reps 1 "
            "--what analysis` (cold-cache, serialised launches: compare shares, not absolutes).\n\n")
    f.write(f"Total kernel time {S/1e6:.1f} ms over {sum(cnt.values())} launches.\n\n| kernel | launches | ms | share |\n|---|---|---|---|\n")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        f.write(f"| `{k}` | {cnt[k]} | {v/1e6:.2f} | {100*v/S:.1f}% |\n")
# ---- bench line
b = os.path.join(g, "bench.log")
if os.path.exists(b):
    line = [l for l in open(b) if l.startswith("{")]
    if line:
        open(os.path.join(out, "bench.json"), "w").write(line[-1])
print(open(os.path.join(out, "launches.md")).read()[:3000])

