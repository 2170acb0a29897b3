"""Round-2 profile summary: gpurun_out/{launches.csv, launches_decomp.csv, r2_*.ncu-rep, bench.log}
-> profiles/round2/{launches.md, ncu_kernels.md, bench.json} and profiles/ncu_summary.json
(the DRAM bytes per pass that bench.py reports as roofline "traffic").

launches.csv: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`
of one C4 build + TC pass + gc_ktruss_analysis(4) (scripts/gpu_profile_r2.sh): cold-cache,
serialised launches -- compare shares, not absolutes."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles", "round2")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ix = {n: h.index(n) for n in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    seq = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        k = int(r[ix["ID"]])
        d = seq.setdefault(k, {"name": r[ix["Kernel Name"]]})
        try:
            v = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1.0)
        except ValueError:
            continue
        d[r[ix["Metric Name"]]] = v
    return list(seq.values())


def short(name):
    return name.split("(")[0].replace("gcx::<unnamed>::", "").replace("gcx::", "").replace("void ", "")[:70]


def sup_flag(name):
    s = short(name)
    if not s.startswith("k_tc_"):
        return None
    args = [a.strip() for a in s[s.index("<") + 1:s.rindex(">")].split(",")]
    return (args[1] if s.startswith("k_tc_warp") else args[0]) == "1"


def seg_sum(ks):
    return {"ms": sum(k.get("gpu__time_duration.sum", 0) for k in ks),
            "dram_bytes": sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in ks),
            "launches": len(ks)}


def table(f, ks, total_ms):
    agg = collections.OrderedDict()
    for k in ks:
        a = agg.setdefault(short(k["name"]), [0, 0.0, 0.0])
        a[0] += 1
        a[1] += k.get("gpu__time_duration.sum", 0)
        a[2] += k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
    f.write("| kernel | launches | ms | share | DRAM GB |\n|---|---|---|---|---|\n")
    for n, (c, ms, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if ms < 0.005 * total_ms and ms < 0.05:
            continue
        f.write(f"| `{n}` | {c} | {ms:.2f} | {100 * ms / total_ms:.1f}% | {b / 1e9:.2f} |\n")


def main():
    os.makedirs(OUT, exist_ok=True)
    seq = launches(os.path.join(G, "launches.csv"))
    i_tc = next(i for i, k in enumerate(seq) if sup_flag(k["name"]) is False)
    i_an = next(i for i, k in enumerate(seq) if sup_flag(k["name"]) is True)
    build, tc_seg, an = seq[:i_tc], seq[i_tc:i_an], seq[i_an:]
    tc = [k for k in tc_seg if sup_flag(k["name"]) is False]
    sup = [k for k in an if sup_flag(k["name"]) is True]
    summ = {"workload": "C4 R-MAT s24", "source": "profiles/round2/launches.md (ncu launch list with DRAM bytes)",
            "build": seg_sum(build), "tc": seg_sum(tc), "support": seg_sum(sup), "ktruss": seg_sum(an)}
    dec_path = os.path.join(G, "launches_decomp.csv")
    if os.path.exists(dec_path):
        dseq = launches(dec_path)
        j = next(i for i, k in enumerate(dseq) if sup_flag(k["name"]) is True)
        summ["decomposition"] = seg_sum(dseq[j:])
        dec_seq = dseq[j:]
    else:
        dec_seq = None
    for key in list(summ):
        if isinstance(summ[key], dict) and "dram_bytes" in summ[key]:
            summ[key]["dram_bytes_per_launch"] = summ[key]["dram_bytes"]
    json.dump(summ, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
    step = build + an
    step_ms = sum(k.get("gpu__time_duration.sum", 0) for k in step)
    with open(os.path.join(OUT, "launches.md"), "w") as f:
        f.write("# ncu launch list — C4 (R-MAT s24), round 2\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` "
                "of `scripts/run_tc.py --config C4 --reps 1 --what tc,analysis --k 4` (scripts/gpu_profile_r2.sh). "
                "Cold-cache, serialised launches: compare shares, not absolutes.\n\n")
        f.write(f"## The bench step: gc_build_csr + gc_ktruss_analysis(4) — {step_ms:.1f} ms of kernels, "
                f"{len(step)} launches\n\n")
        table(f, step, step_ms)
        f.write("\n## Passes\n\n| pass | ms (kernels) | DRAM GB | launches |\n|---|---|---|---|\n")
        for key in ("build", "tc", "support", "ktruss", "decomposition"):
            if key in summ:
                d = summ[key]
                f.write(f"| {key} | {d['ms']:.1f} | {d['dram_bytes'] / 1e9:.1f} | {d['launches']} |\n")
        f.write("\n`ktruss` = every kernel of the gc_ktruss_analysis(4) call (support pass, output scatter, "
                "level scan, symmetric rows, peel rounds); `decomposition` = every kernel of one "
                "gc_truss_decomposition call after its support pass's first kernel (scripts/run_decomp.py).\n")
        if dec_seq:
            dms = sum(k.get("gpu__time_duration.sum", 0) for k in dec_seq)
            f.write(f"\n## gc_truss_decomposition — {dms:.1f} ms of kernels, {len(dec_seq)} launches\n\n")
            table(f, dec_seq, dms)
    # --set full reports
    names = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
             "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_issued.avg.pct_of_peak_sustained_active",
             "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
             "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
    rows = []
    for rep in ("r2_tc_block", "r2_sup_block", "r2_peel_k4"):
        p = os.path.join(G, rep + ".ncu-rep")
        if not os.path.exists(p):
            continue
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        r = list(csv.reader(io.StringIO(out)))
        if len(r) < 3:
            continue
        h, u = r[0], r[1]
        for x in r[2:]:
            d = {n: f"{x[h.index(n)]} {u[h.index(n)]}".strip() for n in names if n in h}
            rows.append((short(x[h.index("Kernel Name")]), rep, d))
    if rows:
        with open(os.path.join(OUT, "ncu_kernels.md"), "w") as f:
            f.write("# ncu --set full, C4, round 2 (scripts/gpu_profile_r2.sh)\n\nSerialised replays of one launch each.\n\n")
            f.write("| kernel | report | " + " | ".join(names) + " |\n|" + "---|" * (len(names) + 2) + "\n")
            for k, rep, d in rows:
                f.write(f"| `{k}` | {rep} | " + " | ".join(d.get(n, "") for n in names) + " |\n")
    b = os.path.join(G, "bench.log")
    if os.path.exists(b):
        line = [ln for ln in open(b) if ln.startswith("{")]
        if line:
            open(os.path.join(OUT, "bench.json"), "w").write(line[-1])
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    sys.exit(main())
