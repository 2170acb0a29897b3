"""Aggregate an ncu report's SASS-level stall samples / instructions by CUDA source line.
usage: python scripts/ncu_lines.py REPORT [launch_skip] [top]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; skip = sys.argv[2] if len(sys.argv) > 2 else "0"; top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", skip, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if len(r) > 5 and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)"); ie = hdr.index("Instructions Executed")
cur = None; src = {}; samp = collections.Counter(); inst = collections.Counter(); fname = ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) <= ie or r is hdr:
        continue
    if r[0] not in ("",):
        cur = (fname, r[0]); src[cur] = r[1].strip()[:100]
        continue
    if cur and r[si].isdigit():
        samp[cur] += int(r[si]); inst[cur] += int(r[ie] or 0)
T = sum(samp.values()) or 1; I = sum(inst.values()) or 1
print(f"samples {T} inst {I}")
for k, v in samp.most_common(top):
    print(f"{100*v/T:5.1f}% smp {100*inst[k]/I:5.1f}% ins {k[0]}:{k[1]:>4s} {src[k]}")
