"""Mutation check of the CPU oracle's pins.

Each mutant is a plausible one-line mistake in oracle/oracle.c.  The script
copies oracle/, gen/ and tests/ into a scratch directory, applies the mutant,
rebuilds liboracle.so there and runs the CPU pins (tests/test_oracle_pins.py);
a mutant that passes every pin is reported as SURVIVED (exit code 1).

    python scripts/mutation_check.py [name ...]
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TIMEOUT_S = 300

# name: (exact text in oracle.c, replacement).  Semantics-preserving edits
# (e.g. never taking a galloping branch, not advancing past a match in a list
# of distinct ids, skipping the dead-entry compaction) are not listed: they
# are equivalent mutants and survive any pin.
MUTANTS = {
    # O-5 alive-subgraph support, galloping branch
    "o5_gallop_no_long_alive": ("&& alive[eid[i]] && alive[eid[p]]) ++c;", "&& alive[eid[i]]) ++c;"),
    "o5_gallop_no_short_alive": ("&& alive[eid[i]] && alive[eid[p]]) ++c;", "&& alive[eid[p]]) ++c;"),
    # O-5 merge branch
    "o5_merge_no_alive": ("else { if (alive[eid[i]] && alive[eid[j]]) ++c; ++i; ++j; }", "else { ++c; ++i; ++j; }"),
    "o5_threshold_off_by_one": ("(int64_t)s[e] < (int64_t)k - 2", "(int64_t)s[e] < (int64_t)k - 3"),
    "o5_x_stays_alive": ("                s[e] = 0xFFFFFFFFu;\n                ++nx;",
                         "                ++nx;"),
    "o5_work_min_not_max": ("work[0] += d[cu[e]] < d[cv[e]] ? d[cu[e]] : d[cv[e]];",
                            "work[0] += d[cu[e]] > d[cv[e]] ? d[cu[e]] : d[cv[e]];"),
    "o5_work_dec_sign": ("if (alive[e]) work[1] += (int64_t)prev[e] - (int64_t)s[e];",
                         "if (alive[e]) work[1] += (int64_t)s[e] - (int64_t)prev[e];"),
    # O-3 intersection
    "o3_gallop_skip_candidate": ("lo = lower_bound32(B, lo, nb, A[i]);", "lo = lower_bound32(B, lo + 1, nb, A[i]);"),
    "o3_gallop_strict": ("if (lo < nb && B[lo] == A[i]) { ++c; ++lo; }", "if (lo + 1 < nb && B[lo] == A[i]) { ++c; ++lo; }"),
    # O-4
    "o4_w_gt_a": ("lower_bound32(C->col, a0, a1, b + 1);       /* w > b in N(a) */\n        int64_t pb = lower_bound32(C->col, b0, b1, b + 1);",
                  "lower_bound32(C->col, a0, a1, a + 1);\n        int64_t pb = lower_bound32(C->col, b0, b1, a + 1);"),
    # O-7
    "o7_no_alive_g": ("if (E[f].pos < 0 || E[g].pos < 0) continue;", "if (E[f].pos < 0) continue;"),
    "o7_no_level_guard": ("if (E[h].s > se) {", "if (E[h].s > 0) {"),
    "o7_gallop_skip_equal": ("if (col[q] != col[p]) continue;", "if (col[q] != col[p]) continue; if (gallop) ++q;"),
    "o7_compact_drops_last": ("len[x] = w - ptr[x];", "len[x] = w - ptr[x] - (w > ptr[x]);"),
    "o7_tau_off_by_one": ("tau[e] = (int32_t)se + 2;", "tau[e] = (int32_t)se + 3;"),
    # O-1
    "o1_keep_duplicates": ("if (i > 0 && keys[i] == keys[i - 1]) continue;", ""),
}


def run(name: str, src: str, old: str, new: str) -> bool:
    assert src.count(old) == 1, f"{name}: anchor not unique / missing"
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "gen", "tests", "paper_1708_06866_b200"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__", "csrc"))
        shutil.copy(os.path.join(ROOT, "Makefile"), tmp)
        open(os.path.join(tmp, "oracle", "oracle.c"), "w").write(src.replace(old, new))
        subprocess.run(["make", "-C", tmp, "gen", "oracle"], check=True, capture_output=True)
        try:
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:warnings", "-p",
                                "no:cacheprovider", os.path.join(tmp, "tests", "test_oracle_pins.py")],
                               cwd=tmp, capture_output=True, text=True, timeout=TIMEOUT_S,
                               env={**os.environ, "PYTHONPATH": tmp})
            killed = r.returncode != 0
            last = [ln for ln in r.stdout.splitlines() if ln.strip()][-1:] or [""]
        except subprocess.TimeoutExpired:
            # a mutant that never terminates (e.g. x never leaves the graph) fails the pins too
            killed, last = True, [f"no result after {TIMEOUT_S} s (the unmutated pins take under a minute)"]
        print(f"{name:28s} {'killed' if killed else 'SURVIVED'}  {last[0][:90]}", flush=True)
        return killed


def main(names):
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    if run("(unmutated)", src, "/* ------------------------------------------------------------------ O-7 --", "/* ------------------------------------------------------------------ O-7 --"):
        print("the pins fail on the unmutated oracle: fix them first")
        return 2
    todo = names or list(MUTANTS)
    survived = [n for n in todo if not run(n, src, *MUTANTS[n])]
    print(f"{len(todo) - len(survived)}/{len(todo)} mutants killed")
    return 1 if survived else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
