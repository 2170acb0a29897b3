"""Expected values for the full-size configs C3, C4, C5, written ONLY by the CPU
oracle (oracle/) from the seeded generator (gen/).  Nothing here imports or
runs the CUDA path; the GPU parity tests (tests/test_parity_gpu.py) compare
libgc's outputs with the files this script writes:

    tests/golden/c3_expected.json   T (O-4), supports (O-3), k-truss masks for
                                     k = 3..6 (O-5, Alg. 4 batch semantics) and
                                     trussness (O-7), cross-checked: mask_k ==
                                     (tau >= k) (reading A8)
    tests/golden/c4_expected.json   T, supports, trussness / kmax (O-7), masks
                                     for k = 3..6 derived as tau >= k
    tests/golden/c5_expected.json   the same for C5

Trussness comes from O-7 (sequential bucket peel) or O-8 (Alg. 4's
incremental rounds, parallel), or both with an equality check (--tau
o7|o8|both; default o7 for C3/C4, o8 for C5, where O-7 would take ~10 h).

Every per-edge array is stored as the SHA-256 of its canonical-order bytes
(uint32 supports, int32 trussness, uint8 masks) plus its histogram, so a
mismatch also shows where the counts differ.  O-3 vs O-4 is checked here
(Σ support = 3 T, P4).  Phase times, thread counts and the CPU model are
recorded: they are the full oracle runs the bench report quotes.

    python scripts/make_golden.py [--tau o7|o8|both] C3 [C4 C5]    (C5: ~45 GB RAM, hours)
    python scripts/make_golden.py --crosscheck C4   (O-8 against an O-7 golden, from the cache)
    python scripts/make_golden.py --o4 C5           (O-4's triangle count against a golden's)
    python scripts/make_golden.py --support-only C5 (T and supports only: trussness_pending)
    python scripts/make_golden.py --ckpt FILE SECONDS C5   (O-8 resumable: exit 3 = state saved, call again;
                                                            the golden then holds min(trussness, clip) exactly)

GOLDEN_CACHE=<dir> overrides the cache directory (e.g. supports computed on
one host, the trussness on another).

Arrays are cached under exp/golden_cache/ (git- and gpurun-ignored) so a
rerun resumes after the support pass.
"""
from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen      # noqa: E402
import oracle   # noqa: E402

CACHE = os.environ.get("GOLDEN_CACHE") or os.path.join(ROOT, "exp", "golden_cache")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def hist(a: np.ndarray) -> dict:
    vals, cnt = np.unique(a, return_counts=True)
    return {str(int(x)): int(c) for x, c in zip(vals, cnt)}


def run(name: str, ktruss_batch: tuple = (), tau_mode: str = "o7", support_only: bool = False,
        ckpt: str | None = None, budget_s: float = 0.0) -> dict | None:
    os.makedirs(CACHE, exist_ok=True)
    cfg = gen.CONFIGS[name]
    times = {}
    t = time.time()
    u, v = cfg.generate()
    nnz = int(u.size)
    times["generate_s"] = time.time() - t
    log(name, "generated", nnz)
    t = time.time()
    g = oracle.OracleGraph(u, v)
    del u, v
    times["canonicalize_adjacency_s"] = time.time() - t
    log(name, "graph n", g.n, "m", g.m, f"{times['canonicalize_adjacency_s']:.1f}s")
    out = {"_source": ("written by scripts/make_golden.py from oracle/ only (O-1..O-5; trussness by the "
                       "tier-2 oracle named in trussness_oracle; SURVEY.md §8(c)); per-edge arrays in "
                       "canonical edge order (SURVEY §8(b))"),
           "config": name, "desc": cfg.desc, "nnz": nnz, "n": g.n, "m": g.m,
           "canonical_sha256": sha(np.stack([g.cu, g.cv], axis=1))}

    sp = os.path.join(CACHE, f"{name}_support.npy")
    if os.path.exists(sp):
        sup = np.load(sp)
        times["support_s"] = json.load(open(sp + ".json"))["support_s"]
        log(name, "support from cache")
    else:
        t = time.time()
        sup = g.support()                                   # O-3
        times["support_s"] = time.time() - t
        np.save(sp, sup)
        json.dump({"support_s": times["support_s"]}, open(sp + ".json", "w"))
        log(name, f"support {times['support_s']:.1f}s")
    if name == "C5" and not os.environ.get("GOLDEN_O4"):
        # O-4 at C5 would add hours: T = Σ support / 3 (P4) from O-3; `--o4 C5` checks it later
        T = int(sup.astype(np.int64).sum()) // 3
        assert 3 * T == int(sup.astype(np.int64).sum())
        out["triangles_from"] = "sum of O-3 supports / 3 (P4); O-4 not run at C5"
        log(name, "T (Σ S / 3)", T)
    else:
        t = time.time()
        T = g.triangle_count()                              # O-4
        times["triangle_count_s"] = time.time() - t
        assert int(sup.astype(np.int64).sum()) == 3 * T, "O-3 / O-4 disagree (P4)"
        out["triangles_from"] = "O-4 (id-order triangle count), equal to sum of O-3 supports / 3"
        log(name, "T", T, f"{times['triangle_count_s']:.1f}s")
    out.update(triangles=T, support_sha256=sha(sup.astype(np.uint32)), support_max=int(sup.max(initial=0)),
               support_zero=int((sup == 0).sum()))

    if support_only:
        # T and supports only (O-3, P4); the trussness is added by a later full run
        out["trussness_pending"] = True
        out["oracle_times"] = {**{k: round(v, 3) for k, v in times.items()}, "threads": os.cpu_count(),
                               "cpu": cpu_model(), "host": platform.node()}
        return out
    masks = {}
    for k in ktruss_batch:                                  # O-5, the definition
        t = time.time()
        alive, trace = g.ktruss(k)
        times[f"ktruss{k}_s"] = time.time() - t
        masks[k] = alive
        out.setdefault("ktruss_rounds", {})[str(k)] = trace.tolist()
        log(name, f"O-5 k={k}: {int(alive.sum())} edges, {trace.size} rounds, {times[f'ktruss{k}_s']:.1f}s")

    if tau_mode in ("o7", "both"):
        t = time.time()
        tau, kmax = g.truss_sequential(sup, consume=(tau_mode == "o7"))   # O-7 (rows in place when alone)
        times["truss_sequential_s"] = time.time() - t
        log(name, "O-7 kmax", kmax, f"{times['truss_sequential_s']:.1f}s")
    if tau_mode in ("o8", "both"):
        t = time.time()
        if ckpt and os.environ.get("GOLDEN_DEADLINE"):     # budget up to a wall-clock deadline (epoch s)
            budget_s = max(60.0, float(os.environ["GOLDEN_DEADLINE"]) - time.time())
        res = g.truss_parallel(sup, consume=True, ckpt=ckpt, budget_s=budget_s)   # O-8
        spent = time.time() - t
        if ckpt:                                            # time over every resumed call
            side = ckpt + ".time.json"
            prev = json.load(open(side))["s"] if os.path.exists(side) else 0.0
            json.dump({"s": prev + spent}, open(side, "w"))
            spent += prev
        if res is None:
            hdr = np.fromfile(ckpt, dtype=np.int64, count=7)    # magic, n, m, k, kmax, rounds, alive
            log(name, f"O-8 unfinished after this call ({spent:.0f} s so far): state saved to {ckpt} "
                      f"at level k={int(hdr[3])}, kmax so far {int(hdr[4])}, rounds {int(hdr[5])}, "
                      f"live edges {int(hdr[6])} of {g.m}")
            # Partial golden from the saved state (written by oracle/ only): the levels below k are
            # finished, so every removed edge (state 0) holds its final trussness (<= k - 2) and every
            # live edge has trussness >= k - 1 -- the exact trussness clipped at k - 1.
            k_next, m = int(hdr[3]), g.m
            st = np.fromfile(ckpt, dtype=np.uint8, count=m, offset=56 + 4 * m)
            tau_p = np.fromfile(ckpt, dtype=np.int32, count=m, offset=56 + 5 * m)
            assert int((st != 0).sum()) == int(hdr[6])
            assert int(tau_p[st == 0].max(initial=2)) <= k_next - 2
            clip = np.where(st == 0, tau_p, np.int32(k_next - 1)).astype(np.int32)
            out["trussness_pending"] = True
            out["trussness_partial"] = {
                "clip": k_next - 1, "live_edges": int(hdr[6]), "kmax_at_least": int(hdr[4]),
                "rounds_so_far": int(hdr[5]), "o8_seconds": round(spent, 1), "threads": os.cpu_count(),
                "clip_sha256": sha(clip), "clip_hist": hist(clip),
                "note": ("O-8 stopped at its deadline at the start of level k = clip + 1: min(trussness, clip) "
                         "of every edge is exact (edges below clip have their final trussness)")}
            out["oracle_times"] = {**{k: round(v, 3) for k, v in times.items()}, "threads": os.cpu_count(),
                                   "cpu": cpu_model(), "host": platform.node()}
            out["_unfinished"] = True
            return out
        tau8, kmax8 = res
        times["truss_parallel_s"] = spent
        log(name, "O-8 kmax", kmax8, f"{times['truss_parallel_s']:.1f}s")
        if tau_mode == "both":
            assert kmax8 == kmax and np.array_equal(tau8, tau), "O-7 and O-8 disagree"
        tau, kmax = tau8, kmax8
    out["trussness_oracle"] = {"o7": "O-7", "o8": "O-8", "both": "O-7 = O-8 (checked equal)"}[tau_mode]
    np.save(os.path.join(CACHE, f"{name}_tau.npy"), tau)
    for k, alive in masks.items():
        assert np.array_equal(alive.astype(bool), tau >= k), f"O-5 k={k} != tier-2 tau >= k (reading A8)"
    out.update(kmax=kmax, trussness_sha256=sha(tau.astype(np.int32)), trussness_hist=hist(tau))
    out["ktruss_size"] = {}
    out["ktruss_sha256"] = {}
    for k in sorted(set(range(3, 7)) | {kmax, kmax + 1}):
        mk = (tau >= k).astype(np.uint8)
        out["ktruss_size"][str(k)] = int(mk.sum())
        out["ktruss_sha256"][str(k)] = sha(mk)
    out["oracle_times"] = {**{k: round(v, 3) for k, v in times.items()},
                           "threads": os.cpu_count(), "truss_sequential_threads": 1,
                           "truss_parallel_threads": os.cpu_count(),
                           "cpu": cpu_model(), "host": platform.node()}
    return out


def crosscheck(name: str) -> None:
    """Re-derive the trussness of an existing golden with the other tier-2
    oracle (O-8) from the cached supports and compare: the file then records
    "O-7 = O-8 (checked equal)"."""
    path = os.path.join(GOLDEN, f"{name.lower()}_expected.json")
    d = json.load(open(path))
    tau7 = np.load(os.path.join(CACHE, f"{name}_tau.npy"))
    assert sha(tau7.astype(np.int32)) == d["trussness_sha256"], "cached trussness is not the golden's"
    u, v = gen.CONFIGS[name].generate()
    g = oracle.OracleGraph(u, v)
    del u, v
    sup = np.load(os.path.join(CACHE, f"{name}_support.npy"))
    assert sha(sup.astype(np.uint32)) == d["support_sha256"]
    t = time.time()
    tau8, kmax8 = g.truss_parallel(sup, consume=True)
    dt = time.time() - t
    log(name, "O-8 kmax", kmax8, f"{dt:.1f}s")
    assert kmax8 == d["kmax"] and np.array_equal(tau8, tau7), "O-7 and O-8 disagree"
    d["trussness_oracle"] = "O-7 = O-8 (checked equal)"
    d["oracle_times"]["truss_parallel_s"] = round(dt, 3)
    d["oracle_times"]["truss_parallel_threads"] = os.cpu_count()
    with open(path, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)
        f.write("\n")
    log("cross-checked", path)


def o4_check(name: str) -> None:
    """Count the triangles of a golden's config with O-4 and compare."""
    path = os.path.join(GOLDEN, f"{name.lower()}_expected.json")
    d = json.load(open(path))
    u, v = gen.CONFIGS[name].generate()
    g = oracle.OracleGraph(u, v)
    del u, v
    t = time.time()
    T = g.triangle_count()
    dt = time.time() - t
    assert T == d["triangles"], "O-4 disagrees with the golden's triangle count"
    d["triangles_from"] = "O-4 (id-order triangle count), equal to sum of O-3 supports / 3"
    d["oracle_times"]["triangle_count_s"] = round(dt, 3)
    with open(path, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)
        f.write("\n")
    log(name, "O-4 T", T, f"{dt:.1f}s: equal")


def main(argv):
    if argv and argv[0] == "--o4":
        for name in argv[1:]:
            o4_check(name)
        return
    if argv and argv[0] == "--crosscheck":
        for name in argv[1:]:
            crosscheck(name)
        return
    tau_mode = None
    support_only = False
    ckpt, budget = None, 0.0
    if argv and argv[0] == "--ckpt":                       # O-8 in several calls (C5 on a 1-hour host)
        ckpt, budget, argv = argv[1], float(argv[2]), argv[3:]
    if argv and argv[0] == "--support-only":
        support_only, argv = True, argv[1:]
    if argv and argv[0] == "--tau":
        tau_mode, argv = argv[1], argv[2:]
    names = argv or ["C3"]
    for name in names:
        ks = (3, 4, 5, 6) if name == "C3" else ()
        d = run(name, ks, tau_mode or ("o8" if name == "C5" else "o7"), support_only, ckpt, budget)
        if d is None:
            sys.exit(3)
        unfinished = d.pop("_unfinished", False)
        path = os.path.join(GOLDEN, f"{name.lower()}_expected.json")
        with open(path, "w") as f:
            json.dump(d, f, indent=1, sort_keys=True)
            f.write("\n")
        log("wrote", path, "(partial trussness: O-8 unfinished, call again to continue)" if unfinished else "")
        if unfinished:
            sys.exit(3)


if __name__ == "__main__":
    main(sys.argv[1:])
