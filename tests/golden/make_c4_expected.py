"""Writes tests/golden/expected_C4-full.json: the oracle's answers for the full
C4 space (8.192e13 candidates per policy) and for four 2^32-candidate slices of
it.  Calls ONLY oracle/ on problems from gen/problems.py; no value comes from
the CUDA path.

  * full space, both policies: oracle O7 (oracle.search_filtered, the
    filtered exhaustive scan of SURVEY.md §8(c) O7, validated against the plain
    scan in tests/test_oracle_o7.py).  Its incumbents are the oracle's own C4r
    results (tests/golden/expected_C4r-*.json, written by make_expected.py):
    C4r is C4 on the 10% quota grid, a subset of C4's 1% grid with identical
    table entries (checked here), so its plans are members of the C4 space; each
    one is re-scored in C4 by oc_score before use.
  * slices: the plain exhaustive scan oracle.search over
    [0, 2^32), a seeded 2^32-aligned slice, and the aligned slices holding the
    O7 winners of each policy.

  * --c4b: the second C4 instance C4b (gen config 7: other draws, QoS 0.8x),
    full space, both policies, by O7.  Its incumbents are the plain-scan optima
    of its own 10% sub-grid problem (C4b restricted to quotas 10..100, the same
    table entries), each re-scored in C4b; for min-resource at the C4b load.

  * --b200: C4 on the modeled-B200 cluster preset (gen PRESETS["b200"]: 8 TB/s,
    180 GiB per GPU), full space, both policies, by O7 with the same 10%
    sub-grid incumbents ("C4 is also run with b200").

    python tests/golden/make_c4_expected.py [threads] [--no-slices] [--c4b | --b200]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from gen import problems as G  # noqa: E402
from oracle import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SLICE = 1 << 32
LOW_LOAD = 0.3   # PAPER.md L1088 (bench.py uses the same float64 product)


def best_dict(b, seconds):
    return dict(index=b.index, T=b.T, u=b.u, U=b.U, n_feasible=b.n_feasible, n_scanned=b.n_scanned,
                hist=b.hist, seconds=seconds)


def c4r_to_c4(c4r, c4, x):
    """Canonical C4r index -> the same plan's canonical C4 index (quota 10k% is
    theta 10k-1 on the 1% grid)."""
    beta, rho, theta = O.decode(c4r, x)
    q = [int(c4r.quota_pct[t]) for t in theta]
    th = [int(np.nonzero(c4.quota_pct == v)[0][0]) for v in q]
    return O.encode(c4, beta, rho, th)


def main(threads, slices=True):
    c4 = G.config_problems(4)[0]
    c4r = G.config_problems(6)[0]
    sub = [int(np.nonzero(c4.quota_pct == q)[0][0]) for q in c4r.quota_pct]
    assert np.array_equal(c4.table[:, :, sub, :], c4r.table), "C4r must be a sub-grid of C4"
    gold = json.load(open(os.path.join(HERE, f"expected_{c4r.name}.json")))
    assert gold["sha256"] == c4r.sha256()
    rec = dict(problem=c4.name, sha256=c4.sha256(), ntot=O.ntot(c4), threads=threads,
               note="written by tests/golden/make_c4_expected.py (oracle only: O7 for the full space, "
                    "the plain scan for the slices)")
    # ---- max-load: incumbent = the C4r optimum, re-scored in C4
    xi = c4r_to_c4(c4r, c4, gold["max_load"]["index"])
    s = O.score(c4, xi)
    assert s.verdict == 0 and s.T == np.float32(gold["max_load"]["T"])
    t = time.time()
    bm = O.search_filtered(c4, T_inc=s.T, threads=threads)
    rec["max_load"] = dict(incumbent=dict(index=xi, T=s.T, source="C4r max-load optimum"),
                           **best_dict(bm, time.time() - t))
    print("max_load", rec["max_load"], flush=True)
    # ---- min-resource at 0.3 T*: incumbent = the C4r min-resource plan if it
    # carries the C4 load, else the C4 max-load plan (always feasible there)
    lam = [LOW_LOAD * bm.T]
    xr = c4r_to_c4(c4r, c4, gold["min_resource"]["index"])
    sr = O.score(c4, xr, loads=[lam])
    if sr.level_verdict == [0]:
        inc = dict(index=xr, u=sr.u, U=sr.U, source="C4r min-resource optimum")
    else:
        sm = O.score(c4, bm.index, loads=[lam])
        assert sm.level_verdict == [0]
        inc = dict(index=bm.index, u=sm.u, U=sm.U, source="C4 max-load optimum")
    t = time.time()
    br = O.search_filtered(c4, "min_resource", load=lam, u_inc=inc["u"], U_inc=inc["U"], threads=threads)
    rec["min_resource"] = dict(loads=[lam], incumbent=inc, **best_dict(br, time.time() - t))
    print("min_resource", rec["min_resource"], flush=True)
    path = os.path.join(HERE, "expected_C4-full.json")
    if slices:
        rng = np.random.Generator(np.random.PCG64(G.SEED_BASE + 4444))
        seeded = int(rng.integers(1, rec["ntot"] // SLICE)) * SLICE
        plan = [("first", 0, "max_load"), ("seeded", seeded, "max_load"),
                ("max_load_winner", (bm.index // SLICE) * SLICE, "max_load"),
                ("min_resource_winner", (br.index // SLICE) * SLICE, "min_resource")]
        rec["slices"] = []
        for name, lo, pol in plan:
            t = time.time()
            kw = dict(loads=[lam]) if pol == "min_resource" else {}
            b = O.search(c4, pol, lo=lo, hi=lo + SLICE, threads=threads, **kw)[0]
            d = dict(name=name, policy=pol, lo=lo, hi=lo + SLICE, **best_dict(b, time.time() - t))
            if pol == "min_resource":
                d["loads"] = [lam]
            rec["slices"].append(d)
            print("slice", d, flush=True)
            with open(path, "w") as f:
                json.dump(rec, f, indent=1)
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)


def sub_grid(prob):
    """The same problem restricted to the quotas 10, 20, .., 100 (a subset of the
    1% grid with the same table entries)."""
    sub = [int(np.nonzero(prob.quota_pct == q)[0][0]) for q in range(10, 101, 10)]
    return prob.with_(name=prob.name + "-10pct", quota_pct=prob.quota_pct[sub].copy(),
                      table=prob.table[:, :, sub, :].copy()), sub


def main_c4b(threads, config=7, preset="v100-dgx2", out="expected_C4b-full.json"):
    p = G.config_problems(config, preset)[0]
    if preset != "v100-dgx2":
        p = p.with_(name=f"{p.name}-{preset}")
    pr, sub = sub_grid(p)

    def to_full(x):
        beta, rho, theta = O.decode(pr, x)
        return O.encode(p, beta, rho, [sub[t] for t in theta])

    rec = dict(problem=p.name, sha256=p.sha256(), ntot=O.ntot(p), threads=threads, preset=preset,
               note="written by tests/golden/make_c4_expected.py --c4b / --b200 (oracle only: O7 with incumbents "
                    "from the plain scan of the 10% sub-grid)")
    t = time.time()
    r = O.search(pr, threads=threads)[0]
    xi = to_full(r.index)
    s = O.score(p, xi)
    assert s.verdict == 0 and s.T == r.T
    bm = O.search_filtered(p, T_inc=s.T, threads=threads)
    rec["max_load"] = dict(incumbent=dict(index=xi, T=s.T, source="10% sub-grid max-load optimum"),
                           **best_dict(bm, time.time() - t))
    print("max_load", rec["max_load"], flush=True)
    lam = [LOW_LOAD * bm.T]
    t = time.time()
    rm = O.search(pr, "min_resource", loads=[lam], threads=threads)[0]
    xr = to_full(rm.index)
    sr = O.score(p, xr, loads=[lam])
    assert sr.level_verdict == [0]
    br = O.search_filtered(p, "min_resource", load=lam, u_inc=sr.u, U_inc=sr.U, threads=threads)
    rec["min_resource"] = dict(loads=[lam], incumbent=dict(index=xr, u=sr.u, U=sr.U,
                                                           source="10% sub-grid min-resource optimum"),
                               **best_dict(br, time.time() - t))
    print("min_resource", rec["min_resource"], flush=True)
    with open(os.path.join(HERE, out), "w") as f:
        json.dump(rec, f, indent=1)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    if "--c4b" in sys.argv:
        main_c4b(int(args[0]) if args else os.cpu_count())
    elif "--b200" in sys.argv:   # C4 on the modeled-B200 preset ("C4 is also run with b200")
        main_c4b(int(args[0]) if args else os.cpu_count(), config=4, preset="b200", out="expected_C4-b200-full.json")
    else:
        main(int(args[0]) if args else os.cpu_count(), slices="--no-slices" not in sys.argv)
