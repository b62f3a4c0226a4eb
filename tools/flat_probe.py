"""Flat (NO_FILTER) exhaustive scan timing of a config (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import _lib as L, api  # noqa: E402

SLICE = int(os.environ.get("FLAT_SLICE", "0"))
for cfg in [int(c) for c in sys.argv[1:]]:
    p = G.config_problems(cfg)[0]
    s = api.Session(p, flags=p.flags | L.F_NO_FILTER)
    ntot = 1
    for _ in range(p.n_apps):
        ntot *= len(p.batch)
    for _ in range(p.n_stages):
        ntot *= p.max_replicas * len(p.quota_pct)
    lo = (ntot // 3) - (ntot // 3) % (p.max_replicas * len(p.quota_pct)) if SLICE else 0
    hi = min(ntot, lo + SLICE) if SLICE else 0
    for rep in range(3):
        r = s.plan_max_load(lo=lo, hi=hi)
        st = s.last_stats()
        nt = (hi - lo) if SLICE else ntot
        print(p.name, "flat", r.index, "ms=%.2f" % (st["t_ns"] / 1e6), "cand/s=%.3g" % (nt / (st["t_ns"] * 1e-9)),
              "leaves/s=%.3g" % (st["cum_scored"] / (st["t_ns"] * 1e-9)), st, flush=True)
