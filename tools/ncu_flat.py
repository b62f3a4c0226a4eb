"""One flat (NO_FILTER) max-load plan of a config (ncu capture target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import _lib as L, api  # noqa: E402

p = G.config_problems(int(sys.argv[1]) if len(sys.argv) > 1 else 6)[0]
slice_ = int(sys.argv[2]) if len(sys.argv) > 2 else 0
s = api.Session(p, flags=p.flags | L.F_NO_FILTER)
nt = 1
for _ in range(p.n_apps):
    nt *= len(p.batch)
for _ in range(p.n_stages):
    nt *= p.max_replicas * len(p.quota_pct)
lo = (nt // 3) - (nt // 3) % (p.max_replicas * len(p.quota_pct)) if slice_ else 0
r = s.plan_max_load(lo=lo, hi=lo + slice_ if slice_ else 0)
print(p.name, r.index, s.last_stats())
