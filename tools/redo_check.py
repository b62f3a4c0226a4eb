import os, sys
sys.path.insert(0, os.getcwd())
from gen import problems as G
from paper_2005_02088_b200 import api
pb = G.config_problems(7)[0]
for cap in ("30000", "300000"):
    for sl in ("1", "8"):
        os.environ["CAMELOT_FRONTIER_CAP"] = cap; os.environ["CAMELOT_TMODE_SLACK"] = sl
        s = api.Session(pb, n_loads=1)
        pm, pr = s.plan_max_then_min(0.3)
        print("cap", cap, "slack", sl, "max-load evaluated", pm.n_evaluated, "index", pm.index, "min-res evaluated", pr.n_evaluated)
