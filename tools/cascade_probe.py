"""Step time (both policies, C4) for several incumbent-cascade stride lists
(CAMELOT_COARSE; development aid).  python tools/cascade_probe.py [config]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = G.config_problems(cfg)[0]
s = api.Session(p, n_loads=1)
ref = None
for spec in (sys.argv[2].split(";") if len(sys.argv) > 2 else ["", "50,20,5", "50,20", "50,10", "50,25,10,5", "50,10,5", "34,10,3", "20,5", "25,5", "50,20,10,5", "50,5"]):
    if spec:
        os.environ["CAMELOT_COARSE"] = spec
    else:
        os.environ.pop("CAMELOT_COARSE", None)
    ts, ev = [], []
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = s.plan_max_load()
        m = s.plan_min_resource([[0.3 * r.objective] * p.n_apps])[0]
        e1.record()
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append(e0.elapsed_time(e1))
            ev.append(r.n_evaluated + m.n_evaluated)
    key = (r.index, m.index)
    ref = ref or key
    print(f"{spec or 'default':>12}: {statistics.median(ts):.3f} ms  evals {statistics.median(ev):.0f}  "
          f"{'same plans' if key == ref else 'DIFFERENT ' + str(key)}", flush=True)
