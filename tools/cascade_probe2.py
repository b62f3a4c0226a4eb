"""Per-policy cascade strides (CAMELOT_COARSE_P0 / _P1): C4 and C4b step times of
camelot_plan_max_then_min (development aid).  python tools/cascade_probe2.py "p0a;p0b" "p1a;p1b" """
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402

P0 = sys.argv[1].split(";")
P1 = sys.argv[2].split(";")
probs = [G.config_problems(4)[0], G.config_problems(7)[0]]
sess = [api.Session(p, n_loads=1) for p in probs]
for s in sess:
    s.upload()
ref = [s.plan_max_then_min(0.3) for s in sess]
for a in P0:
    for b in P1:
        os.environ["CAMELOT_COARSE_P0"] = a
        os.environ["CAMELOT_COARSE_P1"] = b
        out = []
        for s, r in zip(sess, ref):
            ts = []
            for rep in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                pm, pr = s.plan_max_then_min(0.3, resident=True)
                e1.record()
                torch.cuda.synchronize()
                if rep >= 2:
                    ts.append(e0.elapsed_time(e1))
            assert pm.index == r[0].index and pr.index == r[1].index
            out.append(statistics.median(ts))
        print(f"ML {a:>10} MR {b:>10}: C4 {out[0]:.3f} ms  C4b {out[1]:.3f} ms", flush=True)
