"""Cascade stride candidates on several C4-shaped problems (other seeds, QoS scale
1.0 / 0.8; development aid): step time of camelot_plan_max_then_min per candidate.
python tools/cascade_probe3.py "ML1|MR1;ML2|MR2;..." """
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402

cands = [c.split("|") for c in sys.argv[1].split(";")]
probs = [G.config_problems(4)[0], G.config_problems(7)[0]]
for j, rho in ((2, 1.0), (3, 1.0), (4, 0.8), (5, 0.9), (6, 1.0), (7, 0.8)):
    probs.append(G.build_problem(f"C4x{j}", [["p1", "c2", "m2", "c3", "m1"]], 8, 1, G.POW2_128, 4,
                                 G.config_seed(4, j), rho, "v100-dgx2"))
sess = [api.Session(p, n_loads=1) for p in probs]
for s in sess:
    s.upload()
ref = [s.plan_max_then_min(0.3) for s in sess]
print("problems:", [p.name for p in probs], flush=True)
for a, b in cands:
    os.environ["CAMELOT_COARSE_P0"] = a
    os.environ["CAMELOT_COARSE_P1"] = b
    out = []
    for s, r in zip(sess, ref):
        ts = []
        for rep in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            pm, pr = s.plan_max_then_min(0.3, resident=True)
            e1.record()
            torch.cuda.synchronize()
            if rep >= 1:
                ts.append(e0.elapsed_time(e1))
        assert pm.index == r[0].index and pr.index == r[1].index
        out.append(statistics.median(ts))
    print(f"ML {a:>9} MR {b:>9}: " + " ".join(f"{t:7.3f}" for t in out) + f"  | sum {sum(out):.2f} geo "
          f"{statistics.geometric_mean(out):.3f}", flush=True)
