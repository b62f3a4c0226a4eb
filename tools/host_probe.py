"""Host vs device time of the bench step's API calls (development aid):
per call, host wall time of the enqueue (no sync) and the device time between
events recorded before and after it.   python tools/host_probe.py [config] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import _lib as L  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p = G.config_problems(cfg)[0]
s = api.Session(p, n_loads=1)
s.upload()
st = torch.cuda.current_stream()
for rep in range(reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    host = []
    torch.cuda.synchronize()
    ev[0].record(st)
    t0 = time.perf_counter()
    k1 = s.search_local(L.POLICY_MAX_LOAD, resident=True)
    host.append(time.perf_counter() - t0)
    ev[1].record(st)
    t0 = time.perf_counter()
    pm = s.finalize(L.POLICY_MAX_LOAD, k1)[0]
    host.append(time.perf_counter() - t0)
    ev[2].record(st)
    lam = [[0.3 * pm.objective] * p.n_apps]
    t0 = time.perf_counter()
    k2 = s.search_local(L.POLICY_MIN_RESOURCE, lam, resident=True)
    host.append(time.perf_counter() - t0)
    ev[3].record(st)
    t0 = time.perf_counter()
    s.finalize(L.POLICY_MIN_RESOURCE, k2, lam)
    host.append(time.perf_counter() - t0)
    ev[4].record(st)
    torch.cuda.synchronize()
    dev = [ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(4)]
    print(f"rep {rep}: host us " + " ".join(f"{h * 1e6:7.1f}" for h in host) +
          " | device us " + " ".join(f"{d:7.1f}" for d in dev) + f" | total {sum(dev):.1f}")
