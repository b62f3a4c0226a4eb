import os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import torch
from gen import problems as G
from paper_2005_02088_b200 import api
p = G.config_problems(4)[0]
s = api.Session(p, n_loads=1); s.upload()
st = torch.cuda.current_stream()
for _ in range(5): s.plan_max_then_min(0.3, resident=True)
W, D = [], []
for _ in range(30):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); t0 = time.perf_counter()
    s.plan_max_then_min(0.3, resident=True)
    t1 = time.perf_counter(); e1.record(st); torch.cuda.synchronize()
    W.append((t1 - t0) * 1e3); D.append(e0.elapsed_time(e1))
print("wall median %.4f min %.4f | device median %.4f min %.4f" % (statistics.median(W), min(W), statistics.median(D), min(D)))
