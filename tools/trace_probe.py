"""Phase trace of the C4 plan calls (development aid): per search-level launch,
the time between grid barriers.   python tools/trace_probe.py [config] [reps]"""
import os
import struct
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gen import problems as G  # noqa: E402
from paper_2005_02088_b200 import api  # noqa: E402

NAMES = {0: "start", 1: "reset", 2: "filter", 3: "offsets", 32: "cta-red", 4: "f.stage", 5: "f.static", 6: "f.min", 7: "f.round", 8: "f.compact"}


def show(tag, tr, st):
    print(f"== {tag}: kernel {st['t_ns']/1e3:.1f} us, leaves {st['cum_scored']}, nodes {st['cum_nodes']}")
    line, prev = [], None
    t0s = [0]
    for t, ns in tr:
        if t in (200, 201, 202, 203):
            if t in (200, 202):
                kk = ns & 0xFFFFFFFF
                T = struct.unpack("<f", struct.pack("<I", (0xFFFFFFFF - kk) & 0xFFFFFFFF))[0]
                line.append(f"{'sweep ' if t == 202 else ''}key={kk:#x} (T={T:.6g} | u={kk >> 24},U={kk & 0xFFFFFF})")
            else:
                line.append(f"x={ns}")
            continue
        elif t == 0:
            if line:
                print("   " + " ".join(line))
            line = []
            if prev is not None:
                line.append(f"[gap {(ns - prev)/1e3:.1f}]")
        elif 48 <= t < 64:
            line.append(f"fin{t - 48}={(ns - prev)/1e3:.1f}")
            continue
        elif t >= 120:
            line.append(f"tc{t - 120}={ns / 1e3 if t < 123 else ns:.1f}")
            continue
        elif t >= 112:   # item 1 of warp 0, block 0: SM cycles since the pass start -> us at 1.965 GHz
            line.append(f"w{t - 112}={ns / 1965.0:.2f}")
            continue
        elif t >= 64:
            line.append(f"{['par', 'bat', 'maxb'][(t - 64) // 16]}{t % 16}={ns}")
            continue
        else:
            line.append(f"{NAMES.get(t, 'p%d' % (t - 16))}={(ns - prev)/1e3:.1f}")
        prev = ns
    if line:
        print("   " + " ".join(line))


arg = sys.argv[1] if len(sys.argv) > 1 else "4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if arg.startswith("x"):   # C4-shaped problem of tools/cascade_probe3.py: "x<j>" (seed j, QoS rho)
    j = int(arg[1:])
    rho = {2: 1.0, 3: 1.0, 4: 0.8, 5: 0.9, 6: 1.0, 7: 0.8}[j]
    p = G.build_problem(f"C4x{j}", [["p1", "c2", "m2", "c3", "m1"]], 8, 1, G.POW2_128, 4,
                        G.config_seed(4, j), rho, "v100-dgx2")
else:
    p = G.config_problems(int(arg))[0]
s = api.Session(p, n_loads=1)
for rep in range(reps):
    r = s.plan_max_load()
    show(f"max-load rep {rep}", s.trace(), s.last_stats())
    m = s.plan_min_resource([[0.3 * r.objective] * p.n_apps])[0]
    show(f"min-res rep {rep}", s.trace(), s.last_stats())
torch.cuda.synchronize()
