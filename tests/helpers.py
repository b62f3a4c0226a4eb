"""Shared test helpers: hand-built problems (input packing only, no method arithmetic)."""
import numpy as np

from gen import problems as GP
G = GP

FLAG = {"NO_BW_CAP": G.F_NO_BW_CAP, "NO_CONTENTION": G.F_NO_CONTENTION, "SAT": G.F_SAT,
        "PAPER_GLOBAL": G.F_PAPER_GLOBAL, "EQ2_BUDGET": G.F_EQ2_BUDGET,
        "NO_FILTER": G.F_NO_FILTER, "COMM": G.F_COMM}


def flags_of(spec):
    if spec in (0, None):
        return 0
    if isinstance(spec, int):
        return spec
    f = 0
    for k in str(spec).split("|"):
        f |= FLAG[k.strip()]
    return f


def cluster(C=1, R=100, I=48, BW=1e6, FM=1 << 20, G=1e4):  # noqa: N803
    return GP.Cluster(n_gpus=C, quota_per_gpu=R, max_instances=I, bw_gbs=BW, mem_mib=FM, gflops=G)


def table_from(dur, thr, bw):
    """dur/thr/bw: [n][nS][nQ] nested lists -> float32 [n][nS][nQ][4]."""
    d, t, b = (np.asarray(v, np.float64) for v in (dur, thr, bw))
    tab = np.zeros(d.shape + (4,), np.float32)
    tab[..., 0], tab[..., 1], tab[..., 2] = d, t, b
    return tab


def linear_thr_problem(slopes, quota_grid, C=1, R=100, qos=1e9, Rmax=1):
    """Stage i has thr = slopes[i] * p, dur = 1000 / thr (batch 1), no bandwidth."""
    Q = np.asarray(quota_grid, np.float64)
    thr = [[[s * q for q in Q]] for s in slopes]
    dur = [[[1000.0 / (s * q) for q in Q]] for s in slopes]
    bw = [[[0.0 for _ in Q]] for _ in slopes]
    return G.custom_problem("linear", table_from(dur, thr, bw), quota_grid, [1], [qos],
                            cluster(C=C, R=R), max_replicas=Rmax)


def placement_problem(case):
    """Build the explicit problem of a tests/golden/placement_cases.json case.

    Each stage has exactly one option (its p and N) on a quota grid holding
    every p used, so the single candidate is digits (0, [N-1], [theta])."""
    stages = case["stages"]
    ps = sorted({s["p"] for s in stages})
    n = len(stages)
    Rmax = max(s["N"] for s in stages)
    tab = table_from([[[1.0] * len(ps)]] * n, [[[1.0] * len(ps)]] * n, [[[0.0] * len(ps)]] * n)
    cl = cluster(C=case["C"], FM=case["FM"], I=case.get("I", 48))
    prob = G.custom_problem(case["name"], tab, ps, [1], [1e9], cl, max_replicas=Rmax,
                            weights_mib=[s["W"] for s in stages],
                            act_mib_per_item=[s["A"] for s in stages])
    digits = ([0], [s["N"] - 1 for s in stages], [ps.index(s["p"]) for s in stages])
    return prob, digits


def contention_problem(qos, flags=0):
    """SURVEY.md P-K / tests/golden/contention_example.json."""
    tab = table_from(
        [[[40, 20, 16]], [[40, 20, 16]]],
        [[[25, 50, 62.5]], [[25, 50, 62.5]]],
        [[[8, 16, 20]], [[32, 64, 64]]])
    return G.custom_problem("pk", tab, [25, 50, 75], [1], [qos], cluster(C=1, BW=128.0),
                            bw_sensitivity=[0.0, 1.0], flags=flags_of(flags))


def kappa_split_problem(bwA):
    """tests/golden/kappa_split.json: stage A (1 x 50%) then stage B (3 x 50%) on 2 GPUs."""
    tab = table_from([[[10.0]], [[20.0]]], [[[200.0]], [[50.0]]], [[[bwA]], [[32.0]]])
    return G.custom_problem("ksplit", tab, [50], [1], [1e9], cluster(C=2, BW=128.0), max_replicas=3,
                            bw_sensitivity=[0.0, 1.0])


def min_resource_priority_problem():
    """tests/golden/min_resource_priority.json: thr = p per replica, I = 2, two GPUs."""
    Q = [15, 40, 60]
    tab = table_from([[[1000.0 / q for q in Q]]] * 2, [[[float(q) for q in Q]]] * 2, [[[0.0] * 3]] * 2)
    return G.custom_problem("uU", tab, Q, [1], [1e9], cluster(C=2, I=2), max_replicas=2)
