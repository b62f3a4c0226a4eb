"""NEXT-4: tail-latency simulation of chosen plans (reading R32: Poisson
arrivals, batching at the entry, round-robin FIFO replicas with
the plan's contended durations, hand-overs under COMM; p99 = the QoS metric,
L514 / L834).

CPU pins of the oracle simulator (-m "not gpu"): without queueing the latency
of every query is the predicted latency sum; a single FIFO stage with
deterministic service is an M/D/1 queue whose mean sojourn time is given by
Pollaczek-Khinchine (D (1 + rho / (2 (1 - rho)))); with a coupled random stream,
latencies only grow with the load.  GPU parity (-m gpu): p99 and mean of the
device simulator equal the oracle's (same counter-based streams) within 1e-9
relative (the only difference is the libm log), and the Camelot-NC effect
shows at high load.
"""
import numpy as np
import pytest

from gen import problems as G
from tests import helpers as H


def single_stage(D=10.0, N=1):
    tab = H.table_from([[[D]]], [[[1000.0 / D]]], [[[0.0]]])
    return G.custom_problem("mdl", tab, [100], [1], [1e9], H.cluster(C=1), max_replicas=N)


def batch1(prob):
    """The problem restricted to batch size 1 (no batch-formation wait)."""
    b = int(np.nonzero(prob.batch == 1)[0][0])
    return prob.with_(batch=prob.batch[b:b + 1], table=np.ascontiguousarray(prob.table[:, b:b + 1]))


def test_sim_no_queueing_is_predicted_sum(oracle):
    prob = batch1(G.config_problems(2)[2])
    r = oracle.search(prob, threads=8)[0]
    s = oracle.score(prob, r.index)
    # load 1e-3 of the bottleneck: fewer than 1% of the queries wait at all, so the
    # p99 is the predicted sum up to the rounding of the (large) arrival times
    p99, mean = oracle.simulate(prob, r.index, [1e-3 * s.T], 20000, 0)
    assert abs(p99[0] - s.Lsum[0]) <= 1e-7 * s.Lsum[0]
    assert s.Lsum[0] * (1 - 1e-7) <= mean[0] <= s.Lsum[0] * (1 + 1e-3)


def test_sim_md1_pollaczek_khinchine(oracle):
    D = 10.0
    prob = single_stage(D)
    for rho_ in (0.3, 0.5, 0.8):
        lam = rho_ * 1000.0 / D
        _, mean = oracle.simulate(prob, 0, [lam], 1_000_000, 50_000, seed=7)
        pk = D * (1.0 + rho_ / (2.0 * (1.0 - rho_)))
        assert abs(mean[0] / pk - 1.0) < 0.03, (rho_, mean[0], pk)


def test_sim_monotone_in_load(oracle):
    """With batch size 1 and a coupled stream (gaps scale as 1/load), the Lindley
    recursion makes every latency non-decreasing in the load.  (With batching at
    the entry this does not hold: the batch-formation wait shrinks with the load.)"""
    prob = batch1(G.config_problems(2)[4])
    r = oracle.search(prob, threads=8)[0]
    prev = (0.0, 0.0)
    for f in (0.2, 0.5, 0.8, 0.95):
        p99, mean = oracle.simulate(prob, r.index, [f * r.T], 50000, 5000, seed=3)
        assert p99[0] >= prev[0] and mean[0] >= prev[1]
        prev = (p99[0], mean[0])


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2005_02088_b200 import _lib
    _lib.build()
    from paper_2005_02088_b200 import api as A
    return A


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,j", [(1, 0), (2, 3), (2, 11), (3, 0)])
def test_sim_gpu_parity(api, oracle, cfg, j):
    prob = G.config_problems(cfg)[j]
    r = oracle.search(prob, threads=8)[0]
    beta, rho, theta = oracle.decode(prob, r.index)
    batch = [int(prob.batch[b]) for b in beta]
    reps = [int(v) + 1 for v in rho]
    quota = [int(prob.quota_pct[t]) for t in theta]
    s = api.Session(prob)
    for f in (0.3, 0.9):
        lam = [f * r.T] * prob.n_apps
        p99, mean = s.simulate(batch, reps, quota, lam, 30000, 3000, seed=11, n_sims=3)
        for k in range(3):
            rp, rm = oracle.simulate(prob, r.index, lam, 30000, 3000, seed=11, sim=k)
            for a in range(prob.n_apps):
                assert abs(p99[k][a] - rp[a]) <= 1e-9 * rp[a]
                assert abs(mean[k][a] - rm[a]) <= 1e-9 * rm[a]


@pytest.mark.gpu
def test_sim_camelot_nc_effect(api, oracle):
    """Camelot-NC at the level of the simulated tail (reading R18): the plan chosen
    by the contention-blind search, replayed with the contended durations, has a
    simulated p99 at least as long as the contention-blind prediction of it
    (service times only grow, and the queueing recursion is monotone in them),
    and strictly longer for a plan with co-located stages."""
    for prob in G.config_problems(2)[:10]:
        blind = oracle.search(prob, threads=8, flags=prob.flags | G.F_NO_CONTENTION)[0]
        if blind.index is None:
            continue
        beta, rho, theta = oracle.decode(prob, blind.index)
        plan = ([int(prob.batch[beta[0]])], [int(v) + 1 for v in rho], [int(prob.quota_pct[t]) for t in theta])
        lam = [0.8 * blind.T]
        with_c, _ = api.Session(prob).simulate(*plan, lam, 20000, 2000, seed=5)
        without, _ = api.Session(prob, flags=prob.flags | G.F_NO_CONTENTION).simulate(*plan, lam, 20000, 2000, seed=5)
        assert with_c[0][0] >= without[0][0]
        s = oracle.score(prob, blind.index)
        if max(s.kappa) > 1.0:
            assert with_c[0][0] > without[0][0]
            return
    pytest.skip("no co-located contention-blind plan among the samples")
