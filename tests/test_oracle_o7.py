"""Validation of oracle O7 (oracle.search_filtered) against
the plain exhaustive scan (oracle.search) before O7 is trusted for the full C4
golden (tests/golden/make_c4_expected.py).  -m "not gpu".

O7 must return the plain scan's index and objective for every incumbent that is
the objective of a feasible candidate of the space: the tightest one (the
optimum itself, so every filter is exercised at its tie boundary) and looser
ones."""
import json
import os

import numpy as np
import pytest

from gen import problems as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")
f32 = np.float32


def both_policies(oracle, prob, threads=8):
    r = oracle.search(prob, threads=threads)[0]
    if r.index is None:
        f = oracle.search_filtered(prob, T_inc=0.0, threads=threads)
        assert f.index is None
        return
    for T_inc in (r.T, f32(0.5) * f32(r.T), 0.0):
        f = oracle.search_filtered(prob, T_inc=T_inc, threads=threads)
        assert (f.index, f.T, f.u, f.U) == (r.index, r.T, r.u, r.U)
        assert f.n_scanned <= r.n_scanned
    for frac in (0.2, 0.6, 1.0):
        lam = [f32(frac) * f32(r.T)] * prob.n_apps
        rm = oracle.search(prob, "min_resource", loads=[lam], threads=threads)[0]
        wide = (prob.cluster.n_gpus, prob.cluster.n_gpus * prob.cluster.quota_per_gpu)
        if rm.index is None:    # (EQ2_BUDGET) nothing feasible: O7 scores only real candidates
            fm = oracle.search_filtered(prob, "min_resource", load=lam, u_inc=wide[0], U_inc=wide[1],
                                        threads=threads)
            assert fm.index is None
            continue
        incs = [(rm.u, rm.U), wide]
        if oracle.score(prob, r.index, loads=[lam]).level_verdict == [0]:   # a feasible incumbent only
            incs.append((r.u, r.U))
        for inc in incs:
            fm = oracle.search_filtered(prob, "min_resource", load=lam, u_inc=inc[0], U_inc=inc[1],
                                        threads=threads)
            assert (fm.index, fm.u, fm.U) == (rm.index, rm.u, rm.U), (prob.name, frac, inc)


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_o7_equals_plain_scan_configs(oracle, cfg):
    probs = G.config_problems(cfg)
    for prob in (probs if cfg == 1 else probs[:9]):
        both_policies(oracle, prob)


@pytest.mark.parametrize("seed", range(24))
def test_o7_equals_plain_scan_random(oracle, seed):
    rng = np.random.default_rng(700 + seed)
    A = int(rng.integers(1, 3))
    n = int(rng.integers(max(2, A), 5 if A == 1 else 6))
    flag_sets = [0, G.F_NO_BW_CAP, G.F_NO_CONTENTION, G.F_SAT | G.F_NO_BW_CAP, G.F_EQ2_BUDGET,
                 G.F_PAPER_GLOBAL, 0, G.F_COMM]
    flags = flag_sets[seed % len(flag_sets)]
    prob = G.random_small_problem(300 + seed, n_stages=n, n_gpus=int(rng.integers(1, 6)), n_apps=A,
                                  quota_step=int(rng.choice([20, 25, 34])),
                                  batches=(1, 4, 16)[: int(rng.integers(1, 4))],
                                  max_replicas=int(rng.integers(1, 4)),
                                  qos_rho=float(rng.choice([0.8, 1.0, 1.5])), flags=flags)
    if flags & G.F_COMM:
        prob = G.with_comm(prob, seed)
    if oracle.ntot(prob) > 3_000_000:
        pytest.skip("space too large for the in-test plain scan")
    both_policies(oracle, prob)


@pytest.mark.parametrize("name", ["C4r-p1c2m2c3m1", "C5-p2c3m1+p1c1m3"])
def test_o7_equals_plain_scan_large(oracle, name):
    """C4r (8.2e8) and C5 (2.3e9): O7 == the plain-scan goldens of make_expected.py."""
    e = json.load(open(os.path.join(GOLD, f"expected_{name}.json")))
    prob = [p for c in (5, 6) for p in G.config_problems(c) if p.name == name][0]
    assert prob.sha256() == e["sha256"]
    f = oracle.search_filtered(prob, T_inc=e["max_load"]["T"], threads=8)
    assert (f.index, f.T, f.u, f.U) == tuple(e["max_load"][k] for k in ("index", "T", "u", "U"))
    lam = e["min_resource"]["loads"][0]
    r = e["min_resource"]
    fm = oracle.search_filtered(prob, "min_resource", load=lam, u_inc=r["u"], U_inc=r["U"], threads=8)
    assert (fm.index, fm.u, fm.U) == (r["index"], r["u"], r["U"])


def test_o7_filters_are_not_vacuous(oracle):
    """On C3 the tight incumbent leaves a small fraction of the space to score."""
    prob = G.config_problems(3)[0]
    r = oracle.search(prob, threads=8)[0]
    f = oracle.search_filtered(prob, T_inc=r.T, threads=8)
    assert f.n_scanned < r.n_scanned // 100
