"""Parity of the exhaustive leaf-sweep kernel (NO_FILTER scans, camelot_sweep.cuh)
with the CPU oracle, -m gpu.

The sweep scores every candidate of [lo, hi) with the
scoring of DESIGN.md 3; the bar is the north_star's: chosen index bit-exact,
objective bits identical, feasible count identical (n_feasible is exact in
NO_FILTER mode).  Cases cover both policies, one and two applications,
1..4 replicas, 2..8 GPUs, the NO_CONTENTION / NO_BW_CAP / EQ2_BUDGET flags,
unaligned index slices, and the tree search's flat mode (CAMELOT_NO_SWEEP) as
a second reference on a C4 slice.
"""
import os
import struct

import numpy as np
import pytest
import torch

from gen import problems as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2005_02088_b200 import _lib
    _lib.build()
    from paper_2005_02088_b200 import api as A
    return A


def fb(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


CASES = [  # seed, n, C, A, quota step, batches, Rmax, rho
    (11, 2, 2, 1, 10, (1, 4, 16), 4, 1.0),
    (12, 3, 4, 1, 20, (1, 8), 3, 1.25),
    (13, 4, 8, 1, 25, (2, 8), 2, 1.25),
    (14, 5, 8, 1, 34, (1, 4), 2, 1.5),
    (15, 4, 4, 2, 25, (1, 4), 2, 1.25),
    (16, 6, 8, 2, 50, (1, 8), 2, 1.5),
    (17, 3, 2, 1, 10, (4,), 4, 1.0),
]


def _flat(prob, extra=0):
    return prob.flags | G.F_NO_FILTER | extra


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("extra", [0, G.F_NO_CONTENTION, G.F_NO_BW_CAP])
def test_sweep_max_load(api, oracle, case, extra):
    seed, n, C, A, q, b, R, rho = case
    prob = G.random_small_problem(seed, n_stages=n, n_gpus=C, n_apps=A, quota_step=q, batches=b,
                                  max_replicas=R, qos_rho=rho)
    if oracle.ntot(prob) > 6_000_000:
        pytest.skip("space too large for the in-test oracle")
    flags = _flat(prob, extra)
    got = api.Session(prob, flags=flags).plan_max_load()
    ref = oracle.search(prob, threads=8, flags=flags & ~G.F_NO_FILTER)[0]
    assert got.index == ref.index
    assert got.n_feasible == ref.n_feasible
    if ref.index is not None:
        assert fb(got.objective) == fb(ref.T)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("extra", [0, G.F_EQ2_BUDGET])
def test_sweep_min_resource(api, oracle, case, extra):
    seed, n, C, A, q, b, R, rho = case
    prob = G.random_small_problem(seed, n_stages=n, n_gpus=C, n_apps=A, quota_step=q, batches=b,
                                  max_replicas=R, qos_rho=rho)
    if oracle.ntot(prob) > 6_000_000:
        pytest.skip("space too large for the in-test oracle")
    base = oracle.search(prob, threads=8)[0]
    if base.index is None:
        pytest.skip("infeasible problem")
    lam = [[np.float32(0.3) * np.float32(base.T)] * A]
    flags = _flat(prob, extra)
    got = api.Session(prob, n_loads=1, flags=flags).plan_min_resource(lam)[0]
    ref = oracle.search(prob, "min_resource", loads=lam, threads=8, flags=flags & ~G.F_NO_FILTER)[0]
    assert got.index == ref.index
    if ref.index is not None:
        assert (got.gpus_used, got.quota_used) == (ref.u, ref.U)


@pytest.mark.parametrize("cfg", [2, 6])
def test_sweep_unaligned_slices(api, oracle, cfg):
    """Index slices that start and end inside a parent's leaf range."""
    prob = G.config_problems(cfg)[0]
    nt = oracle.ntot(prob)
    rng = np.random.default_rng(cfg)
    s = api.Session(prob, flags=_flat(prob))
    for _ in range(3):
        lo = int(rng.integers(0, nt - 300000))
        hi = lo + int(rng.integers(1, 300000))
        got = s.plan_max_load(lo=lo, hi=hi)
        ref = oracle.search(prob, lo=lo, hi=hi, threads=8)[0]
        assert got.index == ref.index and got.n_feasible == ref.n_feasible, (lo, hi)


def test_sweep_c4_slice_vs_oracle_and_tree(api, oracle):
    """A 2^24-candidate slice of C4 (8 GPUs, 4 replicas, 1% grid): sweep == oracle,
    and == the tree search's flat mode (CAMELOT_NO_SWEEP)."""
    prob = G.config_problems(4)[0]
    nt = oracle.ntot(prob)
    O = prob.max_replicas * len(prob.quota_pct)
    lo = nt // 3 - (nt // 3) % O + 123
    hi = lo + (1 << 24)
    s = api.Session(prob, flags=_flat(prob))
    got = s.plan_max_load(lo=lo, hi=hi)
    ref = oracle.search(prob, lo=lo, hi=hi, threads=8)[0]
    assert got.index == ref.index and got.n_feasible == ref.n_feasible
    assert fb(got.objective) == fb(ref.T)
    os.environ["CAMELOT_NO_SWEEP"] = "1"
    try:
        tree = s.plan_max_load(lo=lo, hi=hi)
    finally:
        del os.environ["CAMELOT_NO_SWEEP"]
    assert tree.index == got.index and tree.n_feasible == got.n_feasible


@pytest.mark.parametrize("case", CASES[:4])
@pytest.mark.parametrize("mode", ["permuted", "scaled"])
def test_sweep_bandwidth_rows(api, oracle, case, mode):
    """permuted: leaf rows whose bandwidth is not non-decreasing in the quota (possible
    for tables built from decision trees) take the sweep's per-quota capacity path
    instead of the quota breakpoints -- every second batch row of every stage gets its
    bandwidths permuted along the quota grid.  scaled: every bandwidth x3 (rows stay
    non-decreasing), so the bandwidth cap binds often and the breakpoint searches
    decide.  The result is the oracle's either way."""
    seed, n, C, A, q, b, R, rho = case
    prob = G.random_small_problem(seed, n_stages=n, n_gpus=C, n_apps=A, quota_step=q, batches=b,
                                  max_replicas=R, qos_rho=rho)
    if oracle.ntot(prob) > 6_000_000:
        pytest.skip("space too large for the in-test oracle")
    rng = np.random.default_rng(seed)
    tab = prob.table.copy()
    if mode == "scaled":
        tab[..., 2] *= np.float32(3.0)
    else:
        for i in range(tab.shape[0]):
            for bi in range(0, tab.shape[1], 2):
                tab[i, bi, :, 2] = tab[i, bi, rng.permutation(tab.shape[2]), 2] * np.float32(1.5)
    prob = prob.with_(table=tab)
    flags = _flat(prob)
    got = api.Session(prob, flags=flags).plan_max_load()
    ref = oracle.search(prob, threads=8)[0]
    assert got.index == ref.index and got.n_feasible == ref.n_feasible
    if ref.index is None:
        return
    lam = [[np.float32(0.3) * np.float32(ref.T)] * A]
    got = api.Session(prob, n_loads=1, flags=flags).plan_min_resource(lam)[0]
    ref = oracle.search(prob, "min_resource", loads=lam, threads=8)[0]
    assert got.index == ref.index
