"""NEXT-3: decision-tree performance models (trained offline
L706) turned into the search's predictor tables.

CPU (-m "not gpu"): the oracle's tree traversal against a hand-written tree
with a closed-form piecewise function; the offline CART trainer (gen/dt.py,
input generation) reproduces noise-free training samples exactly and its
predictions on the profiling grid stay within the measurement noise; the
table of a problem built from its trees is a valid problem whose oracle search
runs.  GPU (-m gpu): the device tables equal the oracle's bit for bit on grids
other than the profiling grid, and the search over them equals the oracle.
"""
import numpy as np
import pytest

from gen import dt as D
from gen import problems as G


def hand_tree():
    """f(s, p) = 10 if p <= 50;  5 if p > 50 and s <= 4;  7 otherwise."""
    return D.Tree(feature=np.array([1, -1, 0, -1, -1], np.int32),
                  threshold=np.array([50, 0, 4, 0, 0], np.int32),
                  left=np.array([1, -1, 3, -1, -1], np.int32),
                  right=np.array([2, -1, 4, -1, -1], np.int32),
                  value=np.array([0, 10, 0, 5, 7], np.float32))


def f_closed(s, p):
    return 10.0 if p <= 50 else (5.0 if s <= 4 else 7.0)


def test_tree_eval_closed_form(oracle):
    t = hand_tree()
    for s in (1, 4, 5, 128):
        for p in (1, 50, 51, 100):
            assert oracle.tree_eval(t, s, p) == f_closed(s, p)


def test_trainer_fits_noise_free_samples(oracle):
    """A full CART on noise-free samples reproduces every training point (the
    samples at one (s, p) are identical, so each leaf is their value)."""
    params = G.config_problems(2)[0].meta["params"][0]
    X, Y = D.profile_samples(params, 897.0, seed=3, noise=0.0, repeats=1)
    for c in range(3):
        tr = D.train_tree(X, Y[:, c], max_depth=20)
        got = np.array([oracle.tree_eval(tr, s, p) for s, p in X], np.float32)
        assert np.array_equal(got, Y[:, c].astype(np.float32))


def test_trained_tables_are_a_valid_problem(oracle):
    prob = G.config_problems(2)[5]
    trees = D.stage_trees(prob, seed=1)
    tab = oracle.tree_tables(trees, prob.batch, prob.quota_pct)
    rel = np.abs(tab[..., :3] / prob.table[..., :3] - 1.0)
    on_grid = np.isin(prob.quota_pct, D.PROFILE_QUOTA)
    assert rel[:, :, on_grid].max() < 0.1          # profiling grid: within the noise
    p2 = prob.with_(table=tab)
    assert oracle.validate(p2) == 0
    r = oracle.search(p2, threads=8)[0]
    assert r.index is not None


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
@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_device_tables_equal_oracle(api, oracle, cfg):
    prob = G.config_problems(cfg)[0]
    trees = D.stage_trees(prob, seed=cfg)
    dev = api.tables_from_trees(trees, prob.batch, prob.quota_pct).cpu().numpy()
    ref = oracle.tree_tables(trees, prob.batch, prob.quota_pct)
    assert np.array_equal(dev.view(np.uint32), ref.view(np.uint32))
    one = api.tables_from_trees([hand_tree()] * 3, [1, 4, 5, 128], [1, 50, 51, 100]).cpu().numpy()
    for b, s in enumerate([1, 4, 5, 128]):
        for q, p in enumerate([1, 50, 51, 100]):
            assert one[0, b, q, 0] == f_closed(s, p)


@pytest.mark.gpu
def test_search_over_tree_tables(api, oracle):
    prob = G.config_problems(2)[7]
    trees = D.stage_trees(prob, seed=7)
    tab = api.tables_from_trees(trees, prob.batch, prob.quota_pct).cpu().numpy()
    p2 = prob.with_(table=tab)
    got = api.Session(p2).plan_max_load()
    ref = oracle.search(p2, threads=8)[0]
    assert got.index == ref.index


@pytest.mark.gpu
def test_tables_from_trees_rejects_malformed(api):
    from paper_2005_02088_b200 import _lib as L
    bad = hand_tree()
    bad.left = np.array([0, -1, 3, -1, -1], np.int32)   # a cycle back to the root
    with pytest.raises(L.CamelotError):
        api.tables_from_trees([bad] * 3, [1], [50])
