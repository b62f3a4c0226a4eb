"""NEXT-3 input side: the paper's per-microservice decision-tree performance
models, trained OFFLINE on profiling samples (one model per
microservice for processing duration, global-memory bandwidth and throughput,
features = input batch size and percentage of computational resources, samples
collected in solo-run mode; L706: "the profiling is done offline").

This module only produces inputs: seeded synthetic "profiling samples" (the
analytic stage model of gen/problems.py measured with multiplicative noise on a
coarse profiling grid) and CART regression trees fitted to them.  Evaluating the
trees on a search grid is the method's step: the CUDA kernel behind
camelot_tables_from_trees does it on the device and oracle.tree_tables on the
CPU.  Tree format (flattened): node k is a leaf when feature[k] < 0 (prediction
value[k]); otherwise x = (s if feature[k] == 0 else p) goes to left[k] when
x <= threshold[k], else to right[k]; children have larger indices than parents.
"""
import dataclasses
from typing import List, Sequence

import numpy as np

from gen import problems as G

PROFILE_BATCH = (1, 2, 4, 8, 16, 32, 64, 128)
PROFILE_QUOTA = tuple(range(10, 101, 10))   # the commented profiling grid of PAPER.md L719


@dataclasses.dataclass
class Tree:
    feature: np.ndarray     # int32[m]  0 = batch, 1 = quota, -1 = leaf
    threshold: np.ndarray   # int32[m]
    left: np.ndarray        # int32[m]
    right: np.ndarray       # int32[m]
    value: np.ndarray       # float32[m]

    @property
    def n_nodes(self) -> int:
        return int(self.feature.shape[0])


def profile_samples(params: dict, bw_gbs: float, seed: int, noise: float = 0.02,
                    batches: Sequence[int] = PROFILE_BATCH, quotas: Sequence[int] = PROFILE_QUOTA,
                    repeats: int = 2):
    """Solo-run measurements of one stage: X int32[m][2] = (s, p), Y float64[m][3] =
    (dur_ms, thr_qps, bw_gbs), each target measured with its own N(1, noise) factor."""
    rng = np.random.Generator(np.random.PCG64(G.SEED_BASE + 970000 + seed))
    X, Y = [], []
    for s in batches:
        for p in quotas:
            dur = params["o"] + s * (params["tc"] / (p / 100.0) ** params["alpha"] + params["tm"])
            thr = 1000.0 * s / dur
            bw = bw_gbs * s * params["tm"] / dur
            for _ in range(repeats):
                f = 1.0 + noise * rng.standard_normal(3)
                X.append((s, p))
                Y.append((dur * f[0], thr * f[1], bw * f[2]))
    return np.asarray(X, np.int32), np.asarray(Y, np.float64)


def train_tree(X: np.ndarray, y: np.ndarray, max_depth: int = 12, min_leaf: int = 1) -> Tree:
    """CART regression (squared error), integer thresholds x <= t between observed
    values; leaves predict the float32 mean of their samples."""
    feat, thr, lef, rig, val = [], [], [], [], []

    def node(idx, depth):
        k = len(feat)
        feat.append(-1)
        thr.append(0)
        lef.append(-1)
        rig.append(-1)
        val.append(np.float32(np.mean(y[idx])))
        if depth >= max_depth or len(idx) < 2 * min_leaf or np.all(y[idx] == y[idx][0]):
            return k
        best = None
        base = np.sum((y[idx] - y[idx].mean()) ** 2)
        for f in (0, 1):
            xs = X[idx, f]
            for t in np.unique(xs)[:-1]:
                lm = xs <= t
                nl, nr = int(lm.sum()), int((~lm).sum())
                if nl < min_leaf or nr < min_leaf:
                    continue
                yl, yr = y[idx][lm], y[idx][~lm]
                sse = np.sum((yl - yl.mean()) ** 2) + np.sum((yr - yr.mean()) ** 2)
                if best is None or sse < best[0] - 1e-12 * base:
                    best = (sse, f, int(t))
        if best is None or best[0] >= base:
            return k
        _, f, t = best
        lm = X[idx, f] <= t
        feat[k], thr[k] = f, t
        lef[k] = node(idx[lm], depth + 1)
        rig[k] = node(idx[~lm], depth + 1)
        return k

    node(np.arange(len(y)), 0)
    return Tree(np.asarray(feat, np.int32), np.asarray(thr, np.int32), np.asarray(lef, np.int32),
                np.asarray(rig, np.int32), np.asarray(val, np.float32))


def stage_trees(prob: "G.Problem", seed: int = 0, noise: float = 0.02, max_depth: int = 12) -> List[Tree]:
    """Three trees per stage (duration, throughput, bandwidth), in table component
    order, trained on that stage's profiling samples."""
    out = []
    for i, params in enumerate(prob.meta["params"]):
        X, Y = profile_samples(params, prob.cluster.bw_gbs, seed * 100 + i, noise)
        for c in range(3):
            out.append(train_tree(X, Y[:, c], max_depth=max_depth))
    return out
