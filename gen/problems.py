"""Seeded synthetic problem generator (input data only).

This module produces the *inputs* of the allocation search: per-stage predictor
tables on the (batch, SM-quota) grid, linear footprint / FLOP coefficients,
QoS targets and the modeled cluster.  It holds none of the method's arithmetic
(no placement, no contention, no scoring, no enumeration): the CPU oracle
(`oracle/`) and the CUDA path (`paper_2005_02088_b200/`) both consume what it
returns and never share anything else.

Shapes follow the paper's workloads:
  * artifact microservices are PCIe-, compute- and memory-intensive kernels
    with configurable intensity ("c3 is configured to be more
    compute intensive than c2 and c1, m1 is more memory intensive than m2 and
    m3"); 27 artifact pipelines are p_i + c_i + m_i triples;
  * the real benchmarks of Table 1 are 2-stage pipelines
    whose bottleneck is stage 1 (img-to-img) or stage 2 (img-to-text)
    (PAPER.md L384);
  * SM quota is a percentage of the GPU ("The amount of computing
    resources of the entire GPU is 100%"), memory footprint is linear in batch
    (PAPER.md L450-460, L700-703), the MPS client cap is 48,
    BW = 897 GB/s for the V100 of the DGX-2.

The per-stage analytic form is SPEC.md's synthetic ground truth:
    Dur(p, s) = o + s * (t_c / (p/100)^alpha + t_m)          [ms]
    Thr = 1000 * s / Dur                                        [queries/s]
    Bw  = BW * s * t_m / Dur                                    [GB/s]
    gamma = t_m / (t_c + t_m)       (memory-boundness; contention sensitivity)
computed in float64 and rounded ONCE to float32.  The recipe (ranges, levels,
seeds) is stated in DESIGN.md "Input recipe".
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import Dict, List, Optional, Sequence

import numpy as np

# flag bits (numbers only; semantics live in the oracle and in the C ABI)
F_NO_BW_CAP = 1
F_NO_CONTENTION = 2
F_SAT = 4
F_PAPER_GLOBAL = 8
F_EQ2_BUDGET = 16
F_NO_FILTER = 32
F_COMM = 64          # NEXT-2: communication-aware QoS (R29)

SEED_BASE = 200502088 * 1000


@dataclasses.dataclass
class Cluster:
    n_gpus: int            # C
    quota_per_gpu: int     # R (%)
    max_instances: int     # I
    bw_gbs: float          # BW
    mem_mib: int           # F
    gflops: float          # G
    # NEXT-2 (R29/R30): cross-GPU hand-over = D2H + H2D memcpy at 3,150 MB/s each
    # -> 1.575 GB/s; same-GPU IPC hand-over = the 0.02 MB
    # crossover of the two mechanisms (L626): 2 x 0.02 MB / 3.15 GB/s = 0.0127 ms
    link_gbs: float = 1.575
    ipc_ms: float = 0.0127


PRESETS = {
    # V100-SXM3 of the DGX-2 (897 GB/s; L779-780: 48 MPS clients)
    "v100-dgx2": dict(quota_per_gpu=100, max_instances=48, bw_gbs=897.0,
                      mem_mib=32768, gflops=15700.0),
    # a B200 as the modeled device (context preset)
    "b200": dict(quota_per_gpu=100, max_instances=48, bw_gbs=8000.0,
                 mem_mib=184320, gflops=80000.0),
}


def make_cluster(n_gpus: int, preset: str = "v100-dgx2") -> Cluster:
    return Cluster(n_gpus=n_gpus, **PRESETS[preset])


@dataclasses.dataclass
class Problem:
    """One allocation problem (Table 2 variables)."""
    name: str
    n_apps: int
    app_of_stage: np.ndarray      # int32[n]
    qos_ms: np.ndarray            # float32[A]
    quota_pct: np.ndarray         # int32[nQ]   SM-quota grid Q
    batch: np.ndarray             # int32[nS]   batch grid S
    max_replicas: int             # Rmax
    table: np.ndarray             # float32[n][nS][nQ][4] = (dur_ms, thr_qps, bw_gbs, 0)
    weights_mib: np.ndarray       # uint32[n]   W_i
    act_mib_per_item: np.ndarray  # uint32[n]   A_i
    gflop_per_item: np.ndarray    # float32[n]  c_i
    bw_sensitivity: np.ndarray    # float32[n]  gamma_i
    cluster: Cluster
    flags: int = 0
    meta: Optional[dict] = None
    comm_mb_per_item: Optional[np.ndarray] = None   # float32[n] MB per item to the next stage (F_COMM)

    @property
    def n_stages(self) -> int:
        return int(self.app_of_stage.shape[0])

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (self.app_of_stage, self.qos_ms, self.quota_pct, self.batch,
                  self.table, self.weights_mib, self.act_mib_per_item,
                  self.gflop_per_item, self.bw_sensitivity):
            h.update(np.ascontiguousarray(a).tobytes())
        c = self.cluster
        h.update(repr((self.n_apps, self.max_replicas, self.flags, c.n_gpus,
                       c.quota_per_gpu, c.max_instances, c.bw_gbs, c.mem_mib,
                       c.gflops)).encode())
        if self.flags & F_COMM:
            h.update(np.ascontiguousarray(self.comm_mb_per_item, np.float32).tobytes())
            h.update(repr((c.link_gbs, c.ipc_ms)).encode())
        return h.hexdigest()

    def with_(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)


# --------------------------------------------------------------------------
# archetypes
# --------------------------------------------------------------------------
# (t_c ms/item at 100%, t_m ms/item, alpha, o ms) uniform ranges
ARCHETYPES = {
    "c": dict(tc=(2.0, 10.0), tm=(0.05, 0.3), alpha=(0.85, 1.0), o=(1.0, 3.0)),
    "m": dict(tc=(0.2, 1.0), tm=(1.0, 4.0), alpha=(0.3, 0.6), o=(1.0, 3.0)),
    "p": dict(tc=(0.1, 0.5), tm=(0.05, 0.2), alpha=(0.2, 0.5), o=(5.0, 20.0)),
}
# intensity multiplier of the dominant coefficient.  PAPER.md L348: c3 more
# compute intensive than c2, c1; m1 more memory intensive than m2, m3.
LEVEL_MULT = {
    "c": {1: 1.0, 2: 2.0, 3: 4.0},
    "m": {1: 4.0, 2: 2.0, 3: 1.0},
    "p": {1: 1.0, 2: 2.0, 3: 4.0},
}
DOMINANT = {"c": "tc", "m": "tm", "p": "o"}


def _draw_stage(rng: np.random.Generator, kind: str, level: int) -> dict:
    a = ARCHETYPES[kind]
    st = {k: float(rng.uniform(*a[k])) for k in ("tc", "tm", "alpha", "o")}
    st[DOMINANT[kind]] *= LEVEL_MULT[kind][level]
    st["W"] = int(rng.integers(512, 4096 + 1))     # MiB
    st["A"] = int(rng.integers(10, 60 + 1))        # MiB / item
    st["kind"] = f"{kind}{level}"
    return st


def _tables(stages: List[dict], Q: np.ndarray, S: np.ndarray, BW: float):
    n, nS, nQ = len(stages), len(S), len(Q)
    tab = np.zeros((n, nS, nQ, 4), dtype=np.float64)
    for i, st in enumerate(stages):
        p = Q.astype(np.float64)[None, :] / 100.0
        s = S.astype(np.float64)[:, None]
        dur = st["o"] + s * (st["tc"] / p ** st["alpha"] + st["tm"])
        tab[i, :, :, 0] = dur
        tab[i, :, :, 1] = 1000.0 * s / dur
        tab[i, :, :, 2] = BW * s * st["tm"] / dur
    return tab.astype(np.float32)


def build_problem(name: str, apps: Sequence[Sequence[str]], n_gpus: int,
                  quota_step: int, batches: Sequence[int], max_replicas: int,
                  seed: int, qos_rho: float = 1.0, preset: str = "v100-dgx2",
                  flags: int = 0) -> Problem:
    """apps: per app, list of stage archetypes such as "c3", "m1", "p2"."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cl = make_cluster(n_gpus, preset)
    Q = np.arange(quota_step, 101, quota_step, dtype=np.int32)
    S = np.asarray(batches, dtype=np.int32)
    stages, app_of = [], []
    for a, app in enumerate(apps):
        for code in app:
            stages.append(_draw_stage(rng, code[0], int(code[1])))
            app_of.append(a)
    tab = _tables(stages, Q, S, cl.bw_gbs)
    # QoS_a = rho * sum_{i in a} Dur_i(50%, s_mid)   ("hundreds of ms")
    s_mid = float(np.median(S.astype(np.float64)))
    qos = []
    for a in range(len(apps)):
        tot = 0.0
        for i, st in enumerate(stages):
            if app_of[i] == a:
                tot += st["o"] + s_mid * (st["tc"] / 0.5 ** st["alpha"] + st["tm"])
        qos.append(qos_rho * tot)
    gflop = [st["tc"] / 1000.0 * cl.gflops for st in stages]   # C(i,s) = c_i * s
    gamma = [st["tm"] / (st["tc"] + st["tm"]) for st in stages]
    return Problem(
        name=name, n_apps=len(apps),
        app_of_stage=np.asarray(app_of, dtype=np.int32),
        qos_ms=np.asarray(qos, dtype=np.float32),
        quota_pct=Q, batch=S, max_replicas=int(max_replicas),
        table=tab,
        weights_mib=np.asarray([st["W"] for st in stages], dtype=np.uint32),
        act_mib_per_item=np.asarray([st["A"] for st in stages], dtype=np.uint32),
        gflop_per_item=np.asarray(gflop, dtype=np.float32),
        bw_sensitivity=np.asarray(gamma, dtype=np.float32),
        cluster=cl, flags=flags,
        meta=dict(stages=[st["kind"] for st in stages], seed=seed, rho=qos_rho,
                  preset=preset, params=[{k: st[k] for k in ("tc", "tm", "alpha", "o")} for st in stages]),
    )


def config_seed(config: int, j: int = 0) -> int:
    return SEED_BASE + 100 * config + j


POW2_64 = [1, 2, 4, 8, 16, 32, 64]
POW2_128 = [1, 2, 4, 8, 16, 32, 64, 128]
POW2_32 = [1, 2, 4, 8, 16, 32]

# C1: the four 2-stage real benchmarks of Table 1 (shape only; archetype
# assignment is a reading: img2img stage-1 bottleneck, img2text stage-2).
C1_APPS = {
    "img2img": ["c3", "m3"],
    "img2text": ["c1", "c3"],
    "text2img": ["m2", "c2"],
    "text2text": ["c2", "m2"],
}

# per-config QoS rho, chosen once so that each config has a non-trivial feasible
# fraction
RHO = {1: 1.0, 2: 1.0, 3: 1.0, 4: 1.0, 5: 1.0}


def config_problems(config: int, preset: str = "v100-dgx2") -> List[Problem]:
    """The problems of BASELINE.json config `config` (1-based; 6 = C4r, 7 = C4b)."""
    out = []
    if config == 1:
        for j, (nm, app) in enumerate(C1_APPS.items()):
            out.append(build_problem(f"C1-{nm}", [app], 1, 10, POW2_32, 1,
                                     config_seed(1, j), RHO[1], preset))
    elif config == 2:
        j = 0
        for lp in (1, 2, 3):
            for lc in (1, 2, 3):
                for lm in (1, 2, 3):
                    out.append(build_problem(
                        f"C2-p{lp}c{lc}m{lm}", [[f"p{lp}", f"c{lc}", f"m{lm}"]],
                        2, 5, POW2_64, 2, config_seed(2, j), RHO[2], preset))
                    j += 1
    elif config == 3:
        out.append(build_problem("C3-p2c2m2c1", [["p2", "c2", "m2", "c1"]], 4, 5,
                                 POW2_64, 2, config_seed(3), RHO[3], preset))
    elif config == 4:
        out.append(build_problem("C4-p1c2m2c3m1", [["p1", "c2", "m2", "c3", "m1"]],
                                 8, 1, POW2_128, 4, config_seed(4), RHO[4], preset))
    elif config == 5:
        out.append(build_problem("C5-p2c3m1+p1c1m3",
                                 [["p2", "c3", "m1"], ["p1", "c1", "m3"]], 8, 10,
                                 POW2_32, 2, config_seed(5), RHO[5], preset))
    elif config == 7:  # C4b: a second C4 instance (other draws, tighter QoS) where pruning is harder
        out.append(build_problem("C4b-p1c2m2c3m1", [["p1", "c2", "m2", "c3", "m1"]],
                                 8, 1, POW2_128, 4, config_seed(4, 1), 0.8, preset))
    elif config == 6:  # C4r: C4 on a 10% grid (same seed -> same stage draws)
        out.append(build_problem("C4r-p1c2m2c3m1", [["p1", "c2", "m2", "c3", "m1"]],
                                 8, 10, POW2_128, 4, config_seed(4), RHO[4], preset))
    else:
        raise ValueError(f"unknown config {config}")
    return out


def with_comm(prob: Problem, seed: int = 0, mb_range=(0.05, 0.5)) -> Problem:
    """The same problem with NEXT-2 hand-over sizes (MB per item to the next stage,
    drawn uniformly; an image-sized activation per item) and the F_COMM flag."""
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 950000 + seed))
    mb = rng.uniform(*mb_range, size=prob.n_stages).astype(np.float32)
    return prob.with_(comm_mb_per_item=mb, flags=prob.flags | F_COMM)


def custom_problem(name: str, table: np.ndarray, quota_pct: Sequence[int],
                   batch: Sequence[int], qos_ms: Sequence[float],
                   cluster: Cluster, max_replicas: int = 1,
                   app_of_stage: Optional[Sequence[int]] = None,
                   weights_mib: Optional[Sequence[int]] = None,
                   act_mib_per_item: Optional[Sequence[int]] = None,
                   gflop_per_item: Optional[Sequence[float]] = None,
                   bw_sensitivity: Optional[Sequence[float]] = None,
                   flags: int = 0) -> Problem:
    """Pack an explicitly given problem (hand-built test cases and pins)."""
    table = np.ascontiguousarray(table, dtype=np.float32)
    n = table.shape[0]
    app = np.zeros(n, np.int32) if app_of_stage is None else np.asarray(app_of_stage, np.int32)
    z = lambda v, dt, d: np.asarray([d] * n if v is None else v, dtype=dt)
    return Problem(
        name=name, n_apps=int(app.max()) + 1, app_of_stage=app,
        qos_ms=np.asarray(qos_ms, np.float32),
        quota_pct=np.asarray(quota_pct, np.int32), batch=np.asarray(batch, np.int32),
        max_replicas=int(max_replicas), table=table,
        weights_mib=z(weights_mib, np.uint32, 0),
        act_mib_per_item=z(act_mib_per_item, np.uint32, 0),
        gflop_per_item=z(gflop_per_item, np.float32, 1.0),
        bw_sensitivity=z(bw_sensitivity, np.float32, 0.0),
        cluster=cluster, flags=flags)


def random_small_problem(seed: int, n_stages: int = 3, n_gpus: int = 2,
                         n_apps: int = 1, quota_step: int = 25,
                         batches: Sequence[int] = (1, 4), max_replicas: int = 2,
                         preset: str = "v100-dgx2", qos_rho: float = 1.0,
                         flags: int = 0) -> Problem:
    """Random mixed-archetype problem small enough for brute force in tests."""
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 900000 + seed))
    kinds = [f"{'cmp'[int(rng.integers(0, 3))]}{int(rng.integers(1, 4))}"
             for _ in range(n_stages)]
    per_app = [kinds[a::n_apps] for a in range(n_apps)]
    return build_problem(f"rand{seed}", per_app, n_gpus, quota_step, batches,
                         max_replicas, SEED_BASE + 910000 + seed, qos_rho, preset, flags)
