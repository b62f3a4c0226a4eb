"""Benchmark of the contention-aware allocation search (BASELINE.json metric:
"allocation candidates/sec and time-to-optimal-plan at 1/2/4/8 B200").

One step = one full plan of BASELINE config C4 (5-stage pipeline, 8 modeled
GPUs, 1% SM-quota grid, batch 1..128, up to 4 replicas/stage: 8.192e13
candidates per policy) for BOTH policies: max peak load (Eq. 1), then minimum
resource at 30% of that peak (Eq. 3).  Each policy is an exact
search of the whole space; value = candidates covered per second
(2 x 8.192e13 / step time), whole job.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1: one rank per GPU (bench.py re-launches itself under
torch.distributed.run when WORLD_SIZE is unset); every rank searches its shard
(chunk c -> rank c mod N) and ONE all_reduce(MIN) of packed int64 keys per
policy goes over NCCL.  With fewer visible GPUs than ranks (e.g. proving the
launcher on a 1-GPU lease) the ranks share devices and the keys go over gloo
(--backend gloo; NCCL forbids two ranks on one device).  --impl reference
times the CPU oracle (oracle/) on a bounded slice of the same workload on the
host cores.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "allocation candidates/sec (time-to-optimal-plan, both policies)"
UNIT = "candidates/s"
WORKLOAD = "C4: 5-stage p1-c2-m2-c3-m1 pipeline, 8 modeled V100 (BW 897 GB/s), 1% quota grid, " \
           "batch 1..128 (pow2), <=4 replicas/stage; max-load then min-resource at 0.3*T*"
LOW_LOAD = 0.3   # low load = 30% of the peak
TRAFFIC_CSV = "r02_v16_ncu_search_raw.csv"   # committed ncu --set full capture of the search launches
FLAT_CSV = "r02_v16_ncu_flat_raw.csv"        # committed ncu --set full capture of the flat sweep (same slice)


def ncu_metric(name, key, launch=0):
    """One metric of one launch of a committed ncu --page raw --csv capture (None if absent)."""
    import csv
    try:
        rows = list(csv.reader(open(os.path.join(ROOT, "profiles", name))))
        v = rows[2 + launch][rows[0].index(key)]
        return float(v.replace(",", ""))
    except (OSError, ValueError, IndexError):
        return None


def ncu_traffic(name, launches_per_step=None):
    """dram__bytes_read.sum + dram__bytes_write.sum summed over the first
    `launches_per_step` launches (one step) of a committed ncu --page raw --csv
    capture under profiles/ (all launches if None; None if the file is absent)."""
    import csv
    path = os.path.join(ROOT, "profiles", name)
    try:
        rows = list(csv.reader(open(path)))
        hdr, units, data = rows[0], rows[1], rows[2:]
        if launches_per_step:
            data = data[:launches_per_step]
        tot = 0.0
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(key)
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1.0)
            tot += sum(float(r[i]) * scale for r in data if r[i] not in ("", "n/a"))
        return tot, "profiles/" + name
    except (OSError, ValueError, IndexError):
        return None, None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region."""

    def __init__(self, dev):
        self.dev, self.samples, self.proc = dev, [], None

    def __enter__(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active," \
            "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
            "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        time.sleep(0.15)
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 3 + k and s[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


T_START = time.perf_counter()


def log(msg):
    """progress on stderr (the JSON line alone goes to stdout)"""
    print(f"[bench {time.perf_counter() - T_START:7.1f}s] {msg}", file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_relaunch(args):
    """--gpus N > 1 without a torchrun environment: re-launch this script with
    N ranks on this node (the driver's own launch sets WORLD_SIZE itself)."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "camelot":
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_reference_leg(prob, args, as_main):
    """The CPU oracle (plain exhaustive scan, as it stands) on a bounded slice of
    the workload: on all host cores, and single-threaded.  Returns the JSON fields."""
    from oracle import oracle as O
    threads = os.cpu_count() or 1
    nt = O.ntot(prob)
    lo = nt // 3
    t0 = time.perf_counter()
    O.search(prob, lo=lo, hi=lo + 200_000, threads=threads)
    rate0 = 200_000 / max(1e-6, time.perf_counter() - t0)
    steps = args.steps if as_main else 1
    warm = args.warmup if as_main else 0
    # the reference arm's whole run stays within ~2.5 minutes for any --steps / --warmup
    per_step = max(0.5, min(args.ref_seconds, 150.0 / (steps + warm))) if as_main else args.cpu_seconds
    n = int(max(100_000, min(5e9, rate0 * per_step)))
    times = []
    for s in range(warm + steps):
        a = lo + s * n
        t0 = time.perf_counter()
        O.search(prob, lo=a, hi=a + n, threads=threads)
        dt = time.perf_counter() - t0
        if s >= warm:
            times.append(dt)
    rate = n * len(times) / sum(times)
    # single thread on a smaller sample of the same slice
    n1 = int(max(20_000, min(2e8, rate0 / threads * args.cpu1_seconds)))
    t0 = time.perf_counter()
    O.search(prob, lo=lo, hi=lo + n1, threads=1)
    rate1 = n1 / (time.perf_counter() - t0)
    sample = f"max-load exhaustive scan of {n} consecutive C4 candidates per step from index {lo} on {threads} " \
             f"threads, and of {n1} candidates on 1 thread (one policy; full C4 = 2 x {nt:.4g} candidates)"
    return dict(value=rate, unit=UNIT, cores=threads, kind="oracle", sample=sample,
                single_thread_value=rate1, cpu_model=cpu_model(),
                ms_per_step=1000 * statistics.mean(times), n_per_step=n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="camelot", choices=["camelot", "reference"])
    ap.add_argument("--config", type=int, default=4, help="BASELINE config (default 4 = C4)")
    ap.add_argument("--backend", default=None, choices=["nccl", "gloo"],
                    help="key all-reduce backend (default: nccl with one GPU per rank, else gloo)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="cpu_baseline sample budget")
    ap.add_argument("--cpu1-seconds", type=float, default=4.0, help="single-thread oracle sample budget")
    ap.add_argument("--ref-seconds", type=float, default=8.0, help="--impl reference seconds per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flat", action="store_true", help="skip the flat-scan roofline leg")
    ap.add_argument("--no-sa", action="store_true", help="skip the simulated-annealing baseline")
    ap.add_argument("--no-comm", action="store_true", help="skip the NEXT-2 communication-aware leg")
    ap.add_argument("--no-sim", action="store_true", help="skip the NEXT-4 tail-simulation leg")
    ap.add_argument("--no-hard", action="store_true", help="skip the second C4 instance (C4b)")
    ap.add_argument("--no-b200", action="store_true", help="skip C4 on the modeled-B200 cluster preset")
    ap.add_argument("--sa-chains", type=int, default=4096)
    ap.add_argument("--sa-iters", type=int, default=500)
    ap.add_argument("--flat-config", type=int, default=4, help="config of the flat scan (4 = C4)")
    ap.add_argument("--flat-slice", type=int, default=1 << 31, help="candidates of the flat-scan slice (0 = all)")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "timing rules: >= 3 warm-up steps"
    maybe_relaunch(args)

    from gen import problems as G
    prob = G.config_problems(args.config)[0]
    rank, world, local = dist_env()

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_reference_leg(prob, args, as_main=True)
        line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": WORKLOAD, "problem": prob.name, "sha256": prob.sha256(),
                           "l2": "n/a (CPU)"},
                "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "oracle",
                                 "sample": r["sample"], "single_thread_value": r["single_thread_value"],
                                 "cpu_model": r["cpu_model"]},
                "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2005_02088_b200 import _lib as L
    from paper_2005_02088_b200 import api

    ndev = torch.cuda.device_count()
    backend = args.backend or ("nccl" if ndev >= world else "gloo")
    dev_idx = local % max(1, ndev)
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    log("session upload")
    stream = torch.cuda.current_stream(dev)
    sess = api.Session(prob, device=dev_idx, n_loads=1)
    sess.upload()
    torch.cuda.synchronize()

    def ntot_of(p):
        t = 1
        for _ in range(p.n_apps):
            t *= len(p.batch)
        for _ in range(p.n_stages):
            t *= p.max_replicas * len(p.quota_pct)
        return t

    ntot = ntot_of(prob)

    def all_reduce_min(keys):
        """THE collective of the path: one all_reduce(MIN) of the packed keys."""
        if world > 1:
            if backend == "nccl":
                dist.all_reduce(keys, op=dist.ReduceOp.MIN)
            else:   # gloo: host-staged (ranks may share one device)
                h = keys.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.MIN)
                keys.copy_(h)

    def max_over_ranks(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if world > 1:
            dist.barrier()

    def step(s_, p_, resident=True, marks=None):
        """Both policies, whole hot path.  One rank: camelot_plan_max_then_min (the
        low load derived on the device, one host synchronisation).  N ranks, or
        marks given (phase breakdown): per policy search shard -> allreduce ->
        finalize.  marks: optional list collecting CUDA events between the phases."""
        if world == 1 and marks is None:
            return s_.plan_max_then_min(LOW_LOAD, resident=resident)

        def mark():
            if marks is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                marks.append(e)
        mark()
        k1 = s_.search_local(L.POLICY_MAX_LOAD, rank=rank, world=world, resident=resident)
        mark()
        all_reduce_min(k1)
        mark()
        pm = s_.finalize(L.POLICY_MAX_LOAD, k1, rank=rank, world=world)[0]
        mark()
        lam = [[LOW_LOAD * pm.objective] * p_.n_apps]
        k2 = s_.search_local(L.POLICY_MIN_RESOURCE, lam, rank=rank, world=world, resident=True)
        mark()
        all_reduce_min(k2)
        mark()
        pr = s_.finalize(L.POLICY_MIN_RESOURCE, k2, lam, rank=rank, world=world)[0]
        mark()
        return pm, pr

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    log(f"rank {rank}/{world} on cuda:{dev_idx} ({backend if world > 1 else 'single'}): warm-up")
    for _ in range(args.warmup):
        step(sess, prob)
    torch.cuda.synchronize()
    barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    wall = []
    launches0 = L.lib().camelot_kernel_launches()
    plans = []
    with ClockSampler(dev_idx) as clk:
        torch.cuda.synchronize()
        barrier()
        for s in range(args.steps):
            flush.fill_(s & 0xFF)            # L2 flush between timed steps (not timed)
            t0 = time.perf_counter()
            ev[s][0].record(stream)
            pm, pr = step(sess, prob)        # plans land in host memory (finalize synchronises)
            ev[s][1].record(stream)
            wall.append((time.perf_counter() - t0) * 1e3)
            plans.append((pm, pr))
        torch.cuda.synchronize()
        barrier()
    launches = (L.lib().camelot_kernel_launches() - launches0) / args.steps
    ms = [a.elapsed_time(b) for a, b in ev]
    ms_step = max_over_ranks(statistics.mean(ms))
    ms_med, ms_min = max_over_ranks(statistics.median(ms)), max_over_ranks(min(ms))
    wall_med, wall_min = max_over_ranks(statistics.median(wall)), max_over_ranks(min(wall))
    covered = 2 * ntot
    value = covered / (ms_step / 1000.0)
    # the search's device time and evaluation count come back in the plans
    evals = sum(pm.n_evaluated + pr.n_evaluated for pm, pr in plans) / args.steps
    k_ns = sum(pm.search_ns + pr.search_ns for pm, pr in plans) / args.steps

    log(f"timed steps done: {statistics.median(ms):.3f} ms median")
    # fixed costs per N: one instrumented step, CUDA events between the phases
    marks = []
    flush.fill_(0)
    barrier()
    step(sess, prob, marks=marks)
    torch.cuda.synchronize()
    names = ["search_local_max_load", "allreduce_max_load", "finalize_max_load",
             "search_local_min_resource", "allreduce_min_resource", "finalize_min_resource"]
    phases = {nm: max_over_ranks(marks[i].elapsed_time(marks[i + 1])) for i, nm in enumerate(names)}
    tr = sess.trace()   # the min-resource search of that step: cascade levels vs main pass
    starts = [ns for t, ns in tr if t == 0]
    ends = [ns for t, ns in tr if t < 64]
    if len(starts) >= 1 and ends:
        phases["min_resource_coop_cascade_levels_ms"] = (starts[-1] - starts[0]) / 1e6
        phases["min_resource_coop_main_pass_ms"] = (ends[-1] - starts[-1]) / 1e6
    phases["note"] = ("device time per phase of one step through the per-policy API (search_local -> "
                      "allreduce -> finalize, max over ranks; the timed N=1 step is the fused "
                      "camelot_plan_max_then_min instead); search_local = incumbent cascade "
                      "(replicated on every rank) + this rank's shard of the main pass; finalize = resolve + "
                      "chunk re-scan (Ntot > 2^32, N > 1) + plan scoring + D2H and the host turnaround")

    # e2e: through the public API with the problem copied from pinned host
    # memory every step (not resident) and the plans read back to the host
    e2e = None
    if not args.no_e2e:
        log("e2e leg")
        for _ in range(2):
            step(sess, prob, resident=False)
        torch.cuda.synchronize()
        barrier()
        ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for s in range(args.steps):
            flush.fill_(s & 0xFF)
            ee[s][0].record(stream)
            step(sess, prob, resident=False)
            ee[s][1].record(stream)
        torch.cuda.synchronize()
        barrier()
        e_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in ee))
        h2d = prob.table.nbytes + prob.quota_pct.nbytes + prob.batch.nbytes + 4 * prob.n_apps
        d2h = 2 * C_sizeof_plan()
        e2e = {"value": covered / (e_ms / 1000.0), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # roofline of the dominant kernel (the main search kernel): ALU/issue bound
    peaks = load_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    clocks = clk.summary()
    ops_per_eval = algorithmic_ops_per_eval(prob)
    achieved = ops_per_eval * evals / (k_ns * 1e-9) / 1e12 if k_ns else None
    peak = n_sm * 4 * 32 * sm_max * 1e6 / 1e12          # lane-instructions/s (issue bound)
    traffic, traffic_src = ncu_traffic(TRAFFIC_CSV, 2)   # one launch per policy
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "traffic_note": f"DRAM bytes read+written per step (sum over the search launches of one step) "
                            f"from the committed ncu --set full capture {traffic_src}; algorithmic bytes ~0 "
                            f"(64 KB of tables, L2/SMEM resident)" if traffic else None,
            "kernel": "pruned search (incumbent cascade and main pass, both policies)",
            "ops_per_eval": ops_per_eval, "evals_per_step": evals,
            "kernel_ms_per_step": k_ns / 1e6,
            "kernel_share_of_step": (k_ns / 1e6) / ms_step if ms_step else None,
            "peak_note": f"{n_sm} SMs x 4 SMSP x 32 lanes x {sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)"}

    # flat exhaustive scan (NO_FILTER: every candidate placed and scored, no
    # pruning), sharded like the main search: chunks dealt round-robin over the
    # ranks, ONE allreduce-min, finalize.  The sustained hot loop, for the
    # issue-roofline view and the near-linear scaling leg.
    flat = None
    if not args.no_flat:
        log("flat-scan leg")
        fp = G.config_problems(args.flat_config)[0]
        fs = api.Session(fp, device=dev_idx, flags=fp.flags | L.F_NO_FILTER)
        fnt = ntot_of(fp)
        flo = (fnt // 3) - (fnt // 3) % (fp.max_replicas * len(fp.quota_pct))
        fhi = min(fnt, flo + args.flat_slice) if args.flat_slice else fnt

        def flat_step():
            k = fs.search_local(L.POLICY_MAX_LOAD, rank=rank, world=world, lo=flo, hi=fhi)
            all_reduce_min(k)
            return k

        for _ in range(2):
            k = flat_step()
            fr = fs.finalize(L.POLICY_MAX_LOAD, k, rank=rank, world=world, lo=flo, hi=fhi)[0]
        torch.cuda.synchronize()
        fts, fsc, fk = [], [], []
        for _ in range(3):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            k = flat_step()
            e1.record(stream)
            st = fs.last_stats()      # this rank's scored leaves and kernel time (synchronises)
            fts.append(e0.elapsed_time(e1))
            fk.append(st["t_ns"] / 1e6)
            fsc.append(st["cum_scored"])
        fr = fs.finalize(L.POLICY_MAX_LOAD, k, rank=rank, world=world, lo=flo, hi=fhi)[0]
        ft_local = statistics.median(fts)
        ft = max_over_ranks(ft_local)
        scored_local = statistics.median(fsc)
        scored_all = scored_local
        if world > 1:
            t = torch.tensor([scored_local], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
            dist.all_reduce(t)
            scored_all = float(t.item())
        fops = algorithmic_ops_per_eval(fp)
        kern = max_over_ranks(statistics.median(fk))
        fach = fops * scored_all / world / (kern * 1e-3) / 1e12
        flat = {"workload": f"{fp.name} max-load, NO_FILTER exhaustive scan of indices [{flo}, {fhi}) "
                            f"({fhi - flo:.4g} candidates), sharded over {world} rank(s)",
                "index": fr.index, "ms": ft, "candidates_per_s": (fhi - flo) / (ft * 1e-3),
                "leaves_scored_per_s": scored_all / (ft * 1e-3),
                "per_rank_leaves_scored_per_s": scored_local / (ft_local * 1e-3),
                "roofline": {"bound": "alu", "achieved": fach, "peak": peak, "unit": "Tops/s",
                             "frac": fach / peak, "ops_per_eval": fops,
                             "note": "per GPU: leaf evaluations x ops_per_eval / sweep kernel time"}}
        # SURVEY.md 8(d)'s issue-bound fraction: scored/s / (issue peak / measured thread-instructions
        # per scored leaf), from the committed ncu capture of the same slice
        ti = ncu_metric(FLAT_CSV, "thread_inst_executed")
        ia = ncu_metric(FLAT_CSV, "smsp__issue_active.avg.pct_of_peak_sustained_active")
        if ti and scored_all:
            ipl = ti / (scored_all / world)
            flat["issue"] = {"thread_instructions_per_leaf": ipl,
                             "frac": (scored_all / world) / (kern * 1e-3) * ipl / (peak * 1e12),
                             "issue_active_pct": ia, "source": "profiles/" + FLAT_CSV,
                             "note": "leaves/s x measured thread-instructions per leaf / issue peak"}

    # further C4 instances, timed like the headline step (median / min):
    #  * C4b: other draws, QoS 0.8x -- pruning is much harder;
    #  * C4 on the modeled-B200 cluster preset (8 TB/s, 180 GiB per GPU; SURVEY.md 8(d):
    #    "C4 is also run with b200") -- memory never binds.
    def instance_leg(hp):
        hs = api.Session(hp, device=dev_idx, n_loads=1)
        hs.upload()
        for _ in range(3):
            step(hs, hp)
        torch.cuda.synchronize()
        hms, hev = [], []
        for s in range(max(3, min(args.steps, 10))):
            flush.fill_(s & 0xFF)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hm, hr = step(hs, hp)
            e1.record(stream)
            torch.cuda.synchronize()
            hms.append(e0.elapsed_time(e1))
            hev.append(hm.n_evaluated + hr.n_evaluated)
        hmed = max_over_ranks(statistics.median(hms))
        return {"problem": hp.name, "sha256": hp.sha256(), "ms_per_step_median": hmed,
                "ms_per_step_min": max_over_ranks(min(hms)),
                "candidates_per_s": 2 * ntot_of(hp) / (hmed * 1e-3), "evals_per_step": statistics.median(hev),
                "max_load": {"index": hm.index, "T": hm.objective},
                "min_resource": {"index": hr.index, "gpus_used": hr.gpus_used, "quota_used": hr.quota_used}}

    hard = b200 = None
    if not args.no_hard:
        log("C4b leg")
        hard = instance_leg(G.config_problems(7)[0])
    if not args.no_b200:
        log("C4 b200-preset leg")
        bp = G.config_problems(4, "b200")[0]
        b200 = instance_leg(bp.with_(name=bp.name + "-b200"))

    # the paper's own solver (simulated annealing, NEXT-1) on the same device:
    # time and quality against the exact plans of this step
    pm, pr = plans[-1]
    sa = None
    if not args.no_sa and rank == 0:
        log("SA leg")
        ss = api.Session(prob, device=dev_idx, n_loads=1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r1 = ss.sa(L.POLICY_MAX_LOAD, seed=1, chains=args.sa_chains, iters=args.sa_iters, p0=0.3, cool=0.995)
        lam_sa = [[LOW_LOAD * pm.objective] * prob.n_apps]
        r2 = ss.sa(L.POLICY_MIN_RESOURCE, lam_sa, seed=2, chains=args.sa_chains, iters=args.sa_iters, p0=0.3,
                   cool=0.995)
        torch.cuda.synchronize()
        sa = {"chains": args.sa_chains, "iters": args.sa_iters, "p0": 0.3, "cool": 0.995,
              "ms_both_policies": (time.perf_counter() - t0) * 1e3,
              "max_load": {"T_sa": r1.objective, "T_exact": pm.objective,
                           "gap_pct": 100.0 * (1.0 - r1.objective / pm.objective) if r1.index is not None else None,
                           "same_plan_as_exact": r1.index == pm.index},
              "min_resource": {"u_U_sa": [r2.gpus_used, r2.quota_used] if r2.index is not None else None,
                               "u_U_exact": [pr.gpus_used, pr.quota_used],
                               "same_plan_as_exact": r2.index == pr.index},
              "note": "PAPER.md L880-888 solver, reading R13; chains bit-identical to the oracle SA"}

    # NEXT-2 on the same workload: the communication-aware QoS (flag COMM, R29) with
    # the generator's hand-over sizes; both policies, exact, time of the step
    comm = None
    if not args.no_comm and rank == 0:
        log("COMM leg")
        cp = G.with_comm(prob, 4)
        cs = api.Session(cp, device=dev_idx, n_loads=1)
        cts = []
        for rep in range(4):
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            c1 = cs.plan_max_load()
            c2 = cs.plan_min_resource([[LOW_LOAD * c1.objective] * cp.n_apps])[0]
            ev1.record()
            torch.cuda.synchronize()
            if rep:
                cts.append(ev0.elapsed_time(ev1))
        comm = {"ms_both_policies": statistics.median(cts), "link_gbs": cp.cluster.link_gbs,
                "ipc_ms": cp.cluster.ipc_ms,
                "max_load": {"index": c1.index, "T": c1.objective, "comm_ms": c1.comm_ms,
                             "e2e_latency_ms": c1.e2e_latency_ms, "same_plan_as_paper_qos": c1.index == pm.index},
                "min_resource": {"index": c2.index, "gpus_used": c2.gpus_used, "quota_used": c2.quota_used},
                "note": "NEXT-2, reading R29/R30: hand-over times in Constraint-5's ordered sum"}

    # NEXT-4: the simulated tail of the step's max-load plan (reading R32)
    tail = None
    if not args.no_sim and rank == 0:
        log("tail-simulation leg")
        ss2 = api.Session(prob, device=dev_idx)
        sims, n_q = 64, 20000
        tail = {"plan": "C4 max-load plan of this step", "queries_per_sim": n_q, "sims": sims, "points": []}
        for f in (0.3, 0.6, 0.9):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            p99, mean = ss2.simulate(pm.batch, pm.replicas, pm.quota_pct, [f * pm.objective] * prob.n_apps,
                                     n_q, 2000, seed=1, n_sims=sims)
            dt = time.perf_counter() - t0
            v = sorted(r[0] for r in p99)
            tail["points"].append({"load_frac_of_T": f, "p99_ms_median_over_sims": v[len(v) // 2],
                                   "mean_ms": statistics.mean(r[0] for r in mean), "sim_ms": dt * 1e3,
                                   "predicted_latency_ms": pm.e2e_latency_ms[0], "qos_ms": float(prob.qos_ms[0])})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        log("CPU oracle leg")
        r = cpu_reference_leg(prob, args, as_main=False)
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "oracle", "sample": r["sample"],
               "single_thread_value": r["single_thread_value"], "cpu_model": r["cpu_model"]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_step_median": ms_med,
                "ms_per_step_min": ms_min, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": WORKLOAD, "problem": prob.name, "sha256": prob.sha256(),
                           "candidates_per_policy": ntot, "policies": 2, "parallelism": f"shard{world}",
                           "api": ("camelot_plan_max_then_min (one call, low load derived on the device)"
                                   if world == 1 else "camelot_search_local -> all_reduce(MIN) -> camelot_finalize "
                                                      "per policy"),
                           "backend": backend if world > 1 else None, "devices": ndev,
                           "l2": "flushed between timed steps (256 MiB write)"},
                "time_to_plan_ms": ms_step,
                "time_to_plan_wall_ms": {"median": wall_med, "min": wall_min,
                                         "note": "host wall clock from the API entry to both plans in host "
                                                 "memory (problem resident, process group warm)"},
                "plans": {"max_load": {"index": pm.index, "T": pm.objective, "replicas": pm.replicas,
                                       "quota_pct": pm.quota_pct, "batch": pm.batch},
                          "min_resource": {"index": pr.index, "gpus_used": pr.gpus_used,
                                           "quota_used": pr.quota_used, "load": LOW_LOAD * pm.objective}},
                "phases_ms": phases, "scored_per_step": evals, "gpu_launches": launches, "roofline": roof,
                "flat_scan": flat, "c4b": hard, "c4_b200": b200, "sa_baseline": sa, "comm_qos": comm, "tail_sim": tail,
                "clocks": clocks,
                "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def C_sizeof_plan():
    import ctypes
    from paper_2005_02088_b200 import _lib as L
    return ctypes.sizeof(L.Plan)


def algorithmic_ops_per_eval(prob):
    """Algorithmic operations of one tree-node / leaf evaluation (DESIGN.md
    "Roofline"): first-fit placement test 4 ops x C GPUs, demand update 2,
    host-max update (n-1), contention factor 4 per stage, latency 1 per stage,
    ordered sum (n-1), QoS compare A, throughput bound 2, key compare 2."""
    n, C, A = prob.n_stages, prob.cluster.n_gpus, prob.n_apps
    return 4 * C + 2 + (n - 1) + 4 * n + n + (n - 1) + A + 2 + 2


if __name__ == "__main__":
    main()
