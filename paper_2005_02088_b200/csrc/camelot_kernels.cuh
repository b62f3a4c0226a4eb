// camelot_kernels.cuh -- the small kernels around the search (sm_100a):
//   filter_kernel   (N3) per (batch, stage) option filtering + compaction,
//   prologue_kernel      a search's prologue: incumbent slots, counters, Eq. 2 estimates,
//   bridge_kernel        camelot_plan_max_then_min between the two searches,
//   reduce_kernel        per-CTA slots -> rank-local best + packed 64-bit keys,
//   resolve_kernel, plan_kernel (N4/N5) keys -> exact index (chunk rescan) -> plan,
//   level_body / search_level_kernel: filter + passes of one pruned search level,
//   score_range_kernel, predict_kernel, flat_search_kernel (N5): full recompute.
#pragma once
#include "../../include/camelot.h"
#include "camelot_device.cuh"
#include "camelot_score.cuh"
#include "camelot_search.cuh"

// Translation units that only instantiate the search templates (camelot_inst_*.cu)
// get private copies of the plain kernels, so that their host stubs do not clash
// with camelot_api.cu's at link time.
#ifdef CAMELOT_INST_TU
#define CAM_GLOBAL static __global__
#else
#define CAM_GLOBAL __global__
#endif

namespace cam {

constexpr int FILTER_THREADS = 512;
constexpr int OMAX = 16 * 128;   // Rmax * nQ upper bound
constexpr int ITEM_SMEM = 256;   // batch combos whose item offsets live in shared memory

struct FilterArgs {
    int policy, prune, stride, nlev;
    const Slot *inc;       // [nlev] incumbent (may be all-none)
    const float *lam;      // [nlev][A]
    OptRec *rec;           // [n][nS][O]
    StageBound *sb;        // [n][nS]
    // fused: search-slot reset and item offsets (last block)
    Slot *slots;
    int nslots;            // grid * nlev slots to reset
    unsigned long long *item_off;
    DevHeader *hdr;
    int d0;
};

CAM_DEVFN void item_offsets(const DevProb &P, const StageBound *sb, int d0, unsigned long long *item_off,
                             DevHeader *hdr);

// One CTA per batch index b: filters the options of every stage at batch b.
// An option survives unless it provably cannot be part of a feasible
// candidate at least as good as the incumbent.
struct FilterSmem {
    float4 tabs[NMAX * CAMELOT_MAX_QUOTAS];   // this batch's table slice (TMA: one bulk copy per stage row)
    unsigned char keep[NMAX][OMAX];
    float mindur[NMAX];
    int minNP[NMAX];
    int Qs[CAMELOT_MAX_QUOTAS];
    unsigned char oth[OMAX], oN[OMAX];        // option code -> (theta, N) (no divisions in the rounds)
    unsigned char ongrid[CAMELOT_MAX_QUOTAS]; // quota theta is on the level's sub-grid
    unsigned char qpass[NMAX][CAMELOT_MAX_QUOTAS];   // (stage, quota): the duration passes the QoS bound
    long long ulim[NMAX];                     // per stage: largest N p passing the quota bounds
};

// Filter body for batch b, executed by one whole CTA (any blockDim multiple of 32).
#ifdef CAMELOT_FTRACE
#define FTRACE(t) if (blockIdx.x == 0 && threadIdx.x == 0) trace_mark(F.hdr, t)
#else
#define FTRACE(t)
#endif
// bar: an initialised mbarrier outside fsm (count 1) whose next phase has parity
// `phase & 1`; the table staging uses one phase (phase is advanced)
CAM_DEVFN void filter_body(const DevProb &P, const FilterArgs &F, int b, FilterSmem &fsm, unsigned long long *bar,
                           unsigned &phase) {
    auto &keep = fsm.keep;
    auto &mindur = fsm.mindur;
    auto &minNP = fsm.minNP;
    auto &tabs = fsm.tabs;
    auto &Qs = fsm.Qs;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int n = P.n, O = P.O, nQ = P.nQ;
    // the per-stage predictor rows of batch b (table [n][nS][nQ] of float4: row (i, b) is
    // nQ x 16 contiguous bytes) -> shared memory with the TMA engine, one bulk copy per stage
    __syncthreads();   // earlier generic accesses of the scratch are complete
    if (tid == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(bar, (uint32_t)(n * nQ * sizeof(float4)));
        for (int i = 0; i < n; ++i)
            bulk_g2s(tabs + i * nQ, P.tab + ((size_t)i * P.nS + b) * nQ, (uint32_t)(nQ * sizeof(float4)), bar);
    }
    for (int q = tid; q < nQ; q += blockDim.x) Qs[q] = P.Q[q];
    for (int o = tid; o < O; o += blockDim.x) {
        fsm.oth[o] = (unsigned char)(o % nQ);
        fsm.oN[o] = (unsigned char)(o / nQ + 1);
    }
    for (int q = tid; q < nQ; q += blockDim.x) fsm.ongrid[q] = F.stride <= 1 || ((nQ - 1 - q) % F.stride) == 0;
    mbar_wait(bar, phase & 1u);
    ++phase;
    __syncthreads();
    FTRACE(4);
    const bool cap = !(P.flags & F_NO_BW_CAP);
    // incumbent
    unsigned long long ikey = 0xFFFFFFFFull;
    for (int k = 0; k < F.nlev; ++k) ikey = (k == 0) ? F.inc[k].key : max(ikey, F.inc[k].key);
    const bool has_inc = ikey < 0xFFFFFFFFull;
    const float Tinc = has_inc ? __uint_as_float(0xFFFFFFFFu - (unsigned)ikey) : 0.0f;
    const int uinc = (int)(ikey >> 24), Uinc = (int)(ikey & 0xFFFFFFu);
    float lam_min[AMAX] = {0.0f, 0.0f};
    if (F.policy == 1)
        for (int a = 0; a < P.A; ++a) {
            float m = F.lam[a];
            for (int k = 1; k < F.nlev; ++k) m = fminf(m, F.lam[k * P.A + a]);
            lam_min[a] = m;
        }
    // static conditions
    const uint32_t Sb = (uint32_t)P.S[b];
    for (int i = 0; i < n; ++i)
    for (int o = tid; o < O; o += blockDim.x) {
        const int th = fsm.oth[o], N = fsm.oN[o];
        const float4 e = tabs[i * nQ + th];
        const uint32_t As = P.Am[i] * Sb;
        bool k = fsm.ongrid[th];
        if (F.prune) {
            if (P.W[i] + As > P.FM) k = false;                 // one replica fits no GPU
            if (cap && e.z > P.BW) k = false;
            if (N > P.C * P.I) k = false;
            const float NT = __fmul_rn((float)N, e.y);
            if (F.policy == 0 && has_inc && NT < Tinc) k = false;   // T <= fl(N thr) < T_inc
            if (F.policy == 1 && NT < (P.app[i] ? lam_min[AMAX - 1] : lam_min[0])) k = false; // load floor at every level
        }
        keep[i][o] = k;
    }
    __syncthreads();
    FTRACE(5);
    const int rounds = F.prune ? 3 : 0;
    for (int it = 0; it <= rounds; ++it) {
        // per-stage minima over surviving options (warp w: stage w)
        for (int i = wid; i < n; i += (int)(blockDim.x >> 5)) {
            float md = __int_as_float(0x7f800000);
            int mn = 0x7fffffff;
            for (int o = lane; o < O; o += 32)
                if (keep[i][o]) {
                    const int th = fsm.oth[o], N = fsm.oN[o];
                    md = fminf(md, tabs[i * nQ + th].x);
                    mn = min(mn, N * Qs[th]);
                }
            for (int off = 16; off; off >>= 1) {
                md = fminf(md, __shfl_xor_sync(0xffffffffu, md, off));
                mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
            }
            if (lane == 0) {
                mindur[i] = md;
                minNP[i] = mn;
            }
        }
        __syncthreads();
        FTRACE(6);
        if (it == rounds) break;
        // The QoS test depends on the option only through its duration, i.e. its quota
        // theta (not N): it is evaluated once per (stage, theta).  The quota tests are
        // monotone in U = N p + rest_i: U <= C R, and (min-resource with an incumbent
        // (u*, U*)) not (ceil(U/R) > u* or (ceil(U/R) >= u* and U > U*)), i.e.
        // U <= min(u* R, max((u* - 1) R, U*)); so N p <= ulim_i (one threshold per stage).
        for (int q = tid; q < n * nQ; q += blockDim.x) {
            const int i = q / nQ, th = q % nQ, a = P.app[i];
            const float dur = tabs[i * nQ + th].x;
            // ordered fp32 sum with this duration at position i and the others' minima
            float ls = 0.0f;
            for (int k2 = P.first_of_app[a]; k2 <= P.last_of_app[a]; ++k2) {
                const float t = (k2 == i) ? dur : mindur[k2];
                if (k2 > P.first_of_app[a] && (P.flags & F_COMM))   // hand-over lower bound (R29)
                    ls = __fadd_rn(ls, fminf(P.ipc_ms, __fmul_rn(__fmul_rn(P.comm_mb[k2 - 1], (float)P.S[b]), P.inv_link)));
                ls = (k2 == P.first_of_app[a]) ? t : __fadd_rn(ls, t);
            }
            fsm.qpass[i][th] = ls <= P.qos[a];
        }
        if (tid < n) {
            const int i = tid, a = P.app[i];
            long long rest = 0;
            for (int k2 = 0; k2 < n; ++k2)
                if (k2 != i) rest += (P.app[k2] == a) ? (long long)minNP[k2] : (long long)Qs[0];
            long long lim = (long long)P.C * P.R;
            if (F.policy == 1 && has_inc)
                lim = min(lim, min((long long)uinc * P.R, max((long long)(uinc - 1) * P.R, (long long)Uinc)));
            fsm.ulim[i] = lim - rest;
        }
        __syncthreads();
        bool changed = false;
        for (int i = 0; i < n; ++i) {
            const long long ul = fsm.ulim[i];
            for (int o = tid; o < O; o += blockDim.x) {
                if (!keep[i][o]) continue;
                const int th = fsm.oth[o], N = fsm.oN[o];
                const bool k = fsm.qpass[i][th] && (long long)N * Qs[th] <= ul;
                if (!k) {
                    keep[i][o] = 0;
                    changed = true;
                }
            }
        }
        // fixpoint reached: the minima of the next round would be the same
        const bool any = __syncthreads_or(changed);
        FTRACE(7);
        if (!any) break;
    }
    // compaction in ascending option code (warp w: stage w) + records
    for (int i = wid; i < n; i += (int)(blockDim.x >> 5)) {
        int cnt = 0;
        float maxNT = 0.0f;
        OptRec *dst = F.rec + ((size_t)i * P.nS + b) * O;
        const uint32_t As = P.Am[i] * (uint32_t)P.S[b];
        for (int o0 = 0; o0 < O; o0 += 32) {
            const int o = o0 + lane;
            const bool k = o < O && keep[i][o];
            const unsigned m = __ballot_sync(0xffffffffu, k);
            if (k) {
                const int th = fsm.oth[o], N = fsm.oN[o];
                const float4 e = tabs[i * nQ + th];
                OptRec r;
                r.code = (uint32_t)o;
                r.p = (uint32_t)Qs[th];
                r.N = (uint32_t)N;
                r.NP = (uint32_t)(N * Qs[th]);
                r.W = P.W[i];
                r.As = As;
                r.MEM = P.W[i] + (uint32_t)N * As;
                r.NB = __fmul_rn((float)N, e.z);
                r.NT = __fmul_rn((float)N, e.y);
                r.bw = e.z;
                r.dur = e.x;
                r.pmul = (65536u + r.p - 1u) / r.p;
                dst[cnt + __popc(m & ((1u << lane) - 1u))] = r;
                maxNT = fmaxf(maxNT, r.NT);
            }
            cnt += __popc(m);
        }
        for (int off = 16; off; off >>= 1) maxNT = fmaxf(maxNT, __shfl_xor_sync(0xffffffffu, maxNT, off));
        if (lane == 0) {
            StageBound s;
            s.cnt = (uint32_t)cnt;
            s.maxNT = maxNT;
            s.mindur = mindur[i];
            s.minNP = (uint32_t)(cnt ? minNP[i] : 0);
            F.sb[(size_t)i * P.nS + b] = s;
        }
    }
    __syncthreads();
    FTRACE(8);
}

// One CTA per batch index b: filters the options of every stage at batch b
// (+ fused: search-slot reset and, by the last block, the item offsets).
CAM_GLOBAL void __launch_bounds__(FILTER_THREADS) filter_kernel(const DevProb P, const FilterArgs F) {
    __shared__ FilterSmem fsm;
    __shared__ unsigned long long bar;
    const int tid = threadIdx.x;
    if (tid == 0) mbar_init(&bar, 1);
    __syncthreads();
    unsigned phase = 0;
    filter_body(P, F, blockIdx.x, fsm, &bar, phase);
    if (F.slots)
        for (int q = blockIdx.x * blockDim.x + tid; q < F.nslots; q += gridDim.x * blockDim.x) {
            F.slots[q].key = 0xFFFFFFFFull;
            F.slots[q].x = ~0ull;
        }
    if (F.item_off) {
        __shared__ int is_last;
        __threadfence();
        __syncthreads();
        if (tid == 0) is_last = atomicAdd(&F.hdr->filt_done, 1u) == gridDim.x - 1;
        __syncthreads();
        if (is_last && tid == 0) {
            __threadfence();
            item_offsets(P, F.sb, F.d0, F.item_off, F.hdr);
            F.hdr->filt_done = 0;
        }
    }
}

CAM_GLOBAL void init_slots_kernel(Slot *s, int n) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        s[k].key = 0xFFFFFFFFull;
        s[k].x = ~0ull;
    }
}

// item space: for batch combo bc, items = prod_{i<d0} cnt_i(b_app(i)), 0 if any stage is empty
CAM_DEVFN void item_offsets(const DevProb &P, const StageBound *sb, int d0, unsigned long long *item_off,
                             DevHeader *hdr) {
    unsigned long long acc = 0;
    for (int bc = 0; bc < P.nbc; ++bc) {
        item_off[bc] = acc;
        int bb[AMAX];   // batch index per application (explicit: no dynamically indexed local array)
        {
            int t = bc;
            bb[AMAX - 1] = t % P.nS;
            if (P.A > 1) t /= P.nS;
            bb[0] = t % P.nS;
        }
        unsigned long long it = 1;
        bool empty = false;
        for (int i = 0; i < P.n; ++i) {
            const unsigned c = sb[(size_t)i * P.nS + (P.app[i] ? bb[AMAX - 1] : bb[0])].cnt;
            if (c == 0) empty = true;
            if (i < d0) it *= c;
        }
        acc += empty ? 0ull : it;
    }
    item_off[P.nbc] = acc;
    hdr->items_total = acc;
}

// The same offsets computed by a whole CTA from shared-memory bounds into shared
// memory (nbc <= ITEM_SMEM): per-combo counts in parallel, then an inclusive scan.
CAM_DEVFN void item_offsets_block(const DevProb &P, const StageBound *sb, int d0, unsigned long long *out) {
    for (int bc = threadIdx.x; bc < P.nbc; bc += blockDim.x) {
        int bb[AMAX];   // batch index per application (explicit: no dynamically indexed local array)
        {
            int t = bc;
            bb[AMAX - 1] = t % P.nS;
            if (P.A > 1) t /= P.nS;
            bb[0] = t % P.nS;
        }
        unsigned long long it = 1;
        bool empty = false;
        for (int i = 0; i < P.n; ++i) {
            const unsigned c = sb[(size_t)i * P.nS + (P.app[i] ? bb[AMAX - 1] : bb[0])].cnt;
            if (c == 0) empty = true;
            if (i < d0) it *= c;
        }
        out[bc + 1] = empty ? 0ull : it;
    }
    if (threadIdx.x == 0) out[0] = 0;
    __syncthreads();
    const int q = threadIdx.x;   // nbc <= ITEM_SMEM <= blockDim.x
    for (int off = 1; off < P.nbc; off <<= 1) {   // Hillis-Steele inclusive scan of out[1..nbc]
        const bool act = q < P.nbc && q >= off;
        const unsigned long long v = act ? out[q + 1 - off] : 0ull;
        __syncthreads();
        if (act) out[q + 1] += v;
        __syncthreads();
    }
}

// slots -> result[k] and packed keys (stand-alone kernel: naive path)
CAM_GLOBAL void reduce_kernel(const DevProb P, const Slot *slots, int nslots, int nlev, Slot *result,
                              long long *keys, const StageBound *sb, const OptRec *rec,
                              const unsigned long long *item_off, int d0, int chunk_items, int flat_shift) {
    __shared__ unsigned long long sk[256], sx[256];
    reduce_slots_block(P, slots, nslots, nlev, result, keys, nullptr, sb, rec, item_off, d0, chunk_items,
                       flat_shift, sk, sx);
}

// keys (after the cross-rank MIN) -> which chunk must be re-scanned / exact index
struct FinalArgs {
    int policy, nlev, world;
    const long long *keys;     // [nlev] reduced, sign-mapped
    const Slot *local;         // [nlev] this rank's exact best
    Slot *winner;              // [nlev] out: (objective key, x) ; x = ~0 if unresolved
    unsigned long long *rescan;// [nlev] out: chunk to re-scan or ~0
};

CAM_GLOBAL void resolve_kernel(const DevProb P, const FinalArgs F) {
    const int k = threadIdx.x;
    if (k >= F.nlev) return;
    const unsigned long long packed = (unsigned long long)F.keys[k] ^ 0x8000000000000000ull;
    Slot w;
    unsigned long long rs = ~0ull;
    if (packed == ~0ull) {
        w.key = 0xFFFFFFFFull;
        w.x = ~0ull;
    } else {
        w.key = packed >> 32;
        const unsigned long long low = packed & 0xFFFFFFFFull;
        if (F.world == 1) w.x = F.local[k].x;
        else if (P.ntot <= (1ull << 32)) w.x = low;
        else {
            w.x = ~0ull;
            rs = low;
        }
    }
    F.winner[k] = w;
    F.rescan[k] = rs;
}

// winner index -> full plan (device), with the search counters
constexpr int PLAN_THREADS = 64;
struct PlanScratch {
    camelot_plan pl;
    FullScore s;
    ScoreScratch scr;
    int beta[AMAX], rho[NMAX], theta[NMAX];
    float dur[NMAX], thr[NMAX], bwv[NMAX];
    int pq[NMAX];
    uint32_t As[NMAX];
    int eq2y;
};
// The full plan of winner w, scored by ONE whole CTA (>= 32 threads; every thread
// calls): thread 0 decodes, warp 0 places in parallel (place_warp; score_digits only
// for PAPER_GLOBAL or a failed placement), the CTA fills the plan in shared memory and
// copies it out.  lamk: this level's loads [A] (min-resource); hdr: the search's counters.
CAM_DEVFN void plan_block(const DevProb &P, int policy, const Slot w, const float *lamk, const DevHeader *hdr,
                          camelot_plan *out, PlanScratch &ps) {
    const int tid = threadIdx.x;
    camelot_plan &pl = ps.pl;
    FullScore &s = ps.s;
    int *beta = ps.beta, *rho = ps.rho, *theta = ps.theta;
    {
        uint32_t *pw = reinterpret_cast<uint32_t *>(&pl);
        for (int q = tid; q < (int)(sizeof(camelot_plan) / 4); q += blockDim.x) pw[q] = 0u;
    }
    __syncthreads();
    for (int q = tid; q < CAMELOT_MAX_STAGES * CAMELOT_MAX_REPLICAS; q += blockDim.x) pl.gpu_of_instance[q] = -1;
    if (tid == 0) {
        pl.n_scored = hdr->n_scored;
        pl.n_evaluated = hdr->cum_scored + hdr->cum_nodes;
        pl.n_feasible = hdr->n_feasible;
        if (w.x == ~0ull) {
            pl.index = ~0ull;
            pl.status = CAMELOT_INFEASIBLE;
            pl.violations = hdr->viol_or;
        }
    }
    // mixed-radix decode (decode_index's digits), one digit per thread: option o_i =
    // (x / O^(n-1-i)) mod O = rho_i nQ + theta_i; the batch combo = x / O^n
    if (w.x != ~0ull) {
        if (tid < P.n) {
            const unsigned o = (unsigned)((w.x / P.opow[P.n - 1 - tid]) % (unsigned long long)P.O);
            rho[tid] = (int)(o / (unsigned)P.nQ);
            theta[tid] = (int)(o % (unsigned)P.nQ);
        } else if (tid == P.n) {
            unsigned bc = (unsigned)(w.x / P.opow[P.n]);
            for (int a = P.A - 1; a >= 0; --a) {
                beta[a] = (int)(bc % (unsigned)P.nS);
                bc /= (unsigned)P.nS;
            }
        }
    }
    __syncthreads();
    // the winner's table rows, quotas and activation sizes, one stage per thread (one
    // round trip instead of a dependent chain per stage)
    if (w.x != ~0ull && tid < P.n) {
        const int i = tid, b = beta[P.app[i]];
        const float4 e = P.tab[((size_t)i * P.nS + b) * P.nQ + theta[i]];
        ps.dur[i] = e.x;
        ps.thr[i] = e.y;
        ps.bwv[i] = e.z;
        ps.pq[i] = P.Q[theta[i]];
        ps.As[i] = P.Am[i] * (uint32_t)P.S[b];
    }
    __syncthreads();
    if (w.x != ~0ull && tid < 32) {
        bool placed = false;
        if (!(P.flags & F_PAPER_GLOBAL)) {
            float dur[NMAX], thr[NMAX], bwv[NMAX], kmax[NMAX];
            uint32_t hm[NMAX];
            for (int i = 0; i < P.n; ++i) {
                dur[i] = ps.dur[i];
                thr[i] = ps.thr[i];
                bwv[i] = ps.bwv[i];
            }
            for (int q = tid; q < NMAX * SCORE_RMAX; q += 32) s.goi[q] = -1;
            __syncwarp();
            int u = 0;
            placed = place_warp(P, rho, ps.pq, ps.As, bwv, kmax, hm, s.goi, u);
            __syncwarp();
            if (placed && tid == 0) {
                int U = 0;
                for (int i = 0; i < P.n; ++i) U += (rho[i] + 1) * ps.pq[i];
                s.U = U;
                score_finish(P, beta, rho, dur, thr, kmax, hm, 0u, u, s);
            }
        }
        if (!placed && tid == 0) score_digits(P, beta, rho, theta, s, &ps.scr);
    }
    __syncthreads();
    if (tid == 0 && w.x != ~0ull) {
        ps.eq2y = policy == 1 ? eq2_gpus(P, beta, lamk) : 0;
        pl.index = w.x;
        pl.status = CAMELOT_OK;
        pl.quota_used = s.U;
        pl.gpus_used = s.u;
        if (policy == 1) {
            pl.eq2_gpus = ps.eq2y;
            pl.violations = level_verdict(P, s, lamk, ps.eq2y);
            pl.objective = (float)s.U;
        } else {
            pl.violations = s.verdict;
            pl.objective = s.T;
        }
    }
    __syncthreads();
    if (w.x != ~0ull) {
        if (tid < P.A) {
            pl.batch[tid] = P.S[beta[tid]];
            pl.e2e_latency_ms[tid] = s.Lsum[tid];
            pl.throughput_qps[tid] = s.Tmin[tid];
        }
        if (tid < P.n) {
            const int i = tid;
            pl.replicas[i] = rho[i] + 1;
            pl.quota_pct[i] = ps.pq[i];
            pl.stage_latency_ms[i] = s.L[i];
            pl.stage_throughput_qps[i] = s.Ti[i];
            pl.kappa[i] = s.kappa[i];
            pl.comm_ms[i] = s.comm[i];
        }
        for (int q = tid; q < P.n * CAMELOT_MAX_REPLICAS; q += blockDim.x) {
            const int i = q / CAMELOT_MAX_REPLICAS, r = q % CAMELOT_MAX_REPLICAS;
            if (r < SCORE_RMAX) pl.gpu_of_instance[q] = s.goi[i * SCORE_RMAX + r];
        }
    }
    __syncthreads();
    const uint32_t *src = reinterpret_cast<const uint32_t *>(&pl);
    uint32_t *dst = reinterpret_cast<uint32_t *>(out);
    for (int q = tid; q < (int)(sizeof(camelot_plan) / 4); q += blockDim.x) dst[q] = src[q];
}

// One block per load level: plan_block of that level's winner.
// keys != nullptr (one rank): the level's packed key is resolved here first (resolve_kernel's
// world-1 rule: objective key from the packed key, index from this rank's exact best
// `local`) and the winner is written back -- one launch instead of two at the end of a plan.
CAM_GLOBAL void __launch_bounds__(PLAN_THREADS) plan_kernel(const DevProb P, int policy, int nlev, Slot *winner,
                                                            const float *lam, const DevHeader *hdr, camelot_plan *out,
                                                            const long long *keys = nullptr,
                                                            const Slot *local = nullptr) {
    const int k = blockIdx.x;
    if (k >= nlev) return;
    __shared__ PlanScratch ps;
    Slot w;
    if (keys) {
        const unsigned long long packed = (unsigned long long)keys[k] ^ 0x8000000000000000ull;
        w.key = packed == ~0ull ? 0xFFFFFFFFull : packed >> 32;
        w.x = packed == ~0ull ? ~0ull : local[k].x;
        if (threadIdx.x == 0) winner[k] = w;
    } else {
        w = winner[k];
    }
    plan_block(P, policy, w, lam + k * P.A, hdr, out + k, ps);
}

// The prologue of a search in ONE launch (one CTA): no incumbent (key 0xFFFFFFFF,
// x = ~0) at every level, the cumulative counters of the call zeroed, and (min
// resource) the Eq. 2 estimates y[bc][k] = eq2_gpus at the levels' loads.
CAM_GLOBAL void prologue_kernel(const DevProb P, Slot *inc, int nlev, int policy, const float *lam, int *y,
                                DevHeader *hdr) {
    const int t = threadIdx.x;
    for (int k = t; k < nlev; k += blockDim.x) {
        inc[k].key = 0xFFFFFFFFull;
        inc[k].x = ~0ull;
    }
    if (t == 0) {
        hdr->cum_scored = 0;
        hdr->cum_nodes = 0;
        hdr->trace_n = 0;
        hdr->trace_pad = 0;
    }
    if (policy == 1)
        for (int idx = t; idx < P.nbc * nlev; idx += blockDim.x) {
            const int bc = idx / nlev, k = idx % nlev;
            int beta[AMAX];
            int r = bc;
            for (int a = P.A - 1; a >= 0; --a) {
                beta[a] = r % P.nS;
                r /= P.nS;
            }
            y[idx] = eq2_gpus(P, beta, lam + k * P.A);
        }
}

// camelot_plan_max_then_min, between the two searches, in ONE launch (one CTA):
//  * resolve the max-load key (world 1: resolve_kernel's rule);
//  * the low load (low load = a fraction of the peak): load_a =
//    fl(frac * T*) for every application, T* read from the winner's objective key
//    (0xFFFFFFFF - bits(T): the same binary32 T the plan reports), the
//    binary32 rounding of the float64 product (as a host caller computing frac * T* in
//    double and storing it as float); +inf when there is no feasible peak (every
//    min-resource candidate then fails LOAD);
//  * a snapshot of the winner and the search counters for the max-load plan_kernel,
//    which runs on a second stream while the min-resource search runs;
//  * the min-resource search's prologue: no incumbent, the Eq. 2 estimates at the low
//    load, the cumulative counters zeroed (what prologue_kernel does for a search).
CAM_GLOBAL void bridge_kernel(const DevProb P, const long long *keys, const Slot *local, Slot *winner, double frac,
                              float *lam, Slot *side_w, DevHeader *side_h, const DevHeader *hdr2, Slot *inc, int *y,
                              DevHeader *hdr) {
    __shared__ Slot w;
    const int t = threadIdx.x;
    if (t == 0) {
        const unsigned long long packed = (unsigned long long)keys[0] ^ 0x8000000000000000ull;
        if (packed == ~0ull) {
            w.key = 0xFFFFFFFFull;
            w.x = ~0ull;
        } else {
            w.key = packed >> 32;
            w.x = local[0].x;
        }
        winner[0] = w;
        *side_w = w;
        inc[0].key = 0xFFFFFFFFull;
        inc[0].x = ~0ull;
    }
    __syncthreads();
    if (t < P.A) {
        const float T = __uint_as_float(0xFFFFFFFFu - (uint32_t)w.key);
        lam[t] = w.x != ~0ull ? __double2float_rn(frac * (double)T) : __int_as_float(0x7f800000);
    }
    const uint32_t *src = reinterpret_cast<const uint32_t *>(hdr2);   // (may be hdr itself)
    uint32_t *dst = reinterpret_cast<uint32_t *>(side_h);
    for (int q = t; q < (int)(offsetof(DevHeader, trace_n) / 4); q += blockDim.x) dst[q] = src[q];
    __syncthreads();   // the snapshot before the counters are zeroed; lam before the Eq. 2 estimates
    if (t == 0) {
        hdr->cum_scored = 0;
        hdr->cum_nodes = 0;
        hdr->trace_n = 0;
        hdr->trace_pad = 0;
    }
    for (int bc = t; bc < P.nbc; bc += blockDim.x) {
        int beta[AMAX];
        int r = bc;
        for (int a = P.A - 1; a >= 0; --a) {
            beta[a] = r % P.nS;
            r /= P.nS;
        }
        y[bc] = eq2_gpus(P, beta, lam);
    }
}

// Naive exhaustive search (kernel N5 as a search): one thread scores one
// candidate from scratch.  Used for PAPER_GLOBAL problems, single-stage
// problems and as the un-hoisted baseline (CAMELOT_EXEC_NAIVE).  Chunks of
// 2^FLAT_SHIFT consecutive indices are dealt to ranks round-robin.
constexpr int FLAT_SHIFT = 15;
constexpr int FLAT_THREADS = 256;

struct FlatArgs {
    int policy, nlev, rank, world;
    unsigned long long lo, hi;
    const float *lam;
    const int *y;
    int ystride, yoff;
    const Slot *inc;
    Slot *slots;
    DevHeader *hdr;
};

CAM_GLOBAL void __launch_bounds__(FLAT_THREADS) flat_search_kernel(const DevProb P, const FlatArgs F) {
    __shared__ unsigned long long bk_s[FLAT_THREADS / 32][LMAX], bx_s[FLAT_THREADS / 32][LMAX];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int k = lane; k < F.nlev; k += 32) {
        bk_s[wid][k] = F.inc[k].key;
        bx_s[wid][k] = F.inc[k].x;
    }
    __syncwarp();
    unsigned long long scored = 0, feasible = 0;
    unsigned viol = 0;
    const unsigned long long CH = 1ull << FLAT_SHIFT;
    const unsigned long long c0 = F.lo >> FLAT_SHIFT, c1 = (F.hi + CH - 1) >> FLAT_SHIFT;
    // chunk c belongs to rank (c mod world); threads of the grid stride over its indices
    const unsigned long long nthreads = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long cfirst = c0 + (unsigned long long)((F.rank - (long long)(c0 % F.world) + F.world) % F.world);
    for (unsigned long long c = cfirst; c < c1; c += F.world) {
        const unsigned long long a = max(c * CH, F.lo), b = min((c + 1) * CH, F.hi);
        for (unsigned long long base = a; base < b; base += nthreads) {
            const unsigned long long x = base + tid;
            const bool v = x < b;
            int beta[AMAX], rho[NMAX], theta[NMAX];
            FullScore s;
            s.verdict = 0xFFu;
            if (v) {
                decode_index(P, x, beta, rho, theta);
                score_digits(P, beta, rho, theta, s);
                ++scored;
                viol |= s.verdict;
                feasible += s.verdict == 0;
            }
            if (F.policy == 0) {
                const bool ok = v && s.verdict == 0;
                const unsigned long long key = ok ? (unsigned long long)objkey_maxload(s.T) : 0xFFFFFFFFull;
                const bool imp = ok && slot_less(key, x, bk_s[wid][0], bx_s[wid][0]);
                unsigned im = __ballot_sync(0xffffffffu, imp);
                if (im) {
                    unsigned long long k2 = imp ? key : ~0ull, x2 = imp ? x : ~0ull;
                    for (int off = 16; off; off >>= 1) {
                        unsigned long long ok2 = __shfl_xor_sync(0xffffffffu, k2, off);
                        unsigned long long ox = __shfl_xor_sync(0xffffffffu, x2, off);
                        if (slot_less(ok2, ox, k2, x2)) { k2 = ok2; x2 = ox; }
                    }
                    __syncwarp();   // all lanes have read the warp best before lane 0 updates it
                    if (lane == 0 && slot_less(k2, x2, bk_s[wid][0], bx_s[wid][0])) {
                        bk_s[wid][0] = k2;
                        bx_s[wid][0] = x2;
                    }
                    __syncwarp();
                }
            } else {
                const unsigned long long key = v ? (unsigned long long)objkey_minres(s.u, s.U) : 0xFFFFFFFFull;
                int bc = 0;
                if (v)
                    for (int q = 0; q < P.A; ++q) bc = bc * P.nS + beta[q];
                for (int k = 0; k < F.nlev; ++k) {
                    bool ok = v && s.verdict == 0;
                    if (ok) ok = level_verdict(P, s, F.lam + k * P.A, F.y[bc * F.ystride + F.yoff + k]) == 0;
                    const bool imp = ok && slot_less(key, x, bk_s[wid][k], bx_s[wid][k]);
                    unsigned im = __ballot_sync(0xffffffffu, imp);
                    if (im) {
                        unsigned long long k2 = imp ? key : ~0ull, x2 = imp ? x : ~0ull;
                        for (int off = 16; off; off >>= 1) {
                            unsigned long long ok2 = __shfl_xor_sync(0xffffffffu, k2, off);
                            unsigned long long ox = __shfl_xor_sync(0xffffffffu, x2, off);
                            if (slot_less(ok2, ox, k2, x2)) { k2 = ok2; x2 = ox; }
                        }
                        __syncwarp();
                        if (lane == 0 && slot_less(k2, x2, bk_s[wid][k], bx_s[wid][k])) {
                            bk_s[wid][k] = k2;
                            bx_s[wid][k] = x2;
                        }
                        __syncwarp();
                    }
                }
            }
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < F.nlev; k += blockDim.x) {
        unsigned long long bk = bk_s[0][k], bx = bx_s[0][k];
        for (int w = 1; w < FLAT_THREADS / 32; ++w)
            if (slot_less(bk_s[w][k], bx_s[w][k], bk, bx)) {
                bk = bk_s[w][k];
                bx = bx_s[w][k];
            }
        F.slots[(size_t)blockIdx.x * F.nlev + k].key = bk;
        F.slots[(size_t)blockIdx.x * F.nlev + k].x = bx;
    }
    for (int off = 16; off; off >>= 1) {
        scored += __shfl_xor_sync(0xffffffffu, scored, off);
        feasible += __shfl_xor_sync(0xffffffffu, feasible, off);
        viol |= __shfl_xor_sync(0xffffffffu, viol, off);
    }
    if (lane == 0) {
        atomicAdd(&F.hdr->n_scored, scored);
        atomicAdd(&F.hdr->n_feasible, feasible);
        atomicOr(&F.hdr->viol_or, viol & 0x7Fu);
    }
}

// explicit plan (predict) -> plan
CAM_GLOBAL void predict_kernel(const DevProb P, unsigned long long x, const float *lam, int nlev, camelot_plan *out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    camelot_plan pl;
    memset(&pl, 0, sizeof(pl));
    for (int i = 0; i < CAMELOT_MAX_STAGES * CAMELOT_MAX_REPLICAS; ++i) pl.gpu_of_instance[i] = -1;
    int beta[AMAX], rho[NMAX], theta[NMAX];
    decode_index(P, x, beta, rho, theta);
    FullScore s;
    score_digits(P, beta, rho, theta, s);
    pl.index = x;
    for (int a = 0; a < P.A; ++a) {
        pl.batch[a] = P.S[beta[a]];
        pl.e2e_latency_ms[a] = s.Lsum[a];
        pl.throughput_qps[a] = s.Tmin[a];
    }
    for (int i = 0; i < P.n; ++i) {
        pl.replicas[i] = rho[i] + 1;
        pl.quota_pct[i] = P.Q[theta[i]];
        pl.stage_latency_ms[i] = s.L[i];
        pl.stage_throughput_qps[i] = s.Ti[i];
        pl.kappa[i] = s.kappa[i];
        pl.comm_ms[i] = s.comm[i];
        for (int r = 0; r < CAMELOT_MAX_REPLICAS && r < SCORE_RMAX; ++r)
            pl.gpu_of_instance[i * CAMELOT_MAX_REPLICAS + r] = s.goi[i * SCORE_RMAX + r];
    }
    pl.quota_used = s.U;
    pl.gpus_used = s.u;
    pl.objective = s.T;
    pl.violations = s.verdict;
    if (nlev > 0 && lam) {
        pl.eq2_gpus = eq2_gpus(P, beta, lam);
        pl.violations = level_verdict(P, s, lam, pl.eq2_gpus);
    }
    pl.status = pl.violations ? CAMELOT_INFEASIBLE : CAMELOT_OK;
    out[0] = pl;
}

CAM_GLOBAL void score_range_kernel(const DevProb P, unsigned long long lo, unsigned long long cnt, uint8_t *verdict,
                                   float *T, int *u, int *U) {
    const unsigned long long t = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    int beta[AMAX], rho[NMAX], theta[NMAX];
    decode_index(P, lo + t, beta, rho, theta);
    FullScore s;
    score_digits(P, beta, rho, theta, s);
    if (verdict) verdict[t] = (uint8_t)s.verdict;
    if (T) T[t] = s.T;
    if (u) u[t] = s.u;
    if (U) U[t] = s.U;
}

}  // namespace cam

// ============================================================================
// Cooperative persistent kernel: ONE launch per search level (incumbent
// cascade level or main search): header reset -> option filter -> item offsets
// -> the n level-synchronous passes -> slot reduction, separated by grid-wide
// barriers instead of kernel boundaries.  Launched with
// cudaLaunchCooperativeKernel (all CTAs co-resident).
#include <cooperative_groups.h>

namespace cam {

struct LevelArgs {
    SearchArgs S;      // shared fields; per-pass fields are set in the kernel
    FilterArgs F;
    void *buf0, *buf1; // frontier ping-pong buffers
    unsigned long long fcap;
    unsigned rec_budget;   // bytes of shared memory for the staged option lists (0: never stage)
};

// Dynamic shared memory of a search level: max(filter scratch, search state +
// StageBound cache + item offsets + list offsets), then the staging mbarrier (16 B),
// then the staged option lists (LevelArgs::rec_budget bytes).
template <int CM>
__host__ __device__ constexpr size_t level_state_bytes() {
    return search_smem_bytes<CM>() + (size_t)NMAX * CAMELOT_MAX_BATCHES * sizeof(StageBound) +
           (ITEM_SMEM + 1) * sizeof(unsigned long long) + (NMAX * CAMELOT_MAX_BATCHES + 1) * sizeof(int);
}
template <int CM>
__host__ __device__ constexpr size_t level_fixed_bytes() {
    return ((level_state_bytes<CM>() > sizeof(FilterSmem) ? level_state_bytes<CM>() : sizeof(FilterSmem)) + 15) /
           16 * 16;
}

// reset a level's header state (the cumulative counters stay); one whole CTA
__device__ __forceinline__ void level_reset(DevHeader *hdr) {
    unsigned *h = reinterpret_cast<unsigned *>(hdr);
    for (int w = threadIdx.x; w < (int)(offsetof(DevHeader, cum_scored) / 4); w += blockDim.x) h[w] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
        hdr->best_obj = 0xFFFFFFFFu;
        hdr->best_packed = ~0ull;
    }
}

// One search level (incumbent cascade level or main pass) executed by the whole
// cooperative grid; levels are chained inside one launch (search_level_kernel).
// first: reset the header (block 0) behind a grid barrier; later levels find it reset
// by the previous level's last CTA.  last: no grid barrier at the end (kernel exit).
template <int CM, int NS, int POLICY>
__device__ __forceinline__ void level_body(const DevProb &P, const LevelArgs &LA, unsigned char *smem_raw,
                                           cooperative_groups::grid_group &grid, unsigned &stage_phase, bool first,
                                           bool last) {
    SearchArgs S = LA.S;
    DevHeader *hdr = S.hdr;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool tr = blockIdx.x == 0 && threadIdx.x == 0;
    if (tr) trace_mark(hdr, 0);
    // phase 0 (first level only): reset the header state
    if (first) {
        if (blockIdx.x == 0) level_reset(hdr);
        grid.sync();
    }
    if (tr) trace_mark(hdr, 1);
    // phase 1: option filter (one CTA per batch) and slot reset
    for (int b = blockIdx.x; b < P.nS; b += gridDim.x) {
        filter_body(P, LA.F, b, *reinterpret_cast<FilterSmem *>(smem_raw),
                    reinterpret_cast<unsigned long long *>(smem_raw + level_fixed_bytes<CM>()), stage_phase);
        __syncthreads();
    }
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < gridDim.x * S.nlev; q += gridDim.x * blockDim.x) {
        S.slots[q].key = 0xFFFFFFFFull;
        S.slots[q].x = ~0ull;
    }
    grid.sync();
    if (tr) trace_mark(hdr, 2);
    // per-CTA copy of the (stage, batch) bounds in shared memory, after the search state,
    // and (phase 2) the item offsets of the chunk ownership: computed by every CTA from
    // its copy (no grid barrier) when there are few batch combos; block 0 also writes
    // them to global memory for a later chunk re-scan
    {
        StageBound *sbs = reinterpret_cast<StageBound *>(smem_raw + search_smem_bytes<CM>());
        for (int q = threadIdx.x; q < P.n * P.nS; q += blockDim.x) sbs[q] = S.sb[q];
        __syncthreads();
        S.sb = sbs;
        if (P.nbc <= ITEM_SMEM) {
            unsigned long long *ioff = reinterpret_cast<unsigned long long *>(sbs + NMAX * CAMELOT_MAX_BATCHES);
            item_offsets_block(P, sbs, S.d0, ioff);
            if (blockIdx.x == 0) {
                for (int t = threadIdx.x; t <= P.nbc; t += blockDim.x) LA.F.item_off[t] = ioff[t];
                if (threadIdx.x == 0) hdr->items_total = ioff[P.nbc];
            }
            S.item_off = ioff;
        } else {
            grid.sync();
            if (blockIdx.x == 0 && threadIdx.x == 0) item_offsets(P, S.sb, S.d0, LA.F.item_off, hdr);
            grid.sync();
        }
        // the level's compacted option lists -> this CTA's shared memory with the TMA
        // engine (cp.async.bulk, one copy per (stage, batch) list), when they fit
        int *recoff = reinterpret_cast<int *>(reinterpret_cast<unsigned long long *>(sbs + NMAX * CAMELOT_MAX_BATCHES) +
                                              ITEM_SMEM + 1);
        unsigned long long *mbar = reinterpret_cast<unsigned long long *>(smem_raw + level_fixed_bytes<CM>());
        OptRec *rec_s = reinterpret_cast<OptRec *>(smem_raw + level_fixed_bytes<CM>() + 16);
        const int nl = P.n * P.nS;
        if (LA.rec_budget > 0 && threadIdx.x == 0) {   // (staging is opt-in: skip the serial scan when off)
            int acc = 0;
            for (int q = 0; q < nl; ++q) {
                recoff[q] = acc;
                acc += (int)sbs[q].cnt;
            }
            recoff[nl] = acc;
        }
        if (LA.rec_budget > 0) __syncthreads();
        const unsigned long long bytes = LA.rec_budget > 0 ? (unsigned long long)recoff[nl] * sizeof(OptRec) : 0ull;
        if (bytes > 0 && bytes <= LA.rec_budget) {
            if (threadIdx.x == 0) {
                fence_proxy_async();   // the filter's generic stores (before the grid barrier) -> async reads
                mbar_arrive_expect_tx(mbar, (uint32_t)bytes);
                for (int q = 0; q < nl; ++q)
                    if (sbs[q].cnt)
                        bulk_g2s(rec_s + recoff[q], S.rec + (size_t)q * P.O, sbs[q].cnt * (uint32_t)sizeof(OptRec), mbar);
            }
            mbar_wait(mbar, stage_phase & 1u);
            ++stage_phase;
            S.rec_stage = rec_s;
            S.rec_off = recoff;
        }
        if (tr) trace_mark(hdr, 3);
    }
    // phase 3: the passes (shared memory now holds the search state)
    Node<CM> *stack_all = reinterpret_cast<Node<CM> *>(smem_raw);
    WarpCtl *ctl_all = reinterpret_cast<WarpCtl *>(stack_all + (size_t)SEARCH_WARPS * NMAX);
    WarpBest *wb_all = reinterpret_cast<WarpBest *>(ctl_all + SEARCH_WARPS);
    Node<CM> *stack = stack_all + (size_t)wid * NMAX;
    WarpCtl *ctl = ctl_all + wid;
    WarpBest *wb = wb_all + wid;
    init_warp_best(S, wb, lane);
    Counters cn = {0, 0, 0, 0};
    const int n = P.n;
    // compact depth-1 frontier (2 words per child of the root pass) when depth 1 is an
    // inner level (testing knob: LevelArgs.S.compact1 = 0 keeps full nodes)
    S.compact1 = S.compact1 && n >= 3;
    for (int j = 0; j < n; ++j) {
        S.level = j;
        S.flevel = (j + 1 <= n - 1) ? j + 1 : -1;
        S.in_nodes = j == 0 ? nullptr : ((j & 1) ? LA.buf1 : LA.buf0);
        S.in_count = &hdr->tail[j];
        S.in_cap = LA.fcap;
        S.out_nodes = ((j + 1) & 1) ? LA.buf1 : LA.buf0;
        S.out_tail = &hdr->tail[j + 1];
        S.out_cap = LA.fcap;
        S.head = &hdr->head[j];
        S.grab = 1;
        // (one call site: pass_body is large.)  A thread-per-parent pass that could outgrow
        // the frontier (optimistic) and did -- children were dropped -- is redone in the
        // warp mode, which descends inline when the frontier is full.
        bool redo = false;
        for (int attempt = 0; attempt < 2; ++attempt) {
            S.no_tmode = attempt;
            const bool optimistic = pass_body<CM, NS, POLICY>(P, S, stack, ctl, wb, lane, cn);
            if (attempt || !optimistic || j == n - 1) break;
            grid.sync();
            redo = *(volatile unsigned long long *)&hdr->tail[j + 1] > LA.fcap;   // (same value in every CTA)
            if (!redo) break;
            grid.sync();   // every CTA has read the tail
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                hdr->tail[j + 1] = 0;
                hdr->head[j] = 0;
            }
            grid.sync();
        }
        S.no_tmode = 0;
        if (j == n - 1) break;   // the last pass ends at the CTA merge below (no grid barrier)
#ifdef CAMELOT_FTRACE
        if (lane == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMax(&hdr->dbg_tend[j], t);
        }
#endif
        grid.sync();
        if (tr) {
#ifdef CAMELOT_FTRACE
            trace_value(hdr, 48 + j, hdr->dbg_tend[j]);
#endif
            trace_mark(hdr, 16 + j);
#ifdef CAMELOT_FTRACE
            trace_value(hdr, 64 + j, j == 0 ? (unsigned long long)P.nbc : hdr->tail[j]);   // parents of pass j
            trace_value(hdr, 80 + j, hdr->dbg_batches[j]);
            trace_value(hdr, 96 + j, hdr->dbg_maxb[j]);
            if (hdr->dbg_tc[j][3]) {   // thread-per-parent chunk of block 0 warp 0: ctx / children / emission ns, parents
                for (int q = 0; q < 4; ++q) trace_value(hdr, 120 + q, hdr->dbg_tc[j][q]);
            }
#endif
        }
    }
    cta_finish<CM>(S, wb_all, lane, wid, cn);
    // phase 4: the LAST CTA to finish reduces the CTA slots (exact local best, packed
    // key, next incumbent) and resets the header for the next level; one grid barrier
    // then separates the levels
    __shared__ int is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = atomicAdd(&hdr->done_ctas, 1u) == gridDim.x - 1;
    __syncthreads();
    if (is_last) {
        __threadfence();
        if (threadIdx.x == 0) {
            trace_mark(hdr, 16 + n - 1);
            trace_mark(hdr, 32);
        }
        unsigned long long *sk = reinterpret_cast<unsigned long long *>(smem_raw);
        reduce_slots_block(P, S.slots, gridDim.x, S.nlev, S.result, S.keys, S.inc_out, S.sb, S.rec, S.item_off, S.d0,
                           S.chunk_items, -1, sk, sk + SEARCH_THREADS);
        if (threadIdx.x == 0) {   // the level's optimum (objective key, canonical index) in the phase trace
            trace_value(hdr, 200, S.result[0].key);
            trace_value(hdr, 201, S.result[0].x);
        }
        __syncthreads();
        if (!last) level_reset(hdr);   // (also zeroes done_ctas)
        else if (threadIdx.x == 0) hdr->done_ctas = 0;
    }
    if (!last) grid.sync();
}


// All pruned levels of one search in ONE cooperative launch: level l+1 reads the
// incumbent that level l's last CTA wrote (with the header reset) before the grid
// barrier that ends level l, so no extra barrier or launch is needed between levels.
constexpr int MAX_LEVELS = 4;
struct LevelSet {
    int count;
    LevelArgs L[MAX_LEVELS];
};

template <int CM, int NS, int POLICY>
__global__ void __launch_bounds__(SEARCH_THREADS, SEARCH_MINB)
search_level_kernel(const DevProb P, const LevelSet LS) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned stage_phase = 0;   // phase of the staging mbarrier (one per staged level)
    if (threadIdx.x == 0) mbar_init(reinterpret_cast<unsigned long long *>(smem_raw + level_fixed_bytes<CM>()), 1);
    __syncthreads();
    for (int l = 0; l < LS.count; ++l) {
        level_body<CM, NS, POLICY>(P, LS.L[l], smem_raw, grid, stage_phase, l == 0, l == LS.count - 1);
        __syncthreads();   // the last CTA's reduction used shared memory
    }
}
}  // namespace cam

// ============================================================================
// The paper's simulated annealing (NEXT-1) as a GPU
// multi-chain baseline: one thread per chain, counter-based randomness
// (splitmix64 of (seed, chain, iteration, purpose)), every
// proposal scored exactly like the search (score_digits).  A worse valid state
// is accepted with probability p_k = p0 * cool^k (decreasing with the
// iterations, R13); invalid states are rejected once the chain is valid; every
// valid proposal that improves the objective updates the chain's best.
namespace cam {

__device__ __forceinline__ unsigned long long sa_sm64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long sa_rng(unsigned long long seed, unsigned long long chain,
                                                     unsigned long long it, unsigned long long purpose) {
    return sa_sm64(sa_sm64(seed ^ (chain * 0xD1B54A32D192ED03ull)) + ((it << 2) | purpose));
}
__device__ __forceinline__ unsigned sa_below(unsigned long long h, unsigned m) {
    return (unsigned)(((h >> 32) * (unsigned long long)m) >> 32);
}

struct SAArgs {
    int policy, chains, iters;
    unsigned long long seed;
    float p0, cool;
    const float *lam;                 // [A] load (min-resource)
    Slot *slots;                      // [gridDim.x] per-CTA best
    unsigned long long *chain_index;  // [chains] or nullptr
    unsigned *chain_key;              // [chains] or nullptr
    unsigned long long *accepted;     // total accepted moves (atomic)
};

__device__ __forceinline__ unsigned sa_key_of(const DevProb &P, int policy, const int *beta, const float *lam,
                                              const FullScore &s) {
    if (policy == 0) return s.verdict ? 0xFFFFFFFFu : objkey_maxload(s.T);
    const int y = eq2_gpus(P, beta, lam);
    return level_verdict(P, s, lam, y) ? 0xFFFFFFFFu : objkey_minres(s.u, s.U);
}

CAM_GLOBAL void __launch_bounds__(256) sa_kernel(const DevProb P, const SAArgs A) {
    __shared__ unsigned long long sk[8], sx[8];
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long bx = ~0ull;
    unsigned bk = 0xFFFFFFFFu;
    unsigned acc = 0;
    if (c < A.chains) {
        const int nA = P.A, n = P.n, K = nA + 2 * n;
        int rad[AMAX + 2 * NMAX], d[AMAX + 2 * NMAX];
        for (int a = 0; a < nA; ++a) rad[a] = P.nS;
        for (int i = 0; i < n; ++i) {
            rad[nA + 2 * i] = P.Rmax;
            rad[nA + 2 * i + 1] = P.nQ;
        }
        for (int k = 0; k < K; ++k) d[k] = (int)sa_below(sa_rng(A.seed, c, k, 3), (unsigned)rad[k]);
        int beta[AMAX], rho[NMAX], theta[NMAX];
        auto unpack = [&](const int *v) {
            for (int a = 0; a < nA; ++a) beta[a] = v[a];
            for (int i = 0; i < n; ++i) {
                rho[i] = v[nA + 2 * i];
                theta[i] = v[nA + 2 * i + 1];
            }
        };
        auto encode = [&](const int *v) {
            unsigned long long x = 0;
            for (int k = 0; k < K; ++k) x = x * (unsigned long long)rad[k] + (unsigned long long)v[k];
            return x;
        };
        FullScore s;
        unpack(d);
        score_digits(P, beta, rho, theta, s);
        unsigned kc = sa_key_of(P, A.policy, beta, A.lam, s);
        bool valid = kc != 0xFFFFFFFFu;
        bk = kc;
        bx = valid ? encode(d) : ~0ull;
        float p = A.p0;
        int e[AMAX + 2 * NMAX];
        for (int it = 0; it < A.iters; ++it) {
            const int k = (int)sa_below(sa_rng(A.seed, c, it, 0), (unsigned)K);
            const int dir = (sa_rng(A.seed, c, it, 1) >> 63) ? 1 : -1;
            const float u = (float)(sa_rng(A.seed, c, it, 2) >> 40) * (1.0f / 16777216.0f);
            for (int q = 0; q < K; ++q) e[q] = d[q];
            if (rad[k] > 1) {
                int nd = d[k] + dir;
                if (nd < 0 || nd >= rad[k]) nd = d[k] - dir;
                e[k] = nd;
            }
            unpack(e);
            score_digits(P, beta, rho, theta, s);
            const unsigned kn = sa_key_of(P, A.policy, beta, A.lam, s);
            const bool vn = kn != 0xFFFFFFFFu;
            const unsigned long long xn = encode(e);
            if (vn && (kn < bk || (kn == bk && xn < bx))) {
                bk = kn;
                bx = xn;
            }
            bool accept;
            if (!valid) accept = true;
            else if (!vn) accept = false;
            else if (kn <= kc) accept = true;
            else accept = u < p;
            if (accept) {
                for (int q = 0; q < K; ++q) d[q] = e[q];
                kc = kn;
                valid = vn;
                ++acc;
            }
            p = __fmul_rn(p, A.cool);
        }
        if (bx == ~0ull) bk = 0xFFFFFFFFu;
        if (A.chain_index) A.chain_index[c] = bx;
        if (A.chain_key) A.chain_key[c] = bk;
    }
    // block best (key, index) -> slot; accepted-move count
    unsigned long long k64 = bk, x64 = bx;
    for (int off = 16; off; off >>= 1) {
        const unsigned long long ok = __shfl_xor_sync(0xffffffffu, k64, off);
        const unsigned long long ox = __shfl_xor_sync(0xffffffffu, x64, off);
        if (slot_less(ok, ox, k64, x64)) {
            k64 = ok;
            x64 = ox;
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, off);
    }
    if (lane == 0) {
        sk[wid] = k64;
        sx[wid] = x64;
        if (acc) atomicAdd(A.accepted, (unsigned long long)acc);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long kb = sk[0], xb = sx[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (slot_less(sk[w], sx[w], kb, xb)) {
                kb = sk[w];
                xb = sx[w];
            }
        A.slots[blockIdx.x].key = kb;
        A.slots[blockIdx.x].x = xb;
    }
}

}  // namespace cam

// ============================================================================
// NEXT-3: decision-tree performance models evaluated on
// the device into the predictor table: one thread per (tree, batch, quota).
namespace cam {

CAM_GLOBAL void tree_table_kernel(int n_trees, const int4 *nodes, const float *values, const int *off,
                                  int nS, const int *batch, int nQ, const int *quota, float *table) {
    const long long total = (long long)n_trees * nS * nQ;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int q = (int)(t % nQ), b = (int)((t / nQ) % nS), tr = (int)(t / ((long long)nQ * nS));
        const int s = batch[b], p = quota[q];
        const int base = off[tr], m = off[tr + 1] - base;
        int k = 0;
        float v = __int_as_float(0x7fc00000);   // NaN: malformed (validated on the host)
        for (int step = 0; step <= m; ++step) {
            const int4 nd = nodes[base + k];
            if (nd.x < 0) {
                v = values[base + k];
                break;
            }
            k = ((nd.x == 0 ? s : p) <= nd.y) ? nd.z : nd.w;
        }
        const int i = tr / 3, c = tr % 3;
        float *cell = table + (((size_t)i * nS + b) * nQ + q) * 4;
        cell[c] = v;
        if (c == 0) cell[3] = 0.0f;
    }
}

}  // namespace cam

// ============================================================================
// NEXT-4: tail-latency simulation of one plan (reading R32; PAPER.md L527
// batching at the entry, L514 / L834 the 99%-ile QoS).  One CTA per
// simulation: thread 0 runs the queueing recursion of each application
// (Poisson arrivals from a counter-based stream, batches of s_a queries,
// round-robin replicas, FIFO, contended durations, hand-overs) and writes the
// measured latencies; the CTA then selects the exact ceil(0.99 M)-th smallest
// by an 8-pass byte radix select on the (positive, hence ordered) double bit
// patterns.
namespace cam {

__device__ __forceinline__ unsigned long long sim_sm64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct SimArgs {
    unsigned long long x;                  // candidate (canonical index)
    float lam[AMAX];                       // load per application (QPS)
    long long n_queries, warmup;
    unsigned long long seed;
    double *lat;                           // [n_sims][n_queries]
    double *out;                           // [n_sims][A][2] = (p99, mean)
};

CAM_GLOBAL void __launch_bounds__(256) simulate_kernel(const DevProb P, const SimArgs A) {
    __shared__ FullScore sc;
    __shared__ double freet[NMAX][CAMELOT_MAX_REPLICAS];
    __shared__ unsigned int hist[256];
    __shared__ unsigned long long sel[2];   // prefix, remaining rank
    __shared__ double s_sum;
    __shared__ int s_ok;
    __shared__ ScoreScratch scr;
    const unsigned long long sim = blockIdx.x;
    double *lat = A.lat + sim * (unsigned long long)A.n_queries;
    int beta[AMAX], rho[NMAX], theta[NMAX];
    decode_index(P, A.x, beta, rho, theta);
    if (threadIdx.x == 0) {
        FullScore f;
        score_digits(P, beta, rho, theta, f, &scr);
        sc = f;
        s_ok = f.place_viol == 0;
    }
    __syncthreads();
    for (int a = 0; a < P.A; ++a) {
        if (threadIdx.x == 0 && s_ok) {
            const int s = P.S[beta[a]];
            const int first = P.first_of_app[a], last = P.last_of_app[a];
            for (int i = 0; i < NMAX; ++i)
                for (int r = 0; r < CAMELOT_MAX_REPLICAS; ++r) freet[i][r] = 0.0;
            const double scale = 1000.0 / (double)A.lam[a];
            const unsigned long long base = sim_sm64(A.seed ^ (sim * 0xD1B54A32D192ED03ull));
            const long long total = A.warmup + A.n_queries;
            const long long nbatch = (total + s - 1) / s;
            double t = 0.0, sum = 0.0;
            long long m = 0;
            for (long long b = 0; b < nbatch; ++b) {
                const double t0 = t;   // arrivals of this batch are regenerated below (no per-batch buffer)
                for (int j = 0; j < s; ++j) {
                    const unsigned long long q = (unsigned long long)(b * s + j);
                    const unsigned long long h = sim_sm64(base + (((unsigned long long)a << 40) | q));
                    const double u = ((double)(h >> 11) + 0.5) * 0x1.0p-53;
                    t = __dadd_rn(t, __dmul_rn(-log(u), scale));
                }
                double ready = t;
                for (int i = first; i <= last; ++i) {
                    const int r = (int)(b % (long long)(rho[i] + 1));
                    const double start = ready > freet[i][r] ? ready : freet[i][r];
                    const double fin = __dadd_rn(start, (double)sc.L[i]);
                    freet[i][r] = fin;
                    ready = fin;
                    if (i < last && (P.flags & F_COMM)) ready = __dadd_rn(ready, (double)sc.comm[i]);
                }
                double ta = t0;
                for (int j = 0; j < s; ++j) {
                    const long long q = b * s + j;
                    const unsigned long long h = sim_sm64(base + (((unsigned long long)a << 40) | (unsigned long long)q));
                    const double u = ((double)(h >> 11) + 0.5) * 0x1.0p-53;
                    ta = __dadd_rn(ta, __dmul_rn(-log(u), scale));
                    if (q < A.warmup || q >= total) continue;
                    const double l = __dsub_rn(ready, ta);
                    lat[m++] = l;
                    sum = __dadd_rn(sum, l);
                }
            }
            s_sum = sum;
            sel[0] = 0;
            sel[1] = (unsigned long long)max(0ll, (long long)ceil(0.99 * (double)m) - 1);
        }
        __syncthreads();
        if (!s_ok) {
            if (threadIdx.x == 0) {
                A.out[(sim * P.A + a) * 2 + 0] = -1.0;
                A.out[(sim * P.A + a) * 2 + 1] = -1.0;
            }
            __syncthreads();
            continue;
        }
        // exact order statistic: byte radix select, most significant byte first
        const long long M = A.n_queries;
        for (int byte = 7; byte >= 0; --byte) {
            for (int t2 = threadIdx.x; t2 < 256; t2 += blockDim.x) hist[t2] = 0u;
            __syncthreads();
            const unsigned long long prefix = sel[0];
            const unsigned long long hmask = byte == 7 ? 0ull : (~0ull << (8 * (byte + 1)));
            for (long long q = threadIdx.x; q < M; q += blockDim.x) {
                const unsigned long long key = (unsigned long long)__double_as_longlong(lat[q]);
                if ((key & hmask) == prefix) atomicAdd(&hist[(key >> (8 * byte)) & 255u], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long k = sel[1];
                int d = 0;
                while (d < 255 && k >= hist[d]) {
                    k -= hist[d];
                    ++d;
                }
                sel[0] = prefix | ((unsigned long long)d << (8 * byte));
                sel[1] = k;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            A.out[(sim * P.A + a) * 2 + 0] = __longlong_as_double((long long)sel[0]);
            A.out[(sim * P.A + a) * 2 + 1] = s_sum / (double)M;
        }
        __syncthreads();
    }
}

}  // namespace cam
