/*
 * camelot.h -- C ABI of the B200-native contention-aware allocation search of
 * Camelot (arXiv 2005.02088).
 *
 * PAPER.md below = the paper's LaTeX source (/root/reference/PAPER.md, line
 * numbers); R<nn> = the numbered readings in DESIGN.md (where the paper is
 * silent, ambiguous or garbled).
 *
 * WHAT IS COMPUTED.  A *candidate plan* fixes, for a pipeline of n
 * microservice stages (one or two applications, stages app-major), one batch
 * size s_a per application ("batch size should also be
 * considered as a variable"), and per stage i a replica count N_i and one SM
 * quota p_i shared by its replicas (the SA state V = [n1..nN, p1..pN],
 * PAPER.md L882-883).  Each candidate is
 *   1. placed on the C modeled GPUs with the paper's deployment scheme
 *      (listing L955-979; readings R14-R16),
 *   2. checked against Eq. 1 / Eq. 3's constraints per GPU after placement
 *      (quota, MPS client cap I = 48 (L779-780), memory, bandwidth; R3, R4),
 *   3. scored by the contention-aware predictor: co-located stages' bandwidth
 *      pressure inflates their latency (L424-429, L1164-1170; R17), pipeline
 *      throughput = min over stages (L384, L766), latency sum vs QoS
 *      (Constraint-5, L834; R1),
 * and the exact optimum is reduced out:
 *   - camelot_plan_max_load: maximise the supported peak load T (Eq. 1,
 *     PAPER.md L825-836);
 *   - camelot_plan_min_resource: minimise (GPUs used, sum N_i p_i)
 *     lexicographically at a given low load ("first minimizes the number of
 *     GPUs ... then the resource usage", L842; Eq. 3; R10, R11),
 *     for several load levels in one pass.
 * Ties go to the smallest canonical candidate index (R20).  The search is
 * exhaustive and exact (a superset of the paper's simulated annealing,
 * L880-888): exact bounds only discard candidates that provably cannot be
 * feasible and at least as good as a known feasible candidate (DESIGN.md
 * "Exact pruning").
 *
 * CANONICAL INDEX.  Digits, most significant first:
 *   beta_1..beta_A (radix nS), then for i = 1..n: rho_i (radix Rmax),
 *   theta_i (radix nQ);   N_i = rho_i + 1, p_i = quota_pct[theta_i],
 *   s_a = batch[beta_a].   Ntot = nS^A * (Rmax*nQ)^n.
 *
 * ARITHMETIC.  IEEE binary32, round-to-nearest-even, no FMA contraction, no
 * FTZ, in the order of DESIGN.md "Scoring definition"; quota, instance and MiB
 * accounting in integers.  Results are bit-identical to the CPU oracle.
 *
 * MEMORY / OWNERSHIP.  All pointers in these structs are caller-owned host
 * pointers unless marked "device".  The library never retains a pointer after
 * a call returns and never allocates device memory: all device memory is the
 * caller's workspace (e.g. a torch uint8 tensor) of camelot_workspace_bytes()
 * bytes, passed in camelot_exec.  Work is enqueued on exec->stream; calls that
 * return host results synchronise that stream before returning.
 *
 * ERRORS.  Every entry point returns a camelot_status.  CAMELOT_INFEASIBLE is
 * a result (no candidate satisfies the constraints), not an error.  On an
 * error (< 0) the out-params are untouched and camelot_last_error() returns a
 * thread-local message.  There is NO CPU fallback: without a CUDA device every
 * compute entry point returns CAMELOT_ENODEV.
 *
 * THREADING.  Inputs are read-only and may be shared between threads; calls on
 * different streams with different workspaces are independent.  A workspace
 * must not be used by two calls concurrently.
 */
#ifndef CAMELOT_H
#define CAMELOT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CAMELOT_MAX_STAGES 8
#define CAMELOT_MAX_APPS 2
#define CAMELOT_MAX_GPUS 16
#define CAMELOT_MAX_REPLICAS 16
#define CAMELOT_MAX_QUOTAS 128
#define CAMELOT_MAX_BATCHES 64
#define CAMELOT_MAX_LOADS 64

typedef enum {
    CAMELOT_OK = 0,
    CAMELOT_INFEASIBLE = 1, /* result: no feasible candidate                   */
    CAMELOT_EINVAL = -1,    /* invalid argument (see camelot_last_error)        */
    CAMELOT_ERANGE = -2,    /* space / key / size limits exceeded               */
    CAMELOT_ECUDA = -3,     /* CUDA runtime error                               */
    CAMELOT_ENODEV = -4,    /* no CUDA device: there is no CPU fallback         */
    CAMELOT_ENOMEM = -5     /* workspace too small                              */
} camelot_status;

/* problem flags (camelot_problem.flags) */
#define CAMELOT_F_NO_BW_CAP 1u      /* drop the per-GPU bandwidth constraint (Constraint-3)      */
#define CAMELOT_F_NO_CONTENTION 2u  /* kappa = 1: contention-blind predictor (Camelot-NC, R18)   */
#define CAMELOT_F_SAT 4u            /* kappa *= max(1, dem/BW) (oversubscription, R17)           */
#define CAMELOT_F_PAPER_GLOBAL 8u   /* literal Eq. 1 global sums, no placement (R3; pins only)   */
#define CAMELOT_F_EQ2_BUDGET 16u    /* min-resource: enforce GPUs used <= Eq. 2's y (R9)         */
#define CAMELOT_F_NO_FILTER 32u     /* exhaustive scan without pruning (flat mode)               */
#define CAMELOT_F_COMM 64u          /* NEXT-2: communication-aware QoS (R29): the hand-over from
                                       stage i to i+1 of an app is added to the latency sum;
                                       same-GPU (global-memory IPC) only when
                                       both stages run entirely on one and the same GPU, else a
                                       host-staged copy (L442-448).  Not with PAPER_GLOBAL.     */

/* first-failing-check bits (camelot_plan.violations, score vectors) */
#define CAMELOT_V_QUOTA 1u  /* placement: SM quota per GPU                 */
#define CAMELOT_V_INST 2u   /* placement: instances per GPU > I            */
#define CAMELOT_V_MEM 4u    /* placement: global memory capacity           */
#define CAMELOT_V_BW 8u     /* placement: global memory bandwidth          */
#define CAMELOT_V_QOS 16u   /* end-to-end latency sum > QoS                */
#define CAMELOT_V_LOAD 32u  /* min-resource: throughput below the load     */
#define CAMELOT_V_EQ2 64u   /* min-resource: GPUs used > Eq. 2 estimate    */

#define CAMELOT_POLICY_MAX_LOAD 0
#define CAMELOT_POLICY_MIN_RESOURCE 1

/* One modeled GPU type, C copies (Table 2). */
typedef struct {
    int32_t n_gpus;        /* C, 1..16                                          */
    int32_t quota_per_gpu; /* R, SM quota of one GPU in %, 1..127 (paper: 100)  */
    int32_t max_instances; /* I, MPS clients per GPU (paper: 48, L779-780)      */
    float bw_gbs;          /* BW, global memory bandwidth per GPU (GB/s, > 0)   */
    uint32_t mem_mib;      /* F, global memory per GPU (MiB), < 2^21            */
    float gflops;          /* G, GFLOPS per GPU (Eq. 2 only, > 0)               */
    float link_gbs;        /* CAMELOT_F_COMM: cross-GPU hand-over bandwidth (GB/s, > 0);
                              t = fl(fl(comm_mb_i * s) * fl(1/link_gbs)) ms         */
    float ipc_ms;          /* CAMELOT_F_COMM: same-GPU hand-over time (ms, >= 0)     */
} camelot_cluster;

/* The allocation problem.  Per-stage predictions are tabulated on the
 * (batch, quota) grid: the paper predicts per (batch, SM%) before allocating
 * (PAPER.md L527 steps 3-4, L664-703). */
typedef struct {
    int32_t n_apps;                /* A, 1 or 2                                       */
    int32_t n_stages;              /* n, 1..8 (sum over apps)                          */
    const int32_t *app_of_stage;   /* [n] 0..A-1, non-decreasing (app-major order)     */
    const float *qos_ms;           /* [A] QoS target per application (ms, > 0)         */
    int32_t n_quota;               /* nQ, 1..128                                       */
    const int32_t *quota_pct;      /* [nQ] strictly ascending, in [1, R]               */
    int32_t n_batch;               /* nS, 1..64                                        */
    const int32_t *batch;          /* [nS] strictly ascending, >= 1                    */
    int32_t max_replicas;          /* Rmax, 1..16: N_i in [1, Rmax]                    */
    const float *table;            /* [n][nS][nQ][4]: dur_ms (>0), thr_qps (>0),
                                      bw_gbs (>=0), unused -- f(p), g(p) of Table 2    */
    const uint32_t *weights_mib;   /* [n] W_i:  M(i,s) = W_i + A_i*s (L700-703)        */
    const uint32_t *act_mib_per_item; /* [n] A_i                                      */
    const float *gflop_per_item;   /* [n] c_i:  C(i,s) = c_i*s (Eq. 2 only)            */
    const float *bw_sensitivity;   /* [n] gamma_i >= 0 (R17; 0 = paper-strict)         */
    uint32_t flags;                /* CAMELOT_F_*                                      */
    const float *comm_mb_per_item; /* [n] CAMELOT_F_COMM: MB per batch item sent from stage i
                                      to stage i+1 of its app (>= 0; unused for the last
                                      stage of an app); may be NULL without the flag   */
} camelot_problem;

/* Execution context.  rank/world shard the candidate space (chunk c is searched
 * by rank c mod world); index_lo/index_hi restrict the search to canonical
 * indices [lo, hi) (0,0 = the whole space). */
#define CAMELOT_EXEC_RESIDENT 1u  /* the workspace already holds this problem
                                     (camelot_upload): skip the host->device copy
                                     and the host scan of the table values (the
                                     uploaded image was validated) */
#define CAMELOT_EXEC_NAIVE 2u     /* use the un-hoisted thread-per-candidate scan
                                     (baseline; always used for PAPER_GLOBAL or n = 1) */
typedef struct {
    int32_t device;           /* CUDA device ordinal                                */
    void *stream;             /* cudaStream_t (e.g. torch.cuda.current_stream())    */
    int32_t rank, world;      /* 0 <= rank < world                                   */
    uint64_t index_lo, index_hi;
    void *workspace;          /* device memory, caller-owned                         */
    size_t workspace_bytes;
    uint32_t exec_flags;      /* CAMELOT_EXEC_*                                      */
} camelot_exec;

/* The result of a plan call (one per load level for min-resource). */
typedef struct {
    uint64_t index;           /* canonical candidate index; UINT64_MAX if none      */
    int32_t status;           /* CAMELOT_OK or CAMELOT_INFEASIBLE                   */
    int32_t batch[CAMELOT_MAX_APPS];                 /* s_a                          */
    int32_t replicas[CAMELOT_MAX_STAGES];            /* N_i                          */
    int32_t quota_pct[CAMELOT_MAX_STAGES];           /* p_i                          */
    int8_t gpu_of_instance[CAMELOT_MAX_STAGES * CAMELOT_MAX_REPLICAS]; /* -1 unused;
                                 replicas of stage i listed by GPU index             */
    float stage_latency_ms[CAMELOT_MAX_STAGES];      /* L_i (contended)              */
    float stage_throughput_qps[CAMELOT_MAX_STAGES];  /* T_i                          */
    float kappa[CAMELOT_MAX_STAGES];                 /* contention inflation         */
    float e2e_latency_ms[CAMELOT_MAX_APPS];          /* Lsum_a                       */
    float throughput_qps[CAMELOT_MAX_APPS];          /* Tmin_a                       */
    float objective;          /* T (max-load) or U (min-resource)                   */
    int32_t quota_used;       /* U = sum N_i p_i                                     */
    int32_t gpus_used;        /* u                                                   */
    int32_t eq2_gpus;         /* y (Eq. 2, R9) at this load level; 0 for max-load    */
    uint32_t violations;      /* first failing check of this plan (0 = feasible);
                                 for INFEASIBLE results: OR of the first-failing checks
                                 of the scanned candidates (placement bits = the
                                 dimensions where fits(g, 1) fails after pass 2,
                                 DESIGN.md 3.2); exact in CAMELOT_F_NO_FILTER mode, a
                                 subset when bounds skip candidates                  */
    uint64_t n_feasible;      /* candidates seen that pass placement and QoS (the   */
                              /* load-independent checks; exact in NO_FILTER mode)  */
    uint64_t n_scored;        /* candidates fully scored by the search               */
    uint64_t n_covered;       /* candidates covered (scored or excluded by a bound)  */
    float comm_ms[CAMELOT_MAX_STAGES];  /* CAMELOT_F_COMM: hand-over time of edge i -> i+1 (ms) */
    uint64_t n_evaluated;     /* leaves + inner nodes evaluated by the whole search
                                 (incumbent cascade + main pass) of this call         */
    uint64_t search_ns;       /* device time of that search (CUDA events on the stream,
                                 ns) when searched and finalized on this thread, else 0 */
} camelot_plan;

/* ------------------------------------------------------------------ entry points */

/* Thread-local message of the last error (never NULL). */
const char *camelot_last_error(void);
const char *camelot_version(void);

/* Bytes of device workspace needed for this problem with up to n_loads load
 * levels (0 for max-load only).  Returns 0 and sets the error on invalid input. */
size_t camelot_workspace_bytes(const camelot_problem *p, const camelot_cluster *c, int n_loads);

/* Validate and copy the problem into the workspace (host->device on
 * exec->stream; asynchronous).  Later calls may pass CAMELOT_EXEC_RESIDENT. */
int camelot_upload(const camelot_problem *p, const camelot_cluster *c, const camelot_exec *exec);

/* Max peak load (Eq. 1).  Single-process entry: searches exec's range (all of
 * it for rank 0 of world 1) and writes the plan to *out (host). */
int camelot_plan_max_load(const camelot_problem *p, const camelot_cluster *c,
                          const camelot_exec *exec, camelot_plan *out);

/* Min resource (Eq. 2-3) at n_loads load levels in one pass.
 * load_qps: host [n_loads][A] (> 0).  out: host [n_loads]. */
int camelot_plan_min_resource(const camelot_problem *p, const camelot_cluster *c,
                              const float *load_qps, int n_loads,
                              const camelot_exec *exec, camelot_plan *out);

/* Both policies back to back, as Camelot uses them (the
 * low-load allocation is planned at 30% of the peak the max-load policy
 * supports): out[0] = the max-load plan (Eq. 1), out[1] = the min-resource plan
 * (Eq. 3) at load_a = fl32(low_load_frac * T*) for every application a, T* =
 * out[0].objective (the float64 product rounded to binary32, as a host caller
 * computing it in double would).  The load is derived ON THE DEVICE from the
 * max-load winner's objective key, so the two exact searches run back to back on
 * exec->stream with one host synchronisation at the end (no host round trip
 * between the policies); the max-load plan itself is scored on an internal second
 * stream of the calling thread while the min-resource search runs, and exec->stream
 * waits for it (an event) before the plans are copied out.  No feasible peak: out[1] is INFEASIBLE with violations = V_LOAD
 * (the min-resource search then runs at load +inf and finds nothing).  Same result
 * as camelot_plan_max_load followed by camelot_plan_min_resource at that load.
 * low_load_frac in (0, 1]; world must be 1; out: host [2].  Returns CAMELOT_OK
 * if both plans are feasible, else CAMELOT_INFEASIBLE (plans still written). */
int camelot_plan_max_then_min(const camelot_problem *p, const camelot_cluster *c,
                              double low_load_frac, const camelot_exec *exec,
                              camelot_plan *out);

/* Score ONE explicit plan (oracle_predict counterpart).  batch: [A] batch SIZES
 * (values on the grid), replicas: [n] N_i, quota_pct: [n] p_i (on the grid);
 * a value off the grid is CAMELOT_EINVAL.  load_qps [n_loads][A] may be NULL.
 * out->violations = first failing check (max-load; with loads: level 0). */
int camelot_predict(const camelot_problem *p, const camelot_cluster *c,
                    const int32_t *batch, const int32_t *replicas, const int32_t *quota_pct,
                    const float *load_qps, int n_loads,
                    const camelot_exec *exec, camelot_plan *out);

/* Score ONE candidate given by its canonical index (0 <= index < Ntot, else
 * CAMELOT_EINVAL): the device decodes the mixed-radix digits (beta_a, rho_i,
 * theta_i; CANONICAL INDEX above) and scores the plan as
 * camelot_predict does.  load_qps [1][A] may be NULL (n_loads = 0). */
int camelot_predict_index(const camelot_problem *p, const camelot_cluster *c, uint64_t index,
                          const float *load_qps, int n_loads, const camelot_exec *exec, camelot_plan *out);

/* Score every candidate of [lo, hi) (hi - lo <= 2^31) on the device.
 * Device outputs (any may be NULL): d_verdict u8 [hi-lo] first failing check
 * (max-load), d_T f32 [hi-lo], d_u i32, d_U i32.  Asynchronous. */
int camelot_score_range(const camelot_problem *p, const camelot_cluster *c,
                        uint64_t lo, uint64_t hi, const camelot_exec *exec,
                        uint8_t *d_verdict, float *d_T, int32_t *d_u, int32_t *d_U);

/* ---- multi-GPU split: the caller's process group does ONE allreduce-min ----
 * camelot_search_local searches this rank's shard and writes n_keys int64
 * keys to DEVICE memory d_keys (n_keys = 1 for max-load, n_loads for
 * min-resource).  Key = (objective key << 32 | chunk-or-index) ^ 2^63, so that
 * a signed int64 MIN over ranks is the unsigned min (INT64_MAX = none).
 * Asynchronous (no host synchronisation).  After
 *     torch.distributed.all_reduce(keys, op=MIN)
 * every rank calls camelot_finalize with the reduced DEVICE keys; it recovers
 * the exact winning index (re-scanning the winning chunk when Ntot > 2^32),
 * scores it and writes the plans to host out[n_keys].
 * Pairing contract: camelot_finalize reads what the LAST camelot_search_local
 * left in the same workspace (local best, filtered option lists, loads), so it
 * must be called with the same problem, policy, n_loads, load_qps, index range,
 * rank and world, and no other call that rewrites the workspace in between
 * (any entry point other than camelot_finalize / camelot_last_stats /
 * camelot_trace does); otherwise it returns CAMELOT_EINVAL. */
int camelot_search_local(const camelot_problem *p, const camelot_cluster *c, int policy,
                         const float *load_qps, int n_loads, const camelot_exec *exec,
                         int64_t *d_keys);
int camelot_finalize(const camelot_problem *p, const camelot_cluster *c, int policy,
                     const float *load_qps, int n_loads, const int64_t *d_keys,
                     const camelot_exec *exec, camelot_plan *out);

/* Statistics of the last search on this workspace (host out[8], synchronises
 * the stream): [0] leaf candidates scored by the main pass, [1] inner tree
 * nodes evaluated by the main pass, [2] feasible candidates seen, [3] device
 * time of the whole search (incumbent cascade + main pass, CUDA events on
 * exec->stream, ns), [4] depth-d0 work items of the main pass, [5] kernels
 * launched by the last plan/search call, [6] leaves and [7] inner nodes
 * evaluated over the cascade and the main pass. */
int camelot_last_stats(const camelot_exec *exec, uint64_t *out8);

/* Phase trace of the last search on this workspace (profiling aid; host
 * out[cap], synchronises the stream).  Block 0 of every search-level launch
 * (incumbent cascade levels, then the main pass) records, after each grid-wide
 * barrier, (tag << 48) | (%globaltimer ns & 2^48-1) with tag 0 = launch start,
 * 1 = header reset, 2 = option filter, 3 = item offsets, 16+j = pass j,
 * 32 = CTA reduction.  Returns the number of entries recorded (may exceed cap;
 * at most 256 are kept) or a negative status. */
int camelot_trace(const camelot_exec *exec, uint64_t *out, int cap);

/* NEXT-3: the paper's decision-tree performance models (one
 * regression tree per microservice and target, features batch size s and SM
 * quota p; trained offline, L706).  Flattened tree: node k is a leaf when
 * feature[k] < 0 (prediction value[k]); otherwise x = (feature[k] == 0 ? s : p)
 * goes to left[k] when x <= threshold[k], else to right[k]; child indices must
 * be larger than their parent's (so every walk ends within n_nodes steps). */
typedef struct {
    int32_t n_nodes;          /* >= 1                                                */
    const int32_t *feature;   /* [n_nodes] 0 = batch size, 1 = SM quota (%), -1 = leaf */
    const int32_t *threshold; /* [n_nodes]                                           */
    const int32_t *left;      /* [n_nodes] child index (internal nodes)              */
    const int32_t *right;     /* [n_nodes]                                           */
    const float *value;       /* [n_nodes] leaf prediction                           */
} camelot_tree;

/* Workspace bytes camelot_tables_from_trees needs (0 on invalid arguments). */
size_t camelot_trees_workspace_bytes(int n_trees, const camelot_tree *trees, int n_batch, int n_quota);

/* Build the predictor table of a problem on the device from its trees: for every
 * stage i, trees[3i + c] (c = 0 duration ms, 1 throughput QPS, 2 bandwidth GB/s)
 * are evaluated at every (batch[b], quota_pct[q]) grid point -- any grid, not
 * only the profiling one -- into d_table[i][b][q][c] (float, [n][nS][nQ][4],
 * component 3 = 0), a DEVICE pointer owned by the caller.  Host inputs are
 * copied into exec->workspace (>= camelot_trees_workspace_bytes).  Asynchronous
 * on exec->stream.  EINVAL: malformed tree (feature not in {-1,0,1}, child index
 * not in (k, n_nodes)), empty grid, null pointers. */
int camelot_tables_from_trees(int n_stages, const camelot_tree *trees, int n_batch, const int32_t *batch,
                              int n_quota, const int32_t *quota_pct, const camelot_exec *exec, float *d_table);

/* NEXT-4: tail-latency simulation of ONE plan (reading R32; PAPER.md L527,
 * L514, L834).  Per application: Poisson arrivals at load_qps[a] from a
 * counter-based stream (u = ((h >> 11) + 0.5) 2^-53, h = splitmix64(splitmix64(
 * seed ^ sim * 0xD1B54A32D192ED03) + (a << 40 | q)), gap = -log(u) 1000/load ms),
 * batches of s_a consecutive queries released at their last arrival, stage i
 * serving batch b on replica b mod N_i FIFO for its contended duration L_i,
 * hand-overs under CAMELOT_F_COMM; latency = completion at the app's last stage
 * - arrival.  n_sims independent simulations (sim = 0..n_sims-1), each
 * discarding `warmup` queries and measuring n_queries: host out p99_ms and
 * mean_ms [n_sims][A] (the ceil(0.99 M)-th smallest latency and the mean; -1
 * when the plan cannot be placed).  The workspace must hold
 * camelot_simulate_workspace_bytes().  Synchronous. */
size_t camelot_simulate_workspace_bytes(const camelot_problem *p, const camelot_cluster *c, int64_t n_queries,
                                        int n_sims);
int camelot_simulate(const camelot_problem *p, const camelot_cluster *c, const int32_t *batch,
                     const int32_t *replicas, const int32_t *quota_pct, const float *load_qps, int64_t n_queries,
                     int64_t warmup, uint64_t seed, int n_sims, const camelot_exec *exec, double *p99_ms,
                     double *mean_ms);

/* Process-wide number of kernels launched by this library so far. */
uint64_t camelot_kernel_launches(void);

/* The paper's own solver (NEXT-1): simulated annealing over V = [n1..nN,
 * p1..pN] plus the batch digit(s) (reading R13), run as
 * `chains` independent chains of `iters` moves on the device.  A move changes
 * one random digit by +-1 (reflected at the grid edge); invalid states are
 * rejected once the chain is valid; a worse valid state is accepted with
 * probability p0 * cool^k at iteration k; every valid proposal that improves
 * the objective updates the best.  Randomness is counter-based:
 *   h(seed, chain, k, purpose) = sm64(sm64(seed ^ chain*0xD1B54A32D192ED03) + (k<<2 | purpose))
 * (sm64 = splitmix64; purposes 0 digit, 1 direction, 2 acceptance, 3 initial
 * digit k), so a chain is reproducible anywhere.  policy: CAMELOT_POLICY_*;
 * load_qps: host [A] (min-resource) or NULL.  out: best plan over all chains
 * (INFEASIBLE if no chain reached a valid state).  Optional DEVICE outputs
 * d_chain_index [chains] (UINT64_MAX = none) and d_chain_key [chains] (the
 * 32-bit objective key of each chain's best).  chains <= 2^20. */
int camelot_sa(const camelot_problem *p, const camelot_cluster *c, int policy, const float *load_qps,
               uint64_t seed, int chains, int iters, float p0, float cool, const camelot_exec *exec,
               camelot_plan *out, uint64_t *d_chain_index, uint32_t *d_chain_key);

#ifdef __cplusplus
}
#endif
#endif /* CAMELOT_H */
