/*
 * camelot_oracle.c -- plain, slow CPU oracle for the Camelot allocation search.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2005_02088_b200/csrc/).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, line numbers):
 *   - the candidate space: one batch size per application (PAPER.md L858,
 *     "batch size should also be considered as a variable"), and per stage i a
 *     replica count N_i and an SM quota p_i shared by its replicas (the SA state
 *     vector V = [n1..nN, p1..pN]), all on given grids;
 *   - the deployment scheme of PAPER.md L916-945 (sort GPUs by remaining
 *     resources, global memory first, fewest resources first; all replicas of a
 *     stage on one GPU if possible; listing PAPER.md) -- DESIGN.md
 *     readings R14-R16;
 *   - the constraints of Eq. 1 / Eq. 3 per GPU
 *     after placement (prose PAPER.md L774-777: bandwidth "on a GPU") -- R3,R4;
 *   - the contention-aware predictor: co-located stages' bandwidth pressure
 *     inflates their latency -- reading R17;
 *   - objectives: Eq. 1 max of min_i N_i f(p_i) and the
 *     min-resource policy "first minimizes the number of GPUs ... then the
 *     resource usage" (Eq. 3) with a load floor -- R10,R11;
 *   - Eq. 2 GPU-count estimate -- reading R9.
 * Arithmetic: IEEE binary32, round-to-nearest-even, no FMA contraction
 * (compiled with -ffp-contract=off), every operation in the order written
 * below.  The paper fixes no precision; binary32 is the kernel's precision and
 * every output of the search is an integer decision (verdict, argmax), which
 * both sides therefore take in the same precision (R21).
 * A float64 re-evaluation of the latencies of a given placement is provided to
 * bound the binary32 rounding error (north_star: latencies within 1e-5 rel).
 *
 * Pins: tests/test_oracle_*.py (worked examples, closed forms, invariants,
 * brute force); see DESIGN.md "Oracle pins".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OC_MAX_STAGES 8
#define OC_MAX_APPS 2
#define OC_MAX_GPUS 16
#define OC_MAX_REPL 16
#define OC_MAX_LOADS 64

/* flags */
#define OC_NO_BW_CAP 1u
#define OC_NO_CONTENTION 2u
#define OC_SAT 4u
#define OC_PAPER_GLOBAL 8u
#define OC_EQ2_BUDGET 16u
#define OC_COMM 64u   /* NEXT-2: communication-aware QoS (R29) */

/* first-failing-check bits */
#define OC_V_QUOTA 1u
#define OC_V_INST 2u
#define OC_V_MEM 4u
#define OC_V_BW 8u
#define OC_V_QOS 16u
#define OC_V_LOAD 32u
#define OC_V_EQ2 64u

typedef struct {
    int32_t A, n;
    const int32_t *app;   /* [n] application of each stage, app-major order */
    const float *qos;     /* [A] QoS target (ms) */
    int32_t nQ;
    const int32_t *Q;     /* SM-quota grid (%) */
    int32_t nS;
    const int32_t *S;     /* batch grid */
    int32_t Rmax;         /* replicas N_i in 1..Rmax */
    const float *tab;     /* [n][nS][nQ][4] = dur_ms, thr_qps, bw_gbs, unused */
    const uint32_t *W;    /* [n] weights footprint (MiB) */
    const uint32_t *Am;   /* [n] activation footprint per batch item (MiB) */
    const float *cflop;   /* [n] GFLOP per item */
    const float *gamma;   /* [n] bandwidth sensitivity */
    uint32_t flags;
    int32_t C, R, I;      /* GPUs, quota per GPU (%), max instances per GPU */
    float BW;             /* GB/s per GPU */
    uint32_t FM;          /* MiB per GPU */
    float G;              /* GFLOPS per GPU */
    /* NEXT-2 (flag OC_COMM; reading R29) */
    const float *comm_mb; /* [n] MB per batch item sent from stage i to stage i+1 of its app */
    float link_gbs;       /* cross-GPU transfer bandwidth (GB/s): data staged through host memory */
    float ipc_ms;         /* same-GPU hand-over (global-memory IPC handle) time (ms) */
} oc_problem;

typedef struct {
    uint32_t verdict;         /* first failing check of the max-load policy (0 = feasible) */
    uint32_t place_viol;      /* placement failure bits (0 = placed) */
    float T;                  /* min over apps of Tmin_a */
    int32_t u, U;             /* GPUs used, sum N_i p_i */
    float Tmin[OC_MAX_APPS];
    float Lsum[OC_MAX_APPS];
    float L[OC_MAX_STAGES], Ti[OC_MAX_STAGES], kappa[OC_MAX_STAGES];
    double L64[OC_MAX_STAGES], T64[OC_MAX_STAGES], Lsum64[OC_MAX_APPS];
    int8_t gpu_of_instance[OC_MAX_STAGES * OC_MAX_REPL];  /* -1 = unused */
    float dem[OC_MAX_GPUS];
    float comm[OC_MAX_STAGES];             /* COMM: hand-over time of edge i -> i+1 (0: none) */
    uint32_t level_verdict[OC_MAX_LOADS];  /* min-resource: first failing check per load level */
    int32_t eq2_y[OC_MAX_LOADS];
} oc_score_t;

typedef struct {
    uint64_t index;       /* UINT64_MAX if no feasible candidate */
    float T;              /* objective (max-load) of the winner */
    int32_t u, U;
    uint64_t n_feasible;
    uint64_t n_scanned;
    uint64_t hist[7];     /* first-failing-check histogram: QUOTA..EQ2 (placement bits counted per bit) */
} oc_best_t;

/* ---------------------------------------------------------------- validation */
static int fin(float v) { return isfinite(v); }

int oc_validate(const oc_problem *P) {
    if (P->n < 1 || P->n > OC_MAX_STAGES) return -1;
    if (P->A < 1 || P->A > OC_MAX_APPS) return -1;
    if (P->C < 1 || P->C > OC_MAX_GPUS) return -2;
    if (P->R < 1 || P->R > 127 || P->I < 1) return -1;
    if (!(P->BW > 0.0f) || !fin(P->BW) || !(P->G > 0.0f) || P->FM < 1) return -1;
    if (P->Rmax < 1 || P->Rmax > OC_MAX_REPL) return -1;
    if (P->nQ < 1 || P->nS < 1) return -1;
    for (int k = 0; k < P->nQ; k++) {
        if (P->Q[k] < 1 || P->Q[k] > P->R) return -1;
        if (k > 0 && P->Q[k] <= P->Q[k - 1]) return -1;
    }
    for (int k = 0; k < P->nS; k++) {
        if (P->S[k] < 1) return -1;
        if (k > 0 && P->S[k] <= P->S[k - 1]) return -1;
    }
    for (int i = 0; i < P->n; i++) {
        if (P->app[i] < 0 || P->app[i] >= P->A) return -1;
        if (i > 0 && P->app[i] < P->app[i - 1]) return -1;
        if (!(P->gamma[i] >= 0.0f) || !fin(P->gamma[i])) return -1;
        if (!fin(P->cflop[i]) || P->cflop[i] < 0.0f) return -1;
    }
    if (P->app[0] != 0 || P->app[P->n - 1] != P->A - 1) return -1;
    if (P->flags & OC_COMM) {
        if (P->flags & OC_PAPER_GLOBAL) return -1;   /* no placement, no co-location */
        if (!(P->link_gbs > 0.0f) || !fin(P->link_gbs) || !(P->ipc_ms >= 0.0f) || !fin(P->ipc_ms)) return -1;
        for (int i = 0; i < P->n; i++)
            if (!(P->comm_mb[i] >= 0.0f) || !fin(P->comm_mb[i])) return -1;
    }
    for (int a = 0; a < P->A; a++)
        if (!(P->qos[a] > 0.0f) || !fin(P->qos[a])) return -1;
    for (long e = 0; e < (long)P->n * P->nS * P->nQ; e++) {
        const float *t = P->tab + 4 * e;
        if (!fin(t[0]) || !fin(t[1]) || !fin(t[2])) return -1;
        if (!(t[0] > 0.0f) || !(t[1] > 0.0f) || !(t[2] >= 0.0f)) return -1;
    }
    return 0;
}

/* Ntot = |S|^A * (Rmax*|Q|)^n ; 0 if >= 2^63 */
uint64_t oc_ntot(const oc_problem *P) {
    unsigned __int128 t = 1;
    for (int a = 0; a < P->A; a++) t *= (unsigned)P->nS;
    for (int i = 0; i < P->n; i++) t *= (unsigned)(P->Rmax * P->nQ);
    if (t >= ((unsigned __int128)1 << 63)) return 0;
    return (uint64_t)t;
}

/* Candidate digits, most significant first: beta_1..beta_A, rho_1, theta_1, ...,
 * rho_n, theta_n (DESIGN.md R-enum).  N_i = rho_i + 1, p_i = Q[theta_i],
 * s_a = S[beta_a]. */
void oc_decode(const oc_problem *P, uint64_t x, int32_t *beta, int32_t *rho, int32_t *theta) {
    for (int i = P->n - 1; i >= 0; i--) {
        theta[i] = (int32_t)(x % (uint64_t)P->nQ);
        x /= (uint64_t)P->nQ;
        rho[i] = (int32_t)(x % (uint64_t)P->Rmax);
        x /= (uint64_t)P->Rmax;
    }
    for (int a = P->A - 1; a >= 0; a--) {
        beta[a] = (int32_t)(x % (uint64_t)P->nS);
        x /= (uint64_t)P->nS;
    }
}

uint64_t oc_encode(const oc_problem *P, const int32_t *beta, const int32_t *rho, const int32_t *theta) {
    uint64_t x = 0;
    for (int a = 0; a < P->A; a++) x = x * (uint64_t)P->nS + (uint64_t)beta[a];
    for (int i = 0; i < P->n; i++) {
        x = x * (uint64_t)P->Rmax + (uint64_t)rho[i];
        x = x * (uint64_t)P->nQ + (uint64_t)theta[i];
    }
    return x;
}

static const float *entry(const oc_problem *P, int i, int b, int q) {
    return P->tab + 4 * (((long)i * P->nS + b) * P->nQ + q);
}

/* ------------------------------------------------------------------ placement
 * PAPER.md L929-945 + listing L955-979, readings R14-R16. */
typedef struct {
    int32_t rq[OC_MAX_GPUS];     /* remaining quota (%) */
    int32_t cnt[OC_MAX_GPUS];    /* instances hosted */
    int64_t rm[OC_MAX_GPUS];     /* remaining memory (MiB) */
    float dem[OC_MAX_GPUS];      /* accumulated bandwidth demand (GB/s) */
    int32_t host[OC_MAX_STAGES][OC_MAX_GPUS];
} oc_state;

/* can GPU g take k more replicas of stage i?  returns 0 if yes, else the
 * failing dimension bits */
static uint32_t fit_bits(const oc_problem *P, const oc_state *st, int i, int g, int k,
                         int32_t p, int64_t s, float bw) {
    uint32_t v = 0;
    if ((int64_t)k * p > st->rq[g]) v |= OC_V_QUOTA;
    if (st->cnt[g] + k > P->I) v |= OC_V_INST;
    int64_t need = (st->host[i][g] == 0 ? (int64_t)P->W[i] : 0) + (int64_t)k * (int64_t)P->Am[i] * s;
    if (need > st->rm[g]) v |= OC_V_MEM;
    if (!(P->flags & OC_NO_BW_CAP)) {
        float add = (float)k * bw;
        float tot = st->dem[g] + add;
        if (tot > P->BW) v |= OC_V_BW;
    }
    return v;
}

static int can_hold(const oc_problem *P, const oc_state *st, int i, int g, int m,
                    int32_t p, int64_t s, float bw) {
    for (int k = m; k >= 1; k--)
        if (fit_bits(P, st, i, g, k, p, s, bw) == 0) return k;
    return 0;
}

static void deploy(const oc_problem *P, oc_state *st, int i, int g, int k, int32_t p,
                   int64_t s, float bw) {
    st->rq[g] -= k * p;
    st->cnt[g] += k;
    st->rm[g] -= (st->host[i][g] == 0 ? (int64_t)P->W[i] : 0) + (int64_t)k * (int64_t)P->Am[i] * s;
    float add = (float)k * bw;
    st->dem[g] = st->dem[g] + add;
    st->host[i][g] += k;
}

/* returns 0 if every stage was placed, else the placement-failure bits */
static uint32_t place_all(const oc_problem *P, const int32_t *beta, const int32_t *rho,
                          const int32_t *theta, oc_state *st) {
    for (int g = 0; g < P->C; g++) {
        st->rq[g] = P->R;
        st->cnt[g] = 0;
        st->rm[g] = (int64_t)P->FM;
        st->dem[g] = 0.0f;
        for (int i = 0; i < P->n; i++) st->host[i][g] = 0;
    }
    for (int i = 0; i < P->n; i++) {
        int b = beta[P->app[i]];
        int64_t s = P->S[b];
        int32_t p = P->Q[theta[i]];
        int N = rho[i] + 1;
        float bw = entry(P, i, b, theta[i])[2];
        /* 1. snapshot order: GPUs by (remaining memory, remaining quota, index) ascending */
        int order[OC_MAX_GPUS];
        for (int g = 0; g < P->C; g++) order[g] = g;
        for (int a = 1; a < P->C; a++) {           /* insertion sort */
            int g = order[a], j = a - 1;
            while (j >= 0) {
                int h = order[j];
                int less = (st->rm[g] < st->rm[h]) ||
                           (st->rm[g] == st->rm[h] && st->rq[g] < st->rq[h]) ||
                           (st->rm[g] == st->rm[h] && st->rq[g] == st->rq[h] && g < h);
                if (!less) break;
                order[j + 1] = h;
                j--;
            }
            order[j + 1] = g;
        }
        /* 2. pass 1: all N_i replicas on the first GPU that holds them */
        int placed = 0;
        for (int j = 0; j < P->C && !placed; j++) {
            int g = order[j];
            if (can_hold(P, st, i, g, N, p, s, bw) == N) {
                deploy(P, st, i, g, N, p, s, bw);
                placed = 1;
            }
        }
        if (placed) continue;
        /* 3. pass 2: fill greedily in the same order */
        int rem = N;
        for (int j = 0; j < P->C && rem > 0; j++) {
            int g = order[j];
            int k = can_hold(P, st, i, g, rem, p, s, bw);
            if (k > 0) {
                deploy(P, st, i, g, k, p, s, bw);
                rem -= k;
            }
        }
        if (rem > 0) {
            uint32_t v = 0;
            for (int j = 0; j < P->C; j++) v |= fit_bits(P, st, i, order[j], 1, p, s, bw);
            return v ? v : OC_V_QUOTA;   /* (v == 0 cannot happen: some g failed k=1) */
        }
    }
    return 0;
}

/* Eq. 2, rate reading R9:
 * y = clamp(max(ceil(sum_a lambda_a * sum_{i in a} c_i / G), ceil(sum_i M(i,s)/F)), 1, C)
 * with M(i,s) = W_i + A_i*s; computed in float64. */
static int32_t eq2_y(const oc_problem *P, const int32_t *beta, const float *lam) {
    double comp = 0.0, mem = 0.0;
    for (int i = 0; i < P->n; i++) {
        comp += (double)lam[P->app[i]] * (double)P->cflop[i];
        mem += (double)P->W[i] + (double)P->Am[i] * (double)P->S[beta[P->app[i]]];
    }
    double y1 = ceil(comp / (double)P->G), y2 = ceil(mem / (double)P->FM);
    double y = y1 > y2 ? y1 : y2;
    if (y < 1.0) y = 1.0;
    if (y > (double)P->C) y = (double)P->C;
    return (int32_t)y;
}

/* ---------------------------------------------------------------- scoring
 * Score one candidate (all checks, no short-cuts).  loads: [L][A] (may be NULL
 * when L == 0).  Returns 0. */
int oc_score(const oc_problem *P, const int32_t *beta, const int32_t *rho, const int32_t *theta,
             const float *loads, int L, oc_score_t *out) {
    memset(out, 0, sizeof(*out));
    for (int k = 0; k < OC_MAX_STAGES * OC_MAX_REPL; k++) out->gpu_of_instance[k] = -1;
    const int n = P->n;
    float dur[OC_MAX_STAGES], thr[OC_MAX_STAGES], bwv[OC_MAX_STAGES];
    int32_t Nn[OC_MAX_STAGES];
    int32_t U = 0;
    for (int i = 0; i < n; i++) {
        const float *e = entry(P, i, beta[P->app[i]], theta[i]);
        dur[i] = e[0];
        thr[i] = e[1];
        bwv[i] = e[2];
        Nn[i] = rho[i] + 1;
        U += Nn[i] * P->Q[theta[i]];
    }
    out->U = U;
    float kmax[OC_MAX_STAGES];
    uint32_t pv = 0;
    static const oc_state zero_state;
    oc_state st = zero_state;
    if (P->flags & OC_PAPER_GLOBAL) {
        /* literal Eq. 1 Constraints 1-4 as global sums (reading R3 flag) */
        int64_t q = 0, ni = 0, mem = 0;
        float bsum = 0.0f;
        for (int i = 0; i < n; i++) {
            int64_t s = P->S[beta[P->app[i]]];
            q += (int64_t)Nn[i] * P->Q[theta[i]];
            ni += Nn[i];
            float t = (float)Nn[i] * bwv[i];
            bsum = bsum + t;
            mem += (int64_t)Nn[i] * ((int64_t)P->W[i] + (int64_t)P->Am[i] * s);
        }
        if (q > (int64_t)P->C * P->R) pv |= OC_V_QUOTA;
        if (ni > (int64_t)P->C * P->I) pv |= OC_V_INST;
        float cap = (float)P->C * P->BW;
        if (!(P->flags & OC_NO_BW_CAP) && bsum > cap) pv |= OC_V_BW;
        if (mem > (int64_t)P->C * (int64_t)P->FM) pv |= OC_V_MEM;
        out->u = 0;
        for (int i = 0; i < n; i++) kmax[i] = 1.0f;
    } else {
        pv = place_all(P, beta, rho, theta, &st);
        int u = 0;
        for (int g = 0; g < P->C; g++) {
            if (st.cnt[g] > 0) u++;
            out->dem[g] = st.dem[g];
        }
        out->u = u;
        /* instance -> GPU map (replica order: by GPU index) */
        for (int i = 0; i < n; i++) {
            int r = 0;
            for (int g = 0; g < P->C; g++)
                for (int k = 0; k < st.host[i][g]; k++) out->gpu_of_instance[i * OC_MAX_REPL + r++] = (int8_t)g;
        }
        /* contention (reading R17): kappa_{i,g} = 1 + gamma_i * (dem_g - bw_i) / BW,
         * x max(1, dem_g/BW) under SAT; worst GPU hosting the stage */
        float invBW = 1.0f / P->BW;
        for (int i = 0; i < n; i++) {
            kmax[i] = 1.0f;
            if (P->flags & OC_NO_CONTENTION) continue;
            for (int g = 0; g < P->C; g++) {
                if (st.host[i][g] == 0) continue;
                float d = st.dem[g] - bwv[i];
                float t = d * invBW;
                float t2 = P->gamma[i] * t;
                float kap = 1.0f + t2;
                if (P->flags & OC_SAT) {
                    float r = st.dem[g] * invBW;
                    if (r > 1.0f) kap = kap * r;
                }
                if (kap > kmax[i]) kmax[i] = kap;
            }
        }
    }
    out->place_viol = pv;
    /* predictions (Table 2: f(p_i) throughput, duration) with contention */
    for (int i = 0; i < n; i++) {
        out->kappa[i] = kmax[i];
        out->L[i] = dur[i] * kmax[i];
        float nt = (float)Nn[i] * thr[i];
        out->Ti[i] = nt / kmax[i];
        out->L64[i] = (double)dur[i] * (double)kmax[i];
        out->T64[i] = (double)Nn[i] * (double)thr[i] / (double)kmax[i];
    }
    /* float64 kappa from float64 demand sums of the same placement */
    if (!(P->flags & OC_PAPER_GLOBAL) && !(P->flags & OC_NO_CONTENTION)) {
        double dem64[OC_MAX_GPUS];
        for (int g = 0; g < P->C; g++) {
            dem64[g] = 0.0;
            for (int i = 0; i < n; i++) dem64[g] += (double)st.host[i][g] * (double)bwv[i];
        }
        for (int i = 0; i < n; i++) {
            double km = 1.0;
            for (int g = 0; g < P->C; g++) {
                if (st.host[i][g] == 0) continue;
                double kap = 1.0 + (double)P->gamma[i] * (dem64[g] - (double)bwv[i]) / (double)P->BW;
                if ((P->flags & OC_SAT) && dem64[g] / (double)P->BW > 1.0) kap *= dem64[g] / (double)P->BW;
                if (kap > km) km = kap;
            }
            out->L64[i] = (double)dur[i] * km;
            out->T64[i] = (double)Nn[i] * (double)thr[i] / km;
        }
    }
    /* NEXT-2, reading R29: the hand-over from stage i to stage i+1 of the same app
     * stays on the GPU (global-memory IPC, ipc_ms) only if both stages run on one
     * and the same GPU (every replica pair co-located; the tail takes the worst
     * pair), otherwise the batch's data crosses GPUs through host memory:
     * fl(fl(comm_mb_i * s) * fl(1 / link_gbs)) ms (MB / (GB/s) = ms). */
    float comm[OC_MAX_STAGES];
    for (int i = 0; i < n; i++) comm[i] = 0.0f;
    if ((P->flags & OC_COMM) && !pv) {
        const float inv_link = 1.0f / P->link_gbs;
        for (int i = 0; i + 1 < n; i++) {
            if (P->app[i] != P->app[i + 1]) continue;
            int gi = -1, same = 1, cnt_gpus = 0;
            for (int g = 0; g < P->C; g++) {
                const int hi = st.host[i][g] > 0, hj = st.host[i + 1][g] > 0;
                if (hi != hj) same = 0;
                if (hi) {
                    cnt_gpus++;
                    gi = g;
                }
            }
            (void)gi;
            const int local = same && cnt_gpus == 1;
            const float s = (float)P->S[beta[P->app[i]]];
            const float bytes = P->comm_mb[i] * s;
            comm[i] = local ? P->ipc_ms : bytes * inv_link;
        }
    }
    for (int i = 0; i < n; i++) out->comm[i] = comm[i];
    /* per app: ordered latency sum vs QoS (Constraint-5, reading R1; with COMM the
     * hand-over times are interleaved: L_f, t_f, L_f+1, t_f+1, ...) and Tmin */
    uint32_t qos_fail = 0;
    float T = 0.0f;
    for (int a = 0; a < P->A; a++) {
        int first = 1;
        float ls = 0.0f, tm = 0.0f;
        double ls64 = 0.0;
        for (int i = 0; i < n; i++) {
            if (P->app[i] != a) continue;
            if (first) {
                ls = out->L[i];
                tm = out->Ti[i];
                first = 0;
            } else {
                if (P->flags & OC_COMM) ls = ls + comm[i - 1];
                ls = ls + out->L[i];
                if (out->Ti[i] < tm) tm = out->Ti[i];
            }
            ls64 += out->L64[i] + (i + 1 < n && P->app[i + 1] == a ? (double)comm[i] : 0.0);
        }
        out->Lsum[a] = ls;
        out->Lsum64[a] = ls64;
        out->Tmin[a] = tm;
        if (ls > P->qos[a]) qos_fail = 1;
        if (a == 0 || tm < T) T = tm;
    }
    out->T = T;
    out->verdict = pv ? pv : (qos_fail ? OC_V_QOS : 0u);
    for (int k = 0; k < L && k < OC_MAX_LOADS; k++) {
        const float *lam = loads + (long)k * P->A;
        int32_t y = eq2_y(P, beta, lam);
        out->eq2_y[k] = y;
        uint32_t v = out->verdict;
        if (v == 0) {
            for (int a = 0; a < P->A; a++)
                if (out->Tmin[a] < lam[a]) v = OC_V_LOAD;
        }
        if (v == 0 && (P->flags & OC_EQ2_BUDGET) && out->u > y) v = OC_V_EQ2;
        out->level_verdict[k] = v;
    }
    return 0;
}

int oc_score_index(const oc_problem *P, uint64_t x, const float *loads, int L, oc_score_t *out) {
    int32_t beta[OC_MAX_APPS], rho[OC_MAX_STAGES], theta[OC_MAX_STAGES];
    oc_decode(P, x, beta, rho, theta);
    return oc_score(P, beta, rho, theta, loads, L, out);
}

/* Verdict/objective vectors over [lo,hi): verdict (max-load), T bits, u, U. */
int oc_score_range(const oc_problem *P, uint64_t lo, uint64_t hi, uint8_t *verdict,
                   float *T, int32_t *u, int32_t *U) {
    oc_score_t sc;
    for (uint64_t x = lo; x < hi; x++) {
        oc_score_index(P, x, NULL, 0, &sc);
        verdict[x - lo] = (uint8_t)sc.verdict;
        T[x - lo] = sc.T;
        u[x - lo] = sc.u;
        U[x - lo] = sc.U;
    }
    return 0;
}

/* ---------------------------------------------------------------- search
 * Plain exhaustive scan in increasing canonical index; keep the best with a
 * STRICT improvement test, so the smallest index wins among ties (R20).
 * policy 0 = max-load (maximise T); 1 = min-resource (minimise (u, U)
 * lexicographically, per load level). */
static void hist_add(uint64_t *h, uint32_t v) {
    for (int b = 0; b < 7; b++)
        if (v & (1u << b)) h[b]++;
}

static void search_range(const oc_problem *P, int policy, const float *loads, int L,
                         uint64_t lo, uint64_t hi, oc_best_t *best) {
    int nb = policy == 0 ? 1 : L;
    for (int k = 0; k < nb; k++) {
        memset(&best[k], 0, sizeof(best[k]));
        best[k].index = UINT64_MAX;
    }
    oc_score_t sc;
    for (uint64_t x = lo; x < hi; x++) {
        oc_score_index(P, x, loads, policy == 0 ? 0 : L, &sc);
        if (policy == 0) {
            best[0].n_scanned++;
            if (sc.verdict) {
                hist_add(best[0].hist, sc.verdict);
                continue;
            }
            best[0].n_feasible++;
            if (best[0].index == UINT64_MAX || sc.T > best[0].T) {
                best[0].index = x;
                best[0].T = sc.T;
                best[0].u = sc.u;
                best[0].U = sc.U;
            }
        } else {
            for (int k = 0; k < L; k++) {
                best[k].n_scanned++;
                uint32_t v = sc.level_verdict[k];
                if (v) {
                    hist_add(best[k].hist, v);
                    continue;
                }
                best[k].n_feasible++;
                int better = best[k].index == UINT64_MAX || sc.u < best[k].u ||
                             (sc.u == best[k].u && sc.U < best[k].U);
                if (better) {
                    best[k].index = x;
                    best[k].T = sc.T;
                    best[k].u = sc.u;
                    best[k].U = sc.U;
                }
            }
        }
    }
}

static int better_than(int policy, const oc_best_t *a, const oc_best_t *b) {
    /* is a strictly better than b (ties -> smaller index) */
    if (a->index == UINT64_MAX) return 0;
    if (b->index == UINT64_MAX) return 1;
    if (policy == 0) {
        if (a->T != b->T) return a->T > b->T;
    } else {
        if (a->u != b->u) return a->u < b->u;
        if (a->U != b->U) return a->U < b->U;
    }
    return a->index < b->index;
}

/* threads > 1: the range is cut into contiguous pieces scanned independently
 * and merged by (objective, index) -- the same result as one scan. */
int oc_search(const oc_problem *P, int policy, const float *loads, int L, uint64_t lo, uint64_t hi,
              int threads, oc_best_t *best) {
    if (oc_validate(P) != 0) return -1;
    if (policy != 0 && (L < 1 || L > OC_MAX_LOADS)) return -1;
    if (policy != 0)
        for (int k = 0; k < L * P->A; k++)
            if (!(loads[k] > 0.0f) || !isfinite(loads[k])) return -1;
    uint64_t nt = oc_ntot(P);
    if (nt == 0) return -2;
    if (hi > nt) hi = nt;
    if (lo > hi) lo = hi;
    int nb = policy == 0 ? 1 : L;
    if (threads < 1) threads = 1;
    if (threads == 1 || hi - lo < (uint64_t)threads * 64) {
        search_range(P, policy, loads, L, lo, hi, best);
        return 0;
    }
    oc_best_t *part = (oc_best_t *)calloc((size_t)threads * nb, sizeof(oc_best_t));
    if (!part) return -3;
    uint64_t len = hi - lo;
#pragma omp parallel for num_threads(threads) schedule(static, 1)
    for (int t = 0; t < threads; t++) {
        uint64_t a = lo + (uint64_t)((unsigned __int128)len * t / threads);
        uint64_t b = lo + (uint64_t)((unsigned __int128)len * (t + 1) / threads);
        search_range(P, policy, loads, L, a, b, part + (size_t)t * nb);
    }
    for (int k = 0; k < nb; k++) {
        oc_best_t acc;
        memset(&acc, 0, sizeof(acc));
        acc.index = UINT64_MAX;
        for (int t = 0; t < threads; t++) {
            const oc_best_t *q = part + (size_t)t * nb + k;
            acc.n_feasible += q->n_feasible;
            acc.n_scanned += q->n_scanned;
            for (int b = 0; b < 7; b++) acc.hist[b] += q->hist[b];
            if (better_than(policy, q, &acc)) {
                acc.index = q->index;
                acc.T = q->T;
                acc.u = q->u;
                acc.U = q->U;
            }
        }
        best[k] = acc;
    }
    free(part);
    return 0;
}

/* ---------------------------------------------------------------- O7: filtered oracle
 * SURVEY.md §8(c) O7 / §8(a) A6.  The same answer as oc_search over the whole
 * space, for spaces too large to scan (full C4), given an INCUMBENT: the
 * objective of a known feasible candidate of the space (max-load: T_inc;
 * min-resource, one load level: (u_inc, U_inc)).  Plain steps:
 *   1. per batch combination and stage i, the option list (rho_i, theta_i) in
 *      canonical order keeps only options that pass every NECESSARY condition of
 *      "feasible and at least as good as the incumbent" (non-strict, so ties
 *      survive), iterated to a fixpoint:
 *        - throughput: T <= T_i <= fl(N_i thr_i) (kappa >= 1, Eq. 1, R12), so
 *          max-load drops fl(N thr) < T_inc and min-resource drops fl(N thr) <
 *          lambda_app (load floor R10);
 *        - QoS (Constraint-5, L834, R1): L_j >= dur_j (kappa >= 1) and the ordered
 *          binary32 sum of non-negative terms is monotone in every term (and only
 *          grows when hand-over terms are inserted), so the ordered sum with this
 *          option's dur at stage i and the smallest surviving dur at the app's
 *          other stages must be <= QoS_a;
 *        - quota (Constraint-2, L831): every GPU holds at most R, so
 *          N p + sum_{j != i} min_j(N p) <= C R;
 *        - min-resource incumbent (L842, R11): U = sum N p exactly and every used
 *          GPU holds at most R, so u >= ceil(U / R) (u = 0 under PAPER_GLOBAL);
 *          with U_lb = N p + sum_{j != i} min_j(N p) and u_lb = ceil(U_lb / R) the
 *          option is dropped iff u_lb > u_inc, or u_lb >= u_inc and U_lb > U_inc;
 *   2. nested loops over the surviving options in canonical order (batch, then
 *      stage 1 .. n), where a prefix whose partial sum N p plus the unplaced
 *      stages' minima already fails the quota or the min-resource test above is
 *      skipped (the same necessary conditions on the partial sum);
 *   3. every remaining candidate is scored by the unchanged oc_score and kept on
 *      STRICT improvement, exactly as oc_search does.
 * Scanning in canonical order with strict improvement returns the smallest
 * index among ties, as oc_search.  The incumbent only ever removes candidates
 * strictly worse than itself, hence strictly worse than the optimum.
 * n_scanned counts the candidates scored; n_feasible those feasible among them. */
typedef struct {
    int32_t cnt[OC_MAX_STAGES];
    int32_t code[OC_MAX_STAGES][OC_MAX_REPL * 128];   /* rho * nQ + theta, ascending */
} oc_optlist;

static int ceil_div(int a, int b) { return (a + b - 1) / b; }

/* step 1 for one batch combination; returns 0 if some stage has no option left */
static int o7_filter(const oc_problem *P, int policy, const float *lam, const int32_t *beta, float T_inc,
                     int32_t u_inc, int32_t U_inc, oc_optlist *ol) {
    const int n = P->n, O = P->Rmax * P->nQ;
    uint8_t alive[OC_MAX_STAGES][OC_MAX_REPL * 128];
    for (int i = 0; i < n; i++)
        for (int k = 0; k < O; k++) alive[i][k] = 1;
    for (int iter = 0;; iter++) {
        float mindur[OC_MAX_STAGES];
        int32_t minnp[OC_MAX_STAGES];
        for (int i = 0; i < n; i++) {
            mindur[i] = INFINITY;
            minnp[i] = INT32_MAX;
            for (int k = 0; k < O; k++) {
                if (!alive[i][k]) continue;
                const int N = k / P->nQ + 1, th = k % P->nQ;
                const float d = entry(P, i, beta[P->app[i]], th)[0];
                if (d < mindur[i]) mindur[i] = d;
                if (N * P->Q[th] < minnp[i]) minnp[i] = N * P->Q[th];
            }
            if (minnp[i] == INT32_MAX) return 0;
        }
        int changed = 0;
        for (int i = 0; i < n; i++) {
            const int a = P->app[i];
            for (int k = 0; k < O; k++) {
                if (!alive[i][k]) continue;
                const int N = k / P->nQ + 1, th = k % P->nQ;
                const float *e = entry(P, i, beta[a], th);
                int drop = 0;
                const float nt = (float)N * e[1];
                if (policy == 0 && nt < T_inc) drop = 1;
                if (policy != 0 && nt < lam[a]) drop = 1;
                /* QoS: ordered sum over the app's stages */
                int first = 1;
                float ls = 0.0f;
                for (int j = 0; j < n; j++) {
                    if (P->app[j] != a) continue;
                    const float t = j == i ? e[0] : mindur[j];
                    ls = first ? t : ls + t;
                    first = 0;
                }
                if (ls > P->qos[a]) drop = 1;
                /* quota and the min-resource incumbent */
                int32_t Ulb = N * P->Q[th];
                for (int j = 0; j < n; j++)
                    if (j != i) Ulb += minnp[j];
                if (Ulb > P->C * P->R) drop = 1;
                if (policy != 0) {
                    const int32_t ulb = (P->flags & OC_PAPER_GLOBAL) ? 0 : ceil_div(Ulb, P->R);
                    if (ulb > u_inc || (ulb >= u_inc && Ulb > U_inc)) drop = 1;
                }
                if (drop) {
                    alive[i][k] = 0;
                    changed = 1;
                }
            }
        }
        if (!changed) break;
    }
    for (int i = 0; i < n; i++) {
        ol->cnt[i] = 0;
        for (int k = 0; k < O; k++)
            if (alive[i][k]) ol->code[i][ol->cnt[i]++] = k;
        if (ol->cnt[i] == 0) return 0;
    }
    return 1;
}

/* steps 2-3: the candidates below a fixed batch combination and stage-1 option */
static int o7_prefix_ok(const oc_problem *P, int policy, int32_t Ulb, int32_t u_inc, int32_t U_inc) {
    if (Ulb > P->C * P->R) return 0;
    if (policy != 0) {
        const int32_t ulb = (P->flags & OC_PAPER_GLOBAL) ? 0 : ceil_div(Ulb, P->R);
        if (ulb > u_inc || (ulb >= u_inc && Ulb > U_inc)) return 0;
    }
    return 1;
}

static void o7_leaf(const oc_problem *P, int policy, const float *lam, const int32_t *beta, const int32_t *rho,
                    const int32_t *theta, oc_best_t *best) {
    oc_score_t sc;
    oc_score(P, beta, rho, theta, lam, policy == 0 ? 0 : 1, &sc);
    best->n_scanned++;
    const uint32_t v = policy == 0 ? sc.verdict : sc.level_verdict[0];
    if (v) {
        hist_add(best->hist, v);
        return;
    }
    best->n_feasible++;
    int better;
    if (policy == 0)
        better = best->index == UINT64_MAX || sc.T > best->T;
    else
        better = best->index == UINT64_MAX || sc.u < best->u || (sc.u == best->u && sc.U < best->U);
    if (better) {
        best->index = oc_encode(P, beta, rho, theta);
        best->T = sc.T;
        best->u = sc.u;
        best->U = sc.U;
    }
}

static void o7_scan(const oc_problem *P, int policy, const float *lam, const int32_t *beta,
                    const oc_optlist *ol, int t0, int32_t u_inc, int32_t U_inc, oc_best_t *best) {
    const int n = P->n;
    int32_t minnp_after[OC_MAX_STAGES + 1];   /* sum of the minimum N p of the stages after i */
    minnp_after[n] = 0;
    for (int i = n - 1; i >= 0; i--) {
        int32_t m = INT32_MAX;
        for (int t = 0; t < ol->cnt[i]; t++) {
            const int k = ol->code[i][t];
            const int32_t np = (k / P->nQ + 1) * P->Q[k % P->nQ];
            if (np < m) m = np;
        }
        minnp_after[i] = minnp_after[i + 1] + m;
    }
    int32_t rho[OC_MAX_STAGES], theta[OC_MAX_STAGES], Upre[OC_MAX_STAGES + 1];
    int pos[OC_MAX_STAGES];
    /* stage 1: the one option of this work item */
    const int k0 = ol->code[0][t0];
    rho[0] = k0 / P->nQ;
    theta[0] = k0 % P->nQ;
    Upre[0] = 0;
    Upre[1] = (rho[0] + 1) * P->Q[theta[0]];
    if (!o7_prefix_ok(P, policy, Upre[1] + minnp_after[1], u_inc, U_inc)) return;
    if (n == 1) {
        o7_leaf(P, policy, lam, beta, rho, theta, best);
        return;
    }
    /* stages 2..n: nested loops (explicit stack), canonical order */
    int depth = 1;
    pos[1] = -1;
    while (depth >= 1) {
        if (++pos[depth] >= ol->cnt[depth]) {
            depth--;
            continue;
        }
        const int k = ol->code[depth][pos[depth]];
        rho[depth] = k / P->nQ;
        theta[depth] = k % P->nQ;
        Upre[depth + 1] = Upre[depth] + (rho[depth] + 1) * P->Q[theta[depth]];
        if (!o7_prefix_ok(P, policy, Upre[depth + 1] + minnp_after[depth + 1], u_inc, U_inc)) continue;
        if (depth + 1 < n) {
            depth++;
            pos[depth] = -1;
            continue;
        }
        o7_leaf(P, policy, lam, beta, rho, theta, best);
    }
}

int oc_search_filtered(const oc_problem *P, int policy, const float *lam, float T_inc, int32_t u_inc,
                       int32_t U_inc, int threads, oc_best_t *best) {
    if (oc_validate(P) != 0) return -1;
    if (P->Rmax * P->nQ > OC_MAX_REPL * 128) return -1;
    if (policy != 0)
        for (int a = 0; a < P->A; a++)
            if (!(lam[a] > 0.0f) || !isfinite(lam[a])) return -1;
    if (oc_ntot(P) == 0) return -2;
    int nb = 1;
    for (int a = 0; a < P->A; a++) nb *= P->nS;
    oc_optlist *ol = (oc_optlist *)malloc(sizeof(oc_optlist) * (size_t)nb);
    int *ok = (int *)malloc(sizeof(int) * (size_t)nb);
    if (!ol || !ok) return -3;
    /* step 1 per batch combination (beta digits, most significant first) */
    int nitems = 0;
    for (int c = 0; c < nb; c++) {
        int32_t beta[OC_MAX_APPS];
        int r = c;
        for (int a = P->A - 1; a >= 0; a--) {
            beta[a] = r % P->nS;
            r /= P->nS;
        }
        ok[c] = o7_filter(P, policy, lam, beta, T_inc, u_inc, U_inc, &ol[c]);
        if (ok[c]) nitems += ol[c].cnt[0];
    }
    /* work items = (batch combination, stage-1 option), in canonical order */
    int *item_c = (int *)malloc(sizeof(int) * (size_t)(nitems + 1));
    int *item_k = (int *)malloc(sizeof(int) * (size_t)(nitems + 1));
    oc_best_t *part = (oc_best_t *)calloc((size_t)(nitems + 1), sizeof(oc_best_t));
    if (!item_c || !item_k || !part) return -3;
    int m = 0;
    for (int c = 0; c < nb; c++)
        if (ok[c])
            for (int t = 0; t < ol[c].cnt[0]; t++) {
                item_c[m] = c;
                item_k[m] = t;
                m++;
            }
    if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
    for (int w = 0; w < nitems; w++) {
        int32_t beta[OC_MAX_APPS];
        int r = item_c[w];
        for (int a = P->A - 1; a >= 0; a--) {
            beta[a] = r % P->nS;
            r /= P->nS;
        }
        memset(&part[w], 0, sizeof(oc_best_t));
        part[w].index = UINT64_MAX;
        o7_scan(P, policy, lam, beta, &ol[item_c[w]], item_k[w], u_inc, U_inc, &part[w]);
    }
    /* merge in canonical order with strict improvement (== one sequential scan) */
    oc_best_t acc;
    memset(&acc, 0, sizeof(acc));
    acc.index = UINT64_MAX;
    for (int w = 0; w < nitems; w++) {
        acc.n_feasible += part[w].n_feasible;
        acc.n_scanned += part[w].n_scanned;
        for (int b = 0; b < 7; b++) acc.hist[b] += part[w].hist[b];
        if (better_than(policy, &part[w], &acc)) {
            acc.index = part[w].index;
            acc.T = part[w].T;
            acc.u = part[w].u;
            acc.U = part[w].U;
        }
    }
    *best = acc;
    free(ol);
    free(ok);
    free(item_c);
    free(item_k);
    free(part);
    return 0;
}

int oc_eq2_y(const oc_problem *P, const int32_t *beta, const float *lam) { return eq2_y(P, beta, lam); }

int oc_sizeof_score(void) { return (int)sizeof(oc_score_t); }
int oc_sizeof_best(void) { return (int)sizeof(oc_best_t); }

/* ---------------------------------------------------------------- simulated annealing
 * The paper's solver: a state V = [n1..nN, p1..pN] (plus the
 * batch digit(s), L858) "randomly moves in one direction"; an invalid new state
 * is rejected; a valid one with a higher objective updates the global optimum;
 * a worse valid state is still accepted with a probability that "decreases with
 * more iterations" (reading R13: p_k = p0 * cool^k, independent of the size of
 * the worsening, exactly as the text states; no temperature-scaled exponent).
 * Counter-based randomness: u64 = splitmix64(splitmix64(seed ^
 * chain*C) + (iter<<2 | purpose)); the CUDA path implements the same generator.
 * Plain, sequential, one chain after the other. */
static uint64_t sm64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t sa_rand(uint64_t seed, uint64_t chain, uint64_t iter, uint64_t purpose) {
    return sm64(sm64(seed ^ (chain * 0xD1B54A32D192ED03ull)) + ((iter << 2) | purpose));
}
static uint32_t sa_uint(uint64_t h, uint32_t m) { return (uint32_t)(((h >> 32) * (uint64_t)m) >> 32); }
static float sa_unif(uint64_t h) { return (float)(h >> 40) * (1.0f / 16777216.0f); }

typedef struct {
    uint64_t best_index;   /* UINT64_MAX: no valid state visited */
    uint32_t best_key;     /* objective key (smaller is better) */
    uint32_t accepted;
    uint64_t final_index;
} oc_sa_chain_t;

/* objective key of a scored candidate for the policy, or 0xFFFFFFFF if invalid */
static uint32_t sa_key(const oc_problem *P, int policy, const oc_score_t *sc) {
    if (policy == 0) {
        if (sc->verdict) return 0xFFFFFFFFu;
        uint32_t bits;
        memcpy(&bits, &sc->T, 4);
        return 0xFFFFFFFFu - bits;
    }
    if (sc->level_verdict[0]) return 0xFFFFFFFFu;
    return ((uint32_t)sc->u << 24) | (uint32_t)sc->U;
}

int oc_sa(const oc_problem *P, int policy, const float *load, uint64_t seed, int chain_lo, int chain_hi,
          int iters, float p0, float cool, oc_sa_chain_t *out) {
    if (oc_validate(P) != 0) return -1;
    const int A = P->A, n = P->n, K = A + 2 * n;
    int radix[OC_MAX_APPS + 2 * OC_MAX_STAGES];
    for (int a = 0; a < A; a++) radix[a] = P->nS;
    for (int i = 0; i < n; i++) {
        radix[A + 2 * i] = P->Rmax;
        radix[A + 2 * i + 1] = P->nQ;
    }
    for (int c = chain_lo; c < chain_hi; c++) {
        int d[OC_MAX_APPS + 2 * OC_MAX_STAGES], e[OC_MAX_APPS + 2 * OC_MAX_STAGES];
        for (int k = 0; k < K; k++) d[k] = (int)sa_uint(sa_rand(seed, (uint64_t)c, (uint64_t)k, 3), (uint32_t)radix[k]);
        oc_score_t sc;
        int32_t beta[OC_MAX_APPS], rho[OC_MAX_STAGES], theta[OC_MAX_STAGES];
        for (int a = 0; a < A; a++) beta[a] = d[a];
        for (int i = 0; i < n; i++) {
            rho[i] = d[A + 2 * i];
            theta[i] = d[A + 2 * i + 1];
        }
        oc_score(P, beta, rho, theta, load, policy == 0 ? 0 : 1, &sc);
        uint32_t kc = sa_key(P, policy, &sc);
        int valid = kc != 0xFFFFFFFFu;
        uint64_t xc = oc_encode(P, beta, rho, theta);
        uint32_t bk = kc;
        uint64_t bx = valid ? xc : UINT64_MAX;
        uint32_t acc = 0;
        float p = p0;
        for (int it = 0; it < iters; it++) {
            int k = (int)sa_uint(sa_rand(seed, (uint64_t)c, (uint64_t)it, 0), (uint32_t)K);
            int dir = (sa_rand(seed, (uint64_t)c, (uint64_t)it, 1) >> 63) ? 1 : -1;
            float u = sa_unif(sa_rand(seed, (uint64_t)c, (uint64_t)it, 2));
            for (int q = 0; q < K; q++) e[q] = d[q];
            if (radix[k] > 1) {
                int nd = d[k] + dir;
                if (nd < 0 || nd >= radix[k]) nd = d[k] - dir;   /* reflect at the grid edge */
                e[k] = nd;
            }
            for (int a = 0; a < A; a++) beta[a] = e[a];
            for (int i = 0; i < n; i++) {
                rho[i] = e[A + 2 * i];
                theta[i] = e[A + 2 * i + 1];
            }
            oc_score(P, beta, rho, theta, load, policy == 0 ? 0 : 1, &sc);
            uint32_t kn = sa_key(P, policy, &sc);
            int vn = kn != 0xFFFFFFFFu;
            uint64_t xn = oc_encode(P, beta, rho, theta);
            /* the global optimum is updated by every valid state with a better objective */
            if (vn && (kn < bk || (kn == bk && xn < bx))) {
                bk = kn;
                bx = xn;
            }
            int accept;
            if (!valid) accept = 1;            /* until the chain reaches a valid state */
            else if (!vn) accept = 0;          /* invalid new states are rejected */
            else if (kn <= kc) accept = 1;     /* not worse */
            else accept = u < p;               /* worse: with decreasing probability */
            if (accept) {
                for (int q = 0; q < K; q++) d[q] = e[q];
                kc = kn;
                valid = vn;
                xc = xn;
                acc++;
            }
            p = p * cool;
        }
        out[c - chain_lo].best_index = bx;
        out[c - chain_lo].best_key = bx == UINT64_MAX ? 0xFFFFFFFFu : bk;
        out[c - chain_lo].accepted = acc;
        out[c - chain_lo].final_index = xc;
    }
    return 0;
}
int oc_sizeof_sa(void) { return (int)sizeof(oc_sa_chain_t); }

/* ---------------------------------------------------------------- NEXT-3
 * The paper's decision-tree performance model: one
 * regression tree per microservice and target (duration, throughput,
 * bandwidth) over the features batch size s and SM quota p.  Node k is a leaf
 * when feature[k] < 0; otherwise x = (feature[k] == 0 ? s : p) goes left when
 * x <= threshold[k].  Plain traversal; NaN for a malformed tree. */
float oc_tree_eval(const int32_t *feature, const int32_t *threshold, const int32_t *left,
                   const int32_t *right, const float *value, int32_t n_nodes, int32_t s, int32_t p) {
    int32_t k = 0;
    for (int32_t step = 0; step <= n_nodes; step++) {
        if (k < 0 || k >= n_nodes) break;
        if (feature[k] < 0) return value[k];
        const int32_t x = feature[k] == 0 ? s : p;
        k = x <= threshold[k] ? left[k] : right[k];
    }
    return NAN;
}

/* ---------------------------------------------------------------- NEXT-4
 * Tail-latency simulation of one plan (reading R32; queries are
 * batched at the entry of an application, then flow through its microservices;
 * L514 / L834: the 99%-ile latency is the QoS metric).  Per application a:
 *   - Poisson arrivals at load lam[a] QPS: gap_q = -log(u_q) * 1000 / lam[a] ms,
 *     u_q = ((h >> 11) + 0.5) * 2^-53, h = sm64(sm64(seed ^ sim * 0xD1B54A32D192ED03)
 *     + (a << 40 | q)) (counter-based: the same stream anywhere);
 *   - every s_a consecutive queries form a batch, released at its last arrival;
 *   - stage i of the app serves batch b on replica b mod N_i, FIFO, for the
 *     plan's contended duration L_i ms; then the hand-over comm_i (COMM) ms;
 *   - latency of a query = completion of its batch at the last stage - arrival.
 * The first `warmup` queries are discarded; p99 = the ceil(0.99 M)-th smallest
 * of the M = n_queries measured latencies; mean = their sum / M (double,
 * in query order).  Times are doubles. */
static int cmp_double(const void *a, const void *b) {
    const double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

int oc_simulate(const oc_problem *P, const int32_t *beta, const int32_t *rho, const int32_t *theta,
                const float *lam, int64_t n_queries, int64_t warmup, uint64_t seed, uint64_t sim,
                double *p99, double *mean) {
    oc_score_t sc;
    oc_score(P, beta, rho, theta, NULL, 0, &sc);
    if (sc.place_viol) return -1;
    if (n_queries < 1 || warmup < 0) return -2;
    double *lat = (double *)malloc(sizeof(double) * (size_t)n_queries);
    if (!lat) return -3;
    for (int a = 0; a < P->A; a++) {
        const int32_t s = P->S[beta[a]];
        int first = -1, last = -1;
        for (int i = 0; i < P->n; i++)
            if (P->app[i] == a) {
                if (first < 0) first = i;
                last = i;
            }
        double freet[OC_MAX_STAGES][OC_MAX_REPL];
        for (int i = 0; i < OC_MAX_STAGES; i++)
            for (int r = 0; r < OC_MAX_REPL; r++) freet[i][r] = 0.0;
        const double scale = 1000.0 / (double)lam[a];
        const uint64_t base = sm64(seed ^ (sim * 0xD1B54A32D192ED03ull));
        const int64_t total = warmup + n_queries;
        const int64_t nbatch = (total + s - 1) / s;
        double t = 0.0, sum = 0.0;
        double arr[OC_MAX_REPL * 8 + 128];   /* arrivals of the current batch (s <= 1024) */
        double *arrv = s <= (int32_t)(sizeof(arr) / sizeof(arr[0])) ? arr : (double *)malloc(sizeof(double) * s);
        int64_t m = 0;
        for (int64_t b = 0; b < nbatch; b++) {
            for (int32_t j = 0; j < s; j++) {
                const uint64_t q = (uint64_t)(b * s + j);
                const uint64_t h = sm64(base + (((uint64_t)a << 40) | q));
                const double u = ((double)(h >> 11) + 0.5) * 0x1.0p-53;
                t = t + (-log(u)) * scale;
                arrv[j] = t;
            }
            double ready = arrv[s - 1];
            for (int i = first; i <= last; i++) {
                const int r = (int)(b % (rho[i] + 1));
                const double start = ready > freet[i][r] ? ready : freet[i][r];
                const double fin = start + (double)sc.L[i];
                freet[i][r] = fin;
                ready = fin;
                if (i < last && (P->flags & OC_COMM)) ready = ready + (double)sc.comm[i];
            }
            for (int32_t j = 0; j < s; j++) {
                const int64_t q = b * s + j;
                if (q < warmup || q >= total) continue;
                const double l = ready - arrv[j];
                lat[m++] = l;
                sum = sum + l;
            }
        }
        if (arrv != arr) free(arrv);
        qsort(lat, (size_t)m, sizeof(double), cmp_double);
        int64_t k = (int64_t)ceil(0.99 * (double)m) - 1;
        if (k < 0) k = 0;
        p99[a] = lat[k];
        mean[a] = sum / (double)m;
    }
    free(lat);
    return 0;
}
