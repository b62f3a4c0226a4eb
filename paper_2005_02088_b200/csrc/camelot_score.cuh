// camelot_score.cuh -- full per-candidate scoring on the device (kernel N5:
// camelot_predict, camelot_score_range, finalize).  One thread scores one
// candidate from scratch: decode -> deployment (readings
// R14-R16) -> contention-aware predictions (R17) -> constraints (Eq. 1 / Eq. 3,
// L825-836, L859-869) -> objective.  Written for clarity: the hot search path
// (camelot_search.cuh) hoists the same arithmetic across candidates.
#pragma once
#include "camelot_device.cuh"

namespace cam {

constexpr int SCORE_CMAX = 16;
constexpr int SCORE_RMAX = 16;

struct FullScore {
    uint32_t verdict;      // first failing check of the max-load policy (0 = feasible)
    uint32_t place_viol;
    float T;               // min over apps of Tmin
    int u, U;
    float Tmin[AMAX], Lsum[AMAX];
    float L[NMAX], Ti[NMAX], kappa[NMAX];
    int8_t goi[NMAX * SCORE_RMAX];
    float comm[NMAX];      // COMM: hand-over time of edge i -> i+1 (ms)
};

__device__ inline void decode_index(const DevProb &P, unsigned long long x, int *beta, int *rho, int *theta) {
    for (int i = P.n - 1; i >= 0; --i) {
        theta[i] = (int)(x % (unsigned)P.nQ);
        x /= (unsigned)P.nQ;
        rho[i] = (int)(x % (unsigned)P.Rmax);
        x /= (unsigned)P.Rmax;
    }
    for (int a = P.A - 1; a >= 0; --a) {
        beta[a] = (int)(x % (unsigned)P.nS);
        x /= (unsigned)P.nS;
    }
}

// can a GPU with (rq, cnt, rm, dem) take k replicas (weights not yet present)?
__device__ __forceinline__ uint32_t fit_viol(const DevProb &P, int rq, int cnt, uint32_t rm, float dem,
                                             int k, int p, uint32_t W, uint32_t As, float bw) {
    uint32_t v = 0;
    if (k * p > rq) v |= V_QUOTA;
    if (cnt + k > P.I) v |= V_INST;
    if (W + (uint32_t)k * As > rm) v |= V_MEM;
    if (!(P.flags & F_NO_BW_CAP)) {
        float tot = __fadd_rn(dem, __fmul_rn((float)k, bw));
        if (tot > P.BW) v |= V_BW;
    }
    return v;
}

// Per-thread scratch of the placement in score_digits; kernels that score few
// candidates on a long serial path (plan_kernel) pass it in shared memory.
struct ScoreScratch {
    int rq[SCORE_CMAX], cnt[SCORE_CMAX], order[SCORE_CMAX];
    uint32_t rm[SCORE_CMAX];
    float dem[SCORE_CMAX];
    uint32_t hmask[NMAX];
    uint8_t hcnt[NMAX][SCORE_CMAX];
};

CAM_DEVFN void score_digits(const DevProb &P, const int *beta, const int *rho, const int *theta,
                             FullScore &out, ScoreScratch *scr = nullptr) {
    const int n = P.n, C = P.C;
    float dur[NMAX], thr[NMAX], bwv[NMAX];
    int U = 0;
    for (int i = 0; i < n; ++i) {
        float4 e = P.tab[((size_t)i * P.nS + beta[P.app[i]]) * P.nQ + theta[i]];
        dur[i] = e.x;
        thr[i] = e.y;
        bwv[i] = e.z;
        U += (rho[i] + 1) * P.Q[theta[i]];
    }
    for (int k = 0; k < NMAX * SCORE_RMAX; ++k) out.goi[k] = -1;
    out.U = U;
    float kmax[NMAX];
    uint32_t out_hmask[NMAX];
    for (int i = 0; i < NMAX; ++i) out_hmask[i] = 0u;
    uint32_t pv = 0;
    int u = 0;
    if (P.flags & F_PAPER_GLOBAL) {
        long long q = 0, ni = 0, mem = 0;
        float bsum = 0.0f;
        for (int i = 0; i < n; ++i) {
            long long s = P.S[beta[P.app[i]]];
            int N = rho[i] + 1;
            q += (long long)N * P.Q[theta[i]];
            ni += N;
            bsum = __fadd_rn(bsum, __fmul_rn((float)N, bwv[i]));
            mem += (long long)N * ((long long)P.W[i] + (long long)P.Am[i] * s);
            kmax[i] = 1.0f;
        }
        if (q > (long long)C * P.R) pv |= V_QUOTA;
        if (ni > (long long)C * P.I) pv |= V_INST;
        if (!(P.flags & F_NO_BW_CAP) && bsum > __fmul_rn((float)C, P.BW)) pv |= V_BW;
        if (mem > (long long)C * (long long)P.FM) pv |= V_MEM;
    } else {
        ScoreScratch loc;
        ScoreScratch &X = scr ? *scr : loc;
        int *rq = X.rq, *cnt = X.cnt;
        uint32_t *rm = X.rm;
        float *dem = X.dem;
        uint32_t *hmask = X.hmask;
        auto &hcnt = X.hcnt;
        for (int g = 0; g < C; ++g) {
            rq[g] = P.R;
            cnt[g] = 0;
            rm[g] = P.FM;
            dem[g] = 0.0f;
        }
        for (int i = 0; i < n && !pv; ++i) {
            hmask[i] = 0;
            for (int g = 0; g < C; ++g) hcnt[i][g] = 0;
            const int p = P.Q[theta[i]];
            const int N = rho[i] + 1;
            const uint32_t As = P.Am[i] * (uint32_t)P.S[beta[P.app[i]]];
            const uint32_t W = P.W[i];
            const float bw = bwv[i];
            // snapshot order: by (remaining MiB, remaining quota, index) ascending
            int *order = X.order;
            for (int g = 0; g < C; ++g) {
                int r = 0;
                for (int h = 0; h < C; ++h) {
                    bool lt = rm[h] < rm[g] || (rm[h] == rm[g] && (rq[h] < rq[g] || (rq[h] == rq[g] && h < g)));
                    r += lt;
                }
                order[r] = g;
            }
            // pass 1: first GPU holding all N replicas
            int gstar = -1;
            for (int j = 0; j < C && gstar < 0; ++j) {
                int g = order[j];
                if (fit_viol(P, rq[g], cnt[g], rm[g], dem[g], N, p, W, As, bw) == 0) gstar = g;
            }
            if (gstar >= 0) {
                rq[gstar] -= N * p;
                cnt[gstar] += N;
                rm[gstar] -= W + (uint32_t)N * As;
                dem[gstar] = __fadd_rn(dem[gstar], __fmul_rn((float)N, bw));
                hcnt[i][gstar] = (uint8_t)N;
                hmask[i] = 1u << gstar;
                continue;
            }
            // pass 2: greedy fill in the same order with min(canHold, remaining)
            int rem = N;
            for (int j = 0; j < C && rem > 0; ++j) {
                int g = order[j];
                int k = rem;
                while (k > 0 && fit_viol(P, rq[g], cnt[g], rm[g], dem[g], k, p, W, As, bw) != 0) --k;
                if (k > 0) {
                    rq[g] -= k * p;
                    cnt[g] += k;
                    rm[g] -= W + (uint32_t)k * As;
                    dem[g] = __fadd_rn(dem[g], __fmul_rn((float)k, bw));
                    hcnt[i][g] = (uint8_t)k;
                    hmask[i] |= 1u << g;
                    rem -= k;
                }
            }
            if (rem > 0) {
                // first-failing dimensions AFTER pass 2 (DESIGN.md 3.2 step 5): fits(g, 1)
                // on the updated state, weights charged only where stage i is not yet hosted
                uint32_t v = 0;
                for (int g = 0; g < C; ++g)
                    v |= fit_viol(P, rq[g], cnt[g], rm[g], dem[g], 1, p, hcnt[i][g] ? 0u : W, As, bw);
                pv = v ? v : V_QUOTA;
            }
        }
        if (!pv) {
            for (int g = 0; g < C; ++g) u += cnt[g] > 0;
            for (int i = 0; i < n; ++i) {
                int r = 0;
                for (int g = 0; g < C; ++g)
                    for (int k = 0; k < hcnt[i][g]; ++k) out.goi[i * SCORE_RMAX + r++] = (int8_t)g;
                float dm = 0.0f;
                for (int g = 0; g < C; ++g)
                    if (hmask[i] >> g & 1u) dm = fmaxf(dm, dem[g]);
                kmax[i] = kappa_of(dm, bwv[i], P.gamma[i], P.invBW, P.flags);
                out_hmask[i] = hmask[i];
            }
        } else {
            for (int i = 0; i < n; ++i) kmax[i] = 1.0f;
        }
    }
    out.u = u;
    out.place_viol = pv;
    for (int i = 0; i < n; ++i) {
        out.kappa[i] = kmax[i];
        out.L[i] = __fmul_rn(dur[i], kmax[i]);
        out.Ti[i] = __fdiv_rn(__fmul_rn((float)(rho[i] + 1), thr[i]), kmax[i]);
    }
    // COMM (R29): hand-over of edge i -> i+1 = ipc when both stages run entirely on
    // one and the same GPU, else the host-staged copy of the batch's data
    for (int i = 0; i < NMAX; ++i) out.comm[i] = 0.0f;
    if ((P.flags & F_COMM) && !pv && !(P.flags & F_PAPER_GLOBAL)) {
        for (int i = 0; i + 1 < n; ++i) {
            if (P.app[i] != P.app[i + 1]) continue;
            const bool local = out_hmask[i] == out_hmask[i + 1] && __popc(out_hmask[i]) == 1;
            out.comm[i] = local ? P.ipc_ms
                                : __fmul_rn(__fmul_rn(P.comm_mb[i], (float)P.S[beta[P.app[i]]]), P.inv_link);
        }
    }
    bool qos_fail = false;
    float T = 0.0f;
    for (int a = 0; a < P.A; ++a) {
        float ls = 0.0f, tm = 0.0f;
        for (int i = P.first_of_app[a]; i <= P.last_of_app[a]; ++i) {
            if (i == P.first_of_app[a]) {
                ls = out.L[i];
                tm = out.Ti[i];
            } else {
                if (P.flags & F_COMM) ls = __fadd_rn(ls, out.comm[i - 1]);
                ls = __fadd_rn(ls, out.L[i]);
                tm = fminf(tm, out.Ti[i]);
            }
        }
        out.Lsum[a] = ls;
        out.Tmin[a] = tm;
        if (ls > P.qos[a]) qos_fail = true;
        T = (a == 0) ? tm : fminf(T, tm);
    }
    out.T = T;
    out.verdict = pv ? pv : (qos_fail ? V_QOS : 0u);
}

// level verdict for min-resource load level (lam: [A]); y = Eq. 2 estimate
__device__ __forceinline__ uint32_t level_verdict(const DevProb &P, const FullScore &s, const float *lam, int y) {
    uint32_t v = s.verdict;
    if (v) return v;
    for (int a = 0; a < P.A; ++a)
        if (s.Tmin[a] < lam[a]) return V_LOAD;
    if ((P.flags & F_EQ2_BUDGET) && s.u > y) return V_EQ2;
    return 0;
}

// Eq. 2, rate reading R9, float64.
__device__ inline int eq2_gpus(const DevProb &P, const int *beta, const float *lam) {
    double comp = 0.0, mem = 0.0;
    for (int i = 0; i < P.n; ++i) {
        comp += (double)lam[P.app[i]] * (double)P.cflop[i];
        mem += (double)P.W[i] + (double)P.Am[i] * (double)P.S[beta[P.app[i]]];
    }
    double y1 = ceil(comp / (double)P.G), y2 = ceil(mem / (double)P.FM);
    double y = fmax(y1, y2);
    y = fmin(fmax(y, 1.0), (double)P.C);
    return (int)y;
}

}  // namespace cam
