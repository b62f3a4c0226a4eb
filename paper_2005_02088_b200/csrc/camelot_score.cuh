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

__device__ __forceinline__ void score_finish(const DevProb &P, const int *beta, const int *rho, const float *dur,
                                             const float *thr, const float *kmax, const uint32_t *out_hmask,
                                             uint32_t pv, int u, FullScore &out);

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
    score_finish(P, beta, rho, dur, thr, kmax, out_hmask, pv, u, out);
}

// The predictions and verdict of a placed candidate (shared by score_digits and the
// warp-parallel placement of plan_kernel): kmax = contention factor per stage,
// hmask = GPU mask per stage, pv = placement failure bits (0 = placed), u = GPUs used.
__device__ __forceinline__ void score_finish(const DevProb &P, const int *beta, const int *rho, const float *dur,
                                             const float *thr, const float *kmax, const uint32_t *out_hmask,
                                             uint32_t pv, int u, FullScore &out) {
    const int n = P.n;
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

// Warp-parallel placement of ONE candidate (plan_kernel; all 32 lanes of a warp):
// lane g < C owns GPU g.  The same deployment as score_digits (DESIGN.md 3.2,
// PAPER.md L929-945): the order is (remaining MiB, remaining quota, id) ascending
// (rank = number of GPUs with a smaller packed key); pass 1 = the GPU of smallest rank
// that fits all N replicas; pass 2 = greedy k_g = min(c_g, N - (capacity of the GPUs
// before g)), with c_g = canHold(g, N) (fits is monotone in k, and deploying on other
// GPUs does not change g's state).  Writes kmax / hmask / goi / u for score_finish.
// Returns false (uniformly) when a stage does not fit: the caller then scores the
// candidate with score_digits, which also derives the failure bits.
__device__ __forceinline__ bool place_warp(const DevProb &P, const int *rho, const int *pq, const uint32_t *Asv,
                                           const float *bwv, float *kmax, uint32_t *hmask, int8_t *goi, int &u) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, C = P.C, n = P.n;
    const bool own = lane < C;
    int rq = own ? P.R : 0, cnt = 0;
    uint32_t rm = own ? P.FM : 0u;
    float dem = 0.0f;
    int hc[NMAX];
#pragma unroll
    for (int i = 0; i < NMAX; ++i) hc[i] = 0;
#pragma unroll
    for (int i = 0; i < NMAX; ++i) {
        if (i < n) {
            const int p = pq[i], N = rho[i] + 1;   // quota and A_i s (gathered by the caller)
            const uint32_t As = Asv[i], W = P.W[i];
            const float bw = bwv[i];
            auto fits = [&](int k) { return own && fit_viol(P, rq, cnt, rm, dem, k, p, W, As, bw) == 0u; };
            const unsigned long long key =
                own ? (((unsigned long long)rm << 12) | ((unsigned long long)(uint32_t)rq << 4) | (unsigned)lane) : ~0ull;
            int rank = 0;
            for (int h = 0; h < C; ++h) rank += __shfl_sync(FULL, key, h) < key;
            int k = 0;
            const int r1 = __reduce_min_sync(FULL, fits(N) ? rank : 0x7fffffff);
            if (r1 != 0x7fffffff) {
                k = (own && rank == r1) ? N : 0;
            } else {
                int c = 0;
                if (own)
                    for (int kk = N; kk >= 1; --kk)
                        if (fits(kk)) {
                            c = kk;
                            break;
                        }
                int pre = 0, tot = 0;
                for (int h = 0; h < C; ++h) {
                    const int ch = __shfl_sync(FULL, c, h), rh = __shfl_sync(FULL, rank, h);
                    tot += ch;
                    if (rh < rank) pre += ch;
                }
                if (tot < N) return false;
                k = own ? min(c, max(0, N - pre)) : 0;
            }
            if (k > 0) {
                rq -= k * p;
                cnt += k;
                rm -= W + (uint32_t)k * As;
                dem = __fadd_rn(dem, __fmul_rn((float)k, bw));
            }
            hc[i] = k;
        }
    }
    u = __popc(__ballot_sync(FULL, own && cnt > 0));
#pragma unroll
    for (int i = 0; i < NMAX; ++i) {
        if (i < n) {
            hmask[i] = __ballot_sync(FULL, hc[i] > 0);
            float dm = hc[i] > 0 ? dem : 0.0f;   // max demand over the GPUs hosting stage i
            for (int off = 16; off; off >>= 1) dm = fmaxf(dm, __shfl_xor_sync(FULL, dm, off));
            kmax[i] = kappa_of(dm, bwv[i], P.gamma[i], P.invBW, P.flags);
            int pre = hc[i];   // inclusive prefix over GPU index: replicas listed by GPU index
            for (int off = 1; off < 32; off <<= 1) {
                const int v = __shfl_up_sync(FULL, pre, off);
                if (lane >= off) pre += v;
            }
            pre -= hc[i];
            for (int r = 0; r < hc[i]; ++r)
                if (pre + r < SCORE_RMAX) goi[i * SCORE_RMAX + pre + r] = (int8_t)lane;
        }
    }
    return true;
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
