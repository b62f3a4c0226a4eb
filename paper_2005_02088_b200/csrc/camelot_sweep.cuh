// camelot_sweep.cuh -- the exhaustive (NO_FILTER) scan as an issue-bound
// "leaf sweep" kernel for sm_100a.
//
// The flat scan scores EVERY candidate of [lo, hi) (the
// state V = [N_1..N_n, p_1..p_n] plus the batch, L858) with the scoring of
// DESIGN.md 3 (placement L929-945, contention R17, Constraint-5 L834).  Unlike
// the pruned tree search it has no data-dependent work, so it is laid out for
// instruction issue:
//   * a warp owns one GRANDPARENT (batch combo + options of stages 0..n-3,
//     warp-uniform state placed once) and 32 of its PARENTS (option of stage
//     n-2): lane = parent, placed by the lane in registers;
//   * each lane then sweeps ALL leaves (options (N, theta) of the last stage)
//     of its parent: per quota theta the per-GPU capacities
//     c_g = canHold(g, Rmax) are computed once and packed as a thermometer
//     code in deployment order (4 bits per GPU), so for every replica count N
//     pass 1 of the deployment heuristic is one shift+ffs and pass 2's greedy
//     prefix is one popc; the code is built per quota from the
//     capacities' quota BREAKPOINTS, packed bytes (one subtract per 4 GPUs);
//   * contention: only the GPU(s) receiving the leaf's replicas change demand,
//     so every placed stage's max demand is updated by a bit test + max;
//   * every lane keeps its own best (objective key, index); one reduction at
//     the end.  No shared-memory stacks, no warp synchronisation in the loop.
// State is indexed by GPU id (no permutation): the deployment order
// (remaining MiB, remaining quota, id) only enters through the rank shifts.
#pragma once
#include "camelot_device.cuh"
#include "camelot_sweep_args.h"

namespace cam {

constexpr int SWEEP_THREADS = 256;
#ifndef SWEEP_MINB
#define SWEEP_MINB 2
#endif

// SweepArgs: camelot_sweep_args.h

// Thread-level placement state indexed by GPU id.
template <int CM, int NS>
struct SwState {
    int rq[CM], cnt[CM];
    uint32_t rm[CM];
    float dem[CM];
    uint32_t hm[NS];     // GPU mask of stage i
    float dm[NS];        // max demand over the GPUs hosting stage i
    int u, U;
};

template <int CM, int NS>
__device__ __forceinline__ void sw_init(const DevProb &P, SwState<CM, NS> &s) {
#pragma unroll
    for (int g = 0; g < CM; ++g) {
        s.rq[g] = g < P.C ? P.R : 0;
        s.cnt[g] = 0;
        s.rm[g] = g < P.C ? P.FM : 0u;
        s.dem[g] = 0.0f;
    }
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        s.hm[i] = 0u;
        s.dm[i] = 0.0f;
    }
    s.u = 0;
    s.U = 0;
}

// Deploy stage i with N replicas of quota p:
// pass 1 = the first GPU in (rm, rq, id) order that holds all N, pass 2 = greedy
// min(canHold, remaining) in the same order.  Returns false if it does not fit.
// Division-free: floor(rq / p) = (rq * pmul) >> 16 with pmul = ceil(2^16 / p) (rq <= 127),
// and the memory capacity counts k = 1..N with W + k As <= rm (N <= 4 in the sweep).
// The deployment order packs (rm, rq, id) into 32 bits (rm < 2^21, rq < 2^7, id < 2^4).
template <int CM, int NS>
__device__ __forceinline__ bool sw_place(const DevProb &P, SwState<CM, NS> &s, int i, int N, int p, uint32_t pmul,
                                         uint32_t W, uint32_t As, float bw) {
    const bool cap = !(P.flags & F_NO_BW_CAP);
    int c[CM];
    uint32_t key[CM];
#pragma unroll
    for (int g = 0; g < CM; ++g) {
        int k = 0;
        if (g < P.C) {
            k = min(N, (int)(((uint32_t)s.rq[g] * pmul) >> 16));
            k = min(k, P.I - s.cnt[g]);
            int km = 0;   // memory: k' <= k with W + k' As <= rm
#pragma unroll
            for (int t = 1; t <= 4; ++t) km += (t <= k) & (W + (uint32_t)t * As <= s.rm[g]);
            k = km;
            if (cap)
                while (k > 0 && __fadd_rn(s.dem[g], __fmul_rn((float)k, bw)) > P.BW) --k;
        }
        c[g] = k;
        key[g] = (s.rm[g] << 11) | ((uint32_t)s.rq[g] << 4) | (uint32_t)g;
    }
    int gs = -1;
    uint32_t best = 0xffffffffu;
#pragma unroll
    for (int g = 0; g < CM; ++g)
        if (c[g] == N && key[g] < best) {
            best = key[g];
            gs = g;
        }
    int kk[CM];
    uint32_t hmask = 0u;
    if (gs >= 0) {
#pragma unroll
        for (int g = 0; g < CM; ++g) kk[g] = g == gs ? N : 0;
    } else {
        int tot = 0;
#pragma unroll
        for (int g = 0; g < CM; ++g) tot += c[g];
        if (tot < N) return false;
#pragma unroll
        for (int g = 0; g < CM; ++g) {
            int pre = 0;   // capacity of the GPUs before g in deployment order
#pragma unroll
            for (int h = 0; h < CM; ++h) pre += (key[h] < key[g]) ? c[h] : 0;
            kk[g] = min(c[g], max(0, N - pre));
        }
    }
#pragma unroll
    for (int g = 0; g < CM; ++g) {
        const int k = kk[g];
        if (k > 0) {
            s.u += s.cnt[g] == 0;
            s.rq[g] -= k * p;
            s.cnt[g] += k;
            s.rm[g] -= W + (uint32_t)k * As;
            s.dem[g] = __fadd_rn(s.dem[g], __fmul_rn((float)k, bw));
            hmask |= 1u << g;
        }
    }
#pragma unroll
    for (int i2 = 0; i2 < NS; ++i2)
        if (i2 == i) s.hm[i2] = hmask;   // stage i is new (i may be a runtime value: no local array)
    // max demand over the hosting GPUs of every placed stage (demand only grows)
#pragma unroll
    for (int i2 = 0; i2 < NS; ++i2) {
        if (i2 <= i) {
            float m = 0.0f;
#pragma unroll
            for (int g = 0; g < CM; ++g)
                if ((s.hm[i2] >> g) & 1u) m = fmaxf(m, s.dem[g]);
            s.dm[i2] = m;
        }
    }
    s.U += N * p;
    return true;
}

// kappa of DESIGN.md 3.3 without SAT (the sweep is not used with SAT); with
// NO_CONTENTION the caller passes gamma = 0, and fl(1 + 0) = 1 exactly.
__device__ __forceinline__ float sw_kappa(float dmax, float bw, float gamma, float invBW) {
    return __fadd_rn(1.0f, __fmul_rn(gamma, __fmul_rn(__fsub_rn(dmax, bw), invBW)));
}

// cold paths of the leaf loop, out of line (instruction-cache footprint)
// First-failing dimensions of a failed deployment of the leaf stage (DESIGN.md 3.2
// step 5): the OR over GPUs of the dimensions in which fits(g, 1) fails AFTER pass 2.
// A failed pass 2 leaves every GPU at its capacity c_g (the popcount of its nibble of
// the thermometer code M, in deployment order; `perm` maps a rank to the GPU id), and
// on that state fits(g, 1) fails exactly in the integer dimensions where fits(g, c_g+1)
// fails on the parent state (the leaf stage is new on every GPU, so its weights are
// charged once), and in bandwidth iff fl(fl(dem + fl(c_g bw)) + bw) > BW.  The same
// for every failing N: pass 2 fills every GPU to capacity.  The parent state is read
// from the per-thread shared-memory copies (rq | cnt << 8, rm, dem).
static __device__ __noinline__ uint32_t sw_fail_bits(const DevProb &P, int p, float bw, uint32_t need1, uint32_t As,
                                              bool cap, uint32_t M, uint32_t perm, const uint32_t *rqc,
                                              const uint32_t *rmv, const float *demv, int stride) {
    uint32_t v = 0;
    for (int r = 0; r < P.C; ++r) {
        const int g = (perm >> (4 * r)) & 0xF;
        const int c = __popc((M >> (4 * r)) & 0xFu);
        const uint32_t w = rqc[g * stride];
        const int rq = (int)(w & 0xFFu), cnt = (int)(w >> 8);
        const float dem = demv[g * stride];
        const int k = c + 1;
        if (k * p > rq) v |= V_QUOTA;
        if (cnt + k > P.I) v |= V_INST;
        if (need1 + (uint32_t)c * As > rmv[g * stride]) v |= V_MEM;
        if (cap && __fadd_rn(__fadd_rn(dem, __fmul_rn((float)c, bw)), bw) > P.BW) v |= V_BW;
    }
    return v ? v : V_QUOTA;
}

// Largest float h with fl(dem + h) <= BW: fl(dem + y) is monotone in y, so
// fl(dem + fl(k bw)) <= BW  <=>  fl(k bw) <= h  (exact).
__device__ __forceinline__ float bw_threshold(float dem, float BW) {
    // start at fl(BW - dem) and step by one ulp (integer steps on the bit pattern of
    // the non-negative / negative float) until the largest admissible value is found
    auto up = [](float v) {   // next float towards +inf
        const uint32_t b = __float_as_uint(v);
        if (b == 0x80000000u) return __uint_as_float(1u);                 // -0 -> +min subnormal
        return __uint_as_float((b >> 31) ? b - 1u : b + 1u);
    };
    auto down = [](float v) {   // next float towards -inf
        const uint32_t b = __float_as_uint(v);
        if (b == 0u) return __uint_as_float(0x80000001u);                 // +0 -> -min subnormal
        return __uint_as_float((b >> 31) ? b + 1u : b - 1u);
    };
    float h = __fsub_rn(BW, dem);
    while (__fadd_rn(dem, h) > BW) h = down(h);
    while (true) {
        const float h2 = up(h);
        if (!(__fadd_rn(dem, h2) <= BW) || isinf(h2)) break;
        h = h2;
    }
    return __fadd_rn(h, 0.0f);   // -0 -> +0 (the sign-bit test of the sweep needs +0)
}

// fits in bandwidth of k replicas of one-replica demand bw under the threshold h of
// bw_threshold: fl(k bw) <= h  <=>  fl(h - fl(k bw)) has a clear sign bit (exact: RN
// keeps the sign and gradual underflow never rounds a non-zero difference to 0)
__device__ __forceinline__ bool bw_fits(float h, float kbw) { return !(__float_as_uint(__fsub_rn(h, kbw)) >> 31); }

// First sub-grid index ts in [0, hi) at which k replicas no longer fit in bandwidth
// (hi if they fit everywhere).  Valid when the row's bw is non-decreasing along the
// sub-grid (then fl(k bw(ts)) is non-decreasing and the fitting ts form a prefix).
__device__ __forceinline__ int bw_break(const float4 *row, int nQ, int qs, int nQs, int k, float h, int hi) {
    auto kbw = [&](int ts) {
        const float bw = row[nQ - 1 - qs * (nQs - 1 - ts)].z;
        return k == 1 ? bw : __fmul_rn((float)k, bw);
    };
    if (hi <= 0 || bw_fits(h, kbw(hi - 1))) return hi;
    int lo = 0, up = hi - 1;   // the answer is in [lo, up]: ts = up fails
    while (lo < up) {
        const int mid = (lo + up) >> 1;
        if (bw_fits(h, kbw(mid))) lo = mid + 1;
        else up = mid;
    }
    return lo;
}

// The thermometer code M of one quota (see the leaf loop) straight from the definition:
// c_g = min(instance+memory capacity, floor(rq/p), #{k in 1..4 : fl(dem + fl(k bw)) <= BW})
// per GPU, c_g ones in the nibble of the GPU's rank.  Out of line: only leaf rows whose
// bandwidth is not non-decreasing in the quota take it (never for the generated tables).
static __device__ __noinline__ uint32_t sw_therm_slow(const DevProb &P, int Rmax, uint32_t WL, uint32_t AsL, int p, float bw,
                                                   bool cap, uint32_t perm, const uint32_t *rqc, const uint32_t *rmv,
                                                   const float *demv, int stride) {
    uint32_t M = 0u;
    for (int r = 0; r < P.C; ++r) {
        const int g = (perm >> (4 * r)) & 0xF;
        const uint32_t w = rqc[g * stride];
        const int rq = (int)(w & 0xFFu), cnt = (int)(w >> 8);
        const float dem = demv[g * stride];
        int c = min(Rmax, P.I - cnt);
        int km = 0;
        for (int t = 1; t <= 4; ++t) km += (t <= c) & (WL + (uint32_t)t * AsL <= rmv[g * stride]);
        c = min(km, rq / p);
        if (cap) {
            int kb = 0;
            for (int t = 1; t <= 4; ++t) kb += __fadd_rn(dem, __fmul_rn((float)t, bw)) <= P.BW;
            c = min(c, kb);
        }
        M += ((1u << c) - 1u) << (4 * r);
    }
    return M;
}

__device__ __forceinline__ void sw_better(unsigned long long key, unsigned long long x, unsigned long long &bk,
                                          unsigned long long &bx) {
    if (key < bk || (key == bk && x < bx)) {
        bk = key;
        bx = x;
    }
}

// The sweep.  NS == n exactly (stage loops carry no runtime guards) unless n > 6.
template <int CM, int NS, int POLICY, bool TWO, bool COMM>
__global__ void __launch_bounds__(SWEEP_THREADS, SWEEP_MINB) sweep_kernel(const DevProb P, const SweepArgs A) {
    static_assert(CM <= 8, "thermometer code holds 8 GPUs x 4 bits");
    __shared__ float dem_s[CM][SWEEP_THREADS];
    __shared__ uint32_t rqc_s[CM][SWEEP_THREADS], rm_s[CM][SWEEP_THREADS];   // cold: failure bits
    __shared__ uint32_t qpm_s[CAMELOT_MAX_QUOTAS];   // p | ceil(2^16/p) << 7
    __shared__ unsigned char qcnt_s[128];            // #{sub-grid ts : p(ts) <= v}, v < 128
    __shared__ unsigned char mono_s[CAMELOT_MAX_BATCHES];   // leaf row of batch b: bw >= 0, non-decreasing
    __shared__ unsigned long long red_k[SWEEP_THREADS / 32], red_x[SWEEP_THREADS / 32];
    __shared__ unsigned long long red_c[SWEEP_THREADS / 32][2];
    __shared__ unsigned red_v[SWEEP_THREADS / 32];
    __shared__ int is_last;
    // per warp: the grandparent's placement state, shared by the chunks of a work item
    struct GSave {
        SwState<CM, NS> st;
        float dur[NS], bwv[NS], ntv[NS];
    };
    __shared__ GSave gsave[SWEEP_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // NS == n for n <= 6 (the host dispatches exact widths), so stage guards fold away
    const int n = NS <= 6 ? NS : P.n;
    const int nQ = P.nQ, O = P.O, Rmax = P.Rmax;
    // quota sub-grid (incumbent cascade): sub index t -> canonical theta; Os options per stage
    const int nQs = A.nQs, qs = A.qstride, Os = Rmax * nQs;
    auto canon = [&](int os) { return (os / nQs) * nQ + (nQ - 1 - qs * (nQs - 1 - os % nQs)); };
    const int jl = n - 1;                     // leaf stage
    const bool cont = !(P.flags & F_NO_CONTENTION);
    const bool cap = !(P.flags & F_NO_BW_CAP);
    // the leaf stage's predictor rows of every batch (nS x nQ float4, contiguous in the
    // [n][nS][nQ] table) -> shared memory with the TMA engine (one bulk copy per CTA)
    extern __shared__ __align__(16) float4 tabL_s[];
    __shared__ unsigned long long tbar;
    const bool staged = A.tabL_bytes > 0;
    if (staged && tid == 0) {
        mbar_init(&tbar, 1);
        fence_proxy_async();
        mbar_arrive_expect_tx(&tbar, A.tabL_bytes);
        bulk_g2s(tabL_s, P.tab + (size_t)jl * P.nS * nQ, A.tabL_bytes, &tbar);
    }
    for (int t = tid; t < nQ; t += blockDim.x) {
        const uint32_t p = (uint32_t)P.Q[t];
        qpm_s[t] = p | (((65536u + p - 1u) / p) << 7);
    }
    for (int v = tid; v < 128; v += blockDim.x) {
        int c = 0;
        for (int ts = 0; ts < nQs; ++ts) c += P.Q[nQ - 1 - qs * (nQs - 1 - ts)] <= v;
        qcnt_s[v] = (unsigned char)c;
    }
    __syncthreads();   // (also publishes the initialised barrier)
    if (staged) mbar_wait(&tbar, 0);
    const float4 *tabLall = staged ? tabL_s : P.tab + (size_t)jl * P.nS * nQ;
    for (int b = tid; b < P.nS; b += blockDim.x) {
        const float4 *row = tabLall + (size_t)b * nQ;
        float prev = 0.0f;
        bool m = true;
        for (int ts = 0; ts < nQs; ++ts) {
            const float z = row[nQ - 1 - qs * (nQs - 1 - ts)].z;
            m = m && z >= prev;   // (false for NaN)
            prev = z;
        }
        mono_s[b] = m;
    }
    __syncthreads();
    unsigned long long bk = A.inc[0].key, bx = A.inc[0].x;
    unsigned long long n_sc = 0, n_fe = 0;
    unsigned viol = 0;
    while (true) {
        unsigned long long it = 0;
        if (lane == 0) it = atomicAdd(&A.hdr->chunk_counter, 1ull);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= A.n_items) break;
        // work item: one grandparent x 32 parents, or (small sub-grids, Os <= 16) gpack
        // grandparents x Os parents, lane = (grandparent, parent) pair
        const int gpk = A.gpack;
        const int lg = gpk == 1 ? 0 : lane / Os;   // this lane's grandparent in the item
        bool lane_ok = true;
        unsigned long long gp;
        int c_begin = 0, c_end = 1;   // this item's parent chunks (32 parents each)
        if (gpk == 1 && it < A.n_grp_items) {
            const unsigned ng = (unsigned)A.ngroups;
            gp = A.g_lo + it / ng;
            const int grp = (int)(it % ng);
            c_begin = grp * A.nchunk / A.ngroups;
            c_end = (grp + 1) * A.nchunk / A.ngroups;
        } else if (gpk == 1) {   // the tail: one chunk per item
            const unsigned long long j = it - A.n_grp_items;
            gp = A.g_lo + A.gp_split + j / (unsigned)A.nchunk;
            c_begin = (int)(j % (unsigned)A.nchunk);
            c_end = c_begin + 1;
        } else {
            const unsigned long long g0 = it * (unsigned long long)gpk + (unsigned long long)lg;
            lane_ok = lg < gpk && g0 < A.n_gp;
            gp = A.g_lo + (lane_ok ? g0 : 0ull);
        }
        // bound: the best objective key found anywhere so far (a feasible candidate), so a
        // leaf whose key bound is strictly worse cannot win (skips only the divisions)
        unsigned long long gkey = 0;
        if (lane == 0) gkey = *(volatile unsigned int *)&A.hdr->best_obj;
        gkey = min(__shfl_sync(0xffffffffu, gkey, 0), bk);
        // ---- grandparent (warp-uniform unless gpack > 1): batch combo + options of stages 0..n-3
        int beta[AMAX];
        int o[NS];
        {
            unsigned long long t = gp;
#pragma unroll
            for (int k = NS - 1; k >= 0; --k)
                if (k < n - 2) {
                    o[k] = canon((int)(t % (unsigned)Os));
                    t /= (unsigned)Os;
                }
            int bc = (int)t;
            beta[0] = beta[1] = 0;
            if (P.A > 1) {
                beta[1] = bc % P.nS;
                bc /= P.nS;
            }
            beta[0] = bc;
        }
        SwState<CM, NS> st;
        float dur[NS], bwv[NS], ntv[NS];
        bool gok = lane_ok;   // the grandparent's stages fit (uniform when gpack == 1)
        for (int ch = c_begin; ch < c_end; ++ch) {
        // ---- parent (per lane): option of stage n-2, its canonical index and range
        const int ops = gpk == 1 ? ch * 32 + lane : lane % Os;   // parent option in the (sub-)grid
        const int op = canon(min(ops, Os - 1));      // canonical option code
        unsigned long long gpc = 0;                  // canonical grandparent index
        {
            const int bc = P.A > 1 ? beta[0] * P.nS + beta[1] : beta[0];
            gpc = (unsigned long long)bc;
#pragma unroll
            for (int k = 0; k < NS; ++k)
                if (k < n - 2) gpc = gpc * (unsigned long long)O + (unsigned long long)o[k];
        }
        const unsigned long long xp = gpc * (unsigned long long)O + (unsigned long long)op;   // parent index
        const unsigned long long xpO = xp * (unsigned long long)O;
        int clo = 0, chi = O;
        if (A.lo > xpO) clo = (int)min(A.lo - xpO, (unsigned long long)O);
        if (A.hi < xpO + O) chi = A.hi > xpO ? (int)(A.hi - xpO) : 0;
        bool act = lane_ok && ops < Os && clo < chi;
        if (act && A.world > 1) {
            const unsigned long long item = xp / P.opow[n - 1 - A.d0];
            act = ((item / 64ull) % (unsigned long long)A.world) == (unsigned long long)A.rank;
        }
        // ---- placement of stages 0..n-2: the grandparent's options (warp-uniform unless
        // gpack > 1; placed once per work item, saved in shared memory for its further
        // chunks), then the lane's parent option.  A rolled loop (one copy of sw_place):
        // this code runs once per chunk, and unrolled it thrashed the instruction cache.
        int i0 = 0;
        if (ch > c_begin) {
            __syncwarp();   // lane 0's save is visible
            st = gsave[wid].st;
#pragma unroll
            for (int i = 0; i < NS; ++i) {
                dur[i] = gsave[wid].dur[i];
                bwv[i] = gsave[wid].bwv[i];
                ntv[i] = gsave[wid].ntv[i];
            }
            i0 = n - 2;
        } else {
            sw_init<CM, NS>(P, st);
#pragma unroll
            for (int i = 0; i < NS; ++i) dur[i] = bwv[i] = ntv[i] = 0.0f;
        }
#pragma unroll 1
        for (int i = i0; i <= n - 2; ++i) {
            if (i == n - 2) {
                if (gpk == 1 && ch == c_begin && c_end - c_begin > 1 && gok && lane == 0) {
                    gsave[wid].st = st;
#pragma unroll
                    for (int k = 0; k < NS; ++k) {
                        gsave[wid].dur[k] = dur[k];
                        gsave[wid].bwv[k] = bwv[k];
                        gsave[wid].ntv[k] = ntv[k];
                    }
                }
                act = act && gok;
                if (!act) break;
            } else if (!gok) {
                break;
            }
            int oi = op;
#pragma unroll
            for (int k = 0; k < NS; ++k)
                if (k == i && k < n - 2) oi = o[k];
            const int b = P.app[i] ? beta[1] : beta[0];
            const int th = oi % nQ, N = oi / nQ + 1;
            const float4 e = __ldg(&P.tab[((size_t)i * P.nS + b) * nQ + th]);
            const uint32_t As = P.Am[i] * (uint32_t)P.S[b];
            const bool ok = sw_place<CM, NS>(P, st, i, N, (int)(qpm_s[th] & 127u), qpm_s[th] >> 7, P.W[i], As, e.z);
            if (i < n - 2) gok = ok;
            else act = ok;
            const float nt = __fmul_rn((float)N, e.y);
#pragma unroll
            for (int k = 0; k < NS; ++k)
                if (k == i) {
                    dur[k] = e.x;
                    bwv[k] = e.z;
                    ntv[k] = nt;
                }
        }
        if (gpk == 1 && !gok) break;   // the grandparent does not fit: no chunk of it has work (uniform)
        if (act) {
        // ---- leaf context: capacities, deployment order, bounds (per lane)
        const int bL = P.app[jl] ? beta[1] : beta[0];
        const uint32_t WL = P.W[jl], AsL = P.Am[jl] * (uint32_t)P.S[bL];
        const float gL = cont ? P.gamma[jl] : 0.0f;
        // COMM (R29): hand-over times of the edges between placed stages (exact), and the
        // cross-GPU time of the edge into the leaf stage (local or not is decided per leaf)
        float te[NS];
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            te[i] = 0.0f;
            if (COMM && i + 1 < n && P.app[i] == P.app[i + 1]) {
                const float tx = __fmul_rn(__fmul_rn(P.comm_mb[i], (float)P.S[P.app[i] ? beta[1] : beta[0]]), P.inv_link);
                te[i] = (i + 1 < jl && st.hm[i] == st.hm[i + 1] && __popc(st.hm[i]) == 1) ? P.ipc_ms : tx;
            }
        }
        const float4 *tabL = tabLall + (size_t)bL * nQ;
        const bool mono = nQs >= A.bp_min_nqs && mono_s[bL];
        // Capacities as BREAKPOINTS in the quota: over the sub-grid
        // ts = 0..nQs-1 the quota p(ts) increases and (mono rows) so does bw(ts), so
        // c_g(ts) >= k  <=>  ts < brk[g][k] with brk[g][k] = the first ts where k replicas
        // no longer fit (0 if k exceeds the instance+memory capacity).  The breakpoints
        // are packed as bytes b | 0x80 (b <= 127): rank r's k-th breakpoint is byte r >> 1
        // of wE[k-1] (even r) or wO[k-1] (odd r), so that per quota one subtraction of
        // (ts + 1) per byte sets bit 7 exactly where c >= k, in rank order.
        uint32_t wE[4], wO[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) wE[k] = wO[k] = 0x80808080u;
        uint32_t perm = 0u, E = 0u;
#pragma unroll
        for (int g = 0; g < CM; ++g) {
            int r = g;
            if (g < P.C) {   // rank in the (rm, rq, id) order: packed 32-bit keys (see sw_place)
                r = 0;
                const uint32_t kg = (st.rm[g] << 11) | ((uint32_t)st.rq[g] << 4) | (uint32_t)g;
#pragma unroll
                for (int h = 0; h < CM; ++h)
                    if (h < P.C) r += ((st.rm[h] << 11) | ((uint32_t)st.rq[h] << 4) | (uint32_t)h) < kg;
                if (st.cnt[g] == 0) E |= 1u << g;
            }
            perm |= (uint32_t)g << (4 * r);
            dem_s[g][tid] = st.dem[g];
            rqc_s[g][tid] = (uint32_t)st.rq[g] | ((uint32_t)st.cnt[g] << 8);
            rm_s[g][tid] = st.rm[g];
        }
        // the breakpoints, rank by rank (rolled; the GPU's state from its shared-memory copy)
        if (mono) {
#pragma unroll 1
            for (int r = 0; r < P.C; ++r) {
                const int g = (perm >> (4 * r)) & 0xF;
                const uint32_t w = rqc_s[g][tid], rm = rm_s[g][tid];
                const int rq = (int)(w & 0xFFu), kc = min(Rmax, P.I - (int)(w >> 8));
                const float hb = cap ? bw_threshold(dem_s[g][tid], P.BW) : __int_as_float(0x7f800000);
                int prev = nQs;
                uint32_t bytes = 0u;   // byte k-1 = the k-th breakpoint (non-increasing in k)
#pragma unroll 1
                for (int k = 1; k <= 4 && prev > 0; ++k) {
                    int b = 0;
                    // instance + memory: k <= cap, WL + k AsL <= rm
                    if (k <= kc && WL + (uint32_t)k * AsL <= rm) {
                        const int ql = k == 1 ? rq : k == 2 ? rq >> 1 : k == 3 ? (rq * 43691) >> 17 : rq >> 2;
                        b = min((int)qcnt_s[ql], prev);   // quota: p(ts) <= floor(rq / k)
                        if (cap) b = bw_break(tabL, nQ, qs, nQs, k, hb, b);
                    }
                    prev = b;
                    bytes |= (uint32_t)b << (8 * (k - 1));
                }
                const int sh = 8 * (r >> 1);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t v = ((bytes >> (8 * k)) & 0xFFu) << sh;
                    if (r & 1) wO[k] |= v;
                    else wE[k] |= v;
                }
            }
        }
        float ptub = __int_as_float(0x7f800000);
#pragma unroll
        for (int i = 0; i < NS; ++i)
            if (i < jl) {
                const float k = sw_kappa(st.dm[i], bwv[i], cont ? P.gamma[i] : 0.0f, P.invBW);
                ptub = fminf(ptub, k == 1.0f ? ntv[i] : __fdiv_rn(ntv[i], k));
            }
        const float qos0 = P.qos[0], qos1 = TWO ? P.qos[1] : 0.0f;
        const int f1 = TWO ? P.first_of_app[1] : n;   // first stage of application 2
        float gam[NS];
#pragma unroll
        for (int i = 0; i < NS; ++i) gam[i] = (cont && i < n) ? P.gamma[i] : 0.0f;
        int ybud = 0x7fffffff;
        float lam0 = 0.0f, lam1 = 0.0f;
        if (POLICY == 1) {
            lam0 = A.lam[0];
            lam1 = TWO ? A.lam[1] : 0.0f;
            if (P.flags & F_EQ2_BUDGET) {
                const int bc = P.A > 1 ? beta[0] * P.nS + beta[1] : beta[0];
                ybud = A.y[bc * A.ystride + A.yoff];
            }
        }
        const unsigned span = (unsigned)(chi - clo);
        const bool full = span == (unsigned)O;
        unsigned c_sc = 0, c_fe = 0;
        // ---- the leaves: quota theta outer (capacities once), replicas N inner.
        // Kept compact (rolled N loop, no per-GPU branches): the hot loop must stay
        // within the ~6 KB L0 instruction cache.
        uint32_t t1 = 0u;   // (ts + 1) in every byte
        for (int ts = 0; ts < nQs; ++ts) {
            const int th = nQ - 1 - qs * (nQs - 1 - ts);
            const float4 e = tabL[th];
            const uint32_t qp = qpm_s[th];
            const float bw = e.z;
            // thermometer code of c_g = canHold(g, Rmax): c_g ones in the nibble of the GPU's
            // rank (4 bits per GPU in deployment order).  Byte b | 0x80 minus (ts + 1) keeps
            // bit 7 iff b > ts (no borrow between bytes: b, ts + 1 <= 127), i.e. iff c >= k;
            // that bit moves to position 4 r + k - 1.
            t1 += 0x01010101u;
            uint32_t M = 0u;
            if (mono) {
#pragma unroll
                for (int k = 1; k <= 4; ++k)
                    M |= (((wE[k - 1] - t1) >> (8 - k)) & (0x80808080u >> (8 - k))) |
                         (((wO[k - 1] - t1) >> (4 - k)) & (0x80808080u >> (4 - k)));
            } else {
                M = sw_therm_slow(P, Rmax, WL, AsL, (int)(qp & 127u), bw, cap, perm, &rqc_s[0][tid], &rm_s[0][tid],
                                  &dem_s[0][tid], SWEEP_THREADS);
            }
            // deployment succeeds iff the total capacity holds N (pass 1 or pass 2)
            const int sumc = __popc(M);
            const int nok = min(sumc, Rmax);
            if (full) {
                c_sc += Rmax;
            } else {
                for (int N = 1; N <= Rmax; ++N) c_sc += (unsigned)((N - 1) * nQ + th - clo) < span;
            }
            // the failing leaves: first-failing dimensions (OR over GPUs, k = 1).  Only an
            // INFEASIBLE result reports them, so they are skipped once a feasible candidate
            // is known (the lane's best, the incumbent or the device-wide best)
            if (nok < Rmax && bk >= 0xFFFFFFFFull && gkey >= 0xFFFFFFFFull) {
                bool any = full;
                for (int N = nok + 1; N <= Rmax && !any; ++N) any = (unsigned)((N - 1) * nQ + th - clo) < span;
                if (any)
                    viol |= sw_fail_bits(P, (int)(qp & 127u), bw, WL + AsL, AsL, cap, M, perm, &rqc_s[0][tid],
                                         &rm_s[0][tid], &dem_s[0][tid], SWEEP_THREADS);
            }
#pragma unroll 1
            for (int N = 1; N <= nok; ++N) {
                const int code = (N - 1) * nQ + th;
                if (!full && (unsigned)(code - clo) >= span) continue;
                // receiving GPUs in deployment order: pass 1 = the first with c >= N (k = N);
                // pass 2 = greedy k = min(c, remaining) over those with c >= 1
                const uint32_t mN = (M >> (N - 1)) & 0x11111111u;
                float dmx[NS];
#pragma unroll
                for (int i = 0; i < NS; ++i) dmx[i] = st.dm[i];
                float dl = 0.0f;
                int du = 0;
                uint32_t lm = 0u;   // GPUs receiving the leaf stage (COMM)
                uint32_t mm = mN ? (mN & (0u - mN)) : (M & 0x11111111u);
                int rem = N;
                do {
                    const int r = __ffs(mm) - 1;
                    mm &= mm - 1u;
                    const int k = min(rem, __popc((M >> r) & 15u));
                    rem -= k;
                    const int g = (perm >> r) & 15u;
                    const float d = __fadd_rn(dem_s[g][tid], __fmul_rn((float)k, bw));
                    dl = fmaxf(dl, d);
                    du += (E >> g) & 1u;
                    if (COMM) lm |= 1u << g;
#pragma unroll
                    for (int i = 0; i < NS; ++i)
                        if (i < jl && ((st.hm[i] >> g) & 1u)) dmx[i] = fmaxf(dmx[i], d);
                } while (rem > 0);
                // contention-aware latencies and the per-application ordered sums (Constraint-5)
                float kap[NS];
                float l0 = 0.0f, l1 = 0.0f;
#pragma unroll
                for (int i = 0; i < NS; ++i) {
                    if (i < n) {
                        if (COMM && i > 0 && P.app[i - 1] == P.app[i]) {   // hand-over before stage i
                            const float t = (i == jl) ? ((st.hm[jl - 1] == lm && __popc(lm) == 1) ? P.ipc_ms : te[jl - 1])
                                                      : te[i - 1];
                            if (!TWO || i < f1) l0 = __fadd_rn(l0, t);
                            else l1 = __fadd_rn(l1, t);
                        }
                        const float k = (i == jl) ? sw_kappa(dl, bw, gL, P.invBW)
                                                  : sw_kappa(dmx[i], bwv[i], gam[i], P.invBW);
                        kap[i] = k;
                        const float L = __fmul_rn(i == jl ? e.x : dur[i], k);
                        if (!TWO || i < f1) l0 = (i == 0) ? L : __fadd_rn(l0, L);
                        else l1 = (i == f1) ? L : __fadd_rn(l1, L);
                    }
                }
                if (!(l0 <= qos0 && (!TWO || l1 <= qos1))) {
                    viol |= V_QOS;
                    continue;
                }
                ++c_fe;
                const unsigned long long x = xpO + (unsigned long long)code;
                const float ntl = __fmul_rn((float)N, e.y);
                if (POLICY == 0) {
                    // T <= min(parent bound, fl(N thr)): the divisions only when it can win
                    const unsigned long long kub = objkey_maxload(fminf(ptub, ntl));
                    if (kub <= gkey && (kub < bk || (kub == bk && x < bx))) {
                        float T = __int_as_float(0x7f800000);
#pragma unroll
                        for (int i = 0; i < NS; ++i)
                            if (i < n) {
                                const float nt = i == jl ? ntl : ntv[i];
                                T = fminf(T, kap[i] == 1.0f ? nt : __fdiv_rn(nt, kap[i]));
                            }
                        sw_better(objkey_maxload(T), x, bk, bx);
                    }
                } else {
                    const int u2 = st.u + du;
                    const unsigned long long key = objkey_minres(u2, st.U + N * (int)(qp & 127u));
                    if (key <= gkey && (key < bk || (key == bk && x < bx)) && u2 <= ybud) {
                        float t0 = __int_as_float(0x7f800000), t1 = __int_as_float(0x7f800000);
#pragma unroll
                        for (int i = 0; i < NS; ++i)
                            if (i < n) {
                                const float nt = i == jl ? ntl : ntv[i];
                                const float ti = kap[i] == 1.0f ? nt : __fdiv_rn(nt, kap[i]);
                                if (!TWO || i < f1) t0 = fminf(t0, ti);
                                else t1 = fminf(t1, ti);
                            }
                        if (t0 >= lam0 && (!TWO || t1 >= lam1)) sw_better(key, x, bk, bx);
                    }
                }
            }
        }
        n_sc += c_sc;
        n_fe += c_fe;
        if (bk < gkey) {
            atomicMin(&A.hdr->best_obj, (unsigned int)bk);
            gkey = bk;
        }
        }   // act
        }   // chunks of the item
    }
    // ---- reduction: lane -> warp -> CTA slot; the last CTA reduces the slots
    for (int off = 16; off; off >>= 1) {
        const unsigned long long ok2 = __shfl_xor_sync(0xffffffffu, bk, off);
        const unsigned long long ox = __shfl_xor_sync(0xffffffffu, bx, off);
        sw_better(ok2, ox, bk, bx);
        n_sc += __shfl_xor_sync(0xffffffffu, n_sc, off);
        n_fe += __shfl_xor_sync(0xffffffffu, n_fe, off);
        viol |= __shfl_xor_sync(0xffffffffu, viol, off);
    }
    if (lane == 0) {
        red_k[wid] = bk;
        red_x[wid] = bx;
        red_c[wid][0] = n_sc;
        red_c[wid][1] = n_fe;
        red_v[wid] = viol;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long k2 = red_k[0], x2 = red_x[0], sc = 0, fe = 0;
        unsigned vi = 0;
        for (int w = 0; w < SWEEP_THREADS / 32; ++w) {
            sw_better(red_k[w], red_x[w], k2, x2);
            sc += red_c[w][0];
            fe += red_c[w][1];
            vi |= red_v[w];
        }
        A.slots[blockIdx.x].key = k2;
        A.slots[blockIdx.x].x = x2;
        if (sc) {
            atomicAdd(&A.hdr->n_scored, sc);
            atomicAdd(&A.hdr->cum_scored, sc);
        }
        if (fe) atomicAdd(&A.hdr->n_feasible, fe);
        if (vi) atomicOr(&A.hdr->viol_or, vi);
        __threadfence();
        is_last = atomicAdd(&A.hdr->done_ctas, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    unsigned long long k2 = ~0ull, x2 = ~0ull;
    for (int s = tid; s < (int)gridDim.x; s += blockDim.x) {
        const unsigned long long vk = *(volatile unsigned long long *)&A.slots[s].key;
        const unsigned long long vx = *(volatile unsigned long long *)&A.slots[s].x;
        sw_better(vk, vx, k2, x2);
    }
    for (int off = 16; off; off >>= 1) {
        const unsigned long long ok2 = __shfl_xor_sync(0xffffffffu, k2, off);
        const unsigned long long ox = __shfl_xor_sync(0xffffffffu, x2, off);
        sw_better(ok2, ox, k2, x2);
    }
    if (lane == 0) {
        red_k[wid] = k2;
        red_x[wid] = x2;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < SWEEP_THREADS / 32; ++w) sw_better(red_k[w], red_x[w], k2, x2);
        if (k2 >= 0xFFFFFFFFull) {
            k2 = 0xFFFFFFFFull;
            x2 = ~0ull;
        }
        A.result[0].key = k2;
        A.result[0].x = x2;
        trace_value(A.hdr, 202, k2);   // the sweep's optimum in the phase trace
        trace_value(A.hdr, 203, x2);
        unsigned long long packed = ~0ull;
        if (k2 != 0xFFFFFFFFull) {
            // chunk id = 64 depth-d0 items (NO_FILTER: item = x / O^(n-d0)), as the tree search
            const unsigned long long low = P.ntot <= (1ull << 32) ? x2 : (x2 / P.opow[n - A.d0]) / 64ull;
            packed = (k2 << 32) | (low & 0xFFFFFFFFull);
        }
        A.keys[0] = (long long)(packed ^ 0x8000000000000000ull);
        A.hdr->done_ctas = 0;
    }
}

}  // namespace cam
