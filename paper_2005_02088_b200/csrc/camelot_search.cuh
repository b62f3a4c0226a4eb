// camelot_search.cuh -- the exact, pruned, warp-cooperative allocation search
// (kernels N1 search, N3 option filter) for sm_100a.
//
// Search order.  The candidate space is the tree  beta-combo -> stage 1 option
// -> ... -> stage n option  (option = (N_i, p_i); batch
// L858).  The top d0 stage levels are flattened into "items" that lanes
// evaluate independently; below, a warp walks the tree depth-first: at each
// node all 32 lanes evaluate 32 children (the next stage's options) in
// parallel against the node's placement state (held once in shared memory),
// ballot the survivors and descend into them in order.  Leaves (the last
// stage) are scored exactly and reduced into the warp's best (objective key,
// canonical index).
//
// Pruning.  A child is dropped only if every
// candidate below it is infeasible or strictly worse than a candidate already
// known to be feasible (the incumbent / best so far): placement failure of the
// placed prefix; QoS lower bound (contention only grows as stages are added,
// so the ordered fp32 latency sum of the current latencies plus the minimum
// durations of the unplaced stages is a lower bound); throughput upper bound
// (T_i <= fl(N_i thr_i)); quota left; min-resource key lower bound.  Ties are
// never pruned, so the smallest index among optimal candidates survives.
#pragma once
#include "camelot_device.cuh"

namespace cam {

constexpr int SEARCH_THREADS = 256;
constexpr int SEARCH_WARPS = SEARCH_THREADS / 32;

struct SearchArgs {
    int policy;                 // 0 max-load, 1 min-resource
    int nlev;                   // number of best slots (1 for max-load)
    int d0;                     // stage levels flattened into items (1 <= d0 <= n-1)
    int chunk_items;            // items per chunk (work unit, key low bits when Ntot > 2^32)
    int rank, world;
    int prune;                  // 0 = flat scan (bounds off)
    unsigned long long lo, hi;  // canonical index range
    const OptRec *rec;          // [n][nS][O] compacted surviving options (ascending code)
    const StageBound *sb;       // [n][nS]
    const unsigned long long *item_off;  // [nbc + 1]
    const float *lam;           // [nlev][A] load levels (min-resource)
    const int *y;               // [nbc][ystride] Eq. 2 estimates (min-resource), level k at yoff + k
    int ystride, yoff;
    const Slot *inc;            // [nlev] incumbent (key, x); key 0xFFFFFFFF.. = none
    DevHeader *hdr;
    Slot *slots;                // [gridDim.x][nlev]
    unsigned long long chunk_lo, chunk_hi;  // owned chunks restricted to [lo, hi) (rescan); hi = 0: all
    // level-synchronous pass: expand parents at depth `level` (stages 0..level-1
    // placed); children at depth `flevel` go to the output frontier (-1: none)
    int level, flevel, grab;
    const void *in_nodes;       // Node<CM>[in_cap] (nullptr: parents are the roots, one per batch combo)
    const unsigned long long *in_count;
    unsigned long long in_cap;
    void *out_nodes;            // Node<CM>[out_cap]
    unsigned long long *out_tail;
    unsigned long long out_cap;
    unsigned long long *head;   // pop counter of this pass
};

// Placement state after the first j stages, in shared memory (one per DFS
// level per warp).  GPU arrays are indexed by GPU id (g*) and by position in
// the deployment order for the NEXT stage (p*: sorted by remaining memory,
// remaining quota, index -- PAPER.md L929-942).
template <int CM>
struct Node {
    int grq[CM], gcnt[CM];
    uint32_t grm[CM];
    float gdem[CM];
    int prq[CM], pkim[CM], pgid[CM];
    float pdem[CM];
    float dur[NMAX], bw[NMAX], nt[NMAX], dmax[NMAX];
    uint32_t hmask[NMAX];
    int kidx[NMAX];         // position of each placed stage's option in its compacted list
    unsigned long long x;   // canonical prefix value
    int U, u, rqsum, bc;
    int b[AMAX];
    float tub;              // min fl(N thr) over placed stages
};

// per-warp DFS bookkeeping (shared memory)
struct WarpCtl {
    int cur[NMAX];
    int base[NMAX];
    unsigned msk[NMAX];
};

// ---------------------------------------------------------------- placement of one stage
// Places option r of the stage being placed onto node nd (positions in order).
// Returns k (replicas) per position in kpos[] and whether it succeeded.
// fits(pos,k): k*p <= rq, k <= kim (instances and memory), fl(dem + fl(k bw)) <= BW.
template <int CM>
__device__ __forceinline__ bool place_stage(const DevProb &P, const Node<CM> &nd, const OptRec &r, int (&kpos)[CM]) {
    const bool cap = !(P.flags & F_NO_BW_CAP);
    const int N = (int)r.N;
    int jstar = -1;
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        kpos[q] = 0;
        if (q < P.C && jstar < 0) {
            bool f = (int)r.NP <= nd.prq[q] && N <= nd.pkim[q];
            if (f && cap) f = __fadd_rn(nd.pdem[q], r.NB) <= P.BW;
            if (f) jstar = q;
        }
    }
    if (jstar >= 0) {
#pragma unroll
        for (int q = 0; q < CM; ++q)
            if (q == jstar) kpos[q] = N;
        return true;
    }
    // pass 2: greedy fill in order, k = min(canHold, remaining)
    int rem = N;
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        if (q < P.C && rem > 0) {
            int kq = (int)(((uint32_t)nd.prq[q] * r.pmul) >> 16);   // floor(rq / p)
            int k = min(min(rem, kq), nd.pkim[q]);
            if (cap)
                while (k > 0 && __fadd_rn(nd.pdem[q], __fmul_rn((float)k, r.bw)) > P.BW) --k;
            kpos[q] = k > 0 ? k : 0;
            rem -= kpos[q];
        }
    }
    return rem == 0;
}

// first-failing placement dimensions of a failed stage (OR over GPUs of fits(g,1) failures)
template <int CM>
__device__ __forceinline__ uint32_t place_fail_bits(const DevProb &P, const Node<CM> &nd, const OptRec &r) {
    uint32_t v = 0;
    for (int q = 0; q < P.C; ++q) {
        if ((int)r.p > nd.prq[q]) v |= V_QUOTA;
        int g = nd.pgid[q];
        if (nd.gcnt[g] + 1 > P.I) v |= V_INST;
        if (r.W + r.As > nd.grm[g]) v |= V_MEM;
        if (!(P.flags & F_NO_BW_CAP) && __fadd_rn(nd.pdem[q], r.bw) > P.BW) v |= V_BW;
    }
    return v ? v : V_QUOTA;
}

__device__ __forceinline__ const OptRec &opt_at(const DevProb &P, const SearchArgs &S, int i, int b, int k) {
    return S.rec[((size_t)i * P.nS + b) * P.O + k];
}
__device__ __forceinline__ const StageBound &sb_at(const DevProb &P, const SearchArgs &S, int i, int b) {
    return S.sb[(size_t)i * P.nS + b];
}

// Child evaluation of stage j (option r) on node nd, by one lane.
// Computes everything needed for (a) the bound test of an inner node, or (b)
// the exact leaf score.  Returns false if the placement fails.
struct ChildEval {
    bool placed;
    float lsum[AMAX];     // exact (leaf) or lower bound (inner)
    float kap[NMAX];      // contention factors of placed stages 0..j
    int u, U;
    unsigned long long x;
};

template <int CM>
__device__ __forceinline__ void eval_child(const DevProb &P, const SearchArgs &S, const Node<CM> &nd, int j,
                                           const OptRec &r, ChildEval &ce) {
    int kpos[CM];
    ce.placed = place_stage<CM>(P, nd, r, kpos);
    ce.x = nd.x * (unsigned long long)P.O + r.code;
    ce.U = nd.U + (int)r.NP;
    if (!ce.placed) return;
    // demand after this stage on the GPUs it uses; update max demand of hosts
    float dm[NMAX];
#pragma unroll
    for (int i = 0; i < NMAX; ++i) dm[i] = (i < j) ? nd.dmax[i] : 0.0f;
    float dself = 0.0f;
    int unew = 0;
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        if (kpos[q] > 0) {
            float d = __fadd_rn(nd.pdem[q], __fmul_rn((float)kpos[q], r.bw));
            dself = fmaxf(dself, d);
            int g = nd.pgid[q];
            unew += nd.gcnt[g] == 0;
#pragma unroll
            for (int i = 0; i < NMAX; ++i)
                if (i < j && ((nd.hmask[i] >> g) & 1u)) dm[i] = fmaxf(dm[i], d);
        }
    }
    ce.u = nd.u + unew;
    // contention factors and ordered latency sums (lower bound for unplaced stages)
#pragma unroll
    for (int a = 0; a < AMAX; ++a) ce.lsum[a] = 0.0f;
    const int b0 = nd.b[0], b1 = nd.b[AMAX - 1];
#pragma unroll
    for (int i = 0; i < NMAX; ++i) {
        if (i >= P.n) break;
        float L;
        if (i < j) {
            float k = kappa_of(dm[i], nd.bw[i], P.gamma[i], P.invBW, P.flags);
            ce.kap[i] = k;
            L = __fmul_rn(nd.dur[i], k);
        } else if (i == j) {
            float k = kappa_of(dself, r.bw, P.gamma[i], P.invBW, P.flags);
            ce.kap[i] = k;
            L = __fmul_rn(r.dur, k);
        } else {
            L = sb_at(P, S, i, P.app[i] == 0 ? b0 : b1).mindur;
        }
        int a = P.app[i];
        if (i == P.first_of_app[a]) ce.lsum[a] = L;
        else ce.lsum[a] = __fadd_rn(ce.lsum[a], L);
    }
}

// ---------------------------------------------------------------- node construction
// Build the child node (stage j placed with option r) into out.  Executed by the
// whole warp with identical inputs (uniform); lanes share the work per GPU.
template <int CM>
__device__ void build_child(const DevProb &P, const SearchArgs &S, const Node<CM> &nd, int j, const OptRec &r,
                            int kopt, Node<CM> &out, int lane) {
    int kpos[CM];
    place_stage<CM>(P, nd, r, kpos);   // succeeded when we get here
    // per-GPU update: lane q (a position) owns GPU pgid[q]
    int k = 0;
#pragma unroll
    for (int q = 0; q < CM; ++q)
        if (q == lane) k = kpos[q];
    int g = lane < P.C ? nd.pgid[lane] : 0;
    int rq = 0, cnt = 0;
    uint32_t rm = 0;
    float dem = 0.0f;
    if (lane < P.C) {
        rq = nd.grq[g] - k * (int)r.p;
        cnt = nd.gcnt[g] + k;
        rm = nd.grm[g] - (k > 0 ? r.W + (uint32_t)k * r.As : 0u);
        dem = k > 0 ? __fadd_rn(nd.gdem[g], __fmul_rn((float)k, r.bw)) : nd.gdem[g];
    }
    unsigned used = __ballot_sync(0xffffffffu, lane < P.C && k > 0);
    // host mask of the new stage (GPU ids)
    unsigned hm = 0;
    for (unsigned m = used; m; m &= m - 1) {
        int q = __ffs(m) - 1;
        hm |= 1u << __shfl_sync(0xffffffffu, g, q);
    }
    // max demand per stage after the update: lane i (< j+1) handles stage i
    float dmi = 0.0f;
    if (lane < j) dmi = nd.dmax[lane];
    for (unsigned m = used; m; m &= m - 1) {
        int q = __ffs(m) - 1;
        float dq = __shfl_sync(0xffffffffu, dem, q);
        int gq = __shfl_sync(0xffffffffu, g, q);
        if (lane < j && ((nd.hmask[lane] >> gq) & 1u)) dmi = fmaxf(dmi, dq);
        if (lane == j) dmi = fmaxf(dmi, dq);
    }
    // order for the next stage: rank of (rm, rq, g) among the C GPUs
    int rank = 0;
    for (int h = 0; h < P.C; ++h) {
        uint32_t rmh = __shfl_sync(0xffffffffu, rm, h);
        int rqh = __shfl_sync(0xffffffffu, rq, h);
        int gh = __shfl_sync(0xffffffffu, g, h);
        bool lt = rmh < rm || (rmh == rm && (rqh < rq || (rqh == rq && gh < g)));
        rank += (lane < P.C && h != lane && lt) ? 1 : 0;
    }
    // instance + memory capacity for the next stage (uniform stage j+1)
    int kim = 0;
    if (j + 1 < P.n && lane < P.C) {
        const int i2 = j + 1;
        const int b2 = nd.b[P.app[i2]];
        const uint32_t W2 = P.W[i2], As2 = P.Am[i2] * (uint32_t)P.S[b2];
        int km = P.Rmax;
        if (rm < W2) km = 0;
        else if (As2 > 0) km = (int)min((uint32_t)P.Rmax, (rm - W2) / As2);
        kim = min(km, min(P.Rmax, P.I - cnt));
        kim = max(kim, 0);
    }
    __syncwarp();
    if (lane < P.C) {
        out.grq[g] = rq;
        out.gcnt[g] = cnt;
        out.grm[g] = rm;
        out.gdem[g] = dem;
        out.prq[rank] = rq;
        out.pkim[rank] = kim;
        out.pgid[rank] = g;
        out.pdem[rank] = dem;
    }
    if (lane < j) {
        out.dur[lane] = nd.dur[lane];
        out.bw[lane] = nd.bw[lane];
        out.nt[lane] = nd.nt[lane];
        out.hmask[lane] = nd.hmask[lane];
        out.kidx[lane] = nd.kidx[lane];
    }
    if (lane <= j) out.dmax[lane] = dmi;
    unsigned unew = __popc(__ballot_sync(0xffffffffu, lane < P.C && k > 0 && nd.gcnt[g] == 0));
    if (lane == 0) {
        out.dur[j] = r.dur;
        out.bw[j] = r.bw;
        out.nt[j] = r.NT;
        out.hmask[j] = hm;
        out.kidx[j] = kopt;
        out.x = nd.x * (unsigned long long)P.O + r.code;
        out.U = nd.U + (int)r.NP;
        out.u = nd.u + (int)unew;
        out.rqsum = nd.rqsum - (int)r.NP;
        out.bc = nd.bc;
        out.b[0] = nd.b[0];
        out.b[AMAX - 1] = nd.b[AMAX - 1];
        out.tub = fminf(nd.tub, r.NT);
    }
    __syncwarp();
}

// root node for beta combo bc (no stage placed), built by the warp
template <int CM>
__device__ void build_root(const DevProb &P, int bc, Node<CM> &out, int lane) {
    int b[AMAX];
    {
        int t = bc;
        for (int a = P.A - 1; a >= 0; --a) {
            b[a] = t % P.nS;
            t /= P.nS;
        }
        if (P.A == 1) b[AMAX - 1] = b[0];
    }
    __syncwarp();
    if (lane < P.C) {
        const int g = lane;
        out.grq[g] = P.R;
        out.gcnt[g] = 0;
        out.grm[g] = P.FM;
        out.gdem[g] = 0.0f;
        // all GPUs equal: order = index
        const uint32_t W0 = P.W[0], As0 = P.Am[0] * (uint32_t)P.S[b[P.app[0]]];
        int km = P.Rmax;
        if (P.FM < W0) km = 0;
        else if (As0 > 0) km = (int)min((uint32_t)P.Rmax, (P.FM - W0) / As0);
        out.prq[g] = P.R;
        out.pkim[g] = max(0, min(km, min(P.Rmax, P.I)));
        out.pgid[g] = g;
        out.pdem[g] = 0.0f;
    }
    if (lane == 0) {
        out.x = (unsigned long long)bc;
        out.U = 0;
        out.u = 0;
        out.rqsum = P.C * P.R;
        out.bc = bc;
        out.b[0] = b[0];
        out.b[AMAX - 1] = b[AMAX - 1];
        out.tub = __int_as_float(0x7f800000);   // +inf
    }
    __syncwarp();
}

// ---------------------------------------------------------------- bounds
struct WarpBest {
    unsigned long long key[LMAX];   // objective key (32 bits used), smaller is better
    unsigned long long x[LMAX];
    unsigned long long bound;       // pruning bound: max over levels of key (conservative)
};

// key lower bound of any completion of a child at stage j (inner node)
template <int CM>
__device__ __forceinline__ unsigned int child_keylb(const DevProb &P, const SearchArgs &S, const Node<CM> &nd, int j,
                                                    const OptRec &r, const ChildEval &ce, float restT, int restU) {
    if (S.policy == 0) {
        float tub = fminf(fminf(nd.tub, r.NT), restT);
        return objkey_maxload(tub);
    }
    int Ulb = ce.U + restU;
    int ulb = max(ce.u, (Ulb + P.R - 1) / P.R);
    return objkey_minres(ulb, Ulb);
}

// inner-node survival test for child (stage j, option r) of nd; exact bounds only
template <int CM>
__device__ __forceinline__ bool inner_survives(const DevProb &P, const SearchArgs &S, const Node<CM> &nd, int j,
                                               const OptRec &r, const ChildEval &ce, unsigned long long bound) {
    if (!ce.placed) return false;
    const int n = P.n;
    const unsigned long long span = P.opow[n - 1 - j];
    const unsigned long long xs = ce.x * span;
    if (xs >= S.hi || xs + span <= S.lo) return false;
    if (!S.prune) return true;
    bool ok = true;
    for (int a = 0; a < P.A; ++a) ok &= ce.lsum[a] <= P.qos[a];
    float restT = __int_as_float(0x7f800000);
    int restU = 0;
    for (int i2 = j + 1; i2 < n; ++i2) {
        const StageBound &bb = sb_at(P, S, i2, nd.b[P.app[i2]]);
        restT = fminf(restT, bb.maxNT);
        restU += (int)bb.minNP;
    }
    if (nd.rqsum - (int)r.NP < restU) ok = false;
    if (ok) {
        unsigned kl = child_keylb<CM>(P, S, nd, j, r, ce, restT, restU);
        if ((unsigned long long)kl > bound) ok = false;
    }
    return ok;
}

// warp-wide min of (key, x) over lanes with imp set; updates slot k of wb
__device__ __forceinline__ void warp_improve(WarpBest *wb, int k, bool imp, unsigned long long key,
                                             unsigned long long x, int lane) {
    unsigned im = __ballot_sync(0xffffffffu, imp);
    if (!im) return;
    unsigned long long bk = imp ? key : ~0ull, bx = imp ? x : ~0ull;
    for (int off = 16; off; off >>= 1) {
        unsigned long long ok2 = __shfl_xor_sync(0xffffffffu, bk, off);
        unsigned long long ox = __shfl_xor_sync(0xffffffffu, bx, off);
        if (slot_less(ok2, ox, bk, bx)) {
            bk = ok2;
            bx = ox;
        }
    }
    __syncwarp();
    if (lane == 0 && slot_less(bk, bx, wb->key[k], wb->x[k])) {
        wb->key[k] = bk;
        wb->x[k] = bx;
    }
    __syncwarp();
}

// does this rank own the node at depth S.d0 (chunk = item / chunk_items,
// item = canonical position of (beta combo, option indices of stages < d0))?
template <int CM>
__device__ __forceinline__ bool owns(const DevProb &P, const SearchArgs &S, const Node<CM> &nd) {
    unsigned long long it = 0;
    for (int i = 0; i < S.d0; ++i) it = it * sb_at(P, S, i, nd.b[P.app[i]]).cnt + (unsigned long long)nd.kidx[i];
    const unsigned long long chunk = (S.item_off[nd.bc] + it) / (unsigned long long)S.chunk_items;
    if (chunk < S.chunk_lo) return false;
    if (S.chunk_hi && chunk >= S.chunk_hi) return false;
    return (chunk % (unsigned long long)S.world) == (unsigned long long)S.rank;
}

template <int CM>
__device__ __forceinline__ void copy_node(Node<CM> &dst, const Node<CM> &src, int lane) {
    static_assert(sizeof(Node<CM>) % 4 == 0, "node size");
    const uint32_t *s = reinterpret_cast<const uint32_t *>(&src);
    uint32_t *d = reinterpret_cast<uint32_t *>(&dst);
    for (int w = lane; w < (int)(sizeof(Node<CM>) / 4); w += 32) d[w] = s[w];
    __syncwarp();
}

// ---------------------------------------------------------------- the search kernel
// One level-synchronous pass: warps pop parents (dynamic, `grab` at a time),
// lanes expand the parent's children 32 at a time, surviving children at depth
// `flevel` are appended to the output frontier (inline depth-first descent when
// the frontier is full), leaves are scored exactly.
template <int CM, int POLICY>
__global__ void __launch_bounds__(SEARCH_THREADS)
search_kernel(const DevProb P, const SearchArgs S) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    Node<CM> *stack_all = reinterpret_cast<Node<CM> *>(smem_raw);
    WarpCtl *ctl_all = reinterpret_cast<WarpCtl *>(stack_all + (size_t)SEARCH_WARPS * NMAX);
    WarpBest *wb_all = reinterpret_cast<WarpBest *>(ctl_all + SEARCH_WARPS);
    Node<CM> *stack = stack_all + (size_t)wid * NMAX;
    WarpCtl *ctl = ctl_all + wid;
    WarpBest *wb = wb_all + wid;
    const int nlev = S.nlev;
    for (int k = lane; k < nlev; k += 32) {
        wb->key[k] = S.inc[k].key;
        wb->x[k] = S.inc[k].x;
    }
    __syncwarp();
    if (lane == 0) {
        unsigned long long m = 0;
        for (int k = 0; k < nlev; ++k) m = max(m, wb->key[k]);
        const unsigned long long g = (unsigned long long)(*(volatile unsigned int *)&S.hdr->best_obj);
        wb->bound = min(m, g);
    }
    __syncwarp();
    unsigned long long scored = 0, feasible = 0, nodes = 0;
    unsigned viol_or = 0;
    const int n = P.n;
    const int jtop = S.level;
    const Node<CM> *in = reinterpret_cast<const Node<CM> *>(S.in_nodes);
    Node<CM> *outf = reinterpret_cast<Node<CM> *>(S.out_nodes);
    const unsigned long long count = in ? min(*(volatile const unsigned long long *)S.in_count, S.in_cap)
                                        : (unsigned long long)P.nbc;

    while (true) {
        unsigned long long e0 = 0;
        if (lane == 0) e0 = atomicAdd(S.head, (unsigned long long)S.grab);
        e0 = __shfl_sync(0xffffffffu, e0, 0);
        if (e0 >= count) break;
        if (lane == 0) {   // refresh the pruning bound from the device-wide best
            const unsigned long long g = (unsigned long long)(*(volatile unsigned int *)&S.hdr->best_obj);
            if (g < wb->bound) wb->bound = g;
        }
        __syncwarp();
        const unsigned long long e1 = min(e0 + (unsigned long long)S.grab, count);
        for (unsigned long long e = e0; e < e1; ++e) {
            if (!in) {
                build_root<CM>(P, (int)e, stack[0], lane);
                if (lane == 0) {
                    for (int i = 0; i < NMAX; ++i) stack[0].kidx[i] = 0;
                }
                __syncwarp();
            } else {
                copy_node<CM>(stack[jtop], in[e], lane);
            }
            // ---- depth-first walk below the parent (normally one level: the
            // surviving children go to the next frontier)
            int j = jtop;
            if (lane == 0) {
                ctl->cur[j] = 0;
                ctl->msk[j] = 0;
            }
            __syncwarp();
            while (true) {
                const Node<CM> &nd = stack[j];
                const int bj = nd.b[P.app[j]];
                const int cntj = (int)sb_at(P, S, j, bj).cnt;
                const unsigned msk = ctl->msk[j];
                if (msk) {
                    const int kk = __ffs(msk) - 1;
                    const int opt = ctl->base[j] + kk;
                    __syncwarp();
                    if (lane == 0) ctl->msk[j] = msk & (msk - 1);
                    build_child<CM>(P, S, nd, j, opt_at(P, S, j, bj, opt), opt, stack[j + 1], lane);
                    if (j + 1 == S.d0 && !owns<CM>(P, S, stack[j + 1])) continue;
                    if (j + 1 == S.flevel) {
                        unsigned long long slot = 0;
                        if (lane == 0) slot = atomicAdd(S.out_tail, 1ull);
                        slot = __shfl_sync(0xffffffffu, slot, 0);
                        if (slot < S.out_cap) {
                            copy_node<CM>(outf[slot], stack[j + 1], lane);
                            continue;
                        }
                    }
                    ++j;   // descend inline (frontier full, or below the frontier level)
                    if (lane == 0) {
                        ctl->cur[j] = 0;
                        ctl->msk[j] = 0;
                    }
                    __syncwarp();
                    continue;
                }
                const int cur = ctl->cur[j];
                if (cur >= cntj) {
                    if (j == jtop) break;
                    --j;
                    continue;
                }
                __syncwarp();
                if (lane == 0) {
                    ctl->base[j] = cur;
                    ctl->cur[j] = cur + 32;
                }
                __syncwarp();
                const int opt = cur + lane;
                const bool valid = opt < cntj;
                const OptRec &r = opt_at(P, S, j, bj, valid ? opt : cur);
                ChildEval ce;
                if (valid) eval_child<CM>(P, S, nd, j, r, ce);
                else ce.placed = false;
                if (j < n - 1) {
                    // ---- inner node
                    nodes += valid;
                    const bool sv = valid && inner_survives<CM>(P, S, nd, j, r, ce, wb->bound);
                    const unsigned m = __ballot_sync(0xffffffffu, sv);
                    if (lane == 0) ctl->msk[j] = m;
                    __syncwarp();
                    continue;
                }
                // ---- leaf: exact score of candidate ce.x
                const bool inr = valid && ce.x >= S.lo && ce.x < S.hi;
                scored += inr;
                if (inr && !ce.placed) viol_or |= place_fail_bits<CM>(P, nd, r);
                bool feas = inr && ce.placed;
                if (feas) {
                    bool q = true;
                    for (int a = 0; a < P.A; ++a) q &= ce.lsum[a] <= P.qos[a];
                    if (!q) viol_or |= V_QOS;
                    feas = q;
                }
                feasible += feas;
                if (POLICY == 0) {
                    unsigned long long key = 0xFFFFFFFFull;
                    if (feas) {
                        // T <= min_i fl(N_i thr_i): skip the divisions when it cannot win
                        const unsigned long long kl = objkey_maxload(fminf(nd.tub, r.NT));
                        if (slot_less(kl, ce.x, wb->key[0], wb->x[0])) {
                            float T = __int_as_float(0x7f800000);
                            for (int i = 0; i < n; ++i) {
                                const float nti = (i < j) ? nd.nt[i] : r.NT;
                                const float ti = ce.kap[i] == 1.0f ? nti : __fdiv_rn(nti, ce.kap[i]);
                                T = fminf(T, ti);
                            }
                            key = objkey_maxload(T);
                        }
                    }
                    const bool imp = key != 0xFFFFFFFFull && slot_less(key, ce.x, wb->key[0], wb->x[0]);
                    warp_improve(wb, 0, imp, key, ce.x, lane);
                    if (lane == 0 && wb->key[0] < wb->bound) {
                        wb->bound = wb->key[0];
                        atomicMin(&S.hdr->best_obj, (unsigned int)wb->key[0]);
                    }
                    __syncwarp();
                } else {
                    const unsigned long long key = objkey_minres(ce.u, ce.U);
                    const bool cand = feas && key <= wb->bound;
                    float tmin[AMAX] = {0.0f, 0.0f};
                    if (cand) {
                        for (int a = 0; a < P.A; ++a) {
                            float tm = __int_as_float(0x7f800000);
                            for (int i = P.first_of_app[a]; i <= P.last_of_app[a]; ++i) {
                                const float nti = (i < j) ? nd.nt[i] : r.NT;
                                const float ti = ce.kap[i] == 1.0f ? nti : __fdiv_rn(nti, ce.kap[i]);
                                tm = fminf(tm, ti);
                            }
                            tmin[a] = tm;
                        }
                    }
                    if (__any_sync(0xffffffffu, cand)) {
                        for (int k = 0; k < nlev; ++k) {
                            bool fk = cand;
                            if (fk) {
                                for (int a = 0; a < P.A; ++a) fk &= tmin[a] >= S.lam[k * P.A + a];
                                if ((P.flags & F_EQ2_BUDGET) && ce.u > S.y[nd.bc * S.ystride + S.yoff + k]) fk = false;
                            }
                            const bool imp = fk && slot_less(key, ce.x, wb->key[k], wb->x[k]);
                            warp_improve(wb, k, imp, key, ce.x, lane);
                        }
                        if (lane == 0) {
                            unsigned long long m = 0;
                            for (int k = 0; k < nlev; ++k) m = max(m, wb->key[k]);
                            if (m < wb->bound) {
                                wb->bound = m;
                                atomicMin(&S.hdr->best_obj, (unsigned int)min(m, 0xFFFFFFFFull));
                            }
                        }
                        __syncwarp();
                    }
                }
            }
        }
    }
    // ---- CTA reduction of warp bests, MERGED into this CTA's slot (slots are
    // reset once per search; every pass may score leaves via inline descent)
    __syncthreads();
    for (int k = threadIdx.x; k < nlev; k += blockDim.x) {
        Slot &sl = S.slots[(size_t)blockIdx.x * nlev + k];
        unsigned long long bk = sl.key, bx = sl.x;
        for (int w = 0; w < SEARCH_WARPS; ++w)
            if (slot_less(wb_all[w].key[k], wb_all[w].x[k], bk, bx)) {
                bk = wb_all[w].key[k];
                bx = wb_all[w].x[k];
            }
        sl.key = bk;
        sl.x = bx;
    }
    for (int off = 16; off; off >>= 1) {
        scored += __shfl_xor_sync(0xffffffffu, scored, off);
        feasible += __shfl_xor_sync(0xffffffffu, feasible, off);
        nodes += __shfl_xor_sync(0xffffffffu, nodes, off);
        viol_or |= __shfl_xor_sync(0xffffffffu, viol_or, off);
    }
    if (lane == 0) {
        atomicAdd(&S.hdr->n_scored, scored);
        atomicAdd(&S.hdr->n_feasible, feasible);
        atomicAdd(&S.hdr->n_nodes, nodes);
        atomicOr(&S.hdr->viol_or, viol_or);
    }
}

}  // namespace cam
