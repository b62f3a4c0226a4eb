// camelot_search.cuh -- the exact, pruned allocation search (kernel N1) for
// sm_100a.
//
// Search order.  The candidate space is the tree  batch combo -> stage-1 option
// -> ... -> stage-n option  (option = (N_i, p_i); batch
// L858).  It is expanded LEVEL-SYNCHRONOUSLY: pass j pops parents (placement
// state after stages 0..j-1) from a global frontier with one atomic per parent,
// hoists the parent into registers, and the 32 lanes of a warp evaluate 32
// children (stage-j options) at a time: placement, contention, latency sums,
// bounds.  Every surviving child is written by its own lane to the next
// frontier; when the frontier is full the warp descends inline (explicit
// per-warp stack, same evaluator).  Leaves (last stage) are scored exactly and
// reduced into the warp's best (objective key, canonical index).
//
// Pruning.  A child is dropped only if no candidate below it
// can be feasible and at least as good as a feasible candidate already known
// (incumbent / best so far): failed placement of the prefix; QoS lower bound
// (contention only grows, ordered fp32 sums are monotone); throughput upper
// bound (T_i <= fl(N_i thr_i) / kappa_i(current)); quota left; min-resource key
// lower bound; ties by index (a subtree that can at best tie and lies entirely
// above the best's index).  Strictly better keys are never pruned.
#pragma once
#include "camelot_device.cuh"
#include "camelot_score.cuh"
#include <cstddef>

namespace cam {

// testing knob (compile time): -DCAMELOT_NO_TMODE keeps every pass in the warp mode
__device__ __forceinline__ bool getenv_tmode_off() {
#ifdef CAMELOT_NO_TMODE
    return true;
#else
    return false;
#endif
}

#ifndef CAMELOT_SEARCH_THREADS
#define CAMELOT_SEARCH_THREADS 256
#endif
constexpr int SEARCH_THREADS = CAMELOT_SEARCH_THREADS;
constexpr int SEARCH_WARPS = SEARCH_THREADS / 32;
#ifndef SEARCH_MINB
#define SEARCH_MINB 1   // measured with the thread-per-parent mode: 255 regs x 1 CTA (no spills) beats 128 x 2 (C4 1.51 vs 1.75 ms)
#endif

struct SearchArgs {
    int policy;                 // 0 max-load, 1 min-resource
    int nlev;                   // number of best slots (1 for max-load)
    int d0;                     // stage levels flattened into items (1 <= d0 <= n-1)
    int chunk_items;            // items per chunk (work unit, key low bits when Ntot > 2^32)
    int rank, world;
    int prune;                  // 0 = flat scan (bounds off)
    unsigned long long lo, hi;  // canonical index range
    const OptRec *rec;          // [n][nS][O] compacted surviving options (ascending code)
    const OptRec *rec_stage;    // per-CTA shared-memory copy of the compacted lists (or nullptr)
    const int *rec_off;         // [n][nS] offset of list (i, b) in rec_stage (when staged)
    const StageBound *sb;       // [n][nS]
    const unsigned long long *item_off;  // [nbc + 1]
    const float *lam;           // [nlev][A] load levels (min-resource)
    int lam_stride;             // A (row stride of lam)
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
    int xshift;                 // index >> xshift fits 32 bits (tie pruning key)
    int tmode_min16;            // thread-per-parent mode from count >= tmode_min16 / 16 x resident warps
    int tmode_inner_gmax;       // inner passes: up to this many lanes per parent (32 children per lane)
    int tmode_leaf_gmax;        // leaf passes: up to this many lanes per parent (32 children per lane)
    int tmode_slack;            // inner thread-per-parent passes allowed up to count x maxc <= slack x out_cap
                                // (> 1: optimistic -- the caller redoes an overflowing pass in the warp mode)
    int no_tmode;               // the redo: warp mode only
    int compact1;               // the depth-1 frontier holds (batch combo, stage-0 option) pairs: the
                                // root pass writes 2 words per child, the depth-1 pass rebuilds the node
    // fused reduction (last pass): the last CTA reduces all slots
    int reduce_last;
    Slot *result;               // [nlev] exact local best
    long long *keys;            // [nlev] packed keys
    Slot *inc_out;              // [nlev] next incumbent (cascade) or nullptr
};

// Placement state after the first j stages (shared-memory DFS stack and the
// global frontier).  Per-GPU arrays are stored in POSITION order of the
// deployment order for the NEXT stage (sorted by remaining memory, remaining
// quota, index -- PAPER.md L929-942); pgid maps a position to its GPU id.
template <int CM>
struct Node {
    int prq[CM], pcnt[CM], pkim[CM], pgid[CM];
    uint32_t prm[CM];
    float pdem[CM];
    float dur[NMAX], bw[NMAX], nt[NMAX], dmax[NMAX];
    uint32_t hmask[NMAX];
    int kidx[NMAX];         // position of each placed stage's option in its compacted list
    unsigned long long x;   // canonical prefix value
    int U, u, rqsum, bc;
    int b[AMAX];
    float tub;              // min fl(N thr) over placed stages
};

// The global frontier is a structure of arrays: 32-bit word w of node k lives at
// base[w * cap + k], so the lanes of a warp that emit consecutive slots write
// every field with one coalesced store (an array-of-structs frontier costs one
// memory transaction per lane and field).
template <int CM>
struct Frontier {
    uint32_t *base;
    unsigned long long cap;
    static constexpr int WORDS = (int)(sizeof(Node<CM>) / 4);
    __device__ __forceinline__ void put(int w, unsigned long long k, uint32_t v) const { base[(size_t)w * cap + k] = v; }
    __device__ __forceinline__ void putf(int w, unsigned long long k, float v) const { put(w, k, __float_as_uint(v)); }
};
#define NODE_W(CM, field) ((int)(offsetof(Node<CM>, field) / 4))

// Read-only view of node k of a structure-of-arrays frontier with the field syntax
// of Node<CM> (nd.prq[q], nd.x, ...), for the thread-per-parent mode: the lanes of
// a warp view consecutive nodes, so every field read is coalesced.
template <typename T>
struct FieldView {
    const uint32_t *p;
    unsigned long long cap;
    __device__ __forceinline__ T operator[](int i) const {
        // read-only during the pass; written by the previous pass, and the grid barrier
        // between the two invalidates L1, so the L1-cached read-only path is coherent
        const uint32_t v = __ldg(p + (size_t)i * cap);
        T t;
        memcpy(&t, &v, 4);
        return t;
    }
};
template <int CM>
struct NodeSoA {
    FieldView<int> prq, pcnt, pkim, pgid, kidx, b;
    FieldView<uint32_t> prm, hmask;
    FieldView<float> pdem, dur, bw, nt, dmax;
    unsigned long long x;
    int U, u, rqsum, bc;
    float tub;
    __device__ __forceinline__ NodeSoA(const Frontier<CM> &F, unsigned long long k) {
        const uint32_t *B = F.base + k;
        const unsigned long long c = F.cap;
        auto at = [&](int w) { return B + (size_t)w * c; };
        prq = {at(NODE_W(CM, prq)), c};
        pcnt = {at(NODE_W(CM, pcnt)), c};
        pkim = {at(NODE_W(CM, pkim)), c};
        pgid = {at(NODE_W(CM, pgid)), c};
        kidx = {at(NODE_W(CM, kidx)), c};
        b = {at(NODE_W(CM, b)), c};
        prm = {at(NODE_W(CM, prm)), c};
        hmask = {at(NODE_W(CM, hmask)), c};
        pdem = {at(NODE_W(CM, pdem)), c};
        dur = {at(NODE_W(CM, dur)), c};
        bw = {at(NODE_W(CM, bw)), c};
        nt = {at(NODE_W(CM, nt)), c};
        dmax = {at(NODE_W(CM, dmax)), c};
        x = (unsigned long long)__ldg(at(NODE_W(CM, x))) | ((unsigned long long)__ldg(at(NODE_W(CM, x) + 1)) << 32);
        U = (int)__ldg(at(NODE_W(CM, U)));
        u = (int)__ldg(at(NODE_W(CM, u)));
        rqsum = (int)__ldg(at(NODE_W(CM, rqsum)));
        bc = (int)__ldg(at(NODE_W(CM, bc)));
        tub = __uint_as_float(__ldg(at(NODE_W(CM, tub))));
    }
};

// per-warp DFS bookkeeping (shared memory)
struct WarpCtl {
    int cur[NMAX];     // next child batch of the node at each depth
    int end[NMAX];     // end of that node's child range
    int base[NMAX];    // first child of the batch whose survivors are pending
    unsigned msk[NMAX];   // pending (inline-descent) survivors of that batch
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

// First-failing placement dimensions of a failed stage (DESIGN.md 3.2 step 5):
// the OR over GPUs of the dimensions in which fits(g, 1) fails AFTER pass 2.  A
// failed pass 2 leaves every GPU at its capacity c = canHold(g, Rmax) (< the
// replicas still to place), and on that state fits(g, 1) fails exactly in the
// integer dimensions where fits(g, c + 1) fails on the parent state (the stage's
// weights are charged once), and in bandwidth iff fl(fl(dem + fl(c bw)) + bw) > BW.
template <int CM>
__device__ __forceinline__ uint32_t place_fail_bits(const DevProb &P, const Node<CM> &nd, const OptRec &r) {
    const bool cap = !(P.flags & F_NO_BW_CAP);
    uint32_t v = 0;
    for (int q = 0; q < P.C; ++q) {
        int c = min((int)(((uint32_t)nd.prq[q] * r.pmul) >> 16), nd.pkim[q]);   // floor(rq / p), inst + mem
        if (cap)
            while (c > 0 && __fadd_rn(nd.pdem[q], __fmul_rn((float)c, r.bw)) > P.BW) --c;
        const int k = c + 1;
        if (k * (int)r.p > nd.prq[q]) v |= V_QUOTA;
        if (nd.pcnt[q] + k > P.I) v |= V_INST;
        if (r.W + (uint32_t)k * r.As > nd.prm[q]) v |= V_MEM;
        if (cap && __fadd_rn(__fadd_rn(nd.pdem[q], __fmul_rn((float)c, r.bw)), r.bw) > P.BW) v |= V_BW;
    }
    return v ? v : V_QUOTA;
}

// compacted option list of (stage i, batch b): the CTA's shared-memory copy when the
// level staged it (TMA bulk copy after the filter), else the global [n][nS][O] array
__device__ __forceinline__ const OptRec *list_of(const DevProb &P, const SearchArgs &S, int i, int b) {
    return S.rec_off ? S.rec_stage + S.rec_off[i * P.nS + b] : S.rec + ((size_t)i * P.nS + b) * P.O;
}
// one 16-byte chunk of a record (generic load: the list may be in shared or global memory)
__device__ __forceinline__ uint4 rec_chunk(const OptRec *r, int c) { return reinterpret_cast<const uint4 *>(r)[c]; }
__device__ __forceinline__ const StageBound &sb_at(const DevProb &P, const SearchArgs &S, int i, int b) {
    return S.sb[(size_t)i * P.nS + b];
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
        rq = nd.prq[lane] - k * (int)r.p;
        cnt = nd.pcnt[lane] + k;
        rm = nd.prm[lane] - (k > 0 ? r.W + (uint32_t)k * r.As : 0u);
        dem = k > 0 ? __fadd_rn(nd.pdem[lane], __fmul_rn((float)k, r.bw)) : nd.pdem[lane];
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
        out.prq[rank] = rq;
        out.pcnt[rank] = cnt;
        out.prm[rank] = rm;
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
    unsigned unew = __popc(__ballot_sync(0xffffffffu, lane < P.C && k > 0 && nd.pcnt[lane] == 0));
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
    int b[AMAX];   // batch index per application (explicit: no dynamically indexed local array)
    {
        int t = bc;
        b[AMAX - 1] = t % P.nS;
        if (P.A > 1) t /= P.nS;
        b[0] = t % P.nS;
    }
    __syncwarp();
    if (lane < P.C) {
        const int g = lane;
        out.pcnt[g] = 0;
        out.prm[g] = P.FM;
        // all GPUs equal: order = index
        const uint32_t W0 = P.W[0], As0 = P.Am[0] * (uint32_t)P.S[P.app[0] ? b[AMAX - 1] : b[0]];
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
    unsigned long long gpack;       // device-wide (key << 32 | x >> xshift) best (1 level)
    float lmin;                     // min-resource, one application: the smallest load level
    int mlev;                       // min-resource, one application, several levels: level-aware bound
    float lam[LMAX];                // (mlev) the load of each level
};

// Can a subtree whose keys are >= kl and whose indices are >= xs still hold
// the answer?  Strictly worse keys cannot; with ONE level, a key equal to the
// best can only tie and ties go to the smallest index, so a subtree entirely
// above the best's index cannot either (exact).
// Min resource with several load levels (one application): a subtree whose completions
// all have T <= tub cannot be feasible at a level with load > tub, so only the levels
// it can carry bound it (their best keys are non-decreasing in the load, the bound is
// the largest of them); no such level: nothing to find.  (wb->bound, the max over all
// levels, is the plain rule.)
__device__ __forceinline__ unsigned long long level_bound(const WarpBest *wb, int nlev, float tub) {
    if (nlev == 1 || !wb->mlev) return wb->bound;
    unsigned long long m = 0;
    for (int k = 0; k < nlev; ++k)
        if (wb->lam[k] <= tub) m = max(m, wb->key[k]);
    return min(m, wb->bound);
}

__device__ __forceinline__ bool can_win(unsigned long long kl, unsigned long long xs, const WarpBest *wb, int nlev,
                                        int xshift, float tub = __builtin_inff()) {
    if (kl > level_bound(wb, nlev, tub)) return false;
    if (nlev == 1) {
        if (kl == wb->key[0] && xs > wb->x[0]) return false;
        if (kl == (wb->gpack >> 32) && (xs >> xshift) > (wb->gpack & 0xFFFFFFFFull)) return false;
    }
    return true;
}

__device__ __forceinline__ void publish_best(const SearchArgs &S, WarpBest *wb) {
    // lane 0 only: the warp's level-0 best to the device-wide packed best
    if (wb->key[0] >= 0xFFFFFFFFull) return;
    const unsigned long long pk = (wb->key[0] << 32) | min(wb->x[0] >> S.xshift, 0xFFFFFFFFull);
    if (pk < wb->gpack) {
        wb->gpack = pk;
        atomicMin(&S.hdr->best_packed, pk);
    }
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

// ---------------------------------------------------------------- register context (fast path)
// The parent's placement state hoisted into registers once per parent.
// Positions are padded to the compile-time width CM (padding: no quota, no
// capacity => never used); stages to NS >= n.
template <int CM, int NS>
struct PCtx {
    int prq[CM], pkim[CM];
    float pdem[CM];
    unsigned empty;                 // bit q: position q hosts no instance yet
    unsigned hp[NS];                // bit q: placed stage i has a replica at position q
    float dmax[NS], dur[NS], bw[NS], nt[NS];   // i < j: placed stage; i > j: dur = min duration
    float tub, restT;
    float lpre;                     // ordered fp32 sum of current L of placed stages of app(j) (-1: none)
    float tx[NS];                   // COMM: cross-GPU hand-over time of edge i -> i+1 (at its app's batch)
    float lother;                   // lower bound of the other application's latency sum (A = 2)
    int u, U, rqsum, restU, bc;
    unsigned long long x;
};

template <int CM, int NS, typename ND = Node<CM>>
__device__ __forceinline__ void load_ctx(const DevProb &P, const SearchArgs &S, const ND &nd, int j,
                                         PCtx<CM, NS> &c) {
    c.empty = 0;
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        const bool in = q < P.C;
        c.prq[q] = in ? nd.prq[q] : 0;
        c.pkim[q] = in ? nd.pkim[q] : 0;
        c.pdem[q] = in ? nd.pdem[q] : 0.0f;
        if (in && nd.pcnt[q] == 0) c.empty |= 1u << q;
    }
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        c.hp[i] = 0;
        c.dmax[i] = 0.0f;
        c.bw[i] = 0.0f;
        c.nt[i] = 0.0f;
        c.dur[i] = 0.0f;
        if (i < j) {
            const unsigned hm = nd.hmask[i];
            unsigned m = 0;
#pragma unroll
            for (int q = 0; q < CM; ++q)
                if (q < P.C && ((hm >> nd.pgid[q]) & 1u)) m |= 1u << q;
            c.hp[i] = m;
            c.dmax[i] = nd.dmax[i];
            c.dur[i] = nd.dur[i];
            c.bw[i] = nd.bw[i];
            c.nt[i] = nd.nt[i];
        } else if (i > j && i < P.n) {
            c.dur[i] = sb_at(P, S, i, nd.b[P.app[i]]).mindur;
        }
    }
    float restT = __int_as_float(0x7f800000);
    int restU = 0;
    for (int i2 = j + 1; i2 < P.n; ++i2) {
        const StageBound &bb = sb_at(P, S, i2, nd.b[P.app[i2]]);
        restT = fminf(restT, bb.maxNT);
        restU += (int)bb.minNP;
    }
    c.restT = restT;
    c.restU = restU;
    // throughput upper bound of every completion: contention only grows, so
    // T_i <= fl(fl(N_i thr_i) / kappa_i(current)) for the placed stages
    float tub = nd.tub;
#pragma unroll
    for (int i = 0; i < NS; ++i)
        if (S.prune && i < j) {
            const float k = kappa_of(c.dmax[i], c.bw[i], P.gamma[i], P.invBW, P.flags);
            if (k != 1.0f) tub = fminf(tub, __fdiv_rn(c.nt[i], k));
        }
    c.tub = tub;
    // QoS prefix of the child's application (current contention; it only grows)
    c.lpre = -1.0f;
    c.lother = 0.0f;
    if (S.prune) {
        const int aj = P.app[j];
        float lp = -1.0f, lo = 0.0f;
        bool lo_started = false;
#pragma unroll
        for (int i = 0; i < NS; ++i)
            if (i < P.n) {
                float L;
                if (i < j) L = __fmul_rn(c.dur[i], kappa_of(c.dmax[i], c.bw[i], P.gamma[i], P.invBW, P.flags));
                else if (i > j) L = c.dur[i];
                else continue;
                if (P.app[i] == aj) {
                    if (i < j) lp = (lp < 0.0f) ? L : __fadd_rn(lp, L);
                } else {
                    lo = lo_started ? __fadd_rn(lo, L) : L;
                    lo_started = true;
                }
            }
        c.lpre = lp;
        c.lother = lo_started ? lo : 0.0f;
    }
    if (P.flags & F_COMM) {
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            c.tx[i] = 0.0f;
            if (i + 1 < P.n && P.app[i] == P.app[i + 1])
                c.tx[i] = __fmul_rn(__fmul_rn(P.comm_mb[i], (float)P.S[nd.b[P.app[i]]]), P.inv_link);
        }
    }
    c.u = nd.u;
    c.U = nd.U;
    c.rqsum = nd.rqsum;
    c.bc = nd.bc;
    c.x = nd.x;
}

struct FastEval {
    bool placed;
    int u, U;
    float lsum[AMAX];
    float kap[NMAX];
    unsigned long long x;
};

// Place stage j with option r on the context and score it (branch-free
// placement: per-position capacities K_q = canHold(q, N); pass 1 = first q with
// K_q == N; pass 2 = greedy min(K_q, remaining) -- DESIGN.md 3.2, R14).
template <int CM, int NS>
__device__ __forceinline__ bool fast_place(const DevProb &P, const PCtx<CM, NS> &c, const OptRec &r, int (&kk)[CM]) {
    const int N = (int)r.N;
    const bool cap = !(P.flags & F_NO_BW_CAP);
    int K[CM];
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        int k = min(min(N, (int)(((uint32_t)c.prq[q] * r.pmul) >> 16)), c.pkim[q]);
        if (cap && k > 0 && __fadd_rn(c.pdem[q], __fmul_rn((float)k, r.bw)) > P.BW) {
            do {
                --k;
            } while (k > 0 && __fadd_rn(c.pdem[q], __fmul_rn((float)k, r.bw)) > P.BW);
        }
        K[q] = k;
    }
    int jstar = CM;
#pragma unroll
    for (int q = CM - 1; q >= 0; --q)
        if (K[q] == N) jstar = q;
    int rem = N;
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        const int g = min(K[q], rem);
        rem -= g;
        kk[q] = (jstar < CM) ? (q == jstar ? N : 0) : g;
    }
    return (jstar < CM) || rem == 0;
}

template <int CM, int NS>
__device__ __forceinline__ void fast_eval(const DevProb &P, const PCtx<CM, NS> &c, int j, const OptRec &r,
                                          FastEval &fe) {
    const int N = (int)r.N;
    const bool cap = !(P.flags & F_NO_BW_CAP);
    int K[CM];
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        int k = min(min(N, (int)(((uint32_t)c.prq[q] * r.pmul) >> 16)), c.pkim[q]);
        if (cap && k > 0 && __fadd_rn(c.pdem[q], __fmul_rn((float)k, r.bw)) > P.BW) {
            do {
                --k;
            } while (k > 0 && __fadd_rn(c.pdem[q], __fmul_rn((float)k, r.bw)) > P.BW);
        }
        K[q] = k;
    }
    int jstar = CM;
#pragma unroll
    for (int q = CM - 1; q >= 0; --q)
        if (K[q] == N) jstar = q;
    int kk[CM];
    int rem = N;
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        const int g = min(K[q], rem);
        rem -= g;
        kk[q] = (jstar < CM) ? (q == jstar ? N : 0) : g;
    }
    fe.placed = (jstar < CM) || rem == 0;
    fe.x = c.x * (unsigned long long)P.O + r.code;
    fe.U = c.U + (int)r.NP;
    float dm[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) dm[i] = c.dmax[i];
    float dself = 0.0f;
    int unew = 0;
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        // demand after the stage (== pdem when no replica lands on q)
        const float d = __fadd_rn(c.pdem[q], __fmul_rn((float)kk[q], r.bw));
        if (kk[q] > 0) {
            dself = fmaxf(dself, d);
            unew += (c.empty >> q) & 1u;
        }
#pragma unroll
        for (int i = 0; i < NS; ++i)
            if ((c.hp[i] >> q) & 1u) dm[i] = fmaxf(dm[i], d);
    }
    fe.u = c.u + unew;
    float l0 = 0.0f, l1 = 0.0f;
    // COMM (R29): positions hosting stage j; an edge whose both stages are placed has
    // its exact hand-over time, otherwise its lower bound min(ipc, cross)
    const bool comm = (P.flags & F_COMM) != 0;
    unsigned jm = 0u;
    if (comm) {
#pragma unroll
        for (int q = 0; q < CM; ++q) jm |= (kk[q] > 0 ? 1u : 0u) << q;
    }
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        if (i < P.n) {
            if (comm && i > 0 && P.app[i - 1] == P.app[i]) {
                float t;
                if (i <= j) {   // both i-1 and i placed
                    const unsigned mp = c.hp[i - 1], mi = (i == j) ? jm : c.hp[i];
                    t = (mp == mi && __popc(mi) == 1) ? P.ipc_ms : c.tx[i - 1];
                } else {
                    t = fminf(P.ipc_ms, c.tx[i - 1]);
                }
                if (P.app[i] == 0) l0 = __fadd_rn(l0, t);
                else l1 = __fadd_rn(l1, t);
            }
            float L;
            if (i < j) {
                const float k = kappa_of(dm[i], c.bw[i], P.gamma[i], P.invBW, P.flags);
                fe.kap[i] = k;
                L = __fmul_rn(c.dur[i], k);
            } else if (i == j) {
                const float k = kappa_of(dself, r.bw, P.gamma[i], P.invBW, P.flags);
                fe.kap[i] = k;
                L = __fmul_rn(r.dur, k);
            } else {
                fe.kap[i] = 1.0f;
                L = c.dur[i];
            }
            // ordered per-application sums (stages are app-major)
            if (P.app[i] == 0) l0 = (i == 0) ? L : __fadd_rn(l0, L);
            else l1 = (i == P.first_of_app[1]) ? L : __fadd_rn(l1, L);
        }
    }
    fe.lsum[0] = l0;
    fe.lsum[1] = l1;
}

// Is min_i fl(nt_i / kap_i) over stages i <= j certainly below the threshold
// T_thr?  __fdividef is within 2 ulp; with the 2^-19 margin the answer "yes" is
// exact-safe (used only to prune; exact values are computed with __fdiv_rn).
template <int NS, typename NtF>
__device__ __forceinline__ bool t_certainly_below(const DevProb &P, int j, const float *kap, NtF nt, float T_thr) {
    float t = __int_as_float(0x7f800000);
#pragma unroll
    for (int i = 0; i < NS; ++i)
        if (i <= j && i < P.n) t = fminf(t, kap[i] == 1.0f ? nt(i) : __fdividef(nt(i), kap[i]));
    return __fmul_rn(t, 1.0f + 1.0f / 524288.0f) < T_thr;
}

struct Counters {
    unsigned long long scored, feasible, nodes;
    unsigned viol;
};

// Exact leaf scoring + warp-level best update (shared by both paths).
// nt(i) = fl(N_i thr_i) of stage i, kap(i) = contention factor.
template <int POLICY, int NS, typename NtF>
__device__ __forceinline__ void score_leaf(const DevProb &P, const SearchArgs &S, WarpBest *wb, int lane, bool inr,
                                           bool placed, const float *lsum, const float *kap, NtF nt, float tub,
                                           int u, int U, int bc, unsigned long long x, Counters &cn) {
    const int pol = POLICY == 2 ? S.policy : POLICY;   // 2: the policy is a runtime argument (shared code)
    cn.scored += inr;
    bool feas = inr && placed;
    if (feas) {
        bool q = lsum[0] <= P.qos[0];
        if (P.A > 1) q &= lsum[1] <= P.qos[1];
        if (!q) cn.viol |= V_QOS;
        feas = q;
    }
    cn.feasible += feas;
    const int n = P.n;
    if (pol == 0) {
        unsigned long long key = 0xFFFFFFFFull;
        if (feas) {
            // T <= min_i fl(N_i thr_i): the divisions only when it can win
            const unsigned long long kl = objkey_maxload(tub);
            bool maybe = slot_less(kl, x, wb->key[0], wb->x[0]);
            if (maybe && wb->key[0] < 0xFFFFFFFFull) {
                const float Tb = __uint_as_float(0xFFFFFFFFu - (unsigned)wb->key[0]);
                if (t_certainly_below<NS>(P, n - 1, kap, nt, Tb)) maybe = false;
            }
            if (maybe) {
                float T = __int_as_float(0x7f800000);
#pragma unroll
                for (int i = 0; i < NS; ++i)
                    if (i < n) {
                        const float ti = kap[i] == 1.0f ? nt(i) : __fdiv_rn(nt(i), kap[i]);
                        T = fminf(T, ti);
                    }
                key = objkey_maxload(T);
            }
        }
        const bool imp = key != 0xFFFFFFFFull && slot_less(key, x, wb->key[0], wb->x[0]);
        warp_improve(wb, 0, imp, key, x, lane);
        if (lane == 0) {
            if (wb->key[0] < wb->bound) {
                wb->bound = wb->key[0];
                atomicMin(&S.hdr->best_obj, (unsigned int)wb->key[0]);
            }
            publish_best(S, wb);
        }
        __syncwarp();
    } else {
        const unsigned long long key = objkey_minres(u, U);
        const bool cand = feas && key <= wb->bound;
        float tm0 = __int_as_float(0x7f800000), tm1 = __int_as_float(0x7f800000);
        if (cand) {
#pragma unroll
            for (int i = 0; i < NS; ++i)
                if (i < n) {
                    const float ti = kap[i] == 1.0f ? nt(i) : __fdiv_rn(nt(i), kap[i]);
                    if (P.app[i] == 0) tm0 = fminf(tm0, ti);
                    else tm1 = fminf(tm1, ti);
                }
        }
        if (__any_sync(0xffffffffu, cand)) {
            const int nlev = S.nlev;
            for (int k = 0; k < nlev; ++k) {
                bool fk = cand;
                if (fk) {
                    fk &= tm0 >= S.lam[k * P.A];
                    if (P.A > 1) fk &= tm1 >= S.lam[k * P.A + 1];
                    if ((P.flags & F_EQ2_BUDGET) && u > S.y[bc * S.ystride + S.yoff + k]) fk = false;
                }
                const bool imp = fk && slot_less(key, x, wb->key[k], wb->x[k]);
                warp_improve(wb, k, imp, key, x, lane);
            }
            if (lane == 0) {
                unsigned long long m = 0;
                for (int k = 0; k < nlev; ++k) m = max(m, wb->key[k]);
                if (m < wb->bound) {
                    wb->bound = m;
                    atomicMin(&S.hdr->best_obj, (unsigned int)min(m, 0xFFFFFFFFull));
                }
                if (nlev == 1) publish_best(S, wb);
            }
            __syncwarp();
        }
    }
}

// does this rank own the node at depth S.d0 (chunk = item / chunk_items,
// item = canonical position of (beta combo, option indices of stages < d0))?
template <int CM>
__device__ __forceinline__ bool owns(const DevProb &P, const SearchArgs &S, const Node<CM> &nd) {
    if (S.world == 1 && S.chunk_lo == 0 && S.chunk_hi == 0) return true;
    unsigned long long it = 0;
    for (int i = 0; i < S.d0; ++i) it = it * sb_at(P, S, i, nd.b[P.app[i]]).cnt + (unsigned long long)nd.kidx[i];
    const unsigned long long chunk = (S.item_off[nd.bc] + it) / (unsigned long long)S.chunk_items;
    if (chunk < S.chunk_lo) return false;
    if (S.chunk_hi && chunk >= S.chunk_hi) return false;
    return (chunk % (unsigned long long)S.world) == (unsigned long long)S.rank;
}

template <int CM>
__device__ __forceinline__ void copy_node(Node<CM> &dst, const Frontier<CM> &F, unsigned long long k, int lane) {
    static_assert(sizeof(Node<CM>) % 4 == 0, "node size");
    uint32_t *d = reinterpret_cast<uint32_t *>(&dst);
    for (int w = lane; w < Frontier<CM>::WORDS; w += 32) d[w] = __ldcg(F.base + (size_t)w * F.cap + k);
    __syncwarp();
}

// Ownership of the child (stage j, option index kopt) of nd at depth S.d0 = j+1.
template <int CM, typename ND = Node<CM>>
__device__ __forceinline__ bool owns_child(const DevProb &P, const SearchArgs &S, const ND &nd, int j,
                                           int kopt) {
    if (S.world == 1 && S.chunk_lo == 0 && S.chunk_hi == 0) return true;   // one rank, no chunk restriction
    unsigned long long it = 0;
    for (int i = 0; i <= j; ++i)
        it = it * sb_at(P, S, i, nd.b[P.app[i]]).cnt + (unsigned long long)(i < j ? nd.kidx[i] : kopt);
    const unsigned long long chunk = (S.item_off[nd.bc] + it) / (unsigned long long)S.chunk_items;
    if (chunk < S.chunk_lo) return false;
    if (S.chunk_hi && chunk >= S.chunk_hi) return false;
    return (chunk % (unsigned long long)S.world) == (unsigned long long)S.rank;
}

// One lane builds its own surviving child (stage j placed with option r) and
// writes it to the global frontier: the same state as build_child (warp
// version), computed independently per lane so that all survivors of a batch
// are emitted in parallel.
template <int CM, int NS, typename ND = Node<CM>>
__device__ __forceinline__ void emit_child(const DevProb &P, const ND &nd, const PCtx<CM, NS> &c, int j,
                                           const OptRec &r, uint32_t p, uint32_t W, uint32_t As, int kopt,
                                           const Frontier<CM> &F, unsigned long long k) {
#define OUT_PUT(field, idx, v) F.put(NODE_W(CM, field) + (idx), k, (uint32_t)(v))
#define OUT_PUTF(field, idx, v) F.putf(NODE_W(CM, field) + (idx), k, (v))
    int kk[CM];
    fast_place<CM, NS>(P, c, r, kk);
    int rq[CM], cnt[CM], g[CM];
    uint32_t rm[CM];
    float dem[CM];
    unsigned hm = 0;
    int unew = 0;
    float dself = 0.0f;
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        rq[q] = 0;
        cnt[q] = 0;
        g[q] = 0;
        rm[q] = 0;
        dem[q] = 0.0f;
        if (q < P.C) {
            const int k = kk[q];
            g[q] = nd.pgid[q];
            rq[q] = c.prq[q] - k * (int)p;
            cnt[q] = nd.pcnt[q] + k;
            rm[q] = nd.prm[q] - (k > 0 ? W + (uint32_t)k * As : 0u);
            dem[q] = k > 0 ? __fadd_rn(c.pdem[q], __fmul_rn((float)k, r.bw)) : c.pdem[q];
            if (k > 0) {
                hm |= 1u << g[q];
                unew += nd.pcnt[q] == 0;
                dself = fmaxf(dself, dem[q]);
            }
        }
    }
    const bool more = j + 1 < P.n;
    uint32_t W2 = 0, As2 = 0;
    if (more) {
        const int i2 = j + 1;
        W2 = P.W[i2];
        As2 = P.Am[i2] * (uint32_t)P.S[nd.b[P.app[i2]]];
    }
    // deployment order for the next stage: (remaining MiB, remaining quota, id) packed
    // into one orderable 32-bit key (rm < 2^21 as FM < 2^21, 0 <= rq <= 127, id < 16)
    uint32_t okey[CM];
#pragma unroll
    for (int q = 0; q < CM; ++q) okey[q] = (rm[q] << 11) | ((uint32_t)rq[q] << 4) | (uint32_t)g[q];
#pragma unroll
    for (int q = 0; q < CM; ++q) {
        if (q < P.C) {
            int rank = 0;
#pragma unroll
            for (int h = 0; h < CM; ++h)
                if (h < P.C && h != q) rank += okey[h] < okey[q];
            int kim = 0;
            if (more) {
                // largest k <= min(Rmax, I - cnt) with W2 + k As2 <= rm (binary search, no
                // division; 32-bit: W + Rmax A s < 2^31 is validated and t <= lim <= Rmax)
                const int lim = min(P.Rmax, P.I - cnt[q]);
                if (lim > 0 && rm[q] >= W2) {
#pragma unroll
                    for (int step = 16; step >= 1; step >>= 1) {
                        const int t = kim + step;
                        if (t <= lim && W2 + (uint32_t)t * As2 <= rm[q]) kim = t;
                    }
                }
            }
            OUT_PUT(prq, rank, rq[q]);
            OUT_PUT(pcnt, rank, cnt[q]);
            OUT_PUT(prm, rank, rm[q]);
            OUT_PUT(pkim, rank, kim);
            OUT_PUT(pgid, rank, g[q]);
            OUT_PUTF(pdem, rank, dem[q]);
        }
    }
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        if (i < j) {
            float dm = nd.dmax[i];
            const unsigned hmi = nd.hmask[i];
#pragma unroll
            for (int q = 0; q < CM; ++q)
                if (q < P.C && kk[q] > 0 && ((hmi >> g[q]) & 1u)) dm = fmaxf(dm, dem[q]);
            OUT_PUTF(dur, i, nd.dur[i]);
            OUT_PUTF(bw, i, nd.bw[i]);
            OUT_PUTF(nt, i, nd.nt[i]);
            OUT_PUTF(dmax, i, dm);
            OUT_PUT(hmask, i, hmi);
            OUT_PUT(kidx, i, nd.kidx[i]);
        } else if (i == j) {
            OUT_PUTF(dur, i, r.dur);
            OUT_PUTF(bw, i, r.bw);
            OUT_PUTF(nt, i, r.NT);
            OUT_PUTF(dmax, i, dself);
            OUT_PUT(hmask, i, hm);
            OUT_PUT(kidx, i, kopt);
        }
    }
    {
        const unsigned long long xv = nd.x * (unsigned long long)P.O + r.code;
        OUT_PUT(x, 0, (uint32_t)xv);
        OUT_PUT(x, 1, (uint32_t)(xv >> 32));
    }
    OUT_PUT(U, 0, nd.U + (int)r.NP);
    OUT_PUT(u, 0, nd.u + unew);
    OUT_PUT(rqsum, 0, nd.rqsum - (int)r.NP);
    OUT_PUT(bc, 0, nd.bc);
    OUT_PUT(b, 0, nd.b[0]);
    OUT_PUT(b, AMAX - 1, nd.b[AMAX - 1]);
    OUT_PUTF(tub, 0, fminf(nd.tub, r.NT));
}

// the same item offsets, but an "empty" batch combo still has a well-defined
// (zero) item range; used by chunk_of()
__device__ inline long long find_code(const OptRec *list, int cnt, uint32_t code) {
    int lo = 0, hi = cnt;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (list[mid].code < code) lo = mid + 1;
        else hi = mid;
    }
    return (lo < cnt && list[lo].code == code) ? lo : -1;
}

__device__ inline unsigned long long item_of(const DevProb &P, const StageBound *sb, const OptRec *rec,
                                             const unsigned long long *item_off, int d0, unsigned long long x) {
    int beta[AMAX], rho[NMAX], theta[NMAX];
    decode_index(P, x, beta, rho, theta);
    int bc = 0;
    for (int a = 0; a < P.A; ++a) bc = bc * P.nS + beta[a];
    unsigned long long it = 0;
    for (int i = 0; i < d0; ++i) {
        const int b = beta[P.app[i]];
        const unsigned c = sb[(size_t)i * P.nS + b].cnt;
        const long long k = find_code(rec + ((size_t)i * P.nS + b) * P.O, (int)c, (uint32_t)(rho[i] * P.nQ + theta[i]));
        it = it * c + (unsigned long long)(k < 0 ? 0 : k);
    }
    return item_off[bc] + it;
}

// slots -> result[k] (exact local best), packed keys and (optionally) the next
// incumbent; executed by ONE block of 256 threads (sk/sx: 256-entry scratch)
CAM_DEVFN void reduce_slots_block(const DevProb &P, const Slot *slots, int nslots, int nlev, Slot *result,
                                   long long *keys, Slot *inc_out, const StageBound *sb, const OptRec *rec,
                                   const unsigned long long *item_off, int d0, int chunk_items, int flat_shift,
                                   unsigned long long *sk, unsigned long long *sx) {
    for (int k = 0; k < nlev; ++k) {
        unsigned long long bk = ~0ull, bx = ~0ull;
        for (int s = threadIdx.x; s < nslots; s += blockDim.x) {
            const Slot v = slots[(size_t)s * nlev + k];
            if (slot_less(v.key, v.x, bk, bx)) {
                bk = v.key;
                bx = v.x;
            }
        }
        sk[threadIdx.x] = bk;
        sx[threadIdx.x] = bx;
        __syncthreads();
        for (int st = blockDim.x / 2; st; st >>= 1) {
            if (threadIdx.x < st && slot_less(sk[threadIdx.x + st], sx[threadIdx.x + st], sk[threadIdx.x], sx[threadIdx.x])) {
                sk[threadIdx.x] = sk[threadIdx.x + st];
                sx[threadIdx.x] = sx[threadIdx.x + st];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            bk = sk[0];
            bx = sx[0];
            if (bk >= 0xFFFFFFFFull) {
                bk = 0xFFFFFFFFull;
                bx = ~0ull;
            }
            result[k].key = bk;
            result[k].x = bx;
            if (inc_out) {   // incumbent-cascade level: its packed key is never read (no item_of walk)
                inc_out[k].key = bk;
                inc_out[k].x = bx;
            }
            unsigned long long packed;
            if (bk == 0xFFFFFFFFull || inc_out) packed = ~0ull;
            else {
                unsigned long long low = (P.ntot <= (1ull << 32)) ? bx
                                         : flat_shift >= 0 ? (bx >> flat_shift)
                                         : item_of(P, sb, rec, item_off, d0, bx) / (unsigned long long)chunk_items;
                packed = (bk << 32) | (low & 0xFFFFFFFFull);
            }
            keys[k] = (long long)(packed ^ 0x8000000000000000ull);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- the search kernel
// One level-synchronous pass: warps pop parents (dynamic, `grab` at a time),
// hoist the parent into registers, lanes evaluate its children 32 at a time;
// surviving children at depth `flevel` are appended to the output frontier
// (generic inline depth-first descent when the frontier is full); leaves are
// scored exactly.
// dynamic shared memory of the search state (DFS stacks, walk control, warp bests)
template <int CM>
__host__ __device__ constexpr size_t search_smem_bytes() {
    return (size_t)SEARCH_WARPS * NMAX * sizeof(Node<CM>) + SEARCH_WARPS * sizeof(WarpCtl) +
           SEARCH_WARPS * sizeof(WarpBest);
}

// warp best + pruning bounds from the incumbent (start of a search level)
__device__ __forceinline__ void init_warp_best(const SearchArgs &S, WarpBest *wb, int lane) {
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
        wb->gpack = *(volatile unsigned long long *)&S.hdr->best_packed;
        if (nlev == 1 && wb->key[0] < 0xFFFFFFFFull)
            wb->gpack = min(wb->gpack, (wb->key[0] << 32) | min(wb->x[0] >> S.xshift, 0xFFFFFFFFull));
        // load floor with contention (min-resource, A = 1): every completion of a node
        // whose placed stages already throttle below the SMALLEST level fails LOAD
        float lm = 0.0f;
        if (S.policy == 1 && S.lam) {
            lm = __int_as_float(0x7f800000);
            for (int k = 0; k < nlev; ++k) lm = fminf(lm, S.lam[k * S.lam_stride]);
        }
        wb->lmin = lm;
        wb->mlev = S.policy == 1 && S.lam && nlev > 1 && S.lam_stride == 1;
        if (wb->mlev)
            for (int k = 0; k < nlev; ++k) wb->lam[k] = S.lam[k];
    }
    __syncwarp();
}

// Thread-per-parent mode of a heavy pass (many parents, one block of children
// each): lane l evaluates ALL children of parent e0 + l sequentially, reading the
// parent from the structure-of-arrays frontier with coalesced loads.  Same bounds
// and scoring as the warp mode (one load level for leaf passes); the lanes' bests
// are merged into the warp best at the end of the chunk.
template <int CM, int NS, int POLICY>
__device__ __forceinline__ void thread_chunk(const DevProb &P, const SearchArgs &S, const Frontier<CM> &in,
                                          const Frontier<CM> &outf, unsigned long long e0, unsigned live, int j,
                                          WarpBest *wb, int lane, Counters &cn, int G) {
    const int pol = POLICY == 2 ? S.policy : POLICY;   // 2: the policy is a runtime argument (shared code)
    // G lanes per parent (leaf passes, and inner passes with more than 32 options): lane l takes parent e0 + l / G
    // and its children sub, sub + G, ... (sub = l % G)
    const int n = P.n, nlev = S.nlev;
    const bool leaf = j == n - 1;
    const unsigned long long span = P.opow[n - 1 - j];
    unsigned long long bk = wb->key[0], bx = wb->x[0];   // lane-local best (leaf passes: one level)
    const int pl = lane / G, sub = lane % G;
    const bool mine = (live >> pl) & 1u;
#ifdef CAMELOT_FTRACE
    const bool tme = lane == 0;
    unsigned long long tt[4] = {0, 0, 0, 0};
    if (tme) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt[0]));
#endif
    {
        // dead lanes view node e0 (valid memory) and have no children
        const NodeSoA<CM> nd(in, e0 + (mine ? pl : 0));
        PCtx<CM, NS> c;
        load_ctx<CM, NS>(P, S, nd, j, c);
        const int bj = nd.b[P.app[j]];
        bool go_node = mine;
        if (go_node) {
            unsigned long long kl;
            if (pol == 0) kl = objkey_maxload(fminf(c.tub, fminf(sb_at(P, S, j, bj).maxNT, c.restT)));
            else {
                const int Ulb = c.U + (int)sb_at(P, S, j, bj).minNP + c.restU;
                kl = objkey_minres(max(c.u, (Ulb + P.R - 1) / P.R), Ulb);
            }
            go_node = can_win(kl, c.x * P.opow[n - j], wb, nlev, S.xshift,
                              nlev > 1 ? fminf(c.tub, fminf(sb_at(P, S, j, bj).maxNT, c.restT)) : __builtin_inff());
            if (pol == 1 && P.A == 1 && c.tub < wb->lmin) go_node = false;
        }
        const int cnt = go_node ? (int)sb_at(P, S, j, bj).cnt : 0;
        const OptRec *list = list_of(P, S, j, bj);
#ifdef CAMELOT_FTRACE
        if (tme) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt[1]));
#endif
        unsigned smask = 0u;   // surviving children of this lane's parent (inner passes)
        const int my_iters = cnt > sub ? (cnt - sub + G - 1) / G : 0;
        const int cntw = __reduce_max_sync(0xffffffffu, my_iters);
        for (int t = 0; t < cntw; ++t) {
            const int k = sub + t * G;
            const bool valid = t < my_iters;
            OptRec r;
            {
                const OptRec *src = list + (valid ? k : 0);
                const uint4 a = rec_chunk(src, 0), b = rec_chunk(src, 1);
                r.code = a.x;
                r.NP = a.y;
                r.N = a.z;
                r.pmul = a.w;
                r.NB = __uint_as_float(b.x);
                r.NT = __uint_as_float(b.y);
                r.bw = __uint_as_float(b.z);
                r.dur = __uint_as_float(b.w);
            }
            const unsigned long long x = c.x * (unsigned long long)P.O + r.code;
            bool go = valid;
            if (go) {
                unsigned long long kl;
                if (pol == 0) {
                    const float t = leaf ? fminf(c.tub, r.NT) : fminf(fminf(c.tub, r.NT), c.restT);
                    kl = objkey_maxload(t);
                } else {
                    const int Ulb = c.U + (int)r.NP + c.restU;
                    kl = objkey_minres(max(c.u, (Ulb + P.R - 1) / P.R), Ulb);
                }
                go = can_win(kl, x * span, wb, nlev, S.xshift,
                             nlev == 1 ? __builtin_inff() : leaf ? fminf(c.tub, r.NT) : fminf(fminf(c.tub, r.NT), c.restT));
                if (go && leaf && pol == 0) go = kl < bk || (kl == bk && x < bx);   // the lane's own best
                if (go && !leaf && c.rqsum - (int)r.NP < c.restU) go = false;
            }
            if (go && !(P.flags & F_COMM)) {
                const int aj = P.app[j];
                float lb = c.lpre < 0.0f ? r.dur : __fadd_rn(c.lpre, r.dur);
#pragma unroll
                for (int i = 0; i < NS; ++i)
                    if (i > j && i < n && P.app[i] == aj) lb = __fadd_rn(lb, c.dur[i]);
                go = lb <= P.qos[aj];
            }
            if (go) {
                const unsigned long long xs = x * span;
                if (xs >= S.hi || xs + span <= S.lo) go = false;
            }
            FastEval fe;
            fe.placed = false;
            if (go) fast_eval<CM, NS>(P, c, j, r, fe);
            const int jj = j;
            auto ntf = [&](int i) { return i < jj ? c.nt[i] : r.NT; };
            if (leaf) {
                if (!go) continue;
                cn.scored += 1;
                bool feas = fe.placed;
                if (feas) {
                    bool q = fe.lsum[0] <= P.qos[0];
                    if (P.A > 1) q &= fe.lsum[1] <= P.qos[1];
                    if (!q) cn.viol |= V_QOS;
                    feas = q;
                }
                cn.feasible += feas;
                if (!feas) continue;
                if (pol == 0) {
                    if (bk < 0xFFFFFFFFull) {
                        const float Tb = __uint_as_float(0xFFFFFFFFu - (unsigned)bk);
                        if (t_certainly_below<NS>(P, n - 1, fe.kap, ntf, Tb)) continue;
                    }
                    float T = __int_as_float(0x7f800000);
#pragma unroll
                    for (int i = 0; i < NS; ++i)
                        if (i < n) T = fminf(T, fe.kap[i] == 1.0f ? ntf(i) : __fdiv_rn(ntf(i), fe.kap[i]));
                    const unsigned long long key = objkey_maxload(T);
                    if (key < bk || (key == bk && x < bx)) {
                        bk = key;
                        bx = x;
                    }
                } else {
                    const unsigned long long key = objkey_minres(fe.u, fe.U);
                    if (key > wb->bound || !(key < bk || (key == bk && x < bx))) continue;
                    float tm0 = __int_as_float(0x7f800000), tm1 = __int_as_float(0x7f800000);
#pragma unroll
                    for (int i = 0; i < NS; ++i)
                        if (i < n) {
                            const float ti = fe.kap[i] == 1.0f ? ntf(i) : __fdiv_rn(ntf(i), fe.kap[i]);
                            if (P.app[i] == 0) tm0 = fminf(tm0, ti);
                            else tm1 = fminf(tm1, ti);
                        }
                    bool fk = tm0 >= S.lam[0];
                    if (P.A > 1) fk &= tm1 >= S.lam[1];
                    if ((P.flags & F_EQ2_BUDGET) && fe.u > S.y[c.bc * S.ystride + S.yoff]) fk = false;
                    if (fk) {
                        bk = key;
                        bx = x;
                    }
                }
                continue;
            }
            // ---- inner node: bounds with the current contention, then emit
            cn.nodes += go;
            bool sv = go && fe.placed;
            if (sv) {
                sv &= fe.lsum[0] <= P.qos[0];
                if (P.A > 1) sv &= fe.lsum[1] <= P.qos[1];
                if (sv && pol == 0 && wb->bound < 0xFFFFFFFFull) {
                    const float Tbest = __uint_as_float(0xFFFFFFFFu - (unsigned)wb->bound);
                    if (t_certainly_below<NS>(P, j, fe.kap, ntf, Tbest)) sv = false;
                }
                if (sv && pol == 1 && P.A == 1 && t_certainly_below<NS>(P, j, fe.kap, ntf, wb->lmin)) sv = false;
                if (sv && pol == 1) {
                    const int Ulb = fe.U + c.restU;
                    sv = (unsigned long long)objkey_minres(max(fe.u, (Ulb + P.R - 1) / P.R), Ulb) <=
                         (nlev == 1 ? wb->bound : level_bound(wb, nlev, fminf(fminf(c.tub, r.NT), c.restT)));
                }
            }
            if (sv && j + 1 == S.d0) sv = owns_child<CM>(P, S, nd, j, k);
            if (sv) smask |= 1u << t;   // emitted after the loop (t < 32: cnt <= 32)
        }
#ifdef CAMELOT_FTRACE
        __syncwarp();
        if (tme) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt[2]));
#endif
        // emission rounds: every lane emits its next survivor in the same round, into
        // consecutive slots (coalesced structure-of-arrays stores); the slots of all
        // rounds come from ONE warp-aggregated atomic (capacity checked by the caller)
        unsigned total = __popc(smask);
        for (int off = 16; off; off >>= 1) total += __shfl_xor_sync(0xffffffffu, total, off);
        unsigned long long fbase = 0;
        if (lane == 0 && total) fbase = atomicAdd(S.out_tail, (unsigned long long)total);
        fbase = __shfl_sync(0xffffffffu, fbase, 0);
        while (true) {
            const unsigned m = __ballot_sync(0xffffffffu, smask != 0u);
            if (!m) break;
            const unsigned long long rbase = fbase;
            fbase += __popc(m);
            if (smask) {
                const int k = sub + (__ffs(smask) - 1) * G;
                smask &= smask - 1u;
                OptRec r;
                {
                    const OptRec *src = list + k;
                    const uint4 a = rec_chunk(src, 0), b = rec_chunk(src, 1);
                    r.code = a.x;
                    r.NP = a.y;
                    r.N = a.z;
                    r.pmul = a.w;
                    r.NB = __uint_as_float(b.x);
                    r.NT = __uint_as_float(b.y);
                    r.bw = __uint_as_float(b.z);
                    r.dur = __uint_as_float(b.w);
                }
                const OptRec &full = list[k];
                const unsigned long long slot = rbase + __popc(m & ((1u << lane) - 1u));
                if (slot < S.out_cap)   // (an optimistic pass may overflow: it is then redone, see pass_body)
                    emit_child<CM, NS>(P, nd, c, j, r, full.p, full.W, full.As, k, outf, slot);
            }
        }
    }
    __syncwarp();
#ifdef CAMELOT_FTRACE
    if (tme) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt[3]));
        atomicMax(&S.hdr->dbg_tc[j][0], tt[1] - tt[0]);   // max over chunks of each phase
        atomicMax(&S.hdr->dbg_tc[j][1], tt[2] - tt[1]);
        atomicMax(&S.hdr->dbg_tc[j][2], tt[3] - tt[2]);
        atomicAdd(&S.hdr->dbg_tc[j][3], 1ull);
    }
#endif
    if (leaf) {   // merge the lanes' bests (converged)
        const bool imp = bk < 0xFFFFFFFFull && slot_less(bk, bx, wb->key[0], wb->x[0]);
        warp_improve(wb, 0, imp, bk, bx, lane);
        if (lane == 0) {
            if (wb->key[0] < wb->bound) {
                wb->bound = wb->key[0];
                atomicMin(&S.hdr->best_obj, (unsigned int)wb->key[0]);
            }
            publish_best(S, wb);
        }
        __syncwarp();
    }
}

// One level-synchronous pass (parents at depth S.level), executed by one warp
// of a persistent grid until the pass's work is exhausted.
template <int CM, int NS, int POLICY>
// Returns true when the pass ran in the thread-per-parent mode with more possible
// children than frontier slots (S.tmode_slack > 1): children that found no slot were
// dropped, so if the frontier overflowed (tail > capacity) the caller must redo the
// pass in the warp mode (S.no_tmode), which descends inline instead.
__device__ __forceinline__ bool pass_body(const DevProb &P, const SearchArgs &S, Node<CM> *stack, WarpCtl *ctl,
                                          WarpBest *wb, int lane, Counters &cn) {
    const int pol = POLICY == 2 ? S.policy : POLICY;   // 2: the policy is a runtime argument (shared code)
    const int nlev = S.nlev;
    const int n = P.n;
    const int jtop = S.level;
    const bool have_in = S.in_nodes != nullptr;
    const Frontier<CM> in{const_cast<uint32_t *>(reinterpret_cast<const uint32_t *>(S.in_nodes)), S.in_cap};
    const Frontier<CM> outf{reinterpret_cast<uint32_t *>(S.out_nodes), S.out_cap};
    const unsigned long long count = have_in ? min(*(volatile const unsigned long long *)S.in_count, S.in_cap)
                                        : (unsigned long long)P.nbc;
    // few parents (shallow passes): each block of 32 children is its own work item;
    // the blocks per parent follow the largest surviving option count of stage jtop
    int maxc = 0;
    for (int b = 0; b < P.nS; ++b) maxc = max(maxc, (int)sb_at(P, S, jtop, b).cnt);
    const int nblk = max(1, (maxc + 31) / 32);
    const int split = (count < 4ull * gridDim.x * SEARCH_WARPS) ? nblk : 1;
    const unsigned long long items = count * (unsigned long long)split;

#ifdef CAMELOT_FTRACE
    unsigned long long dbg_nb = 0;
    unsigned long long dbg_t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int dbg_item = 0;
    const bool dbg_me = blockIdx.x == 0 && threadIdx.x == 0;
#define PTM(k) \
    if (dbg_me && dbg_item <= 1 && dbg_t[k] == 0) dbg_t[k] = (unsigned long long)clock64();   /* SM cycles */
#else
#define PTM(k)
#endif
    PTM(0);
    // the first item of every warp is assigned statically (no atomic queueing at the
    // start of a pass: with few items the pass is latency bound); the rest is dynamic
    // Heavy passes (many parents, one block of children each): a warp takes 32
    // parents at a time and screens them lane-parallel against the current bound
    // from a few coalesced frontier words before copying any survivor.
    const unsigned long long nwarps = (unsigned long long)gridDim.x * SEARCH_WARPS;
    const bool compact_in = S.compact1 && jtop == 1;   // parents are (batch combo, stage-0 option) pairs
    const bool screen = S.prune && have_in && split == 1 && count >= 16ull * nwarps && !compact_in;
    // thread-per-parent mode: leaf passes with one level, or inner passes whose children
    // all fit in the output frontier (no inline descent possible in this mode)
    // (measured: leaf passes with more than 32 options per parent are faster in the warp mode)
    // leaf passes with more than 32 options per parent use G = 2 or 4 lanes per parent
    const bool leafp = S.flevel < 0 && jtop == n - 1 && nlev == 1;
    // lanes per parent (1..8): enough parent groups to occupy the warps (measured: a pass with
    // 7.5k parents kept only 234 of 1184 warps busy at one lane per parent), and for
    // leaf passes at most 32 children per lane
    int G = 1;
    while (G < 8 && count * (unsigned long long)(2 * G) <= 32ull * nwarps) G *= 2;
    if (leafp) G = max(G, maxc <= 32 ? 1 : maxc <= 64 ? 2 : maxc <= 128 ? 4 : 8);
    // inner passes: G lanes per parent also keep <= 32 children per lane (survivor mask)
    const int Gin = max(G, maxc <= 32 ? 1 : maxc <= 64 ? 2 : maxc <= 128 ? 4 : 8);
    const bool inner_t = S.flevel == jtop + 1 && maxc <= 32 * min(Gin, S.tmode_inner_gmax) &&
                         count * (unsigned long long)maxc <= S.out_cap * (unsigned long long)max(1, S.tmode_slack);
    if (!leafp && inner_t) G = Gin;
    const bool tmode = S.prune && have_in && split == 1 && 16ull * count >= (unsigned long long)S.tmode_min16 * nwarps && !getenv_tmode_off() &&
                       !S.no_tmode && !compact_in && ((leafp && maxc <= 32 * min(8, S.tmode_leaf_gmax)) || inner_t);
    const bool optimistic = tmode && !leafp && count * (unsigned long long)maxc > S.out_cap;
    const unsigned grab = tmode ? 32u / (unsigned)G : screen ? 8u : (unsigned)S.grab;
    const unsigned long long nw = nwarps * grab;
    unsigned long long e0 = ((unsigned long long)blockIdx.x * SEARCH_WARPS + (threadIdx.x >> 5)) * grab;
    // Parent prefetch (warp mode on a frontier, jtop >= 1 so stack[0] is free): the next
    // parent's node is copied asynchronously (cp.async) into stack[0] while the current
    // one is searched, and the next work item is popped one item ahead, so neither the
    // queue atomic nor the node copy sits on the warp's critical path.
    const bool pipe = have_in && jtop >= 1 && !tmode && !compact_in;
    unsigned long long pf_e = ~0ull;    // parent node in stack[0] (copy issued)
    unsigned long long top_e = ~0ull;   // parent node in stack[jtop]
    unsigned long long nx_raw = 0;      // lane 0: the popped-ahead item (nx_state == 1)
    int nx_state = 0;                   // 0 none, 1 popped (lane 0 holds it), 2 known (nx_e)
    unsigned long long nx_e = 0;
    auto prefetch = [&](unsigned long long e) {
        uint32_t *d = reinterpret_cast<uint32_t *>(&stack[0]);
        for (int w = lane; w < Frontier<CM>::WORDS; w += 32) cp_async4(d + w, in.base + (size_t)w * in.cap + e);
        cp_async_commit();
        pf_e = e;
    };
    auto parent_of = [&](unsigned long long item) { return split == 1 ? item : item / (unsigned)split; };
    bool first = true;
    while (true) {
        if (!first) {
            if (nx_state == 1) {
                nx_e = __shfl_sync(0xffffffffu, nx_raw, 0);
                nx_state = 2;
            }
            if (nx_state == 2) {
                e0 = nx_e;
                nx_state = 0;
            } else {
                if (nw >= items) break;   // every item was assigned statically: no queue round trip
                if (lane == 0) e0 = nw + atomicAdd(S.head, (unsigned long long)grab);
                e0 = __shfl_sync(0xffffffffu, e0, 0);
            }
        }
        first = false;
        // pop the next item now (its value is read later) -- only when items are plentiful:
        // holding an item ahead starves idle warps in passes with few items per warp
        if (pipe && e0 < items && nw < items && items >= 8ull * nwarps) {
            if (lane == 0) nx_raw = nw + atomicAdd(S.head, (unsigned long long)grab);
            nx_state = 1;
        }
#ifdef CAMELOT_FTRACE
        ++dbg_item;
#endif
        PTM(1);
        if (e0 >= items) break;
        // refresh the pruning bounds from the device-wide best: both loads issued
        // together; the warp mode applies them only after the parent copy (the two
        // round trips overlap)
        unsigned long long g_obj = ~0ull, g_pk = ~0ull;
        if (lane == 0) {
            g_obj = (unsigned long long)(*(volatile unsigned int *)&S.hdr->best_obj);
            g_pk = *(volatile unsigned long long *)&S.hdr->best_packed;
        }
        bool bounds_pending = true;
        auto apply_bounds = [&]() {
            if (lane == 0) {
                if (g_obj < wb->bound) wb->bound = g_obj;
                if (g_pk < wb->gpack) wb->gpack = g_pk;
            }
            __syncwarp();
            bounds_pending = false;
        };
        if (screen || tmode) apply_bounds();
        const unsigned long long e1 = min(e0 + (unsigned long long)grab, items);
        unsigned live = 0xffffffffu;
        if (screen || tmode) {
            const unsigned long long ei = e0 + lane;
            bool lv = ei < e1;
            if (lv) {
                auto word = [&](int w) { return __ldcg(in.base + (size_t)w * in.cap + ei); };
                const int Uq = (int)word(NODE_W(CM, U)), uq = (int)word(NODE_W(CM, u));
                const float tq = __uint_as_float(word(NODE_W(CM, tub)));
                const unsigned long long xq = (unsigned long long)word(NODE_W(CM, x)) |
                                              ((unsigned long long)word(NODE_W(CM, x) + 1) << 32);
                int bq[AMAX];
                bq[0] = (int)word(NODE_W(CM, b));
                bq[AMAX - 1] = (int)word(NODE_W(CM, b) + AMAX - 1);
                float rT = __int_as_float(0x7f800000);
                int rU = 0;
                for (int i2 = jtop + 1; i2 < n; ++i2) {
                    const StageBound &bb = sb_at(P, S, i2, P.app[i2] ? bq[AMAX - 1] : bq[0]);   // (select: no local array)
                    rT = fminf(rT, bb.maxNT);
                    rU += (int)bb.minNP;
                }
                const StageBound &bj = sb_at(P, S, jtop, P.app[jtop] ? bq[AMAX - 1] : bq[0]);
                unsigned long long kl;
                if (pol == 0) kl = objkey_maxload(fminf(tq, fminf(bj.maxNT, rT)));
                else {
                    const int Ulb = Uq + (int)bj.minNP + rU;
                    kl = objkey_minres(max(uq, (Ulb + P.R - 1) / P.R), Ulb);
                }
                lv = can_win(kl, xq * P.opow[n - jtop], wb, nlev, S.xshift, nlev > 1 ? fminf(tq, fminf(bj.maxNT, rT)) : __builtin_inff());
            }
            live = __ballot_sync(0xffffffffu, lv);
        }
        if (tmode) {
            thread_chunk<CM, NS, POLICY>(P, S, in, outf, e0, live, jtop, wb, lane, cn, G);
            continue;
        }
        for (unsigned long long it = e0; it < e1; ++it) {
            if (!((live >> (unsigned)(it - e0)) & 1u)) continue;
            if (screen && it > e0) {   // refresh the bounds per parent
                if (lane == 0) {
                    g_obj = (unsigned long long)(*(volatile unsigned int *)&S.hdr->best_obj);
                    g_pk = *(volatile unsigned long long *)&S.hdr->best_packed;
                }
                apply_bounds();
            }
            const unsigned long long e = split == 1 ? it : it / (unsigned)split;
            const int blk = split == 1 ? 0 : (int)(it % (unsigned)split);
            __syncwarp();   // the previous item's readers of the stack are done (WAR)
            if (!have_in) {
                build_root<CM>(P, (int)e, stack[0], lane);
                if (lane < NMAX) stack[0].kidx[lane] = 0;
                __syncwarp();
            } else if (pipe) {
                if (top_e != e) {   // (consecutive blocks of one parent reuse stack[jtop])
                    if (pf_e != e) prefetch(e);
                    cp_async_wait_all();
                    __syncwarp();
                    const uint32_t *src = reinterpret_cast<const uint32_t *>(&stack[0]);
                    uint32_t *dst = reinterpret_cast<uint32_t *>(&stack[jtop]);
                    for (int w = lane; w < Frontier<CM>::WORDS; w += 32) dst[w] = src[w];
                    __syncwarp();
                    top_e = e;
                    pf_e = ~0ull;
                }
                // prefetch the next parent: the next live one of this item, else the
                // first of the popped-ahead item
                unsigned long long e2 = ~0ull;
                for (unsigned long long it2 = it + 1; it2 < e1; ++it2)
                    if ((live >> (unsigned)(it2 - e0)) & 1u) {
                        e2 = parent_of(it2);
                        break;
                    }
                if (e2 == ~0ull && nx_state != 0) {
                    if (nx_state == 1) {
                        nx_e = __shfl_sync(0xffffffffu, nx_raw, 0);
                        nx_state = 2;
                    }
                    if (nx_e < items) e2 = parent_of(nx_e);
                }
                if (e2 != ~0ull && e2 != top_e && e2 != pf_e) prefetch(e2);
            } else if (compact_in) {   // rebuild the depth-1 node: the root, then stage 0's option
                const int bc = (int)__ldcg(in.base + e);
                const int k0 = (int)__ldcg(in.base + (size_t)in.cap + e);
                build_root<CM>(P, bc, stack[0], lane);
                if (lane < NMAX) stack[0].kidx[lane] = 0;
                __syncwarp();
                const OptRec *l0 = list_of(P, S, 0, stack[0].b[P.app[0]]);
                build_child<CM>(P, S, stack[0], 0, l0[k0], k0, stack[1], lane);
                __syncwarp();
            } else {
                copy_node<CM>(stack[jtop], in, e, lane);
            }
            if (bounds_pending) apply_bounds();
            PTM(2);
            {
                const int cnt0 = (int)sb_at(P, S, jtop, stack[jtop].b[P.app[jtop]]).cnt;
                __syncwarp();
                if (lane == 0) {
                    ctl->cur[jtop] = split > 1 ? blk * 32 : 0;
                    ctl->end[jtop] = split > 1 ? min(cnt0, blk * 32 + 32) : cnt0;
                    ctl->msk[jtop] = 0;
                }
                __syncwarp();
            }
            // ---- explicit-stack walk: normally one level (survivors go to the
            // frontier); inline descents (frontier full) use the same fast path
            int j = jtop;
            bool reload = true;
            PCtx<CM, NS> c;
            while (true) {
                const Node<CM> &nd = stack[j];
                const int bj = nd.b[P.app[j]];
                const OptRec *list = list_of(P, S, j, bj);
                if (reload) {
                    reload = false;
                    load_ctx<CM, NS>(P, S, nd, j, c);
                    PTM(3);
                    // re-check the node against the current bound (it may have tightened)
                    if (S.prune) {
                        unsigned long long kl;
                        if (pol == 0) kl = objkey_maxload(fminf(c.tub, fminf(sb_at(P, S, j, bj).maxNT, c.restT)));
                        else {
                            const int Ulb = c.U + (int)sb_at(P, S, j, bj).minNP + c.restU;
                            kl = objkey_minres(max(c.u, (Ulb + P.R - 1) / P.R), Ulb);
                        }
                        bool live = can_win(kl, c.x * P.opow[n - j], wb, nlev, S.xshift,
                                            nlev > 1 ? fminf(c.tub, fminf(sb_at(P, S, j, bj).maxNT, c.restT)) : __builtin_inff());
                        // T_i <= fl(N_i thr_i / kappa_i(now)) (kappa only grows): below the load floor -> dead
                        if (pol == 1 && P.A == 1 && c.tub < wb->lmin) live = false;
                        if (!live) {
                            __syncwarp();
                            if (lane == 0) {
                                ctl->cur[j] = ctl->end[j];
                                ctl->msk[j] = 0;
                            }
                            __syncwarp();
                        }
                    }
                }
                const unsigned pend = ctl->msk[j];
                if (pend) {
                    // inline descent into the next pending survivor
                    const int kk = __ffs(pend) - 1;
                    const int o2 = ctl->base[j] + kk;
                    __syncwarp();
                    if (lane == 0) ctl->msk[j] = pend & (pend - 1);
                    build_child<CM>(P, S, nd, j, list[o2], o2, stack[j + 1], lane);
                    ++j;
                    const int cntc = (int)sb_at(P, S, j, stack[j].b[P.app[j]]).cnt;
                    if (lane == 0) {
                        ctl->cur[j] = 0;
                        ctl->end[j] = cntc;
                        ctl->msk[j] = 0;
                    }
                    __syncwarp();
                    reload = true;
                    continue;
                }
                const int base = ctl->cur[j];
                if (base >= ctl->end[j]) {
                    if (j == jtop) break;
                    --j;
                    reload = true;
                    continue;
                }
                const int endj = ctl->end[j];
#ifdef CAMELOT_FTRACE
                ++dbg_nb;
#endif
                __syncwarp();
                if (lane == 0) {
                    ctl->base[j] = base;
                    ctl->cur[j] = base + 32;
                }
                __syncwarp();
                const bool leaf = j == n - 1;
                const unsigned long long span = P.opow[n - 1 - j];
                const int opt = base + lane;
                const bool valid = opt < endj;
                OptRec r;
                uint4 cold = make_uint4(0u, 0u, 0u, 0u);   // p, W, A*s, MEM (emission only)
                {
                    const OptRec *src = list + (valid ? opt : base);
                    const uint4 a = rec_chunk(src, 0), b = rec_chunk(src, 1);
                    if (!leaf) cold = rec_chunk(src, 2);
                    r.code = a.x;
                    r.NP = a.y;
                    r.N = a.z;
                    r.pmul = a.w;
                    r.NB = __uint_as_float(b.x);
                    r.NT = __uint_as_float(b.y);
                    r.bw = __uint_as_float(b.z);
                    r.dur = __uint_as_float(b.w);
                }
                const unsigned long long x = c.x * (unsigned long long)P.O + r.code;
                bool go = valid;
                // cheap exact bounds before the placement
                if (S.prune && go) {
                    // prune only when the subtree cannot hold the answer (ties by index)
                    unsigned long long kl;
                    if (pol == 0) {
                        const float t = leaf ? fminf(c.tub, r.NT) : fminf(fminf(c.tub, r.NT), c.restT);
                        kl = objkey_maxload(t);
                    } else {
                        const int Ulb = c.U + (int)r.NP + c.restU;
                        kl = objkey_minres(max(c.u, (Ulb + P.R - 1) / P.R), Ulb);
                    }
                    go = can_win(kl, x * span, wb, nlev, S.xshift,
                                 nlev == 1 ? __builtin_inff() : leaf ? fminf(c.tub, r.NT) : fminf(fminf(c.tub, r.NT), c.restT));
                    if (go && !leaf && c.rqsum - (int)r.NP < c.restU) go = false;
                }
                // QoS lower bound before placement: L_j >= dur, placed stages' L
                // only grow, unplaced stages >= their minimum duration (ordered sum)
                if (S.prune && go && !(P.flags & F_COMM)) {
                    const int aj = P.app[j];
                    float lb = c.lpre < 0.0f ? r.dur : __fadd_rn(c.lpre, r.dur);
#pragma unroll
                    for (int i = 0; i < NS; ++i)
                        if (i > j && i < n && P.app[i] == aj) lb = __fadd_rn(lb, c.dur[i]);
                    go = lb <= P.qos[aj];
                }
                // canonical index range of the child's subtree
                if (go) {
                    const unsigned long long xs = x * span;
                    if (xs >= S.hi || xs + span <= S.lo) go = false;
                }
                FastEval fe;
                fe.placed = false;
                if (go) fast_eval<CM, NS>(P, c, j, r, fe);
                PTM(4);
                if (leaf) {
                    // violation diagnostics are exact (and computed) only in flat mode
                    if (!S.prune && go && !fe.placed) cn.viol |= place_fail_bits<CM>(P, nd, list[opt]);
                    const int jj = j;
                    auto ntf = [&](int i) { return i < jj ? c.nt[i] : r.NT; };
                    score_leaf<POLICY, NS>(P, S, wb, lane, go, fe.placed, fe.lsum, fe.kap, ntf, fminf(c.tub, r.NT),
                                           fe.u, fe.U, c.bc, x, cn);
                    continue;
                }
                // ---- inner: bounds with the current contention
                cn.nodes += go;
                bool sv = go && fe.placed;
                if (sv && S.prune) {
                    sv &= fe.lsum[0] <= P.qos[0];
                    if (P.A > 1) sv &= fe.lsum[1] <= P.qos[1];
                    if (sv && pol == 0 && wb->bound < 0xFFFFFFFFull) {
                        const float Tbest = __uint_as_float(0xFFFFFFFFu - (unsigned)wb->bound);
                        const int jj = j;
                        auto ntf2 = [&](int i) { return i < jj ? c.nt[i] : r.NT; };
                        if (t_certainly_below<NS>(P, j, fe.kap, ntf2, Tbest)) sv = false;
                    }
                    if (sv && pol == 1 && P.A == 1) {
                        const int jj = j;
                        auto ntf3 = [&](int i) { return i < jj ? c.nt[i] : r.NT; };
                        if (t_certainly_below<NS>(P, j, fe.kap, ntf3, wb->lmin)) sv = false;
                    }
                    if (sv && pol == 1) {
                        const int Ulb = fe.U + c.restU;
                        sv = (unsigned long long)objkey_minres(max(fe.u, (Ulb + P.R - 1) / P.R), Ulb) <=
                             (nlev == 1 ? wb->bound : level_bound(wb, nlev, fminf(fminf(c.tub, r.NT), c.restT)));
                    }
                }
                if (sv && j + 1 == S.d0) sv = owns_child<CM>(P, S, nd, j, opt);
                unsigned m = __ballot_sync(0xffffffffu, sv);
                if (m && j + 1 == S.flevel) {
                    // every surviving lane emits its own child into the frontier
                    unsigned long long fbase = 0;
                    if (lane == 0) fbase = atomicAdd(S.out_tail, (unsigned long long)__popc(m));
                    fbase = __shfl_sync(0xffffffffu, fbase, 0);
                    const unsigned long long slot = fbase + __popc(m & ((1u << lane) - 1u));
                    const bool fits = sv && slot < S.out_cap;
                    if (fits) {
                if (S.compact1 && j == 0) {   // compact depth-1 child: (batch combo, option of stage 0)
                    outf.put(0, slot, (uint32_t)c.bc);
                    outf.put(1, slot, (uint32_t)opt);
                } else {
                    emit_child<CM, NS>(P, nd, c, j, r, cold.x, cold.y, cold.z, opt, outf, slot);
                }
            }
                    PTM(5);
                    m = __ballot_sync(0xffffffffu, sv && !fits);   // frontier full: descend inline
                }
                __syncwarp();
                if (lane == 0) ctl->msk[j] = m;
                __syncwarp();
            }
            PTM(6);
        }
    }
    if (pipe) {   // no copy may still be in flight into stack[0] when the pass ends
        cp_async_wait_all();
        __syncwarp();
    }
    PTM(7);
#ifdef CAMELOT_FTRACE
    if (dbg_me)
        for (int k = 1; k < 8; ++k) trace_value(S.hdr, 112 + k, dbg_t[k] ? dbg_t[k] - dbg_t[0] : 0);
    if (lane == 0 && dbg_nb) {
        atomicAdd(&S.hdr->dbg_batches[jtop], dbg_nb);
        atomicMax(&S.hdr->dbg_maxb[jtop], dbg_nb);
    }
#endif
    return optimistic;
}

// End of a search level for one CTA: merge the warps' bests into the CTA's slot
// and add the counters (one atomic per CTA and non-zero counter).
template <int CM>
__device__ __forceinline__ void cta_finish(const SearchArgs &S, WarpBest *wb_all, int lane, int wid, Counters &cn) {
    const int nlev = S.nlev;
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
    // counters: warp -> CTA (shared) -> one atomic per CTA and non-zero counter
    for (int off = 16; off; off >>= 1) {
        cn.scored += __shfl_xor_sync(0xffffffffu, cn.scored, off);
        cn.feasible += __shfl_xor_sync(0xffffffffu, cn.feasible, off);
        cn.nodes += __shfl_xor_sync(0xffffffffu, cn.nodes, off);
        cn.viol |= __shfl_xor_sync(0xffffffffu, cn.viol, off);
    }
    __shared__ unsigned long long cta_cnt[SEARCH_WARPS][3];
    __shared__ unsigned cta_viol[SEARCH_WARPS];
    if (lane == 0) {
        cta_cnt[wid][0] = cn.scored;
        cta_cnt[wid][1] = cn.feasible;
        cta_cnt[wid][2] = cn.nodes;
        cta_viol[wid] = cn.viol;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long sc = 0, fe = 0, no = 0;
        unsigned vi = 0;
        for (int w = 0; w < SEARCH_WARPS; ++w) {
            sc += cta_cnt[w][0];
            fe += cta_cnt[w][1];
            no += cta_cnt[w][2];
            vi |= cta_viol[w];
        }
        if (sc) {
            atomicAdd(&S.hdr->n_scored, sc);
            atomicAdd(&S.hdr->cum_scored, sc);
        }
        if (fe) atomicAdd(&S.hdr->n_feasible, fe);
        if (no) {
            atomicAdd(&S.hdr->n_nodes, no);
            atomicAdd(&S.hdr->cum_nodes, no);
        }
        if (vi) atomicOr(&S.hdr->viol_or, vi);
    }
}

template <int CM, int NS, int POLICY>
__global__ void __launch_bounds__(SEARCH_THREADS, SEARCH_MINB)
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
    init_warp_best(S, wb, lane);
    Counters cn = {0, 0, 0, 0};
    pass_body<CM, NS, POLICY>(P, S, stack, ctl, wb, lane, cn);
    cta_finish<CM>(S, wb_all, lane, wid, cn);
    // ---- fused reduction of the search: the last CTA to finish reduces all slots
    if (S.reduce_last) {
        __shared__ int is_last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) is_last = atomicAdd(&S.hdr->done_ctas, 1u) == gridDim.x - 1;
        __syncthreads();
        if (is_last) {
            __threadfence();
            unsigned long long *sk = reinterpret_cast<unsigned long long *>(smem_raw);
            reduce_slots_block(P, S.slots, gridDim.x, nlev, S.result, S.keys, S.inc_out, S.sb, S.rec, S.item_off,
                               S.d0, S.chunk_items, -1, sk, sk + SEARCH_THREADS);
            if (threadIdx.x == 0) S.hdr->done_ctas = 0;
        }
    }
}

}  // namespace cam
