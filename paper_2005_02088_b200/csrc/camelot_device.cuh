// camelot_device.cuh -- device-side data structures and the scoring arithmetic
// of the allocation search (sm_100a).  Everything here follows DESIGN.md
// "Scoring definition" (placement PAPER.md L929-945; constraints Eq. 1 / Eq. 3
// L825-836, L859-869; contention reading R17).  Floating point uses explicit
// round-to-nearest intrinsics so that no FMA contraction can happen.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Non-inline device functions of the shared headers: private copies in the
// translation units that only instantiate the search templates (camelot_inst_*.cu).
#ifdef CAMELOT_INST_TU
#define CAM_DEVFN static __device__
#else
#define CAM_DEVFN __device__
#endif

namespace cam {

constexpr int NMAX = 8;      // stages
constexpr int AMAX = 2;      // applications
constexpr int LMAX = 64;     // load levels
constexpr int TRACE_MAX = 256;

constexpr uint32_t F_NO_BW_CAP = 1u, F_NO_CONTENTION = 2u, F_SAT = 4u, F_PAPER_GLOBAL = 8u,
                   F_EQ2_BUDGET = 16u, F_NO_FILTER = 32u, F_COMM = 64u;
constexpr uint32_t V_QUOTA = 1u, V_INST = 2u, V_MEM = 4u, V_BW = 8u, V_QOS = 16u,
                   V_LOAD = 32u, V_EQ2 = 64u;

// Problem image passed BY VALUE to every kernel (lives in the constant bank).
struct DevProb {
    int A, n, nQ, nS, Rmax, C, R, I, O, nbc;   // O = Rmax*nQ options per stage, nbc = nS^A
    uint32_t FM, flags;
    float BW, invBW, G;
    float qos[AMAX];
    int app[NMAX];
    int first_of_app[AMAX], last_of_app[AMAX];
    uint32_t W[NMAX], Am[NMAX];
    float gamma[NMAX], cflop[NMAX];
    unsigned long long ntot;
    unsigned long long opow[NMAX + 1];       // O^k
    // NEXT-2 (F_COMM, R29): hand-over of edge i -> i+1 at batch s: local (both stages
    // entirely on one and the same GPU) ipc_ms, else fl(fl(comm_mb[i] * s) * inv_link)
    float comm_mb[NMAX];
    float inv_link, ipc_ms;
    const float4 *tab;                       // [n][nS][nQ] (dur, thr, bw, 0)
    const int *Q, *S;                        // grids
};

// One option (N, theta) of stage i at batch index b, precomputed by the filter kernel.
struct __align__(16) OptRec {
    // hot 32 bytes (two 16-byte loads in the search)
    uint32_t code;     // option code o = rho*nQ + theta
    uint32_t NP;       // N * p
    uint32_t N;        // replicas
    uint32_t pmul;     // ceil(2^16 / p): floor(a/p) = (a*pmul)>>16 for a <= 127
    float NB;          // fl(N * bw)
    float NT;          // fl(N * thr)
    float bw;          // bw of one replica
    float dur;         // duration (ms)
    // cold
    uint32_t p;        // quota (%)
    uint32_t W;        // W_i
    uint32_t As;       // A_i * s
    uint32_t MEM;      // W_i + N*A_i*s  (MiB)
};

// Per (stage, batch) bounds over the surviving options.
struct __align__(16) StageBound {
    float mindur;      // min duration over surviving options
    float maxNT;       // max fl(N*thr) over surviving options
    uint32_t minNP;    // min N*p over surviving options
    uint32_t cnt;      // surviving options
};

// Device header at the start of the workspace.
struct DevHeader {
    unsigned long long chunk_counter;
    unsigned long long n_scored, n_feasible, n_nodes;
    unsigned int best_obj;          // dynamic incumbent objective key (32-bit, smaller better)
    unsigned int viol_or;
    unsigned int done_ctas;         // last-CTA detection of the leaf pass (fused reduction)
    unsigned int filt_done;         // last-CTA detection of the filter (fused item offsets)
    unsigned long long items_total; // number of depth-d0 items of the (filtered) space
    unsigned long long nchunks;
    unsigned long long t_search_ns;
    unsigned int inc_passes;
    unsigned int pad[7];
    unsigned long long best_packed;      // (objective key << 32) | (index >> xshift), atomicMin (1 level)
    unsigned long long head[NMAX + 1];   // pop counter of pass j
    unsigned long long tail[NMAX + 1];   // size of the frontier at depth j (may exceed capacity)
    unsigned long long dbg_batches[NMAX + 1], dbg_maxb[NMAX + 1], dbg_tend[NMAX + 1], dbg_tc[NMAX + 1][4];   // profiling (CAMELOT_FTRACE)
    // cumulative over the incumbent cascade + main search of one call (not reset per pass)
    unsigned long long cum_scored, cum_nodes;
    // phase trace of the last search (camelot_trace): block 0 of every search-level
    // launch appends (tag << 48 | %globaltimer ns) after each grid barrier
    unsigned int trace_n, trace_pad;
    unsigned long long trace[TRACE_MAX];
};

__device__ __forceinline__ void trace_value(DevHeader *h, unsigned tag, unsigned long long v) {
    const unsigned i = h->trace_n;
    if (i < (unsigned)TRACE_MAX) h->trace[i] = ((unsigned long long)tag << 48) | (v & 0xFFFFFFFFFFFFull);
    h->trace_n = i + 1;
}
__device__ __forceinline__ void trace_mark(DevHeader *h, unsigned tag) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned i = h->trace_n;
    if (i < (unsigned)TRACE_MAX) h->trace[i] = ((unsigned long long)tag << 48) | (t & 0xFFFFFFFFFFFFull);
    h->trace_n = i + 1;
}

struct Slot {                      // (objective key, canonical index), smaller is better
    unsigned long long key, x;
};

__device__ __forceinline__ bool slot_less(unsigned long long ka, unsigned long long xa,
                                          unsigned long long kb, unsigned long long xb) {
    return ka < kb || (ka == kb && xa < xb);
}

__device__ __forceinline__ unsigned int objkey_maxload(float T) {
    return 0xFFFFFFFFu - __float_as_uint(T);
}
__device__ __forceinline__ unsigned int objkey_minres(int u, int U) {
    return ((unsigned)u << 24) | (unsigned)U;
}

// contention inflation for a stage with one-replica bandwidth bw, sensitivity
// gamma, on GPUs whose largest accumulated demand is dmax (reading R17; the max
// over hosting GPUs of a monotone function = the function of the max demand).
__device__ __forceinline__ float kappa_of(float dmax, float bw, float gamma, float invBW, uint32_t flags) {
    if (flags & F_NO_CONTENTION) return 1.0f;
    float d = __fsub_rn(dmax, bw);
    float t = __fmul_rn(d, invBW);
    float t2 = __fmul_rn(gamma, t);
    float k = __fadd_rn(1.0f, t2);
    if (flags & F_SAT) {
        float r = __fmul_rn(dmax, invBW);
        if (r > 1.0f) k = __fmul_rn(k, r);
    }
    return k;
}

// ---------------------------------------------------------------- bulk async copies (TMA engine)
// 1-D cp.async.bulk global -> shared with an mbarrier (sm_90+/sm_100a): one thread
// arms the barrier with the expected byte count and issues the copies; every thread
// waits on the barrier's phase.  Sizes and addresses are multiples of 16 bytes.
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // visible to the async proxy
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes, unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    }
}
// 4-byte asynchronous global -> shared copies (cp.async, L1-cached): the parent-node
// prefetch of the search passes; wait_all + a warp barrier before the data is read
__device__ __forceinline__ void cp_async4(void *dst_smem, const void *src_gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// generic-proxy writes (this or other threads, ordered by a barrier) before async-proxy
// accesses of the same memory (the bulk copy reads global records written by the filter,
// and overwrites shared memory read by the previous level)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

}  // namespace cam
