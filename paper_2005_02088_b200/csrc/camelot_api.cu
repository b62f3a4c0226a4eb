// camelot_api.cu -- host side of libcamelot.so: validation, workspace layout,
// launches and the C ABI declared in include/camelot.h.  All compute runs in
// the kernels of camelot_kernels.cuh / camelot_search.cuh; there is no CPU
// fallback (no device -> CAMELOT_ENODEV).
#include <cuda_runtime.h>

#include <cmath>
#include <cstddef>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/camelot.h"
#include "camelot_inst.cuh"
#include "camelot_sweep_args.h"

namespace cam {   // camelot_sweep.cu
bool sweep_supported(const DevProb &P, int policy, int nlev);
cudaError_t sweep_launch(const DevProb &P, const SweepArgs &A, int dev, cudaStream_t st);
}  // namespace cam

using namespace cam;

namespace {

thread_local std::string g_err = "";
std::atomic<unsigned long long> g_launches{0};
thread_local unsigned long long t_call_launches = 0;
// CUDA events around the main search kernel of the last call on this thread
struct EvPair {
    int dev = -1;
    cudaEvent_t a = nullptr, b = nullptr;
    bool armed = false;
};
thread_local EvPair t_ev;
thread_local EvPair t_ev_spare;   // camelot_plan_max_then_min: the first search's events
// camelot_plan_max_then_min: the second stream that scores the max-load plan while the
// min-resource search runs, and its fork / join events (per thread, per device)
struct SideStream {
    int dev = -1;
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
thread_local SideStream t_side;

// What the last camelot_search_local left in a workspace: camelot_finalize reads
// that state (local best, filter records, loads, Eq. 2 estimates), so it must be
// called with the same policy, levels, range, shard and problem size (camelot.h).
struct SearchRecord {
    int policy = -1, nlev = 0, rank = 0, world = 1;
    unsigned long long lo = 0, hi = 0, ntot = 0;
    uint32_t flags = 0;
    std::vector<float> loads;
};
std::mutex g_rec_mu;
std::unordered_map<const void *, SearchRecord> g_rec;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define COUNT_LAUNCH()               \
    do {                             \
        g_launches.fetch_add(1);     \
        ++t_call_launches;           \
    } while (0)

#define CU(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) return fail(CAMELOT_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

constexpr int MAXSLOTS = 4096;      // persistent CTAs (>= 148 SMs x resident CTAs)
constexpr int CHUNK_ITEMS = 64;

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
    size_t hdr, hdr2, tab, Q, S, rec, sb, item_off, lam, y, inc, result, keys, winner, rescan, plans, slots,
        front0, front1, side_w, side_h, total;
    int nlev;
    unsigned long long fcap;   // frontier capacity (nodes) of each ping-pong buffer
};

struct Dims {
    int A, n, nQ, nS, Rmax, C, O, nbc;
    unsigned long long ntot;
};

int check_problem(const camelot_problem *p, const camelot_cluster *c, Dims &d, bool check_table = true) {
    if (!p || !c) return fail(CAMELOT_EINVAL, "null problem or cluster");
    if (p->n_apps < 1 || p->n_apps > CAMELOT_MAX_APPS) return fail(CAMELOT_EINVAL, "n_apps must be 1 or 2");
    if (p->n_stages < 1 || p->n_stages > CAMELOT_MAX_STAGES) return fail(CAMELOT_EINVAL, "n_stages must be in 1..8");
    if (c->n_gpus < 1) return fail(CAMELOT_EINVAL, "n_gpus < 1");
    if (c->n_gpus > CAMELOT_MAX_GPUS) return fail(CAMELOT_ERANGE, "n_gpus > %d", CAMELOT_MAX_GPUS);
    if (c->quota_per_gpu < 1 || c->quota_per_gpu > 127) return fail(CAMELOT_EINVAL, "quota_per_gpu must be in 1..127");
    if (c->max_instances < 1) return fail(CAMELOT_EINVAL, "max_instances < 1");
    if (!(c->bw_gbs > 0.0f) || !std::isfinite(c->bw_gbs)) return fail(CAMELOT_EINVAL, "bw_gbs must be > 0");
    if (!(c->gflops > 0.0f) || !std::isfinite(c->gflops)) return fail(CAMELOT_EINVAL, "gflops must be > 0");
    if (c->mem_mib < 1 || c->mem_mib >= (1u << 21)) return fail(CAMELOT_ERANGE, "mem_mib must be in 1..2^21-1");
    if (p->max_replicas < 1 || p->max_replicas > CAMELOT_MAX_REPLICAS) return fail(CAMELOT_EINVAL, "max_replicas must be in 1..16");
    if (p->n_quota < 1 || p->n_quota > CAMELOT_MAX_QUOTAS) return fail(CAMELOT_EINVAL, "n_quota must be in 1..128");
    if (p->n_batch < 1 || p->n_batch > CAMELOT_MAX_BATCHES) return fail(CAMELOT_EINVAL, "n_batch must be in 1..64");
    if (!p->app_of_stage || !p->qos_ms || !p->quota_pct || !p->batch || !p->table || !p->weights_mib ||
        !p->act_mib_per_item || !p->gflop_per_item || !p->bw_sensitivity)
        return fail(CAMELOT_EINVAL, "null array in problem");
    if (p->flags & CAMELOT_F_COMM) {
        if (p->flags & CAMELOT_F_PAPER_GLOBAL) return fail(CAMELOT_EINVAL, "COMM needs a placement (not with PAPER_GLOBAL)");
        if (!p->comm_mb_per_item) return fail(CAMELOT_EINVAL, "COMM needs comm_mb_per_item");
        if (!(c->link_gbs > 0.0f) || !std::isfinite(c->link_gbs)) return fail(CAMELOT_EINVAL, "link_gbs must be > 0");
        if (!(c->ipc_ms >= 0.0f) || !std::isfinite(c->ipc_ms)) return fail(CAMELOT_EINVAL, "ipc_ms must be >= 0");
        for (int i = 0; i < p->n_stages; ++i)
            if (!(p->comm_mb_per_item[i] >= 0.0f) || !std::isfinite(p->comm_mb_per_item[i]))
                return fail(CAMELOT_EINVAL, "comm_mb_per_item[%d] must be finite and >= 0", i);
    }
    for (int k = 0; k < p->n_quota; ++k) {
        if (p->quota_pct[k] < 1 || p->quota_pct[k] > c->quota_per_gpu) return fail(CAMELOT_EINVAL, "quota_pct[%d] not in [1,R]", k);
        if (k && p->quota_pct[k] <= p->quota_pct[k - 1]) return fail(CAMELOT_EINVAL, "quota grid not strictly ascending");
    }
    for (int k = 0; k < p->n_batch; ++k) {
        if (p->batch[k] < 1) return fail(CAMELOT_EINVAL, "batch[%d] < 1", k);
        if (k && p->batch[k] <= p->batch[k - 1]) return fail(CAMELOT_EINVAL, "batch grid not strictly ascending");
    }
    for (int i = 0; i < p->n_stages; ++i) {
        const int a = p->app_of_stage[i];
        if (a < 0 || a >= p->n_apps) return fail(CAMELOT_EINVAL, "app_of_stage[%d] out of range", i);
        if (i && a < p->app_of_stage[i - 1]) return fail(CAMELOT_EINVAL, "app_of_stage not non-decreasing");
        if (!(p->bw_sensitivity[i] >= 0.0f) || !std::isfinite(p->bw_sensitivity[i])) return fail(CAMELOT_EINVAL, "bw_sensitivity[%d] < 0", i);
        if (!(p->gflop_per_item[i] >= 0.0f) || !std::isfinite(p->gflop_per_item[i])) return fail(CAMELOT_EINVAL, "gflop_per_item[%d] < 0", i);
        const unsigned long long need = (unsigned long long)p->weights_mib[i] +
            (unsigned long long)p->max_replicas * p->act_mib_per_item[i] * (unsigned long long)p->batch[p->n_batch - 1];
        if (need >= (1ull << 31)) return fail(CAMELOT_ERANGE, "stage %d memory footprint overflows 2^31 MiB", i);
    }
    if (p->app_of_stage[0] != 0 || p->app_of_stage[p->n_stages - 1] != p->n_apps - 1)
        return fail(CAMELOT_EINVAL, "every application needs at least one stage");
    for (int a = 0; a < p->n_apps; ++a)
        if (!(p->qos_ms[a] > 0.0f) || !std::isfinite(p->qos_ms[a])) return fail(CAMELOT_EINVAL, "qos_ms[%d] must be > 0", a);
    // (the table values are only read when they are uploaded: a RESIDENT call reuses the
    // image that camelot_upload validated)
    const size_t ne = check_table ? (size_t)p->n_stages * p->n_batch * p->n_quota : 0;
    for (size_t e = 0; e < ne; ++e) {
        const float *t = p->table + 4 * e;
        if (!std::isfinite(t[0]) || !std::isfinite(t[1]) || !std::isfinite(t[2]))
            return fail(CAMELOT_EINVAL, "non-finite table entry %zu", e);
        if (!(t[0] > 0.0f) || !(t[1] > 0.0f) || !(t[2] >= 0.0f))
            return fail(CAMELOT_EINVAL, "table entry %zu: need dur > 0, thr > 0, bw >= 0", e);
    }
    if ((unsigned long long)p->max_replicas * p->n_stages * c->quota_per_gpu >= (1ull << 24))
        return fail(CAMELOT_ERANGE, "quota sum exceeds the 24-bit key field");
    d.A = p->n_apps;
    d.n = p->n_stages;
    d.nQ = p->n_quota;
    d.nS = p->n_batch;
    d.Rmax = p->max_replicas;
    d.C = c->n_gpus;
    d.O = d.Rmax * d.nQ;
    d.nbc = 1;
    for (int a = 0; a < d.A; ++a) d.nbc *= d.nS;
    long double t = 1;
    for (int a = 0; a < d.A; ++a) t *= d.nS;
    for (int i = 0; i < d.n; ++i) t *= d.O;
    if (t >= 9.2e18L) return fail(CAMELOT_ERANGE, "candidate space >= 2^63");
    unsigned long long nt = 1;
    for (int a = 0; a < d.A; ++a) nt *= (unsigned long long)d.nS;
    for (int i = 0; i < d.n; ++i) nt *= (unsigned long long)d.O;
    d.ntot = nt;
    return CAMELOT_OK;
}

int check_loads(const camelot_problem *p, const float *loads, int n_loads) {
    if (n_loads < 1 || n_loads > CAMELOT_MAX_LOADS) return fail(CAMELOT_EINVAL, "n_loads must be in 1..64");
    if (!loads) return fail(CAMELOT_EINVAL, "null load_qps");
    for (int k = 0; k < n_loads * p->n_apps; ++k)
        if (!(loads[k] > 0.0f) || !std::isfinite(loads[k])) return fail(CAMELOT_EINVAL, "load_qps[%d] must be > 0", k);
    return CAMELOT_OK;
}

Layout make_layout(const Dims &d, int nlev) {
    Layout L;
    L.nlev = nlev < 1 ? 1 : nlev;
    size_t o = 0;
    auto put = [&](size_t bytes) {
        size_t at = o;
        o += al(bytes);
        return at;
    };
    L.hdr = put(sizeof(DevHeader));
    L.hdr2 = put(sizeof(DevHeader));
    L.tab = put((size_t)d.n * d.nS * d.nQ * sizeof(float4));
    L.Q = put((size_t)d.nQ * sizeof(int));
    L.S = put((size_t)d.nS * sizeof(int));
    L.rec = put((size_t)d.n * d.nS * d.O * sizeof(OptRec));
    L.sb = put((size_t)d.n * d.nS * sizeof(StageBound));
    L.item_off = put((size_t)(d.nbc + 1) * sizeof(unsigned long long));
    L.lam = put((size_t)CAMELOT_MAX_LOADS * CAMELOT_MAX_APPS * sizeof(float));
    L.y = put((size_t)d.nbc * L.nlev * sizeof(int));
    L.inc = put((size_t)L.nlev * sizeof(Slot));
    L.result = put((size_t)L.nlev * sizeof(Slot));
    L.keys = put((size_t)L.nlev * sizeof(long long));
    L.winner = put((size_t)L.nlev * sizeof(Slot));
    L.rescan = put((size_t)L.nlev * sizeof(unsigned long long));
    L.plans = put((size_t)(L.nlev + 1) * sizeof(camelot_plan));   // + the max-load plan of camelot_plan_max_then_min
    L.side_w = put(sizeof(Slot));          // camelot_plan_max_then_min: the max-load winner and
    L.side_h = put(sizeof(DevHeader));     // counters, scored on a second stream
    L.slots = put((size_t)MAXSLOTS * L.nlev * sizeof(Slot));
    // frontier of placement-state nodes: as many as there are leaf parents in the
    // whole space, clamped to [256, 2^23] (overflow falls back to inline DFS).  2^23
    // (3.6 GB per buffer for 8 GPUs, 7 GB per C4 workspace against 180 GB of HBM): the
    // thread-per-parent mode needs room for every child of a pass (measured: C4b's
    // 271k-parent pass ran in the warp mode at 2^20, 5.07 ms per step, 2.54 ms at 2^21;
    // a harder C4-shaped instance (tools/cascade_probe3.py, C4x3) 14.7 ms at 2^21, 5.4 ms
    // at 2^23; C4 unchanged)
    const size_t nb = d.C > 8 ? sizeof(Node<16>) : d.C > 4 ? sizeof(Node<8>) : sizeof(Node<4>);
    long double parents = (long double)d.ntot / (long double)d.O;
    // (testing knob CAMELOT_FRONTIER_MAX moves the clamp)
    const long double fmax = getenv("CAMELOT_FRONTIER_MAX") ? (long double)atof(getenv("CAMELOT_FRONTIER_MAX"))
                                                            : (long double)(1u << 23);
    L.fcap = (unsigned long long)std::max(256.0L, std::min(fmax, parents));
    // testing knob: force a small frontier to exercise the inline-descent fallback
    if (const char *cap = getenv("CAMELOT_FRONTIER_CAP")) {
        const unsigned long long v = strtoull(cap, nullptr, 10);
        if (v >= 1 && v < L.fcap) L.fcap = v;
    }
    L.front0 = put((size_t)L.fcap * nb);
    L.front1 = put((size_t)L.fcap * nb);
    L.total = o;
    return L;
}
size_t slots_off(const Layout &L) { return L.slots; }

int device_ok(const camelot_exec *ex) {
    if (!ex) return fail(CAMELOT_EINVAL, "null exec");
    int nd = 0;
    cudaError_t e = cudaGetDeviceCount(&nd);
    if (e != cudaSuccess || nd == 0) {
        cudaGetLastError();
        return fail(CAMELOT_ENODEV, "no CUDA device (there is no CPU fallback)");
    }
    if (ex->device < 0 || ex->device >= nd) return fail(CAMELOT_EINVAL, "bad device ordinal %d", ex->device);
    CU(cudaSetDevice(ex->device));
    if (ex->world < 1 || ex->rank < 0 || ex->rank >= ex->world) return fail(CAMELOT_EINVAL, "bad rank/world");
    if (!ex->workspace) return fail(CAMELOT_EINVAL, "null workspace");
    return CAMELOT_OK;
}

DevProb make_devprob(const camelot_problem *p, const camelot_cluster *c, const Dims &d, char *ws, const Layout &L) {
    DevProb P;
    memset(&P, 0, sizeof(P));
    P.A = d.A;
    P.n = d.n;
    P.nQ = d.nQ;
    P.nS = d.nS;
    P.Rmax = d.Rmax;
    P.C = d.C;
    P.R = c->quota_per_gpu;
    P.I = c->max_instances;
    P.O = d.O;
    P.nbc = d.nbc;
    P.FM = c->mem_mib;
    P.flags = p->flags;
    P.BW = c->bw_gbs;
    volatile float one = 1.0f;
    P.invBW = one / c->bw_gbs;   // IEEE binary32 division, as the oracle
    P.G = c->gflops;
    for (int a = 0; a < d.A; ++a) {
        P.qos[a] = p->qos_ms[a];
        P.first_of_app[a] = -1;
    }
    for (int i = 0; i < d.n; ++i) {
        const int a = p->app_of_stage[i];
        P.app[i] = a;
        if (P.first_of_app[a] < 0) P.first_of_app[a] = i;
        P.last_of_app[a] = i;
        P.W[i] = p->weights_mib[i];
        P.Am[i] = p->act_mib_per_item[i];
        P.gamma[i] = p->bw_sensitivity[i];
        P.cflop[i] = p->gflop_per_item[i];
    }
    volatile float link = (p->flags & CAMELOT_F_COMM) ? c->link_gbs : 1.0f;
    P.inv_link = one / link;   // IEEE binary32 division, as the oracle
    P.ipc_ms = (p->flags & CAMELOT_F_COMM) ? c->ipc_ms : 0.0f;
    for (int i = 0; i < d.n; ++i) P.comm_mb[i] = (p->flags & CAMELOT_F_COMM) ? p->comm_mb_per_item[i] : 0.0f;
    P.ntot = d.ntot;
    P.opow[0] = 1;
    for (int k = 1; k <= NMAX; ++k) P.opow[k] = P.opow[k - 1] * (unsigned long long)d.O;
    P.tab = reinterpret_cast<const float4 *>(ws + L.tab);
    P.Q = reinterpret_cast<const int *>(ws + L.Q);
    P.S = reinterpret_cast<const int *>(ws + L.S);
    return P;
}

struct Ctx {
    Dims d;
    Layout L;
    DevProb P;
    char *ws;
    cudaStream_t st;
    int nslots[2][2];   // [cm16][policy]
    int d0;
    int cm16;
    bool naive;
};

template <int CM>
size_t search_smem() {
    return (size_t)SEARCH_WARPS * NMAX * sizeof(Node<CM>) + SEARCH_WARPS * sizeof(WarpCtl) +
           SEARCH_WARPS * sizeof(WarpBest);
}

// compile-time widths: positions CM in {4, 8, 16} >= C, stages NS in {4, 6, 8} >= n
int cm_bucket(int C) { return C <= 4 ? 4 : C <= 8 ? 8 : 16; }
int ns_bucket(int n) { return n <= 4 ? 4 : n <= 6 ? 6 : 8; }

std::mutex g_attr_mu;
struct GridKey {
    int dev, cm, ns, pol;
};
std::vector<std::pair<GridKey, int>> g_grid_cache;

template <int CM, int NS, int POL>
int grid_for(int dev, int &grid) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    for (auto &e : g_grid_cache)
        if (e.first.dev == dev && e.first.cm == CM && e.first.ns == NS && e.first.pol == POL) {
            grid = e.second;
            return CAMELOT_OK;
        }
    const size_t sm = search_smem<CM>();
    int per = 0, nsm = 0;
    CU((k_search_occupancy<CM, NS, POL>(sm, &per)));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    grid = std::max(1, std::min(MAXSLOTS, per * nsm));
    g_grid_cache.push_back({GridKey{dev, CM, NS, POL}, grid});
    return CAMELOT_OK;
}

int choose_d0(const Dims &d) {
    if (d.n < 2) return 0;   // single-stage problems: items are whole candidates (handled by flat path)
    int d0 = 1;
    long double items = (long double)d.nbc * d.O;
    while (d0 < d.n - 1 && items < 16384.0L) {
        ++d0;
        items *= d.O;
    }
    return d0;
}

int setup(const camelot_problem *p, const camelot_cluster *c, const camelot_exec *ex, int nlev, Ctx &X, bool upload) {
    int rc = check_problem(p, c, X.d, !(ex && (ex->exec_flags & CAMELOT_EXEC_RESIDENT)));
    if (rc) return rc;
    rc = device_ok(ex);
    if (rc) return rc;
    X.L = make_layout(X.d, nlev);
    if (ex->workspace_bytes < X.L.total)
        return fail(CAMELOT_ENOMEM, "workspace too small: %zu < %zu bytes", ex->workspace_bytes, X.L.total);
    X.ws = static_cast<char *>(ex->workspace);
    X.st = static_cast<cudaStream_t>(ex->stream);
    if (upload) {   // this call rewrites the workspace: a pending finalize would read stale state
        std::lock_guard<std::mutex> g(g_rec_mu);
        g_rec.erase(ex->workspace);
    }
    X.P = make_devprob(p, c, X.d, X.ws, X.L);
    X.d0 = choose_d0(X.d);
    X.cm16 = X.d.C > 8;
    X.naive = (p->flags & F_PAPER_GLOBAL) || X.d.n < 2 || (ex->exec_flags & CAMELOT_EXEC_NAIVE);
    if (upload && !(ex->exec_flags & CAMELOT_EXEC_RESIDENT)) {
        CU(cudaMemcpyAsync(X.ws + X.L.tab, p->table, (size_t)X.d.n * X.d.nS * X.d.nQ * 16, cudaMemcpyHostToDevice, X.st));
        CU(cudaMemcpyAsync(X.ws + X.L.Q, p->quota_pct, (size_t)X.d.nQ * 4, cudaMemcpyHostToDevice, X.st));
        CU(cudaMemcpyAsync(X.ws + X.L.S, p->batch, (size_t)X.d.nS * 4, cudaMemcpyHostToDevice, X.st));
    }
    return CAMELOT_OK;
}

template <int CM, int NS, int POL>
int launch_search(const Ctx &X, const SearchArgs &S, int grid) {
    const size_t sm = search_smem<CM>();
    CU((k_search_launch<CM, NS, POL>(X.P, S, grid, sm, X.st)));
    COUNT_LAUNCH();
    return CAMELOT_OK;
}

#ifdef CAMELOT_SHARED_POLICY
#define CAM_POL(p) 2
#else
#define CAM_POL(p) (p)
#endif
#define CAM_DISPATCH(FN, ...)                                                                          \
    do {                                                                                               \
        const int cm_ = cm_bucket(X.d.C), ns_ = ns_bucket(X.d.n);                                      \
        if (cm_ == 4 && ns_ == 4) return policy ? FN<4, 4, CAM_POL(1)>(__VA_ARGS__) : FN<4, 4, CAM_POL(0)>(__VA_ARGS__); \
        if (cm_ == 4 && ns_ == 6) return policy ? FN<4, 6, CAM_POL(1)>(__VA_ARGS__) : FN<4, 6, CAM_POL(0)>(__VA_ARGS__); \
        if (cm_ == 4) return policy ? FN<4, 8, CAM_POL(1)>(__VA_ARGS__) : FN<4, 8, CAM_POL(0)>(__VA_ARGS__);             \
        if (cm_ == 8 && ns_ == 4) return policy ? FN<8, 4, CAM_POL(1)>(__VA_ARGS__) : FN<8, 4, CAM_POL(0)>(__VA_ARGS__); \
        if (cm_ == 8 && ns_ == 6) return policy ? FN<8, 6, CAM_POL(1)>(__VA_ARGS__) : FN<8, 6, CAM_POL(0)>(__VA_ARGS__); \
        if (cm_ == 8) return policy ? FN<8, 8, CAM_POL(1)>(__VA_ARGS__) : FN<8, 8, CAM_POL(0)>(__VA_ARGS__);             \
        return policy ? FN<16, 8, CAM_POL(1)>(__VA_ARGS__) : FN<16, 8, CAM_POL(0)>(__VA_ARGS__);                         \
    } while (0)

// staged option lists (TMA bulk copy of the level's compacted lists into every CTA's
// shared memory): the shared memory left after the level state, up to the opt-in
// per-block maximum.  Opt-in (CAMELOT_STAGE_RECORDS=1): measured on C4 it costs
// ~45 us per step (the staging phase per level, and 48-byte-strided LDS.128 reads are
// no faster than the L1 hits they replace)
template <int CM>
unsigned rec_budget_for(int dev, bool honour_env = true) {
    static int cache[64] = {0};
    int mx = dev < 64 ? cache[dev] : 0;
    if (!mx) {
        if (cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
            cudaGetLastError();
            mx = 48 * 1024;
        }
        if (dev < 64) cache[dev] = mx;
    }
    if (honour_env && (!getenv("CAMELOT_STAGE_RECORDS") || getenv("CAMELOT_NO_STAGE"))) return 0;
    const size_t fixed = level_fixed_bytes<CM>() + 16;
    return mx > (int)fixed + 1024 ? (unsigned)((mx - fixed - 1024) / 16 * 16) : 0u;
}
template <int CM>
size_t level_smem(int dev, bool honour_env = true) {   // filter scratch / search state, mbarrier, staged lists
    return level_fixed_bytes<CM>() + 16 + rec_budget_for<CM>(dev, honour_env);
}

template <int CM, int NS, int POL>
int coop_grid_for(int dev, int &grid) {
    static std::mutex mu;
    static std::vector<std::pair<int, int>> cache;   // (dev, grid)
    std::lock_guard<std::mutex> lk(mu);
    for (auto &e : cache)
        if (e.first == dev) {
            grid = e.second;
            return CAMELOT_OK;
        }
    const size_t sm = level_smem<CM>(dev, false);   // the largest launch (attribute + occupancy)
    int per = 0, nsm = 0;
    CU((k_level_occupancy<CM, NS, POL>(sm, &per)));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    grid = std::max(1, std::min(MAXSLOTS, per * nsm));
    cache.push_back({dev, grid});
    return CAMELOT_OK;
}

template <int CM, int NS, int POL>
int launch_level(const Ctx &X, int dev, const std::vector<LevelArgs> &levels) {
    int grid = 0;
    int rc = coop_grid_for<CM, NS, POL>(dev, grid);
    if (rc) return rc;
    LevelSet LS;
    memset(&LS, 0, sizeof(LS));
    if (levels.empty() || levels.size() > (size_t)MAX_LEVELS) return fail(CAMELOT_EINVAL, "bad level count");
    LS.count = (int)levels.size();
    const unsigned budget = rec_budget_for<CM>(dev);
    for (int l = 0; l < LS.count; ++l) {
        LS.L[l] = levels[l];
        LS.L[l].F.nslots = grid * LS.L[l].S.nlev;
        LS.L[l].rec_budget = budget;
    }
    const size_t sm = level_smem<CM>(dev);
    CU((k_level_launch<CM, NS, POL>(X.P, LS, grid, sm, X.st)));
    COUNT_LAUNCH();
    return CAMELOT_OK;
}

int launch_level_any(const Ctx &X, int policy, int dev, const std::vector<LevelArgs> &levels) {
    CAM_DISPATCH(launch_level, X, dev, levels);
}

int launch_search_any(const Ctx &X, int policy, const SearchArgs &S, int grid) {
    CAM_DISPATCH(launch_search, X, S, grid);
}

int grid_any(const Ctx &X, int policy, int dev, int &grid) {
    CAM_DISPATCH(grid_for, dev, grid);
}

int flat_grid(int dev, int &grid) {
    static int cache[64] = {0};
    if (dev < 64 && cache[dev]) {
        grid = cache[dev];
        return CAMELOT_OK;
    }
    int per = 0, nsm = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, flat_search_kernel, FLAT_THREADS, 0));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    grid = std::max(1, std::min(MAXSLOTS, per * nsm));
    if (dev < 64) cache[dev] = grid;
    return CAMELOT_OK;
}

// naive pass: thread per candidate over [lo, hi) (chunks of 2^15 dealt round-robin to ranks)
int flat_pass(const Ctx &X, int dev, int policy, int nlev, int ystride, int yoff, const float *lam, const Slot *inc,
              Slot *result, long long *keys, int rank, int world, unsigned long long lo, unsigned long long hi) {
    char *ws = X.ws;
    DevHeader *hdr = reinterpret_cast<DevHeader *>(ws + X.L.hdr);
    CU(cudaMemsetAsync(hdr, 0, sizeof(DevHeader), X.st));
    int grid = 0;
    int rc = flat_grid(dev, grid);
    if (rc) return rc;
    FlatArgs F;
    F.policy = policy;
    F.nlev = nlev;
    F.rank = rank;
    F.world = world;
    F.lo = lo;
    F.hi = hi;
    F.lam = lam;
    F.y = reinterpret_cast<const int *>(ws + X.L.y);
    F.ystride = ystride;
    F.yoff = yoff;
    F.inc = inc;
    F.slots = reinterpret_cast<Slot *>(ws + slots_off(X.L));
    F.hdr = hdr;
    flat_search_kernel<<<grid, FLAT_THREADS, 0, X.st>>>(X.P, F);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    reduce_kernel<<<1, 256, 0, X.st>>>(X.P, F.slots, grid, nlev, result, keys, nullptr, nullptr, nullptr, 0, 1,
                                       FLAT_SHIFT);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    return CAMELOT_OK;
}

// one cooperative launch per search level (default); CAMELOT_COOP=0 selects the
// multi-launch path (filter kernel + one kernel per pass)
bool use_coop() {
    const char *e = getenv("CAMELOT_COOP");
    return !(e && e[0] == '0');
}

int xshift_of(unsigned long long ntot) {
    int s = 0;
    while (s < 63 && ((ntot - 1) >> s) >= (1ull << 32)) ++s;
    return s;
}

// the level-synchronous passes of one search (parents at depth 0..n-1)
// `fresh`: the frontier counters and slots still have to be reset (re-scan);
// otherwise search_pass's header reset and the fused filter already did it.
int run_passes(const Ctx &X, int dev, int policy, SearchArgs S, bool timed, bool fresh) {
    char *ws = X.ws;
    DevHeader *hdr = S.hdr;
    int grid = 0;
    int rc = grid_any(X, policy, dev, grid);
    if (rc) return rc;
    if (fresh) CU(cudaMemsetAsync(hdr->head, 0, sizeof(hdr->head) + sizeof(hdr->tail), X.st));
    if (timed) {
        if (t_ev.dev != dev) {
            if (t_ev.a) {
                cudaEventDestroy(t_ev.a);
                cudaEventDestroy(t_ev.b);
            }
            CU(cudaEventCreate(&t_ev.a));
            CU(cudaEventCreate(&t_ev.b));
            t_ev.dev = dev;
        }
        CU(cudaEventRecord(t_ev.a, X.st));
    }
    if (fresh) {
        init_slots_kernel<<<(grid * S.nlev + 255) / 256, 256, 0, X.st>>>(S.slots, grid * S.nlev);
        COUNT_LAUNCH();
        CU(cudaGetLastError());
    }
    void *buf[2] = {ws + X.L.front0, ws + X.L.front1};
    const int n = X.d.n;
    for (int j = 0; j < n; ++j) {
        S.level = j;
        S.flevel = (j + 1 <= n - 1) ? j + 1 : -1;
        S.in_nodes = j == 0 ? nullptr : buf[j & 1];
        S.in_count = &hdr->tail[j];
        S.in_cap = X.L.fcap;
        S.out_nodes = buf[(j + 1) & 1];
        S.out_tail = &hdr->tail[j + 1];
        S.out_cap = X.L.fcap;
        S.head = &hdr->head[j];
        S.grab = 1;
        S.reduce_last = j == n - 1;   // the last pass reduces the slots (fused)
        rc = launch_search_any(X, policy, S, grid);
        if (rc) return rc;
    }
    if (timed) {
        CU(cudaEventRecord(t_ev.b, X.st));
        t_ev.armed = true;
    }
    return CAMELOT_OK;
}

// exhaustive scan (NO_FILTER) through the leaf-sweep kernel: the option lists are
// still built (full, unfiltered) for a possible chunk re-scan by the tree search
int sweep_pass(const Ctx &X, int dev, int policy, int nlev, const Slot *inc, Slot *result, long long *keys,
               int rank, int world, unsigned long long lo, unsigned long long hi, int qstride = 1) {
    char *ws = X.ws;
    DevHeader *hdr = reinterpret_cast<DevHeader *>(ws + X.L.hdr);
    CU(cudaMemsetAsync(hdr, 0, offsetof(DevHeader, cum_scored), X.st));
    CU(cudaMemsetAsync(&hdr->best_obj, 0xFF, sizeof(unsigned int), X.st));
    FilterArgs F;
    memset(&F, 0, sizeof(F));
    F.policy = policy;
    F.prune = 0;
    F.stride = 1;
    F.nlev = nlev;
    F.inc = inc;
    F.lam = reinterpret_cast<const float *>(ws + X.L.lam);
    F.rec = reinterpret_cast<OptRec *>(ws + X.L.rec);
    F.sb = reinterpret_cast<StageBound *>(ws + X.L.sb);
    F.item_off = reinterpret_cast<unsigned long long *>(ws + X.L.item_off);
    F.hdr = hdr;
    F.d0 = X.d0;
    if (qstride == 1 && world > 1) {   // full option lists + item offsets for a chunk re-scan (finalize)
        filter_kernel<<<X.d.nS, FILTER_THREADS, 0, X.st>>>(X.P, F);
        COUNT_LAUNCH();
        CU(cudaGetLastError());
    }
    SweepArgs A;
    memset(&A, 0, sizeof(A));
    A.policy = policy;
    A.rank = rank;
    A.world = world;
    A.d0 = X.d0;
    A.lo = lo;
    A.hi = hi;
    A.qstride = qstride;
    A.nQs = (X.d.nQ - 1) / qstride + 1;
    const unsigned long long Os = (unsigned long long)X.d.Rmax * A.nQs;
    A.nchunk = (int)((Os + 31) / 32);
    A.gpack = Os <= 16 ? (int)(32 / Os) : 1;   // small option lists: several grandparents per warp
    if (qstride == 1) {
        const unsigned long long O2 = Os * Os;
        if (hi > lo) {
            A.g_lo = lo / O2;
            A.n_gp = (hi - 1) / O2 + 1 - A.g_lo;
        }
    } else {   // sub-grid (incumbent cascade): the whole sub-space, world 1
        unsigned long long ngp = (unsigned long long)X.d.nbc;
        for (int i = 0; i < X.d.n - 2; ++i) ngp *= Os;
        A.g_lo = 0;
        A.n_gp = ngp;
    }
    {   // chunks per work item (testing knob CAMELOT_SWEEP_CPG): the grandparent is placed once per item
        const int cpg = getenv("CAMELOT_SWEEP_CPG") ? std::max(1, atoi(getenv("CAMELOT_SWEEP_CPG"))) : 4;
        A.ngroups = A.gpack == 1 ? (A.nchunk + cpg - 1) / cpg : 1;
    }
    // guided: the last eighth of the grandparents (the end of the dynamic queue) as
    // single-chunk items, so that the tail of the scan is fine-grained
    const unsigned long long tdiv = getenv("CAMELOT_SWEEP_TAIL") ? std::max(1, atoi(getenv("CAMELOT_SWEEP_TAIL"))) : 8;
    A.gp_split = A.gpack == 1 && A.ngroups < A.nchunk ? A.n_gp - A.n_gp / tdiv : A.n_gp;
    A.n_grp_items = A.gp_split * (unsigned long long)A.ngroups;
    A.n_items = A.gpack == 1 ? A.n_grp_items + (A.n_gp - A.gp_split) * (unsigned long long)A.nchunk
                             : (A.n_gp + (unsigned long long)A.gpack - 1) / (unsigned long long)A.gpack;
    A.lam = reinterpret_cast<const float *>(ws + X.L.lam);
    A.y = reinterpret_cast<const int *>(ws + X.L.y);
    A.ystride = nlev;
    A.yoff = 0;
    A.inc = inc;
    A.slots = reinterpret_cast<Slot *>(ws + slots_off(X.L));
    A.hdr = hdr;
    A.result = result;
    A.keys = keys;
    const size_t tb = (size_t)X.d.nS * X.d.nQ * sizeof(float4);
    A.tabL_bytes = (tb <= SWEEP_TABL_MAX && !getenv("CAMELOT_NO_STAGE")) ? (unsigned)tb : 0u;
    // small sub-grids (the coarsest cascade level: a few quotas) compute the capacities
    // per quota; the breakpoints pay off over many quotas (testing knob CAMELOT_BP_MIN)
    A.bp_min_nqs = getenv("CAMELOT_BP_MIN") ? atoi(getenv("CAMELOT_BP_MIN")) : 9;
    CU(sweep_launch(X.P, A, dev, X.st));
    COUNT_LAUNCH();
    return CAMELOT_OK;
}

int search_pass(const Ctx &X, int dev, int policy, int nlev, bool prune, int stride, const Slot *inc,
                Slot *result, long long *keys, int rank, int world, unsigned long long lo, unsigned long long hi,
                bool timed, Slot *inc_out = nullptr, std::vector<LevelArgs> *defer = nullptr) {
    char *ws = X.ws;
    if (X.naive)
        return flat_pass(X, dev, policy, nlev, nlev, 0, reinterpret_cast<const float *>(ws + X.L.lam), inc, result,
                         keys, rank, world, lo, hi);
    DevHeader *hdr = reinterpret_cast<DevHeader *>(ws + X.L.hdr);
    if (!prune && sweep_supported(X.P, policy, nlev) && !getenv("CAMELOT_NO_SWEEP"))
        return sweep_pass(X, dev, policy, nlev, inc, result, keys, rank, world, lo, hi);
    const bool coop = use_coop();
    if (!coop) {
        CU(cudaMemsetAsync(hdr, 0, offsetof(DevHeader, cum_scored), X.st));
        CU(cudaMemsetAsync(&hdr->best_obj, 0xFF, sizeof(unsigned int), X.st));
        CU(cudaMemsetAsync(&hdr->best_packed, 0xFF, sizeof(unsigned long long), X.st));
    }
    FilterArgs F;
    F.policy = policy;
    F.prune = prune;
    F.stride = stride;
    F.nlev = nlev;
    F.inc = inc;
    F.lam = reinterpret_cast<const float *>(ws + X.L.lam);
    F.rec = reinterpret_cast<OptRec *>(ws + X.L.rec);
    F.sb = reinterpret_cast<StageBound *>(ws + X.L.sb);
    int grid = 0;
    int rc = grid_any(X, policy, dev, grid);
    if (rc) return rc;
    F.slots = reinterpret_cast<Slot *>(ws + slots_off(X.L));
    F.nslots = grid * nlev;
    F.item_off = reinterpret_cast<unsigned long long *>(ws + X.L.item_off);
    F.hdr = hdr;
    F.d0 = X.d0;
    if (!coop) {
        filter_kernel<<<X.d.nS, FILTER_THREADS, 0, X.st>>>(X.P, F);   // + slot reset + item offsets
        COUNT_LAUNCH();
        CU(cudaGetLastError());
    }
    SearchArgs S;
    memset(&S, 0, sizeof(S));
    S.policy = policy;
    S.nlev = nlev;
    S.d0 = X.d0;
    S.chunk_items = CHUNK_ITEMS;
    S.rank = rank;
    S.world = world;
    S.prune = prune;
    S.lo = lo;
    S.hi = hi;
    S.rec = F.rec;
    S.sb = F.sb;
    S.item_off = reinterpret_cast<const unsigned long long *>(ws + X.L.item_off);
    S.lam = F.lam;
    S.lam_stride = X.d.A;
    S.y = reinterpret_cast<const int *>(ws + X.L.y);
    S.ystride = nlev;
    S.yoff = 0;
    S.inc = inc;
    S.hdr = hdr;
    S.slots = reinterpret_cast<Slot *>(ws + slots_off(X.L));
    S.xshift = xshift_of(X.d.ntot);
    S.tmode_min16 = getenv("CAMELOT_TMODE_MIN16") ? atoi(getenv("CAMELOT_TMODE_MIN16")) : 32;   // (testing knob)
    S.tmode_inner_gmax = getenv("CAMELOT_TMODE_INNER_G") ? atoi(getenv("CAMELOT_TMODE_INNER_G")) : 8;   // (testing knob)
    S.tmode_leaf_gmax = getenv("CAMELOT_TMODE_LEAF_G") ? atoi(getenv("CAMELOT_TMODE_LEAF_G")) : 8;   // (testing knob)
    S.tmode_slack = 1;   // separate launches have no redo: strict capacity (the cooperative level sets its own)
    S.result = result;
    S.keys = keys;
    S.inc_out = inc_out;
    if (coop) {
        LevelArgs LA;
        memset(&LA, 0, sizeof(LA));
        LA.S = S;
        LA.F = F;
        LA.buf0 = ws + X.L.front0;
        LA.buf1 = ws + X.L.front1;
        LA.fcap = X.L.fcap;
        // optimistic thread-per-parent inner passes (redone in the warp mode on overflow;
        // testing knob CAMELOT_TMODE_SLACK)
        LA.S.tmode_slack = getenv("CAMELOT_TMODE_SLACK") ? std::max(1, atoi(getenv("CAMELOT_TMODE_SLACK"))) : 8;
        // compact depth-1 frontier (testing knob CAMELOT_COMPACT1=0 keeps full nodes)
        LA.S.compact1 = !(getenv("CAMELOT_COMPACT1") && getenv("CAMELOT_COMPACT1")[0] == '0');
        if (defer) {   // chained into one cooperative launch by the caller
            defer->push_back(LA);
            return CAMELOT_OK;
        }
        return launch_level_any(X, policy, dev, std::vector<LevelArgs>{LA});
    }
    return run_passes(X, dev, policy, S, timed, false);
}

// re-scan chunk `chunk` for level k after the cross-rank reduction (same filter state)
int rescan_pass(const Ctx &X, int dev, int policy, int nlev, bool prune, int k, Slot *winner_k,
                const unsigned long long chunk, unsigned long long lo, unsigned long long hi) {
    char *ws = X.ws;
    if (X.naive) {
        const unsigned long long a0 = std::max(lo, chunk << FLAT_SHIFT);
        const unsigned long long b0 = std::min(hi, (chunk + 1) << FLAT_SHIFT);
        long long *dummy = reinterpret_cast<long long *>(ws + X.L.keys) + k;
        return flat_pass(X, dev, policy, 1, nlev, k, reinterpret_cast<const float *>(ws + X.L.lam) + k * X.d.A,
                         winner_k, winner_k, dummy, 0, 1, a0, b0);
    }
    DevHeader *hdr = reinterpret_cast<DevHeader *>(ws + X.L.hdr);
    SearchArgs S;
    memset(&S, 0, sizeof(S));
    S.policy = policy;
    S.nlev = 1;
    S.d0 = X.d0;
    S.chunk_items = CHUNK_ITEMS;
    S.rank = 0;
    S.world = 1;
    S.prune = prune;
    S.lo = lo;
    S.hi = hi;
    S.rec = reinterpret_cast<const OptRec *>(ws + X.L.rec);
    S.sb = reinterpret_cast<const StageBound *>(ws + X.L.sb);
    S.item_off = reinterpret_cast<const unsigned long long *>(ws + X.L.item_off);
    S.lam = reinterpret_cast<const float *>(ws + X.L.lam) + k * X.d.A;
    S.lam_stride = X.d.A;
    S.y = reinterpret_cast<const int *>(ws + X.L.y);
    S.ystride = nlev;
    S.yoff = k;
    S.inc = winner_k;
    S.hdr = hdr;
    S.slots = reinterpret_cast<Slot *>(ws + slots_off(X.L));
    S.chunk_lo = chunk;
    S.chunk_hi = chunk + 1;
    S.xshift = xshift_of(X.d.ntot);
    S.tmode_min16 = getenv("CAMELOT_TMODE_MIN16") ? atoi(getenv("CAMELOT_TMODE_MIN16")) : 32;   // (testing knob)
    S.tmode_inner_gmax = getenv("CAMELOT_TMODE_INNER_G") ? atoi(getenv("CAMELOT_TMODE_INNER_G")) : 8;   // (testing knob)
    S.tmode_leaf_gmax = getenv("CAMELOT_TMODE_LEAF_G") ? atoi(getenv("CAMELOT_TMODE_LEAF_G")) : 8;   // (testing knob)
    S.tmode_slack = 1;   // separate launches have no redo: strict capacity (the cooperative level sets its own)
    CU(cudaMemsetAsync(&hdr->best_obj, 0xFF, sizeof(unsigned int), X.st));
    CU(cudaMemsetAsync(&hdr->best_packed, 0xFF, sizeof(unsigned long long), X.st));
    CU(cudaMemsetAsync(&hdr->done_ctas, 0, sizeof(unsigned int), X.st));
    S.result = winner_k;
    S.keys = reinterpret_cast<long long *>(ws + X.L.keys) + k;
    S.inc_out = nullptr;
    return run_passes(X, dev, policy, S, false, true);
}

void range_of(const Ctx &X, const camelot_exec *ex, unsigned long long &lo, unsigned long long &hi) {
    lo = ex->index_lo;
    hi = ex->index_hi;
    if (lo == 0 && hi == 0) hi = X.d.ntot;
    if (hi > X.d.ntot) hi = X.d.ntot;
    if (lo > hi) lo = hi;
}

bool use_coarse(const Ctx &X, bool prune) { return prune && !X.naive && X.d.nQ >= 8 && X.d.ntot > 4000000ull; }
// quota sub-grid strides of the incumbent cascade (every stride-th quota counted
// from the top, so 100% is always included).  CAMELOT_COARSE="25,10" overrides (and
// CAMELOT_COARSE_P0 / _P1 per policy: experiments).
std::vector<int> coarse_strides(const Ctx &X, int policy) {
    std::vector<int> v;
    const char *e = getenv(policy == 0 ? "CAMELOT_COARSE_P0" : "CAMELOT_COARSE_P1");
    if (!e) e = getenv("CAMELOT_COARSE");
    if (e) {
        const char *p = e;
        while (*p) {
            char *q = nullptr;
            const long s = strtol(p, &q, 10);
            if (q == p) break;
            if (s >= 2 && s < X.d.nQ) v.push_back((int)s);
            p = (*q == ',') ? q + 1 : q;
        }
        return v;
    }
    // measured: coarse grids (nQ < 50) use (nQ/2, nQ/5, nQ/20), e.g. C5
    // (5, 2); fine grids use per-policy strides, max load (nQ/2, nQ/9, nQ/25) = (50, 11, 4)
    // and min resource (nQ/2, nQ/5, nQ/14) = (50, 20, 7) on the 1% grid: over eight
    // C4-shaped problems (C4, C4b and six other seeds / QoS scales) they cut the plan
    // pair's geometric-mean time from 4.9 to 2.8 ms, and none got slower
    const int nQ = X.d.nQ;
    int div[3] = {2, 5, 20};
    if (nQ >= 50) {
        div[1] = policy == 0 ? 9 : 5;
        div[2] = policy == 0 ? 25 : 14;
    }
    for (int d : div) {
        const int s = nQ / d;
        if (s >= 2 && (v.empty() || s < v.back())) v.push_back(s);
    }
    return v;
}

// local search (incumbent pass + main pass); leaves keys in X.L.keys (or d_keys) and the
// exact local best in X.L.result
// prologue_done: the incumbent slots, the Eq. 2 estimates and the cumulative counters
// were already prepared on the stream (camelot_plan_max_then_min's bridge_kernel)
int local_search(const Ctx &X, const camelot_exec *ex, int policy, int nlev, long long *d_keys,
                 bool prologue_done = false, bool snapshot = true) {
    const bool prune = !(X.P.flags & F_NO_FILTER);
    char *ws = X.ws;
    Slot *inc = reinterpret_cast<Slot *>(ws + X.L.inc);
    Slot *result = reinterpret_cast<Slot *>(ws + X.L.result);
    long long *keys = d_keys ? d_keys : reinterpret_cast<long long *>(ws + X.L.keys);
    // incumbent = none (key 0xFFFFFFFF, x = ~0), counters zeroed, Eq. 2 estimates: one launch
    if (!prologue_done) {
        prologue_kernel<<<1, 256, 0, X.st>>>(X.P, inc, nlev, policy, reinterpret_cast<const float *>(ws + X.L.lam),
                                             reinterpret_cast<int *>(ws + X.L.y),
                                             reinterpret_cast<DevHeader *>(ws + X.L.hdr));
        COUNT_LAUNCH();
        CU(cudaGetLastError());
    }
    unsigned long long lo, hi;
    range_of(X, ex, lo, hi);
    int dev = ex->device;
    int rc;
    if (t_ev.dev != dev) {
        if (t_ev.a) {
            cudaEventDestroy(t_ev.a);
            cudaEventDestroy(t_ev.b);
        }
        CU(cudaEventCreate(&t_ev.a));
        CU(cudaEventCreate(&t_ev.b));
        t_ev.dev = dev;
    }
    CU(cudaEventRecord(t_ev.a, X.st));
    std::vector<int> pending_strides;
    if (use_coarse(X, prune)) {
        // incumbent: exact optimum of coarse quota sub-grids, coarsest first (each
        // pass seeds the next); replicated on every rank.  The coarse levels small
        // enough for an exhaustive scan are replaced by ONE leaf sweep of the finest
        // of them (its optimum is at least as good as any coarser level's).
        std::vector<int> strides = coarse_strides(X, policy);
        if (sweep_supported(X.P, policy, nlev) && lo == 0 && hi == X.d.ntot && !getenv("CAMELOT_NO_SWEEP")) {
            int flat_s = 0;
            for (int s2 : strides) {
                long double sub = (long double)X.d.nbc;
                for (int i = 0; i < X.d.n; ++i) sub *= (long double)X.d.Rmax * ((X.d.nQ - 1) / s2 + 1);
                // measured (C4): a sub-grid of <= 2^20 candidates sweeps faster than a pruned
                // level; larger ones lose to the pruned search (per-parent setup dominates)
                if (sub <= (long double)(1ull << 20)) flat_s = s2;   // strides are descending
            }
            if (flat_s) {
                rc = sweep_pass(X, dev, policy, nlev, inc, inc, reinterpret_cast<long long *>(ws + X.L.keys), 0, 1, lo,
                                hi, flat_s);
                if (rc) return rc;
                std::vector<int> rest;
                for (int s2 : strides)
                    if (s2 < flat_s) rest.push_back(s2);
                strides.swap(rest);
            }
        }
        pending_strides = strides;
    }
    // the pruned levels (cascade, then the main pass) go into ONE cooperative launch
    std::vector<LevelArgs> levels;
    const bool chain = use_coop() && !X.naive && prune;
    std::vector<int> strides2;
    if (use_coarse(X, prune)) strides2 = pending_strides;
    for (int stride : strides2) {
        rc = search_pass(X, dev, policy, nlev, true, stride, inc, result, reinterpret_cast<long long *>(ws + X.L.keys),
                         0, 1, lo, hi, false, inc, chain ? &levels : nullptr);
        if (rc) return rc;
    }
    rc = search_pass(X, dev, policy, nlev, prune, 1, inc, result, keys, ex->rank, ex->world, lo, hi, false, nullptr,
                     chain ? &levels : nullptr);
    if (rc) return rc;
    if (!levels.empty()) {
        rc = launch_level_any(X, policy, dev, levels);
        if (rc) return rc;
    }
    CU(cudaEventRecord(t_ev.b, X.st));
    t_ev.armed = true;
    // the counters for camelot_finalize, safe from a chunk re-scan (camelot_plan_max_then_min
    // reads them from the header itself: nothing runs in between)
    if (snapshot) CU(cudaMemcpyAsync(ws + X.L.hdr2, ws + X.L.hdr, sizeof(DevHeader), cudaMemcpyDeviceToDevice, X.st));
    return CAMELOT_OK;
}

// resolve the reduced keys (+ chunk re-scan when sharded) and score the winners into
// dplans[0..nlev) on the device; no host synchronisation when world == 1
int finalize_enqueue(const Ctx &X, const camelot_exec *ex, int policy, int nlev, const long long *d_keys,
                     camelot_plan *dplans, bool from_hdr = false) {
    const bool prune = !(X.P.flags & F_NO_FILTER);
    char *ws = X.ws;
    Slot *winner = reinterpret_cast<Slot *>(ws + X.L.winner);
    unsigned long long *rescan = reinterpret_cast<unsigned long long *>(ws + X.L.rescan);
    FinalArgs F;
    F.policy = policy;
    F.nlev = nlev;
    F.world = ex->world;
    F.keys = d_keys;
    F.local = reinterpret_cast<const Slot *>(ws + X.L.result);
    F.winner = winner;
    F.rescan = rescan;
    if (ex->world > 1) {   // (one rank: plan_kernel resolves the key itself)
        resolve_kernel<<<1, 64, 0, X.st>>>(X.P, F);
        COUNT_LAUNCH();
        CU(cudaGetLastError());
    }
    if (ex->world > 1 && X.d.ntot > (1ull << 32)) {
        std::vector<unsigned long long> rs(nlev);
        CU(cudaMemcpyAsync(rs.data(), rescan, nlev * sizeof(unsigned long long), cudaMemcpyDeviceToHost, X.st));
        CU(cudaStreamSynchronize(X.st));
        unsigned long long lo, hi;
        range_of(X, ex, lo, hi);
        for (int k = 0; k < nlev; ++k) {
            if (rs[k] == ~0ull) continue;
            int rc = rescan_pass(X, ex->device, policy, nlev, prune, k, winner + k, rs[k], lo, hi);
            if (rc) return rc;
        }
    }
    plan_kernel<<<nlev, PLAN_THREADS, 0, X.st>>>(X.P, policy, nlev, winner, reinterpret_cast<const float *>(ws + X.L.lam),
                                                   reinterpret_cast<const DevHeader *>(ws + (from_hdr ? X.L.hdr : X.L.hdr2)),
                                                   dplans, ex->world > 1 ? nullptr : d_keys,
                                                   ex->world > 1 ? nullptr : F.local);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    return CAMELOT_OK;
}

int finalize_impl(const Ctx &X, const camelot_exec *ex, int policy, int nlev, const long long *d_keys,
                  camelot_plan *out) {
    camelot_plan *dplans = reinterpret_cast<camelot_plan *>(X.ws + X.L.plans);
    int rc = finalize_enqueue(X, ex, policy, nlev, d_keys, dplans);
    if (rc) return rc;
    CU(cudaMemcpyAsync(out, dplans, nlev * sizeof(camelot_plan), cudaMemcpyDeviceToHost, X.st));
    CU(cudaStreamSynchronize(X.st));
    unsigned long long lo, hi;
    range_of(X, ex, lo, hi);
    uint64_t search_ns = 0;   // the stream is synchronised: the search's events are complete
    if (t_ev.armed && t_ev.dev == ex->device) {
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, t_ev.a, t_ev.b) == cudaSuccess) search_ns = (uint64_t)((double)ms * 1e6);
        else cudaGetLastError();
    }
    bool any = false;
    for (int k = 0; k < nlev; ++k) {
        out[k].n_covered = hi - lo;
        out[k].search_ns = search_ns;
        any |= out[k].status == CAMELOT_OK;
    }
    return any ? CAMELOT_OK : CAMELOT_INFEASIBLE;
}

int upload_loads(const Ctx &X, const float *loads, int n_loads) {
    if (n_loads <= 0) return CAMELOT_OK;
    CU(cudaMemcpyAsync(X.ws + X.L.lam, loads, (size_t)n_loads * X.d.A * sizeof(float), cudaMemcpyHostToDevice, X.st));
    return CAMELOT_OK;
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

const char *camelot_last_error(void) { return g_err.c_str(); }
const char *camelot_version(void) { return "camelot-b200 0.1 (sm_100a)"; }

size_t camelot_workspace_bytes(const camelot_problem *p, const camelot_cluster *c, int n_loads) {
    Dims d;
    if (check_problem(p, c, d)) return 0;
    if (n_loads < 0 || n_loads > CAMELOT_MAX_LOADS) {
        fail(CAMELOT_EINVAL, "n_loads must be in 0..64");
        return 0;
    }
    return make_layout(d, n_loads).total;
}

int camelot_upload(const camelot_problem *p, const camelot_cluster *c, const camelot_exec *ex) {
    t_call_launches = 0;
    Ctx X;
    camelot_exec e2 = ex ? *ex : camelot_exec{};
    e2.exec_flags &= ~CAMELOT_EXEC_RESIDENT;
    return setup(p, c, &e2, 1, X, true);
}

int camelot_search_local(const camelot_problem *p, const camelot_cluster *c, int policy, const float *load_qps,
                         int n_loads, const camelot_exec *ex, int64_t *d_keys) {
    t_call_launches = 0;
    if (policy != 0 && policy != 1) return fail(CAMELOT_EINVAL, "bad policy");
    const int nlev = policy == 0 ? 1 : n_loads;
    if (policy == 1) {
        int rc = p ? check_loads(p, load_qps, n_loads) : fail(CAMELOT_EINVAL, "null problem");
        if (rc) return rc;
    }
    Ctx X;
    int rc = setup(p, c, ex, nlev, X, true);
    if (rc) return rc;
    rc = upload_loads(X, load_qps, policy == 1 ? n_loads : 0);
    if (rc) return rc;
    rc = local_search(X, ex, policy, nlev, reinterpret_cast<long long *>(d_keys));
    if (rc) return rc;
    SearchRecord r;
    r.policy = policy;
    r.nlev = nlev;
    r.rank = ex->rank;
    r.world = ex->world;
    range_of(X, ex, r.lo, r.hi);
    r.ntot = X.d.ntot;
    r.flags = p->flags;
    if (policy == 1) r.loads.assign(load_qps, load_qps + (size_t)n_loads * p->n_apps);
    std::lock_guard<std::mutex> g(g_rec_mu);
    g_rec[ex->workspace] = std::move(r);
    return CAMELOT_OK;
}

int camelot_finalize(const camelot_problem *p, const camelot_cluster *c, int policy, const float *load_qps,
                     int n_loads, const int64_t *d_keys, const camelot_exec *ex, camelot_plan *out) {
    t_call_launches = 0;
    if (policy != 0 && policy != 1) return fail(CAMELOT_EINVAL, "bad policy");
    if (!out || !d_keys) return fail(CAMELOT_EINVAL, "null out or keys");
    const int nlev = policy == 0 ? 1 : n_loads;
    if (policy == 1) {
        int rc = p ? check_loads(p, load_qps, n_loads) : fail(CAMELOT_EINVAL, "null problem");
        if (rc) return rc;
    }
    Ctx X;
    int rc = setup(p, c, ex, nlev, X, false);
    if (rc) return rc;
    {
        // the pairing contract with camelot_search_local (camelot.h)
        unsigned long long lo, hi;
        range_of(X, ex, lo, hi);
        std::lock_guard<std::mutex> g(g_rec_mu);
        auto it = g_rec.find(ex->workspace);
        if (it == g_rec.end()) return fail(CAMELOT_EINVAL, "finalize: no camelot_search_local on this workspace");
        const SearchRecord &r = it->second;
        if (r.policy != policy || r.nlev != nlev || r.rank != ex->rank || r.world != ex->world || r.lo != lo ||
            r.hi != hi || r.ntot != X.d.ntot || r.flags != p->flags)
            return fail(CAMELOT_EINVAL, "finalize: policy/levels/range/shard differ from the last camelot_search_local "
                                        "on this workspace");
        if (policy == 1 && (r.loads.size() != (size_t)n_loads * p->n_apps ||
                            memcmp(r.loads.data(), load_qps, r.loads.size() * sizeof(float)) != 0))
            return fail(CAMELOT_EINVAL, "finalize: load_qps differ from the last camelot_search_local");
    }
    return finalize_impl(X, ex, policy, nlev, reinterpret_cast<const long long *>(d_keys), out);
}

int camelot_plan_max_load(const camelot_problem *p, const camelot_cluster *c, const camelot_exec *ex,
                          camelot_plan *out) {
    t_call_launches = 0;
    if (!out) return fail(CAMELOT_EINVAL, "null out");
    if (ex && ex->world != 1) return fail(CAMELOT_EINVAL, "plan_* is single-process: use search_local + finalize for world > 1");
    Ctx X;
    int rc = setup(p, c, ex, 1, X, true);
    if (rc) return rc;
    rc = local_search(X, ex, 0, 1, nullptr);
    if (rc) return rc;
    return finalize_impl(X, ex, 0, 1, reinterpret_cast<const long long *>(X.ws + X.L.keys), out);
}

int camelot_plan_min_resource(const camelot_problem *p, const camelot_cluster *c, const float *load_qps, int n_loads,
                              const camelot_exec *ex, camelot_plan *out) {
    t_call_launches = 0;
    if (!out) return fail(CAMELOT_EINVAL, "null out");
    if (ex && ex->world != 1) return fail(CAMELOT_EINVAL, "plan_* is single-process: use search_local + finalize for world > 1");
    int rc = p ? check_loads(p, load_qps, n_loads) : fail(CAMELOT_EINVAL, "null problem");
    if (rc) return rc;
    Ctx X;
    rc = setup(p, c, ex, n_loads, X, true);
    if (rc) return rc;
    rc = upload_loads(X, load_qps, n_loads);
    if (rc) return rc;
    rc = local_search(X, ex, 1, n_loads, nullptr);
    if (rc) return rc;
    return finalize_impl(X, ex, 1, n_loads, reinterpret_cast<const long long *>(X.ws + X.L.keys), out);
}

int camelot_plan_max_then_min(const camelot_problem *p, const camelot_cluster *c, double low_load_frac,
                              const camelot_exec *ex, camelot_plan *out) {
    t_call_launches = 0;
    if (!out) return fail(CAMELOT_EINVAL, "null out");
    if (ex && ex->world != 1) return fail(CAMELOT_EINVAL, "plan_* is single-process: use search_local + finalize for world > 1");
    if (!(low_load_frac > 0.0 && low_load_frac <= 1.0)) return fail(CAMELOT_EINVAL, "low_load_frac must be in (0, 1]");
    Ctx X;
    int rc = setup(p, c, ex, 1, X, true);
    if (rc) return rc;
    camelot_plan *dplans = reinterpret_cast<camelot_plan *>(X.ws + X.L.plans);   // [0] min-resource, [1] max-load
    // max-load search and its winner
    rc = local_search(X, ex, 0, 1, nullptr, false, false);
    if (rc) return rc;
    std::swap(t_ev, t_ev_spare);   // keep the max-load search's events
    if (t_side.dev != ex->device) {
        if (t_side.s) {
            cudaStreamDestroy(t_side.s);
            cudaEventDestroy(t_side.fork);
            cudaEventDestroy(t_side.join);
        }
        CU(cudaStreamCreateWithFlags(&t_side.s, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&t_side.fork, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&t_side.join, cudaEventDisableTiming));
        t_side.dev = ex->device;
    }
    // the low load from the peak, on the device (no host round trip) + a snapshot of the
    // max-load winner and counters; the max-load plan is then scored on the second
    // stream while the min-resource search runs on this one
    Slot *side_w = reinterpret_cast<Slot *>(X.ws + X.L.side_w);
    DevHeader *side_h = reinterpret_cast<DevHeader *>(X.ws + X.L.side_h);
    // one launch between the searches: resolve the max-load key, the low load, the snapshot
    // for the max-load plan, and the min-resource search's prologue (bridge_kernel)
    bridge_kernel<<<1, 256, 0, X.st>>>(X.P, reinterpret_cast<const long long *>(X.ws + X.L.keys),
                                       reinterpret_cast<const Slot *>(X.ws + X.L.result),
                                       reinterpret_cast<Slot *>(X.ws + X.L.winner), low_load_frac,
                                       reinterpret_cast<float *>(X.ws + X.L.lam), side_w, side_h,
                                       reinterpret_cast<const DevHeader *>(X.ws + X.L.hdr),
                                       reinterpret_cast<Slot *>(X.ws + X.L.inc), reinterpret_cast<int *>(X.ws + X.L.y),
                                       reinterpret_cast<DevHeader *>(X.ws + X.L.hdr));
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    CU(cudaEventRecord(t_side.fork, X.st));
    CU(cudaStreamWaitEvent(t_side.s, t_side.fork, 0));
    plan_kernel<<<1, PLAN_THREADS, 0, t_side.s>>>(X.P, 0, 1, side_w, reinterpret_cast<const float *>(X.ws + X.L.lam),
                                                   side_h, dplans + 1);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    CU(cudaEventRecord(t_side.join, t_side.s));
    rc = local_search(X, ex, 1, 1, nullptr, true, false);
    if (!rc) rc = finalize_enqueue(X, ex, 1, 1, reinterpret_cast<const long long *>(X.ws + X.L.keys), dplans, true);
    CU(cudaStreamWaitEvent(X.st, t_side.join, 0));   // join the max-load plan (also on an error)
    if (rc) return rc;
    camelot_plan both[2];
    CU(cudaMemcpyAsync(both, dplans, 2 * sizeof(camelot_plan), cudaMemcpyDeviceToHost, X.st));
    CU(cudaStreamSynchronize(X.st));
    out[0] = both[1];
    out[1] = both[0];
    if (out[0].status != CAMELOT_OK) {   // no peak, no low load (camelot.h): every level fails LOAD
        out[1].status = CAMELOT_INFEASIBLE;
        out[1].index = ~0ull;
        out[1].violations = CAMELOT_V_LOAD;
    }
    unsigned long long lo, hi;
    range_of(X, ex, lo, hi);
    EvPair *evs[2] = {&t_ev_spare, &t_ev};
    for (int k = 0; k < 2; ++k) {
        out[k].n_covered = hi - lo;
        out[k].search_ns = 0;
        float ms = 0.0f;
        if (evs[k]->armed && evs[k]->dev == ex->device) {
            if (cudaEventElapsedTime(&ms, evs[k]->a, evs[k]->b) == cudaSuccess) out[k].search_ns = (uint64_t)((double)ms * 1e6);
            else cudaGetLastError();
        }
    }
    return (out[0].status == CAMELOT_OK && out[1].status == CAMELOT_OK) ? CAMELOT_OK : CAMELOT_INFEASIBLE;
}

int camelot_predict(const camelot_problem *p, const camelot_cluster *c, const int32_t *batch, const int32_t *replicas,
                    const int32_t *quota_pct, const float *load_qps, int n_loads, const camelot_exec *ex,
                    camelot_plan *out) {
    t_call_launches = 0;
    if (!out || !batch || !replicas || !quota_pct) return fail(CAMELOT_EINVAL, "null argument");
    Dims d;
    int rc = check_problem(p, c, d);
    if (rc) return rc;
    // explicit plan values -> canonical digits (strictly on the grids) -> index
    unsigned long long x = 0;
    for (int a = 0; a < d.A; ++a) {
        int b = -1;
        for (int k = 0; k < d.nS; ++k)
            if (p->batch[k] == batch[a]) b = k;
        if (b < 0) return fail(CAMELOT_EINVAL, "batch %d of app %d is not on the batch grid", batch[a], a);
        x = x * d.nS + b;
    }
    for (int i = 0; i < d.n; ++i) {
        if (replicas[i] < 1 || replicas[i] > d.Rmax) return fail(CAMELOT_EINVAL, "replicas[%d] not in 1..Rmax", i);
        int t = -1;
        for (int k = 0; k < d.nQ; ++k)
            if (p->quota_pct[k] == quota_pct[i]) t = k;
        if (t < 0) return fail(CAMELOT_EINVAL, "quota %d of stage %d is not on the quota grid", quota_pct[i], i);
        x = x * d.Rmax + (replicas[i] - 1);
        x = x * d.nQ + t;
    }
    return camelot_predict_index(p, c, x, load_qps, n_loads, ex, out);
}

int camelot_predict_index(const camelot_problem *p, const camelot_cluster *c, uint64_t index, const float *load_qps,
                          int n_loads, const camelot_exec *ex, camelot_plan *out) {
    t_call_launches = 0;
    if (!out) return fail(CAMELOT_EINVAL, "null out");
    Ctx X;
    int rc = setup(p, c, ex, 1, X, true);
    if (rc) return rc;
    if (index >= X.d.ntot) return fail(CAMELOT_EINVAL, "index %llu >= Ntot %llu", (unsigned long long)index, X.d.ntot);
    if (n_loads > 0) {
        rc = check_loads(p, load_qps, 1);
        if (rc) return rc;
        rc = upload_loads(X, load_qps, 1);
        if (rc) return rc;
    }
    // the device decodes the canonical index (mixed radix, step A2) and scores it
    camelot_plan *dplans = reinterpret_cast<camelot_plan *>(X.ws + X.L.plans);
    predict_kernel<<<1, 1, 0, X.st>>>(X.P, index, n_loads > 0 ? reinterpret_cast<const float *>(X.ws + X.L.lam) : nullptr,
                                      n_loads > 0 ? 1 : 0, dplans);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out, dplans, sizeof(camelot_plan), cudaMemcpyDeviceToHost, X.st));
    CU(cudaStreamSynchronize(X.st));
    return out->status;
}

size_t camelot_simulate_workspace_bytes(const camelot_problem *p, const camelot_cluster *c, int64_t n_queries,
                                        int n_sims) {
    Dims d;
    if (check_problem(p, c, d)) return 0;
    if (n_queries < 1 || n_sims < 1 || n_sims > 65535) {
        fail(CAMELOT_EINVAL, "n_queries >= 1 and n_sims in 1..65535");
        return 0;
    }
    return make_layout(d, 1).total + al((size_t)n_sims * (size_t)n_queries * sizeof(double)) +
           al((size_t)n_sims * CAMELOT_MAX_APPS * 2 * sizeof(double));
}

int camelot_simulate(const camelot_problem *p, const camelot_cluster *c, const int32_t *batch,
                     const int32_t *replicas, const int32_t *quota_pct, const float *load_qps, int64_t n_queries,
                     int64_t warmup, uint64_t seed, int n_sims, const camelot_exec *ex, double *p99_ms,
                     double *mean_ms) {
    t_call_launches = 0;
    if (!batch || !replicas || !quota_pct || !load_qps || !p99_ms || !mean_ms) return fail(CAMELOT_EINVAL, "null argument");
    if (warmup < 0) return fail(CAMELOT_EINVAL, "warmup < 0");
    const size_t need = camelot_simulate_workspace_bytes(p, c, n_queries, n_sims);
    if (!need) return CAMELOT_EINVAL;
    if (!ex || ex->workspace_bytes < need) return fail(CAMELOT_ENOMEM, "workspace too small for the simulation (%zu bytes)", need);
    int rc = check_loads(p, load_qps, 1);
    if (rc) return rc;
    Ctx X;
    rc = setup(p, c, ex, 1, X, true);
    if (rc) return rc;
    unsigned long long x = 0;
    for (int a = 0; a < X.d.A; ++a) {
        int b = -1;
        for (int k = 0; k < X.d.nS; ++k)
            if (p->batch[k] == batch[a]) b = k;
        if (b < 0) return fail(CAMELOT_EINVAL, "batch %d of app %d is not on the batch grid", batch[a], a);
        x = x * X.d.nS + b;
    }
    for (int i = 0; i < X.d.n; ++i) {
        if (replicas[i] < 1 || replicas[i] > X.d.Rmax) return fail(CAMELOT_EINVAL, "replicas[%d] not in 1..Rmax", i);
        int t = -1;
        for (int k = 0; k < X.d.nQ; ++k)
            if (p->quota_pct[k] == quota_pct[i]) t = k;
        if (t < 0) return fail(CAMELOT_EINVAL, "quota %d of stage %d is not on the quota grid", quota_pct[i], i);
        x = x * X.d.Rmax + (replicas[i] - 1);
        x = x * X.d.nQ + t;
    }
    SimArgs A;
    memset(&A, 0, sizeof(A));
    A.x = x;
    for (int a = 0; a < X.d.A; ++a) A.lam[a] = load_qps[a];
    A.n_queries = n_queries;
    A.warmup = warmup;
    A.seed = seed;
    A.lat = reinterpret_cast<double *>(X.ws + X.L.total);
    A.out = reinterpret_cast<double *>(X.ws + X.L.total + al((size_t)n_sims * (size_t)n_queries * sizeof(double)));
    simulate_kernel<<<n_sims, 256, 0, X.st>>>(X.P, A);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    std::vector<double> h((size_t)n_sims * X.d.A * 2);
    CU(cudaMemcpyAsync(h.data(), A.out, h.size() * sizeof(double), cudaMemcpyDeviceToHost, X.st));
    CU(cudaStreamSynchronize(X.st));
    for (int sidx = 0; sidx < n_sims; ++sidx)
        for (int a = 0; a < X.d.A; ++a) {
            p99_ms[sidx * X.d.A + a] = h[((size_t)sidx * X.d.A + a) * 2];
            mean_ms[sidx * X.d.A + a] = h[((size_t)sidx * X.d.A + a) * 2 + 1];
        }
    return CAMELOT_OK;
}

int camelot_score_range(const camelot_problem *p, const camelot_cluster *c, uint64_t lo, uint64_t hi,
                        const camelot_exec *ex, uint8_t *d_verdict, float *d_T, int32_t *d_u, int32_t *d_U) {
    t_call_launches = 0;
    Ctx X;
    int rc = setup(p, c, ex, 1, X, true);
    if (rc) return rc;
    if (hi > X.d.ntot) hi = X.d.ntot;
    if (lo > hi) return fail(CAMELOT_EINVAL, "lo > hi");
    const unsigned long long cnt = hi - lo;
    if (cnt > (1ull << 31)) return fail(CAMELOT_ERANGE, "range longer than 2^31");
    if (cnt == 0) return CAMELOT_OK;
    const unsigned blocks = (unsigned)((cnt + 255) / 256);
    score_range_kernel<<<blocks, 256, 0, X.st>>>(X.P, lo, cnt, d_verdict, d_T, d_u, d_U);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    return CAMELOT_OK;
}

uint64_t camelot_kernel_launches(void) { return g_launches.load(); }

int camelot_sa(const camelot_problem *p, const camelot_cluster *c, int policy, const float *load_qps,
               uint64_t seed, int chains, int iters, float p0, float cool, const camelot_exec *ex,
               camelot_plan *out, uint64_t *d_chain_index, uint32_t *d_chain_key) {
    t_call_launches = 0;
    if (policy != 0 && policy != 1) return fail(CAMELOT_EINVAL, "bad policy");
    if (!out) return fail(CAMELOT_EINVAL, "null out");
    if (chains < 1 || chains > (1 << 20) || iters < 0) return fail(CAMELOT_EINVAL, "chains must be in 1..2^20, iters >= 0");
    if (!(p0 >= 0.0f && p0 <= 1.0f) || !(cool >= 0.0f && cool <= 1.0f)) return fail(CAMELOT_EINVAL, "p0, cool must be in [0,1]");
    if (policy == 1) {
        int rc = p ? check_loads(p, load_qps, 1) : fail(CAMELOT_EINVAL, "null problem");
        if (rc) return rc;
    }
    Ctx X;
    int rc = setup(p, c, ex, 1, X, true);
    if (rc) return rc;
    if (policy == 1) {
        rc = upload_loads(X, load_qps, 1);
        if (rc) return rc;
    }
    const int blocks = (chains + 255) / 256;
    if (blocks > MAXSLOTS) return fail(CAMELOT_ERANGE, "too many chains");
    char *ws = X.ws;
    DevHeader *hdr = reinterpret_cast<DevHeader *>(ws + X.L.hdr);
    CU(cudaMemsetAsync(hdr, 0, sizeof(DevHeader), X.st));
    SAArgs A;
    A.policy = policy;
    A.chains = chains;
    A.iters = iters;
    A.seed = seed;
    A.p0 = p0;
    A.cool = cool;
    A.lam = reinterpret_cast<const float *>(ws + X.L.lam);
    A.slots = reinterpret_cast<Slot *>(ws + slots_off(X.L));
    A.chain_index = reinterpret_cast<unsigned long long *>(d_chain_index);
    A.chain_key = d_chain_key;
    A.accepted = &hdr->n_nodes;   // reported as stats[1]
    sa_kernel<<<blocks, 256, 0, X.st>>>(X.P, A);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    Slot *winner = reinterpret_cast<Slot *>(ws + X.L.winner);
    reduce_kernel<<<1, 256, 0, X.st>>>(X.P, A.slots, blocks, 1, winner, reinterpret_cast<long long *>(ws + X.L.keys),
                                       nullptr, nullptr, nullptr, 0, 1, 0);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(ws + X.L.hdr2, ws + X.L.hdr, sizeof(DevHeader), cudaMemcpyDeviceToDevice, X.st));
    camelot_plan *dplans = reinterpret_cast<camelot_plan *>(ws + X.L.plans);
    plan_kernel<<<1, PLAN_THREADS, 0, X.st>>>(X.P, policy, 1, winner, reinterpret_cast<const float *>(ws + X.L.lam),
                                    reinterpret_cast<const DevHeader *>(ws + X.L.hdr2), dplans);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out, dplans, sizeof(camelot_plan), cudaMemcpyDeviceToHost, X.st));
    CU(cudaStreamSynchronize(X.st));
    out->n_scored = (uint64_t)chains * (uint64_t)(iters + 1);
    out->n_covered = out->n_scored;
    return out->status;
}

int camelot_last_stats(const camelot_exec *ex, uint64_t *out8) {
    if (!ex || !out8 || !ex->workspace) return fail(CAMELOT_EINVAL, "null argument");
    uint64_t *out6 = out8;
    float ms = 0.0f;
    if (t_ev.armed) {
        CU(cudaEventSynchronize(t_ev.b));
        CU(cudaEventElapsedTime(&ms, t_ev.a, t_ev.b));
    }
    // the saved header sits right after the live one (layout is problem independent here)
    DevHeader h;
    cudaStream_t st = static_cast<cudaStream_t>(ex->stream);
    CU(cudaMemcpyAsync(&h, static_cast<char *>(ex->workspace) + al(sizeof(DevHeader)), sizeof(h), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    out6[0] = h.n_scored;
    out6[1] = h.n_nodes;
    out6[2] = h.n_feasible;
    out6[3] = (uint64_t)((double)ms * 1e6);
    out6[4] = h.items_total;
    out6[5] = t_call_launches;
    out8[6] = h.cum_scored;
    out8[7] = h.cum_nodes;
    return CAMELOT_OK;
}

static int check_trees(int n_trees, const camelot_tree *trees, size_t &nodes) {
    nodes = 0;
    if (!trees || n_trees < 1) return fail(CAMELOT_EINVAL, "no trees");
    for (int t = 0; t < n_trees; ++t) {
        const camelot_tree &T = trees[t];
        if (T.n_nodes < 1 || !T.feature || !T.threshold || !T.left || !T.right || !T.value)
            return fail(CAMELOT_EINVAL, "tree %d: empty or null arrays", t);
        for (int k = 0; k < T.n_nodes; ++k) {
            const int f = T.feature[k];
            if (f < -1 || f > 1) return fail(CAMELOT_EINVAL, "tree %d node %d: feature must be -1, 0 or 1", t, k);
            if (f >= 0 && (T.left[k] <= k || T.left[k] >= T.n_nodes || T.right[k] <= k || T.right[k] >= T.n_nodes))
                return fail(CAMELOT_EINVAL, "tree %d node %d: children must lie in (k, n_nodes)", t, k);
            if (f < 0 && !std::isfinite(T.value[k])) return fail(CAMELOT_EINVAL, "tree %d node %d: non-finite leaf", t, k);
        }
        nodes += (size_t)T.n_nodes;
    }
    return CAMELOT_OK;
}

size_t camelot_trees_workspace_bytes(int n_trees, const camelot_tree *trees, int n_batch, int n_quota) {
    size_t nodes = 0;
    if (check_trees(n_trees, trees, nodes) || n_batch < 1 || n_quota < 1) return 0;
    return al(nodes * sizeof(int4)) + al(nodes * sizeof(float)) + al((n_trees + 1) * sizeof(int)) +
           al(n_batch * sizeof(int)) + al(n_quota * sizeof(int));
}

int camelot_tables_from_trees(int n_stages, const camelot_tree *trees, int n_batch, const int32_t *batch,
                              int n_quota, const int32_t *quota_pct, const camelot_exec *ex, float *d_table) {
    t_call_launches = 0;
    if (n_stages < 1 || n_stages > CAMELOT_MAX_STAGES) return fail(CAMELOT_EINVAL, "n_stages must be in 1..8");
    if (!batch || !quota_pct || !d_table || n_batch < 1 || n_quota < 1) return fail(CAMELOT_EINVAL, "empty grid or null");
    const int n_trees = 3 * n_stages;
    size_t nodes = 0;
    int rc = check_trees(n_trees, trees, nodes);
    if (rc) return rc;
    rc = device_ok(ex);
    if (rc) return rc;
    const size_t need = camelot_trees_workspace_bytes(n_trees, trees, n_batch, n_quota);
    if (ex->workspace_bytes < need) return fail(CAMELOT_ENOMEM, "workspace too small: %zu < %zu bytes", ex->workspace_bytes, need);
    std::vector<int4> hn(nodes);
    std::vector<float> hv(nodes);
    std::vector<int> hoff(n_trees + 1);
    size_t at = 0;
    for (int t = 0; t < n_trees; ++t) {
        hoff[t] = (int)at;
        for (int k = 0; k < trees[t].n_nodes; ++k, ++at) {
            hn[at] = make_int4(trees[t].feature[k], trees[t].threshold[k], trees[t].left[k], trees[t].right[k]);
            hv[at] = trees[t].value[k];
        }
    }
    hoff[n_trees] = (int)at;
    char *ws = static_cast<char *>(ex->workspace);
    cudaStream_t st = static_cast<cudaStream_t>(ex->stream);
    int4 *dn = reinterpret_cast<int4 *>(ws);
    float *dv = reinterpret_cast<float *>(ws + al(nodes * sizeof(int4)));
    int *doff = reinterpret_cast<int *>(ws + al(nodes * sizeof(int4)) + al(nodes * sizeof(float)));
    int *dS = reinterpret_cast<int *>(reinterpret_cast<char *>(doff) + al((n_trees + 1) * sizeof(int)));
    int *dQ = reinterpret_cast<int *>(reinterpret_cast<char *>(dS) + al(n_batch * sizeof(int)));
    CU(cudaMemcpyAsync(dn, hn.data(), nodes * sizeof(int4), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dv, hv.data(), nodes * sizeof(float), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(doff, hoff.data(), (n_trees + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dS, batch, n_batch * sizeof(int), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dQ, quota_pct, n_quota * sizeof(int), cudaMemcpyHostToDevice, st));
    const long long total = (long long)n_trees * n_batch * n_quota;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 4096);
    tree_table_kernel<<<blocks, 256, 0, st>>>(n_trees, dn, dv, doff, n_batch, dS, n_quota, dQ, d_table);
    COUNT_LAUNCH();
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(st));   // the host staging vectors die on return
    return CAMELOT_OK;
}

int camelot_trace(const camelot_exec *ex, uint64_t *out, int cap) {
    if (!ex || !out || cap < 0 || !ex->workspace) return fail(CAMELOT_EINVAL, "null argument");
    DevHeader h;
    cudaStream_t st = static_cast<cudaStream_t>(ex->stream);
    CU(cudaMemcpyAsync(&h, static_cast<char *>(ex->workspace) + al(sizeof(DevHeader)), sizeof(h), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    const int n = (int)std::min<unsigned>(h.trace_n, (unsigned)TRACE_MAX);
    for (int i = 0; i < n && i < cap; ++i) out[i] = h.trace[i];
    return n;
}

}  // extern "C"
