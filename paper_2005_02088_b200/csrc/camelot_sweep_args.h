// camelot_sweep_args.h -- launch arguments of the exhaustive leaf-sweep kernel
// (camelot_sweep.cuh); shared with the host launcher in camelot_api.cu.
#pragma once
#include "camelot_device.cuh"

namespace cam {

constexpr unsigned SWEEP_TABL_MAX = 20 * 1024;   // staged leaf-stage rows (static smem ~25 KB: 2 CTAs/SM)

struct SweepArgs {
    int policy;                       // 0 max-load, 1 min-resource (one load level)
    int rank, world, d0;              // chunk ownership: chunk = (x / O^(n-d0)) / 64
    unsigned long long lo, hi;        // canonical index range [lo, hi)
    unsigned long long g_lo;          // first grandparent
    unsigned long long n_items;       // grandparents x nchunk
    int nchunk;                       // ceil(Os / 32) parent chunks per grandparent
    int ngroups;                      // work items per grandparent (gpack == 1): chunk ranges that
                                      // share one placement of the grandparent
    unsigned long long gp_split;      // grandparents [0, gp_split) in ngroups items each, the rest
    unsigned long long n_grp_items;   // (the tail of the scan) one item per chunk; = gp_split * ngroups
    int gpack;                        // grandparents per warp item: 1, or 32 / Os when Os <= 16
                                      // (lane = (grandparent, parent) pair; nchunk = 1)
    unsigned long long n_gp;          // grandparents in [g_lo, g_lo + n_gp) (bound for gpack > 1)
    int qstride;                      // quota sub-grid: every qstride-th quota from the top (1 = all)
    int nQs;                          // sub-grid size (nQ - 1) / qstride + 1; Os = Rmax * nQs
    const float *lam;                 // [A] load level (min-resource)
    const int *y;                     // Eq. 2 estimates [nbc][ystride] at + yoff
    int ystride, yoff;
    const Slot *inc;                  // incumbent (key, x) (none: key 0xFFFFFFFF)
    Slot *slots;                      // [gridDim.x]
    DevHeader *hdr;
    Slot *result;                     // exact local best
    long long *keys;                  // packed key (NCCL transport)
    unsigned tabL_bytes;              // leaf-stage table rows staged in shared memory (0: read global)
    int bp_min_nqs;                   // quota breakpoints only for sub-grids of >= this many quotas
};

}  // namespace cam
