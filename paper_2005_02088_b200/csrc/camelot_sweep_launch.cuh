// camelot_sweep_launch.cuh -- host-side launch templates of the leaf sweep
// (persistent grid per instantiation, dispatch on n / policy / applications).
// Included by camelot_sweep.cu (F_COMM off) and camelot_sweep_comm.cu (F_COMM
// on), two translation units that compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "../../include/camelot.h"
#include "camelot_sweep.cuh"

namespace cam {

namespace {
std::mutex g_mu;
int g_grid[64][8][2][2][2];   // [device][NS][policy][two apps][comm] persistent grid (0 = unknown)

template <int NS, int POL, bool TWO, bool COMM>
cudaError_t launch_ns(const DevProb &P, const SweepArgs &A, int dev, cudaStream_t st) {
    int grid = 0;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int &gg = g_grid[dev & 63][NS - 1][POL][TWO][COMM];
        if (!gg) {
            int per = 0, nsm = 0;
            cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sweep_kernel<8, NS, POL, TWO, COMM>,
                                                                          SWEEP_THREADS, SWEEP_TABL_MAX);
            if (e != cudaSuccess) return e;
            e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            if (e != cudaSuccess) return e;
            gg = std::max(1, std::min(4096, per * nsm));
        }
        grid = gg;
    }
    // small scans (the coarsest cascade level): at most one work item per warp -- idle
    // CTAs only add to the end-of-kernel reduction (testing knob CAMELOT_SWEEP_FIT=0)
    static const bool fit = !(getenv("CAMELOT_SWEEP_FIT") && getenv("CAMELOT_SWEEP_FIT")[0] == '0');
    if (fit) {
        const unsigned long long per_cta = SWEEP_THREADS / 32;
        grid = (int)std::max(1ull, std::min((unsigned long long)grid, (A.n_items + per_cta - 1) / per_cta));
    }
    sweep_kernel<8, NS, POL, TWO, COMM><<<grid, SWEEP_THREADS, A.tabL_bytes, st>>>(P, A);
    return cudaGetLastError();
}

template <int POL, bool TWO, bool COMM>
cudaError_t launch_pol(const DevProb &P, const SweepArgs &A, int dev, cudaStream_t st) {
    switch (P.n) {
        case 2: return launch_ns<2, POL, TWO, COMM>(P, A, dev, st);
        case 3: return launch_ns<3, POL, TWO, COMM>(P, A, dev, st);
        case 4: return launch_ns<4, POL, TWO, COMM>(P, A, dev, st);
        case 5: return launch_ns<5, POL, TWO, COMM>(P, A, dev, st);
        case 6: return launch_ns<6, POL, TWO, COMM>(P, A, dev, st);
        default: return launch_ns<8, POL, TWO, COMM>(P, A, dev, st);
    }
}

template <bool COMM>
cudaError_t launch_comm(const DevProb &P, const SweepArgs &A, int dev, cudaStream_t st) {
    if (P.A > 1) return A.policy == 0 ? launch_pol<0, true, COMM>(P, A, dev, st) : launch_pol<1, true, COMM>(P, A, dev, st);
    return A.policy == 0 ? launch_pol<0, false, COMM>(P, A, dev, st) : launch_pol<1, false, COMM>(P, A, dev, st);
}
}  // namespace

}  // namespace cam
