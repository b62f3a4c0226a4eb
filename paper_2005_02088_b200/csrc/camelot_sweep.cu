// camelot_sweep.cu -- instantiations and the host launcher of the exhaustive
// leaf-sweep kernel (camelot_sweep.cuh).  Its own translation unit so that it
// compiles in parallel with camelot_api.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "../../include/camelot.h"
#include "camelot_sweep.cuh"

namespace cam {

namespace {
std::mutex g_mu;
int g_grid[64][8][2][2];   // [device][NS][policy][two apps] persistent grid (0 = unknown)

template <int NS, int POL, bool TWO>
cudaError_t launch_ns(const DevProb &P, const SweepArgs &A, int dev, cudaStream_t st) {
    int grid = 0;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        int &gg = g_grid[dev & 63][NS - 1][POL][TWO];
        if (!gg) {
            int per = 0, nsm = 0;
            cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sweep_kernel<8, NS, POL, TWO>, SWEEP_THREADS, 0);
            if (e != cudaSuccess) return e;
            e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            if (e != cudaSuccess) return e;
            gg = std::max(1, std::min(4096, per * nsm));
        }
        grid = gg;
    }
    sweep_kernel<8, NS, POL, TWO><<<grid, SWEEP_THREADS, 0, st>>>(P, A);
    return cudaGetLastError();
}

template <int POL, bool TWO>
cudaError_t launch_pol(const DevProb &P, const SweepArgs &A, int dev, cudaStream_t st) {
    switch (P.n) {
        case 2: return launch_ns<2, POL, TWO>(P, A, dev, st);
        case 3: return launch_ns<3, POL, TWO>(P, A, dev, st);
        case 4: return launch_ns<4, POL, TWO>(P, A, dev, st);
        case 5: return launch_ns<5, POL, TWO>(P, A, dev, st);
        case 6: return launch_ns<6, POL, TWO>(P, A, dev, st);
        default: return launch_ns<8, POL, TWO>(P, A, dev, st);
    }
}
}  // namespace

// Whether the sweep handles this problem (else the tree search runs flat).
bool sweep_supported(const DevProb &P, int policy, int nlev) {
    return P.n >= 2 && P.n <= NMAX && P.C <= 8 && P.Rmax <= 4 && nlev == 1 && (policy == 0 || policy == 1) &&
           !(P.flags & (F_PAPER_GLOBAL | F_SAT));
}

cudaError_t sweep_launch(const DevProb &P, const SweepArgs &A, int dev, cudaStream_t st) {
    if (P.A > 1) return A.policy == 0 ? launch_pol<0, true>(P, A, dev, st) : launch_pol<1, true>(P, A, dev, st);
    return A.policy == 0 ? launch_pol<0, false>(P, A, dev, st) : launch_pol<1, false>(P, A, dev, st);
}

}  // namespace cam
