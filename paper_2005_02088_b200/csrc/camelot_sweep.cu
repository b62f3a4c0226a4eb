// camelot_sweep.cu -- instantiations and the host launcher of the exhaustive
// leaf-sweep kernel (camelot_sweep.cuh).  Its own translation unit so that it
// compiles in parallel with camelot_api.cu.
#include <cuda_runtime.h>


#include "../../include/camelot.h"
#include "camelot_sweep_launch.cuh"

namespace cam {

cudaError_t sweep_launch_comm(const DevProb &P, const SweepArgs &A, int dev, cudaStream_t st);   // camelot_sweep_comm.cu


// Whether the sweep handles this problem (else the tree search runs flat).
bool sweep_supported(const DevProb &P, int policy, int nlev) {
    return P.n >= 2 && P.n <= NMAX && P.C <= 8 && P.Rmax <= 4 && nlev == 1 && (policy == 0 || policy == 1) &&
           !(P.flags & (F_PAPER_GLOBAL | F_SAT));
}

cudaError_t sweep_launch(const DevProb &P, const SweepArgs &A, int dev, cudaStream_t st) {
    return (P.flags & F_COMM) ? sweep_launch_comm(P, A, dev, st) : launch_comm<false>(P, A, dev, st);
}

}  // namespace cam
