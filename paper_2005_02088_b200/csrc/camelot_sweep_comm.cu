// camelot_sweep_comm.cu -- the leaf-sweep instantiations with the NEXT-2
// communication-aware QoS (F_COMM); a translation unit of its own so that it
// compiles in parallel with camelot_sweep.cu.
#include "camelot_sweep_launch.cuh"

namespace cam {

cudaError_t sweep_launch_comm(const DevProb &P, const SweepArgs &A, int dev, cudaStream_t st) {
    return launch_comm<true>(P, A, dev, st);
}

}  // namespace cam
