// camelot_inst.cuh -- host launchers of the templated search kernels
// (search_kernel, search_level_kernel) per compile-time width (CM positions,
// NS stages) and policy.  camelot_api.cu sees only the declarations; the
// definitions are instantiated in camelot_inst_*.cu, several translation units
// that compile in parallel (the kernels are large).
#pragma once
#include <cuda_runtime.h>

#include "camelot_kernels.cuh"

namespace cam {

// occupancy (resident CTAs per SM) with `sm` bytes of dynamic shared memory; sets the
// kernel's dynamic shared-memory limit first
template <int CM, int NS, int POL> cudaError_t k_search_occupancy(size_t sm, int *per);
template <int CM, int NS, int POL> cudaError_t k_level_occupancy(size_t sm, int *per);
// one launch on stream st (the level kernel is cooperative: all CTAs co-resident)
template <int CM, int NS, int POL>
cudaError_t k_search_launch(const DevProb &P, const SearchArgs &S, int grid, size_t sm, cudaStream_t st);
template <int CM, int NS, int POL>
cudaError_t k_level_launch(const DevProb &P, const LevelSet &LS, int grid, size_t sm, cudaStream_t st);

#ifdef CAMELOT_INST_TU
template <int CM, int NS, int POL> cudaError_t k_search_occupancy(size_t sm, int *per) {
    cudaError_t e = cudaFuncSetAttribute(search_kernel<CM, NS, POL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per, search_kernel<CM, NS, POL>, SEARCH_THREADS, sm);
}
template <int CM, int NS, int POL> cudaError_t k_level_occupancy(size_t sm, int *per) {
    cudaError_t e =
        cudaFuncSetAttribute(search_level_kernel<CM, NS, POL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per, search_level_kernel<CM, NS, POL>, SEARCH_THREADS, sm);
}
template <int CM, int NS, int POL>
cudaError_t k_search_launch(const DevProb &P, const SearchArgs &S, int grid, size_t sm, cudaStream_t st) {
    search_kernel<CM, NS, POL><<<grid, SEARCH_THREADS, sm, st>>>(P, S);
    return cudaGetLastError();
}
template <int CM, int NS, int POL>
cudaError_t k_level_launch(const DevProb &P, const LevelSet &LS, int grid, size_t sm, cudaStream_t st) {
    void *args[] = {(void *)&P, (void *)&LS};
    return cudaLaunchCooperativeKernel((const void *)search_level_kernel<CM, NS, POL>, dim3(grid),
                                       dim3(SEARCH_THREADS), args, sm, st);
}
#define CAMELOT_INSTANTIATE(CM, NS, POL)                                                                        \
    template cudaError_t k_search_occupancy<CM, NS, POL>(size_t, int *);                                       \
    template cudaError_t k_level_occupancy<CM, NS, POL>(size_t, int *);                                        \
    template cudaError_t k_search_launch<CM, NS, POL>(const DevProb &, const SearchArgs &, int, size_t,        \
                                                      cudaStream_t);                                           \
    template cudaError_t k_level_launch<CM, NS, POL>(const DevProb &, const LevelSet &, int, size_t, cudaStream_t);
#endif

}  // namespace cam
