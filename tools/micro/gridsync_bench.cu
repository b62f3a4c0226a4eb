// Micro-benchmark (development aid): cost of one grid-wide barrier on the B200 with
// the search's cooperative geometry (148 CTAs x 256 threads): cooperative_groups
// grid.sync() vs a minimal sense-reversing barrier (one atomic per CTA, acquire spin).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}

__device__ unsigned int g_count = 0;
__device__ volatile unsigned int g_gen = 0;
__global__ void k_custom(int iters) {
    unsigned int gen = 0;
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            gen = g_gen;
            __threadfence();
            if (atomicAdd(&g_count, 1u) == gridDim.x - 1) {
                g_count = 0;
                __threadfence();
                g_gen = gen + 1;
            } else {
                unsigned int v;
                do {
                    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"((const unsigned int *)&g_gen));
                } while (v == gen);
            }
        }
        __syncthreads();
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int t = 256; t <= 256; t *= 2) {
        for (int rep = 0; rep < 3; ++rep) {
            int iters = 2000;
            void *args[] = {&iters};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void *)k_cg, nsm, t, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("cg grid.sync: %d CTAs x %d: %.3f us per barrier\n", nsm, t, ms * 1e3 / iters);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void *)k_custom, nsm, t, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("custom barrier: %d CTAs x %d: %.3f us per barrier (%s)\n", nsm, t, ms * 1e3 / iters,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
