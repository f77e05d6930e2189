// barrier_bench.cu -- measures the cost of one grid-wide barrier on this GPU
// (cooperative_groups grid.sync vs a hand-rolled generation barrier), for
// several grid sizes.  Design input for the persistent exploit kernel
// (DESIGN.md section 6).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o /tmp/barrier_bench tools/barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_cg(int iters) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}

// generation barrier: one arrival atomic per block, spin on the generation word
__device__ __forceinline__ void gen_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks,
                                            unsigned& my_gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned target = my_gen + 1;
        __threadfence();
        const unsigned arrived = atomicAdd(count, 1u) + 1u;
        if (arrived == nblocks * target) {
            *gen = target;
        } else {
            unsigned g;
            do {
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(gen));
            } while (g < target);
        }
        my_gen = target;
    }
    __syncthreads();
}

__global__ void k_gen(int iters, unsigned* count, unsigned* gen) {
    unsigned my_gen = 0;
    for (int i = 0; i < iters; ++i) gen_barrier(count, gen, gridDim.x, my_gen);
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    unsigned *count, *gen;
    cudaMalloc(&count, 4);
    cudaMalloc(&gen, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000;
    for (int threads : {256, 512, 1024}) {
        for (int mult : {1, 2}) {
            int blocks = sms * mult;
            if (threads * mult > 2048) continue;
            for (int kind = 0; kind < 2; ++kind) {
                float best = 1e30f;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaMemset(count, 0, 4);
                    cudaMemset(gen, 0, 4);
                    int it = iters;
                    void* args_cg[] = {&it};
                    void* args_gen[] = {&it, &count, &gen};
                    cudaEventRecord(e0);
                    cudaError_t err;
                    if (kind == 0)
                        err = cudaLaunchCooperativeKernel((void*)k_cg, blocks, threads, args_cg, 0, 0);
                    else
                        err = cudaLaunchCooperativeKernel((void*)k_gen, blocks, threads, args_gen, 0, 0);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    if (err != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(err)); break; }
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                printf("%-6s blocks=%4d threads=%4d : %.3f us per barrier\n", kind ? "gen" : "cg",
                       blocks, threads, 1e3f * best / iters);
            }
        }
    }
    // single block __syncthreads reference
    return 0;
}
