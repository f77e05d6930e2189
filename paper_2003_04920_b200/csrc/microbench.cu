// microbench.cu -- "achievable gather bandwidth" microkernels for the
// roofline denominators of SURVEY.md section 8(d): (i) a stream of CSR rows
// (idx i32 + cost f64) read in random row order, warp per row, and (ii)
// random 8-byte gathers from an n-sized array (L2- or HBM-resident).
// Measurement helpers only (include/pirrt_bench.h); not on the PI path.
#include <cuda_runtime.h>

#include <cstdint>

#include "pirrt_bench.h"

namespace {

__global__ void k_rows(const long long* __restrict__ off, const int* __restrict__ idx,
                       const double* __restrict__ cost, const int* __restrict__ order, int nrows,
                       double* sink) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (int r = w; r < nrows; r += nw) {
        const int v = order[r];
        const long long k0 = __ldg(&off[v]), k1 = __ldg(&off[v + 1]);
        for (long long k = k0 + lane; k < k1; k += 32) acc += __ldg(&cost[k]) + (double)__ldg(&idx[k]);
    }
    if (acc == -1.0) *sink = acc;   // keep the loads alive
}

// rows + g[u] gathers + a min per row (what one relaxation pass costs when
// nothing else happens): 20 B algorithmic per entry
__global__ void k_relax(const long long* __restrict__ off, const int* __restrict__ idx,
                        const double* __restrict__ cost, const double* __restrict__ g,
                        const int* __restrict__ order, int nrows, double* out) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = w; r < nrows; r += nw) {
        // order == nullptr: a fixed pseudo-random permutation (2^31 - 1 is
        // prime and larger than nrows)
        const int v = order ? order[r] : (int)(((long long)r * 2147483647LL) % nrows);
        const long long k0 = __ldg(&off[v]), k1 = __ldg(&off[v + 1]);
        double best = 1e300;
        for (long long k = k0 + lane; k < k1; k += 32) {
            const double cand = __ldg(&cost[k]) + __ldcg(&g[__ldg(&idx[k])]);
            best = cand < best ? cand : best;
        }
        for (int o = 16; o; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) out[v] = best;
    }
}

__global__ void k_gather(const double* __restrict__ src, const int* __restrict__ idx, long long n,
                         double* sink) {
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        acc += __ldcg(&src[__ldg(&idx[i])]);
    if (acc == -1.0) *sink = acc;
}

float time_it(void (*launch)(void*), void* arg, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch(arg);                                   // warm-up
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch(arg);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ms / reps;
}

struct RowsArg { const long long* off; const int* idx; const double* cost; const int* order; int n; double* sink; int blocks; };
struct RelaxArg { const long long* off; const int* idx; const double* cost; const double* g; const int* order; int n; double* out; int blocks; };
struct GatherArg { const double* src; const int* idx; long long n; double* sink; int blocks; };

}  // namespace

extern "C" {

int pirrt_bench_rows(const long long* off, const int* idx, const double* cost, const int* order,
                     int32_t nrows, int32_t reps, float* ms_out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return -3;
    RowsArg a{off, idx, cost, order, nrows, sink, sms * 8};
    *ms_out = time_it([](void* p) {
        RowsArg* r = (RowsArg*)p;
        k_rows<<<r->blocks, 256>>>(r->off, r->idx, r->cost, r->order, r->n, r->sink);
    }, &a, reps);
    cudaFree(sink);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

int pirrt_bench_relax(const long long* off, const int* idx, const double* cost, const double* g,
                      const int* order, int32_t nrows, double* out, int32_t reps, float* ms_out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    RelaxArg a{off, idx, cost, g, order, nrows, out, sms * 8};
    *ms_out = time_it([](void* p) {
        RelaxArg* r = (RelaxArg*)p;
        k_relax<<<r->blocks, 256>>>(r->off, r->idx, r->cost, r->g, r->order, r->n, r->out);
    }, &a, reps);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

int pirrt_bench_gather(const double* src, const int* idx, int64_t n, int32_t reps, float* ms_out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* sink;
    if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return -3;
    GatherArg a{src, idx, n, sink, sms * 8};
    *ms_out = time_it([](void* p) {
        GatherArg* g = (GatherArg*)p;
        k_gather<<<g->blocks, 256>>>(g->src, g->idx, g->n, g->sink);
    }, &a, reps);
    cudaFree(sink);
    return cudaGetLastError() == cudaSuccess ? 0 : -4;
}

}  // extern "C"
