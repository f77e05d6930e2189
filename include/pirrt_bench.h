/*
 * pirrt_bench.h -- measurement helpers of libpirrt (not part of the PI path):
 * the "achievable gather bandwidth" microkernels of SURVEY.md section 8(d).
 * All pointers are device pointers; calls run on the default stream and
 * return 0, or -3 (allocation) / -4 (CUDA error).  *ms_out = mean time of
 * one pass over `reps` passes (CUDA events, after one warm-up pass).
 */
#ifndef PIRRT_BENCH_H
#define PIRRT_BENCH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Stream whole CSR rows (idx i32 + cost f64 per entry, rows [off[v], off[v+1]))
 * visiting the rows in the given order (warp per row): 12 B per entry. */
int pirrt_bench_rows(const long long* off, const int* idx, const double* cost, const int* order,
                     int32_t nrows, int32_t reps, float* ms_out);

/* One relaxation pass: rows in `order` (warp per row), out[v] = min over the
 * row of cost + g[idx] -- 12 B streamed + one 8 B gather per entry. */
int pirrt_bench_relax(const long long* off, const int* idx, const double* cost, const double* g,
                      const int* order, int32_t nrows, double* out, int32_t reps, float* ms_out);

/* The same relaxation pass over a context's own base CSR (rows in a fixed
 * pseudo-random order, g = the context's cost-to-come): the achievable rate
 * on exactly the graph the exploit runs on.  *entries_out = entries per pass.
 * Runs on the context's device after completing its pending work. */
typedef struct pirrt_ctx pirrt_ctx;
int pirrt_bench_relax_ctx(const pirrt_ctx* ctx, int32_t reps, float* ms_out, int64_t* entries_out);

/* n random 8-byte gathers src[idx[i]] (idx streamed): 4 B + one 8 B gather each. */
int pirrt_bench_gather(const double* src, const int* idx, int64_t n, int32_t reps, float* ms_out);

#ifdef __cplusplus
}
#endif
#endif
