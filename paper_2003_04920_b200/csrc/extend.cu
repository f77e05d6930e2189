// extend.cu -- device-side Extend: the
// exploration half of a BE-RRT# batch on the GPU, so that a batch crosses
// PCIe as S sample points instead of ~2 x S x degree edge triples.
//
// PAPER.md:182-188 (Extend: "the new vertex is connected to all vertices
// within the connection radius ... a small exploitation determines whether the
// new vertex is promising") and the RRG rule the workloads use (DESIGN.md
// section 4): new vertex i connects to every earlier j < i with
// |x_i - x_j| <= r(i+1) whose segment misses every axis-aligned box (slab
// test); cost = |x_i - x_j| (fp64, squared differences summed in coordinate
// order, IEEE sqrt); h(i) = |x_i - x_goal|.  The radii r(i+1) are computed on
// the host (abi.cu) and passed in, so every decision is an IEEE comparison.
//
// Kernels: a uniform grid of cell side >= the batch's largest radius over all
// points so far (cell id, histogram, scan, scatter), then one warp per new
// vertex over its 3^d neighbour cells (cells the R-ball misses dropped),
// twice -- count, then write the COO triples (src = j, dst = i, cost) at
// scanned offsets.  The triples feed the
// ordinary append (a1) with device pointers; nothing is committed here.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "internal.cuh"

namespace pirrt {
namespace {

constexpr int kXT = 256;

inline int xgrid(long long n, int bt = kXT, int cap = 148 * 16) {
    long long g = (n + bt - 1) / bt;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

__device__ __forceinline__ int cell_coord(double x, int m) {
    int c = (int)floor(x * m);
    return c < 0 ? 0 : (c >= m ? m - 1 : c);
}

__global__ void k_cell_of(const double* pts, int n, int d, int m, int* cell) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        long long c = 0;
        for (int k = 0; k < d; ++k) c = c * m + cell_coord(pts[(long long)i * d + k], m);
        cell[i] = (int)c;
    }
}

__global__ void k_cell_count(const int* cell, int n, long long* cnt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd((unsigned long long*)&cnt[cell[i]], 1ull);
}

__global__ void k_cell_scatter(const int* cell, int n, long long* cur, int* cpts) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        cpts[atomicAdd((unsigned long long*)&cur[cell[i]], 1ull)] = i;
}

// h of the new vertices: |x - x_goal| (admissible heuristic)
__global__ void k_new_h(const double* pts, int n_old, int n_new, int d, const double* xg, double* h) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_new; t += gridDim.x * blockDim.x) {
        const double* p = pts + (long long)(n_old + t) * d;
        double s = 0.0;
        for (int k = 0; k < d; ++k) {
            const double u = p[k] - xg[k];
            s += u * u;
        }
        h[t] = sqrt(s);
    }
}

// segment q -> p meets the closed box [lo, hi] (slab test)
__device__ __forceinline__ bool seg_hits_box(const double* q, const double* p, const double* box,
                                             int d) {
    double t0 = 0.0, t1 = 1.0;
    for (int k = 0; k < d; ++k) {
        const double lo = box[k], hi = box[d + k];
        const double dk = p[k] - q[k];
        if (dk == 0.0) {
            if (q[k] < lo || q[k] > hi) return false;
            continue;
        }
        double ta = (lo - q[k]) / dk, tb = (hi - q[k]) / dk;
        if (ta > tb) { const double x = ta; ta = tb; tb = x; }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
        if (t0 > t1) return false;
    }
    return true;
}

// one warp per new vertex i = n_old + t: every earlier j in the 3^d cells
// around x_i (or all j < i when brute) with |x_i - x_j| <= R_t and a free
// segment.  WRITE = false: count into cnt[t]; true: write at off[t].
// The stencil is taken 32 cells at a time (one per lane): a lane drops a
// cell the R-ball misses and loads the range of a kept one; the candidates
// of the kept cells, concatenated by a warp scan of their counts, are then
// tested 32 at a time (owner cell of a candidate by a binary search over the
// lanes' prefix), so every lane works whatever the cell occupancy.
template <bool WRITE>
// 4 blocks per SM (64 registers, no spill): the count pass is bound by the
// latency of its candidate gathers, so resident warps matter (ncu: 68
// registers and 3 blocks before; profiles/r2/extend_count_ncu.json)
__global__ void __launch_bounds__(kXT, 4) k_neighbours(const double* __restrict__ pts, int n_old, int n_new, int d, int m,
                             int brute, const long long* __restrict__ cstart,
                             const int* __restrict__ cpts, const double* __restrict__ R,
                             const double* __restrict__ boxes, int n_boxes, long long* cnt,
                             const long long* __restrict__ off, int* src, int* dst, double* cost,
                             int hcap, int* __restrict__ hj, double* __restrict__ hd) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    unsigned lt;
    asm("mov.u32 %0, %lanemask_lt;" : "=r"(lt));
    for (int t = w; t < n_new; t += nw) {                 // warp-uniform
        const int i = n_old + t;
        const double* p = pts + (long long)i * d;
        const double Ri = R[t];
        const double R2cut = Ri * Ri * (1.0 + 1e-9);      // conservative: never prunes a neighbour
        const double inv_m = 1.0 / m;
        long long found = 0;
        const long long base = WRITE ? off[t] : 0;
        if (WRITE && hcap > 0 && off[t + 1] - base <= hcap) {
            // every hit is in the count pass's cache, in output order
            const int nh = (int)(off[t + 1] - base);
            const long long h0 = (long long)t * hcap;
            for (int k = lane; k < nh; k += 32) {
                src[base + k] = hj[h0 + k]; dst[base + k] = i; cost[base + k] = hd[h0 + k];
            }
            continue;
        }
        int lo[16], rad[16];
        int N = 1;
        if (!brute) {
            for (int k = 0; k < d; ++k) {
                const int c = cell_coord(p[k], m);
                lo[k] = c > 0 ? c - 1 : 0;
                rad[k] = (c < m - 1 ? c + 1 : m - 1) - lo[k] + 1;
                N *= rad[k];
            }
        }
        for (int s0 = 0; s0 < N; s0 += 32) {
            // this lane's stencil cell
            long long a0 = 0;
            int len = 0;
            const int sidx = s0 + lane;
            if (brute) {
                if (lane == 0) len = i;                   // all j < i, in id order
            } else if (sidx < N) {
                int r = sidx;
                long long c = 0;
                double gap2 = 0.0;                        // squared distance from x_i to the closed cell
                for (int k = d - 1; k >= 0; --k) {        // mixed-radix digits, last axis fastest
                    const int cc = lo[k] + r % rad[k];
                    r /= rad[k];
                    const double clo = cc * inv_m, chi = (cc + 1) * inv_m;
                    const double g = p[k] < clo ? clo - p[k] : (p[k] > chi ? p[k] - chi : 0.0);
                    gap2 += g * g;
                }
                if (gap2 <= R2cut) {
                    r = sidx;
                    long long mult = 1;
                    for (int k = d - 1; k >= 0; --k) {
                        c += (long long)(lo[k] + r % rad[k]) * mult;
                        r /= rad[k];
                        mult *= m;
                    }
                    a0 = cstart[c];
                    len = (int)(cstart[c + 1] - a0);
                }
            }
            int incl = len;                               // warp scan of the candidate counts
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int excl = incl - len;
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            for (int k0 = 0; k0 < total; k0 += 32) {       // warp-uniform
                const int k = k0 + lane;
                int own = 0;                              // last lane whose prefix <= k
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const int cand = own + step;
                    const int ex = __shfl_sync(0xffffffffu, excl, cand);
                    if (ex <= k) own = cand;
                }
                const long long ba = __shfl_sync(0xffffffffu, a0, own);
                const int be = __shfl_sync(0xffffffffu, excl, own);
                bool hit = false;
                int j = -1;
                double dd = 0.0;
                if (k < total) {
                    const long long e = ba + (k - be);
                    j = brute ? (int)e : cpts[e];
                    if (j < i) {
                        const double* q = pts + (long long)j * d;
                        double s2 = 0.0;
                        for (int kk = 0; kk < d; ++kk) {
                            const double u = p[kk] - q[kk];
                            s2 += u * u;
                        }
                        dd = sqrt(s2);
                        if (!(dd > Ri)) {
                            hit = true;
                            for (int b = 0; b < n_boxes && hit; ++b)
                                if (seg_hits_box(q, p, boxes + (long long)b * 2 * d, d)) hit = false;
                        }
                    }
                }
                const unsigned mask = __ballot_sync(0xffffffffu, hit);
                if (WRITE && hit) {
                    const long long o = base + found + __popc(mask & lt);
                    src[o] = j; dst[o] = i; cost[o] = dd;
                }
                if (!WRITE && hit && hcap > 0) {
                    const long long o = found + __popc(mask & lt);
                    if (o < hcap) { hj[(long long)t * hcap + o] = j; hd[(long long)t * hcap + o] = dd; }
                }
                found += __popc(mask);
            }
            if (brute) break;
        }
        if (!WRITE && lane == 0) cnt[t] = found;
    }
}

}  // namespace

cudaError_t launch_extend_grid(const ExtendArgs& a, cudaStream_t s) {
    // cell ids of every point [0, n_all), histogram, exclusive scan, scatter
    const int n_all = a.n_old + a.n_new;
    cudaError_t e;
    if (!a.brute) {
        ++g_kernel_launches;
        k_cell_of<<<xgrid(n_all), kXT, 0, s>>>(a.pts, n_all, a.d, a.m, a.cell);
        if ((e = cudaMemsetAsync(a.ccnt, 0, sizeof(long long) * (a.ncell + 1), s)) != cudaSuccess) return e;
        ++g_kernel_launches;
        k_cell_count<<<xgrid(n_all), kXT, 0, s>>>(a.cell, n_all, a.ccnt);
        if ((e = scan_exclusive(a.ccnt, a.cstart, a.ncell, a.scan_tmp, s)) != cudaSuccess) return e;
        if ((e = cudaMemcpyAsync(a.ccnt, a.cstart, sizeof(long long) * a.ncell, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
        ++g_kernel_launches;
        k_cell_scatter<<<xgrid(n_all), kXT, 0, s>>>(a.cell, n_all, a.ccnt, a.cpts);
    }
    ++g_kernel_launches;
    k_new_h<<<xgrid(a.n_new), kXT, 0, s>>>(a.pts, a.n_old, a.n_new, a.d, a.x_goal, a.h_new);
    ++g_kernel_launches;
    k_neighbours<false><<<xgrid((long long)a.n_new * 32), kXT, 0, s>>>(
        a.pts, a.n_old, a.n_new, a.d, a.m, a.brute, a.cstart, a.cpts, a.R, a.boxes, a.n_boxes,
        a.ecnt, nullptr, nullptr, nullptr, nullptr, a.hcap, a.hj, a.hd);
    if ((e = scan_exclusive(a.ecnt, a.eoff, a.n_new, a.scan_tmp, s)) != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_extend_edges(const ExtendArgs& a, cudaStream_t s) {
    ++g_kernel_launches;
    k_neighbours<true><<<xgrid((long long)a.n_new * 32), kXT, 0, s>>>(
        a.pts, a.n_old, a.n_new, a.d, a.m, a.brute, a.cstart, a.cpts, a.R, a.boxes, a.n_boxes,
        nullptr, a.eoff, a.src, a.dst, a.cost, a.hcap, a.hj, a.hd);
    return cudaGetLastError();
}

}  // namespace pirrt
