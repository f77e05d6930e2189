// store.cu -- the device-resident in-edge graph store and its append path
// (row a1 of SURVEY.md section 8(a)).
//
// Layout: in-edge rows by destination vertex, stored
// as a BASE CSR (boff i64[n+1], bidx i32[], bcost f64[]) plus a DELTA CSR of
// the same shape holding every edge appended since the last compaction.
// The paper rebuilds one CSR per Replan by radix sort + merge of the new
// edges, O(|E|) per replan; here an append costs
// O(n + |delta| + m) (counting-sort merge of the new edges into the delta)
// and the delta is folded into the base when it exceeds a fraction of it
// (geometric, amortised O(1) per edge).  Row order inside a row is not
// significant: Improve takes a lexicographic (cost, id) minimum.
//
// Every kernel that writes committed state is gated on ctl->err == 0, and
// the append path writes only locations that are invisible until the host
// commits (the inactive delta buffers and vertex slots >= n_old), so a
// rejected batch leaves the context unchanged.
#include <cooperative_groups.h>

#include <climits>
#include <cmath>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace pirrt {
namespace {

constexpr int kBT = 256;      // block size of the plain kernels
constexpr int kCopyChunk = kAppendCopyChunk;   // old-delta entries per copy chunk (append P4)
constexpr int kScanTile = 2048;

inline int grid_for(long long n, int bt = kBT, int cap = 148 * 16) {
    long long g = (n + bt - 1) / bt;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

__device__ __forceinline__ bool failed(const DevCtl* c) { return *(volatile const int*)&c->err != 0; }

// ------------------------------------------------------------------ scan
__global__ void k_scan_reduce(const long long* in, long long L, long long* part) {
    __shared__ long long sm[kBT / 32];
    const long long base = (long long)blockIdx.x * kScanTile;
    long long s = 0;
    for (int i = threadIdx.x; i < kScanTile; i += kBT) {
        long long j = base + i;
        if (j < L) s += in[j];
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < kBT / 32; ++w) t += sm[w];
        part[blockIdx.x] = t;
    }
}

// single block: exclusive scan of the partials in place; part[P] = total
__global__ void k_scan_partials(long long* part, long long P) {
    __shared__ long long carry;
    __shared__ long long sm[kBT / 32 + 1];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (long long base = 0; base < P; base += kBT) {
        long long i = base + threadIdx.x;
        long long x = i < P ? part[i] : 0;
        long long inc = x;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) sm[w] = inc;
        __syncthreads();
        if (threadIdx.x == 0) {
            long long r = 0;
            for (int k = 0; k < kBT / 32; ++k) { long long t = sm[k]; sm[k] = r; r += t; }
            sm[kBT / 32] = r;
        }
        __syncthreads();
        if (i < P) part[i] = carry + sm[w] + inc - x;
        __syncthreads();
        if (threadIdx.x == 0) carry += sm[kBT / 32];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[P] = carry;
}

__global__ void k_scan_apply(const long long* in, long long L, const long long* part, long long* out) {
    __shared__ long long sm[kBT / 32 + 1];
    __shared__ long long carry;
    const long long base = (long long)blockIdx.x * kScanTile;
    if (threadIdx.x == 0) carry = part[blockIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int t = 0; t < kScanTile; t += kBT) {
        long long i = base + t + threadIdx.x;
        long long x = i < L ? in[i] : 0;
        long long inc = x;
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) sm[w] = inc;
        __syncthreads();
        if (threadIdx.x == 0) {
            long long r = 0;
            for (int k = 0; k < kBT / 32; ++k) { long long q = sm[k]; sm[k] = r; r += q; }
            sm[kBT / 32] = r;
        }
        __syncthreads();
        if (i < L) out[i] = carry + sm[w] + inc - x;
        __syncthreads();
        if (threadIdx.x == 0) carry += sm[kBT / 32];
        __syncthreads();
    }
}

__global__ void k_set_ll(long long* p, long long v) { *p = v; }

// warp per new vertex with a given parent: pc(v) = cost of the stored edge
// (parent -> v); its absence is an error.  VALIDATE: g_new == g[p] + pc.
__global__ void k_find_pc(const long long* boff, const int* bidx, const double* bcost,
                          const long long* doff, const int* didx, const double* dcost,
                          const int* parent, const double* g, double* pc, int v0, int v1,
                          int validate, DevCtl* ctl) {
    if (failed(ctl)) return;
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int v = v0 + w; v < v1; v += nw) {
        const int p = parent[v];
        if (p < 0) continue;
        // the lowest stored position holding p (duplicates are the caller's problem)
        long long best = LLONG_MAX;
        double c = 0.0;
        for (long long k = boff[v] + lane; k < boff[v + 1]; k += 32)
            if (bidx[k] == p && k < best) { best = k; c = bcost[k]; }
        for (long long k = doff[v] + lane; k < doff[v + 1]; k += 32)
            if (didx[k] == p && (1LL << 62) + k < best) { best = (1LL << 62) + k; c = dcost[k]; }
        for (int o = 16; o; o >>= 1) {
            long long ob = __shfl_xor_sync(kFull, best, o);
            double oc = __shfl_xor_sync(kFull, c, o);
            if (ob < best) { best = ob; c = oc; }
        }
        if (lane == 0) {
            if (best == LLONG_MAX) atomicOr(&ctl->err, kErrPcMissing);
            else {
                pc[v] = c;
                if (validate && g[v] != g[p] + c) atomicOr(&ctl->err, kErrGNew);
            }
        }
    }
}

// B list rebuild (set_policy): flags then scan then scatter in id order
__global__ void k_b_flags(const unsigned char* b, int n, long long* cnt) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        cnt[v] = (v != kRoot && b[v] == 1) ? 1 : 0;
}

__global__ void k_b_scatter(const unsigned char* b, int n, const long long* off, int* list,
                            int* count_out) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        if (v != kRoot && b[v] == 1) list[1 + off[v]] = v;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        list[0] = kRoot;
        *count_out = (int)off[n];
    }
}

// ------------------------------------------------------------------ compaction
__device__ __forceinline__ bool row_kept(int v, int own_n, int own_r) {
    return own_n <= 1 || v % own_n == own_r;
}

// row lengths of the merged store, and the first row of every
// kCopyChunk-entry chunk of the base and of the delta (k_base_merge)
__global__ void k_base_count(CompactArgs a) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * blockDim.x) {
        const long long b0 = a.boff[v], b1 = a.boff[v + 1], d0 = a.doff[v], d1 = a.doff[v + 1];
        a.cnt[v] = row_kept(v, a.own_n, a.own_r) ? (b1 - b0) + (d1 - d0) : 0;
        for (long long k = (b0 + kCopyChunk - 1) / kCopyChunk; k * kCopyChunk < b1; ++k) a.markA[k] = v;
        for (long long k = (d0 + kCopyChunk - 1) / kCopyChunk; k * kCopyChunk < d1; ++k) a.markB[k] = v;
    }
}

// The fold's move: row v of the new base = base row v, then delta row v.
// As the append's old-delta copy (P4): fixed chunks of source entries, the
// destinations of a chunk written to shared memory one thread per row, then
// the entries moved with consecutive threads on consecutive entries (a warp
// per row used ~60 of every 128 lanes' worth of a base row and stalled on
// the row bounds).  Rows not kept (partitioned store) are skipped.
__global__ void __launch_bounds__(kBT) k_base_merge(CompactArgs a) {
    __shared__ long long s_dst[kCopyChunk];
    const long long ncA = (a.Eb + kCopyChunk - 1) / kCopyChunk;
    const long long ncB = (a.Ed + kCopyChunk - 1) / kCopyChunk;
    for (long long ch = blockIdx.x; ch < ncA + ncB; ch += gridDim.x) {
        const bool A = ch < ncA;
        const long long k = A ? ch : ch - ncA;
        const long long* off = A ? a.boff : a.doff;
        const int* mark = A ? a.markA : a.markB;
        const long long c0 = k * kCopyChunk, c1 = min(c0 + kCopyChunk, A ? a.Eb : a.Ed);
        const int r0 = mark[k];
        const int r1 = k + 1 < (A ? ncA : ncB) ? mark[k + 1] : a.n - 1;
#pragma unroll 4
        for (int r = r0 + (int)threadIdx.x; r <= r1; r += kBT) {
            const long long o0 = off[r], o1 = min(off[r + 1], c1);
            long long base = a.boff_new[r];
            if (!A) base += a.boff[r + 1] - a.boff[r];
            const bool keep = row_kept(r, a.own_n, a.own_r);
            for (long long e = max(o0, c0); e < o1; ++e) s_dst[e - c0] = keep ? base + (e - o0) : -1;
        }
        __syncthreads();
        const int* sidx = A ? a.bidx : a.didx;
        const double* scost = A ? a.bcost : a.dcost;
        constexpr int U = 4;
        for (long long g0 = c0; g0 < c1; g0 += U * kBT) {
            int xi[U];
            double xc[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const long long e = g0 + threadIdx.x + j * kBT;
                if (e < c1) {
                    xi[j] = __ldcs(&sidx[e]);
                    if (a.bcost_new) xc[j] = __ldcs(&scost[e]);
                }
            }
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const long long e = g0 + threadIdx.x + j * kBT;
                if (e < c1) {
                    const long long d = s_dst[e - c0];
                    if (d >= 0) {
                        a.bidx_new[d] = xi[j];
                        if (a.bcost_new) a.bcost_new[d] = xc[j];
                    }
                }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ policy
// validate a policy snapshot (no writes: the host commits after the check)
__global__ void k_check_policy(const int* parent_in, const double* g_in, int n, DevCtl* ctl) {
    int err = 0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int p = parent_in[v];
        const double gv = g_in[v];
        if (p < -1 || p >= n || p == v) err |= kErrRange;
        if (!(gv >= 0.0)) err |= kErrGNew;
        if (v == kRoot && (p != -1 || gv != 0.0)) err |= kErrRoot;
    }
    if (err) atomicOr(&ctl->err, err);
}

// VALIDATE duplicate check: staged edge e = (u -> v) (and v -> u when
// undirected) is a duplicate iff u occurs more than once in v's in-row after
// the merge (base row + the NEW delta row, which holds e itself).
__global__ void k_dup_check(const int* src, const int* dst, long long m, int undirected,
                            const long long* boff, const int* bidx, const long long* doff,
                            const int* didx, int n_old, DevCtl* ctl) {
    const int lane = threadIdx.x & 31;
    const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long items = undirected ? 2 * m : m;
    for (long long it = w0; it < items; it += nw) {        // one warp per directed edge
        const long long e = undirected ? it >> 1 : it;
        const bool rev = undirected && (it & 1);
        const int u = rev ? dst[e] : src[e], v = rev ? src[e] : dst[e];
        int cnt = 0;
        if (v < n_old)
            for (long long k = boff[v] + lane; k < boff[v + 1]; k += 32) cnt += bidx[k] == u;
        for (long long k = doff[v] + lane; k < doff[v + 1]; k += 32) cnt += didx[k] == u;
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
        if (lane == 0 && cnt > 1) atomicOr(&ctl->err, kErrDup);
    }
}

// Parent-cycle check by pointer jumping over the (integer) parent array:
// after R rounds anc(v) is the 2^R-th ancestor, or -1 once the chain ended;
// with 2^R >= n every acyclic chain has ended, so a remaining ancestor means
// a cycle.  Integer work only (no re-associated sums of g).
__global__ void k_jump(const int* in, int* out, int n, int first, const int* parent) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int x = first ? parent[v] : in[v];
        out[v] = (x < 0 || x >= n) ? -1 : (first ? parent[x] : in[x]);
    }
}
__global__ void k_jump_any(const int* anc, int n, DevCtl* ctl) {
    int bad = 0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        bad |= anc[v] >= 0;
    if (bad) atomicOr(&ctl->err, kErrCycle);
}

// Best goal (R4: lowest g over the existing goals, lowest id on ties) and
// its branch (Alg. 1 lines 8-12).
// out[0] = length (-1: cycle), out[1] = best goal (-1: none reached),
// out[2..3] = its g bits, out[4..] = goal..root
// head (nullable): the header and the first head_n entries again (a
// deferred step reads them back together with the control block)
__global__ void k_best_path(const int* parent, const double* g, int n, const int* goals,
                            int n_goals, int* out, int* head, int head_n) {
    int best = -1;
    double gb = INFINITY;
    for (int i = 0; i < n_goals; ++i) {                 // ascending ids: strict < keeps the lowest
        const int t = goals[i];
        if (t >= n) break;
        if (g[t] < gb) { gb = g[t]; best = t; }
    }
    out[1] = best;
    *(double*)&out[2] = gb;
    int v = best, len = 0;
    while (v != -1 && len <= n) {
        if (head && len < head_n) head[4 + len] = v;
        out[4 + len++] = v;
        v = parent[v];
    }
    out[0] = (v == -1) ? len : -1;
    if (head) {
        head[0] = out[0];
        head[1] = best;
        *(double*)&head[2] = gb;
    }
}


// ------------------------------------------------------------------ fused append
// One cooperative launch for the whole append (row a1): validation, the
// counting-sort merge of the batch into both delta stores (in-edge rows with
// costs, out-edge ids), base-row extension, new-vertex init, Extend's local
// relaxation (R14) or the given policy's edge costs, and the promising test.
// Grid barriers replace ~20 dependent kernel launches.

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ long long blk_sum_ll(long long x, long long* sm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    __syncthreads();
    if (lane == 0) sm[w] = x;
    __syncthreads();
    long long t = 0;
    for (int i = 0; i < kBT / 32; ++i) t += sm[i];
    return t;                                            // every thread
}

// exclusive block scan of one long long per thread; *total = block sum
__device__ __forceinline__ long long blk_excl_scan_ll(long long x, long long* sm, long long* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long inc = x;
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
    }
    __syncthreads();
    if (lane == 31) sm[w] = inc;
    __syncthreads();
    long long before = 0, all = 0;
    for (int i = 0; i < kBT / 32; ++i) {
        if (i < w) before += sm[i];
        all += sm[i];
    }
    *total = all;
    return before + inc - x;
}

// ---- P8 of the append: the next exploit's first Improve, prebuilt.
// The incremental Improve scans only the members of I
// whose result can differ from the previous Improve's: (a) its commits,
// (b) vertices whose g an Evaluate changed since, and their out-neighbours,
// (c) members that joined I since, (d) out-neighbours of the vertices
// appended since, (e) the goals.  Between exploits (c) and (d) come from
// appends only, so the append lists them here -- from this batch's own edge
// list (thread per edge: a new vertex's out-neighbours are the heads of its
// new edges) -- and the exploit's first Improve takes the list as prebuilt
// (no discovery phase, no grid barrier).  The first append after an Improve
// also lists (a), (b), (e) and whatever earlier appends added (exactly the
// exploit's own discovery); later appends continue the list.  Stamps per
// Improve k: 4k an Evaluate's prebuilt list, 4k + 1 the append's, 4k + 2 a
// discovery (which runs whenever no valid list exists), so each replaces
// the ones below it.  Once an append of the epoch could not list its sources
// (conditions, rejection), the epoch is poisoned: no later append continues.  The full Improve's counters over I (Sum of
// in-degrees, |I|: the paper's relaxation count) are recomputed by every
// append, since new in-edges change the members' in-degrees.  Valid under the
// incremental Improve's own conditions (evaluated here on the same device
// state); app_pre_k = k marks it valid.
__device__ __forceinline__ bool app_in_I(const AppendArgs& a, int v) {
    return v != kRoot && (a.b[v] || is_goal(a.goals, a.n_goals, v));
}

// membership and the list stamp in one round trip (see exploit.cu list_candidate)
__device__ __forceinline__ bool app_candidate(const AppendArgs& a, int v, unsigned ks) {
    const bool fresh = atomicMax(&a.istamp[v], ks) < ks;
    return app_in_I(a, v) && fresh;
}

__device__ __forceinline__ long long app_in_degree(const AppendArgs& a, int v) {
    return (a.boff[v + 1] - a.boff[v]) + (a.doff_new[v + 1] - a.doff_new[v]);
}

__device__ __forceinline__ void app_list_push(int* buf, int* cnt, bool want, int v) {
    const unsigned m = __ballot_sync(kFull, want);
    if (!m) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(cnt, __popc(m));
    base = __shfl_sync(kFull, base, leader);
    unsigned lt;
    asm("mov.u32 %0, %lanemask_lt;" : "=r"(lt));
    if (want) buf[base + __popc(m & lt)] = v;
}

// The current B list (the previous step's, for a deferred step) and its length.
__device__ __forceinline__ const int* app_list(const AppendArgs& a, int* bc) {
    if (a.dev_list) {                                     // written by the previous step's exploit
        *bc = *(volatile const int*)&a.ctl->dev_Bcount;
        return *(volatile const int*)&a.ctl->dev_Bsel ? a.Bq1 : a.Bq0;
    }
    *bc = a.Bcount;
    return a.Blist;
}

// The incremental Improve's own conditions (exploit_kernel), decided before
// the promising test with nprom <= n_new as the bound (an append that would
// pass only with its exact count leaves the discovery to the exploit).
__device__ __forceinline__ bool app_prebuild_ok(const AppendArgs& a, unsigned k, int bc) {
    const DevCtl* ctl = a.ctl;
    const int n_all = a.n_old + a.n_new;
    const int imp_full = *(volatile const int*)&ctl->imp_full;
    const int gc_n = *(volatile const int*)&ctl->gc_count[(k - 1) & 1];
    const int c_n = *(volatile const int*)&ctl->c_n;
    const int L_imp = *(volatile const int*)&ctl->L_imp, n_imp = *(volatile const int*)&ctl->n_imp;
    const int live_min = bc - *(volatile const int*)&ctl->holes;
    return !imp_full && gc_n < a.inc_max && c_n < a.inc_max && L_imp <= bc && n_imp <= n_all &&
           (long long)bc + a.n_new - L_imp <= a.inc_max &&
           (a.inc_imp > 1 || 4LL * (gc_n + (n_all - n_imp)) < (long long)live_min);
}

// Everything but this batch's new members (listed by the promising test
// itself): runs in the promising test's phase, on state that phase does not
// change (old list entries, old vertices' b, the row store after P5).
// rx / tk carry the counters of the new members this thread listed.
__device__ void append_prebuild(const AppendArgs& a, unsigned k, bool first, int tid, int nthreads,
                                long long rx, long long tk, long long* sm) {
    DevCtl* ctl = a.ctl;
    const int lane = threadIdx.x & 31;
    const int gwarp = tid >> 5, nwarps = nthreads >> 5;
    const int n_old = a.n_old, n_all = a.n_old + a.n_new;
    int bc;
    const int* bl = app_list(a, &bc);
    const int gc_n = *(volatile const int*)&ctl->gc_count[(k - 1) & 1];
    const int c_n = *(volatile const int*)&ctl->c_n, c_buf = *(volatile const int*)&ctl->c_buf;
    const int L_imp = *(volatile const int*)&ctl->L_imp, n_imp = *(volatile const int*)&ctl->n_imp;
    int* tl = a.alist + (size_t)(k & 1u) * a.acap;
    int* tc = &ctl->pre_count[k & 1];
    const unsigned ks = 4u * k + 1u;       // above an Evaluate's list (4k), below a discovery (4k + 2)
    // the full Improve's counters over I: the old list entries, every
    // existing goal (+ the new members, counted when listed)
    for (int t = tid; t < bc; t += nthreads) {
        const int v = bl[1 + t];
        if (v < 0 || is_goal(a.goals, a.n_goals, v)) continue;
        rx += app_in_degree(a, v);
        ++tk;
    }
    for (int t = tid; t < a.n_goals; t += nthreads) {
        const int v = a.goals[t];
        if (v >= n_all) continue;
        rx += app_in_degree(a, v);
        ++tk;
    }
    rx = blk_sum_ll(rx, sm);
    tk = blk_sum_ll(tk, sm);
    if (threadIdx.x == 0) {
        if (rx) atomicAdd((unsigned long long*)&ctl->pre_relax[k & 1], (unsigned long long)rx);
        if (tk) atomicAdd(&ctl->pre_tasks[k & 1], (int)tk);
    }
    // (a) commits [first], (c) list slots of earlier appends since the last
    // Improve [first], (e) goals (every existing one [first], else those this
    // batch created)
    const int cn = first ? c_n : 0;
    const int ns = first ? bc - L_imp : 0;
    const int tot1 = cn + ns + a.n_goals;
    const int* cl = a.dirty + (size_t)c_buf * a.dcap;
    for (int base = gwarp * 32; base < tot1; base += nwarps * 32) {        // warp-uniform
        const int t = base + lane;
        int v = -1;
        if (t < cn) v = cl[t];
        else if (t < cn + ns) v = bl[1 + L_imp + (t - cn)];
        else if (t < tot1) {
            v = a.goals[t - cn - ns];
            if (v >= n_all || (!first && v < n_old)) v = -1;
        }
        const bool want = v >= 0 && app_candidate(a, v, ks);
        app_list_push(tl, tc, want, v);
    }
    // (b) [first] g-changed vertices and their out-neighbours, (d) [first]
    // vertices appended by earlier appends since the last Improve: out-rows
    if (first) {
        const int* gl = a.gcl + (size_t)((k - 1) & 1) * a.dcap;
        const int tot2 = gc_n + max(0, n_old - n_imp);
        for (int i = gwarp; i < tot2; i += nwarps) {                      // warp-uniform
            const int x = i < gc_n ? gl[i] : n_imp + (i - gc_n);
            if (i < gc_n) {
                const bool want = lane == 0 && app_candidate(a, x, ks);
                app_list_push(tl, tc, want, x);
            }
            const long long o0 = a.oboff[x], o1 = a.oboff[x + 1];
            const long long q0 = a.odoff_new[x], q1 = a.odoff_new[x + 1];
            const long long L1 = o1 - o0, L = L1 + (q1 - q0);
            for (long long kb = 0; kb < L; kb += 32) {
                const long long e = kb + lane;
                int w = -1;
                if (e < L) w = e < L1 ? a.obidx[o0 + e] : a.odidx_new[q0 + (e - L1)];
                // (new heads are members -- listed by the promising test --
                // or goals of this batch -- listed above -- or not in I)
                const bool want = w >= 0 && w < n_old && app_candidate(a, w, ks);
                app_list_push(tl, tc, want, w);
            }
        }
    }
    // (d) this batch: the old heads of its edges whose tail is a new vertex
    const long long m = a.m;
    for (long long b0 = (long long)gwarp * 32; b0 < m; b0 += (long long)nwarps * 32) {   // warp-uniform
        const long long e = b0 + lane;
        int y0 = -1, y1 = -1;
        if (e < m) {
            const int sv = a.src[e], dv = a.dst[e];
            if (sv >= n_old && dv < n_old) y0 = dv;           // sv -> dv
            if (a.undirected && dv >= n_old && sv < n_old) y1 = sv;   // dv -> sv
        }
        const bool w0 = y0 >= 0 && app_candidate(a, y0, ks);
        app_list_push(tl, tc, w0, y0);
        const bool w1 = y1 >= 0 && app_candidate(a, y1, ks);
        app_list_push(tl, tc, w1, y1);
    }
}

__global__ void __launch_bounds__(kBT) k_append_fused(AppendArgs a, long long* cnt1,
                                                      long long* bsum) {
    cg::grid_group grid = cg::this_grid();
    __shared__ long long sm[kBT / 32];
    DevCtl* ctl = a.ctl;
    const int n_old = a.n_old, n_new = a.n_new, n_all = n_old + n_new;
    const long long m = a.m;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nthreads = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int gw = tid >> 5, nw = nthreads >> 5;
    long long* cnt0 = a.cnt;
    unsigned long long t_ph = tid == 0 ? globaltimer_ns() : 0ull;
#define APP_MARK(k)                                                                \
    if (tid == 0) {                                                                \
        const unsigned long long t_ = globaltimer_ns();                            \
        ctl->app_ns[k] += t_ - t_ph;                                               \
        t_ph = t_;                                                                 \
    }
    // promising threshold of the new vertices: the goal cost before the batch
    // (R4; g of old vertices is not written by an append), read once here
    __shared__ double s_thr;
    if (threadIdx.x < 32) {
        const double t = warp_goal_cost(a.g, a.goals, a.n_goals, n_old);
        if (threadIdx.x == 0) s_thr = t;
    }
    // the next exploit's first Improve (P8): its counters are recomputed by
    // every append, its task list continued while no Improve ran in between
    // (app_pre_k: k = Improve k's list is valid; k | kPrePoison = an append
    // since Improve k - 1 could not list its sources, so no later one may
    // continue: the exploit discovers them itself)
    const unsigned pre_k = *(volatile const unsigned*)&ctl->imp_count + 1u;
    const unsigned pre_st = *(volatile const unsigned*)&ctl->app_pre_k;
    const bool pre_on = a.pre_ok && pre_st != (pre_k | kPrePoison);
    const bool pre_first = pre_st != pre_k;
    if (tid == 0) {
        if (pre_on) {
            ctl->pre_relax[pre_k & 1] = 0;
            ctl->pre_tasks[pre_k & 1] = 0;
            if (pre_first) ctl->pre_count[pre_k & 1] = 0;
        } else {
            ctl->app_pre_k = pre_k | kPrePoison;
        }
    }
    // ---- P0 validation (R12)
    {
        int err = 0;
        bool oldold = false;
        for (long long e = tid; e < m; e += nthreads) {
            const int sv = a.src[e], dv = a.dst[e];
            const double c = a.cost[e];
            if (sv < 0 || sv >= n_all || dv < 0 || dv >= n_all) err |= kErrRange;
            else if (sv == dv) err |= kErrSelfLoop;
            else if (sv < n_old && dv < n_old) oldold = true;
            if (!(c >= 0.0) || isinf(c)) err |= kErrCost;
        }
        // an edge between two old vertices gives an old vertex a new in-edge
        // that the incremental Improve's sources (appended vertices and
        // their out-neighbours) do not cover: the next Improve is a full one
        // (set even if the batch is rejected later: only a full Improve more)
        if (oldold) ctl->imp_full = 1;
        for (int i = tid; i < n_new; i += nthreads) {
            const double hv = a.h_in[i];
            if (!(hv >= 0.0) || isinf(hv)) err |= kErrH;
            if (a.parent_in) {
                const int pp = a.parent_in[i];
                const double gv = a.g_in[i];
                if (pp < -1 || pp >= n_all || pp == n_old + i) err |= kErrRange;
                else if (pp < 0 && !isinf(gv)) err |= kErrGNew;
                else if (pp >= 0 && (!(gv >= 0.0) || isinf(gv))) err |= kErrGNew;
            }
        }
        if (err) atomicOr(&ctl->err, err);
    }
    grid.sync();
    APP_MARK(0);
    if (failed(ctl)) {                                    // uniform: err is final
        if (tid == 0) ctl->app_pre_k = pre_k | kPrePoison;   // (its counters were zeroed)
        return;
    }
    // ---- P1 old delta row lengths (both stores)
    //      and, for the copy in P4, the row holding the first entry of each
    //      kCopyChunk-entry chunk of the old deltas
#pragma unroll 4
    for (int v = tid; v <= n_all; v += nthreads) {
        long long l0 = 0, l1 = 0;
        if (v < n_old) {
            const long long a0 = a.doff_old[v], a1 = a.doff_old[v + 1];
            const long long b0 = a.odoff_old[v], b1 = a.odoff_old[v + 1];
            l0 = a1 - a0;
            l1 = b1 - b0;
            for (long long k = (a0 + kCopyChunk - 1) / kCopyChunk; k * kCopyChunk < a1; ++k)
                a.chunk_in[k] = v;
            for (long long k = (b0 + kCopyChunk - 1) / kCopyChunk; k * kCopyChunk < b1; ++k)
                a.chunk_out[k] = v;
        }
        cnt0[v] = l0;
        cnt1[v] = l1;
    }
    grid.sync();
    APP_MARK(1);
    // ---- P2 histogram of the new edges by row
    for (long long e = tid; e < m; e += nthreads) {
        const int sv = a.src[e], dv = a.dst[e];
        atomicAdd((unsigned long long*)&cnt0[dv], 1ull);
        atomicAdd((unsigned long long*)&cnt1[sv], 1ull);
        if (a.undirected) {
            atomicAdd((unsigned long long*)&cnt0[sv], 1ull);
            atomicAdd((unsigned long long*)&cnt1[dv], 1ull);
        }
    }
    grid.sync();
    APP_MARK(2);
    // ---- P3 exclusive scans -> new delta row offsets (chunk per block)
    const int G = gridDim.x;
    const int chunk = (n_all + G - 1) / G;
    const int c0 = min(n_all, (int)blockIdx.x * chunk), c1 = min(n_all, c0 + chunk);
    {
        long long s0 = 0, s1 = 0;
        for (int v = c0 + threadIdx.x; v < c1; v += kBT) { s0 += cnt0[v]; s1 += cnt1[v]; }
        s0 = blk_sum_ll(s0, sm);
        s1 = blk_sum_ll(s1, sm);
        if (threadIdx.x == 0) { bsum[blockIdx.x] = s0; bsum[G + blockIdx.x] = s1; }
    }
    grid.sync();
    APP_MARK(3);
    {
        long long p0 = 0, p1 = 0, t0 = 0, t1 = 0;
        for (int i = threadIdx.x; i < G; i += kBT) {
            const long long x0 = bsum[i], x1 = bsum[G + i];
            if (i < (int)blockIdx.x) { p0 += x0; p1 += x1; }
            t0 += x0; t1 += x1;
        }
        p0 = blk_sum_ll(p0, sm); p1 = blk_sum_ll(p1, sm);
        t0 = blk_sum_ll(t0, sm); t1 = blk_sum_ll(t1, sm);
        // warp-contiguous sub-ranges of the block's chunk, lanes on
        // consecutive rows (coalesced): pass 1 the warps' sums, pass 2 a
        // warp scan per 32 rows carried along the sub-range
        constexpr int W = kBT / 32;
        const int wl = threadIdx.x >> 5;
        const int wc = ((chunk + W - 1) / W + 31) & ~31;
        const int w0 = min(c1, c0 + wl * wc), w1 = min(c1, w0 + wc);
        __shared__ long long s_w[2][W];
        long long q0 = 0, q1 = 0;
#pragma unroll 4
        for (int v = w0 + lane; v < w1; v += 32) { q0 += cnt0[v]; q1 += cnt1[v]; }
        for (int o = 16; o; o >>= 1) {
            q0 += __shfl_xor_sync(kFull, q0, o);
            q1 += __shfl_xor_sync(kFull, q1, o);
        }
        if (lane == 0) { s_w[0][wl] = q0; s_w[1][wl] = q1; }
        __syncthreads();
        for (int i = 0; i < wl; ++i) { p0 += s_w[0][i]; p1 += s_w[1][i]; }
        for (int base = w0; base < w1; base += 32) {
            const int v = base + lane;
            const long long x0 = v < w1 ? cnt0[v] : 0, x1 = v < w1 ? cnt1[v] : 0;
            long long i0 = x0, i1 = x1;
            for (int o = 1; o < 32; o <<= 1) {
                const long long y0 = __shfl_up_sync(kFull, i0, o), y1 = __shfl_up_sync(kFull, i1, o);
                if (lane >= o) { i0 += y0; i1 += y1; }
            }
            if (v < w1) { a.doff_new[v] = p0 + i0 - x0; a.odoff_new[v] = p1 + i1 - x1; }
            p0 += __shfl_sync(kFull, i0, 31);
            p1 += __shfl_sync(kFull, i1, 31);
        }
        if (tid == 0) { a.doff_new[n_all] = t0; a.odoff_new[n_all] = t1; }
    }
    grid.sync();
    APP_MARK(4);
    // ---- P4 copy the old delta rows to their new offsets (each at the
    //      start of its row); base rows of the new vertices are empty.  The
    //      copy runs over fixed chunks of old-delta entries (not rows: delta
    //      rows hold ~6 entries, a thread or warp per row leaves most of each
    //      transaction unused): a block first writes every entry's
    //      destination into shared memory, one thread per row the chunk
    //      touches (from the chunk's first row, marked in P1), then moves
    //      the chunk with consecutive threads on consecutive entries
    const unsigned long long t_p4 = tid == 0 ? globaltimer_ns() : 0ull;
    {
        __shared__ long long s_dst[kCopyChunk];
        const long long E0 = a.doff_old[n_old], E1 = a.odoff_old[n_old];
        const long long nc0 = (E0 + kCopyChunk - 1) / kCopyChunk;
        const long long nc1 = (E1 + kCopyChunk - 1) / kCopyChunk;
        for (long long ch = blockIdx.x; ch < nc0 + nc1; ch += gridDim.x) {
            const bool in = ch < nc0;
            const long long k = in ? ch : ch - nc0;
            const long long* off_old = in ? a.doff_old : a.odoff_old;
            const long long* off_new = in ? a.doff_new : a.odoff_new;
            const long long c0 = k * kCopyChunk, c1 = min(c0 + kCopyChunk, in ? E0 : E1);
            // rows [r0, r1]: from the row of the chunk's first entry to the
            // row of the next chunk's first entry (loads independent of any
            // test, so a thread's rows are fetched in parallel)
            const int* crow = in ? a.chunk_in : a.chunk_out;
            const long long ncs = in ? nc0 : nc1;
            const int r0 = crow[k];
            const int r1 = k + 1 < ncs ? crow[k + 1] : n_old - 1;
#pragma unroll 4
            for (int r = r0 + (int)threadIdx.x; r <= r1; r += kBT) {
                const long long o0 = off_old[r], o1 = min(off_old[r + 1], c1);
                const long long sh = off_new[r] - o0;
                for (long long e = max(o0, c0); e < o1; ++e) s_dst[e - c0] = e + sh;
            }
            __syncthreads();
            // every thread moves kCopyChunk / kBT entries, U at a time with
            // all loads issued before the first store (memory-level parallelism)
            constexpr int U = 4;
            for (long long g0 = c0; g0 < c1; g0 += U * kBT) {
                if (in) {
                    int xi[U];
                    double xc[U];
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const long long e = g0 + threadIdx.x + j * kBT;
                        if (e < c1) { xi[j] = __ldcs(&a.didx_old[e]); xc[j] = __ldcs(&a.dcost_old[e]); }
                    }
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const long long e = g0 + threadIdx.x + j * kBT;
                        if (e < c1) {
                            const long long d = s_dst[e - c0];
                            a.didx_new[d] = xi[j];
                            a.dcost_new[d] = xc[j];
                        }
                    }
                } else {
                    int xi[U];
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const long long e = g0 + threadIdx.x + j * kBT;
                        if (e < c1) xi[j] = __ldcs(&a.odidx_old[e]);
                    }
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const long long e = g0 + threadIdx.x + j * kBT;
                        if (e < c1) a.odidx_new[s_dst[e - c0]] = xi[j];
                    }
                }
            }
            __syncthreads();
        }
    }
    if (tid == 0) ctl->app_ns[10] += globaltimer_ns() - t_p4;
    for (int v = n_old + 1 + tid; v <= n_all; v += nthreads) {
        a.boff_w[v] = a.base_edges;
        a.oboff_w[v] = a.obase_edges;
    }
    grid.sync();
    APP_MARK(5);
    // ---- P5 scatter the new edges; init the new vertices
    //      (cnt still holds each row's new length, old + new entries: the
    //      new ones fill the row from its end, behind the copied old ones)
    for (long long e = tid; e < m; e += nthreads) {
        const int sv = a.src[e], dv = a.dst[e];
        const double c = a.cost[e] + 0.0;                // -0.0 -> +0.0 (R12)
        long long p = a.doff_new[dv] + (long long)atomicAdd((unsigned long long*)&cnt0[dv], ~0ull) - 1;
        a.didx_new[p] = sv; a.dcost_new[p] = c;
        p = a.odoff_new[sv] + (long long)atomicAdd((unsigned long long*)&cnt1[sv], ~0ull) - 1;
        a.odidx_new[p] = dv;
        if (a.undirected) {
            p = a.doff_new[sv] + (long long)atomicAdd((unsigned long long*)&cnt0[sv], ~0ull) - 1;
            a.didx_new[p] = dv; a.dcost_new[p] = c;
            p = a.odoff_new[dv] + (long long)atomicAdd((unsigned long long*)&cnt1[dv], ~0ull) - 1;
            a.odidx_new[p] = sv;
        }
    }
    for (int i = tid; i < n_new; i += nthreads) {
        const int v = n_old + i;
        a.h[v] = a.h_in[i] + 0.0;
        if (a.parent_in) { a.parent[v] = a.parent_in[i]; a.g[v] = a.g_in[i] + 0.0; }
        else { a.parent[v] = -1; a.g[v] = INFINITY; }
        a.pc[v] = 0.0;
        a.b[v] = 0;
    }
    grid.sync();
    APP_MARK(6);
    // ---- P6 policy of the new vertices
    if (a.parent_in) {
        // given policy: pc(v) = cost of the stored edge (parent -> v)
        for (int i = gw; i < n_new; i += nw) {
            const int v = n_old + i;
            const int p = a.parent[v];
            if (p < 0) continue;
            long long best = LLONG_MAX;
            double c = 0.0;
            for (long long k = a.boff[v] + lane; k < a.boff[v + 1]; k += 32)
                if (a.bidx[k] == p && k < best) { best = k; c = a.bcost[k]; }
            for (long long k = a.doff_new[v] + lane; k < a.doff_new[v + 1]; k += 32)
                if (a.didx_new[k] == p && (1LL << 62) + k < best) { best = (1LL << 62) + k; c = a.dcost_new[k]; }
            for (int o = 16; o; o >>= 1) {
                const long long ob = __shfl_xor_sync(kFull, best, o);
                const double oc = __shfl_xor_sync(kFull, c, o);
                if (ob < best) { best = ob; c = oc; }
            }
            if (lane == 0) {
                if (best == LLONG_MAX) atomicOr(&ctl->err, kErrPcMissing);
                else {
                    a.pc[v] = c;
                    if (a.validate && a.g[v] != a.g[p] + c) atomicOr(&ctl->err, kErrGNew);
                }
            }
        }
    } else if (n_new > 0) {
        // Extend's local relaxation (R14) in ONE dataflow pass:
        // in increasing id order g(v) = min over in-edges (u -> v), u < v,
        // of g(u) + c (lowest u on ties).  A warp takes new vertices in
        // increasing id order; where an in-neighbour u is itself new, the
        // lane waits until u is final (rdone[u] == this append's id, stored
        // with release after u's g / parent / pc).  Every dependency points
        // to a lower id and all warps are co-resident (cooperative launch),
        // so the lowest unfinished vertex can always proceed: the result is
        // the sequential id-order result bit for bit, without the grid-wide
        // sweeps of a Jacobi relaxation.
        const unsigned aid = a.app_id;
        for (int i = gw; i < n_new; i += nw) {
            const int v = n_old + i;
            double best = INFINITY;
            int arg = INT_MAX;
            double argc = 0.0;
            for (long long k = a.boff[v] + lane; k < a.boff[v + 1]; k += 32) {
                const int u = a.bidx[k];
                if (u >= v) continue;
                if (u >= n_old) while (ld_acquire_u32(&a.rdone[u]) != aid) {}
                const double c = a.bcost[k];
                const double cand = *(volatile const double*)&a.g[u] + c;
                if (cand < best || (cand == best && u < arg)) { best = cand; arg = u; argc = c; }
            }
            for (long long k = a.doff_new[v] + lane; k < a.doff_new[v + 1]; k += 32) {
                const int u = a.didx_new[k];
                if (u >= v) continue;
                if (u >= n_old) while (ld_acquire_u32(&a.rdone[u]) != aid) {}
                const double c = a.dcost_new[k];
                const double cand = *(volatile const double*)&a.g[u] + c;
                if (cand < best || (cand == best && u < arg)) { best = cand; arg = u; argc = c; }
            }
            double wb = best;
            int wa = arg;
            for (int o = 16; o; o >>= 1) {
                const double ob = __shfl_xor_sync(kFull, wb, o);
                const int oa = __shfl_xor_sync(kFull, wa, o);
                if (ob < wb || (ob == wb && oa < wa)) { wb = ob; wa = oa; }
            }
            const unsigned mm = __ballot_sync(kFull, best == wb && arg == wa);
            const double c = __shfl_sync(kFull, argc, __ffs(mm) - 1);
            if (lane == 0) {
                if (wb < INFINITY) {
                    *(volatile double*)&a.g[v] = wb;
                    a.parent[v] = wa;
                    a.pc[v] = c;
                }                                          // (else: -1 / +inf / 0 from P5)
                st_release_u32(&a.rdone[v], aid);
            }
            __syncwarp();
        }
        if (tid == 0) ctl->sweeps = 1;
    }
    grid.sync();
    APP_MARK(7);
    if (failed(ctl)) return;
    // ---- P7 b(v) = g(v) + h(v) < g(x_goal); promising ones join the B list
    // (goal set, R4: the goal cost before the batch)
    const double thr = s_thr;
    int bc_list;
    int* const blist = const_cast<int*>(app_list(a, &bc_list));
    const bool pre_go = pre_on && app_prebuild_ok(a, pre_k, bc_list);   // (uniform)
    const unsigned pre_ks = 4u * pre_k + 1u;
    long long pre_rx = 0, pre_tk = 0;
    for (int base = blockIdx.x * blockDim.x; base < n_new; base += nthreads) {
        const int i = base + threadIdx.x;
        const int v = n_old + i;
        const bool p = (i < n_new) && (a.g[v] + a.h[v] < thr);
        if (i < n_new) {
            a.b[v] = p ? 1 : 0;
            // the new vertex is a child of its parent in the policy tree
            // (incremental Evaluate's child counts); VALIDATE appends may
            // still be rejected after this kernel: the host counts those
            // after its commit
            const int pv = a.parent[v];
            if (!a.validate && pv >= 0) atomicAdd(&a.ccd[pv].x, 1);
        }
        const unsigned mm = __ballot_sync(kFull, p);
        if (mm) {
            const int leader = __ffs(mm) - 1;
            int pos = 0;
            if (lane == leader) pos = atomicAdd(&ctl->nprom, __popc(mm));
            pos = __shfl_sync(kFull, pos, leader);
            unsigned lt;
            asm("mov.u32 %0, %lanemask_lt;" : "=r"(lt));
            if (p) blist[1 + bc_list + pos + __popc(mm & lt)] = v;
        }
        if (pre_go) {
            // (c) of the next exploit's first Improve: the new members
            const bool want = p && atomicMax(&a.istamp[v], pre_ks) < pre_ks;
            if (want && !is_goal(a.goals, a.n_goals, v)) { pre_rx += app_in_degree(a, v); ++pre_tk; }
            app_list_push(a.alist + (size_t)(pre_k & 1u) * a.acap, &ctl->pre_count[pre_k & 1], want, v);
        }
    }
    if (pre_go) append_prebuild(a, pre_k, pre_first, tid, nthreads, pre_rx, pre_tk, sm);
    APP_MARK(8);
    if (tid == 0 && pre_on) ctl->app_pre_k = pre_go ? pre_k : (pre_k | kPrePoison);
    if (tid == 0) ctl->app_ns[9] += 1;
#undef APP_MARK
}

}  // namespace

thread_local long long g_kernel_launches = 0;

size_t scan_tmp_elems(long long L) { return (size_t)((L + kScanTile - 1) / kScanTile + 2); }

cudaError_t scan_exclusive(const long long* in, long long* out, long long L, long long* tmp,
                           cudaStream_t s) {
    if (L <= 0) {
        ++g_kernel_launches;
        k_set_ll<<<1, 1, 0, s>>>(out, 0);
        return cudaGetLastError();
    }
    const long long P = (L + kScanTile - 1) / kScanTile;
    ++g_kernel_launches;
    k_scan_reduce<<<(unsigned)P, kBT, 0, s>>>(in, L, tmp);
    ++g_kernel_launches;
    k_scan_partials<<<1, kBT, 0, s>>>(tmp, P);
    ++g_kernel_launches;
    k_scan_apply<<<(unsigned)P, kBT, 0, s>>>(in, L, tmp, out);
    // out[L] = total = tmp[P]
    cudaMemcpyAsync(out + L, tmp + P, sizeof(long long), cudaMemcpyDeviceToDevice, s);
    return cudaGetLastError();
}

cudaError_t launch_dup_check(const AppendArgs& a, cudaStream_t s) {
    if (a.m == 0) return cudaSuccess;
    const long long items = a.undirected ? 2 * a.m : a.m;
    ++g_kernel_launches;
    k_dup_check<<<grid_for(items * 32), kBT, 0, s>>>(a.src, a.dst, a.m, a.undirected, a.boff,
                                                     a.bidx, a.doff_new, a.didx_new, a.n_old,
                                                     a.ctl);
    return cudaGetLastError();
}

cudaError_t launch_cycle_check(const int* parent, int n, int* tmp, DevCtl* ctl, cudaStream_t s) {
    if (n <= 1) return cudaSuccess;
    int* buf[2] = {tmp, tmp + n};
    // round 0 writes the 2nd ancestor; round r the 2^(r+1)-th
    int r = 0, cur = 0;
    ++g_kernel_launches;
    k_jump<<<grid_for(n), kBT, 0, s>>>(nullptr, buf[0], n, 1, parent);
    for (r = 1; (1LL << r) < (long long)n; ++r) {
        ++g_kernel_launches;
        k_jump<<<grid_for(n), kBT, 0, s>>>(buf[cur], buf[cur ^ 1], n, 0, nullptr);
        cur ^= 1;
    }
    ++g_kernel_launches;
    k_jump_any<<<grid_for(n), kBT, 0, s>>>(buf[cur], n, ctl);
    return cudaGetLastError();
}

cudaError_t launch_append_fused(const AppendArgs& a, long long* cnt1, long long* bsum,
                                int max_blocks, const L2Window& w, cudaStream_t s) {
    // a.per_sm: occupancy of k_append_fused, computed once per context at
    // pirrt_create (append_blocks_per_sm) -- device-specific, so not cached here
    int blocks = a.per_sm * (a.grid_blocks > 0 ? a.grid_blocks : 148);
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    AppendArgs args = a;
    void* params[] = {&args, &cnt1, &bsum};
    ++g_kernel_launches;
    return launch_coop((const void*)k_append_fused, blocks, kBT, params, w, s);
}

// policy-tree child counts of the parents of [v0, v1) (incremental
// Evaluate)
__global__ void k_child_count(const int* parent, int v0, int v1, int2* ccd) {
    for (int v = v0 + (int)(blockIdx.x * blockDim.x + threadIdx.x); v < v1; v += gridDim.x * blockDim.x) {
        const int p = parent[v];
        if (p >= 0) atomicAdd(&ccd[p].x, 1);
    }
}

cudaError_t launch_child_count(const int* parent, int v0, int v1, int2* ccd, cudaStream_t s) {
    if (v1 <= v0) return cudaSuccess;
    ++g_kernel_launches;
    k_child_count<<<grid_for(v1 - v0), kBT, 0, s>>>(parent, v0, v1, ccd);
    return cudaGetLastError();
}

int append_blocks_per_sm() {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_append_fused, kBT, 0);
    return per_sm;
}

cudaError_t launch_compact(const CompactArgs& a, cudaStream_t s) {
    cudaError_t e;
    ++g_kernel_launches;
    k_base_count<<<grid_for(a.n), kBT, 0, s>>>(a);
    if ((e = scan_exclusive(a.cnt, a.boff_new, a.n, a.scan_tmp, s)) != cudaSuccess) return e;
    ++g_kernel_launches;
    const long long chunks = (a.Eb + kCopyChunk - 1) / kCopyChunk + (a.Ed + kCopyChunk - 1) / kCopyChunk;
    k_base_merge<<<grid_for(chunks, 1), kBT, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_set_policy(const PolicyArgs& a, cudaStream_t s) {
    // a.parent/a.g/a.pc are STAGING arrays here; the caller commits them
    ++g_kernel_launches;
    k_check_policy<<<grid_for(a.n), kBT, 0, s>>>(a.parent_in, a.g_in, a.n, a.ctl);
    ++g_kernel_launches;
    k_find_pc<<<grid_for((long long)a.n * 32), kBT, 0, s>>>(a.boff, a.bidx, a.bcost, a.doff, a.didx,
                                                            a.dcost, a.parent_in, a.g_in, a.pc, 0,
                                                            a.n, 0, a.ctl);
    return cudaGetLastError();
}

cudaError_t launch_rebuild_blist(const unsigned char* b, int n, int* list, int* count_out,
                                 long long* cnt, long long* scan_tmp, cudaStream_t s) {
    cudaError_t e;
    ++g_kernel_launches;
    k_b_flags<<<grid_for(n), kBT, 0, s>>>(b, n, cnt);
    if ((e = scan_exclusive(cnt, cnt + n + 1, n, scan_tmp, s)) != cudaSuccess) return e;
    ++g_kernel_launches;
    k_b_scatter<<<grid_for(n), kBT, 0, s>>>(b, n, cnt + n + 1, list, count_out);
    return cudaGetLastError();
}

cudaError_t launch_best_path(const int* parent, const double* g, int n, const int* goals,
                             int n_goals, int* out, cudaStream_t s, int* head, int head_n) {
    ++g_kernel_launches;
    k_best_path<<<1, 1, 0, s>>>(parent, g, n, goals, n_goals, out, head, head_n);
    return cudaGetLastError();
}

}  // namespace pirrt
