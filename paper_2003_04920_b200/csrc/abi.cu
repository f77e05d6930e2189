// abi.cu -- the C ABI of include/pirrt.h: context, device memory, staging,
// and the host side of every call.  The hot path (exploit) is one
// cooperative kernel launch; append is a short chain of kernels with one
// host synchronisation at the end (for n_new_promising and the validation
// verdict).  No CPU fallback exists: every result is computed on the device.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"
#include "pirrt_bench.h"

using namespace pirrt;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CU(call)                                                                   \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess)                                                     \
            return fail(PIRRT_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// device allocation that grows geometrically; keep_bytes are preserved
template <class T>
int grow(T*& p, int64_t& cap, int64_t need, int64_t keep, cudaStream_t s) {
    if (need <= cap) return 0;
    int64_t nc = std::max<int64_t>(need, cap + cap / 2);
    nc = std::max<int64_t>(nc, 64);
    T* q = nullptr;
    if (cudaMalloc(&q, (size_t)nc * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        return fail(PIRRT_E_NOMEM, "cudaMalloc failed");
    }
    if (p) {
        if (keep > 0) CU(cudaMemcpyAsync(q, p, (size_t)keep * sizeof(T), cudaMemcpyDeviceToDevice, s));
        CU(cudaStreamSynchronize(s));
        CU(cudaFree(p));
    }
    p = q;
    cap = nc;
    return 0;
}

std::string err_bits(int e) {
    std::string m;
    if (e & kErrRange) m += " id out of range;";
    if (e & kErrSelfLoop) m += " self-loop;";
    if (e & kErrCost) m += " cost not finite and >= 0;";
    if (e & kErrH) m += " h not finite and >= 0;";
    if (e & kErrGNew) m += " bad g (given policy);";
    if (e & kErrPcMissing) m += " policy edge (parent -> v) not stored;";
    if (e & kErrRoot) m += " root must have parent -1 and g 0;";
    if (e & kErrDup) m += " duplicate (src,dst) edge (VALIDATE);";
    if (e & kErrCycle) m += " parent cycle (VALIDATE);";
    return m;
}

// NCCL is loaded lazily (dlopen), only when a context is sharded: a
// single-GPU user needs no NCCL.  If torch already loaded libnccl.so.2 the
// same library is reused.
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;   // optional
    ncclResult_t (*commAbort)(ncclComm_t) = nullptr;                           // optional
};

NcclApi* nccl_api() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        // RTLD_LOCAL: a libnccl.so.2 torch loads later (its own build) must
        // not resolve against this one; if torch loaded one first, the same
        // soname returns that copy
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (h) {
            api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
            api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
            api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
            api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
            api.errorString = (decltype(api.errorString))dlsym(h, "ncclGetErrorString");
            api.commGetAsyncError = (decltype(api.commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
            api.commAbort = (decltype(api.commAbort))dlsym(h, "ncclCommAbort");
            if (api.getUniqueId && api.commInitRank && api.allGather && api.commDestroy &&
                api.errorString)
                api.h = h;
        }
    }
    return api.h ? &api : nullptr;
}

#define NC(call)                                                                   \
    do {                                                                           \
        ncclResult_t r_ = (call);                                                  \
        if (r_ != ncclSuccess)                                                     \
            return fail(PIRRT_E_NCCL, std::string(#call) + ": " + nccl_api()->errorString(r_)); \
    } while (0)

}  // namespace

struct pirrt_ctx {
    pirrt_config cfg;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 0;
    int grid_blocks = 0;
    int append_per_sm = 0;        // k_append_fused occupancy (computed at create)
    int n = 0;
    int64_t vcap = 0;
    // vertex SoA
    double* g = nullptr; int64_t g_cap = 0;
    double* h = nullptr; int64_t h_cap = 0;
    double* pc = nullptr; int64_t pc_cap = 0;
    int* parent = nullptr; int64_t parent_cap = 0;
    unsigned char* b = nullptr; int64_t b_cap = 0;
    // base CSR
    long long* boff = nullptr; int64_t boff_cap = 0;
    int* bidx = nullptr; int64_t bidx_cap = 0;
    double* bcost = nullptr; int64_t bcost_cap = 0;
    // spare base buffers: a fold writes the merged CSR here and swaps, so a
    // steady-state fold allocates and frees nothing
    long long* sboff = nullptr; int64_t sboff_cap = 0;
    int* sbidx = nullptr; int64_t sbidx_cap = 0;
    double* sbcost = nullptr; int64_t sbcost_cap = 0;
    int64_t base_edges = 0;       // edges in the base CSR (this rank's rows when partitioned)
    int64_t edges_total = 0;      // directed edges appended (pirrt_num_edges)
    // partitioned in-edge store (sharded, nranks > 1, no VALIDATE): a fold
    // keeps only the rows of the vertices this rank's Improve owns
    int own_n = 0, own_r = 0;
    // delta CSR, double-buffered (cur = committed)
    long long* doff[2] = {nullptr, nullptr}; int64_t doff_cap[2] = {0, 0};
    int* didx[2] = {nullptr, nullptr}; int64_t didx_cap[2] = {0, 0};
    double* dcost[2] = {nullptr, nullptr}; int64_t dcost_cap[2] = {0, 0};
    int cur = 0;
    int64_t delta_edges = 0;
    // out-edge index (rows by source, ids only): base + delta (double-buffered with `cur`)
    long long* oboff = nullptr; int64_t oboff_cap = 0;
    int* obidx = nullptr; int64_t obidx_cap = 0;
    long long* soboff = nullptr; int64_t soboff_cap = 0;
    int* sobidx = nullptr; int64_t sobidx_cap = 0;
    int64_t obase_edges = 0;
    long long* odoff[2] = {nullptr, nullptr}; int64_t odoff_cap[2] = {0, 0};
    int* odidx[2] = {nullptr, nullptr}; int64_t odidx_cap[2] = {0, 0};
    // Evaluate stamps and the B lists (entry 0 = root)
    unsigned* stamp = nullptr; int64_t stamp_cap = 0;
    unsigned* pstamp = nullptr;                          // incremental Evaluate: dirty marks,
    int2* ccd = nullptr;                                 // child counts + depths,
    int* dirty = nullptr;                                // dirty lists (all in the hot slab),
    unsigned* istamp = nullptr;                          // incremental Improve: task stamps,
    int* gcl = nullptr;                                  // g-changed lists,
    int* alist = nullptr;                                // task list
    int64_t dcap = 0;                                    // entries per dirty / g-changed buffer
    int inc_imp = 1;                                     // PIRRT_INC_IMPROVE (0 off, 1 auto, 2 always)
    int small_grid = -1;                                 // PIRRT_SMALL_GRID: blocks for small exploits
                                                         // (-1: one per SM; 0: off)
    int64_t small_max = 65536;                           // PIRRT_SMALL_MAX: |B| + appended vertices bound
    int64_t n_last_exploit = 0;                          // |V| at the last exploit's launch
    int x_blocks = 0;                                    // grid of the running exploit
    int inc_max = 8192;                                  // PIRRT_INC_MAX (0: full Evaluates only)
    int inc_validate = 0;                                // PIRRT_INC_VALIDATE=1 (test hook)
    int* Bq[2] = {nullptr, nullptr}; int64_t Bq_cap[2] = {0, 0};
    // work-queue Evaluate items (slot 0 = root, the rest -1 between Evaluates)
    int* qv = nullptr; double* qg = nullptr; int* qdepth = nullptr; int64_t q_cap = 0;
    char* slab = nullptr; size_t slab_bytes = 0;          // hot per-vertex arrays (one allocation)
    bool l2_persist = false;                             // PIRRT_L2_PERSIST=1 enables (measured: no
                                                         // exploit gain, and the carve-out halves the
                                                         // append's streaming bandwidth)
    int64_t persist_max = 0, window_max = 0;
    L2Window l2win;
    int Bsel = 0;
    int Bcount = 0;
    unsigned ev_next = 1;
    // scratch
    long long* cnt = nullptr; int64_t cnt_cap = 0;
    long long* scan_tmp = nullptr; int64_t scan_cap = 0;
    int* path = nullptr; int64_t path_cap = 0;   // best_path scratch (n + 1)
    DevCtl* ctl = nullptr;
    DevCtl* ctl_host = nullptr;   // pinned mirror
    // staging for host inputs
    int* s_src = nullptr; int64_t s_src_cap = 0;
    int* s_dst = nullptr; int64_t s_dst_cap = 0;
    double* s_cost = nullptr; int64_t s_cost_cap = 0;
    double* s_h = nullptr; int64_t s_h_cap = 0;
    int* s_parent = nullptr; int64_t s_parent_cap = 0;
    double* s_g = nullptr; int64_t s_g_cap = 0;
    double* s_pc = nullptr; int64_t s_pc_cap = 0;
    unsigned char* s_b = nullptr; int64_t s_b_cap = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool broken = false;
    // sharded mode (nranks > 1, or PIRRT_F_SHARDED): vertex-cyclic Improve,
    // all-gather of the Improve records, replicated Evaluate
    bool sharded = false;
    int rank = 0, nranks = 1;
    ncclComm_t comm = nullptr;
    ShardRec* rec_local = nullptr; int64_t rec_local_cap = 0;
    ShardRec* rec_all = nullptr; int64_t rec_all_cap = 0;
    cudaEvent_t xev = nullptr, xev2 = nullptr;               // in-process group exchange ordering
    int shard_blocks = 0;
    unsigned long long watchdog_ns = 60ull * 1000000000ull;   // PIRRT_WATCHDOG_MS
    double compact_min = 32768.0;                            // PIRRT_COMPACT_MIN (edges)
    int wq_keep = 32;                                        // PIRRT_WQ_KEEP
    int wq_tail = -1;                                        // PIRRT_WQ_TAIL (-1: 16 per block)
    int wq_wide = -1;                                        // PIRRT_WQ_WIDE (-1: 10 per block, 0: off)
    int wide_tasks = 131072;                                 // PIRRT_WIDE_TASKS: |I| for the wide Improve (0: off)
    int kids_min = -1;                                       // PIRRT_KIDS_MIN: |B| for the children index
                                                             // (-1: 4 n / mean degree; 0: never)
    long long* app_bsum = nullptr; int64_t app_bsum_cap = 0;
    int* app_chunk = nullptr; int64_t app_chunk_cap = 0;   // append P4 chunk rows (both deltas)
    unsigned* rdone = nullptr; int64_t rdone_cap = 0;      // append local relaxation stamps
    int* fold_mark = nullptr; int64_t fold_mark_cap = 0;   // fold: chunk rows of base + delta
    int wide_lpv = 0;                                      // PIRRT_WIDE_LPV (16 / 32; 0: by mean degree)
    int prebuild_max = 1024;                               // PIRRT_PREBUILD_MAX: largest batch whose
                                                           // append lists the next first Improve
    unsigned app_id = 0;                                   // appends launched
    int64_t launches = 0;         // kernels launched (diagnostics, bench gpu_launches)
    // goal set G (R4): sorted unique ids incl. x_goal (device copy + host copy)
    int* goals = nullptr; int64_t goals_cap = 0;
    std::vector<int> goals_host;
    // asynchronous exploit (pirrt_exploit_async / pirrt_exploit_wait)
    bool inflight = false;        // an exploit was launched and not finished
    ExploitArgs x_args;           // its first launch's arguments (hand-offs reuse them)
    int x_rc = 0;                 // sharded loop result
    bool kept = false;            // finished implicitly by another call: result kept
    int kept_rc = 0;
    pirrt_exploit_stats kept_stats;
    cudaStream_t copy_stream = nullptr;   // H2D of the next batch while an exploit runs
    cudaEvent_t copy_done = nullptr;
    // device-side Extend (pirrt_set_world / pirrt_extend_batch)
    int w_d = 0, w_nboxes = 0;
    double w_gamma = 0.0;
    double* w_boxes = nullptr; int64_t w_boxes_cap = 0;
    double* w_goal = nullptr; int64_t w_goal_cap = 0;
    double* pts = nullptr; int64_t pts_cap = 0;           // [n][d] every vertex's point
    int* x_cell = nullptr; int64_t x_cell_cap = 0;
    int* x_cpts = nullptr; int64_t x_cpts_cap = 0;
    long long* x_ccnt = nullptr; int64_t x_ccnt_cap = 0;
    long long* x_cstart = nullptr; int64_t x_cstart_cap = 0;
    long long* x_tmp = nullptr; int64_t x_tmp_cap = 0;
    double* x_R = nullptr; int64_t x_R_cap = 0;
    double* x_h = nullptr; int64_t x_h_cap = 0;
    long long* x_ecnt = nullptr; int64_t x_ecnt_cap = 0;
    long long* x_eoff = nullptr; int64_t x_eoff_cap = 0;
    int* x_src = nullptr; int64_t x_src_cap = 0;
    int* x_dst = nullptr; int64_t x_dst_cap = 0;
    double* x_cost = nullptr; int64_t x_cost_cap = 0;
    int* x_hj = nullptr; int64_t x_hj_cap = 0;           // the count pass's hit cache
    double* x_hd = nullptr; int64_t x_hd_cap = 0;
    int x_hcap = 128;             // hit-cache slots per new vertex (from the last batch's mean)
    bool in_extend = false;       // the append is pirrt_extend_batch's own
    // deferred BE-RRT# steps (pirrt_step_async / pirrt_step_wait): a ring of
    // kStepDepth slots, each the step's read-back (control block tail, best
    // path head) in pinned memory, its own device best-path buffer and events
    struct StepSlot {
        DevCtl* ctl = nullptr;            // pinned; the tail from `status` on
        int* head = nullptr;              // pinned; best_path header + kStepHead entries
        int* dpath = nullptr; int64_t dpath_cap = 0;
        cudaEvent_t e0 = nullptr, e1 = nullptr, done = nullptr;
        int blocks = 0;
    } slot[2];
    int steps_out = 0;            // steps enqueued and not yet waited
    int step_head = 0;            // slot of the oldest of them
    cudaEvent_t app_done = nullptr;   // after the last step's append (staging free again)
};

constexpr int kStepDepth = 2;
constexpr int kStepHead = 1020;
constexpr size_t kStepHeadBytes = sizeof(int) * (4 + kStepHead);

namespace {

int set_device(const pirrt_ctx* c, bool steps_ok = false) {
    CU(cudaSetDevice(c->cfg.device));
    if (c->broken) return fail(PIRRT_E_STATE, "context unusable after an earlier CUDA error");
    if (c->steps_out > 0 && !steps_ok)
        return fail(PIRRT_E_STATE, "a deferred step is outstanding (pirrt_step_wait first)");
    return 0;
}

// The per-vertex arrays every PI phase gathers from (g, pc, h, parent, stamp,
// b and the two B lists) live in ONE allocation, so a single L2 access-policy
// window can keep them resident (persisting lines survive other traffic, e.g.
// the benchmark's L2 flush).  Growth copies each sub-array.
int grow_hot_slab(pirrt_ctx* c, int64_t cap) {
    cudaStream_t s = c->stream;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t sz_g = al(8 * cap), sz_pc = al(8 * cap), sz_h = al(8 * cap);
    // B lists: members + holes stay below 4/3 n (the incremental Evaluate
    // runs only while holes <= length / 4), so 2 cap + 2 entries suffice
    const size_t sz_par = al(4 * cap), sz_st = al(4 * cap), sz_bq = al(4 * (2 * cap + 2)), sz_b = al(cap);
    // dirty and g-changed lists: two buffers each (by Evaluate / Improve
    // parity), dcap = cap + 64 entries per buffer; the incremental Improve's
    // task list: cap entries
    const int64_t dcap = cap + 64;
    const size_t sz_ccd = al(8 * cap), sz_dirty = al(4 * 2 * dcap), sz_al = al(4 * 2 * cap);
    const size_t total = sz_g + sz_pc + sz_h + sz_par + 3 * sz_st + 2 * sz_bq + sz_b + sz_ccd +
                         2 * sz_dirty + sz_al;
    char* slab = nullptr;
    if (cudaMalloc(&slab, total) != cudaSuccess) { cudaGetLastError(); return fail(PIRRT_E_NOMEM, "cudaMalloc (vertex slab) failed"); }
    char* q = slab;
    double* g = (double*)q; q += sz_g;
    double* pc = (double*)q; q += sz_pc;
    double* h = (double*)q; q += sz_h;
    int* parent = (int*)q; q += sz_par;
    unsigned* stamp = (unsigned*)q; q += sz_st;
    unsigned* pstamp = (unsigned*)q; q += sz_st;
    unsigned* istamp = (unsigned*)q; q += sz_st;
    int2* ccd = (int2*)q; q += sz_ccd;
    int* dirty = (int*)q; q += sz_dirty;
    int* gcl = (int*)q; q += sz_dirty;
    int* alist = (int*)q; q += sz_al;
    int* bq0 = (int*)q; q += sz_bq;
    int* bq1 = (int*)q; q += sz_bq;
    unsigned char* b = (unsigned char*)q;
    const int64_t n = c->n;
    // stamps of fresh slots read as "never visited"; list slots beyond the
    // live entries are -1 (work-queue invariant), slot 0 = root; fresh
    // vertices have no children
    CU(cudaMemsetAsync(stamp, 0, (size_t)cap * sizeof(unsigned), s));
    CU(cudaMemsetAsync(pstamp, 0, (size_t)cap * sizeof(unsigned), s));
    CU(cudaMemsetAsync(istamp, 0, (size_t)cap * sizeof(unsigned), s));
    CU(cudaMemsetAsync(ccd, 0, (size_t)cap * sizeof(int2), s));
    CU(cudaMemsetAsync(bq0, 0xFF, (size_t)(2 * cap + 2) * sizeof(int), s));
    CU(cudaMemsetAsync(bq1, 0xFF, (size_t)(2 * cap + 2) * sizeof(int), s));
    CU(cudaMemsetAsync(bq0, 0, sizeof(int), s));
    CU(cudaMemsetAsync(bq1, 0, sizeof(int), s));
    if (c->slab) {
        auto cp = [&](void* dst, const void* src, size_t bytes) {
            return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s) : cudaSuccess;
        };
        int* nbq[2] = {bq0, bq1};
        const int64_t keep_cur = 1 + c->Bcount;
        if (cp(g, c->g, 8 * n) || cp(pc, c->pc, 8 * n) || cp(h, c->h, 8 * n) ||
            cp(parent, c->parent, 4 * n) || cp(stamp, c->stamp, 4 * n) || cp(b, c->b, n) ||
            cp(pstamp, c->pstamp, 4 * n) || cp(istamp, c->istamp, 4 * n) || cp(ccd, c->ccd, 8 * n) ||
            cp(dirty, c->dirty, 4 * std::min<int64_t>(n, c->dcap)) ||
            cp(dirty + dcap, c->dirty + c->dcap, 4 * std::min<int64_t>(n, c->dcap)) ||
            cp(gcl, c->gcl, 4 * std::min<int64_t>(n, c->dcap)) ||
            cp(gcl + dcap, c->gcl + c->dcap, 4 * std::min<int64_t>(n, c->dcap)) ||
            // both task-list slots (an append's prebuilt list lives across
            // appends; slot k & 1 starts at (k & 1) x capacity)
            cp(alist, c->alist, 4 * std::min<int64_t>(n, c->g_cap)) ||
            cp(alist + cap, c->alist + c->g_cap, 4 * std::min<int64_t>(n, c->g_cap)) ||
            cp(nbq[c->Bsel], c->Bq[c->Bsel], 4 * keep_cur))
            return fail(PIRRT_E_CUDA, "vertex slab copy failed");
        CU(cudaStreamSynchronize(s));
        CU(cudaFree(c->slab));
    }
    c->slab = slab; c->slab_bytes = total;
    c->g = g; c->pc = pc; c->h = h; c->parent = parent; c->stamp = stamp; c->b = b;
    c->pstamp = pstamp; c->ccd = ccd; c->dirty = dirty;
    c->istamp = istamp; c->gcl = gcl; c->alist = alist; c->dcap = dcap;
    c->Bq[0] = bq0; c->Bq[1] = bq1; c->Bq_cap[0] = c->Bq_cap[1] = 2 * cap + 2;
    c->g_cap = c->pc_cap = c->h_cap = c->parent_cap = c->b_cap = c->stamp_cap = cap;
    // L2 persistence for the slab
    if (c->l2_persist) {
        size_t lim = std::min<size_t>(total, (size_t)c->persist_max);
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim);
        c->l2win.base = slab;
        c->l2win.bytes = std::min<size_t>(total, (size_t)c->window_max);
        c->l2win.hit = c->l2win.bytes ? std::min(1.0f, (float)lim / (float)c->l2win.bytes) : 0.f;
        cudaGetLastError();
    }
    return 0;
}

// make every per-vertex array hold at least `need` vertices (+1 for offsets)
int ensure_vertices(pirrt_ctx* c, int64_t need) {
    if (need <= c->vcap) return 0;
    // vertex ids travel as (id << 1 | tag) inside the Evaluate scan
    if (need > kMaxVertices) return fail(PIRRT_E_RANGE, "more than 2^30 - 2^14 vertices");
    int64_t cap = std::max<int64_t>(need, c->vcap + c->vcap / 2);
    cap = std::min<int64_t>(std::max<int64_t>(cap, 1024), kMaxVertices);
    const int64_t n = c->n;
    cudaStream_t s = c->stream;
    int rc;
    if ((rc = grow_hot_slab(c, cap))) return rc;
    if ((rc = grow(c->boff, c->boff_cap, cap + 1, n + 1, s))) return rc;
    if ((rc = grow(c->sboff, c->sboff_cap, cap + 1, 0, s))) return rc;
    if ((rc = grow(c->doff[c->cur], c->doff_cap[c->cur], cap + 1, n + 1, s))) return rc;
    if ((rc = grow(c->doff[1 - c->cur], c->doff_cap[1 - c->cur], cap + 1, 0, s))) return rc;
    if ((rc = grow(c->cnt, c->cnt_cap, 2 * (cap + 1), 0, s))) return rc;
    if ((rc = grow(c->scan_tmp, c->scan_cap, (int64_t)scan_tmp_elems(cap + 1), 0, s))) return rc;
    if ((rc = grow(c->oboff, c->oboff_cap, cap + 1, n + 1, s))) return rc;
    if ((rc = grow(c->soboff, c->soboff_cap, cap + 1, 0, s))) return rc;
    if ((rc = grow(c->odoff[c->cur], c->odoff_cap[c->cur], cap + 1, n + 1, s))) return rc;
    if ((rc = grow(c->odoff[1 - c->cur], c->odoff_cap[1 - c->cur], cap + 1, 0, s))) return rc;
    if (cap + 2 + kMaxGridBlocks > c->q_cap) {
        // fresh queue: every slot unpublished (-1) except slot 0 = the root (g 0, depth 0)
        const int64_t qc = cap + 2 + kMaxGridBlocks;
        int64_t c1 = 0, c2 = 0, c3 = 0;
        if (c->qv) { CU(cudaStreamSynchronize(s)); cudaFree(c->qv); cudaFree(c->qg); cudaFree(c->qdepth); }
        c->qv = nullptr; c->qg = nullptr; c->qdepth = nullptr;
        if ((rc = grow(c->qv, c1, qc, 0, s))) return rc;
        if ((rc = grow(c->qg, c2, qc, 0, s))) return rc;
        if ((rc = grow(c->qdepth, c3, qc, 0, s))) return rc;
        CU(cudaMemsetAsync(c->qv, 0xff, (size_t)qc * sizeof(int), s));
        CU(cudaMemsetAsync(c->qv, 0, sizeof(int), s));
        CU(cudaMemsetAsync(c->qg, 0, (size_t)qc * sizeof(double), s));
        CU(cudaMemsetAsync(c->qdepth, 0, (size_t)qc * sizeof(int), s));
        c->q_cap = qc;
    }
    if ((rc = grow(c->path, c->path_cap, cap + 8, 0, s))) return rc;
    {
        // stamps of the local relaxation: only this append's new vertices are
        // read, and their ids were never stamped with a later id -- zeroed once
        const int64_t before = c->rdone_cap;
        if ((rc = grow(c->rdone, c->rdone_cap, cap, 0, s))) return rc;
        if (c->rdone_cap != before) CU(cudaMemsetAsync(c->rdone, 0, (size_t)c->rdone_cap * sizeof(unsigned), s));
    }
    c->vcap = cap;
    return 0;
}

void free_all(pirrt_ctx* c) {
    void* ptrs[] = {c->slab, c->boff, c->bidx, c->bcost,
                    c->sboff, c->sbidx, c->sbcost, c->soboff, c->sobidx,
                    c->doff[0], c->doff[1], c->didx[0], c->didx[1], c->dcost[0], c->dcost[1],
                    c->oboff, c->obidx, c->odoff[0], c->odoff[1], c->odidx[0], c->odidx[1],
                    c->qv, c->qg, c->qdepth, c->path, c->cnt, c->scan_tmp, c->ctl,
                    c->s_src, c->s_dst, c->s_cost, c->s_h, c->s_parent, c->s_g, c->s_pc, c->s_b,
                    c->rec_local, c->rec_all, c->app_bsum, c->goals,
                    c->w_boxes, c->w_goal, c->pts, c->x_cell, c->x_cpts, c->x_ccnt, c->x_cstart,
                    c->x_tmp, c->x_R, c->x_h, c->x_ecnt, c->x_eoff, c->x_src, c->x_dst, c->x_cost,
                    c->x_hj, c->x_hd};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (c->ctl_host) cudaFreeHost(c->ctl_host);
    if (c->app_chunk) cudaFree(c->app_chunk);
    if (c->rdone) cudaFree(c->rdone);
    if (c->fold_mark) cudaFree(c->fold_mark);
    for (auto& sl : c->slot) {
        if (sl.ctl) cudaFreeHost(sl.ctl);                 // (head lives inside it)
        if (sl.dpath) cudaFree(sl.dpath);
        for (cudaEvent_t e : {sl.e0, sl.e1, sl.done})
            if (e) cudaEventDestroy(e);
    }
    if (c->app_done) cudaEventDestroy(c->app_done);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->copy_done) cudaEventDestroy(c->copy_done);
    if (c->xev) cudaEventDestroy(c->xev);
    if (c->xev2) cudaEventDestroy(c->xev2);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    if (c->comm && nccl_api()) nccl_api()->commDestroy(c->comm);
}

template <class T>
int stage(pirrt_ctx* c, const T* src, int64_t count, bool device, T*& buf, int64_t& cap,
          const T** out, cudaStream_t s = nullptr) {
    if (count == 0 || src == nullptr) { *out = src; return 0; }
    if (device) { *out = src; return 0; }
    if (!s) s = c->stream;
    int rc;
    if ((rc = grow(buf, cap, count, 0, s))) return rc;
    CU(cudaMemcpyAsync(buf, src, (size_t)count * sizeof(T), cudaMemcpyHostToDevice, s));
    *out = buf;
    return 0;
}

int read_ctl(pirrt_ctx* c) {
    // everything after the per-iteration counters (the host never reads those)
    const size_t o = offsetof(DevCtl, status);
    CU(cudaMemcpyAsync((char*)c->ctl_host + o, (const char*)c->ctl + o, sizeof(DevCtl) - o,
                       cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return 0;
}

// fold one delta CSR into its base CSR: merge into the spare base buffers,
// clear the delta, swap current and spare (cost arrays NULL for the out-index)
int fold(pirrt_ctx* c, long long*& boff, int64_t& boff_cap, int*& bidx, int64_t& bidx_cap,
         double*& bcost, int64_t& bcost_cap, long long*& sboff, int64_t& sboff_cap, int*& sbidx,
         int64_t& sbidx_cap, double*& sbcost, int64_t& sbcost_cap, long long* doff,
         const int* didx, const double* dcost, int64_t E, bool partition) {
    int rc;
    if ((rc = grow(sboff, sboff_cap, c->vcap + 1, 0, c->stream))) return rc;
    if ((rc = grow(sbidx, sbidx_cap, E, 0, c->stream))) return rc;
    if (bcost && (rc = grow(sbcost, sbcost_cap, E, 0, c->stream))) return rc;
    CompactArgs a;
    a.boff = boff; a.bidx = bidx; a.bcost = bcost;
    a.doff = doff; a.didx = didx; a.dcost = dcost;
    a.boff_new = sboff; a.bidx_new = sbidx; a.bcost_new = bcost ? sbcost : nullptr;
    a.cnt = c->cnt; a.scan_tmp = c->scan_tmp; a.n = c->n;
    // the base holds boff[n] entries (this rank's rows on a partitioned
    // store), the delta E - base_edges; chunk marks for the merge
    a.Eb = bcost ? c->base_edges : c->obase_edges;
    a.Ed = E - a.Eb;
    const int64_t nA = a.Eb / kAppendCopyChunk + 2, nB = a.Ed / kAppendCopyChunk + 2;
    if ((rc = grow(c->fold_mark, c->fold_mark_cap, nA + nB, 0, c->stream))) return rc;
    a.markA = c->fold_mark; a.markB = c->fold_mark + nA;
    a.own_n = partition ? c->own_n : 0;
    a.own_r = c->own_r;
    const long long l0 = g_kernel_launches;
    CU(launch_compact(a, c->stream));
    c->launches += g_kernel_launches - l0;
    CU(cudaMemsetAsync(doff, 0, (size_t)(c->n + 1) * sizeof(long long), c->stream));
    std::swap(boff, sboff); std::swap(boff_cap, sboff_cap);
    std::swap(bidx, sbidx); std::swap(bidx_cap, sbidx_cap);
    if (bcost) { std::swap(bcost, sbcost); std::swap(bcost_cap, sbcost_cap); }
    return 0;
}

int compact_if_needed(pirrt_ctx* c, int64_t m_dir, bool sync = true) {
    // fold the deltas into the bases when they outgrow sqrt(2 m |base|) (and
    // 32k edges): minimises (mean delta copied per append) + (|E| fold cost
    // amortised over the appends between folds)
    double thr = std::sqrt(2.0 * (double)std::max<int64_t>(m_dir, 1) * (double)c->base_edges);
    thr = std::max(thr, c->compact_min);
    if ((double)c->delta_edges <= thr) return 0;
    const int64_t E = c->base_edges + c->delta_edges;
    int rc;
    if ((rc = fold(c, c->boff, c->boff_cap, c->bidx, c->bidx_cap, c->bcost, c->bcost_cap,
                   c->sboff, c->sboff_cap, c->sbidx, c->sbidx_cap, c->sbcost, c->sbcost_cap,
                   c->doff[c->cur], c->didx[c->cur], c->dcost[c->cur], E, true)))
        return rc;
    int64_t Eb = E;
    if (c->own_n > 1) {                                   // this rank's rows only
        long long e_local = 0;
        CU(cudaMemcpyAsync(&e_local, c->boff + c->n, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        Eb = e_local;
    }
    double* no_cost = nullptr;
    double* no_scost = nullptr;
    int64_t no_cap = 0, no_scap = 0;
    if ((rc = fold(c, c->oboff, c->oboff_cap, c->obidx, c->obidx_cap, no_cost, no_cap,
                   c->soboff, c->soboff_cap, c->sobidx, c->sobidx_cap, no_scost, no_scap,
                   c->odoff[c->cur], c->odidx[c->cur], nullptr, c->obase_edges + c->delta_edges, false)))
        return rc;
    c->base_edges = Eb;
    c->obase_edges += c->delta_edges;
    c->delta_edges = 0;
    // the fold belongs to this append: finish it before returning, so that
    // it is neither hidden in nor charged to the next call on the stream
    // (a deferred step leaves it in the stream order)
    if (sync) CU(cudaStreamSynchronize(c->stream));
    return 0;
}

// the fused append kernel's arguments (pirrt_graph_append_batch, pirrt_step_async)
void fill_append_args(pirrt_ctx* c, AppendArgs& a, int nb, int n_old, int n_new, const double* d_h,
                      const int* d_parent, const double* d_g, const int* d_src, const int* d_dst,
                      const double* d_cost, int64_t n_edges, bool undirected, bool validate) {
    std::memset(&a, 0, sizeof(a));
    a.boff = c->boff; a.bidx = c->bidx; a.bcost = c->bcost;
    a.doff_old = c->doff[c->cur]; a.didx_old = c->didx[c->cur]; a.dcost_old = c->dcost[c->cur];
    a.doff_new = c->doff[nb]; a.didx_new = c->didx[nb]; a.dcost_new = c->dcost[nb];
    a.boff_w = c->boff;
    a.oboff = c->oboff; a.obidx = c->obidx;
    a.odoff_old = c->odoff[c->cur]; a.odidx_old = c->odidx[c->cur];
    a.odoff_new = c->odoff[nb]; a.odidx_new = c->odidx[nb];
    a.oboff_w = c->oboff;
    a.obase_edges = c->obase_edges;
    a.Blist = c->Bq[c->Bsel]; a.Bcount = c->Bcount;
    a.Bq0 = c->Bq[0]; a.Bq1 = c->Bq[1];
    a.rdone = c->rdone;
    a.app_id = ++c->app_id;
    // P8: prebuild the next exploit's first Improve (single GPU, the
    // incremental Improve's own preconditions; a VALIDATE append may still be
    // rejected after the kernel, a given policy forces a full Improve)
    // (small batches only: for S = 4096 at the bench workload the append's
    // listing cost 18 us for the 10 us discovery phase it saves the exploit;
    // for S = 1 (configs[1]) it takes the exploit median from 33.6 to 23.5 us)
    a.pre_ok = (!c->sharded && c->inc_imp > 0 && !validate && !d_parent && n_new <= c->prebuild_max &&
                !(c->cfg.flags & (PIRRT_F_PRUNE_OFF | PIRRT_F_NEIGHBOURS))) ? 1 : 0;
    a.inc_max = (int)std::min<int64_t>(c->inc_max, c->dcap - 64);
    a.inc_imp = c->inc_imp;
    a.istamp = c->istamp; a.alist = c->alist; a.acap = (int)c->g_cap;
    a.dirty = c->dirty; a.gcl = c->gcl; a.dcap = (int)c->dcap;
    const int64_t nch = c->delta_edges / kAppendCopyChunk + 2;
    a.chunk_in = c->app_chunk; a.chunk_out = c->app_chunk + nch;
    a.cnt = c->cnt; a.scan_tmp = c->scan_tmp;
    a.h_in = d_h; a.parent_in = d_parent; a.g_in = d_g;
    a.src = d_src; a.dst = d_dst; a.cost = d_cost; a.m = n_edges;
    a.undirected = undirected ? 1 : 0;
    a.validate = validate ? 1 : 0;
    a.g = c->g; a.h = c->h; a.parent = c->parent; a.pc = c->pc; a.b = c->b;
    a.ccd = c->ccd;
    a.n_old = n_old; a.n_new = n_new; a.base_edges = c->base_edges;
    a.ctl = c->ctl;
    a.grid_blocks = c->num_sms;
    a.per_sm = c->append_per_sm;
    a.goals = c->goals; a.n_goals = (int)c->goals_host.size();
}

int complete_pending(pirrt_ctx* c);   // below, with the exploit

// The next Evaluate must be a full one (create, set_policy, an append with
// a given policy); list_rebuilt: the B list was rebuilt without holes
// (create, set_policy).  Stream-ordered.
cudaError_t set_need_full(pirrt_ctx* c, bool list_rebuilt) {
    static const int one = 1;
    cudaError_t e = cudaMemcpyAsync(&c->ctl->need_full, &one, sizeof(int), cudaMemcpyHostToDevice,
                                    c->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&c->ctl->imp_full, &one, sizeof(int), cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess && list_rebuilt) e = cudaMemsetAsync(&c->ctl->holes, 0, sizeof(int), c->stream);
    return e;
}

}  // namespace

extern "C" {

void pirrt_config_init(pirrt_config* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->nranks = 1;
    cfg->root = kRoot;
    cfg->goal = kGoal;
}

const char* pirrt_last_error(void) { return g_err.c_str(); }

int pirrt_create(const pirrt_config* cfg_in, pirrt_ctx** out) {
    if (!cfg_in || !out) return fail(PIRRT_E_INVAL, "create: NULL argument");
    const pirrt_config& cfg = *cfg_in;
    if (!(cfg.h_root >= 0.0) || !(cfg.h_goal >= 0.0) || std::isinf(cfg.h_root) ||
        std::isinf(cfg.h_goal) || !(cfg.epsilon >= 0.0) || cfg.max_iterations < 0)
        return fail(PIRRT_E_INVAL, "create: invalid h_root/h_goal/epsilon/max_iterations");
    if (cfg.nranks < 1 || cfg.rank < 0 || cfg.rank >= cfg.nranks)
        return fail(PIRRT_E_INVAL, "create: bad nranks/rank");
    const bool local_group = (cfg.flags & PIRRT_F_LOCAL_GROUP) != 0;
    if (cfg.nranks > 1 && !cfg.nccl_unique_id && !local_group)
        return fail(PIRRT_E_INVAL, "create: nranks > 1 needs nccl_unique_id (or PIRRT_F_LOCAL_GROUP)");
    if (local_group && cfg.nccl_unique_id)
        return fail(PIRRT_E_INVAL, "create: PIRRT_F_LOCAL_GROUP takes no nccl_unique_id");
    if (cfg.n_goals < 0 || (cfg.n_goals > 0 && !cfg.goals))
        return fail(PIRRT_E_INVAL, "create: bad goals/n_goals");
    if ((cfg.flags & PIRRT_F_NEIGHBOURS) &&
        (cfg.nranks > 1 || (cfg.flags & (PIRRT_F_SHARDED | PIRRT_F_LOCAL_GROUP))))
        return fail(PIRRT_E_INVAL, "create: PIRRT_F_NEIGHBOURS is single-GPU only");
    // R15: x_init and x_goal are the first two vertices created
    if (cfg.root != kRoot || cfg.goal != kGoal)
        return fail(PIRRT_E_INVAL, "create: root/goal must be 0/1 (pirrt_config_init; reading R15)");
    std::vector<int> goal_ids = {kGoal};
    for (int32_t i = 0; i < cfg.n_goals; ++i) {
        if (cfg.goals[i] < 1 || cfg.goals[i] >= kMaxVertices)
            return fail(PIRRT_E_RANGE, "create: goal id must be >= 1 (not the root)");
        goal_ids.push_back(cfg.goals[i]);
    }
    std::sort(goal_ids.begin(), goal_ids.end());
    goal_ids.erase(std::unique(goal_ids.begin(), goal_ids.end()), goal_ids.end());
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (cfg.device < 0 || cfg.device >= ndev) return fail(PIRRT_E_INVAL, "create: bad device");
    CU(cudaSetDevice(cfg.device));
    pirrt_ctx* c = new pirrt_ctx();
    c->cfg = cfg;
    c->cfg.goals = nullptr;                     // the caller's array is not kept
    c->goals_host = goal_ids;
    if (const char* w = std::getenv("PIRRT_WATCHDOG_MS"))
        c->watchdog_ns = (unsigned long long)std::strtoull(w, nullptr, 10) * 1000000ull;
    if (const char* w = std::getenv("PIRRT_COMPACT_MIN")) c->compact_min = std::atof(w);
    if (const char* w = std::getenv("PIRRT_WQ_KEEP")) c->wq_keep = std::max(1, std::min(64, std::atoi(w)));
    if (const char* w = std::getenv("PIRRT_WQ_TAIL")) c->wq_tail = std::atoi(w);
    if (const char* w = std::getenv("PIRRT_WQ_WIDE")) c->wq_wide = std::atoi(w);
    if (const char* w = std::getenv("PIRRT_WIDE_TASKS")) c->wide_tasks = std::max(0, std::atoi(w));
    if (const char* w = std::getenv("PIRRT_KIDS_MIN")) c->kids_min = std::atoi(w);
    if (const char* w = std::getenv("PIRRT_INC_MAX")) c->inc_max = std::max(0, std::atoi(w));
    if (const char* w = std::getenv("PIRRT_INC_VALIDATE")) c->inc_validate = std::atoi(w) != 0;
    if (const char* w = std::getenv("PIRRT_INC_IMPROVE")) c->inc_imp = std::max(0, std::atoi(w));
    if (const char* w = std::getenv("PIRRT_SMALL_GRID")) c->small_grid = std::max(-1, std::atoi(w));
    if (const char* w = std::getenv("PIRRT_SMALL_MAX")) c->small_max = std::max(0, std::atoi(w));
    if (const char* w = std::getenv("PIRRT_PREBUILD_MAX")) c->prebuild_max = std::atoi(w);
    if (const char* w = std::getenv("PIRRT_WIDE_LPV")) c->wide_lpv = std::atoi(w) == 32 ? 32 : 16;
    auto bail = [&](int rc) { free_all(c); delete c; return rc; };
    if (cfg.stream) {
        c->stream = (cudaStream_t)cfg.stream;
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(PIRRT_E_CUDA, "create: stream"));
        c->own_stream = true;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cfg.device) != cudaSuccess)
        return bail(fail(PIRRT_E_CUDA, "create: device properties"));
    c->num_sms = prop.multiProcessorCount;
    c->persist_max = prop.persistingL2CacheMaxSize;
    c->window_max = prop.accessPolicyMaxWindowSize;
    if (const char* w = std::getenv("PIRRT_L2_PERSIST")) c->l2_persist = std::atoi(w) != 0;
    if (c->persist_max <= 0 || c->window_max <= 0) c->l2_persist = false;
    if (!prop.cooperativeLaunch) return bail(fail(PIRRT_E_STATE, "create: no cooperative launch"));
    int per_sm = exploit_blocks_per_sm();
    if (per_sm < 1) return bail(fail(PIRRT_E_CUDA, "create: exploit kernel does not fit an SM"));
    c->append_per_sm = append_blocks_per_sm();
    if (c->append_per_sm < 1) return bail(fail(PIRRT_E_CUDA, "create: append kernel does not fit an SM"));
    c->grid_blocks = cfg.grid_blocks > 0 ? std::min(cfg.grid_blocks, per_sm * c->num_sms)
                                         : per_sm * c->num_sms;
    c->grid_blocks = std::min(c->grid_blocks, kMaxGridBlocks);
    // per-batch exploits are grid-barrier bound: one block per SM measured
    // 10% faster than two at the bench workload and 14% at configs[1]
    // (tools/grid_probe.py, profiles/r2/grid_probe.jsonl)
    if (c->small_grid < 0) c->small_grid = c->num_sms;
    int rc;
    int64_t vcap0 = std::max<int64_t>(cfg.vertex_capacity, 1024);
    if ((rc = ensure_vertices(c, vcap0))) return bail(rc);
    int64_t ecap0 = std::max<int64_t>(cfg.edge_capacity, 4096);
    for (int k = 0; k < 2; ++k) {
        if ((rc = grow(c->didx[k], c->didx_cap[k], ecap0, 0, c->stream))) return bail(rc);
        if ((rc = grow(c->dcost[k], c->dcost_cap[k], ecap0, 0, c->stream))) return bail(rc);
    }
    // base and spare base stores: reserve the caller's edge-capacity hint up
    // front so that folds in steady state never allocate
    const int64_t bcap0 = std::max<int64_t>(cfg.edge_capacity, 64);
    if ((rc = grow(c->bidx, c->bidx_cap, bcap0, 0, c->stream))) return bail(rc);
    if ((rc = grow(c->bcost, c->bcost_cap, bcap0, 0, c->stream))) return bail(rc);
    if ((rc = grow(c->obidx, c->obidx_cap, bcap0, 0, c->stream))) return bail(rc);
    if (cfg.edge_capacity > 0) {
        if ((rc = grow(c->sbidx, c->sbidx_cap, bcap0, 0, c->stream))) return bail(rc);
        if ((rc = grow(c->sbcost, c->sbcost_cap, bcap0, 0, c->stream))) return bail(rc);
        if ((rc = grow(c->sobidx, c->sobidx_cap, bcap0, 0, c->stream))) return bail(rc);
    }
    if ((rc = grow(c->app_bsum, c->app_bsum_cap, 2 * kAppendMaxBlocks + 2, 0, c->stream))) return bail(rc);
    for (int k = 0; k < 2; ++k)
        if ((rc = grow(c->odidx[k], c->odidx_cap[k], ecap0, 0, c->stream))) return bail(rc);
    if ((rc = grow(c->goals, c->goals_cap, (int64_t)goal_ids.size(), 0, c->stream))) return bail(rc);
    if (cudaMemcpyAsync(c->goals, goal_ids.data(), goal_ids.size() * sizeof(int),
                        cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
        return bail(fail(PIRRT_E_CUDA, "create: goals copy"));
    // the control block, followed by a deferred step's best-path head (one
    // read-back per step)
    if (cudaMalloc(&c->ctl, sizeof(DevCtl) + kStepHeadBytes) != cudaSuccess) return bail(fail(PIRRT_E_NOMEM, "ctl"));
    if (cudaMallocHost(&c->ctl_host, sizeof(DevCtl)) != cudaSuccess)
        return bail(fail(PIRRT_E_NOMEM, "ctl host"));
    if (cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->copy_done, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(PIRRT_E_CUDA, "events"));
    if (cfg.nranks > 1 || (cfg.flags & (PIRRT_F_SHARDED | PIRRT_F_LOCAL_GROUP))) {
        if (!local_group) {
            NcclApi* api = nccl_api();
            if (!api) return bail(fail(PIRRT_E_NCCL, "create: libnccl.so.2 not loadable"));
            ncclUniqueId id;
            if (cfg.nccl_unique_id) std::memcpy(&id, cfg.nccl_unique_id, sizeof(id));
            else if (api->getUniqueId(&id) != ncclSuccess) return bail(fail(PIRRT_E_NCCL, "create: ncclGetUniqueId"));
            if (api->commInitRank(&c->comm, cfg.nranks, id, cfg.rank) != ncclSuccess)
                return bail(fail(PIRRT_E_NCCL, "create: ncclCommInitRank"));
        }
        if (cudaEventCreateWithFlags(&c->xev, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->xev2, cudaEventDisableTiming) != cudaSuccess)
            return bail(fail(PIRRT_E_CUDA, "create: events"));
        c->sharded = true;
        c->rank = cfg.rank;
        c->nranks = cfg.nranks;
        // partitioned in-edge store (the owner holds the
        // in-edge rows of its vertices): folds keep only the owned rows.
        // Not with VALIDATE, whose duplicate check reads every row
        if (cfg.nranks > 1 && !(cfg.flags & PIRRT_F_VALIDATE)) { c->own_n = cfg.nranks; c->own_r = cfg.rank; }
        int per_sm = shard_evaluate_blocks_per_sm();
        if (per_sm < 1) return bail(fail(PIRRT_E_CUDA, "create: shard kernel does not fit an SM"));
        c->shard_blocks = cfg.grid_blocks > 0 ? std::min(cfg.grid_blocks, per_sm * c->num_sms)
                                              : per_sm * c->num_sms;
        c->shard_blocks = std::min(c->shard_blocks, kMaxGridBlocks);
    }
    // V = {x_init, x_goal}, E = {}, B = {}
    const double g0[2] = {0.0, INFINITY};
    const double h0[2] = {cfg.h_root + 0.0, cfg.h_goal + 0.0};
    const int p0[2] = {-1, -1};
    cudaStream_t s = c->stream;
    if (cudaMemcpyAsync(c->g, g0, sizeof g0, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(c->h, h0, sizeof h0, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(c->parent, p0, sizeof p0, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemsetAsync(c->pc, 0, 2 * sizeof(double), s) != cudaSuccess ||
        cudaMemsetAsync(c->b, 0, 2, s) != cudaSuccess ||
        cudaMemsetAsync(c->boff, 0, 3 * sizeof(long long), s) != cudaSuccess ||
        cudaMemsetAsync(c->doff[0], 0, 3 * sizeof(long long), s) != cudaSuccess ||
        cudaMemsetAsync(c->oboff, 0, 3 * sizeof(long long), s) != cudaSuccess ||
        cudaMemsetAsync(c->odoff[0], 0, 3 * sizeof(long long), s) != cudaSuccess ||

        cudaMemsetAsync(c->ctl, 0, sizeof(DevCtl), s) != cudaSuccess ||
        set_need_full(c, true) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return bail(fail(PIRRT_E_CUDA, "create: init copies"));
    c->n = 2;
    *out = c;
    return PIRRT_OK;
}

int pirrt_destroy(pirrt_ctx* c) {
    if (!c) return PIRRT_OK;
    cudaSetDevice(c->cfg.device);
    cudaStreamSynchronize(c->stream);
    free_all(c);
    delete c;
    return PIRRT_OK;
}

int64_t pirrt_num_vertices(const pirrt_ctx* c) { return c ? c->n : 0; }
int64_t pirrt_num_edges(const pirrt_ctx* c) { return c ? c->edges_total : 0; }
int64_t pirrt_kernel_launches(const pirrt_ctx* c) { return c ? c->launches : 0; }

int pirrt_graph_append_batch(pirrt_ctx* c, int32_t n_new, const double* h_new,
                             const pirrt_vid* parent_new, const double* g_new, int64_t n_edges,
                             const pirrt_vid* src, const pirrt_vid* dst, const double* cost,
                             uint32_t flags, int32_t* n_new_promising) {
    if (!c) return fail(PIRRT_E_INVAL, "append: NULL context");
    int rc;
    if ((rc = set_device(c))) return rc;
    if (n_new < 0 || n_edges < 0) return fail(PIRRT_E_INVAL, "append: negative size");
    if ((parent_new == nullptr) != (g_new == nullptr))
        return fail(PIRRT_E_INVAL, "append: parent_new and g_new must both be given or both NULL");
    if (n_new > 0 && !h_new) return fail(PIRRT_E_INVAL, "append: h_new is NULL");
    if (n_edges > 0 && (!src || !dst || !cost)) return fail(PIRRT_E_INVAL, "append: NULL edge array");
    if ((int64_t)c->n + n_new > INT32_MAX - 1) return fail(PIRRT_E_RANGE, "append: too many vertices");
    if (c->w_d != 0 && !c->in_extend && n_new > 0)
        return fail(PIRRT_E_STATE, "append: a context with a world grows through pirrt_extend_batch");
    const bool dev = (flags & PIRRT_F_DEVICE_PTRS) != 0;
    const bool undirected = (flags & PIRRT_F_EDGES_UNDIRECTED) != 0;
    const int64_t m_dir = undirected ? 2 * n_edges : n_edges;
    cudaStream_t s = c->stream;
    // inputs.  While an exploit started by pirrt_exploit_async still runs,
    // host inputs are copied on the side stream so that the H2D overlaps it
    // (SURVEY.md section 8(f) NEXT-1); the append itself waits for it.
    const double *d_h = nullptr, *d_g = nullptr, *d_cost = nullptr;
    const int *d_parent = nullptr, *d_src = nullptr, *d_dst = nullptr;
    const bool early = c->inflight && !dev;
    const bool dbg = std::getenv("PIRRT_DEBUG_HOST") != nullptr;
    auto now_us = []() {
        return std::chrono::duration<double, std::micro>(
                   std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double t_in = dbg ? now_us() : 0.0;
    double t_staged = 0.0, t_pending = 0.0;
    auto stage_all = [&](cudaStream_t ss) -> int {
        int r;
        if ((r = stage(c, h_new, n_new, dev, c->s_h, c->s_h_cap, &d_h, ss))) return r;
        if ((r = stage(c, parent_new, n_new, dev, c->s_parent, c->s_parent_cap, &d_parent, ss))) return r;
        if ((r = stage(c, g_new, n_new, dev, c->s_g, c->s_g_cap, &d_g, ss))) return r;
        if ((r = stage(c, src, n_edges, dev, c->s_src, c->s_src_cap, &d_src, ss))) return r;
        if ((r = stage(c, dst, n_edges, dev, c->s_dst, c->s_dst_cap, &d_dst, ss))) return r;
        return stage(c, cost, n_edges, dev, c->s_cost, c->s_cost_cap, &d_cost, ss);
    };
    if (early) {
        if ((rc = stage_all(c->copy_stream))) return rc;
        CU(cudaEventRecord(c->copy_done, c->copy_stream));
    }
    if (dbg) t_staged = now_us();
    if ((rc = complete_pending(c))) return rc;
    if (dbg) t_pending = now_us();
    const int n_old = c->n, n_all = c->n + n_new;
    // capacity (growth does not change state)
    if ((rc = ensure_vertices(c, n_all))) return rc;
    const int nb = 1 - c->cur;
    const int64_t dneed = c->delta_edges + m_dir;
    if ((rc = grow(c->didx[nb], c->didx_cap[nb], dneed, 0, s))) return rc;
    if ((rc = grow(c->dcost[nb], c->dcost_cap[nb], dneed, 0, s))) return rc;
    if ((rc = grow(c->odidx[nb], c->odidx_cap[nb], dneed, 0, s))) return rc;
    if (early) CU(cudaStreamWaitEvent(s, c->copy_done, 0));
    else if ((rc = stage_all(s))) return rc;
    static_assert(offsetof(DevCtl, nprom) == offsetof(DevCtl, err) + 2 * sizeof(int), "DevCtl layout");
    CU(cudaMemsetAsync(&c->ctl->err, 0, 3 * sizeof(int), s));   // err, sweeps, nprom
    if ((rc = grow(c->app_chunk, c->app_chunk_cap, 2 * (c->delta_edges / kAppendCopyChunk + 2), 0, s)))
        return rc;
    AppendArgs a;
    fill_append_args(c, a, nb, n_old, n_new, d_h, parent_new ? d_parent : nullptr, g_new ? d_g : nullptr,
                     d_src, d_dst, d_cost, n_edges, undirected,
                     ((flags | c->cfg.flags) & PIRRT_F_VALIDATE) != 0);
    const long long l0 = g_kernel_launches;
    cudaError_t e = launch_append_fused(a, c->cnt + (c->cnt_cap / 2), c->app_bsum, kAppendMaxBlocks,
                                        c->l2win, s);
    if (e == cudaSuccess && a.validate) {
        // VALIDATE: duplicates against the stored graph and inside the batch;
        // a given policy must not close a parent cycle
        e = launch_dup_check(a, s);
        if (e == cudaSuccess && parent_new) e = launch_cycle_check(c->parent, n_all, (int*)c->cnt, c->ctl, s);
    }
    c->launches += g_kernel_launches - l0;
    if (e != cudaSuccess) { c->broken = true; return fail(PIRRT_E_CUDA, std::string("append: ") + cudaGetErrorString(e)); }
    if ((rc = read_ctl(c))) { c->broken = true; return rc; }
    if (dbg) std::fprintf(stderr, "pirrt host: append m=%lld %s: early-staged +%.1f, pending done +%.1f, "
                          "kernel done +%.1f us\n", (long long)n_edges, dev ? "device" : "host",
                          t_staged ? t_staged - t_in : 0.0, t_pending - t_in, now_us() - t_in);
    const int err = c->ctl_host->err;
    if (err) {
        int code = (err & (kErrRange)) ? PIRRT_E_RANGE
                 : (err & kErrCycle && !(err & ~kErrCycle)) ? PIRRT_E_CORRUPT : PIRRT_E_INVAL;
        return fail(code, "append rejected:" + err_bits(err));
    }
    // commit
    c->cur = nb;
    c->n = n_all;
    c->delta_edges += m_dir;
    c->edges_total += m_dir;
    c->Bcount += c->ctl_host->nprom;
    if (a.validate) {
        // the fused kernel leaves the child counts of a VALIDATE append (which
        // the checks after it may still reject) to this point
        const long long l2 = g_kernel_launches;
        CU(launch_child_count(c->parent, n_old, n_all, c->ccd, s));
        c->launches += g_kernel_launches - l2;
    }
    if (parent_new) CU(set_need_full(c, false));   // a given policy: the next Evaluate is a full one
    if (n_new_promising) *n_new_promising = c->ctl_host->nprom;
    if ((rc = compact_if_needed(c, m_dir))) { c->broken = true; return rc; }
    return PIRRT_OK;
}

// the exploit-kernel instantiation with the children-index Evaluate is used
// when a large Evaluate is possible: PRUNE_OFF, or |B| already >= kids_min
static int kids_variant(const ExploitArgs& a, int Bcount) {
    return a.kids_min > 0 && (a.prune_off || (int64_t)Bcount + a.n_goals >= a.kids_min) ? 1 : 0;
}

static void fill_exploit_args(pirrt_ctx* c, ExploitArgs& a, int blocks) {
    std::memset(&a, 0, sizeof(a));
    a.boff = c->boff; a.bidx = c->bidx; a.bcost = c->bcost;
    a.doff = c->doff[c->cur]; a.didx = c->didx[c->cur]; a.dcost = c->dcost[c->cur];
    a.oboff = c->oboff; a.obidx = c->obidx;
    a.odoff = c->odoff[c->cur]; a.odidx = c->odidx[c->cur];
    a.g = c->g; a.h = c->h; a.parent = c->parent; a.pc = c->pc; a.b = c->b;
    a.stamp = c->stamp;
    a.pstamp = c->pstamp; a.ccd = c->ccd; a.dirty = c->dirty;
    a.istamp = c->istamp; a.gcl = c->gcl; a.alist = c->alist; a.dcap = (int)c->dcap;
    a.acap = (int)c->g_cap;                               // (the hot slab's vertex capacity)
    a.inc_max = (int)std::min<int64_t>(c->inc_max, c->dcap - 64);
    a.inc_imp = c->inc_imp;
    a.inc_validate = c->inc_validate;
    a.Bq0 = c->Bq[0]; a.Bq1 = c->Bq[1]; a.Bsel = c->Bsel; a.Bcount = c->Bcount;
    a.old_Bcount = 0; a.pending = 0;
    a.ev_base = c->ev_next;
    a.ctl = c->ctl;
    a.n = c->n;
    a.max_it = c->cfg.max_iterations;
    a.eps = c->cfg.epsilon;
    a.prune_off = (c->cfg.flags & PIRRT_F_PRUNE_OFF) ? 1 : 0;
    a.watchdog_ns = c->watchdog_ns;
    a.wq_keep = c->wq_keep;
    // the hand-over frontier must fit the blocks' local frontiers (64 each)
    a.wq_tail = c->wq_tail < 0 ? 16 * blocks : std::min(c->wq_tail, 64 * blocks);
    a.wq_wide = c->wq_wide < 0 ? 10 * blocks : c->wq_wide;
    a.debug = std::getenv("PIRRT_DEBUG") != nullptr;
    a.qv = c->qv; a.qg = c->qg; a.qdepth = c->qdepth;
    a.goals = c->goals; a.n_goals = (int)c->goals_host.size();
    a.parent_form = (c->cfg.flags & PIRRT_F_PARENT_FORM) ? 1 : 0;
    a.neighbours = (c->cfg.flags & PIRRT_F_NEIGHBOURS) && !a.prune_off ? 1 : 0;
    // children index for large Evaluates: worth it once |B| x mean out-degree
    // exceeds ~4 n row entries; built in the append scratch (idle during an
    // exploit): cnt holds 4 (vcap + 1) ints, app_bsum >= kMaxGridBlocks ints
    const double E = (double)c->edges_total;
    const double mean_deg = c->n > 0 ? std::max(1.0, E / c->n) : 1.0;
    a.kids_min = c->kids_min >= 0 ? c->kids_min
                                  : (int)std::min<double>(INT32_MAX, std::max(4096.0, 4.0 * c->n / mean_deg));
    a.coff = (int*)c->cnt;
    a.kids = (int*)c->cnt + (c->vcap + 1);
    a.kids_bsum = (int*)c->app_bsum;
    a.kids_variant = kids_variant(a, c->Bcount);
    // wide Improve: a warp per vertex for long rows (measured: gamma* mean
    // degree 1,138 +14% with 32 lanes; gamma_k ~60-80 +30% slower with 32)
    a.wide_lpv = c->wide_lpv > 0 ? c->wide_lpv : (mean_deg >= 192.0 ? 32 : 16);
    a.num_sms = c->num_sms;
}

// Sharded exploit: per PI iteration
//   1. Improve over the owned part of I (v mod P == rank) -> records,
//   2. exchange: every rank's block of K + 1 records (its count in slot 0)
//      gathered into every rank's buffer -- one ncclAllGather (one process
//      per GPU), or device copies between the contexts of an in-process
//      group (pirrt_group_exploit: P ranks emulated on one GPU),
//   3. every rank applies all records and runs the identical Evaluate.
// The global Delta g is the max over the gathered records: no all-reduce.
// The loop state lives on the device and a kernel enqueued after the stop
// returns at once, so the host enqueues iterations in chunks (2, 4, 8, 16)
// and synchronises once per chunk instead of twice per iteration.  A rank
// that emitted more than K records stops the loop everywhere before any
// record is applied (every rank sees the same counts); the host then
// re-gathers that iteration with a larger K and carries on.
static int shard_exchange(std::vector<pirrt_ctx*>& cs, int K) {
    int rc = 0;
    (void)rc;
    const size_t bytes = (size_t)(K + 1) * sizeof(ShardRec);
    if (cs.size() == 1 && cs[0]->comm) {
        pirrt_ctx* c = cs[0];
        NC(nccl_api()->allGather(c->rec_local, c->rec_all, bytes, ncclChar, c->comm, c->stream));
        return 0;
    }
    // in-process group: rank q's block -> every rank's buffer, after q's Improve
    for (pirrt_ctx* q : cs) CU(cudaEventRecord(q->xev, q->stream));
    for (pirrt_ctx* c : cs)
        for (pirrt_ctx* q : cs) {
            if (q != c) CU(cudaStreamWaitEvent(c->stream, q->xev, 0));
            CU(cudaMemcpyAsync((char*)c->rec_all + (size_t)q->rank * bytes, q->rec_local, bytes,
                               cudaMemcpyDeviceToDevice, c->stream));
        }
    // a rank's Evaluate resets its record count: only after every copy of it
    for (pirrt_ctx* c : cs) CU(cudaEventRecord(c->xev2, c->stream));
    for (pirrt_ctx* q : cs)
        for (pirrt_ctx* c : cs)
            if (c != q) CU(cudaStreamWaitEvent(q->stream, c->xev2, 0));
    return 0;
}

static int nccl_async_check(pirrt_ctx* c) {
    if (!c->comm) return 0;                               // (an in-process group loads no NCCL)
    NcclApi* api = nccl_api();
    if (!api || !api->commGetAsyncError) return 0;
    ncclResult_t e = ncclSuccess;
    if (api->commGetAsyncError(c->comm, &e) != ncclSuccess || e != ncclSuccess) {
        c->broken = true;
        return fail(PIRRT_E_NCCL, std::string("exploit: NCCL asynchronous error: ") + api->errorString(e));
    }
    return 0;
}

static int exploit_sharded(std::vector<pirrt_ctx*>& cs) {
    int rc;
    pirrt_ctx* c0 = cs[0];
    const int P = c0->nranks;
    const size_t G = cs.size();
    std::vector<ExploitArgs> A(G);
    // records per rank: at most one per owned vertex of I
    const int64_t rec_max = (int64_t)c0->n / P + 2;
    int K = (int)std::min<int64_t>(rec_max, std::max<int64_t>(256, 2 * ((int64_t)c0->Bcount + 1) / P + 64));
    for (size_t i = 0; i < G; ++i) {
        pirrt_ctx* c = cs[i];
        ExploitArgs& a = A[i];
        fill_exploit_args(c, a, c->shard_blocks);
        a.shard_rank = c->rank;
        a.shard_n = P;
        a.shard_dev = 1;
        a.shard_K = K;
        a.wide_tasks = c->wide_tasks;
        // (sized by the vertex capacity, which grows geometrically, not by n:
        // a reallocation inside the loop's first launch cost tens of ms)
        if ((rc = grow(c->rec_local, c->rec_local_cap, std::max<int64_t>(rec_max, c->vcap / P + 2) + 1, 0,
                       c->stream)))
            return rc;
        if ((rc = grow(c->rec_all, c->rec_all_cap, (int64_t)P * (K + 1), 0, c->stream))) return rc;
        a.rec_count = &c->rec_local[0].v;
        a.rec_out = c->rec_local + 1;
        // the device-resident loop state (DevCtl was zeroed by the caller)
        const int st4[4] = {c->Bsel, c->Bcount, 0, 0};   // Bsel_out, Bcount_out, old_Bcount_out, pending_out
        static_assert(offsetof(DevCtl, Bcount_out) == offsetof(DevCtl, Bsel_out) + 4 &&
                      offsetof(DevCtl, old_Bcount_out) == offsetof(DevCtl, Bsel_out) + 8 &&
                      offsetof(DevCtl, pending_out) == offsetof(DevCtl, Bsel_out) + 12, "DevCtl layout");
        CU(cudaMemcpyAsync(&c->ctl->Bsel_out, st4, sizeof st4, cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemcpyAsync(&c->ctl->ev_out, &c->ev_next, sizeof(unsigned), cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemsetAsync(c->rec_local, 0, sizeof(ShardRec), c->stream));
        CU(cudaStreamSynchronize(c->stream));           // (host sources above are on the stack)
    }
    int Bc_known = c0->Bcount, stop = 0, it = 1;
    const bool dbg = std::getenv("PIRRT_DEBUG_HOST") != nullptr;
    auto now_us = []() {
        return std::chrono::duration<double, std::micro>(
                   std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double t_in = dbg ? now_us() : 0.0;
    auto evaluate_all = [&](int itv) -> int {
        for (size_t i = 0; i < G; ++i) {
            A[i].shard_K = K;
            A[i].pending = 0;
            A[i].kids_variant = kids_variant(A[i], Bc_known);
            CU(launch_shard_evaluate(A[i], itv, cs[i]->rec_all, P, cs[i]->shard_blocks, cs[i]->stream));
            cs[i]->launches += 1;
        }
        return 0;
    };
    for (int chunk = 2;; chunk = std::min(2 * chunk, 16)) {
        for (int j = 0; j < chunk; ++j, ++it) {
            for (size_t i = 0; i < G; ++i) {
                pirrt_ctx* c = cs[i];
                // the device picks one of the two Improve launches (|I| vs wide_tasks)
                if (c->wide_tasks > 0) { CU(launch_improve_wide(A[i], it, c->num_sms, c->stream)); c->launches += 1; }
                CU(launch_shard_improve(A[i], it, c->shard_blocks, c->stream));
                c->launches += 1;
            }
            if ((rc = shard_exchange(cs, K))) return rc;
            if ((rc = evaluate_all(it))) return rc;
        }
        const double t_enq = dbg ? now_us() : 0.0;
        stop = 0;
        for (size_t i = 0; i < G; ++i) {
            if ((rc = read_ctl(cs[i]))) return rc;
            if ((rc = nccl_async_check(cs[i]))) return rc;
            const int si = cs[i]->ctl_host->shard_stop;
            if (i > 0 && si != stop) { cs[i]->broken = true; return fail(PIRRT_E_CORRUPT, "exploit: ranks disagree on the stop"); }
            stop = si;
        }
        const DevCtl& h = *c0->ctl_host;
        if (dbg) std::fprintf(stderr, "pirrt host: sharded chunk %d (it %d): enqueued +%.1f us, done +%.1f us, stop %d\n",
                              chunk, it, t_enq - t_in, now_us() - t_in, h.shard_stop);
        Bc_known = h.Bcount_out;
        if (stop == 4) {                                  // a rank had more than K records
            const int it_o = h.shard_over_it;
            K = (int)std::min<int64_t>(rec_max, std::max<int64_t>(2LL * h.shard_over, 2LL * K));
            for (size_t i = 0; i < G; ++i) {
                pirrt_ctx* c = cs[i];
                if ((rc = grow(c->rec_all, c->rec_all_cap, (int64_t)P * (K + 1), 0, c->stream))) return rc;
                CU(cudaMemsetAsync(&c->ctl->shard_stop, 0, sizeof(int), c->stream));
            }
            if ((rc = shard_exchange(cs, K))) return rc;
            if ((rc = evaluate_all(it_o))) return rc;
            it = it_o + 1;
            continue;
        }
        if (stop || h.abort_at) break;
    }
    if (stop == 3) {                                      // R11 cap: finish the pending leave_B
        for (size_t i = 0; i < G; ++i) {
            pirrt_ctx* c = cs[i];
            if (c->ctl_host->pending_out) {
                A[i].shard_finish = 1;
                CU(launch_shard_improve(A[i], it, c->shard_blocks, c->stream));
                c->launches += 1;
                CU(cudaStreamSynchronize(c->stream));
            }
        }
    }
    for (pirrt_ctx* c : cs) {
        const DevCtl& h = *c->ctl_host;
        c->Bsel = h.Bsel_out;
        c->Bcount = h.Bcount_out;
        c->ev_next = h.ev_out;
    }
    return stop == 3 ? PIRRT_E_NOCONV : 0;
}

}  // extern "C"

namespace {

// Exploit, split for the asynchronous form:
// exploit_launch enqueues the first persistent launch (single GPU) and
// returns; exploit_finish reads the control block, serves wide-Improve
// hand-offs and fills the stats.  The sharded loop is host-driven (NCCL
// between the phases), so it runs entirely inside exploit_launch.
int exploit_launch(pirrt_ctx* c) {
    cudaStream_t s = c->stream;
    CU(cudaMemsetAsync(c->ctl, 0, offsetof(DevCtl, err), s));
    CU(cudaEventRecord(c->ev0, s));
    c->x_rc = 0;
    if (c->sharded) {
        if (!c->comm) return fail(PIRRT_E_STATE, "exploit: an in-process group rank runs only through pirrt_group_exploit");
        std::vector<pirrt_ctx*> cs{c};
        c->x_rc = exploit_sharded(cs);
        if (c->x_rc != 0 && c->x_rc != PIRRT_E_NOCONV && c->nranks > 1) {
            // a rank that fails on its own (e.g. an allocation) must not leave
            // its peers blocked in the next all-gather: abort the communicator
            NcclApi* api = nccl_api();
            if (api && api->commAbort) { api->commAbort(c->comm); c->comm = nullptr; }
        }
        if (c->x_rc != 0 && c->x_rc != PIRRT_E_NOCONV) { c->broken = true; return c->x_rc; }
        CU(cudaEventRecord(c->ev1, s));
        return 0;
    }
    // size-adaptive grid: a small improve set and
    // few appended vertices since the last exploit -> a small persistent
    // grid (cheaper grid barriers; the phases have little parallel work)
    c->x_blocks = c->grid_blocks;
    if (c->small_grid > 0 && (int64_t)c->Bcount + (c->n - c->n_last_exploit) <= c->small_max)
        c->x_blocks = std::min(c->small_grid, c->grid_blocks);
    c->n_last_exploit = c->n;
    fill_exploit_args(c, c->x_args, c->x_blocks);
    c->x_args.wide_tasks = c->wide_tasks;
    c->x_args.it_base = 1;
    const long long l0 = g_kernel_launches;
    cudaError_t e = launch_exploit(c->x_args, c->x_blocks, c->l2win, s);
    c->launches += g_kernel_launches - l0;
    if (e != cudaSuccess) { c->broken = true; return fail(PIRRT_E_CUDA, std::string("exploit launch: ") + cudaGetErrorString(e)); }
    CU(cudaEventRecord(c->ev1, s));                      // re-recorded after every resume
    return 0;
}

// the exploit counters of a control-block read-back (pirrt_exploit_stats)
void stats_from(const DevCtl& h, pirrt_exploit_stats* st, int blocks, float device_ms) {
    std::memset(st, 0, sizeof(*st));
    st->iterations = h.iterations;
    st->evaluations = h.evaluations;
    st->last_delta_g = h.last_dg;
    st->relaxations = h.relaxations;
    st->eval_visits = h.eval_visits;
    st->max_level = h.max_level;
    st->promising = h.promising;
    st->stalled = h.stalled;
    st->grid_blocks = blocks;
    st->device_ms = device_ms;
    st->improve_ms = (float)(h.t_improve * 1e-6);
    st->evaluate_ms = (float)(h.t_evaluate * 1e-6);
    st->improve_set = h.improve_set;
    st->eval_scanned = h.eval_scanned;
    st->barriers = h.barriers;
    st->eval_work = h.work_visits;
    st->full_evaluations = h.full_evals;
    st->inc_evaluations = h.inc_evals;
    st->relax_work = h.relax_work;
    st->improve_work = h.improve_work;
    st->inc_improves = h.inc_imps;
}

int exploit_finish(pirrt_ctx* c, pirrt_exploit_stats* st) {
    cudaStream_t s = c->stream;
    int rc;
    const bool dbg = std::getenv("PIRRT_DEBUG_HOST") != nullptr;
    auto now_us = []() {
        return std::chrono::duration<double, std::micro>(
                   std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double t_in = dbg ? now_us() : 0.0;
    if ((rc = read_ctl(c))) { c->broken = true; return rc; }
    if (dbg) std::fprintf(stderr, "pirrt host: first launch done +%.1f us (handoff=%d it=%d)\n",
                          now_us() - t_in, c->ctl_host->handoff, c->ctl_host->handoff_it);
    if (!c->sharded) {
        // wide-Improve hand-offs (large improve sets): Improve of iteration
        // handoff_it at full occupancy, then the loop resumes after it
        const long long l0 = g_kernel_launches;
        while (c->ctl_host->handoff && !c->ctl_host->abort_at) {
            const DevCtl& h = *c->ctl_host;
            ExploitArgs w = c->x_args;
            w.Bsel = h.Bsel_out; w.Bcount = h.Bcount_out; w.old_Bcount = h.old_Bcount_out;
            w.pending = h.pending_out;
            w.ev_base = c->ev_next + (unsigned)h.evaluations;
            w.kids_variant = w.kids_variant || kids_variant(w, w.Bcount);
            const int it = h.handoff_it;
            CU(cudaMemsetAsync(&c->ctl->handoff, 0, 2 * sizeof(int) + 2 * sizeof(unsigned long long), s));
            cudaError_t e;
            if ((e = launch_improve_wide(w, it, c->num_sms, s)) == cudaSuccess) {
                ExploitArgs r = w;
                r.pending = 0;
                r.it_base = it;
                r.resume = 1;
                e = launch_exploit(r, c->x_blocks, c->l2win, s);
            }
            if (e != cudaSuccess) { c->broken = true; return fail(PIRRT_E_CUDA, std::string("exploit launch: ") + cudaGetErrorString(e)); }
            CU(cudaEventRecord(c->ev1, s));
            if ((rc = read_ctl(c))) { c->broken = true; return rc; }
            if (dbg) std::fprintf(stderr, "pirrt host: wide Improve it=%d + resume done +%.1f us "
                                  "(wide span %.1f us, next handoff=%d)\n", it, now_us() - t_in,
                                  (c->ctl_host->t_wide1 - ~c->ctl_host->t_wide0) * 1e-3,
                                  c->ctl_host->handoff);
        }
        c->launches += g_kernel_launches - l0;
        c->Bsel = c->ctl_host->Bsel_out;
        c->Bcount = c->ctl_host->Bcount_out;
        c->ev_next += (unsigned)c->ctl_host->evaluations;
    }
    const DevCtl& h = *c->ctl_host;
    if (st) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev0, c->ev1);
        stats_from(h, st, c->sharded ? c->shard_blocks : c->x_blocks, ms);
    }
    if (h.abort_at) {
        c->broken = true;
        return fail(PIRRT_E_STATE, "exploit: watchdog fired (PIRRT_WATCHDOG_MS); context unusable");
    }
    if (c->x_rc == PIRRT_E_NOCONV || h.status == PIRRT_E_NOCONV)
        return fail(PIRRT_E_NOCONV, "exploit: iteration cap exceeded");
    return PIRRT_OK;
}

// Complete an exploit started by pirrt_exploit_async before any other call
// touches the context; its result is kept for pirrt_exploit_wait.  Returns
// nonzero only if the context became unusable.
int complete_pending(pirrt_ctx* c) {
    if (!c->inflight) return 0;
    c->inflight = false;
    c->kept_rc = exploit_finish(c, &c->kept_stats);
    c->kept = true;
    return c->broken ? c->kept_rc : 0;
}

// A new exploit discards an unwaited kept result -- unless that result was a
// failure (e.g. E_NOCONV of an asynchronous exploit another call completed):
// then the new exploit is not started and the failure is reported now.
int step_slot_init(pirrt_ctx* c, pirrt_ctx::StepSlot& sl) {
    if (!sl.ctl) {
        if (cudaMallocHost(&sl.ctl, sizeof(DevCtl) + kStepHeadBytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(PIRRT_E_NOMEM, "step_async: pinned slot");
        }
        sl.head = (int*)(sl.ctl + 1);                     // the best-path head after the block
        CU(cudaEventCreate(&sl.e0));
        CU(cudaEventCreate(&sl.e1));
        CU(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    }
    return grow(sl.dpath, sl.dpath_cap, c->vcap + 8, 0, c->stream);
}

// every outstanding step's kernels done; the host mirror of the B-list state
// refreshed from the device (before a capacity growth, which copies the list)
int drain_steps(pirrt_ctx* c) {
    CU(cudaStreamSynchronize(c->stream));
    int v[3];
    CU(cudaMemcpy(v, &c->ctl->dev_Bsel, sizeof v, cudaMemcpyDeviceToHost));
    c->Bsel = v[0];
    c->Bcount = v[1];
    c->ev_next = (unsigned)v[2];
    return 0;
}

int take_kept_failure(pirrt_ctx* c) {
    if (!c->kept) return 0;
    c->kept = false;
    if (c->kept_rc == PIRRT_OK) return 0;
    return fail(c->kept_rc, "the previous asynchronous exploit failed (reported late; no new "
                            "exploit was started)");
}

}  // namespace

extern "C" {

int pirrt_exploit(pirrt_ctx* c, pirrt_exploit_stats* st) {
    if (!c) return fail(PIRRT_E_INVAL, "exploit: NULL context");
    int rc;
    if ((rc = set_device(c))) return rc;
    if ((rc = complete_pending(c))) return rc;
    if ((rc = take_kept_failure(c))) return rc;
    if ((rc = exploit_launch(c))) return rc;
    return exploit_finish(c, st);
}

int pirrt_group_exploit(pirrt_ctx* const* ctxs, int32_t n, pirrt_exploit_stats* stats) {
    if (!ctxs || n < 1) return fail(PIRRT_E_INVAL, "group_exploit: bad arguments");
    std::vector<pirrt_ctx*> cs(ctxs, ctxs + n);
    for (int32_t i = 0; i < n; ++i) {
        pirrt_ctx* c = cs[i];
        if (!c) return fail(PIRRT_E_INVAL, "group_exploit: NULL context");
        if (!(c->cfg.flags & PIRRT_F_LOCAL_GROUP) || c->nranks != n || c->rank != i || c->n != cs[0]->n)
            return fail(PIRRT_E_STATE, "group_exploit: contexts must be ranks 0..n-1 of one PIRRT_F_LOCAL_GROUP "
                                       "group with the same graph");
        if (c->broken) return fail(PIRRT_E_STATE, "group_exploit: context unusable");
    }
    int rc;
    for (pirrt_ctx* c : cs) {
        if ((rc = set_device(c))) return rc;
        if ((rc = complete_pending(c))) return rc;
        c->kept = false;
        CU(cudaMemsetAsync(c->ctl, 0, offsetof(DevCtl, err), c->stream));
        CU(cudaEventRecord(c->ev0, c->stream));
        c->x_rc = 0;
    }
    const int lrc = exploit_sharded(cs);
    if (lrc != 0 && lrc != PIRRT_E_NOCONV) {
        for (pirrt_ctx* c : cs) c->broken = true;
        return lrc;
    }
    int out = PIRRT_OK;
    for (int32_t i = 0; i < n; ++i) {
        pirrt_ctx* c = cs[i];
        c->x_rc = lrc;
        CU(cudaEventRecord(c->ev1, c->stream));
        const int r = exploit_finish(c, stats ? &stats[i] : nullptr);
        if (r != PIRRT_OK && out == PIRRT_OK) out = r;
    }
    return out;
}

int pirrt_exploit_async(pirrt_ctx* c) {
    if (!c) return fail(PIRRT_E_INVAL, "exploit_async: NULL context");
    int rc;
    if ((rc = set_device(c))) return rc;
    if ((rc = complete_pending(c))) return rc;
    if ((rc = take_kept_failure(c))) return rc;
    if ((rc = exploit_launch(c))) return rc;
    c->inflight = true;
    return PIRRT_OK;
}

int pirrt_exploit_wait(pirrt_ctx* c, pirrt_exploit_stats* st) {
    if (!c) return fail(PIRRT_E_INVAL, "exploit_wait: NULL context");
    int rc;
    if ((rc = set_device(c))) return rc;
    if (c->inflight) {
        c->inflight = false;
        return exploit_finish(c, st);
    }
    if (!c->kept) return fail(PIRRT_E_STATE, "exploit_wait: no exploit was started");
    c->kept = false;
    if (st) *st = c->kept_stats;
    return c->kept_rc == PIRRT_OK ? PIRRT_OK : fail(c->kept_rc, "exploit: failed (reported late)");
}

// ---- deferred BE-RRT# steps
//
// One call enqueues a whole step of Alg. 3 -- Extend's append,
// the guarded Replan (R10) and the path read-out -- with
// no host synchronisation: the inputs' H2D runs on the copy stream behind the
// previous step's append (so it overlaps that step's exploit), the kernels
// take the B-list state the previous step left on the device (DevCtl dev_*)
// and the Alg. 3 guard is decided by the exploit kernel itself (nprom == 0:
// it returns at once).  The results land in the slot's pinned buffers.
int pirrt_step_async(pirrt_ctx* c, int32_t n_new, const double* h_new, int64_t n_edges,
                     const pirrt_vid* src, const pirrt_vid* dst, const double* cost, uint32_t flags) {
    if (!c) return fail(PIRRT_E_INVAL, "step_async: NULL context");
    int rc;
    if ((rc = set_device(c, true))) return rc;
    if (c->steps_out >= kStepDepth) return fail(PIRRT_E_STATE, "step_async: two steps outstanding (pirrt_step_wait first)");
    if (c->sharded) return fail(PIRRT_E_STATE, "step_async: single-GPU contexts only");
    if (c->w_d != 0) return fail(PIRRT_E_STATE, "step_async: a context with a world grows through pirrt_extend_batch");
    if ((flags | c->cfg.flags) & PIRRT_F_VALIDATE)
        return fail(PIRRT_E_INVAL, "step_async: PIRRT_F_VALIDATE needs the synchronous append");
    if (n_new < 0 || n_edges < 0) return fail(PIRRT_E_INVAL, "step_async: negative size");
    if (n_new > 0 && !h_new) return fail(PIRRT_E_INVAL, "step_async: h_new is NULL");
    if (n_edges > 0 && (!src || !dst || !cost)) return fail(PIRRT_E_INVAL, "step_async: NULL edge array");
    if ((int64_t)c->n + n_new > INT32_MAX - 1) return fail(PIRRT_E_RANGE, "step_async: too many vertices");
    if ((rc = complete_pending(c))) return rc;            // an exploit_async still running
    if ((rc = take_kept_failure(c))) return rc;
    const bool dev = (flags & PIRRT_F_DEVICE_PTRS) != 0;
    const bool undirected = (flags & PIRRT_F_EDGES_UNDIRECTED) != 0;
    const int64_t m_dir = undirected ? 2 * n_edges : n_edges;
    cudaStream_t s = c->stream;
    const int n_old = c->n, n_all = c->n + n_new;
    const int nb = 1 - c->cur;
    const int64_t dneed = c->delta_edges + m_dir;
    // a capacity growth copies the B list by the host's count: bring the
    // host mirror up to date first (rare: capacities grow geometrically)
    const bool growth = n_all > c->vcap || dneed > c->didx_cap[nb] || dneed > c->dcost_cap[nb] ||
                        dneed > c->odidx_cap[nb] ||
                        (!dev && (n_new > c->s_h_cap || n_edges > c->s_src_cap ||
                                  n_edges > c->s_dst_cap || n_edges > c->s_cost_cap));
    if (growth && c->steps_out > 0 && (rc = drain_steps(c))) { c->broken = true; return rc; }
    if ((rc = ensure_vertices(c, n_all))) return rc;
    if ((rc = grow(c->didx[nb], c->didx_cap[nb], dneed, 0, s))) return rc;
    if ((rc = grow(c->dcost[nb], c->dcost_cap[nb], dneed, 0, s))) return rc;
    if ((rc = grow(c->odidx[nb], c->odidx_cap[nb], dneed, 0, s))) return rc;
    pirrt_ctx::StepSlot& sl = c->slot[(c->step_head + c->steps_out) % kStepDepth];
    if ((rc = step_slot_init(c, sl))) return rc;
    if (!c->app_done) CU(cudaEventCreateWithFlags(&c->app_done, cudaEventDisableTiming));
    // inputs: H2D on the copy stream once the previous step's append has
    // consumed the staging buffers -- it overlaps that step's exploit
    const double* d_h = h_new;
    const int *d_src = src, *d_dst = dst;
    const double* d_cost = cost;
    if (!dev) {
        CU(cudaStreamWaitEvent(c->copy_stream, c->app_done, 0));
        if ((rc = stage(c, h_new, n_new, false, c->s_h, c->s_h_cap, &d_h, c->copy_stream))) return rc;
        if ((rc = stage(c, src, n_edges, false, c->s_src, c->s_src_cap, &d_src, c->copy_stream))) return rc;
        if ((rc = stage(c, dst, n_edges, false, c->s_dst, c->s_dst_cap, &d_dst, c->copy_stream))) return rc;
        if ((rc = stage(c, cost, n_edges, false, c->s_cost, c->s_cost_cap, &d_cost, c->copy_stream))) return rc;
        CU(cudaEventRecord(c->copy_done, c->copy_stream));
        CU(cudaStreamWaitEvent(s, c->copy_done, 0));
    }
    // append (Extend's local relaxation and promising test, R14 / P:184-188)
    static_assert(offsetof(DevCtl, nprom) == offsetof(DevCtl, err) + 2 * sizeof(int), "DevCtl layout");
    CU(cudaMemsetAsync(&c->ctl->err, 0, 3 * sizeof(int), s));   // err, sweeps, nprom
    if ((rc = grow(c->app_chunk, c->app_chunk_cap, 2 * (c->delta_edges / kAppendCopyChunk + 2), 0, s)))
        return rc;
    AppendArgs a;
    fill_append_args(c, a, nb, n_old, n_new, d_h, nullptr, nullptr, d_src, d_dst, d_cost, n_edges,
                     undirected, false);
    a.dev_list = c->steps_out > 0 ? 1 : 0;                // the list as the previous step left it
    const long long l0 = g_kernel_launches;
    cudaError_t e = launch_append_fused(a, c->cnt + (c->cnt_cap / 2), c->app_bsum, kAppendMaxBlocks,
                                        c->l2win, s);
    if (e != cudaSuccess) { c->broken = true; return fail(PIRRT_E_CUDA, std::string("step_async: append: ") + cudaGetErrorString(e)); }
    CU(cudaEventRecord(c->app_done, s));
    // commit the host side (a rejected batch is reported by pirrt_step_wait
    // and leaves the context unusable)
    c->cur = nb;
    c->n = n_all;
    c->delta_edges += m_dir;
    c->edges_total += m_dir;
    if ((rc = compact_if_needed(c, m_dir, false))) { c->broken = true; return rc; }
    // Replan, guarded on the device (R10).  Grid size and the instantiation
    // are chosen from the host's last known |B| plus this batch (an upper
    // bound of its new members); neither changes the result
    const int64_t bc_est = (int64_t)c->Bcount + n_new;
    int blocks = c->grid_blocks;
    if (c->small_grid > 0 && bc_est + (c->n - c->n_last_exploit) <= c->small_max)
        blocks = std::min(c->small_grid, c->grid_blocks);
    c->n_last_exploit = c->n;
    ExploitArgs x;
    fill_exploit_args(c, x, blocks);
    x.kids_variant = kids_variant(x, (int)std::min<int64_t>(bc_est, INT32_MAX));
    x.wide_tasks = 0;                                     // no host hand-off inside a step
    x.it_base = 1;
    x.step_mode = c->steps_out > 0 ? 2 : 1;
    CU(cudaMemsetAsync(c->ctl, 0, offsetof(DevCtl, err), s));
    CU(cudaEventRecord(sl.e0, s));
    if ((e = launch_exploit(x, blocks, c->l2win, s)) != cudaSuccess) {
        c->broken = true;
        return fail(PIRRT_E_CUDA, std::string("step_async: exploit: ") + cudaGetErrorString(e));
    }
    CU(cudaEventRecord(sl.e1, s));
    sl.blocks = blocks;
    // path read-out (Alg. 1 lines 8-12) into the slot
    CU(launch_best_path(c->parent, c->g, c->n, c->goals, (int)c->goals_host.size(), sl.dpath, s,
                        (int*)(c->ctl + 1), kStepHead));
    c->launches += g_kernel_launches - l0;
    // one read-back: the control block's tail and the best-path head after it
    const size_t o = offsetof(DevCtl, status);
    CU(cudaMemcpyAsync((char*)sl.ctl + o, (const char*)c->ctl + o, sizeof(DevCtl) - o + kStepHeadBytes,
                       cudaMemcpyDeviceToHost, s));
    CU(cudaEventRecord(sl.done, s));
    ++c->steps_out;
    return PIRRT_OK;
}

int pirrt_step_wait(pirrt_ctx* c, pirrt_step_result* out, pirrt_vid* path_out, int64_t cap) {
    if (!c) return fail(PIRRT_E_INVAL, "step_wait: NULL context");
    int rc;
    if ((rc = set_device(c, true))) return rc;
    if (c->steps_out == 0) return fail(PIRRT_E_STATE, "step_wait: no step outstanding");
    pirrt_ctx::StepSlot& sl = c->slot[c->step_head];
    CU(cudaEventSynchronize(sl.done));
    c->step_head = (c->step_head + 1) % kStepDepth;
    --c->steps_out;
    const DevCtl& h = *sl.ctl;
    if (h.err) {
        c->broken = true;
        return fail((h.err & kErrRange) ? PIRRT_E_RANGE : PIRRT_E_INVAL,
                    "step: append rejected (context unusable):" + err_bits(h.err));
    }
    if (h.abort_at) {
        c->broken = true;
        return fail(PIRRT_E_STATE, "step: watchdog fired (PIRRT_WATCHDOG_MS); context unusable");
    }
    // the host mirror of the B-list state (exact once no step is outstanding)
    c->Bsel = h.dev_Bsel;
    c->Bcount = h.dev_Bcount;
    c->ev_next = h.dev_ev;
    pirrt_step_result r;
    std::memset(&r, 0, sizeof r);
    r.n_new_promising = h.nprom;
    r.replanned = h.nprom > 0 ? 1 : 0;
    if (r.replanned) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, sl.e0, sl.e1);
        stats_from(h, &r.stats, sl.blocks, ms);
    } else {
        r.stats.promising = h.promising;
    }
    const int len = sl.head[0];
    double gg;
    std::memcpy(&gg, &sl.head[2], sizeof(double));
    r.goal = -1;
    r.path_cost = INFINITY;
    if (!std::isinf(gg)) {
        if (len <= 0) return fail(PIRRT_E_CORRUPT, "step: best path: parent cycle");
        r.path_len = len;
        r.path_cost = gg;
        r.goal = sl.head[1];
    }
    if (out) *out = r;
    if (r.path_len > 0 && path_out) {
        if (cap < r.path_len) return fail(PIRRT_E_RANGE, "step_wait: path capacity too small");
        std::vector<int> rev(len);
        std::copy(sl.head + 4, sl.head + 4 + std::min(len, kStepHead), rev.begin());
        if (len > kStepHead)                              // the slot's buffer stays until its reuse
            CU(cudaMemcpy(rev.data() + kStepHead, sl.dpath + 4 + kStepHead,
                          (size_t)(len - kStepHead) * sizeof(int), cudaMemcpyDeviceToHost));
        if (rev.back() != kRoot) return fail(PIRRT_E_CORRUPT, "step: best path does not reach the root");
        for (int i = 0; i < len; ++i) path_out[i] = rev[len - 1 - i];
    }
    if (h.status == PIRRT_E_NOCONV) return fail(PIRRT_E_NOCONV, "step: exploit iteration cap exceeded");
    return PIRRT_OK;
}

int pirrt_steps_outstanding(const pirrt_ctx* c) { return c ? c->steps_out : 0; }

int pirrt_nccl_unique_id(void* out, int64_t cap) {
    if (!out || cap < (int64_t)sizeof(ncclUniqueId)) return fail(PIRRT_E_RANGE, "nccl_unique_id: need 128 bytes");
    NcclApi* api = nccl_api();
    if (!api) return fail(PIRRT_E_NCCL, "nccl_unique_id: libnccl.so.2 not loadable");
    ncclUniqueId id;
    NC(api->getUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
    return PIRRT_OK;
}

static int get_array(const pirrt_ctx* c, void* out, const void* dsrc, size_t elem, int64_t cap,
                     const char* what) {
    if (!c || !out) return fail(PIRRT_E_INVAL, std::string(what) + ": NULL argument");
    int rc;
    if ((rc = set_device(c))) return rc;
    if ((rc = complete_pending(const_cast<pirrt_ctx*>(c)))) return rc;
    if (cap < c->n) return fail(PIRRT_E_RANGE, std::string(what) + ": capacity too small");
    CU(cudaMemcpyAsync(out, dsrc, (size_t)c->n * elem, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return PIRRT_OK;
}

int pirrt_get_policy(const pirrt_ctx* c, pirrt_vid* out, int64_t cap) {
    return get_array(c, out, c ? c->parent : nullptr, sizeof(int), cap, "get_policy");
}
int pirrt_get_costs(const pirrt_ctx* c, double* out, int64_t cap) {
    return get_array(c, out, c ? c->g : nullptr, sizeof(double), cap, "get_costs");
}
int pirrt_get_promising(const pirrt_ctx* c, uint8_t* out, int64_t cap) {
    return get_array(c, out, c ? c->b : nullptr, 1, cap, "get_promising");
}
int pirrt_get_parent_costs(const pirrt_ctx* c, double* out, int64_t cap) {
    return get_array(c, out, c ? c->pc : nullptr, sizeof(double), cap, "get_parent_costs");
}

int pirrt_get_in_edges(const pirrt_ctx* cc, int64_t* off_out, int64_t cap_v, pirrt_vid* src_out,
                       double* cost_out, int64_t cap_e) {
    pirrt_ctx* c = const_cast<pirrt_ctx*>(cc);
    if (!c || !off_out || !src_out || !cost_out) return fail(PIRRT_E_INVAL, "get_in_edges: NULL argument");
    int rc;
    if ((rc = set_device(c))) return rc;
    if ((rc = complete_pending(c))) return rc;
    const int64_t n = c->n, Eb = c->base_edges, Ed = c->delta_edges;
    if (cap_v < n + 1 || cap_e < Eb + Ed) return fail(PIRRT_E_RANGE, "get_in_edges: capacity too small");
    // base row of v, then its delta row (a copy of the store; no arithmetic)
    std::vector<long long> bo(n + 1, 0), dq(n + 1, 0);
    std::vector<int> bi(Eb), di(Ed);
    std::vector<double> bc(Eb), dc(Ed);
    cudaStream_t s = c->stream;
    CU(cudaMemcpyAsync(bo.data(), c->boff, (n + 1) * sizeof(long long), cudaMemcpyDeviceToHost, s));
    if (Eb) {
        CU(cudaMemcpyAsync(bi.data(), c->bidx, Eb * sizeof(int), cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(bc.data(), c->bcost, Eb * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    if (Ed) {
        CU(cudaMemcpyAsync(dq.data(), c->doff[c->cur], (n + 1) * sizeof(long long), cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(di.data(), c->didx[c->cur], Ed * sizeof(int), cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(dc.data(), c->dcost[c->cur], Ed * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    CU(cudaStreamSynchronize(s));
    int64_t k = 0;
    for (int64_t v = 0; v < n; ++v) {
        off_out[v] = k;
        for (long long e = bo[v]; e < bo[v + 1]; ++e, ++k) { src_out[k] = bi[e]; cost_out[k] = bc[e]; }
        for (long long e = dq[v]; e < dq[v + 1]; ++e, ++k) { src_out[k] = di[e]; cost_out[k] = dc[e]; }
    }
    off_out[n] = k;
    if (k != Eb + Ed) return fail(PIRRT_E_CORRUPT, "get_in_edges: row offsets disagree with the edge count");
    return PIRRT_OK;
}

int pirrt_bench_relax_ctx(const pirrt_ctx* cc, int32_t reps, float* ms_out, int64_t* entries_out) {
    pirrt_ctx* c = const_cast<pirrt_ctx*>(cc);
    if (!c || !ms_out || reps < 1) return fail(PIRRT_E_INVAL, "bench_relax_ctx: bad arguments");
    int rc;
    if ((rc = set_device(c))) return rc;
    if ((rc = complete_pending(c))) return rc;
    CU(cudaStreamSynchronize(c->stream));
    double* out = nullptr;
    if (cudaMalloc(&out, (size_t)std::max(c->n, 1) * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return fail(PIRRT_E_NOMEM, "bench_relax_ctx: scratch");
    }
    const int r = pirrt_bench_relax(c->boff, c->bidx, c->bcost, c->g, nullptr, c->n, out, reps, ms_out);
    cudaFree(out);
    if (r) return fail(PIRRT_E_CUDA, "bench_relax_ctx: kernel failed");
    if (entries_out) *entries_out = c->base_edges;
    return PIRRT_OK;
}

int pirrt_best_path(const pirrt_ctx* cc, pirrt_vid* path_out, int64_t cap, int64_t* len_out,
                    double* cost_out, pirrt_vid* goal_out) {
    pirrt_ctx* c = const_cast<pirrt_ctx*>(cc);
    if (!c) return fail(PIRRT_E_INVAL, "best_path: NULL context");
    int rc;
    if ((rc = set_device(c))) return rc;
    if ((rc = complete_pending(c))) return rc;
    cudaStream_t s = c->stream;
    // one small read-back (header + the first kHead entries); a second copy
    // only for paths longer than that
    constexpr int kHead = 1020;
    const long long l0 = g_kernel_launches;
    CU(launch_best_path(c->parent, c->g, c->n, c->goals, (int)c->goals_host.size(), c->path, s));
    c->launches += g_kernel_launches - l0;
    const int first = std::min<int64_t>(kHead, c->n + 1);
    std::vector<int> buf(4 + first);
    CU(cudaMemcpyAsync(buf.data(), c->path, sizeof(int) * (4 + first), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const int len = buf[0];
    double gg;
    std::memcpy(&gg, &buf[2], sizeof(double));
    if (std::isinf(gg)) {
        if (len_out) *len_out = 0;
        if (cost_out) *cost_out = INFINITY;
        if (goal_out) *goal_out = -1;
        return PIRRT_OK;
    }
    if (len < 0) return fail(PIRRT_E_CORRUPT, "best_path: parent cycle");
    std::vector<int> rev(len);
    std::copy(buf.begin() + 4, buf.begin() + 4 + std::min(len, first), rev.begin());
    if (len > first) {
        CU(cudaMemcpyAsync(rev.data() + first, c->path + 4 + first, (size_t)(len - first) * sizeof(int),
                           cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
    }
    if (len == 0 || rev.back() != kRoot)
        return fail(PIRRT_E_CORRUPT, "best_path: goal branch does not reach the root");
    if (cap < len) return fail(PIRRT_E_RANGE, "best_path: capacity too small");
    if (!path_out) return fail(PIRRT_E_INVAL, "best_path: NULL path_out");
    for (int i = 0; i < len; ++i) path_out[i] = rev[len - 1 - i];
    if (len_out) *len_out = len;
    if (cost_out) *cost_out = gg;
    if (goal_out) *goal_out = buf[1];
    return PIRRT_OK;
}

int pirrt_set_policy(pirrt_ctx* c, const pirrt_vid* parent, const double* g, const uint8_t* b) {
    if (!c) return fail(PIRRT_E_INVAL, "set_policy: NULL context");
    if (!parent || !g) return fail(PIRRT_E_INVAL, "set_policy: NULL array");
    if (c->own_n > 1)
        return fail(PIRRT_E_STATE, "set_policy: the policy-edge costs of other ranks' vertices are not "
                                   "stored on this rank (partitioned sharded store)");
    int rc;
    if ((rc = set_device(c))) return rc;
    if ((rc = complete_pending(c))) return rc;
    cudaStream_t s = c->stream;
    const int n = c->n;
    const int* d_parent;
    const double* d_g;
    const unsigned char* d_b = nullptr;
    // host-side canonicalisation of the snapshot: -0.0 -> +0.0, b -> {0,1}
    std::vector<double> gh(g, g + n);
    for (double& x : gh) x = x + 0.0;
    std::vector<unsigned char> bh;
    if (b) {
        bh.resize(n);
        for (int v = 0; v < n; ++v) bh[v] = b[v] ? 1 : 0;
    }
    if ((rc = stage(c, parent, n, false, c->s_parent, c->s_parent_cap, &d_parent))) return rc;
    if ((rc = stage(c, (const double*)gh.data(), n, false, c->s_g, c->s_g_cap, &d_g))) return rc;
    if (b && (rc = stage(c, (const unsigned char*)bh.data(), n, false, c->s_b, c->s_b_cap, &d_b))) return rc;
    if ((rc = grow(c->s_pc, c->s_pc_cap, n, 0, s))) return rc;
    CU(cudaMemsetAsync(c->s_pc, 0, (size_t)n * sizeof(double), s));
    CU(cudaMemsetAsync(&c->ctl->err, 0, sizeof(int), s));
    PolicyArgs a;
    a.boff = c->boff; a.bidx = c->bidx; a.bcost = c->bcost;
    a.doff = c->doff[c->cur]; a.didx = c->didx[c->cur]; a.dcost = c->dcost[c->cur];
    a.parent_in = d_parent; a.g_in = d_g; a.b_in = d_b;
    a.parent = nullptr; a.g = nullptr; a.pc = c->s_pc; a.b = nullptr;
    a.n = n; a.ctl = c->ctl;
    const long long l0 = g_kernel_launches;
    CU(launch_set_policy(a, s));
    if (c->cfg.flags & PIRRT_F_VALIDATE) CU(launch_cycle_check(d_parent, n, (int*)c->cnt, c->ctl, s));
    c->launches += g_kernel_launches - l0;
    if ((rc = read_ctl(c))) return rc;
    if (c->ctl_host->err) {
        const int err = c->ctl_host->err;
        const int code = (err & kErrRange) ? PIRRT_E_RANGE
                       : (err & kErrCycle) ? PIRRT_E_CORRUPT : PIRRT_E_INVAL;
        return fail(code, "set_policy rejected:" + err_bits(err));
    }
    // commit (g canonicalised: -0.0 -> +0.0 is irrelevant for validated g >= 0)
    CU(cudaMemcpyAsync(c->parent, d_parent, (size_t)n * sizeof(int), cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(c->g, d_g, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(c->pc, c->s_pc, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (d_b) {
        CU(cudaMemcpyAsync(c->b, d_b, (size_t)n, cudaMemcpyDeviceToDevice, s));
    } else {
        CU(cudaMemsetAsync(c->b, 0, (size_t)n, s));
    }
    // the B list is the device-side representation of b;
    // both list buffers restart from the all -1 state
    for (int k = 0; k < 2; ++k)
        CU(cudaMemsetAsync(c->Bq[k] + 1, 0xFF, (size_t)(c->Bq_cap[k] - 1) * sizeof(int), s));
    int* cnt_dev = c->path + (c->path_cap - 1);
    const long long l1 = g_kernel_launches;
    CU(launch_rebuild_blist(c->b, n, c->Bq[c->Bsel], cnt_dev, c->cnt, c->scan_tmp, s));
    c->launches += g_kernel_launches - l1;
    // policy-tree child counts of the restored policy; the next Evaluate
    // is a full one (the incremental form needs the last Evaluate's B)
    CU(cudaMemsetAsync(c->ccd, 0, (size_t)n * sizeof(int2), s));
    const long long l2 = g_kernel_launches;
    CU(launch_child_count(c->parent, 0, n, c->ccd, s));
    c->launches += g_kernel_launches - l2;
    CU(set_need_full(c, true));
    int bc = 0;
    CU(cudaMemcpyAsync(&bc, cnt_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    c->Bcount = bc;
    return PIRRT_OK;
}


// ---- device-side Extend

int pirrt_set_world(pirrt_ctx* c, int32_t d, int32_t n_boxes, const double* boxes,
                    const double* x_init, const double* x_goal, double gamma) {
    if (!c) return fail(PIRRT_E_INVAL, "set_world: NULL context");
    if (d < 1 || d > 16 || n_boxes < 0 || (n_boxes > 0 && !boxes) || !x_init || !x_goal ||
        !(gamma > 0.0) || std::isinf(gamma))
        return fail(PIRRT_E_INVAL, "set_world: bad arguments");
    int rc;
    if ((rc = set_device(c))) return rc;
    if ((rc = complete_pending(c))) return rc;
    if (c->n != 2) return fail(PIRRT_E_STATE, "set_world: must precede the first append");
    for (int64_t k = 0; k < (int64_t)n_boxes * 2 * d; ++k)
        if (!std::isfinite(boxes[k])) return fail(PIRRT_E_INVAL, "set_world: non-finite box");
    for (int k = 0; k < d; ++k)
        if (!std::isfinite(x_init[k]) || !std::isfinite(x_goal[k]))
            return fail(PIRRT_E_INVAL, "set_world: non-finite point");
    cudaStream_t s = c->stream;
    if ((rc = grow(c->w_boxes, c->w_boxes_cap, std::max<int64_t>(1, (int64_t)n_boxes * 2 * d), 0, s))) return rc;
    if ((rc = grow(c->w_goal, c->w_goal_cap, d, 0, s))) return rc;
    if ((rc = grow(c->pts, c->pts_cap, std::max<int64_t>(2, c->vcap) * d, 0, s))) return rc;
    if (n_boxes) CU(cudaMemcpyAsync(c->w_boxes, boxes, sizeof(double) * n_boxes * 2 * d, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(c->w_goal, x_goal, sizeof(double) * d, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(c->pts, x_init, sizeof(double) * d, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(c->pts + d, x_goal, sizeof(double) * d, cudaMemcpyHostToDevice, s));
    CU(cudaStreamSynchronize(s));
    c->w_d = d; c->w_nboxes = n_boxes; c->w_gamma = gamma;
    return PIRRT_OK;
}

int pirrt_extend_batch(pirrt_ctx* c, int32_t n_new, const double* points, uint32_t flags,
                       int32_t* n_new_promising, int64_t* n_edges_out) {
    if (!c) return fail(PIRRT_E_INVAL, "extend: NULL context");
    int rc;
    if ((rc = set_device(c))) return rc;
    if ((rc = complete_pending(c))) return rc;
    if (c->w_d == 0) return fail(PIRRT_E_STATE, "extend: no world (pirrt_set_world)");
    if (n_new < 0 || (n_new > 0 && !points)) return fail(PIRRT_E_INVAL, "extend: bad arguments");
    if ((int64_t)c->n + n_new > INT32_MAX - 1) return fail(PIRRT_E_RANGE, "extend: too many vertices");
    const int d = c->w_d, n_old = c->n, n_all = c->n + n_new;
    const bool dev = (flags & PIRRT_F_DEVICE_PTRS) != 0;
    cudaStream_t s = c->stream;
    if (n_new == 0) {
        if (n_edges_out) *n_edges_out = 0;
        return pirrt_graph_append_batch(c, 0, nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr,
                                        0, n_new_promising);
    }
    // points of the new vertices go to slots >= n (invisible until the append commits)
    if ((rc = grow(c->pts, c->pts_cap, (int64_t)n_all * d, (int64_t)n_old * d, s))) return rc;
    CU(cudaMemcpyAsync(c->pts + (int64_t)n_old * d, points, sizeof(double) * n_new * d,
                       dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    // connection radii r(i + 1) = gamma (ln m / m)^(1/d), m = i + 1 (host libm,
    // the same as the CPU generator's), and the grid: cells of side >= the
    // largest radius of the batch (that of its first vertex), so a neighbour
    // lies in the 3^d cells around a point; at most 4 n_all cells
    std::vector<double> R(n_new);
    for (int t = 0; t < n_new; ++t) {
        const double m = (double)(n_old + t) + 1.0;
        R[t] = m < 2.0 ? 1e300 : c->w_gamma * std::pow(std::log(m) / m, 1.0 / d);
    }
    int mc = R[0] >= 1.0 ? 1 : (int)std::floor(1.0 / (R[0] * (1.0 + 1e-9)));
    while (mc > 1 && std::pow((double)mc, d) > 4.0 * (double)n_all) --mc;
    const int brute = mc < 3 ? 1 : 0;
    long long ncell = 1;
    if (!brute) for (int k = 0; k < d; ++k) ncell *= mc;
    if ((rc = grow(c->x_R, c->x_R_cap, n_new, 0, s))) return rc;
    if ((rc = grow(c->x_h, c->x_h_cap, n_new, 0, s))) return rc;
    if ((rc = grow(c->x_ecnt, c->x_ecnt_cap, n_new + 1, 0, s))) return rc;
    if ((rc = grow(c->x_eoff, c->x_eoff_cap, n_new + 1, 0, s))) return rc;
    if ((rc = grow(c->x_tmp, c->x_tmp_cap, (int64_t)std::max(scan_tmp_elems(ncell + 1), scan_tmp_elems(n_new + 1)), 0, s))) return rc;
    if (!brute) {
        if ((rc = grow(c->x_cell, c->x_cell_cap, n_all, 0, s))) return rc;
        if ((rc = grow(c->x_cpts, c->x_cpts_cap, n_all, 0, s))) return rc;
        if ((rc = grow(c->x_ccnt, c->x_ccnt_cap, ncell + 1, 0, s))) return rc;
        if ((rc = grow(c->x_cstart, c->x_cstart_cap, ncell + 1, 0, s))) return rc;
    }
    CU(cudaMemcpyAsync(c->x_R, R.data(), sizeof(double) * n_new, cudaMemcpyHostToDevice, s));
    // hit cache: the count pass keeps up to hcap (neighbour, distance) pairs
    // per new vertex, so the write pass copies them instead of searching
    // again (only vertices with more hits are searched twice); bounded to
    // 1 GiB, off when the expected degree is beyond the cap
    int hcap = c->x_hcap;
    if ((int64_t)n_new * hcap * 12 > (1ll << 30)) hcap = (int)((1ll << 30) / (12ll * n_new));
    if (hcap < 16) hcap = 0;
    if (hcap > 0) {
        if ((rc = grow(c->x_hj, c->x_hj_cap, (int64_t)n_new * hcap, 0, s))) return rc;
        if ((rc = grow(c->x_hd, c->x_hd_cap, (int64_t)n_new * hcap, 0, s))) return rc;
    }
    ExtendArgs a;
    a.hcap = hcap; a.hj = c->x_hj; a.hd = c->x_hd;
    a.pts = c->pts; a.n_old = n_old; a.n_new = n_new; a.d = d; a.m = mc; a.brute = brute;
    a.ncell = ncell; a.cell = c->x_cell; a.ccnt = c->x_ccnt; a.cstart = c->x_cstart; a.cpts = c->x_cpts;
    a.scan_tmp = c->x_tmp; a.R = c->x_R; a.boxes = c->w_boxes; a.n_boxes = c->w_nboxes;
    a.x_goal = c->w_goal; a.h_new = c->x_h; a.ecnt = c->x_ecnt; a.eoff = c->x_eoff;
    a.src = nullptr; a.dst = nullptr; a.cost = nullptr;
    const long long l0 = g_kernel_launches;
    CU(launch_extend_grid(a, s));
    long long total = 0;
    CU(cudaMemcpyAsync(&total, c->x_eoff + n_new, sizeof(long long), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if ((rc = grow(c->x_src, c->x_src_cap, std::max<long long>(1, total), 0, s))) return rc;
    if ((rc = grow(c->x_dst, c->x_dst_cap, std::max<long long>(1, total), 0, s))) return rc;
    if ((rc = grow(c->x_cost, c->x_cost_cap, std::max<long long>(1, total), 0, s))) return rc;
    a.src = c->x_src; a.dst = c->x_dst; a.cost = c->x_cost;
    if (total > 0) CU(launch_extend_edges(a, s));
    c->launches += g_kernel_launches - l0;
    {   // next batch's cache: twice this batch's mean hits, a power of two in [32, 512], else off
        const double mean = (double)total / n_new;
        int hc = 32;
        while (hc < 2.0 * mean && hc < 1024) hc *= 2;
        c->x_hcap = hc > 512 ? 0 : hc;
    }
    if (n_edges_out) *n_edges_out = total;
    // the ordinary append (a1): store, Extend's local relaxation, promising test
    c->in_extend = true;
    rc = pirrt_graph_append_batch(c, n_new, c->x_h, nullptr, nullptr, total, c->x_src, c->x_dst,
                                  c->x_cost,
                                  PIRRT_F_EDGES_UNDIRECTED | PIRRT_F_DEVICE_PTRS | (flags & PIRRT_F_VALIDATE),
                                  n_new_promising);
    c->in_extend = false;
    return rc;
}

int pirrt_get_points(const pirrt_ctx* c, double* out, int64_t cap) {
    if (!c || !out) return fail(PIRRT_E_INVAL, "get_points: NULL argument");
    if (c->w_d == 0) return fail(PIRRT_E_STATE, "get_points: no world");
    int rc;
    if ((rc = set_device(c))) return rc;
    if (cap < (int64_t)c->n * c->w_d) return fail(PIRRT_E_RANGE, "get_points: capacity too small");
    CU(cudaMemcpyAsync(out, c->pts, sizeof(double) * c->n * c->w_d, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return PIRRT_OK;
}

}  // extern "C"

// ---- debug-only export (not part of include/pirrt.h): the device B list
// diagnostics (not part of the ABI header): the last exploit's phase
// timeline, DevCtl::phase_ns
extern "C" int pirrt_debug_phases(const pirrt_ctx* c, unsigned long long* out, int n) {
    if (!c || !out || n < 8) return fail(PIRRT_E_INVAL, "debug_phases: bad arguments");
    std::memcpy(out, c->ctl_host->phase_ns, 8 * sizeof(unsigned long long));
    return PIRRT_OK;
}

// append phase timeline (DevCtl::app_ns, accumulated since create; valid
// after a synchronous append): 12 entries
extern "C" int pirrt_debug_append_phases(const pirrt_ctx* c, unsigned long long* out, int n) {
    if (!c || !out || n < 12) return fail(PIRRT_E_INVAL, "debug_append_phases: bad arguments");
    std::memcpy(out, c->ctl_host->app_ns, 12 * sizeof(unsigned long long));
    return PIRRT_OK;
}

// debug: the incremental Improve's bookkeeping in DevCtl (synchronous read):
// out[0..11] = imp_count, app_pre_k, pre_count[0], pre_count[1], c_buf, c_n,
// L_imp, n_imp, gc_count[0], gc_count[1], imp_full, dirty_count[c_buf];
// list (nullable): task list slot (imp_count + 1) & 1, up to cap entries
extern "C" int pirrt_debug_inc(const pirrt_ctx* c, long long* out, int32_t* list, int64_t cap) {
    if (!c || !out) return fail(PIRRT_E_INVAL, "debug_inc: bad arguments");
    CU(cudaStreamSynchronize(c->stream));
    DevCtl h;
    CU(cudaMemcpy(&h, c->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost));
    const long long v[12] = {h.imp_count, h.app_pre_k, h.pre_count[0], h.pre_count[1], h.c_buf, h.c_n,
                             h.L_imp, h.n_imp, h.gc_count[0], h.gc_count[1], h.imp_full,
                             h.dirty_count[h.c_buf & 1]};
    std::memcpy(out, v, sizeof v);
    if (list && cap > 0) {
        const int slot = (int)((h.imp_count + 1) & 1);
        const int64_t nl = std::min<int64_t>(cap, std::max(0, h.pre_count[slot]));
        if (nl) CU(cudaMemcpy(list, c->alist + (size_t)slot * c->g_cap, nl * sizeof(int), cudaMemcpyDeviceToHost));
    }
    return PIRRT_OK;
}

extern "C" int pirrt_debug_blist(const pirrt_ctx* c, int32_t* out, int64_t cap, int32_t* count) {
    if (!c || !out || !count) return fail(PIRRT_E_INVAL, "debug_blist: NULL");
    int rc;
    if ((rc = set_device(c))) return rc;
    if ((rc = complete_pending(const_cast<pirrt_ctx*>(c)))) return rc;
    *count = c->Bcount;
    if (cap < c->Bcount + 1) return fail(PIRRT_E_RANGE, "debug_blist: capacity");
    CU(cudaMemcpyAsync(out, c->Bq[c->Bsel], (size_t)(c->Bcount + 1) * sizeof(int),
                       cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return PIRRT_OK;
}
