// internal.cuh -- shared declarations of the libpirrt CUDA implementation.
// Product code (no oracle includes).  Layout of device memory: DESIGN.md
// section 5.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "pirrt.h"

namespace pirrt {

constexpr int kRoot = 0;          // x_init
constexpr int kGoal = 1;          // x_goal
#ifndef PIRRT_THREADS
#define PIRRT_THREADS 512
#endif
constexpr int kThreads = PIRRT_THREADS;   // persistent-kernel block size
constexpr int kMaxGridBlocks = 8192;  // queue slack: claims beyond the last published slot
constexpr long long kMaxVertices = (1LL << 30) - (1LL << 14);
constexpr unsigned kFull = 0xffffffffu;

// validation error bits (append / set_policy)
enum : int {
    kErrRange = 1, kErrSelfLoop = 2, kErrCost = 4, kErrH = 8,
    kErrParent = 16, kErrPcMissing = 32, kErrGNew = 64, kErrRoot = 128,
    kErrDup = 256, kErrCycle = 512    // VALIDATE: duplicate (src,dst); parent cycle
};

// Per-iteration counters of the exploit loop, double-buffered by iteration
// parity so that one phase can reset the other copy without a race.
struct IterCtl {
    // Every counter that all blocks update (one atomic per block per phase or
    // level) or poll has its own 128-byte line: on a shared line ~300 blocks'
    // atomics and polls serialise at one L2 slice (4-5% of the bench step).
    alignas(128) unsigned long long dg_bits;   // atomicMax of Delta g (non-negative f64 bits)
    alignas(128) long long relax;              // relaxations this Improve
    alignas(128) int tasks;                    // |I|
    alignas(128) int ptr_changed;              // some parent value changed in Improve
    alignas(128) long long visits;             // children visited this Evaluate
    long long scanned;                         // out-row entries scanned this Evaluate
    int g_changed;                             // some g bit changed in Evaluate
    int both;                                  // |old B  n  new B|
    struct alignas(128) Level {                // rotating per-level slots
        int push;                              // expanded vertices of the level
        int vis;                               // "some child visited" at the level
    } lv[3];
    // work-queue Evaluate: queue slot 0 holds the root permanently; waiting
    // blocks poll qhead / qtail / qout while working blocks update qtail,
    // qout and bcnt
    alignas(128) int qhead;                    // slots claimed by blocks
    alignas(128) int qtail;                    // slots reserved by publishers
    alignas(128) int qout;                     // (children created - items expanded): -F0 = done
    alignas(128) int bcnt;                     // entries written to the new B list
    alignas(128) int l1cnt;                    // fused root levels: expanded children of the root
    // incremental Evaluate (one atomic per block each)
    alignas(128) int removed;                  // B-list members that left B
    int orphan;                                // a removed member had children: validate the list
    int maxd;                                  // levels of the equivalent full Evaluate
    long long work_visits;                     // children actually visited (the algorithmic
                                               // count, Sum over B u {root} of children, is `visits`)
    // incremental Improve: the task list's length, and the work actually
    // done (relax / tasks are the full Improve's counts, identical in both forms)
    alignas(128) int acount;
    alignas(128) long long relax_work;
    alignas(128) int tasks_work;
    alignas(128) int wide_next;                // improve_wide_kernel: next unclaimed task
};

// One Improve result in sharded mode (all-gathered between ranks).
struct ShardRec {
    int v, parent, changed, pad;
    double pc, delta;
};

// Device control block (one per context, cudaMalloc'ed, 8-byte aligned).
// Everything up to `err` is zeroed before each exploit.
struct DevCtl {
    IterCtl it[2];
    // exploit outputs
    int status;                   // 0 ok, PIRRT_E_NOCONV
    int iterations, evaluations, max_level, promising, stalled;
    int Bsel_out, Bcount_out;     // B list after the exploit
    int old_Bcount_out, pending_out;  // pending leave_B (sharded host loop)
    int shard_stop;               // sharded: 0 continue, 1 converged, 2 stalled/aborted,
                                  // 3 iteration cap (E_NOCONV), 4 record overflow (re-gather)
    unsigned ev_out;              // sharded: id of the next Evaluate (device-resident loop state
                                  // with Bsel_out, Bcount_out, old_Bcount_out, pending_out)
    int shard_over, shard_over_it;    // record overflow: largest count, iteration
    int barriers;
    int abort_at;                 // watchdog: barrier index at which all threads stop
    double last_dg;
    long long relaxations, eval_visits, improve_set, eval_scanned;
    long long work_visits;        // children actually visited (incremental Evaluates visit fewer)
    int full_evals, inc_evals;    // Evaluates run in full / incremental form
    long long relax_work, improve_work;   // relaxations / vertices actually scanned by Improve
    int full_imps, inc_imps;      // Improves run in full / incremental form
    unsigned long long t_improve, t_evaluate;
    // phase timeline (lead thread, %globaltimer ns between grid barriers;
    // pirrt_debug_phases): 0 Improve discovery, 1 Improve scan, 2 incremental
    // Evaluate E2 (walk-ups + traversal), 3 its E3 (bookkeeping + next task
    // list), 4 its validation fixpoint, 5 full Evaluates, 6 incremental
    // Evaluates (count), 7 in-kernel Improves (count)
    unsigned long long phase_ns[8];
    unsigned long long dbg_work_ns;   // PIRRT_DEBUG level trace
    unsigned long long dbg[8];        // PIRRT_LEVEL_TRACE work-queue counters
    unsigned long long dbg_imp[6];    // PIRRT_LEVEL_TRACE Improve timeline
    unsigned long long dbg_lv[32][6]; // PIRRT_LEVEL_TRACE per level: ~min start, max start,
                                      // max work end, max flush end, lead exit, frontier
    // wide-Improve hand-off: the persistent kernel stopped before the Improve
    // of iteration handoff_it (|I| >= wide_tasks); the host runs
    // improve_wide_kernel for it and resumes the loop after that Improve
    int handoff, handoff_it;
    unsigned long long t_wide0, t_wide1;   // ~min start / max end of the wide Improve
    // append / set_policy (the words every block may update on their own lines)
    // (err, sweeps, nprom: one memset before each append)
    alignas(128) int err;         // bitmask of kErr*
    int sweeps;                   // local-relaxation passes (1: the dataflow pass)
    int nprom;                    // new promising vertices (one atomic per warp that has some)
    // append phase timeline (lead thread, %globaltimer ns, accumulated over
    // appends; pirrt_debug_append_phases): 0 validation, 1 old row lengths,
    // 2 histogram, 3 scan partials, 4 row offsets, 5 old-delta copy, 6
    // scatter + init, 7 local relaxation, 8 promising test, 9 appends;
    // 10 block 0's own time in the P4 chunk copy, 11 the prebuild (P8)
    alignas(128) unsigned long long app_ns[12];
    // ---- persistent across exploits (zeroed only at create): the state
    // the incremental Evaluate needs ("incremental
    // Evaluate").  Written by the lead thread after an Evaluate's last grid
    // barrier (or by the host between calls), read at the next Evaluate.
    alignas(128) int dirty_count[2];  // Improve commits pending for Evaluate ev, slot ev & 1
    alignas(128) int need_full;       // next Evaluate must be full (create, set_policy, given policy)
    int n_eval;                       // |V| at the last Evaluate (ids >= n_eval: appended since)
    int Bc_eval;                      // B-list length after the last Evaluate (later slots: appends)
    int holes;                        // -1 slots in the current B list (removed members)
    double thr_prev;                  // thr of the last Evaluate
    // incremental Improve (same rules): gc_count[k & 1] = vertices whose g
    // an Evaluate changed after Improve k (list gcl + (k & 1) * dcap)
    alignas(128) int gc_count[2];
    alignas(128) int imp_full;        // next Improve must be full (create, set_policy, full Evaluate)
    unsigned imp_count;               // Improves so far (k of the last one)
    int L_imp;                        // B-list length at the last Improve
    int n_imp;                        // |V| at the last Improve
    int c_buf, c_n;                   // its commits: dirty list c_buf, entries [0, c_n)
    // task list of Improve k prebuilt by the incremental Evaluate before it
    // (slot k & 1; alist + (k & 1) * acap): entries and the full Improve's
    // counters over I (Sum of in-degrees, |I|)
    alignas(128) int pre_count[2];
    alignas(128) long long pre_relax[2];
    alignas(128) int pre_tasks[2];
    // deferred BE-RRT# steps (pirrt_step_async): the current B list as the
    // last exploit kernel left it (selector, length) and the id of the next
    // Evaluate -- the state the host mirrors in pirrt_ctx after a synchronous
    // call, kept here so that a step enqueued behind another one can read it
    // without a host round trip.  Written by every exploit kernel (lead,
    // loop_state_out), read by the next step's append and exploit kernels.
    alignas(128) int dev_Bsel;
    int dev_Bcount;
    unsigned dev_ev;
    // the append prebuilt the task list (and counters) of Improve app_pre_k
    // (0: none), slot app_pre_k & 1 of alist / pre_count / pre_relax / pre_tasks
    unsigned app_pre_k;
};
constexpr unsigned kPrePoison = 0x80000000u;   // app_pre_k | this: epoch without a prebuilt list

// Everything the persistent exploit kernel touches.
struct ExploitArgs {
    // in-edge store (rows by destination): base CSR + delta CSR -- Improve
    const long long* __restrict__ boff;
    const int* __restrict__ bidx;
    const double* __restrict__ bcost;
    const long long* __restrict__ doff;
    const int* __restrict__ didx;
    const double* __restrict__ dcost;
    // out-edge index (rows by source, ids only): base + delta -- Evaluate
    const long long* __restrict__ oboff;
    const int* __restrict__ obidx;
    const long long* __restrict__ odoff;
    const int* __restrict__ odidx;
    // vertex SoA + policy-edge cost pc (R9)
    double* g;
    const double* h;
    int* parent;
    double* pc;
    unsigned char* b;
    unsigned* stamp;              // 2e: visited in Evaluate e; 2e+1: expanded in e
    unsigned* pstamp;             // e: (parent, pc) committed by an Improve since Evaluate e-1
    int2* ccd;                    // per vertex {children in the policy tree, depth at last visit}
    int* dirty;                   // Improve commits awaiting Evaluate e: dirty + (e & 1) * dcap
    int* gcl;                     // g changed by the Evaluate after Improve k: gcl + (k & 1) * dcap
    int dcap;                     // capacity of each dirty / gcl buffer
    unsigned* istamp;             // k: the incremental Improve k has v in its task list
    int* alist;                   // that task list: Improve k's at alist + (k & 1) * acap
    int acap;
    int inc_max;                  // incremental Evaluate when its start items <= this (0: never)
    int inc_imp;                  // incremental Improve: 0 never, 1 when its sources are small
                                  // next to |I| (default), 2 whenever valid (PIRRT_INC_IMPROVE)
    int inc_validate;             // test hook: always run the incremental list validation
    // work-queue Evaluate: item of queue slot i (qv[i] == -1: not yet published)
    int* qv;
    double* qg;
    int* qdepth;
    // B lists (entry 0 = root, B = [1, 1 + count)); Bq[Bsel] is current
    int* Bq0;
    int* Bq1;
    int Bsel;
    int Bcount;
    int old_Bcount;               // previous list still awaiting leave_B (sharded loop)
    int pending;
    unsigned ev_base;             // id of this exploit's first Evaluate
    int shard_rank, shard_n;      // sharded Improve: owned vertices v % shard_n == shard_rank
    ShardRec* rec_out;            // sharded Improve records
    int* rec_count;
    int shard_dev;                // sharded loop: the loop state lives in DevCtl (Bsel_out,
                                  // Bcount_out, old_Bcount_out, pending_out, ev_out) and a
                                  // kernel of an iteration enqueued after the stop returns at once
    int shard_K;                  // records per rank in the gathered buffer (stride K + 1:
                                  // slot 0 of each rank's block holds its count)
    int shard_finish;             // only finish the last Evaluate's leave_B (after E_NOCONV)
    DevCtl* ctl;
    int n;
    int max_it;
    double eps;
    int prune_off;
    unsigned long long watchdog_ns;   // abort the loop after this long (diagnostic guard)
    int wq_keep;                      // work-queue Evaluate: items a block keeps per local level
    int wq_tail;                      // level-synchronous: hand a shrinking frontier of at most
                                      // this many items to the work queue (0: never)
    int wq_wide;                      // ... and any frontier of at least this many (0: never)
    int debug;                        // PIRRT_DEBUG: device diagnostics
    // goal set G (R4): sorted ascending ids, contains x_goal; ids >= n inactive
    const int* goals;
    int n_goals;
    int parent_form;                  // PIRRT_F_PARENT_FORM: P:263 literal test (NEXT-4)
    int neighbours;                   // PIRRT_F_NEIGHBOURS (and not PRUNE_OFF): I = B u
                                      // N+(B u {root}) u G (R16, NEXT-4)
    int wide_tasks;                   // hand an Improve with |I| >= this to improve_wide_kernel (0: never)
    int wide_lpv;                     // its lanes per vertex (16 or 32, by the mean degree)
    int num_sms;                      // the device's SMs (a grid of at most one block per SM
                                      // runs the one-block-per-SM instantiation)
    int it_base;                      // first PI iteration of this launch (1 = a fresh exploit)
    int resume;                       // 1: iteration it_base's Improve already ran (wide kernel)
    // children index for large Evaluates (build_children): |B| >= kids_min (0: never)
    int kids_min;
    int* coff;                        // [n]: after the build row(p) = [p ? coff[p-1] : 0, coff[p])
    int* kids;                        // [n]
    int* kids_bsum;                   // [grid blocks] scan partials
    int kids_variant;                 // launch the instantiation that can use the index
    // deferred step (pirrt_step_async): 0 off; 1 the B list / Evaluate id are
    // the host's (Bsel, Bcount, ev_base); 2 they are DevCtl's dev_* (a step
    // enqueued behind another).  In both the step's append has pushed nprom
    // new members after them, and the kernel returns at once (Alg. 3 guard,
    // R10) when nprom == 0 or the append was rejected (err != 0)
    int step_mode;
};

// ---- goal set (reading R4, goal-set form) ----
// v in G?  G is sorted; the single-goal case is the paper's x_goal.
__device__ __forceinline__ bool is_goal(const int* goals, int n_goals, int v) {
    if (n_goals == 1) return v == kGoal;
    int lo = 0, hi = n_goals - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(&goals[mid]) < v) lo = mid + 1; else hi = mid;
    }
    return __ldg(&goals[lo]) == v;
}

// Goal cost min over the goals among the first n_exist vertices of g (the
// promising threshold, P:263 with R3/R4).  Warp-collective: every lane of a
// converged warp calls it and receives the value.
__device__ __forceinline__ double warp_goal_cost(const double* g, const int* goals, int n_goals,
                                                 int n_exist) {
    if (n_goals == 1) return *(volatile const double*)&g[kGoal];
    double m = INFINITY;
    for (int i = (threadIdx.x & 31); i < n_goals; i += 32) {
        const int t = __ldg(&goals[i]);
        if (t < n_exist) m = fmin(m, *(volatile const double*)&g[t]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmin(m, __shfl_xor_sync(kFull, m, o));
    return m;
}

// kernels launched by this host thread (diagnostics; abi.cu attributes the
// delta of each call to its context)
extern thread_local long long g_kernel_launches;

// L2 access-policy window (persisting) for the hot vertex slab; bytes == 0: none
struct L2Window {
    void* base = nullptr;
    size_t bytes = 0;
    float hit = 0.f;
};

// cudaLaunchKernelEx helper: cooperative launch + optional persisting window
cudaError_t launch_coop(const void* fn, int blocks, int threads, void** params,
                        const L2Window& w, cudaStream_t s);

// ---- launchers (store.cu / exploit.cu) ----
cudaError_t launch_exploit(const ExploitArgs& a, int blocks, const L2Window& w, cudaStream_t s);
cudaError_t launch_shard_improve(const ExploitArgs& a, int it, int blocks, cudaStream_t s);
cudaError_t launch_shard_evaluate(const ExploitArgs& a, int it, const ShardRec* recs, int nranks,
                                  int blocks, cudaStream_t s);
int exploit_blocks_per_sm();
// a3 Improve of iteration `it` as its own high-occupancy launch (large I)
cudaError_t launch_improve_wide(const ExploitArgs& a, int it, int num_sms, cudaStream_t s);
int shard_evaluate_blocks_per_sm();

struct AppendArgs {
    // committed store (read)
    const long long* boff; const int* bidx; const double* bcost;
    const long long* doff_old; const int* didx_old; const double* dcost_old;
    // new delta (write)
    long long* doff_new; int* didx_new; double* dcost_new;
    // out-edge index: committed base/delta (read) and new delta (write)
    const long long* oboff; const int* obidx;
    const long long* odoff_old; const int* odidx_old;
    long long* odoff_new; int* odidx_new;
    long long* oboff_w;
    long long* boff_w;            // writable base offsets (rows n_old+1..n_all filled)
    long long* cnt;               // [n_all+1] scratch counts / cursors
    long long* scan_tmp;          // scan partials
    // incoming batch (device)
    const double* h_in; const int* parent_in; const double* g_in;
    const int* src; const int* dst; const double* cost;
    long long m;                  // triples
    int undirected;
    int validate;
    // vertex SoA (write slots >= n_old only)
    double* g; double* h; int* parent; double* pc; unsigned char* b;
    int2* ccd;                    // child counts (parents of the new vertices gain one)
    int n_old, n_new;
    long long base_edges;
    long long obase_edges;
    int* Blist;                   // current B list; new promising vertices go to [1+Bcount+k]
    int Bcount;
    // P8: the next exploit's first Improve prebuilt (pre_ok: single GPU, no
    // PRUNE_OFF / NEIGHBOURS / VALIDATE / given policy, incremental Improve on)
    int pre_ok;
    int inc_max, inc_imp;
    unsigned* istamp; int* alist; int acap;
    const int* dirty; const int* gcl; int dcap;
    unsigned* rdone;              // local relaxation: rdone[v] == app_id once v is final
    unsigned app_id;              // this append's id (> every earlier one)
    int* chunk_in; int* chunk_out;   // scratch: first row of each old-delta copy chunk
                                     // (|delta| / kCopyChunk + 2 entries each)
    int dev_list;                 // 1: the list is Bq[ctl->dev_Bsel] of length ctl->dev_Bcount
    int* Bq0; int* Bq1;           //    (a deferred step behind another, pirrt_step_async)
    DevCtl* ctl;
    int grid_blocks;
    int per_sm;                   // k_append_fused blocks per SM (append_blocks_per_sm)
    const int* goals;             // goal set (R4); the promising threshold of the
    int n_goals;                  // new vertices is the goal cost before the batch
};
// one cooperative kernel for the whole append; bsum needs 2 * max_blocks entries
// child counts ccd[p].x += 1 for every parent p of [v0, v1)
cudaError_t launch_child_count(const int* parent, int v0, int v1, int2* ccd, cudaStream_t s);
cudaError_t launch_append_fused(const AppendArgs& a, long long* cnt1, long long* bsum,
                                int max_blocks, const L2Window& w, cudaStream_t s);
constexpr int kAppendMaxBlocks = 2048;
constexpr int kAppendCopyChunk = 2048;   // old-delta entries per append copy chunk (16 KB of smem destinations)
int append_blocks_per_sm();

// fold a delta CSR into its base CSR (cost arrays may be NULL: out-index)
struct CompactArgs {
    const long long* boff; const int* bidx; const double* bcost;
    const long long* doff; const int* didx; const double* dcost;
    long long* boff_new; int* bidx_new; double* bcost_new;
    long long* cnt; long long* scan_tmp;
    int* markA; int* markB;       // scratch: first row of each kAppendCopyChunk-entry chunk of
                                  // the base / the delta (Eb / C + 2, Ed / C + 2 entries)
    long long Eb, Ed;             // entries of the base / the delta
    int n;
    int own_n, own_r;             // partitioned store (sharded, P > 1): keep only the rows of
                                  // v with v % own_n == own_r (own_n = 0: every row)
};
cudaError_t launch_compact(const CompactArgs& a, cudaStream_t s);

struct PolicyArgs {
    const long long* boff; const int* bidx; const double* bcost;
    const long long* doff; const int* didx; const double* dcost;
    const int* parent_in; const double* g_in; const unsigned char* b_in;
    int* parent; double* g; double* pc; unsigned char* b;
    int n; DevCtl* ctl;
};
cudaError_t launch_set_policy(const PolicyArgs& a, cudaStream_t s);

// VALIDATE: a staged batch whose edges duplicate a
// stored (src,dst) pair or each other -> kErrDup (run after the append merged
// the batch into the new delta, before the host commits); a parent array with
// a cycle -> kErrCycle (integer pointer jumping; tmp holds 2 n ints).
cudaError_t launch_dup_check(const AppendArgs& a, cudaStream_t s);
cudaError_t launch_cycle_check(const int* parent, int n, int* tmp, DevCtl* ctl, cudaStream_t s);

// B list = {v : b[v] == 1} in ascending order into list[1..]; count -> *count_out
cudaError_t launch_rebuild_blist(const unsigned char* b, int n, int* list, int* count_out,
                                 long long* cnt, long long* scan_tmp, cudaStream_t s);

// best goal (lowest g, lowest id on ties) and its branch; see k_best_path
// device-side Extend (extend.cu)
struct ExtendArgs {
    const double* pts;            // all points [n_old + n_new][d] (new ones staged)
    int n_old, n_new, d;
    int m, brute;                 // grid cells per axis (cell side >= every radius); brute: no grid
    long long ncell;
    int* cell;                    // [n_all] cell id per point
    long long* ccnt;              // [ncell + 1] counts / cursors
    long long* cstart;            // [ncell + 1] exclusive scan
    int* cpts;                    // [n_all] point ids by cell
    long long* scan_tmp;
    const double* R;              // [n_new] r(i + 1), computed on the host
    const double* boxes;          // [n_boxes][2][d]
    int n_boxes;
    const double* x_goal;         // [d]
    double* h_new;                // [n_new] out
    long long* ecnt;              // [n_new + 1] edges per new vertex
    long long* eoff;              // [n_new + 1] their offsets (eoff[n_new] = total)
    int* src; int* dst; double* cost;   // [total] COO out (undirected: j -> i stored once)
    int hcap;                     // hit-cache slots per new vertex (0: none)
    int* hj; double* hd;          // [n_new][hcap] the count pass's hits, in output order
};
cudaError_t launch_extend_grid(const ExtendArgs& a, cudaStream_t s);   // grid, h, counts, offsets
cudaError_t launch_extend_edges(const ExtendArgs& a, cudaStream_t s);  // the triples

cudaError_t launch_best_path(const int* parent, const double* g, int n, const int* goals,
                             int n_goals, int* out, cudaStream_t s, int* head = nullptr, int head_n = 0);

// device-wide exclusive scan: out[0..L] with out[L] = total
cudaError_t scan_exclusive(const long long* in, long long* out, long long L,
                           long long* tmp, cudaStream_t s);
size_t scan_tmp_elems(long long L);

}  // namespace pirrt
