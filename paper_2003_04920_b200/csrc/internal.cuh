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
constexpr int kThreads = 512;     // persistent-kernel block size
constexpr unsigned kFull = 0xffffffffu;

// validation error bits (append / set_policy)
enum : int {
    kErrRange = 1, kErrSelfLoop = 2, kErrCost = 4, kErrH = 8,
    kErrParent = 16, kErrPcMissing = 32, kErrGNew = 64, kErrRoot = 128
};

// Per-iteration counters of the exploit loop, double-buffered by iteration
// parity so that one phase can reset the other copy without a race.
struct IterCtl {
    unsigned long long dg_bits;   // atomicMax of Delta g (non-negative f64 bits)
    long long relax;              // relaxations this Improve
    long long visits;             // children visited this Evaluate
    int I_count;                  // |I|
    int oldB;                     // |B| before Evaluate
    int ptr_changed;              // some parent value changed in Improve
    int g_changed;                // some g bit changed in Evaluate
    int newB;                     // |B| after Evaluate
    int both;                     // |old B  n  new B|
    int pad[2];
};

// Device control block (one per context, cudaMalloc'ed, 8-byte aligned).
struct DevCtl {
    IterCtl it[2];
    int fcount[3];                // frontier sizes (3-rotation over levels)
    int vcount[3];                // "visited at this level" flags
    // exploit outputs
    int status;                   // 0 ok, PIRRT_E_NOCONV
    int iterations, evaluations, max_level, promising, stalled;
    double last_dg;
    long long relaxations, eval_visits, improve_set, children_index;
    unsigned long long t_compact, t_improve, t_evaluate;
    // append / set_policy
    int err;                      // bitmask of kErr*
    int nprom;                    // new promising vertices
    int sweeps;                   // local-relaxation sweeps
    int sweep_changed[2];
    int pad2;
};

// Everything the persistent exploit kernel touches.
struct ExploitArgs {
    // in-edge store: base CSR + delta CSR, rows by destination vertex
    const long long* __restrict__ boff;
    const int* __restrict__ bidx;
    const double* __restrict__ bcost;
    const long long* __restrict__ doff;
    const int* __restrict__ didx;
    const double* __restrict__ dcost;
    // vertex SoA + policy-edge cost pc (R9)
    double* g;
    const double* h;
    int* parent;
    double* pc;
    unsigned char* b;
    // workspace
    int* Ilist;                   // [n] improve set
    int* kcnt;                    // [n+1] children counts
    int* krank;                   // [n] rank of v among its parent's children
    int* koff;                    // [n+1] children offsets
    int* kids;                    // [n] children index
    int* front0;                  // [n] BFS frontier buffers
    int* front1;
    long long* bsum;              // [grid] block partial sums
    DevCtl* ctl;
    int n;
    int max_it;
    double eps;
    int prune_off;
};

// kernels launched by this host thread (diagnostics; abi.cu attributes the
// delta of each call to its context)
extern thread_local long long g_kernel_launches;

// ---- launchers (store.cu / exploit.cu) ----
cudaError_t launch_exploit(const ExploitArgs& a, int blocks, cudaStream_t s);
int exploit_blocks_per_sm();

struct AppendArgs {
    // committed store (read)
    const long long* boff; const int* bidx; const double* bcost;
    const long long* doff_old; const int* didx_old; const double* dcost_old;
    // new delta (write)
    long long* doff_new; int* didx_new; double* dcost_new;
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
    int n_old, n_new;
    long long base_edges;
    DevCtl* ctl;
    int grid_blocks;
};
cudaError_t launch_append(const AppendArgs& a, cudaStream_t s);

struct CompactArgs {
    const long long* boff; const int* bidx; const double* bcost;
    const long long* doff; const int* didx; const double* dcost;
    long long* boff_new; int* bidx_new; double* bcost_new;
    long long* cnt; long long* scan_tmp;
    int n;
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

cudaError_t launch_best_path(const int* parent, int n, int* path_rev, int* len_out,
                             cudaStream_t s);

// device-wide exclusive scan: out[0..L] with out[L] = total
cudaError_t scan_exclusive(const long long* in, long long* out, long long L,
                           long long* tmp, cudaStream_t s);
size_t scan_tmp_elems(long long L);

}  // namespace pirrt
