/*
 * pirrt.h -- C ABI of the B200-native PI-RRT# exploitation library
 * (libpirrt.so, paper_2003_04920_b200/lib/).
 *
 * Method: the exploitation phase of PI-RRT# / BE-RRT#, arXiv 2003.04920
 * ("PAPER.md" below): policy iteration on the random geometric graph
 * G = (V, E) with edge costs c : E -> R+, a root x_init, a goal x_goal and an
 * admissible heuristic h : V -> R+ (problem statement PAPER.md:168-178),
 * iterated to a fixed point after each single or batched graph extension
 * (Alg. 2; Alg. 3).  Ambiguities of the
 * listing are resolved by the readings R1-R14 of DESIGN.md section 3.
 *
 * Conventions for every call:
 *   - Vertex ids are dense int32 0..n-1; -1 means "no vertex".  Vertex 0 is
 *     x_init (g = 0) and vertex 1 is x_goal (g = +inf); both exist after
 *     pirrt_create (Alg. 1 line 1).
 *   - All floating point is IEEE binary64.  Costs and h must be finite and
 *     >= 0; -0.0 is stored as +0.0 (R12).
 *   - Ownership: the caller owns every input and output array; the library
 *     copies inputs before returning and owns all device memory.  Unless the
 *     call's flags contain PIRRT_F_DEVICE_PTRS, pointers are host pointers
 *     (pinned host memory makes the H2D copies asynchronous DMA).  Every call
 *     except pirrt_exploit_async and pirrt_step_async is synchronous with
 *     respect to the context's stream: when it returns, results are visible
 *     to the caller.
 *   - Errors: every call returns PIRRT_OK (0) or a negative PIRRT_E_* code and
 *     sets a thread-local message readable with pirrt_last_error().  On error
 *     the context state (graph, policy, costs, promising set) is unchanged,
 *     except after PIRRT_E_CUDA, which leaves the context unusable.
 *   - A context is single-threaded; separate contexts are independent.
 */
#ifndef PIRRT_H
#define PIRRT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pirrt_ctx pirrt_ctx;  /* opaque; owned by the library */
typedef int32_t pirrt_vid;           /* vertex id, dense; -1 = none  */

enum {
    PIRRT_OK = 0,
    PIRRT_E_INVAL = -1,   /* bad argument: NaN/inf/negative cost or h, self-loop, NULL */
    PIRRT_E_RANGE = -2,   /* vertex id out of range, or output capacity too small   */
    PIRRT_E_NOMEM = -3,   /* device or pinned host allocation failed                 */
    PIRRT_E_CUDA = -4,    /* CUDA runtime error (context unusable afterwards)        */
    PIRRT_E_NCCL = -5,    /* multi-GPU communication error                           */
    PIRRT_E_NOCONV = -6,  /* exploit exceeded max_iterations (R11)       */
    PIRRT_E_STATE = -7,   /* call out of order / unsupported configuration           */
    PIRRT_E_CORRUPT = -8  /* parent cycle or missing policy edge detected            */
};

enum {
    /* config flags */
    PIRRT_F_PRUNE_OFF = 1u,        /* I = V \ {root}, thr = +inf: classical PI (test/cold mode) */
    PIRRT_F_VALIDATE = 2u,         /* extra checks on append / set_policy: duplicate (src,dst)
                                      pairs, in the batch or against the stored graph ->
                                      E_INVAL; a parent cycle in a given
                                      policy (set_policy, or parent_new) -> E_CORRUPT (S:179,
                                      S:237); g_new == g(parent) + c consistency -> E_INVAL    */
    PIRRT_F_SHARDED = 16u,         /* use the sharded (NCCL) exploit loop even with nranks == 1 */
    PIRRT_F_PARENT_FORM = 32u,     /* Evaluate's promising test on the parent v, h(v)+g(v) < thr,
                                      as printed at PAPER.md:263 (variant of reading R2)         */
    PIRRT_F_NEIGHBOURS = 64u,      /* "promising vertices and their neighbors are re-evaluated"
                                      (NEXT-4 variant, reading R16): the
                                      Improve set is I = B u N+(B u {x_init}) u G \ {x_init},
                                      N+(X) = heads of the edges leaving X.  Not with
                                      PIRRT_F_SHARDED / nranks > 1 (E_INVAL)                  */
    PIRRT_F_LOCAL_GROUP = 128u,    /* this context is rank `rank` of an in-process group of
                                      `nranks` contexts (no NCCL; e.g. P ranks emulated on one
                                      GPU for parity tests): the sharded exploit runs through
                                      pirrt_group_exploit; pirrt_exploit returns E_STATE        */
    /* append flags */
    PIRRT_F_EDGES_UNDIRECTED = 4u, /* each (src,dst,cost) is stored in both directions         */
    PIRRT_F_DEVICE_PTRS = 8u       /* input arrays are device pointers (e.g. torch CUDA tensors)*/
};

typedef struct {
    int64_t vertex_capacity;  /* initial reservation (hint; grows up to 2^30 - 2^14 vertices,
                                 beyond which append returns PIRRT_E_RANGE)                 */
    int64_t edge_capacity;    /* initial directed-edge reservation (hint)                    */
    double h_root;            /* h(x_init); default 0                                       */
    double h_goal;            /* h(x_goal); default 0                                       */
    double epsilon;           /* stop when Delta g <= epsilon (R5); default 0               */
    int32_t max_iterations;   /* Improve cap per exploit; 0 -> 10 |V| (R11)                  */
    uint32_t flags;           /* PIRRT_F_PRUNE_OFF | PIRRT_F_VALIDATE | PIRRT_F_PARENT_FORM  */
    int32_t device;           /* CUDA device ordinal                                        */
    void* stream;             /* cudaStream_t to run on (e.g. a torch stream; the legacy
                                 default stream is cudaStreamLegacy, (void*)1); NULL: the
                                 context creates its own non-blocking stream, which does
                                 not synchronise with the caller's default stream          */
    int32_t grid_blocks;      /* persistent-kernel grid; 0 = auto (SMs x occupancy)          */
    int32_t nranks;           /* multi-GPU SPMD: ranks (1 = single GPU), one process per GPU */
    int32_t rank;             /* this process's rank                                        */
    const void* nccl_unique_id; /* ncclUniqueId (128 B, pirrt_nccl_unique_id on one rank,
                                   broadcast by the caller) when nranks > 1; NULL otherwise  */
    /* Goal set (reading R4, goal-set form; the paper's case is the single
     * x_goal): G = {x_goal} u goals[0..n_goals).  Ids must be >= 1 and may name
     * vertices appended later (a goal joins G when its vertex exists).  The
     * promising threshold is min over existing goals of g (P:263 with R3);
     * every existing goal is in the Improve set; best_path follows the best
     * goal (lowest g, lowest id on ties).  New vertices of a batch are
     * promising against the goal cost before that batch.  Copied at create;
     * NULL/0 = {x_goal}.  E_RANGE: an id < 1. */
    const pirrt_vid* goals;
    int32_t n_goals;
    /* Ids of x_init and x_goal.  The two vertices are the
     * first created (Alg. 1 line 1) and ids are dense in
     * creation order, so the only valid values are root = 0, goal = 1
     * (reading R15); anything else -> E_INVAL.
     * pirrt_config_init sets them. */
    pirrt_vid root;
    pirrt_vid goal;
} pirrt_config;

typedef struct {
    int32_t iterations;      /* Improve calls (Alg. 2)                          */
    int32_t evaluations;     /* Evaluate calls                                           */
    double last_delta_g;     /* Delta g of the final Improve                             */
    int64_t relaxations;     /* sum over Improves of sum_{v in I} indeg(v)               */
    int64_t eval_visits;     /* children visited, summed over Evaluates                  */
    int32_t max_level;       /* deepest Evaluate BFS level reached (root = 0)            */
    int32_t promising;       /* |B| on return                                            */
    int32_t stalled;         /* 1 if the R13 stall guard ended the loop                  */
    int32_t grid_blocks;     /* persistent grid used                                     */
    float device_ms;         /* exploit kernel time, CUDA events on the context stream   */
    float improve_ms;        /* time inside Improve phases (device %globaltimer)         */
    float evaluate_ms;       /* time inside Evaluate phases (device %globaltimer)        */
    int32_t barriers;        /* grid-wide barriers executed                              */
    int64_t improve_set;     /* sum over Improves of |I| (vertices examined)             */
    int64_t eval_scanned;    /* out-edge entries scanned by Evaluate for children        */
    int64_t eval_work;       /* children actually visited (an incremental Evaluate visits
                                only the changed subtrees; eval_visits is the count of the
                                paper's full traversal, identical in both forms)          */
    int32_t full_evaluations;   /* Evaluates run as the full traversal ...               */
    int32_t inc_evaluations;    /* ... and in the incremental form  */
    int64_t relax_work;      /* relaxations actually made (an incremental Improve scans only
                                the rows whose result can change; `relaxations` is the
                                paper's full Improve count, identical in both forms)      */
    int64_t improve_work;    /* vertices actually scanned (`improve_set` = sum of |I|)    */
    int32_t inc_improves;    /* Improves run in the incremental form                     */
    int32_t pad_;
} pirrt_exploit_stats;

/* Fill *cfg with the defaults listed above. */
void pirrt_config_init(pirrt_config* cfg);

/* Create a context on cfg->device: V = {x_init (g=0, h=h_root), x_goal
 * (g=+inf, h=h_goal)}, E = {}, B = {} (Alg. 1 line 1). */
int pirrt_create(const pirrt_config* cfg, pirrt_ctx** out);
int pirrt_destroy(pirrt_ctx* ctx);

/* Append one extension batch (Alg. 3 lines 6-8; data flow
 * each edge is sent to the device exactly once).
 *   n_new       new vertices; they get ids [n, n + n_new) in caller order.
 *   h_new       [n_new] heuristic of the new vertices.
 *   parent_new, g_new  [n_new] the new vertices' policy and cost-to-come, or
 *               both NULL: the library then performs Extend's local
 *               relaxation (reading R14): in increasing id
 *               order g(v) = min over edges (u -> v), u < v, of g(u) + c(u,v),
 *               lowest u on ties; +inf and parent -1 if there is none.  When
 *               given, the edge (parent_new[i] -> new vertex i) must be in the
 *               batch (its cost becomes the policy-edge cost).
 *   n_edges, src, dst, cost  [n_edges] COO edges; (src, dst, c) means "dst
 *               may take src as parent at cost c" = c(n, v) with n = src,
 *               v = dst.  Endpoints may be old or new vertices.
 *               With PIRRT_F_EDGES_UNDIRECTED each triple is stored both ways.
 *   n_new_promising (out, nullable)  number of new vertices with
 *               g + h < g(x_goal), i.e. |B'| - |B| for the
 *               Alg. 3 replan guard (reading R10).
 * Errors: E_RANGE endpoint >= n + n_new or < 0; E_INVAL non-finite/negative
 * cost or h, self-loop, only one of parent_new/g_new given, missing parent
 * edge; with PIRRT_F_VALIDATE (config or call flags) also a duplicate
 * (src,dst) pair in the batch or against the stored graph (E_INVAL, SPEC
 * S:128), a g_new != g(parent) + c (E_INVAL) and a parent cycle in
 * parent_new (E_CORRUPT).  Without VALIDATE duplicates are accepted and
 * stored: Improve then takes the cheapest of them (lowest id on ties, R6) and
 * Evaluate visits a child reached through several entries once. */
int pirrt_graph_append_batch(pirrt_ctx* ctx, int32_t n_new, const double* h_new,
                             const pirrt_vid* parent_new, const double* g_new,
                             int64_t n_edges, const pirrt_vid* src, const pirrt_vid* dst,
                             const double* cost, uint32_t flags, int32_t* n_new_promising);

/* Replan (Alg. 2) to a fixed point, entirely on the device:
 * loop { Improve over I = B u {x_goal} \ {x_init};
 *        if Delta g <= epsilon break; Evaluate }.
 * Improve: each v in I takes the lowest-id argmin over its in-edges of
 * g(u) + c(u,v) if strictly below g(v); g is not written (Jacobi).
 * Evaluate: thr = g(x_goal) snapshot; truncated BFS of the policy tree from
 * x_init, g(n) = g(parent) + c(parent, n), expand and mark promising iff
 * g(n) + h(n) < thr.  stats (nullable) receives counters and timings.
 * Errors: E_NOCONV after max_iterations Improves (state as left). */
int pirrt_exploit(pirrt_ctx* ctx, pirrt_exploit_stats* stats);

/* Asynchronous exploit (PAPER.md:565-574:
 * "asynchronous policy iteration exploitation concurrent with exploration").
 * pirrt_exploit_async enqueues the same exploit on the context's stream and
 * returns at once, so the caller's exploration (sampling, collision checks,
 * building the next batch) runs while the GPU exploits.  pirrt_exploit_wait
 * completes it and returns its stats and result code (as pirrt_exploit).
 * Any other call on the context first completes a pending exploit (its
 * result is kept for the next pirrt_exploit_wait) -- except that
 * pirrt_graph_append_batch with host inputs first starts their H2D copies
 * on a side stream, overlapping the running exploit, and only then waits.
 * Results are identical to pirrt_exploit; Alg. 3's order (append after the
 * previous Replan) is unchanged.  Sharded contexts run the exploit inside
 * pirrt_exploit_async.  E_STATE: wait without a started exploit. */
int pirrt_exploit_async(pirrt_ctx* ctx);
int pirrt_exploit_wait(pirrt_ctx* ctx, pirrt_exploit_stats* stats);

/* Deferred BE-RRT# step (PAPER.md:565-574,
 * "asynchronous policy iteration exploitation concurrent with exploration").
 * pirrt_step_async enqueues one whole iteration of Alg. 3
 * and returns without waiting for the device:
 *   append the batch (as pirrt_graph_append_batch with parent_new = g_new =
 *   NULL: Extend's local relaxation, R14; flags may hold
 *   PIRRT_F_EDGES_UNDIRECTED and PIRRT_F_DEVICE_PTRS), then Replan
 *   (pirrt_exploit) iff the batch brought a new promising vertex (Alg. 3
 *   line 9, R10 -- decided on the device), then the best-path
 *   read-out (pirrt_best_path).
 * Up to two steps may be outstanding: the H2D of step k+1's inputs overlaps
 * step k's exploit, and the host never sits between the kernels of a step.
 * Host inputs are read asynchronously: they must stay valid and unchanged
 * until this step's pirrt_step_wait returns (pinned memory makes the copy a
 * DMA).  pirrt_step_wait completes the oldest outstanding step and returns
 * its result in *out (nullable) and its best path root..goal in
 * path_out[0..out->path_len) (nullable; E_RANGE if cap is smaller, the rest
 * of *out is still filled).  Results are identical to the synchronous calls.
 * While a step is outstanding every other call on the context returns
 * E_STATE, except pirrt_step_wait, pirrt_steps_outstanding, the counters
 * (pirrt_num_vertices / num_edges / kernel_launches: the vertices and edges
 * of every enqueued step are counted) and pirrt_destroy (which waits).
 * Errors of step_async: E_INVAL as the append's argument checks, and
 * PIRRT_F_VALIDATE (use the synchronous append); E_STATE two steps already
 * outstanding, a sharded context, or a context with a world.  A batch the
 * device rejects (an id out of range, a bad cost or h: the append's E_RANGE /
 * E_INVAL) is reported by its pirrt_step_wait and leaves the context
 * unusable; E_NOCONV as pirrt_exploit. */
typedef struct {
    int32_t n_new_promising;   /* as pirrt_graph_append_batch                          */
    int32_t replanned;         /* 1: the exploit ran (n_new_promising > 0)              */
    int64_t path_len;          /* best path (0: no goal reached)                        */
    double path_cost;          /* its g (+inf: none)                                    */
    pirrt_vid goal;            /* its goal (-1: none)                                   */
    int32_t pad_;
    pirrt_exploit_stats stats; /* the exploit's (zero if !replanned, except promising) */
} pirrt_step_result;

int pirrt_step_async(pirrt_ctx* ctx, int32_t n_new, const double* h_new, int64_t n_edges,
                     const pirrt_vid* src, const pirrt_vid* dst, const double* cost,
                     uint32_t flags);
int pirrt_step_wait(pirrt_ctx* ctx, pirrt_step_result* out, pirrt_vid* path_out, int64_t cap);
int pirrt_steps_outstanding(const pirrt_ctx* ctx);   /* steps enqueued and not yet waited */

/* Read-out of the vertex state the paper's GPU version keeps per vertex
 * (the cost-to-come g, the parent pointer of the policy
 * T(v) = (parent(v), v) of PAPER.md:208-212, and the promising flag b of
 * B), plus pc(v) = c(parent(v), v) (reading R9).  Host
 * outputs of n = pirrt_num_vertices elements, indexed by vertex id; parent -1
 * and g +inf for a vertex not reached.  A pending asynchronous exploit is
 * completed first.  E_INVAL NULL; E_RANGE cap < n (nothing written). */
int pirrt_get_policy(const pirrt_ctx* ctx, pirrt_vid* parent_out, int64_t cap);
int pirrt_get_costs(const pirrt_ctx* ctx, double* g_out, int64_t cap);
int pirrt_get_promising(const pirrt_ctx* ctx, uint8_t* b_out, int64_t cap);
int pirrt_get_parent_costs(const pirrt_ctx* ctx, double* pc_out, int64_t cap);

/* Read-out of the stored graph (the CSR the Improve kernel reads, PAPER.md:
 * 296-307, 351-369), rows by destination: the in-edges (u -> v, c(u, v)) of
 * vertex v are src_out[off_out[v] .. off_out[v + 1]) with their costs in
 * cost_out, in storage order (unspecified; Improve's result does not depend
 * on it, R6).  off_out has n + 1 entries (cap_v >= n + 1), src_out/cost_out
 * pirrt_num_edges entries (cap_e).  For tests and diagnostics (a full copy of
 * the store; not for the per-batch path).  E_INVAL NULL; E_RANGE a capacity
 * too small (nothing written). */
int pirrt_get_in_edges(const pirrt_ctx* ctx, int64_t* off_out, int64_t cap_v, pirrt_vid* src_out,
                       double* cost_out, int64_t cap_e);

/* Policy-tree extraction (Alg. 1 lines 8-12): the branch
 * root..goal of the best goal (lowest g over the goal set, lowest id on ties;
 * reading R4) into path_out[0..len); *cost_out = its g, *goal_out = its id
 * (outputs nullable).  No goal reached: *len_out = 0, *cost_out = +inf,
 * *goal_out = -1.  E_RANGE if cap < path length (nothing written);
 * E_CORRUPT if the branch does not reach the root. */
int pirrt_best_path(const pirrt_ctx* ctx, pirrt_vid* path_out, int64_t cap,
                    int64_t* len_out, double* cost_out, pirrt_vid* goal_out);

/* Restore a policy snapshot (host arrays of length n): parent, g, and b
 * (nullable -> B = {}).  The policy-edge cost of v is re-read from the stored
 * edge (parent(v) -> v) (R9); E_INVAL if it is missing or the root is not
 * (parent -1, g 0). */
int pirrt_set_policy(pirrt_ctx* ctx, const pirrt_vid* parent, const double* g,
                     const uint8_t* b);

int64_t pirrt_num_vertices(const pirrt_ctx* ctx);
int64_t pirrt_num_edges(const pirrt_ctx* ctx);   /* directed edges stored */
/* Multi-GPU mode.  With nranks > 1 every rank makes
 * the same call sequence with the same arguments (SPMD); the graph and the
 * policy are replicated, Improve is split by vertex (v mod nranks == rank),
 * its records are all-gathered with NCCL once per PI iteration, and every
 * rank runs the identical Evaluate, so results are bit-identical to one GPU.
 * Stats: relaxations / improve_set count this rank's share.
 * Storage (nranks > 1, without PIRRT_F_VALIDATE): the in-edge rows a fold
 * moves into the base CSR are kept only for the vertices this rank owns, so
 * the Improve store shrinks to ~1/nranks per rank (the out-edge index,
 * 4 B per edge, and the vertex arrays stay replicated for the Evaluate);
 * pirrt_get_in_edges then returns this rank's rows plus the unfolded delta,
 * and pirrt_set_policy returns E_STATE (it needs every policy edge's cost).
 * pirrt_nccl_unique_id writes the 128-byte ncclUniqueId (call on one rank). */
int pirrt_nccl_unique_id(void* out, int64_t cap);

/* The sharded exploit of an in-process group (the same
 * kernels and loop as one process per GPU, with the record all-gather done as
 * device copies between the contexts' buffers): ctxs[i] is rank i of n, each
 * created with nranks = n, rank = i, PIRRT_F_LOCAL_GROUP, and fed the same
 * appends (SPMD).  stats (nullable) receives n entries.  The contexts may
 * share one device and one stream.  Errors as pirrt_exploit; E_STATE if the
 * contexts do not form such a group. */
int pirrt_group_exploit(pirrt_ctx* const* ctxs, int32_t n, pirrt_exploit_stats* stats);

/* Device-side Extend: the
 * graph-growth half of a BE-RRT# batch on the GPU, so that a batch crosses
 * PCIe as n_new sample points instead of ~2 x n_new x degree edge triples.
 *
 * pirrt_set_world: the configuration space [0,1]^d with n_boxes axis-aligned
 * obstacle boxes (boxes[b][0][k] = lower, boxes[b][1][k] = upper corner,
 * row-major [n_boxes][2][d]), x_init / x_goal (the points of vertices 0 and
 * 1) and the connection constant gamma.  Call once, before the first append
 * (E_STATE otherwise); afterwards the context grows only through
 * pirrt_extend_batch (a plain append returns E_STATE).
 *
 * pirrt_extend_batch: points [n_new][d] (host, or device with
 * PIRRT_F_DEVICE_PTRS; the caller samples them, e.g. uniformly outside the
 * boxes) become vertices [n, n + n_new) in order.  New vertex i connects to
 * every earlier j < i with |x_i - x_j| <= r(i + 1), r(m) = gamma (ln m /
 * m)^(1/d), whose segment misses every box (closed boxes, slab test); cost =
 * |x_i - x_j| (fp64, squared differences summed in coordinate order), both
 * directions; h(i) = |x_i - x_goal|.  The triples are built on the device
 * (uniform grid, one warp per new vertex) and appended as by
 * pirrt_graph_append_batch with PIRRT_F_EDGES_UNDIRECTED (local relaxation,
 * promising test; flags may add PIRRT_F_VALIDATE).  *n_edges_out (nullable)
 * = undirected pairs created.  Errors as the append; state unchanged.
 *
 * pirrt_get_points: the points of all n vertices ([n][d], host). */
int pirrt_set_world(pirrt_ctx* ctx, int32_t d, int32_t n_boxes, const double* boxes,
                    const double* x_init, const double* x_goal, double gamma);
int pirrt_extend_batch(pirrt_ctx* ctx, int32_t n_new, const double* points, uint32_t flags,
                       int32_t* n_new_promising, int64_t* n_edges_out);
int pirrt_get_points(const pirrt_ctx* ctx, double* points_out, int64_t cap);

/* Number of CUDA kernels this context has launched so far (diagnostics). */
int64_t pirrt_kernel_launches(const pirrt_ctx* ctx);
const char* pirrt_last_error(void);              /* thread-local; valid until the next call */

#ifdef __cplusplus
}
#endif
#endif /* PIRRT_H */
