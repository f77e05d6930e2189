// oracle.cpp -- plain, slow, serial CPU oracle of the PI-RRT# exploitation
// phase (arXiv 2003.04920).  TEST INFRASTRUCTURE: see oracle.h for who may
// call it.  It shares no code with the CUDA library.
//
// Every function cites the PAPER.md passage it follows (P:line) and the
// DESIGN.md reading (R#) used where the paper is silent or ambiguous.
// Data layout is the paper's CPU baseline: an adjacency list per vertex
// ("the format used for graph representation in the CPU
// benchmark implementation"), here holding IN-edges (reading R7).
//
// Pins (tests/test_oracle_pins.py): SPEC worked examples (Improve, Evaluate,
// Replan, path), PRUNE_OFF == scipy Dijkstra bit-exact, the promising-subgraph
// Bellman certificate, the unit lattice closed form, the straight-line bound,
// brute-force sequential local relaxation, invariants.  Parity pinned for
// every function here except the R2/R3/R4 choices themselves, which no
// printed paper value separates ("parity unpinned" for those readings; see
// DESIGN.md section 3).
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <utility>
#include <vector>

namespace {

const double kInf = std::numeric_limits<double>::infinity();
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

}  // namespace

struct orc_ctx {
    // SoA vertex properties, PAPER.md:296-307 (g, h, parent p, promising b),
    // plus pc = cost of the policy edge (parent(v), v) (reading R9).
    std::vector<double> g, h, pc;
    std::vector<int32_t> parent;
    std::vector<uint8_t> b;
    // in(v) = list of (u, c(u,v)): the edges Improve scans (R7).
    std::vector<std::vector<std::pair<int32_t, double>>> in;
    double epsilon;
    int32_t max_iterations;
    uint32_t flags;
    int64_t n_edges;
    // goal set G = {x_goal} u extra goal ids (reading R4, goal-set form),
    // sorted ascending; ids >= |V| are inactive until appended
    std::vector<int32_t> goals;
};

static const int32_t kRoot = 0;  // x_init
static const int32_t kGoal = 1;  // x_goal

extern "C" const char* orc_last_error(void) { return g_err.c_str(); }

// Does the parent array p[0..n) contain a cycle (the
// policy is a tree)?  Plain three-colour walk up the parent chains.
static bool has_parent_cycle(const std::vector<int32_t>& p) {
    const size_t n = p.size();
    std::vector<uint8_t> state(n, 0);   // 0 unseen, 1 on the current walk, 2 done
    std::vector<int32_t> walk;
    for (size_t s = 0; s < n; ++s) {
        walk.clear();
        int32_t v = (int32_t)s;
        while (v >= 0 && (size_t)v < n && state[v] == 0) {
            state[v] = 1;
            walk.push_back(v);
            v = p[v];
        }
        if (v >= 0 && (size_t)v < n && state[v] == 1) return true;   // came back onto this walk
        for (int32_t w : walk) state[w] = 2;
    }
    return false;
}

extern "C" orc_ctx* orc_create(double h_root, double h_goal, double epsilon,
                               int32_t max_iterations, uint32_t flags) {
    // Alg. 1 line 1: V <- {x_init, x_goal}, E <- {}, B <- {}.
    // g(x_init) = 0; g(x_goal) = +inf with no parent (reading R4).
    if (!(h_root >= 0.0) || !(h_goal >= 0.0) || std::isinf(h_root) ||
        std::isinf(h_goal) || !(epsilon >= 0.0) || max_iterations < 0) {
        g_err = "orc_create: invalid argument";
        return nullptr;
    }
    orc_ctx* c = new orc_ctx();
    c->g = {0.0, kInf};
    c->h = {h_root + 0.0, h_goal + 0.0};
    c->pc = {0.0, 0.0};
    c->parent = {-1, -1};
    c->b = {0, 0};
    c->in.resize(2);
    c->epsilon = epsilon;
    c->max_iterations = max_iterations;
    c->flags = flags;
    c->n_edges = 0;
    c->goals = {1};
    return c;
}

extern "C" void orc_destroy(orc_ctx* c) { delete c; }

extern "C" int64_t orc_num_vertices(const orc_ctx* c) {
    return (int64_t)c->g.size();
}

static bool is_goal(const orc_ctx* c, int64_t v) {
    return std::binary_search(c->goals.begin(), c->goals.end(), (int32_t)v);
}

// Goal cost used as the promising threshold: g(x_goal); for
// a goal set, the minimum over the goals that exist among the first n_exist
// vertices (R4).  *best receives the best goal: the lowest id attaining the
// minimum, or -1 if every such goal has g = +inf.
static double goal_cost(const orc_ctx* c, int64_t n_exist, int32_t* best = nullptr) {
    double m = kInf;
    int32_t arg = -1;
    for (int32_t t : c->goals) {          // ascending ids: strict < keeps the lowest
        if (t >= n_exist) break;
        if (c->g[t] < m) { m = c->g[t]; arg = t; }
    }
    if (best) *best = arg;
    return m;
}

// Extra goal vertices (R4, goal-set form): G = {x_goal} u ids.  Ids may name
// vertices not appended yet; they join G when they exist.
extern "C" int orc_set_goals(orc_ctx* c, const int32_t* ids, int32_t n) {
    if (n < 0 || (n > 0 && !ids)) return fail(-1, "set_goals: bad arguments");
    std::vector<int32_t> gs = {1};
    for (int32_t i = 0; i < n; ++i) {
        if (ids[i] < 1) return fail(-2, "set_goals: goal id must be >= 1 (not the root)");
        gs.push_back(ids[i]);
    }
    std::sort(gs.begin(), gs.end());
    gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
    c->goals = gs;
    return 0;
}

// Append one batch: S new vertices and their edges (Alg. 3 lines 6-8,
// PAPER.md:456-460), then the "small exploitation" of Extend on each new
// vertex, in increasing id order (reading R14):
//   g(v) = min over in-edges (u -> v) with u < v of g(u) + c(u, v),
//   lowest u among equal minima (R6); promising iff g(v) + h(v) < g(x_goal).
extern "C" int orc_append(orc_ctx* c, int32_t n_new, const double* h_new,
                          const int32_t* parent_new, const double* g_new,
                          int64_t n_edges, const int32_t* src,
                          const int32_t* dst, const double* cost,
                          uint32_t flags, int32_t* n_new_promising) {
    if (n_new < 0 || n_edges < 0) return fail(-1, "append: negative size");
    if ((parent_new == nullptr) != (g_new == nullptr))
        return fail(-1, "append: parent_new and g_new must both be given or both NULL");
    if (n_new > 0 && h_new == nullptr) return fail(-1, "append: h_new is NULL");
    if (n_edges > 0 && (src == nullptr || dst == nullptr || cost == nullptr))
        return fail(-1, "append: edge array is NULL");
    const int64_t n_old = (int64_t)c->g.size();
    const int64_t n_all = n_old + n_new;
    if (n_all > INT32_MAX) return fail(-2, "append: too many vertices");
    // ---- validate everything before committing (state unchanged on error) ----
    for (int32_t i = 0; i < n_new; ++i) {
        if (!(h_new[i] >= 0.0) || std::isinf(h_new[i]))
            return fail(-1, "append: h must be finite and >= 0 (R12)");
    }
    for (int64_t e = 0; e < n_edges; ++e) {
        if (src[e] < 0 || src[e] >= n_all || dst[e] < 0 || dst[e] >= n_all)
            return fail(-2, "append: edge endpoint out of range");
        if (src[e] == dst[e]) return fail(-1, "append: self-loop");
        if (!(cost[e] >= 0.0) || std::isinf(cost[e]))
            return fail(-1, "append: cost must be finite and >= 0 (R12)");
    }
    const bool undirected = (flags & ORC_F_EDGES_UNDIRECTED) != 0;
    // given policy for the new vertices: the edge (parent -> v) must be in
    // this batch (v is new, so all its in-edges are); its cost becomes pc(v).
    std::vector<double> pc_new(parent_new ? n_new : 0, 0.0);
    if (parent_new) {
        for (int32_t i = 0; i < n_new; ++i) {
            int32_t p = parent_new[i];
            int64_t v = n_old + i;
            if (p < -1 || p >= n_all || p == v)
                return fail(-2, "append: parent_new out of range");
            if (p < 0) {
                if (!std::isinf(g_new[i])) return fail(-1, "append: g_new must be +inf without a parent");
                continue;
            }
            if (!(g_new[i] >= 0.0) || std::isinf(g_new[i])) return fail(-1, "append: bad g_new");
            bool found = false;
            for (int64_t e = 0; e < n_edges && !found; ++e) {
                if (dst[e] == v && src[e] == p) { pc_new[i] = cost[e] + 0.0; found = true; }
                else if (undirected && src[e] == v && dst[e] == p) { pc_new[i] = cost[e] + 0.0; found = true; }
            }
            if (!found) return fail(-1, "append: edge (parent_new -> v) not in the batch");
            if ((flags | c->flags) & ORC_F_VALIDATE) {
                double gp = p < n_old ? c->g[p] : g_new[p - n_old];
                if (g_new[i] != gp + pc_new[i]) return fail(-1, "append: g_new != g[parent] + c");
            }
        }
    }
    if ((flags | c->flags) & ORC_F_VALIDATE) {
        // duplicate (src,dst) check over the whole graph
        std::vector<std::vector<int32_t>> seen(n_all);
        for (int64_t v = 0; v < n_old; ++v)
            for (auto& uc : c->in[v]) seen[v].push_back(uc.first);
        for (int64_t e = 0; e < n_edges; ++e) {
            seen[dst[e]].push_back(src[e]);
            if (undirected) seen[src[e]].push_back(dst[e]);
        }
        for (int64_t v = 0; v < n_all; ++v) {
            auto& s = seen[v];
            for (size_t i = 0; i < s.size(); ++i)
                for (size_t j = i + 1; j < s.size(); ++j)
                    if (s[i] == s[j]) return fail(-1, "append: duplicate edge");
        }
    }
    if (parent_new && ((flags | c->flags) & ORC_F_VALIDATE)) {
        std::vector<int32_t> p(c->parent);
        p.insert(p.end(), parent_new, parent_new + n_new);
        if (has_parent_cycle(p)) return fail(-8, "append: given policy has a parent cycle");
    }
    // ---- commit: vertices (SoA) and edges (COO -> in-lists) ----
    // promising threshold of the new vertices: the goal cost before the
    // batch (old goals only; a new goal vertex does not lower it for its own
    // batch), so the test does not depend on the order inside the batch
    const double thr = goal_cost(c, n_old);
    c->g.resize(n_all, kInf);
    c->h.resize(n_all, 0.0);
    c->pc.resize(n_all, 0.0);
    c->parent.resize(n_all, -1);
    c->b.resize(n_all, 0);
    c->in.resize(n_all);
    for (int32_t i = 0; i < n_new; ++i) c->h[n_old + i] = h_new[i] + 0.0;  // -0 -> +0
    for (int64_t e = 0; e < n_edges; ++e) {
        double w = cost[e] + 0.0;  // canonicalise -0.0 (R12)
        c->in[dst[e]].push_back({src[e], w});
        if (undirected) c->in[src[e]].push_back({dst[e], w});
    }
    c->n_edges += undirected ? 2 * n_edges : n_edges;
    // ---- local relaxation of each new vertex, in id order (R14) ----
    int32_t n_prom = 0;
    for (int64_t v = n_old; v < n_all; ++v) {
        if (parent_new) {
            c->parent[v] = parent_new[v - n_old];
            c->g[v] = g_new[v - n_old] + 0.0;
            c->pc[v] = pc_new[v - n_old];
        } else {
            double best = kInf;
            int32_t arg = -1;
            double argc = 0.0;
            for (auto& uc : c->in[v]) {
                int32_t u = uc.first;
                if (u >= v) continue;  // only vertices inserted before v
                double cand = c->g[u] + uc.second;
                if (cand < best || (cand == best && arg >= 0 && u < arg)) {
                    best = cand; arg = u; argc = uc.second;
                }
            }
            if (best < kInf) {
                c->g[v] = best; c->parent[v] = arg; c->pc[v] = argc;
            } else {
                c->g[v] = kInf; c->parent[v] = -1; c->pc[v] = 0.0;
            }
        }
        // "This small exploitation determines whether the new vertex is
        // promising, in which case it is added to the set B".
        c->b[v] = (c->g[v] + c->h[v] < thr) ? 1 : 0;
        n_prom += c->b[v];
    }
    if (n_new_promising) *n_new_promising = n_prom;
    return 0;
}

// Improve (Alg. 2).  Jacobi: g is read-only here
// (P:277-278).  I = B u {x_goal} \ {x_init} (R4); PRUNE_OFF: I = V \ {x_init};
// NEIGHBOURS (R16): I also holds every v with an in-edge from B u {x_init}.
// For each v in I, the min over in-edges of c(n,v) + g(n) with lowest-id tie
// break (R6); the policy changes only on a strict improvement over g(v)
// (P:246).  Delta g = max over I of g(v) - g_hat (R1).
static void improve(orc_ctx* c, double* dg_out, int32_t* changed_out,
                    int64_t* relax_out) {
    const int64_t n = (int64_t)c->g.size();
    const bool prune_off = (c->flags & ORC_F_PRUNE_OFF) != 0;
    // R16 (NEIGHBOURS variant): v also joins I when one of its
    // in-edges (u -> v) leaves a promising vertex or the root, i.e. when v is
    // a graph neighbour that could take a member of B u {root} as parent.
    // Membership is fixed before any change (b is not written by Improve).
    std::vector<uint8_t> nbr;
    if ((c->flags & ORC_F_NEIGHBOURS) && !prune_off) {
        nbr.assign(n, 0);
        for (int64_t v = 0; v < n; ++v)
            for (auto& uc : c->in[v])
                if (uc.first == kRoot || c->b[uc.first]) { nbr[v] = 1; break; }
    }
    double dg = 0.0;
    int32_t changed = 0;
    int64_t relax = 0;
    for (int64_t v = 0; v < n; ++v) {
        if (v == kRoot) continue;
        if (!(prune_off || c->b[v] || is_goal(c, v) || (!nbr.empty() && nbr[v]))) continue;
        double best = kInf;
        int32_t arg = -1;
        double argc = 0.0;
        for (auto& uc : c->in[v]) {
            double cand = uc.second + c->g[uc.first];  // c(n,v) + g_T(n)
            if (cand < best || (cand == best && arg >= 0 && uc.first < arg)) {
                best = cand; arg = uc.first; argc = uc.second;
            }
        }
        relax += (int64_t)c->in[v].size();
        if (best < c->g[v]) {  // strict
            double d = c->g[v] - best;
            if (d > dg) dg = d;
            if (c->parent[v] != arg) changed = 1;
            c->parent[v] = arg;
            c->pc[v] = argc;
        }
    }
    *dg_out = dg;
    *changed_out = changed;
    *relax_out = relax;
}

// Evaluate (Alg. 2): truncated breadth-first traversal of
// the policy tree from x_init.  thr = g(x_goal) snapshot at entry (R3); the
// promising test is applied to the child n (R2): g(n) + h(n) < thr.  Children
// failing the test get g updated but are not expanded.  B is
// rebuilt from scratch.  Returns whether any g bit or b bit changed
// (used only by the R13 stall guard).
static void evaluate(orc_ctx* c, int32_t* changed_out, int64_t* visits_out,
                     int32_t* levels_out) {
    const int64_t n = (int64_t)c->g.size();
    const double thr = (c->flags & ORC_F_PRUNE_OFF) ? kInf : goal_cost(c, n);
    const bool parent_form = (c->flags & ORC_F_PARENT_FORM) != 0;
    // child(T, v) = { n : parent(n) == v }, listed in id order.
    std::vector<std::vector<int32_t>> kids(n);
    for (int64_t v = 0; v < n; ++v)
        if (c->parent[v] >= 0) kids[c->parent[v]].push_back((int32_t)v);
    std::vector<double> g_old = c->g;
    std::vector<uint8_t> b_old = c->b;
    std::fill(c->b.begin(), c->b.end(), 0);  // B <- {}
    std::vector<int32_t> frontier = {kRoot}, next;  // Q <- {x_init}
    int64_t visits = 0;
    int32_t level = 0;  // depth of the deepest visited child (root depth 0)
    int32_t depth = 0;  // depth of the current frontier
    while (!frontier.empty()) {  // level order; order inside a level is irrelevant
        next.clear();
        bool visited = false;
        for (int32_t p : frontier) {
            for (int32_t v : kids[p]) {
                c->g[v] = c->g[p] + c->pc[v];  // g(n) <- c(v,n) + g(v)
                ++visits;
                visited = true;
                // child form (R2) g(n) + h(n) < thr, or the literal
                // parent form h(v) + g(v) < thr (NEXT-4 variant)
                const bool pass = parent_form ? (c->g[p] + c->h[p] < thr)
                                              : (c->g[v] + c->h[v] < thr);
                if (pass) {
                    c->b[v] = 1;                // B <- B u {n}
                    next.push_back(v);          // push(Q, n)
                }
            }
        }
        if (visited) level = depth + 1;
        ++depth;
        frontier.swap(next);
    }
    int32_t changed = 0;
    for (int64_t v = 0; v < n && !changed; ++v) {
        if (c->b[v] != b_old[v]) changed = 1;
        if (std::memcmp(&c->g[v], &g_old[v], sizeof(double)) != 0) changed = 1;
    }
    *changed_out = changed;
    *visits_out = visits;
    *levels_out = level;
}

extern "C" int orc_improve_step(orc_ctx* c, double* delta_g,
                                int32_t* parent_changed, int64_t* relaxations) {
    double dg; int32_t ch; int64_t r;
    improve(c, &dg, &ch, &r);
    if (delta_g) *delta_g = dg;
    if (parent_changed) *parent_changed = ch;
    if (relaxations) *relaxations = r;
    return 0;
}

extern "C" int orc_evaluate_step(orc_ctx* c, int32_t* changed, int64_t* visits,
                                 int32_t* levels) {
    int32_t ch, lv; int64_t vi;
    evaluate(c, &ch, &vi, &lv);
    if (changed) *changed = ch;
    if (visits) *visits = vi;
    if (levels) *levels = lv;
    return 0;
}

// Replan (Alg. 2): loop { Improve; if Delta g <= eps break
// (R5); Evaluate }.  R13: stop when an iteration changed no parent value and
// the following Evaluate changed no g bit and no b bit (a true fixed point of
// the iteration map).  R11: cap of max_iterations Improves (default 10 |V|).
extern "C" int orc_exploit(orc_ctx* c, orc_stats* out) {
    orc_stats st;
    std::memset(&st, 0, sizeof(st));
    const int64_t n = (int64_t)c->g.size();
    const int64_t cap = c->max_iterations > 0 ? c->max_iterations : 10 * n;
    int rc = 0;
    for (;;) {
        if (st.iterations >= cap) { rc = fail(-6, "exploit: iteration cap exceeded"); break; }
        double dg; int32_t ptr_changed; int64_t relax;
        improve(c, &dg, &ptr_changed, &relax);
        st.iterations += 1;
        st.last_delta_g = dg;
        st.relaxations += relax;
        if (dg <= c->epsilon) break;  // P:236 with R5
        int32_t changed, levels; int64_t visits;
        evaluate(c, &changed, &visits, &levels);
        st.evaluations += 1;
        st.eval_visits += visits;
        if (levels > st.max_level) st.max_level = levels;
        if (!ptr_changed && !changed) { st.stalled = 1; break; }  // R13
    }
    int32_t prom = 0;
    for (int64_t v = 0; v < n; ++v) prom += c->b[v];
    st.promising = prom;
    if (out) *out = st;
    return rc;
}

extern "C" int orc_get_state(const orc_ctx* c, int32_t* parent, double* g,
                             double* pc, uint8_t* b, int64_t cap) {
    const int64_t n = (int64_t)c->g.size();
    if (cap < n) return fail(-2, "get_state: capacity too small");
    for (int64_t v = 0; v < n; ++v) {
        if (parent) parent[v] = c->parent[v];
        if (g) g[v] = c->g[v];
        if (pc) pc[v] = c->pc[v];
        if (b) b[v] = c->b[v];
    }
    return 0;
}

// Restore a policy snapshot (parent, g, b); pc(v) is re-read from the stored
// edge (parent(v) -> v) (R9).  b == NULL means B = {}.
extern "C" int orc_set_policy(orc_ctx* c, const int32_t* parent,
                              const double* g, const uint8_t* b) {
    const int64_t n = (int64_t)c->g.size();
    if (!parent || !g) return fail(-1, "set_policy: NULL array");
    if (parent[kRoot] != -1 || g[kRoot] != 0.0)
        return fail(-1, "set_policy: root must have g=0 and no parent");
    std::vector<double> pc(n, 0.0);
    for (int64_t v = 0; v < n; ++v) {
        int32_t p = parent[v];
        if (p < -1 || p >= n || p == v) return fail(-2, "set_policy: parent out of range");
        if (!(g[v] >= 0.0)) return fail(-1, "set_policy: bad g");
        if (p >= 0) {
            bool found = false;
            for (auto& uc : c->in[v])
                if (uc.first == p) { pc[v] = uc.second; found = true; break; }
            if (!found) return fail(-1, "set_policy: parent edge not in graph");
        }
    }
    if (c->flags & ORC_F_VALIDATE) {
        if (has_parent_cycle(std::vector<int32_t>(parent, parent + n)))
            return fail(-8, "set_policy: parent cycle");
    }
    for (int64_t v = 0; v < n; ++v) {
        c->parent[v] = parent[v];
        c->g[v] = g[v] + 0.0;
        c->pc[v] = pc[v];
        c->b[v] = b ? (b[v] ? 1 : 0) : 0;
    }
    return 0;
}

// Policy-tree extraction (Alg. 1 lines 8-12): the branch
// of the best goal (lowest g, lowest id on ties), root..goal.  Unreached
// goal set: length 0, cost +inf, goal -1.
extern "C" int orc_best_path(const orc_ctx* c, int32_t* path, int64_t cap,
                             int64_t* len, double* cost, int32_t* goal) {
    const int64_t n = (int64_t)c->g.size();
    int32_t best = -1;
    double gc = goal_cost(c, n, &best);   // best goal: lowest id at the minimum (R4, R6)
    if (std::isinf(gc)) {
        if (len) *len = 0;
        if (cost) *cost = kInf;
        if (goal) *goal = -1;
        return 0;
    }
    std::vector<int32_t> rev;
    int32_t v = best;
    while (v != -1) {
        rev.push_back(v);
        if ((int64_t)rev.size() > n) return fail(-8, "best_path: parent cycle");
        v = c->parent[v];
    }
    if (rev.back() != kRoot) return fail(-8, "best_path: goal branch does not reach the root");
    if ((int64_t)rev.size() > cap) return fail(-2, "best_path: capacity too small");
    for (size_t i = 0; i < rev.size(); ++i) path[i] = rev[rev.size() - 1 - i];
    if (len) *len = (int64_t)rev.size();
    if (cost) *cost = gc;
    if (goal) *goal = best;
    return 0;
}
