/*
 * oracle.h -- serial CPU oracle for the PI-RRT# exploitation phase.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this
 * library.  The product path (paper_2003_04920_b200/) never does, and shares
 * no code, header, helper or constant with it.
 *
 * The oracle follows Alg. 2 of arXiv 2003.04920 with the
 * readings R1-R14 listed in DESIGN.md section 3.  All floating point is IEEE
 * binary64 (the paper does not fix a precision).
 *
 * Vertex 0 is x_init (root, g = 0) and vertex 1 is x_goal (g = +inf),
 * created by orc_create (Alg. 1 line 1).
 *
 * Error codes: 0 ok, -1 invalid argument, -2 range, -6 no convergence,
 * -7 bad state, -8 corrupt (cycle).  On error the state is unchanged
 * (append validates before it commits).
 */
#ifndef PIRRT_ORACLE_H
#define PIRRT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_ctx orc_ctx;

#define ORC_F_PRUNE_OFF 1u        /* I = V \ {root}, thr = +inf (classical PI) */
#define ORC_F_VALIDATE 2u         /* duplicate-edge and g_new consistency checks */
#define ORC_F_EDGES_UNDIRECTED 4u /* append: each (src,dst,cost) stored both ways */
#define ORC_F_PARENT_FORM 8u      /* Evaluate tests the parent, h(v)+g(v) < thr, as
                                     printed at PAPER.md:263 (NEXT-4 variant of R2) */
#define ORC_F_NEIGHBOURS 16u      /* "promising vertices and their neighbors are
                                     re-evaluated" (NEXT-4, reading
                                     R16): I = B u N+(B u {root}) u G \ {root}       */

typedef struct {
    int32_t iterations;     /* number of Improve calls (Alg. 2)            */
    double last_delta_g;    /* Delta g of the final Improve                          */
    int64_t relaxations;    /* sum over Improves of sum_{v in I} indeg(v)            */
    int64_t eval_visits;    /* children visited, summed over Evaluates               */
    int32_t max_level;      /* deepest BFS level reached by any Evaluate (root = 0)  */
    int32_t promising;      /* |B| on return                                         */
    int32_t stalled;        /* 1 if the R13 stall guard stopped the loop             */
    int32_t evaluations;    /* number of Evaluate calls                              */
} orc_stats;

orc_ctx* orc_create(double h_root, double h_goal, double epsilon,
                    int32_t max_iterations, uint32_t flags);
void orc_destroy(orc_ctx* c);
const char* orc_last_error(void);
int64_t orc_num_vertices(const orc_ctx* c);

int orc_append(orc_ctx* c, int32_t n_new, const double* h_new,
               const int32_t* parent_new, const double* g_new, int64_t n_edges,
               const int32_t* src, const int32_t* dst, const double* cost,
               uint32_t flags, int32_t* n_new_promising);

int orc_exploit(orc_ctx* c, orc_stats* out);

/* Goal set (reading R4, goal-set form): G = {x_goal} u ids[0..n).  Ids may
 * name vertices appended later.  Threshold = min over existing goals of g;
 * every existing goal is in the Improve set. */
int orc_set_goals(orc_ctx* c, const int32_t* ids, int32_t n);

/* single steps, for the worked-example pins */
int orc_improve_step(orc_ctx* c, double* delta_g, int32_t* parent_changed,
                     int64_t* relaxations);
int orc_evaluate_step(orc_ctx* c, int32_t* changed, int64_t* visits,
                      int32_t* levels);

int orc_get_state(const orc_ctx* c, int32_t* parent, double* g, double* pc,
                  uint8_t* b, int64_t cap);
int orc_set_policy(orc_ctx* c, const int32_t* parent, const double* g,
                   const uint8_t* b);
int orc_best_path(const orc_ctx* c, int32_t* path, int64_t cap, int64_t* len,
                  double* cost, int32_t* goal);

#ifdef __cplusplus
}
#endif
#endif
