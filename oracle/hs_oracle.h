/*
 * hs_oracle.h -- CPU restatement of the hetsched scheduler hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * sm_100a product path (paper_2206_01288_b200/csrc).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it.  The product path never links or calls it.
 *
 * It restates /root/reference/pkg/src/hetsched/{costmodel,combinatorics,
 * scheduler,evaluation}.py in plain C, including numpy's float-order and
 * PCG64 stream contracts, and is pinned against golden vectors produced by
 * running the reference itself (tests/golden/make_golden.py).
 */
#ifndef HS_ORACLE_H
#define HS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* numpy.random.PCG64 + Generator buffered-uint32 state. */
typedef struct {
    uint64_t state_hi, state_lo, inc_hi, inc_lo;
    int32_t has_uint32;
    uint32_t uinteger;
} orc_pcg64;

typedef struct orc_inst orc_inst;

/* dp_num = 8.0*c_dp, pp_num = 8.0*c_pp, sw_num = 8.0*(c_pp + c_dp), each
 * formed on the host with Python's own arithmetic. */
orc_inst *orc_create(int n, const double *lat, const double *bw, int d_pp, int d_dp,
                     double dp_num, double pp_num, double sw_num);
void orc_destroy(orc_inst *in);
void orc_tables(const orc_inst *in, double *dp, double *pp, double *sw);

/* one partition: groups[k*m], members ascending.  order may be NULL. */
int orc_comm_cost(const orc_inst *in, const int32_t *groups, double *out3,
                  double *per_group, int32_t *order);
int orc_comm_cost_heuristic(const orc_inst *in, const int32_t *groups, double *out3, int32_t *order);
/* batch over int16 [P][k][m]; nthreads <= 0 -> 1 */
int orc_comm_cost_batch(const orc_inst *in, const int16_t *groups, int64_t P,
                        double *total, double *datap, double *pipelinep, int nthreads);

double orc_datap_group(const orc_inst *in, const int32_t *members, int cnt);
double orc_bottleneck_value(const double *w, int m);
int orc_bottleneck_matching(const double *w, int m, int32_t *pairs, double *value);
/* exact Held-Karp; returns 0 ok, -1 if k > 16 */
int orc_open_loop_tsp(const double *w, int k, double *total, int32_t *order);
int orc_open_loop_tsp_heuristic(const double *w, int k, double *total, int32_t *order);
double orc_path_cost(const double *w, int k, const int32_t *order, int len);

/* RNG primitives (numpy Generator semantics) */
uint64_t orc_next64(orc_pcg64 *g);
uint32_t orc_next32(orc_pcg64 *g);
int64_t orc_integers(orc_pcg64 *g, int64_t low, int64_t high);
void orc_permutation(orc_pcg64 *g, int n, int32_t *out);
void orc_choice_noreplace_sorted(orc_pcg64 *g, int pop, int size, int32_t *out);
double orc_uniform(orc_pcg64 *g, double lo, double hi);

void orc_random_partition(orc_pcg64 *g, int n, int k, int m, int32_t *groups);
void orc_crossover(const int32_t *p1, const int32_t *p2, int k, int m, orc_pcg64 *g,
                   int32_t *out);

/* surrogate gains on the instance's SW table */
double orc_gain_ours(const orc_inst *in, const int32_t *groups, int j, int j2, int d1,
                     int d2, int d1p, int d2p);
double orc_gain_kl(const orc_inst *in, const int32_t *groups, int d, int d2);
void orc_fast_edge(const orc_inst *in, const int32_t *grp, int cnt, int32_t *out2);

/* kind: 0 = ours, 1 = kl.  groups_inout[k*m]. returns evaluations made. */
int orc_local_search(const orc_inst *in, int32_t *groups_inout, int kind, orc_pcg64 *g,
                     int max_passes);
/* one refinement pass on a balanced partition (phase used by ours). */
int orc_pass(const orc_inst *in, int32_t *groups_inout, int kind, orc_pcg64 *g, int phase);

typedef struct {
    int pop_size, generations, kind /*0 ours 1 kl 2 none*/, max_passes, patience /*<=0 none*/;
} orc_ga_cfg;

/* trace_best/trace_mean sized generations; returns number of trace rows,
 * or <0 on error.  best_groups[k*m] canonical; best3 = (total, datap,
 * pipelinep); best_per_group[k]; best_order[k]. */
int orc_evolve(const orc_inst *in, const orc_ga_cfg *cfg, orc_pcg64 *g, int32_t *best_groups,
               double *best3, double *best_per_group, int32_t *best_order, double *trace_best,
               double *trace_mean, int64_t *evaluations);

/* fixed-layout pricing (evaluation.py) */
int orc_random_assignment(orc_pcg64 *g, int n, int k, int m, int32_t *grid /*m*k*/,
                          int32_t *order);
int orc_evaluate_assignment(const orc_inst *in, const int32_t *grid /*m rows x k cols*/,
                            double *out3, double *per_col);
int orc_materialize(const orc_inst *in, const int32_t *groups, int32_t *grid, int32_t *order);

#ifdef __cplusplus
}
#endif
#endif
