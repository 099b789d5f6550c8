/*
 * hetsched_b200.h -- C-ABI of libhetsched_sm100a.so, the B200-native hot path
 * of the arXiv 2206.01288 layout scheduler (reference: hetsched 0.1.0,
 * /root/reference/pkg/src/hetsched).
 *
 * Plain pointers and sizes only; no torch types.  Every call returns 0 on
 * success and a negative code on failure (hs_last_error() has the message);
 * nothing throws.  Input validation that the reference reports as
 * ValueError subclasses stays in the Python mirror
 * (paper_2206_01288_b200/), which calls these entry points through ctypes.
 * Device-pointer entry points are asynchronous on `stream` (a cudaStream_t,
 * NULL = legacy default stream); *_host entry points take host buffers and
 * return after the results are in them.
 *
 * Numerators are formed by the caller with the reference's own scalar
 * arithmetic:  dp_num = 8.0*c_dp, pp_num = 8.0*c_pp, sw_num = 8.0*(c_pp+c_dp)
 * (costmodel.py:136,141; scheduler.py:85).
 */
#ifndef HETSCHED_B200_H
#define HETSCHED_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hs_instance hs_instance;

/* numpy.random.PCG64 state plus Generator's buffered uint32
 * (bit_generator.state: state, inc, has_uint32, uinteger). */
typedef struct {
    uint64_t state_hi, state_lo, inc_hi, inc_lo;
    int32_t has_uint32;
    uint32_t uinteger;
} hs_pcg64;

int hs_version(void);
const char *hs_last_error(void);
/* Measurement helper (no reference counterpart): shared-memory bandwidth of
 * `device` in bytes/s over all SMs (conflict-free 16-byte loads), the
 * measured denominator of bench.py's on-chip roofline; *ms (optional) is
 * one probe launch. */
int hs_probe_smem_bandwidth(int device, double *bytes_per_s, double *ms);

/* One network instance + workload on one device: uploads lat/bw (n*n
 * float64, symmetric, bw diagonal +inf) and builds the DP/PP/SW pair tables
 * (K0) and the PP rank table.  Replaces the per-call np.ix_ gathers of
 * costmodel.py:154-183 and SurrogateWeights.from_instance
 * (scheduler.py:84-88), which the reference rebuilds on every call.
 * On error nothing is leaked and *h is untouched.
 *
 * Threading: every entry point is re-entrant per handle.  Calls on
 * different streams never share device scratch (d_pp 9..16 / > 16 calls
 * take a per-call scratch set from the handle's pool); the host-buffer
 * entry serialises on the handle.  The search / GA / assignment entries
 * raise the device's per-thread stack limit to 8 KiB if it is lower
 * (cudaLimitStackSize, process-wide). */
int hs_instance_create(const double *lat, const double *bw, int n, int d_pp, int d_dp, double dp_num,
                       double pp_num, double sw_num, int device, hs_instance **out);
int hs_instance_destroy(hs_instance *h);
/* copy the device pair tables back (any pointer may be NULL) */
int hs_instance_tables(hs_instance *h, double *dp, double *pp, double *sw);

/* K1: bi-level cost of P partitions.  groups: int16 [P][d_pp][d_dp], members
 * ascending (the Partition invariant, costmodel.py:58-72).  Outputs
 * total/datap/pipelinep [P] float64 (CostBreakdown, costmodel.py:114-131);
 * per_group [P][d_pp] (per_group_datap) and order [P][d_pp]
 * (pipeline_order) are optional (NULL).  Malformed candidates get NaN and
 * are counted in *invalid (device int, optional).  Replaces comm_cost
 * (costmodel.py:217-229) and the population map of evolve
 * (scheduler.py:537-542).  All pointers are device pointers. */
int hs_eval_batch(hs_instance *h, const int16_t *groups, int64_t P, double *total, double *datap,
                  double *pipelinep, double *per_group, int8_t *order, int32_t *invalid, void *stream);

/* hs_eval_batch with heuristic=True semantics (comm_cost(..., heuristic=True),
 * costmodel.py:217): d_pp > 16 orders stages with nearest-neighbour + 2-opt
 * (combinatorics.py:299-342) instead of exact Held-Karp; d_pp <= 16 is
 * exact either way.  Partitions are not validated here (callers do). */
int hs_eval_batch_ex(hs_instance *h, const int16_t *groups, int64_t P, double *total, double *datap, double *pipelinep,
                     double *per_group, int8_t *order, int32_t *invalid, int heuristic, void *stream);

/* Same, host buffers (pinned for full overlap); copies in, evaluates and
 * copies out as a pipeline over device-held spans (at N = 64, 8x8 one kernel
 * per span consumes chunks as they land), returns when done.  *invalid
 * (host) receives the malformed-candidate count.  Replaces the per-layout
 * comm_cost loop of scheduler.py:537-542 for host arrays. */
int hs_eval_batch_host(hs_instance *h, const int16_t *groups, int64_t P, double *total, double *datap,
                       double *pipelinep, double *per_group, int8_t *order, int32_t *invalid);

/* bottleneck_value (combinatorics.py:128-131) of B matrices [B][m][m],
 * m <= 64, entries finite and >= 0 (device pointers). */
int hs_bottleneck_batch(const double *w, int m, int64_t B, double *out, int device, void *stream);

/* open_loop_tsp(heuristic=True) for any 2 <= k <= 64: nearest neighbour from
 * every start + first-improvement 2-opt (combinatorics.py:299-342); device
 * pointers, one thread per matrix. */
int hs_path_heuristic_batch(const double *w, int k, int64_t B, double *total, int8_t *order, int device, void *stream);

/* exact open_loop_tsp (combinatorics.py:232-296, Held-Karp) of B symmetric
 * [B][k][k] matrices, k <= 8: total [B] and lexicographically smallest
 * optimal order [B][k] (order may be NULL).  Device pointers. */
int hs_path_batch(const double *w, int k, int64_t B, double *total, int8_t *order, int device, void *stream);


/* ---------------- search: K2 (swap gains / local search), K3 (GA) ----------
 * All search entry points reproduce numpy's PCG64 stream draw for draw: the
 * caller passes bit_generator.state and receives the advanced state back
 * (so later caller draws stay aligned, scheduler.py:490-512). */

typedef struct {
    int32_t pop_size, generations, kind /* 0 ours, 1 kl, 2 none */, max_passes, patience /* <= 0: none */;
} hs_ga_config;

typedef struct hs_ga hs_ga;

/* A GA session of `islands` independent steady-state GAs, one CTA each, with
 * island i seeded by rng[i] (evolve, scheduler.py:515-574; the numpy
 * Generator(PCG64(seed)) state of :528).  Population and RNG stay on the
 * device between hs_ga_run calls, so a run can be cut into epochs. */
int hs_ga_create(hs_instance *h, const hs_ga_config *cfg, int islands, const hs_pcg64 *rng, hs_ga **out);
/* mode 0: one CTA per island (all warps price each generation's snapshots in
 * parallel; lowest single-island latency).  mode 1: one warp per island
 * (d_pp <= 8; up to 8 islands per CTA sharing the staged tables; highest
 * island throughput).  Results are identical in both modes. */
int hs_ga_create_ex(hs_instance *h, const hs_ga_config *cfg, int islands, const hs_pcg64 *rng, int mode, hs_ga **out);
/* advance every island to generation `until` (or its patience stop) */
int hs_ga_run(hs_ga *ga, int until, void *stream);
/* island migration (no reference counterpart): export each
 * island's `elites` best members (cost, then index) as int16 [islands][E][k*m]
 * + float64 [islands][E] device buffers; import replaces the island's worst
 * members (first maximum, one per migrant, only if the migrant is strictly
 * cheaper) with migrants[src[i]] for island i. */
int hs_ga_export(hs_ga *ga, int elites, int16_t *groups, double *costs, void *stream);
int hs_ga_import(hs_ga *ga, int elites, const int16_t *groups, const double *costs, const int32_t *src, void *stream);
/* finalize (canonical best, priced once more, :570-574) and copy results to
 * host buffers: best_groups [islands][k*m], best3 [islands][3] (total, datap,
 * pipelinep), best_per_group [islands][k], best_order [islands][k],
 * trace_best / trace_mean [islands][generations], trace_len [islands],
 * evaluations [islands], rng [islands] (advanced states).  NULL skips.
 * Synchronizes the stream of the session's latest run / export / import
 * first; returns -2 if an island is neither stopped (patience) nor run to
 * `generations` (call hs_ga_run(ga, generations, ...) first). */
int hs_ga_result(hs_ga *ga, int16_t *best_groups, double *best3, double *best_per_group, int8_t *best_order,
                 double *trace_best, double *trace_mean, int32_t *trace_len, int64_t *evaluations, hs_pcg64 *rng);
int hs_ga_destroy(hs_ga *ga);

/* local_search (scheduler.py:490-512, _refine :455-487) on B partitions,
 * each with its own stream; host buffers. */
int hs_local_search(hs_instance *h, int kind, int max_passes, int B, const int16_t *groups, hs_pcg64 *rng,
                    int16_t *out, double *out_total, int32_t *evaluations);
/* one refinement pass (_pass_ours phase / _pass_kl, scheduler.py:394-449) */
int hs_refine_pass(hs_instance *h, int kind, int phase, int B, const int16_t *groups, hs_pcg64 *rng, int16_t *out,
                   int32_t *changed);
/* crossover (scheduler.py:139-174) on B parent pairs of shape d_pp x d_dp
 * (n = d_pp*d_dp), one stream each; host buffers */
int hs_crossover(int n, int d_pp, int d_dp, int device, int B, const int16_t *p1, const int16_t *p2, hs_pcg64 *rng,
                 int16_t *out);
/* gain_ours (kind 0, q = j, j2, d1, d2, d1', d2') / gain_kl (kind 1, q = d, d2,
 * group(d), group(d2)), scheduler.py:181-230, on any n x n surrogate table
 * sw (SurrogateWeights.w); host buffers, q is int32 [B][6] */
int hs_gains(int n, int d_pp, int d_dp, int device, const double *sw, int kind, int B, const int16_t *groups,
             const int32_t *q, double *out);
/* init_population / random_partition (scheduler.py:114-136): B sequential
 * random_partition draws from one stream into int16 [B][n] (groups of d_dp,
 * members ascending) */
int hs_random_partitions(int n, int d_pp, int d_dp, int device, int B, hs_pcg64 *rng, int16_t *out);

/* ---------------- exhaustive search (costmodel.py:232-266) ------------------ */

/* number of balanced partitions of n devices into groups of d_dp (-1 if
 * d_dp does not divide n) */
int64_t hs_count_partitions(int n, int d_dp);
/* partitions [start, start+count) of the reference's enumeration order
 * (_balanced_partitions: lexicographic canonical keys) as int16
 * [count][d_pp][d_dp] into device memory; n <= 64 */
int hs_unrank_partitions(int n, int d_pp, int d_dp, int64_t start, int64_t count, int16_t *out, void *stream);

/* ---------------- fixed layouts (evaluation.py) ---------------------------- */

/* materialize (evaluation.py:162-192): grid int16 [B][d_dp][d_pp] (row i =
 * macro-batch chain, column b = stage) and stage order int8 [B][d_pp] of B
 * partitions, using the lexicographically smallest bottleneck pairing
 * (combinatorics.py:147-189) between consecutive stages; host buffers,
 * d_pp <= 8. */
int hs_materialize(hs_instance *h, int64_t B, const int16_t *groups, int16_t *grid, int8_t *order);
/* evaluate_assignment (evaluation.py:195-229) of B grids int16
 * [B][d_dp][d_pp]: out3 [B][3] (total, datap, pipelinep), per_col [B][d_pp]
 * (nullable); host buffers.  Grids must be valid assignments. */
int hs_evaluate_assignments(hs_instance *h, int64_t B, const int16_t *grids, double *out3, double *per_col);
/* random_assignment (evaluation.py:232-243) for B independent streams:
 * grids int16 [B][d_dp][d_pp], orders int8 [B][d_pp]; host buffers. */
int hs_random_assignments(int n, int d_pp, int d_dp, int device, int B, hs_pcg64 *rng, int16_t *grids, int8_t *orders);

/* ---------------- single-matrix solvers behind coarsen() ------------------- */

/* bottleneck_perfect_matching (combinatorics.py:134-144) of B matrices
 * [B][m][m], m <= 64, entries finite and >= 0: value [B] (an exact entry)
 * and the lexicographically smallest optimal pairing pairs [B][m] (row ->
 * column; nullable).  Device pointers; replaces the per-pair Python loop
 * in coarsen (costmodel.py:186-197). */
int hs_bottleneck_match_batch(const double *w, int m, int64_t B, double *value, int8_t *pairs, int device,
                              void *stream);
/* datap_cost_group (costmodel.py:154-168) of G groups from gathered raw
 * blocks lat/bw [G][m][m] (rows and columns = sorted members), m <= 128:
 * out [G] = max row of numpy-pairwise sums of 2.0*(lat + dp_num/(ddp*bw))
 * with a 0.0 diagonal.  ddp = (double)d_dp, dp_num = 8.0*c_dp (host
 * formed).  Device pointers. */
int hs_datap_group_batch(const double *lat, const double *bw, int m, int64_t G, double ddp, double dp_num, double *out,
                         int device, void *stream);
/* The reference's exhaustive oracles over all k! permutations, k <= 10, of
 * one k x k matrix (device pointers): kind 0 = brute_force_bottleneck_
 * matching (combinatorics.py:192-207, value = largest selected entry), kind
 * 1 = brute_force_open_loop_tsp (:345-361, value = right-to-left path
 * cost).  perm [k] = the first permutation in itertools order attaining the
 * minimum, as the reference's strict `<` scan keeps. */
int hs_brute_force(const double *w, int k, int kind, double *value, int8_t *perm, int device, void *stream);

#ifdef __cplusplus
}
#endif
#endif
