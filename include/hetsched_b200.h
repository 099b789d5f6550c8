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

/* One network instance + workload on one device: uploads lat/bw (n*n
 * float64, symmetric, bw diagonal +inf) and builds the DP/PP/SW pair tables
 * (K0) and the PP rank table.  Replaces the per-call np.ix_ gathers of
 * costmodel.py:154-183 and SurrogateWeights.from_instance
 * (scheduler.py:84-88), which the reference rebuilds on every call. */
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

/* Same, host buffers (pinned for full overlap); copies in, evaluates in
 * double-buffered chunks, copies out, returns when done.  *invalid (host)
 * receives the malformed-candidate count. */
int hs_eval_batch_host(hs_instance *h, const int16_t *groups, int64_t P, double *total, double *datap,
                       double *pipelinep, double *per_group, int8_t *order, int32_t *invalid);

/* bottleneck_value (combinatorics.py:128-131) of B matrices [B][m][m],
 * m <= 64, entries finite and >= 0 (device pointers). */
int hs_bottleneck_batch(const double *w, int m, int64_t B, double *out, int device, void *stream);

/* exact open_loop_tsp (combinatorics.py:232-296, Held-Karp) of B symmetric
 * [B][k][k] matrices, k <= 8: total [B] and lexicographically smallest
 * optimal order [B][k] (order may be NULL).  Device pointers. */
int hs_path_batch(const double *w, int k, int64_t B, double *total, int8_t *order, int device, void *stream);

#ifdef __cplusplus
}
#endif
#endif
