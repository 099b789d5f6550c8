// hs_cluster.h -- host interface of the cluster Held-Karp path (9 <= d_pp <= 16,
// pricing without a stage order).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hs_internal.h"

namespace hs {

constexpr int kStageES = 17;                  // padded stage-graph row (= kES16)
constexpr int kStageStride = 16 * kStageES;   // doubles per staged candidate

// Two-layer Held-Karp schedule, "push" form.  Layer p holds the entries
// h[s][u], |s| = p, u in s, at slot (rank_p(s) - sbeg[p][q]) * p + (rank of u
// in s) of CTA q, where rank_p orders the p-subsets as integers and CTA q owns
// the sets sbeg[p][q] .. sbeg[p][q + 1] (a balanced split by whole sets, so a
// set's entries never straddle two CTAs).  Layer p is produced r-major: the
// CTA that owns r (|r| = p - 1) loads h[r][.] from its own shared memory once
// and computes h[r | u][u] = min_v (w[u][v] + h[r][v]) for every u not in r,
// pushing each result into the owner of r | u with an asynchronous DSMEM
// store that completes on the owner's mbarrier for layer p.
//   rwords[i]: one work item: r (16) | local slot of h[r][first member] (15)
//              << 16 | index of the item's first destination word (21) << 31
//              | j0 (4) << 52 | cnt (5) << 56 -- the item relaxes the u not
//              in r after skipping the j0 lowest, cnt of them (layers with
//              few sources split a source's u over several items)
//   dwords[j]: destination CTA (4) << 17 | local slot (17), one per u not in
//              r, ascending u
// The items of layer p on CTA q are rwords[rbeg[p][q] .. rbeg[p][q + 1]).
struct HKTwo {
    const uint64_t* rwords;
    const uint32_t* dwords;
    int rbeg[18][17];
    int sbeg[18][17];  // owned p-subsets per CTA (prefix counts)
    int C[18];    // slice length per layer (entries, max over the CTAs)
    int Cmax;     // buffer length (max over layers)
    int cs;       // CTAs per cluster (1, 2, 4, 8 or 16)
};

int get_hk_two(int device, int k, HKTwo* out);
size_t cluster_smem_bytes(const HKTwo& t);
// grid in CTAs for one pricing launch (a multiple of t.cs)
int cluster_grid(const HKTwo& t, int sm_count);  // CTAs: co-resident clusters x cs

// Stage kernel: validation, datap / per_group and the padded stage graph
// E[b] (16 x 17 doubles) of partitions [0, P) of a.groups; bad[b] = 1 for
// malformed ones (their outputs are NaN, a.invalid counts them).
int launch_stage(const EvalArgs& a, double* E, double* datap, uint8_t* bad, int blocks, bool m8, cudaStream_t s);

// Held-Karp totals of B stage graphs: E + b * estride, row stride es; when
// `add` is given, out_total[b] = add[b] + path and out_pipe[b] = path,
// else out_total[b] = path; bad[b] (nullable) skips a graph (NaN outputs).
int launch_hk_cluster(const double* E, int es, int64_t estride, int k, int64_t B, const HKTwo& t, int grid,
                      const double* add, const uint8_t* bad, double* out_total, double* out_pipe, cudaStream_t s);

}  // namespace hs
