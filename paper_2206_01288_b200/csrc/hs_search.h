// hs_search.h -- host/device interface of the search kernels (K2/K3).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hetsched_b200.h"
#include "hs_internal.h"

namespace hs {

// Per-island GA state kept in global memory between launches (epochs).
struct GAState {
    hs_pcg64 rng;
    double best_total;
    long long evaluations;
    int best_idx, since, gen, stopped, initialized, finalized;
};

struct GAArgs {
    int n, k, m;
    const double* sw;
    const double* dp;
    const void* rank;
    const double* vals;
    HKTables hk;
    int pop, generations, kind /*0 ours 1 kl 2 none*/, max_passes, patience /*<=0: none*/;
    int islands;
    HKBig hkb;            // d_pp > 8: CTA pricing schedule
    double* hk_scratch;   // d_pp > 8: per-island Held-Karp slices
    size_t hk_size;
    int gen_end;   // run generations [state.gen, gen_end)
    int finalize;  // price the canonical best when the run is over
    GAState* state;      // [islands]
    int16_t* pop_buf;    // [islands][pop][k*m]
    double* cost_buf;    // [islands][pop]
    int16_t* best_buf;   // [islands][k*m]
    double* trace_best;  // [islands][generations] (nullable)
    double* trace_mean;
    double* out3;        // [islands][3] total, datap, pipelinep
    double* out_pg;      // [islands][k]
    int8_t* out_order;   // [islands][k]
    int16_t* out_groups; // [islands][k*m] canonical best
    long long* prof;     // optional driver-phase cycle counters (island 0), see hs_search.cu
    // batch-priced generations (d_pp 9..16 with the cluster Held-Karp path):
    // phase 1 runs one generation up to its snapshots and writes them to
    // snap_buf (island i: slots [i * snap_stride, + snap_cnt[i]), the rest
    // marked invalid; the initial population on the first call), phase 2
    // commits that generation from snap_cost; phase 0 prices in-kernel
    int phase;
    int snap_stride;
    int16_t* snap_buf;   // [islands][snap_stride][k*m]
    double* snap_cost;   // [islands][snap_stride] (totals)
    int* snap_cnt;       // [islands]
};

struct RefineArgs {
    int n, k, m;
    const double* sw;
    const double* dp;
    const void* rank;
    const double* vals;
    HKTables hk;
    HKBig hkb;
    double* hk_scratch;
    size_t hk_size;
    int kind, max_passes, single_pass, phase;
    const int16_t* groups;  // [B][k*m]
    hs_pcg64* rng;          // [B] in/out
    int16_t* out_groups;    // [B][k*m]
    double* out_cost;       // [B]
    int* evaluations;       // [B]
    int* changed;           // [B] (single_pass)
    // batch pricing (d_pp 9..16): the passes' snapshots go to snap_buf
    // (partition b: slots [b * snap_stride, + snap_cnt[b]), the rest marked
    // invalid) instead of being priced in-kernel; refine_commit picks
    int16_t* snap_buf;
    int* snap_cnt;
    int snap_stride;
};

// first-minimum snapshot per partition from the batch-priced snap_cost
int launch_refine_commit(const RefineArgs& a, const double* snap_cost, int B, cudaStream_t st);

// one pass, no pricing (any d_pp <= 32)
struct PassArgs {
    int n, k, m, kind, phase;
    const double* sw;
    const int16_t* groups;  // [B][k*m]
    hs_pcg64* rng;          // [B]
    int16_t* out_groups;
    int* changed;
    double* mean;     // [B][n*k] global scratch
    uint32_t* mver;   // [B][n*k]
};

struct SearchShape {
    int n, k, m, max_passes, nvals;
    bool key16;
    HKTables hk;
};

struct SearchPlan {
    int warps;
    bool smem_tables, m8, cta, warp_islands;
    size_t smem;
};

int search_plan(const SearchShape& sh, int P, size_t smem_optin, SearchPlan* plan, bool warp_islands = false);
int launch_ga(const GAArgs& a, const SearchPlan& plan, int islands, bool key16, cudaStream_t st);
// one GA as a speculative generation pipeline over a thread-block cluster
// (hs_search_ga_spec.cu): cluster size for this plan (0 = unavailable), launch
int ga_spec_cluster(const GAArgs& a, const SearchPlan& plan, bool key16, size_t smem_optin);
int launch_ga_spec(const GAArgs& a, const SearchPlan& plan, int cluster, bool key16, cudaStream_t st);
int launch_refine(const RefineArgs& a, const SearchPlan& plan, int B, bool key16, cudaStream_t st);
int launch_crossover(int n, int k, int m, const int16_t* p1, const int16_t* p2, hs_pcg64* rngs, int16_t* out, int B,
                     cudaStream_t st);
int launch_gains(int n, int k, int m, const double* sw, const int16_t* groups, const int32_t* q, int kind, int B,
                 double* out, cudaStream_t st);

int launch_export(int islands, int P, int km, int E, const int16_t* pop, const double* cost, int16_t* out,
                  double* out_cost, cudaStream_t st);
int launch_import(int islands, int P, int km, int E, int16_t* pop, double* cost, int16_t* best, GAState* state,
                  const int16_t* mig, const double* mig_cost, const int32_t* src, cudaStream_t st);
int launch_pass(const PassArgs& a, int B, cudaStream_t st);
int launch_random_partitions(int n, int k, int m, int B, hs_pcg64* rng, int16_t* out, cudaStream_t st);

}  // namespace hs
