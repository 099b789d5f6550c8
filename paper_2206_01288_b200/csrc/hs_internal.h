// hs_internal.h -- host-side declarations shared by the kernels and the C-ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hs {

// Held-Karp schedule for one k (<= 8): packed state words grouped by layer
// (see hs_eval.cuh), layer starts, and compact offsets off[s].
struct HKTables {
    const uint4* states;  // 16-byte pre-decoded states (hs_eval.cuh, warp_held_karp)
    int nstates;
    int lay[18];
    const uint16_t* hoff;
    int nhoff;
    int final_off;  // first of the full set's k entries in h
    int hsize;      // doubles of h the schedule touches
};

// Held-Karp schedule for 9 <= k <= 16 (one CTA per candidate): 64-bit state
// words off[r] (20) | dst (20) | u (4) | r (16) grouped by layer, and the
// compact offsets off[s] (2^k entries).
struct HKBig {
    const uint64_t* states;
    int nstates;
    int lay[18];
    const uint32_t* off;
    int noff;
};

struct EvalArgs {
    int n, k, m;
    const double* dp;    // n*n data-parallel pair seconds (0 diagonal)
    const void* rank;    // n*n rank of PP entries among distinct values (u16 or u32)
    bool key16;          // rank table is uint16
    int nvals;           // distinct PP values
    const double* vals;  // distinct PP values, ascending
    HKTables hk;
    HKTables hk_roll;       // two-layer (ping-pong) schedule: no order reconstruction
    const int16_t* groups;  // [P][k][m], members ascending
    int64_t P;
    double* total;
    double* datap;
    double* pipe;
    double* per_group;  // [P][k] or null
    int8_t* order;      // [P][k] or null
    int* invalid;       // count of malformed candidates
    // streamed batch (eval8 only, null otherwise): the layouts arrive while
    // the kernel runs, in chunks [0, c0), then c-sized ones; chunk i may be
    // read once (int32)(arrived[i] - epoch) >= 0; each warp adds the quads it
    // finished in chunk i to finished[i] (outputs fenced before)
    const uint32_t* arrived;
    uint32_t* finished;
    uint32_t epoch;
    int64_t c0, c;
};

struct EvalPlan {
    bool smem_tables, m8;
    int warps, blocks;
    size_t smem;
    // no order output: two-layer Held-Karp schedule, smaller scratch, more warps
    bool roll_smem_tables;
    int roll_warps;
    size_t roll_smem;
};


int launch_build_tables(int n, const double* lat, const double* bw, int d_dp, double dp_num, double pp_num,
                        double sw_num, double* dp, double* pp, double* sw, cudaStream_t s);
int launch_rank(int64_t nn, const double* pp, const double* vals, int nvals, uint32_t* rank, cudaStream_t s);
int eval_plan(const EvalArgs& a, int sm_count, size_t smem_optin, EvalPlan* plan);
int launch_eval(const EvalArgs& a, const EvalPlan& plan, cudaStream_t s);
// paper shape (8 x 8, N = 64, u16 keys, no stage order): four candidates per warp
bool eval8_applicable(const EvalArgs& a, size_t smem_optin);
int launch_eval8(const EvalArgs& a, int sm_count, cudaStream_t s);
int64_t eval8_wave(int sm_count);
int launch_bottleneck_batch(const double* w, int m, int64_t B, double* out, cudaStream_t s);
int launch_narrow(int64_t nn, const uint32_t* src, uint16_t* dst, cudaStream_t s);
int launch_path_batch(const double* w, int k, int64_t B, const HKTables& t, double* total, int8_t* order,
                      int sm_count, cudaStream_t s);

}  // namespace hs
