// hs_instance.h -- the C-ABI handle and shared host helpers.
#pragma once
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hetsched_b200.h"
#include "hs_cluster.h"
#include "hs_internal.h"

namespace hsx {

int fail(int code, const char* what, cudaError_t e = cudaSuccess);
int get_hk(int device, int k, hs::HKTables* out, bool roll = false);
int get_hk_big(int device, int k, hs::HKBig* out);
// The search / assignment kernels' call chains (GA driver -> crossover /
// passes -> warp evaluator) need more than the default 1 KiB per-thread
// stack: raise the current device's limit to 8 KiB if it is lower (a
// process-wide setting; documented in include/hetsched_b200.h).
int ensure_search_stack();

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace hsx

#define CK(call, what)                                              \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return hsx::fail(-1, what, e_);      \
    } while (0)

// Per-call device scratch of the d_pp > 8 eval paths.  A call takes a set
// from the handle's pool (a new one when every set is in use), so calls on
// different streams never share buffers; a set handed back records `done`
// on the call's stream and its next user waits on that event before
// touching the buffers (HS C-ABI re-entrancy).
struct hs_scratch {
    double* two_E[2] = {};        // stage graphs, ping-pong (stage + cluster Held-Karp)
    double* two_dp[2] = {};
    uint8_t* two_bad[2] = {};
    cudaStream_t side = nullptr;  // stage kernels beside the Held-Karp kernel
    cudaEvent_t ev_stage[2] = {}, ev_hk[2] = {}, ev_in = nullptr;
    double* big = nullptr;        // per-CTA Held-Karp slices (eval_cta_kernel, stage order wanted)
    double* heur_E = nullptr;     // d_pp > 16: per-CTA stage graphs of the heuristic path
    cudaEvent_t done = nullptr;   // recorded on the last user's stream
    bool used = false;
};

struct hs_instance {
    int device = 0, n = 0, k = 0, m = 0, sm_count = 0;
    size_t smem_optin = 0;
    double *lat = nullptr, *bw = nullptr, *dp = nullptr, *pp = nullptr, *sw = nullptr, *vals = nullptr;
    uint32_t* rank = nullptr;
    uint16_t* rank16 = nullptr;
    int nvals = 0;
    hs::HKTables hk{};
    hs::HKTables hk_roll{};        // two-layer schedule: batch pricing without stage order
    hs::HKBig hkb{};               // d_pp > 8: CTA evaluator schedule
    int big_blocks = 0;
    // d_pp 9..16 without stage order: stage kernel + cluster Held-Karp (hs_cluster.cu)
    hs::HKTwo two{};
    int two_grid = 0, stage_blocks = 0;
    int64_t two_chunk = 0;
    // scratch pool (hs_scratch above)
    std::mutex pool_mu;
    std::vector<hs_scratch*> pool_all, pool_free;
    int* invalid = nullptr;
    hs::EvalPlan plan{};
    // host-buffer path
    std::mutex mu;
    int64_t chunk = 0;   // layouts per kernel launch (chunked path)
    int64_t schunk = 0;  // layouts per announced chunk (streamed path)
    int64_t span = 0;                 // layouts the host-path device buffers hold
    int16_t* cg[2] = {nullptr, nullptr};  // [0]: inputs of a span (cg[1] unused)
    double* co[2] = {nullptr, nullptr};   // [0]: outputs of a span (co[1] unused)
    int* cinv = nullptr;
    cudaStream_t cs[2] = {nullptr, nullptr};  // compute (alternating: a launch backfills the previous one's tail)
    cudaStream_t cup = nullptr, cdown = nullptr;  // H2D / D2H copy streams
    std::vector<cudaEvent_t> ev_in, ev_out;       // per chunk: inputs landed / outputs written
    // streamed batches (eval8): one kernel per span consumes chunks as the
    // copy stream's value writes announce them (epoch), and counts finished
    // quads per chunk for the D2H stream's value waits
    uint32_t* arrived = nullptr;
    uint32_t* finished = nullptr;
    std::vector<uint32_t> fin_target;
    int64_t nslots = 0;
    uint32_t epoch = 0;
};

