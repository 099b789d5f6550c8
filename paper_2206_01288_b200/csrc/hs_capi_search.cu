// hs_capi_search.cu -- C-ABI of the search kernels (include/hetsched_b200.h).
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "hs_big.h"
#include "hs_instance.h"
#include "hs_search.h"

using hsx::DeviceGuard;
using hsx::fail;

namespace {

hs::SearchShape shape_of(const hs_instance* h, int max_passes) {
    hs::SearchShape sh;
    sh.n = h->n;
    sh.k = h->k;
    sh.m = h->m;
    sh.max_passes = max_passes;
    sh.nvals = h->nvals;
    sh.key16 = h->rank16 != nullptr;
    sh.hk = h->hk;
    return sh;
}

const void* rank_of(const hs_instance* h) { return h->rank16 ? (const void*)h->rank16 : (const void*)h->rank; }

// Per-call device scratch from a stream-ordered pool of this library's own
// per device (allocated and freed on the legacy stream the calls use; the
// pool keeps the memory between calls -- a batch of 1,024 config-5
// partitions needs 400 MB of mean caches, which cudaMalloc / cudaFree would
// hand back and re-map every call).  The device's default pool, which other
// code in the process may use, is left alone.
constexpr int kMaxPoolDevices = 64;

cudaMemPool_t scratch_pool() {
    static std::mutex mu;
    static cudaMemPool_t pools[kMaxPoolDevices] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxPoolDevices) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool = nullptr;
        if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        pools[dev] = pool;
    }
    return pools[dev];
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, 0);
    }
    cudaError_t alloc(size_t n) {
        cudaMemPool_t pool = scratch_pool();
        if (!pool) return cudaErrorMemoryAllocation;
        return cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), std::max<size_t>(1, n) * sizeof(T), pool, 0);
    }
};

int check_search_shape(const hs_instance* h, int kind, int max_passes) {
    if (kind < 0 || kind > 2) return fail(-2, "kind must be 0 (ours), 1 (kl) or 2 (none)");
    if (max_passes < 1) return fail(-2, "max_passes must be >= 1");
    if (kind == 0 && h->k == 1 && h->m >= 2)
        return fail(-4, "zero-size array to reduction operation maximum which has no identity");
    if (h->n > 1024) return fail(-3, "search kernels support n <= 1024");
    if (h->k > 16) return fail(-3, "the device GA / local search cover d_pp <= 16");
    return 0;
}

}  // namespace

struct hs_ga {
    hs_instance* h = nullptr;
    hs_ga_config cfg{};
    int islands = 0;
    hs::SearchPlan plan{};
    hs::GAState* state = nullptr;
    int16_t* pop = nullptr;
    double* cost = nullptr;
    int16_t* best = nullptr;
    double* trace_best = nullptr;
    double* trace_mean = nullptr;
    double* out3 = nullptr;
    double* out_pg = nullptr;
    int8_t* out_order = nullptr;
    int16_t* out_groups = nullptr;
    double* hk_scratch = nullptr;
    long long* prof = nullptr;  // HS_GA_PROFILE=1: driver-phase cycle counters of island 0
    cudaStream_t last = nullptr;  // stream of the latest run / export / import (hs_ga_result syncs it)
    int spec = -1;                // speculative pipeline cluster size (0: off, -1: not probed yet)
    bool started = false;         // the population has been initialised by a launch
    // batch-priced generations (d_pp 9..16 on the cluster Held-Karp path):
    // every island's snapshots of a generation are priced in one batch
    bool batch = false;
    int snap_stride = 0;
    int host_gen = 0;             // generations run so far (islands advance in lockstep)
    int16_t* snap_buf = nullptr;
    double* snap_cost = nullptr;
    int* snap_cnt = nullptr;
    int32_t* invalid = nullptr;   // the batch pricer's count (padding slots count as malformed)
};

static hs::GAArgs ga_args(hs_ga* ga, int until, int finalize) {
    hs_instance* h = ga->h;
    hs::GAArgs a{};
    a.n = h->n;
    a.k = h->k;
    a.m = h->m;
    a.sw = h->sw;
    a.dp = h->dp;
    a.rank = rank_of(h);
    a.vals = h->vals;
    a.hk = h->hk;
    a.pop = ga->cfg.pop_size;
    a.generations = ga->cfg.generations;
    a.islands = ga->islands;
    a.kind = ga->cfg.kind;
    a.max_passes = ga->cfg.max_passes;
    a.patience = ga->cfg.patience;
    a.gen_end = until;
    a.finalize = finalize;
    a.state = ga->state;
    a.pop_buf = ga->pop;
    a.cost_buf = ga->cost;
    a.best_buf = ga->best;
    a.trace_best = ga->trace_best;
    a.trace_mean = ga->trace_mean;
    a.out3 = ga->out3;
    a.out_pg = ga->out_pg;
    a.out_order = ga->out_order;
    a.out_groups = ga->out_groups;
    a.hkb = h->hkb;
    a.hk_scratch = ga->hk_scratch;
    a.hk_size = h->k > 8 ? hs::hk_big_size(h->k) : 0;
    a.prof = ga->prof;
    return a;
}

extern "C" {

int hs_ga_create(hs_instance* h, const hs_ga_config* cfg, int islands, const hs_pcg64* rng, hs_ga** out) {
    return hs_ga_create_ex(h, cfg, islands, rng, 0, out);
}

int hs_ga_create_ex(hs_instance* h, const hs_ga_config* cfg, int islands, const hs_pcg64* rng, int mode,
                    hs_ga** out) {
    if (!h || !cfg || !rng || !out) return fail(-2, "null argument");
    if (islands < 1) return fail(-2, "islands must be >= 1");
    if (cfg->pop_size < 2) return fail(-2, "pop_size must be >= 2");
    if (cfg->pop_size > 256) return fail(-3, "pop_size > 256 is not supported");
    if (cfg->generations < 1) return fail(-2, "generations must be >= 1");
    int rc = check_search_shape(h, cfg->kind, cfg->max_passes);
    if (rc) return rc;
    DeviceGuard dg(h->device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    hs_ga* ga = new hs_ga();
    ga->h = h;
    ga->cfg = *cfg;
    ga->islands = islands;
    if (hs::search_plan(shape_of(h, cfg->max_passes), cfg->pop_size, h->smem_optin, &ga->plan, mode == 1)) {
        delete ga;
        return fail(-3, "GA working set does not fit shared memory");
    }
    const int km = h->k * h->m;
    std::vector<hs::GAState> st(islands);
    for (int i = 0; i < islands; i++) {
        st[i] = hs::GAState{};
        st[i].rng = rng[i];
    }
    CK(cudaMalloc(&ga->state, sizeof(hs::GAState) * islands), "cudaMalloc");
    CK(cudaMalloc(&ga->pop, (size_t)islands * cfg->pop_size * km * 2), "cudaMalloc");
    CK(cudaMalloc(&ga->cost, (size_t)islands * cfg->pop_size * 8), "cudaMalloc");
    CK(cudaMalloc(&ga->best, (size_t)islands * km * 2), "cudaMalloc");
    CK(cudaMalloc(&ga->trace_best, (size_t)islands * cfg->generations * 8), "cudaMalloc");
    CK(cudaMalloc(&ga->trace_mean, (size_t)islands * cfg->generations * 8), "cudaMalloc");
    CK(cudaMalloc(&ga->out3, (size_t)islands * 3 * 8), "cudaMalloc");
    CK(cudaMalloc(&ga->out_pg, (size_t)islands * h->k * 8), "cudaMalloc");
    CK(cudaMalloc(&ga->out_order, (size_t)islands * h->k), "cudaMalloc");
    CK(cudaMalloc(&ga->out_groups, (size_t)islands * km * 2), "cudaMalloc");
    if (h->k > 8) CK(cudaMalloc(&ga->hk_scratch, (size_t)islands * hs::hk_big_size(h->k) * 8), "cudaMalloc");
    // d_pp 9..16: a generation's snapshots (all islands) are priced together
    // by the stage + cluster Held-Karp kernels (HS_GA_BATCH=0: in-kernel CTA
    // pricing, one snapshot at a time)
    const char* benv = getenv("HS_GA_BATCH");
    if (h->k > 8 && h->two.rwords && !(benv && benv[0] == '0')) {
        ga->batch = true;
        ga->snap_stride = std::max(cfg->pop_size, 1 + cfg->max_passes);
        const size_t slots = (size_t)islands * ga->snap_stride;
        CK(cudaMalloc(&ga->snap_buf, slots * km * 2), "cudaMalloc");
        CK(cudaMalloc(&ga->snap_cost, slots * 8), "cudaMalloc");
        CK(cudaMalloc(&ga->snap_cnt, (size_t)islands * 4), "cudaMalloc");
        CK(cudaMalloc(&ga->invalid, 4), "cudaMalloc");
    }
    CK(cudaMemcpy(ga->state, st.data(), sizeof(hs::GAState) * islands, cudaMemcpyHostToDevice), "upload state");
    if (getenv("HS_GA_PROFILE")) {
        CK(cudaMalloc(&ga->prof, 16 * sizeof(long long)), "cudaMalloc");
        CK(cudaMemset(ga->prof, 0, 16 * sizeof(long long)), "memset");
    }
    *out = ga;
    return 0;
}

// One batch-priced step: phase 1 (snapshots out), the stage + cluster
// Held-Karp pricing of every island's slots, phase 2 (commit).
static int ga_batch_step(hs_ga* ga, int until, bool key16, cudaStream_t st) {
    hs::GAArgs a = ga_args(ga, until, 0);
    a.snap_stride = ga->snap_stride;
    a.snap_buf = ga->snap_buf;
    a.snap_cost = ga->snap_cost;
    a.snap_cnt = ga->snap_cnt;
    a.phase = 1;
    if (hs::launch_ga(a, ga->plan, ga->islands, key16, st)) return fail(-1, "ga emit launch", cudaGetLastError());
    const int64_t P = (int64_t)ga->islands * ga->snap_stride;
    if (int rc = hs_eval_batch(ga->h, ga->snap_buf, P, ga->snap_cost, nullptr, nullptr, nullptr, nullptr, ga->invalid,
                               st))
        return rc;
    a.phase = 2;
    if (hs::launch_ga(a, ga->plan, ga->islands, key16, st)) return fail(-1, "ga commit launch", cudaGetLastError());
    return 0;
}

int hs_ga_run(hs_ga* ga, int until, void* stream) {
    if (!ga) return fail(-2, "null handle");
    DeviceGuard dg(ga->h->device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    until = std::min(until, ga->cfg.generations);
    cudaStream_t st = (cudaStream_t)stream;
    const bool key16 = ga->h->rank16 != nullptr;
    if (ga->batch) {
        if (!ga->started)
            if (int rc = ga_batch_step(ga, 0, key16, st)) return rc;  // init_population + its pricing
        ga->started = true;
        for (; ga->host_gen < until; ga->host_gen++)
            if (int rc = ga_batch_step(ga, ga->host_gen + 1, key16, st)) return rc;
        if (until >= ga->cfg.generations) {  // canonical best of every island
            hs::GAArgs af = ga_args(ga, until, 1);
            if (hs::launch_ga(af, ga->plan, ga->islands, key16, st))
                return fail(-1, "ga finalize launch", cudaGetLastError());
        }
        ga->last = st;
        return 0;
    }
    if (ga->spec < 0) {
        // one GA: generations as a speculative pipeline over a thread-block
        // cluster (hs_search_ga_spec.cu); HS_GA_SPEC=0 keeps the one-CTA kernel
        const char* env = getenv("HS_GA_SPEC");
        const bool want = ga->islands == 1 && !ga->prof && !(env && env[0] == '0');
        ga->spec = want ? hs::ga_spec_cluster(ga_args(ga, until, 0), ga->plan, key16, ga->h->smem_optin) : 0;
        cudaGetLastError();
    }
    if (ga->spec > 1) {
        if (!ga->started) {  // init_population + pricing (no generation runs)
            hs::GAArgs a0 = ga_args(ga, 0, 0);
            if (hs::launch_ga(a0, ga->plan, 1, key16, st)) return fail(-1, "ga init launch", cudaGetLastError());
        }
        hs::GAArgs a = ga_args(ga, until, 0);
        if (hs::launch_ga_spec(a, ga->plan, ga->spec, key16, st))
            return fail(-1, "ga speculative launch", cudaGetLastError());
        if (until >= ga->cfg.generations) {  // finalize (no generation left to run)
            hs::GAArgs af = ga_args(ga, until, 1);
            if (hs::launch_ga(af, ga->plan, 1, key16, st)) return fail(-1, "ga finalize launch", cudaGetLastError());
        }
    } else {
        hs::GAArgs a = ga_args(ga, until, until >= ga->cfg.generations);
        if (hs::launch_ga(a, ga->plan, ga->islands, key16, st)) return fail(-1, "ga launch", cudaGetLastError());
    }
    ga->started = true;
    ga->last = st;
    return 0;
}

int hs_ga_export(hs_ga* ga, int elites, int16_t* groups, double* costs, void* stream) {
    if (!ga) return fail(-2, "null handle");
    if (elites < 1 || elites > ga->cfg.pop_size) return fail(-2, "elites must be in 1..pop_size");
    DeviceGuard dg(ga->h->device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    if (hs::launch_export(ga->islands, ga->cfg.pop_size, ga->h->k * ga->h->m, elites, ga->pop, ga->cost, groups, costs,
                          (cudaStream_t)stream))
        return fail(-1, "export launch", cudaGetLastError());
    ga->last = (cudaStream_t)stream;
    return 0;
}

int hs_ga_import(hs_ga* ga, int elites, const int16_t* groups, const double* costs, const int32_t* src, void* stream) {
    if (!ga) return fail(-2, "null handle");
    if (elites < 1 || elites > ga->cfg.pop_size) return fail(-2, "elites must be in 1..pop_size");
    DeviceGuard dg(ga->h->device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    if (hs::launch_import(ga->islands, ga->cfg.pop_size, ga->h->k * ga->h->m, elites, ga->pop, ga->cost, ga->best,
                          ga->state, groups, costs, src, (cudaStream_t)stream))
        return fail(-1, "import launch", cudaGetLastError());
    ga->last = (cudaStream_t)stream;
    return 0;
}

int hs_ga_result(hs_ga* ga, int16_t* best_groups, double* best3, double* best_per_group, int8_t* best_order,
                 double* trace_best, double* trace_mean, int32_t* trace_len, int64_t* evaluations, hs_pcg64* rng) {
    if (!ga) return fail(-2, "null handle");
    DeviceGuard dg(ga->h->device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    // the session's work may still be in flight on the caller's (possibly
    // non-blocking) stream: drain it before reading the island states
    CK(cudaStreamSynchronize(ga->last), "ga sync");
    std::vector<hs::GAState> st(ga->islands);
    CK(cudaMemcpy(st.data(), ga->state, sizeof(hs::GAState) * ga->islands, cudaMemcpyDeviceToHost), "download state");
    bool need = false;
    for (auto& x : st) {
        if (!x.stopped && x.gen < ga->cfg.generations)
            return fail(-2, "GA session not finished: run it to `generations` (hs_ga_run) before reading results");
        need |= !x.finalized;
    }
    if (need) {
        // islands stopped by patience before `generations` still price their
        // canonical best; no island runs further generations
        hs::GAArgs a = ga_args(ga, ga->cfg.generations, 1);
        if (hs::launch_ga(a, ga->plan, ga->islands, ga->h->rank16 != nullptr, ga->last))
            return fail(-1, "ga finalize", cudaGetLastError());
        CK(cudaStreamSynchronize(ga->last), "ga sync");
        CK(cudaMemcpy(st.data(), ga->state, sizeof(hs::GAState) * ga->islands, cudaMemcpyDeviceToHost), "download");
    }
    const int I = ga->islands, k = ga->h->k, km = k * ga->h->m, G = ga->cfg.generations;
    if (best_groups) CK(cudaMemcpy(best_groups, ga->out_groups, (size_t)I * km * 2, cudaMemcpyDeviceToHost), "D2H");
    if (best3) CK(cudaMemcpy(best3, ga->out3, (size_t)I * 3 * 8, cudaMemcpyDeviceToHost), "D2H");
    if (best_per_group) CK(cudaMemcpy(best_per_group, ga->out_pg, (size_t)I * k * 8, cudaMemcpyDeviceToHost), "D2H");
    if (best_order) CK(cudaMemcpy(best_order, ga->out_order, (size_t)I * k, cudaMemcpyDeviceToHost), "D2H");
    if (trace_best) CK(cudaMemcpy(trace_best, ga->trace_best, (size_t)I * G * 8, cudaMemcpyDeviceToHost), "D2H");
    if (trace_mean) CK(cudaMemcpy(trace_mean, ga->trace_mean, (size_t)I * G * 8, cudaMemcpyDeviceToHost), "D2H");
    if (ga->prof) {
        long long pv[16];
        CK(cudaMemcpy(pv, ga->prof, sizeof(pv), cudaMemcpyDeviceToHost), "D2H");
        fprintf(stderr,
                "[hs_ga_profile] cycles: crossover %lld sweep %lld chains %lld price %lld | chain rounds %lld "
                "(caches at start %lld) moves %lld (cache refresh %lld) | best_candidate %lld calls %lld cycles, "
                "swaps %lld, fast_edge computes %lld (%lld cycles)\n",
                pv[0], pv[1], pv[2], pv[3], pv[5], pv[4], pv[7], pv[6], pv[8], pv[12], pv[11], pv[10], pv[9]);
    }
    for (int i = 0; i < I; i++) {
        if (trace_len) trace_len[i] = st[i].gen;
        if (evaluations) evaluations[i] = st[i].evaluations;
        if (rng) rng[i] = st[i].rng;
    }
    return 0;
}

int hs_ga_destroy(hs_ga* ga) {
    if (!ga) return 0;
    DeviceGuard dg(ga->h->device);
    for (void* p : {(void*)ga->state, (void*)ga->pop, (void*)ga->cost, (void*)ga->best, (void*)ga->trace_best,
                    (void*)ga->trace_mean, (void*)ga->out3, (void*)ga->out_pg, (void*)ga->out_order,
                    (void*)ga->out_groups, (void*)ga->hk_scratch, (void*)ga->prof, (void*)ga->snap_buf,
                    (void*)ga->snap_cost, (void*)ga->snap_cnt, (void*)ga->invalid})
        if (p) cudaFree(p);
    delete ga;
    return 0;
}

static int refine_common(hs_instance* h, int kind, int max_passes, int single, int phase, int B,
                         const int16_t* groups, hs_pcg64* rng, int16_t* out, double* out_total, int32_t* evals,
                         int32_t* changed) {
    if (!h) return fail(-2, "null handle");
    if (B < 0) return fail(-2, "negative batch");
    if (B == 0) return 0;
    if (kind < 0 || kind > 1) return fail(-2, "kind must be 0 (ours) or 1 (kl)");
    int rc = check_search_shape(h, kind, max_passes);
    if (rc) return rc;
    DeviceGuard dg(h->device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    hs::SearchPlan plan;
    if (hs::search_plan(shape_of(h, max_passes), 2, h->smem_optin, &plan)) return fail(-3, "does not fit smem");
    const int km = h->k * h->m;
    DevBuf<int16_t> dg_in, dg_out;
    DevBuf<hs_pcg64> drng;
    DevBuf<double> dcost;
    DevBuf<int> dev, dch;
    DevBuf<double> hks;
    const char* benv = getenv("HS_GA_BATCH");
    // d_pp 9..16: every partition's snapshots priced in one batch through
    // the stage + cluster Held-Karp kernels (HS_GA_BATCH=0: in-kernel, one
    // 4.2 MB Held-Karp slice per partition)
    const bool batch = !single && h->k > 8 && h->two.rwords && !(benv && benv[0] == '0');
    if (h->k > 8 && !batch) CK(hks.alloc((size_t)B * hs::hk_big_size(h->k)), "cudaMalloc");
    CK(dg_in.alloc((size_t)B * km), "cudaMalloc");
    CK(dg_out.alloc((size_t)B * km), "cudaMalloc");
    CK(drng.alloc(B), "cudaMalloc");
    CK(dcost.alloc(B), "cudaMalloc");
    CK(dev.alloc(B), "cudaMalloc");
    CK(dch.alloc(B), "cudaMalloc");
    CK(cudaMemcpy(dg_in.p, groups, (size_t)B * km * 2, cudaMemcpyHostToDevice), "H2D");
    CK(cudaMemcpy(drng.p, rng, sizeof(hs_pcg64) * B, cudaMemcpyHostToDevice), "H2D");
    hs::RefineArgs a{};
    a.n = h->n;
    a.k = h->k;
    a.m = h->m;
    a.sw = h->sw;
    a.dp = h->dp;
    a.rank = rank_of(h);
    a.vals = h->vals;
    a.hk = h->hk;
    a.kind = kind;
    a.max_passes = max_passes;
    a.single_pass = single;
    a.phase = phase;
    a.groups = dg_in.p;
    a.rng = drng.p;
    a.out_groups = dg_out.p;
    a.out_cost = dcost.p;
    a.evaluations = dev.p;
    a.changed = dch.p;
    a.hkb = h->hkb;
    a.hk_scratch = hks.p;
    a.hk_size = h->k > 8 ? hs::hk_big_size(h->k) : 0;
    DevBuf<int16_t> dsnap;
    DevBuf<double> dscost;
    DevBuf<int> dscnt, dinv;
    if (batch) {
        a.snap_stride = 1 + max_passes;
        CK(dsnap.alloc((size_t)B * a.snap_stride * km), "cudaMalloc");
        CK(dscost.alloc((size_t)B * a.snap_stride), "cudaMalloc");
        CK(dscnt.alloc(B), "cudaMalloc");
        CK(dinv.alloc(1), "cudaMalloc");
        a.snap_buf = dsnap.p;
        a.snap_cnt = dscnt.p;
    }
    if (hs::launch_refine(a, plan, B, h->rank16 != nullptr, 0)) return fail(-1, "refine launch", cudaGetLastError());
    if (batch) {
        if (int rc2 = hs_eval_batch(h, dsnap.p, (int64_t)B * a.snap_stride, dscost.p, nullptr, nullptr, nullptr,
                                    nullptr, dinv.p, nullptr))
            return rc2;
        if (hs::launch_refine_commit(a, dscost.p, B, 0)) return fail(-1, "refine commit launch", cudaGetLastError());
    }
    CK(cudaDeviceSynchronize(), "refine");
    CK(cudaMemcpy(out, dg_out.p, (size_t)B * km * 2, cudaMemcpyDeviceToHost), "D2H");
    CK(cudaMemcpy(rng, drng.p, sizeof(hs_pcg64) * B, cudaMemcpyDeviceToHost), "D2H");
    if (out_total) CK(cudaMemcpy(out_total, dcost.p, (size_t)B * 8, cudaMemcpyDeviceToHost), "D2H");
    if (evals) CK(cudaMemcpy(evals, dev.p, (size_t)B * 4, cudaMemcpyDeviceToHost), "D2H");
    if (changed) CK(cudaMemcpy(changed, dch.p, (size_t)B * 4, cudaMemcpyDeviceToHost), "D2H");
    return 0;
}

int hs_local_search(hs_instance* h, int kind, int max_passes, int B, const int16_t* groups, hs_pcg64* rng,
                    int16_t* out, double* out_total, int32_t* evaluations) {
    return refine_common(h, kind, max_passes, 0, 0, B, groups, rng, out, out_total, evaluations, nullptr);
}

int hs_refine_pass(hs_instance* h, int kind, int phase, int B, const int16_t* groups, hs_pcg64* rng, int16_t* out,
                   int32_t* changed) {
    // one pass never prices, so any d_pp <= 32 works (config 5 gains-only stress)
    if (!h) return fail(-2, "null handle");
    if (B <= 0) return B == 0 ? 0 : fail(-2, "negative batch");
    if (kind < 0 || kind > 1) return fail(-2, "kind must be 0 (ours) or 1 (kl)");
    if (kind == 0 && h->k == 1 && h->m >= 2)
        return fail(-4, "zero-size array to reduction operation maximum which has no identity");
    if (h->k > 32 || h->m > 64) return fail(-3, "passes support d_pp <= 32, d_dp <= 64");
    DeviceGuard dg(h->device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    const int km = h->k * h->m;
    DevBuf<int16_t> gi, go;
    DevBuf<hs_pcg64> r;
    DevBuf<int> ch;
    DevBuf<double> mean;
    DevBuf<uint32_t> mver;
    CK(gi.alloc((size_t)B * km), "cudaMalloc");
    CK(go.alloc((size_t)B * km), "cudaMalloc");
    CK(r.alloc(B), "cudaMalloc");
    CK(ch.alloc(B), "cudaMalloc");
    CK(mean.alloc((size_t)B * h->n * h->k), "cudaMalloc");
    CK(mver.alloc((size_t)B * h->n * h->k), "cudaMalloc");
    CK(cudaMemcpy(gi.p, groups, (size_t)B * km * 2, cudaMemcpyHostToDevice), "H2D");
    CK(cudaMemcpy(r.p, rng, sizeof(hs_pcg64) * B, cudaMemcpyHostToDevice), "H2D");
    hs::PassArgs a{};
    a.n = h->n;
    a.k = h->k;
    a.m = h->m;
    a.kind = kind;
    a.phase = phase;
    a.sw = h->sw;
    a.groups = gi.p;
    a.rng = r.p;
    a.out_groups = go.p;
    a.changed = ch.p;
    a.mean = mean.p;
    a.mver = mver.p;
    if (hs::launch_pass(a, B, 0)) return fail(-1, "pass launch", cudaGetLastError());
    CK(cudaDeviceSynchronize(), "pass");
    CK(cudaMemcpy(out, go.p, (size_t)B * km * 2, cudaMemcpyDeviceToHost), "D2H");
    CK(cudaMemcpy(rng, r.p, sizeof(hs_pcg64) * B, cudaMemcpyDeviceToHost), "D2H");
    if (changed) CK(cudaMemcpy(changed, ch.p, (size_t)B * 4, cudaMemcpyDeviceToHost), "D2H");
    return 0;
}

int hs_crossover(int n, int d_pp, int d_dp, int device, int B, const int16_t* p1, const int16_t* p2, hs_pcg64* rng,
                 int16_t* out) {
    if (B <= 0) return B == 0 ? 0 : fail(-2, "negative batch");
    if (n != d_pp * d_dp || d_dp > 64 || n > 32767) return fail(-2, "bad shape");
    DeviceGuard dg(device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    const int km = n;
    DevBuf<int16_t> a1, a2, o;
    DevBuf<hs_pcg64> r;
    CK(a1.alloc((size_t)B * km), "cudaMalloc");
    CK(a2.alloc((size_t)B * km), "cudaMalloc");
    CK(o.alloc((size_t)B * km), "cudaMalloc");
    CK(r.alloc(B), "cudaMalloc");
    CK(cudaMemcpy(a1.p, p1, (size_t)B * km * 2, cudaMemcpyHostToDevice), "H2D");
    CK(cudaMemcpy(a2.p, p2, (size_t)B * km * 2, cudaMemcpyHostToDevice), "H2D");
    CK(cudaMemcpy(r.p, rng, sizeof(hs_pcg64) * B, cudaMemcpyHostToDevice), "H2D");
    if (hs::launch_crossover(n, d_pp, d_dp, a1.p, a2.p, r.p, o.p, B, 0)) return fail(-1, "crossover launch");
    CK(cudaDeviceSynchronize(), "crossover");
    CK(cudaMemcpy(out, o.p, (size_t)B * km * 2, cudaMemcpyDeviceToHost), "D2H");
    CK(cudaMemcpy(rng, r.p, sizeof(hs_pcg64) * B, cudaMemcpyDeviceToHost), "D2H");
    return 0;
}

int hs_gains(int n, int d_pp, int d_dp, int device, const double* sw, int kind, int B, const int16_t* groups,
             const int32_t* q, double* out) {
    if (B <= 0) return B == 0 ? 0 : fail(-2, "negative batch");
    if (n != d_pp * d_dp || d_dp > 64) return fail(-2, "bad shape");
    DeviceGuard dg(device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    DevBuf<int16_t> g;
    DevBuf<int32_t> dq;
    DevBuf<double> o, w;
    CK(g.alloc((size_t)B * n), "cudaMalloc");
    CK(dq.alloc((size_t)B * 6), "cudaMalloc");
    CK(o.alloc(B), "cudaMalloc");
    CK(w.alloc((size_t)n * n), "cudaMalloc");
    CK(cudaMemcpy(g.p, groups, (size_t)B * n * 2, cudaMemcpyHostToDevice), "H2D");
    CK(cudaMemcpy(dq.p, q, (size_t)B * 6 * 4, cudaMemcpyHostToDevice), "H2D");
    CK(cudaMemcpy(w.p, sw, (size_t)n * n * 8, cudaMemcpyHostToDevice), "H2D");
    if (hs::launch_gains(n, d_pp, d_dp, w.p, g.p, dq.p, kind, B, o.p, 0)) return fail(-1, "gains launch");
    CK(cudaMemcpy(out, o.p, (size_t)B * 8, cudaMemcpyDeviceToHost), "D2H");
    return 0;
}

int hs_random_partitions(int n, int d_pp, int d_dp, int device, int B, hs_pcg64* rng, int16_t* out) {
    if (B <= 0) return B == 0 ? 0 : fail(-2, "negative batch");
    if (n != d_pp * d_dp || n > 32767) return fail(-2, "bad shape");
    DeviceGuard dg(device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    DevBuf<int16_t> o;
    DevBuf<hs_pcg64> r;
    CK(o.alloc((size_t)B * n), "cudaMalloc");
    CK(r.alloc(1), "cudaMalloc");
    CK(cudaMemcpy(r.p, rng, sizeof(hs_pcg64), cudaMemcpyHostToDevice), "H2D");
    if (hs::launch_random_partitions(n, d_pp, d_dp, B, r.p, o.p, 0)) return fail(-1, "partitions launch");
    CK(cudaMemcpy(out, o.p, (size_t)B * n * 2, cudaMemcpyDeviceToHost), "D2H");
    CK(cudaMemcpy(rng, r.p, sizeof(hs_pcg64), cudaMemcpyDeviceToHost), "D2H");
    return 0;
}

}  // extern "C"
