// hs_capi.cu -- the C-ABI (include/hetsched_b200.h) over the sm_100a kernels.
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sort.h>
#include <thrust/unique.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hetsched_b200.h"
#include "hs_big.h"
#include "hs_eval.cuh"
#include <cuda.h>

#include "hs_instance.h"

namespace hsx {

thread_local std::string g_err;

int fail(int code, const char* what, cudaError_t e) {
    char buf[512];
    if (e != cudaSuccess)
        snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
    else
        snprintf(buf, sizeof buf, "%s", what);
    g_err = buf;
    return code;
}

int ensure_search_stack() {
    size_t stack = 0;
    CK(cudaDeviceGetLimit(&stack, cudaLimitStackSize), "cudaDeviceGetLimit");
    if (stack < 8192) CK(cudaDeviceSetLimit(cudaLimitStackSize, 8192), "cudaDeviceSetLimit");
    return 0;
}


// Held-Karp schedule for k <= 8 (see hs_eval.cuh, warp_held_karp): compact
// offsets off[s] (entries for |s| >= 2, s ascending), and per state (s, u)
// with r = s \ u the pre-decoded 16-byte word (byte offsets of h[r][.] and
// h[s][u], the byte offsets v*8 of r's members ascending, u*kES), grouped
// by layer |s|.
void hk_schedule(int k, std::vector<uint4>& st, std::vector<uint16_t>& hoff, int lay[18]) {
    st.clear();
    hoff.assign((size_t)1 << k, 0);
    int acc = 0;
    for (int s = 0; s < (1 << k); s++) {
        hoff[s] = (uint16_t)acc;
        if (__builtin_popcount(s) >= 2) acc += __builtin_popcount(s);
    }
    for (int i = 0; i < 18; i++) lay[i] = 0;
    // r-major within a layer: the k-|r| states sharing r = s \ u sit on
    // adjacent lanes and read the same h[r][.] row (smem broadcast).
    for (int p = 0; p < 18; p++) {
        lay[p] = (int)st.size();
        if (p < 2 || p > k) continue;
        for (int r = 0; r < (1 << k); r++) {
            if (__builtin_popcount(r) != p - 1) continue;
            for (int u = 0; u < k; u++) {
                if (r >> u & 1) continue;
                int s = r | (1 << u);
                uint32_t dst = hoff[s] + __builtin_popcount(s & ((1 << u) - 1));
                uint32_t offr = __builtin_popcount(r) >= 2 ? hoff[r] : 0;
                uint32_t vb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                int nv = 0;
                for (int v = 0; v < k; v++)
                    if (r >> v & 1) vb[nv++] = (uint32_t)v * 8;
                uint4 w;
                w.x = offr * 8 | (dst * 8) << 16;
                w.y = vb[0] | vb[1] << 8 | vb[2] << 16 | vb[3] << 24;
                w.z = vb[4] | vb[5] << 8 | vb[6] << 16 | ((uint32_t)u * hs::kES) << 24;
                w.w = (uint32_t)r | (uint32_t)u << 8;
                st.push_back(w);
            }
        }
    }
}

// Two-layer (ping-pong) variant: layer p's entries live in buffer p & 1 (each
// buffer as large as the widest layer), so h needs 2 * max_p C(k,p)*p
// doubles instead of k*2^(k-1) - k.  Same state words, offsets re-based; the
// compact table (and so order reconstruction) is not kept.
void hk_schedule_roll(int k, std::vector<uint4>& st, int lay[18], int* final_off, int* hsize) {
    st.clear();
    std::vector<uint32_t> loc((size_t)1 << k, 0), cnt(k + 1, 0);
    for (int s = 0; s < (1 << k); s++) {
        int p = __builtin_popcount(s);
        loc[s] = cnt[p] * p;
        cnt[p]++;
    }
    uint32_t S = 0;
    for (int p = 2; p <= k; p++) S = std::max<uint32_t>(S, cnt[p] * p);
    auto base = [&](int p) { return (p & 1) ? S : 0u; };
    for (int i = 0; i < 18; i++) lay[i] = 0;
    for (int p = 0; p < 18; p++) {
        lay[p] = (int)st.size();
        if (p < 2 || p > k) continue;
        for (int r = 0; r < (1 << k); r++) {
            if (__builtin_popcount(r) != p - 1) continue;
            for (int u = 0; u < k; u++) {
                if (r >> u & 1) continue;
                int s = r | (1 << u);
                uint32_t dst = base(p) + loc[s] + __builtin_popcount(s & ((1 << u) - 1));
                uint32_t offr = p - 1 >= 2 ? base(p - 1) + loc[r] : 0;
                uint32_t vb[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                int nv = 0;
                for (int v = 0; v < k; v++)
                    if (r >> v & 1) vb[nv++] = (uint32_t)v * 8;
                uint4 w;
                w.x = offr * 8 | (dst * 8) << 16;
                w.y = vb[0] | vb[1] << 8 | vb[2] << 16 | vb[3] << 24;
                w.z = vb[4] | vb[5] << 8 | vb[6] << 16 | ((uint32_t)u * hs::kES) << 24;
                w.w = (uint32_t)r | (uint32_t)u << 8;
                st.push_back(w);
            }
        }
    }
    *final_off = (int)base(k);
    *hsize = (int)(2 * S);
}

struct DeviceHK {
    uint4* st = nullptr;
    uint16_t* hoff = nullptr;
    hs::HKTables t{};
};

std::mutex g_hk_mu;
std::map<std::pair<int, int>, DeviceHK> g_hk;  // (device, k) compact; (device, -k) two-layer

int get_hk(int device, int k, hs::HKTables* out, bool roll) {
    std::lock_guard<std::mutex> lk(g_hk_mu);
    auto key = std::make_pair(device, roll ? -k : k);
    auto it = g_hk.find(key);
    if (it == g_hk.end()) {
        DeviceHK d;
        std::vector<uint4> st;
        std::vector<uint16_t> hoff;
        hk_schedule(k, st, hoff, d.t.lay);
        d.t.final_off = (k << (k - 1)) - 2 * k;
        d.t.hsize = (k << (k - 1)) - k;
        if (roll) hk_schedule_roll(k, st, d.t.lay, &d.t.final_off, &d.t.hsize);
        CK(cudaMalloc(&d.st, std::max<size_t>(16, st.size() * 16)), "cudaMalloc hk");
        CK(cudaMalloc(&d.hoff, hoff.size() * 2), "cudaMalloc hk");
        if (!st.empty()) CK(cudaMemcpy(d.st, st.data(), st.size() * 16, cudaMemcpyHostToDevice), "upload hk");
        CK(cudaMemcpy(d.hoff, hoff.data(), hoff.size() * 2, cudaMemcpyHostToDevice), "upload hk");
        d.t.states = d.st;
        d.t.nstates = (int)st.size();
        d.t.hoff = d.hoff;
        d.t.nhoff = (int)hoff.size();
        it = g_hk.emplace(key, d).first;
    }
    *out = it->second.t;
    return 0;
}

// 9 <= k <= 16: same layout as hk_schedule with 64-bit words
struct DeviceHKBig {
    uint64_t* st = nullptr;
    uint32_t* off = nullptr;
    hs::HKBig t{};
};
std::map<std::pair<int, int>, DeviceHKBig> g_hkb;

int get_hk_big(int device, int k, hs::HKBig* out) {
    std::lock_guard<std::mutex> lk(g_hk_mu);
    auto key = std::make_pair(device, k);
    auto it = g_hkb.find(key);
    if (it == g_hkb.end()) {
        DeviceHKBig d;
        std::vector<uint32_t> off((size_t)1 << k, 0);
        uint32_t acc = 0;
        for (int s = 0; s < (1 << k); s++) {
            off[s] = acc;
            if (__builtin_popcount(s) >= 2) acc += __builtin_popcount(s);
        }
        std::vector<uint64_t> st;
        for (int p = 0; p < 18; p++) {
            d.t.lay[p] = (int)st.size();
            if (p < 2 || p > k) continue;
            for (int r = 0; r < (1 << k); r++) {
                if (__builtin_popcount(r) != p - 1) continue;
                for (int u = 0; u < k; u++) {
                    if (r >> u & 1) continue;
                    int s = r | (1 << u);
                    uint64_t dst = off[s] + __builtin_popcount(s & ((1 << u) - 1));
                    uint64_t offr = __builtin_popcount(r) >= 2 ? off[r] : 0;
                    st.push_back(offr | (dst << 20) | ((uint64_t)u << 40) | ((uint64_t)r << 44));
                }
            }
        }
        CK(cudaMalloc(&d.st, std::max<size_t>(8, st.size() * 8)), "cudaMalloc hkb");
        CK(cudaMalloc(&d.off, off.size() * 4), "cudaMalloc hkb");
        if (!st.empty()) CK(cudaMemcpy(d.st, st.data(), st.size() * 8, cudaMemcpyHostToDevice), "upload hkb");
        CK(cudaMemcpy(d.off, off.data(), off.size() * 4, cudaMemcpyHostToDevice), "upload hkb");
        d.t.states = d.st;
        d.t.nstates = (int)st.size();
        d.t.off = d.off;
        d.t.noff = (int)off.size();
        it = g_hkb.emplace(key, d).first;
    }
    *out = it->second.t;
    return 0;
}

}  // namespace hsx

using hsx::fail;
using hsx::get_hk;
using hsx::get_hk_big;
using hsx::DeviceGuard;
using hsx::g_err;

static hs::EvalArgs base_args(const hs_instance* h) {
    hs::EvalArgs a{};
    a.n = h->n;
    a.k = h->k;
    a.m = h->m;
    a.dp = h->dp;
    a.key16 = h->rank16 != nullptr;
    a.rank = a.key16 ? (const void*)h->rank16 : (const void*)h->rank;
    a.nvals = h->nvals;
    a.vals = h->vals;
    a.hk = h->hk;
    a.hk_roll = h->hk_roll;
    return a;
}

// ---- per-call scratch (hs_scratch, hs_instance.h) ---------------------------

static void scratch_free(hs_scratch* x) {
    for (int i = 0; i < 2; i++) {
        if (x->two_E[i]) cudaFree(x->two_E[i]);
        if (x->two_dp[i]) cudaFree(x->two_dp[i]);
        if (x->two_bad[i]) cudaFree(x->two_bad[i]);
        if (x->ev_stage[i]) cudaEventDestroy(x->ev_stage[i]);
        if (x->ev_hk[i]) cudaEventDestroy(x->ev_hk[i]);
    }
    if (x->side) cudaStreamDestroy(x->side);
    if (x->ev_in) cudaEventDestroy(x->ev_in);
    if (x->big) cudaFree(x->big);
    if (x->heur_E) cudaFree(x->heur_E);
    if (x->done) cudaEventDestroy(x->done);
    delete x;
}

// Take a set for one call on stream s: a free one (s waits until its last
// user's work is done) or a new one.
static int scratch_acquire(hs_instance* h, cudaStream_t s, hs_scratch** out) {
    hs_scratch* x = nullptr;
    {
        std::lock_guard<std::mutex> lk(h->pool_mu);
        if (!h->pool_free.empty()) {
            x = h->pool_free.back();
            h->pool_free.pop_back();
        }
    }
    if (!x) {
        x = new hs_scratch();
        cudaError_t e = cudaEventCreateWithFlags(&x->done, cudaEventDisableTiming);
        if (e != cudaSuccess) {
            delete x;
            return hsx::fail(-1, "event", e);
        }
        std::lock_guard<std::mutex> lk(h->pool_mu);
        h->pool_all.push_back(x);
    }
    if (x->used) {
        cudaError_t e = cudaStreamWaitEvent(s, x->done, 0);
        if (e != cudaSuccess) {
            std::lock_guard<std::mutex> lk(h->pool_mu);
            h->pool_free.push_back(x);
            return hsx::fail(-1, "wait", e);
        }
    }
    *out = x;
    return 0;
}

// Hand the set back once every use of it is enqueued on s (work on the
// side stream is joined into s before this).
static int scratch_release(hs_instance* h, hs_scratch* x, cudaStream_t s, int rc) {
    cudaError_t e = cudaEventRecord(x->done, s);
    x->used = true;
    {
        std::lock_guard<std::mutex> lk(h->pool_mu);
        h->pool_free.push_back(x);
    }
    if (!rc && e != cudaSuccess) return hsx::fail(-1, "event", e);
    return rc;
}

// d_pp 9..16 without stage order: chunks of stage kernel -> cluster Held-Karp.
// The stage kernel of chunk c+1 runs on the set's side stream while the
// Held-Karp kernel of chunk c runs on `s` (the stage CTAs fit beside the
// cluster CTAs' shared memory); ping-pong stage buffers, event-ordered.
static int launch_two(hs_instance* h, const hs::EvalArgs& a, hs_scratch* x, cudaStream_t s) {
    const bool m8 = a.key16 && a.m == 8;
    if (!x->two_E[0]) {
        for (int i = 0; i < 2; i++) {
            CK(cudaMalloc(&x->two_E[i], (size_t)h->two_chunk * hs::kStageStride * 8), "cudaMalloc stage graphs");
            CK(cudaMalloc(&x->two_dp[i], (size_t)h->two_chunk * 8), "cudaMalloc stage datap");
            CK(cudaMalloc(&x->two_bad[i], (size_t)h->two_chunk), "cudaMalloc stage flags");
            CK(cudaEventCreateWithFlags(&x->ev_stage[i], cudaEventDisableTiming), "event");
            CK(cudaEventCreateWithFlags(&x->ev_hk[i], cudaEventDisableTiming), "event");
        }
        CK(cudaStreamCreateWithFlags(&x->side, cudaStreamNonBlocking), "stream");
        CK(cudaEventCreateWithFlags(&x->ev_in, cudaEventDisableTiming), "event");
    }
    CK(cudaEventRecord(x->ev_in, s), "event");  // inputs produced on s before this call
    CK(cudaStreamWaitEvent(x->side, x->ev_in, 0), "wait");
    int64_t c = 0;
    for (int64_t lo = 0; lo < a.P; lo += h->two_chunk, c++) {
        const int i = (int)(c & 1);
        const int64_t cnt = std::min<int64_t>(h->two_chunk, a.P - lo);
        hs::EvalArgs ca = a;
        ca.groups = a.groups + lo * a.k * a.m;
        ca.P = cnt;
        ca.datap = a.datap ? a.datap + lo : nullptr;
        ca.per_group = a.per_group ? a.per_group + lo * a.k : nullptr;
        if (c >= 2) CK(cudaStreamWaitEvent(x->side, x->ev_hk[i], 0), "wait");  // buffer i is free again
        if (hs::launch_stage(ca, x->two_E[i], x->two_dp[i], x->two_bad[i], h->stage_blocks, m8, x->side))
            return hsx::fail(-1, "stage launch", cudaGetLastError());
        CK(cudaEventRecord(x->ev_stage[i], x->side), "event");
        CK(cudaStreamWaitEvent(s, x->ev_stage[i], 0), "wait");
        if (hs::launch_hk_cluster(x->two_E[i], hs::kStageES, hs::kStageStride, a.k, cnt, h->two, h->two_grid,
                                  x->two_dp[i], x->two_bad[i], a.total + lo, a.pipe ? a.pipe + lo : nullptr, s))
            return hsx::fail(-1, "cluster Held-Karp launch", cudaGetLastError());
        CK(cudaEventRecord(x->ev_hk[i], s), "event");
    }
    return 0;
}

static int launch_cta(hs_instance* h, const hs::EvalArgs& a, hs_scratch* x, cudaStream_t s) {
    if (!x->big) CK(cudaMalloc(&x->big, (size_t)h->big_blocks * hs::hk_big_size(h->k) * 8), "cudaMalloc scratch");
    return hs::launch_eval_cta(a, h->hkb, x->big, h->big_blocks, a.key16 && a.m == 8, s);
}

static int launch_heur(hs_instance* h, const hs::EvalArgs& a, hs_scratch* x, cudaStream_t s) {
    if (!x->heur_E) CK(cudaMalloc(&x->heur_E, (size_t)h->big_blocks * h->k * h->k * 8), "cudaMalloc heuristic E");
    if (hs::launch_eval_heur(a, x->heur_E, h->big_blocks, s)) return hsx::fail(-1, "heuristic eval launch");
    return 0;
}

static int launch_any(hs_instance* h, const hs::EvalArgs& a, cudaStream_t s) {
    if (h->k > 16) return hsx::fail(-3, "exact pricing is limited to d_pp <= 16 (Held-Karp); use heuristic paths");
    if (h->k <= hs::kWarpK) {  // no per-call scratch
        const int rc = hs::eval8_applicable(a, h->smem_optin) ? hs::launch_eval8(a, h->sm_count, s)
                                                               : hs::launch_eval(a, h->plan, s);
        return rc ? hsx::fail(-1, "eval launch", cudaGetLastError()) : 0;
    }
    hs_scratch* x = nullptr;
    int rc = scratch_acquire(h, s, &x);
    if (rc) return rc;
    if (!a.order && h->two.rwords) {
        rc = launch_two(h, a, x, s);
    } else {
        rc = launch_cta(h, a, x, s);
        if (rc > 0 || (rc < 0 && hsx::g_err.empty())) rc = hsx::fail(-1, "eval launch", cudaGetLastError());
    }
    return scratch_release(h, x, s, rc);
}

// Tables and schedules of a new handle; any error leaves partial state for
// hs_instance_destroy to free.
static int instance_init(hs_instance* h, const double* lat, const double* bw, double dp_num, double pp_num,
                         double sw_num) {
    const int n = h->n, d_pp = h->k, d_dp = h->m;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, h->device), "cudaGetDeviceProperties");
    h->sm_count = prop.multiProcessorCount;
    h->smem_optin = prop.sharedMemPerBlockOptin;
    size_t nn = (size_t)n * n;
    CK(cudaMalloc(&h->lat, nn * 8), "cudaMalloc");
    CK(cudaMalloc(&h->bw, nn * 8), "cudaMalloc");
    CK(cudaMalloc(&h->dp, nn * 8), "cudaMalloc");
    CK(cudaMalloc(&h->pp, nn * 8), "cudaMalloc");
    CK(cudaMalloc(&h->sw, nn * 8), "cudaMalloc");
    CK(cudaMalloc(&h->vals, nn * 8), "cudaMalloc");
    CK(cudaMalloc(&h->rank, nn * 4), "cudaMalloc");
    CK(cudaMalloc(&h->invalid, sizeof(int)), "cudaMalloc");
    CK(cudaMemcpy(h->lat, lat, nn * 8, cudaMemcpyHostToDevice), "upload lat");
    CK(cudaMemcpy(h->bw, bw, nn * 8, cudaMemcpyHostToDevice), "upload bw");
    if (hs::launch_build_tables(n, h->lat, h->bw, d_dp, dp_num, pp_num, sw_num, h->dp, h->pp, h->sw, 0))
        return fail(-1, "build_tables launch");
    CK(cudaMemcpy(h->vals, h->pp, nn * 8, cudaMemcpyDeviceToDevice), "copy pp");
    thrust::device_ptr<double> v(h->vals);
    thrust::sort(thrust::device, v, v + nn);
    h->nvals = (int)(thrust::unique(thrust::device, v, v + nn) - v);
    if (hs::launch_rank((int64_t)nn, h->pp, h->vals, h->nvals, h->rank, 0)) return fail(-1, "rank launch");
    if (h->nvals <= 0xFFFF) {
        CK(cudaMalloc(&h->rank16, nn * 2), "cudaMalloc");
        if (hs::launch_narrow((int64_t)nn, h->rank, h->rank16, 0)) return fail(-1, "narrow launch");
    }
    CK(cudaDeviceSynchronize(), "instance tables");
    int rc = get_hk(h->device, std::min(d_pp, (int)hs::kWarpK), &h->hk, false);
    if (!rc) rc = get_hk(h->device, std::min(d_pp, (int)hs::kWarpK), &h->hk_roll, true);
    if (rc) return rc;
    if (d_pp > 16) {
        // exact pricing is limited to 16 stages (combinatorics.py:243-249);
        // such instances serve the heuristic and pass-only entry points
        h->big_blocks = 2 * h->sm_count;
    } else if (d_pp > hs::kWarpK) {
        rc = get_hk_big(h->device, d_pp, &h->hkb);
        if (rc) return rc;
        h->big_blocks = hs::big_blocks(h->sm_count, d_pp);
        if (!hs::get_hk_two(h->device, d_pp, &h->two)) {
            h->two_grid = hs::cluster_grid(h->two, h->sm_count);
            h->stage_blocks = h->sm_count * 16;
            h->two_chunk = getenv("HS_TWO_CHUNK") ? std::max(64, atoi(getenv("HS_TWO_CHUNK"))) : 1024;
        }
    } else {
        hs::EvalArgs a = base_args(h);
        if (hs::eval_plan(a, h->sm_count, h->smem_optin, &h->plan)) return fail(-3, "shape does not fit shared memory");
    }
    return 0;
}


extern "C" {

int hs_version(void) { return 1; }

const char* hs_last_error(void) { return g_err.c_str(); }

int hs_instance_create(const double* lat, const double* bw, int n, int d_pp, int d_dp, double dp_num,
                       double pp_num, double sw_num, int device, hs_instance** out) {
    if (!out || !lat || !bw) return fail(-2, "null argument");
    if (n < 1 || d_pp < 1 || d_dp < 1 || (int64_t)d_pp * d_dp != n) return fail(-2, "d_pp*d_dp must equal n");
    if (d_dp > hs::kMaxM) return fail(-3, "d_dp > 64 is not supported");
    if (d_pp > 64) return fail(-3, "d_pp > 64 is not supported");
    if (n > 32767) return fail(-3, "n > 32767 is not supported (int16 device ids)");
    DeviceGuard dg(device);
    hs_instance* h = new hs_instance();
    h->device = device;
    h->n = n;
    h->k = d_pp;
    h->m = d_dp;
    const int rc = instance_init(h, lat, bw, dp_num, pp_num, sw_num);
    if (rc) {  // free whatever the partial init allocated
        const std::string err = g_err;
        hs_instance_destroy(h);
        g_err = err;
        return rc;
    }
    *out = h;
    return 0;
}

int hs_instance_destroy(hs_instance* h) {
    if (!h) return 0;
    DeviceGuard dg(h->device);
    cudaFree(h->lat);
    cudaFree(h->bw);
    cudaFree(h->dp);
    cudaFree(h->pp);
    cudaFree(h->sw);
    cudaFree(h->vals);
    cudaFree(h->rank);
    if (h->rank16) cudaFree(h->rank16);
    for (hs_scratch* x : h->pool_all) scratch_free(x);
    cudaFree(h->invalid);
    for (int i = 0; i < 2; i++) {
        if (h->cg[i]) cudaFree(h->cg[i]);
        if (h->co[i]) cudaFree(h->co[i]);
        if (h->cs[i]) cudaStreamDestroy(h->cs[i]);
    }
    if (h->cup) cudaStreamDestroy(h->cup);
    if (h->cdown) cudaStreamDestroy(h->cdown);
    for (cudaEvent_t e : h->ev_in) cudaEventDestroy(e);
    for (cudaEvent_t e : h->ev_out) cudaEventDestroy(e);
    if (h->cinv) cudaFree(h->cinv);
    if (h->arrived) cudaFree(h->arrived);
    if (h->finished) cudaFree(h->finished);
    delete h;
    return 0;
}

int hs_instance_tables(hs_instance* h, double* dp, double* pp, double* sw) {
    if (!h) return fail(-2, "null handle");
    DeviceGuard dg(h->device);
    size_t nn = (size_t)h->n * h->n * 8;
    if (dp) CK(cudaMemcpy(dp, h->dp, nn, cudaMemcpyDeviceToHost), "download dp");
    if (pp) CK(cudaMemcpy(pp, h->pp, nn, cudaMemcpyDeviceToHost), "download pp");
    if (sw) CK(cudaMemcpy(sw, h->sw, nn, cudaMemcpyDeviceToHost), "download sw");
    return 0;
}

int hs_eval_batch(hs_instance* h, const int16_t* groups, int64_t P, double* total, double* datap,
                  double* pipelinep, double* per_group, int8_t* order, int32_t* invalid, void* stream) {
    if (!h) return fail(-2, "null handle");
    if (P < 0) return fail(-2, "negative batch");
    if (P == 0) return 0;
    if (!groups || !total) return fail(-2, "null buffer");
    DeviceGuard dg(h->device);
    hs::EvalArgs a = base_args(h);
    a.groups = groups;
    a.P = P;
    a.total = total;
    a.datap = datap;
    a.pipe = pipelinep;
    a.per_group = per_group;
    a.order = order;
    a.invalid = invalid ? invalid : h->invalid;
    int rc = launch_any(h, a, (cudaStream_t)stream);
    if (rc) return rc;
    return 0;
}

int hs_eval_batch_ex(hs_instance* h, const int16_t* groups, int64_t P, double* total, double* datap, double* pipelinep,
                     double* per_group, int8_t* order, int32_t* invalid, int heuristic, void* stream) {
    if (!h) return fail(-2, "null handle");
    if (h->k <= 16 || !heuristic)
        return hs_eval_batch(h, groups, P, total, datap, pipelinep, per_group, order, invalid, stream);
    if (P < 0) return fail(-2, "negative batch");
    if (P == 0) return 0;
    DeviceGuard dg(h->device);
    hs::EvalArgs a = base_args(h);
    a.groups = groups;
    a.P = P;
    a.total = total;
    a.datap = datap;
    a.pipe = pipelinep;
    a.per_group = per_group;
    a.order = order;
    a.invalid = invalid ? invalid : h->invalid;
    cudaStream_t s = (cudaStream_t)stream;
    hs_scratch* x = nullptr;
    int rc = scratch_acquire(h, s, &x);
    if (rc) return rc;
    return scratch_release(h, x, s, launch_heur(h, a, x, s));
}

int hs_path_heuristic_batch(const double* w, int k, int64_t B, double* total, int8_t* order, int device, void* stream) {
    if (k < 2 || k > 64) return fail(-3, "heuristic path: k must be in 2..64");
    if (B <= 0) return B == 0 ? 0 : fail(-2, "negative batch");
    DeviceGuard dg(device);
    int8_t* scratch = nullptr;
    CK(cudaMalloc(&scratch, (size_t)B * 2 * k), "cudaMalloc");
    int rc = hs::launch_path_heuristic(w, k, B, total, order, scratch, (cudaStream_t)stream);
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    cudaFree(scratch);
    if (rc || e != cudaSuccess) return fail(-1, "heuristic path launch", e);
    return 0;
}

// cuStreamWriteValue32 / cuStreamWaitValue32 through the runtime's driver
// entry points (no link-time libcuda dependency); null if unavailable
namespace {
using PFN_val32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct StreamMemOps {
    PFN_val32 write = nullptr, wait = nullptr;
};
const StreamMemOps& stream_mem_ops() {
    static StreamMemOps ops = [] {
        StreamMemOps o;
        cudaDriverEntryPointQueryResult q1{}, q2{};
        void *w = nullptr, *t = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
            cudaGetDriverEntryPoint("cuStreamWaitValue32", &t, cudaEnableDefault, &q2) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
            o.write = reinterpret_cast<PFN_val32>(w);
            o.wait = reinterpret_cast<PFN_val32>(t);
        }
        cudaGetLastError();
        return o;
    }();
    return ops;
}
}  // namespace

static int host_batch(hs_instance* h, const int16_t* groups, int64_t P, double* total, double* datap,
                      double* pipelinep, double* per_group, int8_t* order, int32_t* invalid) {
    const int km = h->k * h->m;
    // Decoupled pipeline over a span of up to 2^22 layouts held on the
    // device: all H2D chunk copies back to back on one copy stream (the host
    // link never waits for a kernel), D2H copies on a third stream.  Streamed
    // (eval8, 8x8 at N = 64): ONE kernel per span consumes the chunks as the
    // copy stream announces them (cuStreamWriteValue32 behind each H2D) and
    // counts finished quads per chunk, which the D2H stream waits on
    // (cuStreamWaitValue32).  Otherwise one launch per chunk on alternating
    // compute streams (a launch backfills the previous one's tail), ordered
    // by events.
    constexpr int64_t kSpan = (int64_t)1 << 22;
    if (!h->chunk) {
        h->chunk = 1 << 16;  // layouts per kernel launch (measured best for e2e: 2^14..2^20 swept)
        if (const char* e = getenv("HS_HOST_CHUNK_LOG2")) h->chunk = (int64_t)1 << std::max(10, std::min(24, atoi(e)));
        hs::EvalArgs probe = base_args(h);
        probe.groups = nullptr;  // 16-byte aligned by construction (cudaMalloc)
        if (hs::eval8_applicable(probe, h->smem_optin)) {
            // whole waves of the eval8 kernel per launch: every warp gets the
            // same number of quads, no half-empty last iteration
            const int64_t wave = hs::eval8_wave(h->sm_count);
            h->chunk = std::max<int64_t>(1, (h->chunk + wave / 2) / wave) * wave;
        }
        // streamed path: one kernel per span, so the chunk only sets the
        // grain of the copy / announce / D2H pipeline (measured best 2^15 of
        // 2^13..2^17: 2.88e8 e2e at P = 2^20)
        h->schunk = (int64_t)1 << 15;
        if (const char* e = getenv("HS_HOST_CHUNK_LOG2")) h->schunk = (int64_t)1 << std::max(10, std::min(24, atoi(e)));
        for (int i = 0; i < 2; i++) CK(cudaStreamCreateWithFlags(&h->cs[i], cudaStreamNonBlocking), "stream");
        CK(cudaStreamCreateWithFlags(&h->cup, cudaStreamNonBlocking), "stream");
        CK(cudaStreamCreateWithFlags(&h->cdown, cudaStreamNonBlocking), "stream");
        CK(cudaMalloc(&h->cinv, sizeof(int)), "cudaMalloc");
    }
    const int64_t span = std::min<int64_t>(P, kSpan);
    if (span > h->span) {
        if (h->cg[0]) cudaFree(h->cg[0]);
        if (h->co[0]) cudaFree(h->co[0]);
        h->cg[0] = nullptr;
        h->co[0] = nullptr;
        h->span = 0;
        CK(cudaMalloc(&h->cg[0], (size_t)span * km * 2), "cudaMalloc host-path inputs");
        CK(cudaMalloc(&h->co[0], (size_t)span * (3 + h->k) * 8 + (size_t)span * h->k), "cudaMalloc host-path outputs");
        h->span = span;
    }
    const StreamMemOps& ops = stream_mem_ops();
    hs::EvalArgs probe8 = base_args(h);
    probe8.groups = h->cg[0];
    const char* senv = getenv("HS_HOST_STREAMED");
    const bool streamed = ops.write && ops.wait && !order && hs::eval8_applicable(probe8, h->smem_optin) &&
                          !(senv && senv[0] == '0');
    const int64_t chunk = streamed ? h->schunk : h->chunk;
    const int64_t nch_max = (span + chunk - 1) / chunk + 2;  // chunks per span (first and last small)
    while ((int64_t)h->ev_in.size() < nch_max) {
        cudaEvent_t e1, e2;
        CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming), "event");
        CK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming), "event");
        h->ev_in.push_back(e1);
        h->ev_out.push_back(e2);
    }
    if (streamed && h->nslots < nch_max) {
        if (h->arrived) cudaFree(h->arrived);
        if (h->finished) cudaFree(h->finished);
        h->arrived = nullptr;
        h->finished = nullptr;
        h->nslots = 0;
        CK(cudaMalloc(&h->arrived, (size_t)nch_max * 4), "cudaMalloc");
        CK(cudaMalloc(&h->finished, (size_t)nch_max * 4), "cudaMalloc");
        CK(cudaMemset(h->arrived, 0, (size_t)nch_max * 4), "memset");
        CK(cudaMemset(h->finished, 0, (size_t)nch_max * 4), "memset");
        h->fin_target.assign((size_t)nch_max, 0u);
        h->epoch = 0;
        h->nslots = nch_max;
    }
    CK(cudaMemsetAsync(h->cinv, 0, sizeof(int), h->cup), "memset");
    hs::EvalArgs a = base_args(h);
    a.invalid = h->cinv;
    const int64_t S = h->span;
    double* const o_total = h->co[0];
    double* const o_datap = o_total + S;
    double* const o_pipe = o_total + 2 * S;
    double* const o_pg = o_total + 3 * S;
    int8_t* const o_order = reinterpret_cast<int8_t*>(o_total + (3 + h->k) * S);
    for (int64_t base = 0; base < P; base += S) {
        const int64_t n = std::min<int64_t>(S, P - base);
        if (base) CK(cudaStreamSynchronize(h->cdown), "sync");  // the span's buffers are free again
        // chunk plan: a small first chunk (short exposed H2D), a small last
        // one (short exposed D2H), full chunks between
        std::vector<std::pair<int64_t, int64_t>> ch;
        for (int64_t lo = 0; lo < n;) {
            const int64_t small = std::max<int64_t>(4, chunk / 8 / 4 * 4), left = n - lo;
            int64_t cnt = ch.empty() ? small : chunk;
            if (!streamed && !ch.empty() && left > small && left <= chunk + small) cnt = left - small;
            cnt = std::min<int64_t>(cnt, left);
            ch.emplace_back(lo, cnt);
            lo += cnt;
        }
        if (streamed) {
            // one kernel for the span: chunk c is announced by a value write
            // behind its H2D copy, its D2H waits for the kernel's count of
            // finished quads (no per-chunk launches, no tails between them)
            // the kernel is enqueued first: it waits for its chunks on the GPU
            const uint32_t ep = ++h->epoch;
            a.groups = h->cg[0];
            a.P = n;
            a.total = o_total;
            a.datap = o_datap;
            a.pipe = o_pipe;
            a.per_group = per_group ? o_pg : nullptr;
            a.order = nullptr;
            a.arrived = h->arrived;
            a.finished = h->finished;
            a.epoch = ep;
            a.c0 = ch[0].second;
            a.c = chunk;
            if (int rc = launch_any(h, a, h->cs[0])) return rc;
            a.arrived = nullptr;
            a.finished = nullptr;
            for (size_t c = 0; c < ch.size(); c++) {
                const int64_t lo = ch[c].first, cnt = ch[c].second;
                CK(cudaMemcpyAsync(h->cg[0] + lo * km, groups + (base + lo) * km, (size_t)cnt * km * 2,
                                   cudaMemcpyHostToDevice, h->cup), "H2D");
                if (ops.write(h->cup, (CUdeviceptr)(h->arrived + c), ep, 0) != CUDA_SUCCESS)
                    return fail(-1, "cuStreamWriteValue32");
            }
            for (size_t c = 0; c < ch.size(); c++) {
                const int64_t lo = ch[c].first, cnt = ch[c].second, g = base + lo;
                cudaStream_t s = h->cdown;
                h->fin_target[c] += (uint32_t)((cnt + 3) / 4);
                if (ops.wait(s, (CUdeviceptr)(h->finished + c), h->fin_target[c], CU_STREAM_WAIT_VALUE_GEQ) !=
                    CUDA_SUCCESS)
                    return fail(-1, "cuStreamWaitValue32");
                CK(cudaMemcpyAsync(total + g, o_total + lo, (size_t)cnt * 8, cudaMemcpyDeviceToHost, s), "D2H");
                if (datap) CK(cudaMemcpyAsync(datap + g, o_datap + lo, (size_t)cnt * 8, cudaMemcpyDeviceToHost, s), "D2H");
                if (pipelinep)
                    CK(cudaMemcpyAsync(pipelinep + g, o_pipe + lo, (size_t)cnt * 8, cudaMemcpyDeviceToHost, s), "D2H");
                if (per_group)
                    CK(cudaMemcpyAsync(per_group + g * h->k, o_pg + lo * h->k, (size_t)cnt * h->k * 8,
                                       cudaMemcpyDeviceToHost, s), "D2H");
            }
            continue;
        }
        for (size_t c = 0; c < ch.size(); c++) {
            const int64_t lo = ch[c].first, cnt = ch[c].second;
            CK(cudaMemcpyAsync(h->cg[0] + lo * km, groups + (base + lo) * km, (size_t)cnt * km * 2,
                               cudaMemcpyHostToDevice, h->cup), "H2D");
            CK(cudaEventRecord(h->ev_in[c], h->cup), "event");
        }
        for (size_t c = 0; c < ch.size(); c++) {
            const int64_t lo = ch[c].first, cnt = ch[c].second;
            cudaStream_t s = h->cs[c & 1];
            CK(cudaStreamWaitEvent(s, h->ev_in[c], 0), "wait");
            a.groups = h->cg[0] + lo * km;
            a.P = cnt;
            a.total = o_total + lo;
            a.datap = o_datap + lo;
            a.pipe = o_pipe + lo;
            a.per_group = per_group ? o_pg + lo * h->k : nullptr;
            a.order = order ? o_order + lo * h->k : nullptr;
            int rc = launch_any(h, a, s);
            if (rc) return rc;
            CK(cudaEventRecord(h->ev_out[c], s), "event");
        }
        for (size_t c = 0; c < ch.size(); c++) {
            const int64_t lo = ch[c].first, cnt = ch[c].second, g = base + lo;
            cudaStream_t s = h->cdown;
            CK(cudaStreamWaitEvent(s, h->ev_out[c], 0), "wait");
            CK(cudaMemcpyAsync(total + g, o_total + lo, (size_t)cnt * 8, cudaMemcpyDeviceToHost, s), "D2H");
            if (datap) CK(cudaMemcpyAsync(datap + g, o_datap + lo, (size_t)cnt * 8, cudaMemcpyDeviceToHost, s), "D2H");
            if (pipelinep)
                CK(cudaMemcpyAsync(pipelinep + g, o_pipe + lo, (size_t)cnt * 8, cudaMemcpyDeviceToHost, s), "D2H");
            if (per_group)
                CK(cudaMemcpyAsync(per_group + g * h->k, o_pg + lo * h->k, (size_t)cnt * h->k * 8,
                                   cudaMemcpyDeviceToHost, s), "D2H");
            if (order)
                CK(cudaMemcpyAsync(order + g * h->k, o_order + lo * h->k, (size_t)cnt * h->k, cudaMemcpyDeviceToHost, s),
                   "D2H");
        }
    }
    CK(cudaStreamSynchronize(h->cdown), "sync");
    CK(cudaStreamSynchronize(h->cs[0]), "sync");
    CK(cudaStreamSynchronize(h->cs[1]), "sync");
    if (invalid) CK(cudaMemcpy(invalid, h->cinv, sizeof(int), cudaMemcpyDeviceToHost), "D2H invalid");
    return 0;
}

int hs_eval_batch_host(hs_instance* h, const int16_t* groups, int64_t P, double* total, double* datap,
                       double* pipelinep, double* per_group, int8_t* order, int32_t* invalid) {
    if (!h) return fail(-2, "null handle");
    if (P < 0) return fail(-2, "negative batch");
    if (invalid) *invalid = 0;
    if (P == 0) return 0;
    std::lock_guard<std::mutex> lk(h->mu);
    DeviceGuard dg(h->device);
    const int rc = host_batch(h, groups, P, total, datap, pipelinep, per_group, order, invalid);
    if (rc) {  // nothing of a failed call may still run into the next one's buffers
        for (cudaStream_t s : {h->cup, h->cs[0], h->cs[1], h->cdown})
            if (s) cudaStreamSynchronize(s);
        // the streamed kernel counts every chunk it finished, also those
        // whose D2H wait was never enqueued: restart from the device counts
        if (h->finished && h->nslots &&
            cudaMemcpy(h->fin_target.data(), h->finished, (size_t)h->nslots * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
            h->nslots = 0;  // unknown counts: the next streamed call reallocates and zeroes them
        cudaGetLastError();
    }
    return rc;
}

int hs_bottleneck_batch(const double* w, int m, int64_t B, double* out, int device, void* stream) {
    if (m < 1 || m > hs::kMaxM) return fail(-3, "bottleneck: m must be in 1..64");
    DeviceGuard dg(device);
    if (hs::launch_bottleneck_batch(w, m, B, out, (cudaStream_t)stream))
        return fail(-1, "bottleneck launch", cudaGetLastError());
    return 0;
}

int hs_path_batch(const double* w, int k, int64_t B, double* total, int8_t* order, int device, void* stream) {
    if (k < 1 || k > 16) return fail(-3, "path: k must be in 1..16");
    DeviceGuard dg(device);
    if (k == 1) {
        // a single vertex: empty path (combinatorics.py:241-242)
        std::vector<double> z((size_t)B, 0.0);
        std::vector<int8_t> o((size_t)B, 0);
        CK(cudaMemcpyAsync(total, z.data(), (size_t)B * 8, cudaMemcpyHostToDevice, (cudaStream_t)stream), "H2D");
        if (order) CK(cudaMemcpyAsync(order, o.data(), (size_t)B, cudaMemcpyHostToDevice, (cudaStream_t)stream), "H2D");
        CK(cudaStreamSynchronize((cudaStream_t)stream), "sync");
        return 0;
    }
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device), "props");
    if (k > hs::kWarpK) {
        hs::HKBig t;
        int rc = get_hk_big(device, k, &t);
        if (rc) return rc;
        int blocks = (int)std::min<int64_t>(B, hs::big_blocks(prop.multiProcessorCount, k));
        double* scratch = nullptr;
        CK(cudaMalloc(&scratch, (size_t)std::max(blocks, 1) * hs::hk_big_size(k) * 8), "cudaMalloc scratch");
        int lrc = hs::launch_path_cta(w, k, B, t, scratch, blocks, total, order, (cudaStream_t)stream);
        cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
        cudaFree(scratch);
        if (lrc || e != cudaSuccess) return fail(-1, "path launch", e);
        return 0;
    }
    hs::HKTables t;
    int rc = get_hk(device, k, &t);
    if (rc) return rc;
    if (hs::launch_path_batch(w, k, B, t, total, order, prop.multiProcessorCount, (cudaStream_t)stream))
        return fail(-1, "path launch", cudaGetLastError());
    return 0;
}

}  // extern "C"
