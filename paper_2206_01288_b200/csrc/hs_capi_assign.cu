// hs_capi_assign.cu -- C-ABI of the fixed-layout kernels.
#include <algorithm>

#include "hs_assign.h"
#include "hs_instance.h"

using hsx::DeviceGuard;
using hsx::fail;

namespace {
template <typename T>
struct Buf {
    T* p = nullptr;
    ~Buf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t n) { return cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)); }
};
}  // namespace

extern "C" {

int hs_materialize(hs_instance* h, int64_t B, const int16_t* groups, int16_t* grid, int8_t* order) {
    if (!h) return fail(-2, "null handle");
    if (B <= 0) return B == 0 ? 0 : fail(-2, "negative batch");
    if (h->k > 8) return fail(-3, "GPU materialize covers d_pp <= 8");
    DeviceGuard dg(h->device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    const int km = h->k * h->m;
    Buf<int16_t> g, gr;
    Buf<int8_t> od;
    CK(g.alloc((size_t)B * km), "cudaMalloc");
    CK(gr.alloc((size_t)B * km), "cudaMalloc");
    CK(od.alloc((size_t)B * h->k), "cudaMalloc");
    CK(cudaMemcpy(g.p, groups, (size_t)B * km * 2, cudaMemcpyHostToDevice), "H2D");
    hs::MaterializeArgs a{};
    a.n = h->n;
    a.k = h->k;
    a.m = h->m;
    a.nvals = h->nvals;
    a.key16 = h->rank16 != nullptr;
    a.dp = h->dp;
    a.rank = a.key16 ? (const void*)h->rank16 : (const void*)h->rank;
    a.vals = h->vals;
    a.hk = h->hk;
    a.groups = g.p;
    a.B = B;
    a.grid = gr.p;
    a.order = od.p;
    if (hs::launch_materialize(a, h->sm_count, 0)) return fail(-1, "materialize launch", cudaGetLastError());
    CK(cudaDeviceSynchronize(), "materialize");
    CK(cudaMemcpy(grid, gr.p, (size_t)B * km * 2, cudaMemcpyDeviceToHost), "D2H");
    CK(cudaMemcpy(order, od.p, (size_t)B * h->k, cudaMemcpyDeviceToHost), "D2H");
    return 0;
}

int hs_evaluate_assignments(hs_instance* h, int64_t B, const int16_t* grids, double* out3, double* per_col) {
    if (!h) return fail(-2, "null handle");
    if (B <= 0) return B == 0 ? 0 : fail(-2, "negative batch");
    if (h->k > 16) return fail(-3, "d_pp > 16");
    DeviceGuard dg(h->device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    const int km = h->k * h->m;
    Buf<int16_t> g;
    Buf<double> o, pc;
    CK(g.alloc((size_t)B * km), "cudaMalloc");
    CK(o.alloc((size_t)B * 3), "cudaMalloc");
    CK(pc.alloc((size_t)B * h->k), "cudaMalloc");
    CK(cudaMemcpy(g.p, grids, (size_t)B * km * 2, cudaMemcpyHostToDevice), "H2D");
    if (hs::launch_evaluate(h->n, h->k, h->m, h->dp, h->pp, g.p, B, o.p, per_col ? pc.p : nullptr, h->sm_count, 0))
        return fail(-1, "evaluate launch", cudaGetLastError());
    CK(cudaDeviceSynchronize(), "evaluate");
    CK(cudaMemcpy(out3, o.p, (size_t)B * 3 * 8, cudaMemcpyDeviceToHost), "D2H");
    if (per_col) CK(cudaMemcpy(per_col, pc.p, (size_t)B * h->k * 8, cudaMemcpyDeviceToHost), "D2H");
    return 0;
}

int hs_random_assignments(int n, int d_pp, int d_dp, int device, int B, hs_pcg64* rng, int16_t* grids, int8_t* orders) {
    if (B <= 0) return B == 0 ? 0 : fail(-2, "negative batch");
    if (n != d_pp * d_dp || n > 32767 || d_pp > 64) return fail(-2, "bad shape");
    DeviceGuard dg(device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    Buf<hs_pcg64> r;
    Buf<int16_t> sc, gr;
    Buf<int8_t> od;
    CK(r.alloc(B), "cudaMalloc");
    CK(sc.alloc((size_t)B * n), "cudaMalloc");
    CK(gr.alloc((size_t)B * n), "cudaMalloc");
    CK(od.alloc((size_t)B * d_pp), "cudaMalloc");
    CK(cudaMemcpy(r.p, rng, sizeof(hs_pcg64) * B, cudaMemcpyHostToDevice), "H2D");
    if (hs::launch_random_assign(n, d_pp, d_dp, B, r.p, sc.p, gr.p, od.p, 0)) return fail(-1, "random launch");
    CK(cudaDeviceSynchronize(), "random");
    CK(cudaMemcpy(grids, gr.p, (size_t)B * n * 2, cudaMemcpyDeviceToHost), "D2H");
    CK(cudaMemcpy(orders, od.p, (size_t)B * d_pp, cudaMemcpyDeviceToHost), "D2H");
    CK(cudaMemcpy(rng, r.p, sizeof(hs_pcg64) * B, cudaMemcpyDeviceToHost), "D2H");
    return 0;
}

int hs_bottleneck_match_batch(const double* w, int m, int64_t B, double* value, int8_t* pairs, int device,
                              void* stream) {
    if (m < 1 || m > 64) return fail(-3, "bottleneck matching: m must be in 1..64");
    if (B < 0) return fail(-2, "negative batch");
    if (B && (!w || !value)) return fail(-2, "null argument");
    DeviceGuard dg(device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    if (hs::launch_bottleneck_match(w, m, B, value, pairs, (cudaStream_t)stream))
        return fail(-1, "bottleneck matching launch", cudaGetLastError());
    return 0;
}

int hs_datap_group_batch(const double* lat, const double* bw, int m, int64_t G, double ddp, double dp_num, double* out,
                         int device, void* stream) {
    if (m < 1 || m > 128) return fail(-3, "datap group: m must be in 1..128");
    if (G < 0) return fail(-2, "negative batch");
    if (G && (!lat || !bw || !out)) return fail(-2, "null argument");
    DeviceGuard dg(device);
    if (int rc_ = hsx::ensure_search_stack()) return rc_;
    if (hs::launch_datap_group(lat, bw, m, G, ddp, dp_num, out, (cudaStream_t)stream))
        return fail(-1, "datap group launch", cudaGetLastError());
    return 0;
}

}  // extern "C"
