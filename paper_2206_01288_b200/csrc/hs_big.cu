// hs_big.cu -- batch pricing and exact path search for 9 <= d_pp <= 16:
// one CTA per candidate (hs_cta_eval.cuh), persistent grid, each CTA owning
// a slice of the global Held-Karp scratch.
#include <algorithm>

#include "hs_big.h"
#include "hs_cta_eval.cuh"

namespace hs {

template <typename KeyT, bool kM8>
__global__ void __launch_bounds__(256) eval_cta_kernel(EvalArgs a, HKBig t, double* scratch, size_t hk_size) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int k = a.k, m = kM8 ? 8 : a.m, km = k * m;
    CtaScratch cs = cta_scratch_at(smem, k, m);
    size_t off = cta_scratch_bytes(k, m);
    int16_t* mem = reinterpret_cast<int16_t*>(smem + off);
    off += ((size_t)km * 2 + 15) & ~(size_t)15;
    uint32_t* seen = reinterpret_cast<uint32_t*>(smem + off);
    __shared__ int bad;
    double* h = scratch + (size_t)blockIdx.x * hk_size;
    const KeyT* RK = reinterpret_cast<const KeyT*>(a.rank);
    const int nwords = (a.n + 31) >> 5;
    for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
        const int16_t* gsrc = a.groups + p * km;
        for (int i = threadIdx.x; i < km; i += blockDim.x) mem[i] = gsrc[i];
        for (int i = threadIdx.x; i < nwords; i += blockDim.x) seen[i] = 0;
        if (threadIdx.x == 0) bad = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < km; i += blockDim.x) {
            int d = mem[i];
            if (d < 0 || d >= a.n || (i % m != 0 && mem[i - 1] >= d))
                bad = 1;
            else
                atomicOr(&seen[d >> 5], 1u << (d & 31));
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nwords; i += blockDim.x) {
            int bits = min(32, a.n - i * 32);
            uint32_t want = bits == 32 ? 0xffffffffu : ((1u << bits) - 1u);
            if (seen[i] != want) bad = 1;
        }
        __syncthreads();
        if (bad) {
            if (threadIdx.x == 0) {
                const double nan = __longlong_as_double(0x7ff8000000000000LL);
                a.total[p] = nan;
                if (a.datap) a.datap[p] = nan;
                if (a.pipe) a.pipe[p] = nan;
                atomicAdd(a.invalid, 1);
            }
            __syncthreads();
            continue;
        }
        double datap, pipe;
        cta_price<KeyT, kM8>(a.n, k, m, a.dp, RK, a.vals, t, cs, h, mem, datap, pipe);
        if (threadIdx.x == 0) {
            a.total[p] = datap + pipe;
            if (a.datap) a.datap[p] = datap;
            if (a.pipe) a.pipe[p] = pipe;
            if (a.order) held_karp_order_big(k, cs.E, h, t.off, pipe, a.order + p * k);
        }
        if (a.per_group && threadIdx.x < k) a.per_group[p * k + threadIdx.x] = cs.pg[threadIdx.x];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) path_cta_kernel(const double* __restrict__ w, int k, int64_t B, HKBig t,
                                                        double* scratch, size_t hk_size, double* __restrict__ total,
                                                        int8_t* __restrict__ order) {
    __shared__ double E[16 * kES16];
    __shared__ double red[2];
    double* h = scratch + (size_t)blockIdx.x * hk_size;
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        const double* src = w + b * k * k;
        for (int i = threadIdx.x; i < k * k; i += blockDim.x) E[(i / k) * kES16 + (i % k)] = src[i];
        __syncthreads();
        double tt = cta_held_karp(k, E, h, t, red);
        if (threadIdx.x == 0) {
            total[b] = tt;
            if (order) held_karp_order_big(k, E, h, t.off, tt, order + b * k);
        }
        __syncthreads();
    }
}

size_t hk_big_size(int k) { return ((size_t)k << (k - 1)) - (size_t)k; }

int big_blocks(int sm_count, int k) {
    size_t per = hk_big_size(k) * 8;
    int per_sm = per <= (256u << 10) ? 8 : 2;
    return sm_count * per_sm;
}

template <typename KT, bool M8>
static void launch_cta_t(const EvalArgs& a, const HKBig& t, double* scratch, int blocks, cudaStream_t s) {
    size_t smem = cta_scratch_bytes(a.k, M8 ? 8 : a.m) + (((size_t)a.k * a.m * 2 + 15) & ~(size_t)15) + 32 * 4 * 4;
    cudaFuncSetAttribute(eval_cta_kernel<KT, M8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    eval_cta_kernel<KT, M8><<<blocks, 256, smem, s>>>(a, t, scratch, hk_big_size(a.k));
}

int launch_eval_cta(const EvalArgs& a, const HKBig& t, double* scratch, int blocks, bool m8, cudaStream_t s) {
    if (a.P == 0) return 0;
    blocks = (int)std::min<int64_t>(blocks, a.P);
    if (m8)
        launch_cta_t<uint16_t, true>(a, t, scratch, blocks, s);
    else if (a.key16)
        launch_cta_t<uint16_t, false>(a, t, scratch, blocks, s);
    else
        launch_cta_t<uint32_t, false>(a, t, scratch, blocks, s);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_path_cta(const double* w, int k, int64_t B, const HKBig& t, double* scratch, int blocks, double* total,
                    int8_t* order, cudaStream_t s) {
    if (B == 0) return 0;
    blocks = (int)std::min<int64_t>(blocks, B);
    path_cta_kernel<<<blocks, 256, 0, s>>>(w, k, B, t, scratch, hk_big_size(k), total, order);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace hs

namespace hs {

// open_loop_tsp(heuristic=True), one thread per matrix (any k <= 64)
__global__ void path_heuristic_kernel(const double* __restrict__ w, int k, int64_t B, double* __restrict__ total,
                                      int8_t* __restrict__ order, int8_t* __restrict__ scratch) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;
    int8_t* best = scratch + b * 2 * k;
    int8_t* o = best + k;
    total[b] = nn_two_opt(w + b * k * k, k, k, best, o);
    if (order)
        for (int i = 0; i < k; i++) order[b * k + i] = best[i];
}

int launch_path_heuristic(const double* w, int k, int64_t B, double* total, int8_t* order, int8_t* scratch,
                          cudaStream_t s) {
    if (B == 0) return 0;
    path_heuristic_kernel<<<(unsigned)((B + 63) / 64), 64, 0, s>>>(w, k, B, total, order, scratch);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// comm_cost(heuristic=True) for 16 < d_pp <= 64: one CTA per candidate,
// datap rows and bottleneck edges in parallel, heuristic path on thread 0.
template <typename KeyT>
__global__ void __launch_bounds__(256) eval_heur_kernel(EvalArgs a, double* Ebuf) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int k = a.k, m = a.m, km = k * m, n = a.n, es = k;
    double* rows = reinterpret_cast<double*>(smem);
    double* pg = rows + km;
    int16_t* mem = reinterpret_cast<int16_t*>(pg + 64);
    int8_t* ord = reinterpret_cast<int8_t*>(mem + km + 8);
    double* E = Ebuf + (size_t)blockIdx.x * k * k;
    const KeyT* RK = reinterpret_cast<const KeyT*>(a.rank);
    for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
        for (int i = threadIdx.x; i < km; i += blockDim.x) mem[i] = a.groups[p * km + i];
        __syncthreads();
        for (int r = threadIdx.x; r < km; r += blockDim.x) {
            int g = r / m;
            const int16_t* gm = mem + g * m;
            const double* row = a.dp + (size_t)gm[r - g * m] * n;
            rows[r] = pairwise_sum(m, [&](int c) { return row[gm[c]]; });
        }
        __syncthreads();
        if (threadIdx.x < k) {
            double mx = rows[threadIdx.x * m];
            for (int i = 1; i < m; i++) mx = dmax(mx, rows[threadIdx.x * m + i]);
            pg[threadIdx.x] = mx;
        }
        const int npairs = k * (k - 1) / 2;
        for (int t = threadIdx.x; t < npairs; t += blockDim.x) {
            int j, j2;
            decode_pair(t, k, j, j2);
            const int16_t* A = mem + j * m;
            const int16_t* Bg = mem + j2 * m;
            uint32_t L = bottleneck_threshold<uint32_t>(
                m, [&](int r, int c) { return (uint32_t)RK[(size_t)A[r] * n + Bg[c]]; }, 0xffffffffu);
            double v = a.vals[L];
            E[j * es + j2] = v;
            E[j2 * es + j] = v;
        }
        if (threadIdx.x < k) E[threadIdx.x * es + threadIdx.x] = 0.0;
        __syncthreads();
        if (threadIdx.x == 0) {
            double pipe = nn_two_opt(E, es, k, ord, ord + 64);
            double dp = pg[0];
            for (int g = 1; g < k; g++) dp = dmax(dp, pg[g]);
            a.total[p] = dp + pipe;
            if (a.datap) a.datap[p] = dp;
            if (a.pipe) a.pipe[p] = pipe;
            if (a.order)
                for (int i = 0; i < k; i++) a.order[p * k + i] = ord[i];
        }
        if (a.per_group && threadIdx.x < k) a.per_group[p * k + threadIdx.x] = pg[threadIdx.x];
        __syncthreads();
    }
}

int launch_eval_heur(const EvalArgs& a, double* Ebuf, int blocks, cudaStream_t s) {
    if (a.P == 0) return 0;
    blocks = (int)std::min<int64_t>(blocks, a.P);
    size_t smem = (size_t)a.k * a.m * 8 + 64 * 8 + ((size_t)a.k * a.m + 8) * 2 + 160;
    if (a.key16) {
        cudaFuncSetAttribute(eval_heur_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        eval_heur_kernel<uint16_t><<<blocks, 256, smem, s>>>(a, Ebuf);
    } else {
        cudaFuncSetAttribute(eval_heur_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        eval_heur_kernel<uint32_t><<<blocks, 256, smem, s>>>(a, Ebuf);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace hs
