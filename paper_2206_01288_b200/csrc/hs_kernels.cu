// hs_kernels.cu -- sm_100a kernels for the hetsched fitness hot path.
//
//   K0 build_tables_kernel : DP / PP / SW pair tables (costmodel.py:134-141,
//                            scheduler.py:84-88), exact op order, no FMA.
//   rank_kernel            : order-preserving rank of every PP entry among the
//                            distinct PP values, so bottleneck searches compare
//                            uint32 keys; the winning key maps back to the exact
//                            double the reference returns (an entry of w).
//   K1 eval_warp_kernel    : one warp per candidate layout (comm_cost,
//                            costmodel.py:217-229): datap (pairwise row sums,
//                            max), C(k,2) bottleneck matchings (one lane each),
//                            Held-Karp over the coarsened graph (warp, smem).
//                            Persistent grid, pair tables staged in smem.
//   bottleneck_batch / path_batch : the public single-matrix solvers
//                            (combinatorics.py:128-131,232-251) over a batch.
#include "hs_eval.cuh"
#include "hs_internal.h"

#include <algorithm>

namespace hs {

__global__ void build_tables_kernel(int n, const double* __restrict__ lat, const double* __restrict__ bw,
                                    double ddp, double dp_num, double pp_num, double sw_num,
                                    double* __restrict__ dp, double* __restrict__ pp, double* __restrict__ sw) {
    int64_t nn = (int64_t)n * n;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nn; x += (int64_t)gridDim.x * blockDim.x) {
        int i = (int)(x / n), j = (int)(x - (int64_t)i * n);
        double l = lat[x], b = bw[x];
        dp[x] = (i == j) ? 0.0 : 2.0 * (l + dp_num / (ddp * b));
        pp[x] = 2.0 * (l + pp_num / b);
        sw[x] = (i == j) ? 0.0 : l + sw_num / b;
    }
}

__global__ void rank_kernel(int64_t nn, const double* __restrict__ pp, const double* __restrict__ vals, int nvals,
                            uint32_t* __restrict__ rank) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nn; x += (int64_t)gridDim.x * blockDim.x) {
        double v = pp[x];
        int lo = 0, hi = nvals - 1;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (vals[mid] < v)
                lo = mid + 1;
            else
                hi = mid;
        }
        rank[x] = (uint32_t)lo;
    }
}

__device__ __forceinline__ void decode_pair(int t, int k, int& j, int& j2) {
    j = 0;
    while (t >= k - 1 - j) {
        t -= k - 1 - j;
        j++;
    }
    j2 = j + 1 + t;
}

struct WarpLayout {
    int h_off, e_off, pg_off, mem_off, seen_off, bytes;
};

template <bool kSmemTables>
__global__ void __launch_bounds__(512) eval_warp_kernel(EvalArgs a, WarpLayout wl) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int n = a.n, k = a.k, m = a.m, km = k * m;
    size_t off = 0;
    uint16_t* st = reinterpret_cast<uint16_t*>(smem);
    off += (size_t)((a.nstates * 2 + 15) & ~15);
    int* soff = reinterpret_cast<int*>(smem + off);
    off += 96;
    const double* DP;
    const uint32_t* RK;
    if (kSmemTables) {
        double* sdp = reinterpret_cast<double*>(smem + off);
        off += (size_t)n * n * 8;
        uint32_t* srk = reinterpret_cast<uint32_t*>(smem + off);
        off += ((size_t)n * n * 4 + 15) & ~(size_t)15;
        for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
            sdp[i] = a.dp[i];
            srk[i] = a.rank[i];
        }
        DP = sdp;
        RK = srk;
    } else {
        DP = a.dp;
        RK = a.rank;
    }
    for (int i = threadIdx.x; i < a.nstates; i += blockDim.x) st[i] = a.states[i];
    if (threadIdx.x < 18) soff[threadIdx.x] = a.off[threadIdx.x];
    unsigned char* wbase = smem + off + (size_t)wid * wl.bytes;
    double* h = reinterpret_cast<double*>(wbase + wl.h_off);
    double* E = reinterpret_cast<double*>(wbase + wl.e_off);
    double* pg = reinterpret_cast<double*>(wbase + wl.pg_off);
    int16_t* mem = reinterpret_cast<int16_t*>(wbase + wl.mem_off);
    uint32_t* seen = reinterpret_cast<uint32_t*>(wbase + wl.seen_off);
    __syncthreads();

    const int nwords = (n + 31) >> 5;
    const int npairs = k * (k - 1) / 2;
    for (int64_t p = (int64_t)blockIdx.x * W + wid; p < a.P; p += (int64_t)gridDim.x * W) {
        const int16_t* gsrc = a.groups + p * km;
        for (int i = lane; i < km; i += kWarp) mem[i] = gsrc[i];
        for (int i = lane; i < nwords; i += kWarp) seen[i] = 0;
        __syncwarp();
        // Partition invariants (costmodel.py:58-72): in range, ascending
        // within each group, and covering 0..n-1 (k*m == n, so covering
        // implies disjoint).
        bool bad = false;
        for (int i = lane; i < km; i += kWarp) {
            int d = mem[i];
            if (d < 0 || d >= n) {
                bad = true;
            } else {
                if (i % m != 0 && mem[i - 1] >= d) bad = true;
                atomicOr(&seen[d >> 5], 1u << (d & 31));
            }
        }
        __syncwarp();
        for (int i = lane; i < nwords; i += kWarp) {
            int bits = min(32, n - i * 32);
            uint32_t want = bits == 32 ? 0xffffffffu : ((1u << bits) - 1u);
            if (seen[i] != want) bad = true;
        }
        if (__any_sync(0xffffffffu, bad)) {
            if (lane == 0) {
                const double nan = __longlong_as_double(0x7ff8000000000000LL);
                a.total[p] = nan;
                if (a.datap) a.datap[p] = nan;
                if (a.pipe) a.pipe[p] = nan;
                atomicAdd(a.invalid, 1);
            }
            __syncwarp();
            continue;
        }
        // data-parallel level (costmodel.py:154-175): per-row numpy pairwise
        // sum over the sorted members (diagonal 0.0 in its slot), max per group
        for (int r = lane; r < km; r += kWarp) {
            int g = r / m;
            const int16_t* gm = mem + g * m;
            const double* row = DP + (size_t)gm[r - g * m] * n;
            h[r] = pairwise_sum(m, [&](int c) { return row[gm[c]]; });
        }
        __syncwarp();
        if (lane < k) {
            double mx = h[lane * m];
            for (int i = 1; i < m; i++) mx = dmax(mx, h[lane * m + i]);
            pg[lane] = mx;
        }
        // pipeline edges (costmodel.py:200-208): bottleneck of each group pair
        for (int t = lane; t < npairs; t += kWarp) {
            int j, j2;
            decode_pair(t, k, j, j2);
            const int16_t* A = mem + j * m;
            const int16_t* B = mem + j2 * m;
            uint32_t L = bottleneck_threshold<uint32_t>(
                m, [&](int r, int c) { return RK[(size_t)A[r] * n + B[c]]; }, 0xffffffffu);
            double v = a.vals[L];
            E[j * kHS + j2] = v;
            E[j2 * kHS + j] = v;
        }
        if (lane < k) E[lane * kHS + lane] = 0.0;
        __syncwarp();
        double pipe = warp_held_karp(k, E, h, st, soff, lane);
        double datap = pg[0];
        for (int g = 1; g < k; g++) datap = dmax(datap, pg[g]);
        if (lane == 0) {
            a.total[p] = datap + pipe;
            if (a.datap) a.datap[p] = datap;
            if (a.pipe) a.pipe[p] = pipe;
            if (a.order) held_karp_order(k, E, h, pipe, a.order + p * k);
        }
        if (a.per_group && lane < k) a.per_group[p * k + lane] = pg[lane];
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// public single-matrix solvers, batched

__global__ void bottleneck_batch_kernel(const double* __restrict__ w, int m, int64_t B, double* __restrict__ out) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
        const double* W = w + b * m * m;
        out[b] = bottleneck_threshold<double>(m, [&](int r, int c) { return W[r * m + c]; }, kInf);
    }
}

__global__ void path_batch_kernel(const double* __restrict__ w, int k, int64_t B, const uint16_t* __restrict__ states,
                                  int nstates, PathOff po, double* __restrict__ total, int8_t* __restrict__ order) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    uint16_t* st = reinterpret_cast<uint16_t*>(smem);
    size_t off = (size_t)((nstates * 2 + 15) & ~15);
    int* soff = reinterpret_cast<int*>(smem + off);
    off += 96;
    const int hsz = (1 << k) * kHS;
    double* h = reinterpret_cast<double*>(smem + off) + (size_t)wid * (hsz + kHS * kHS);
    double* E = h + hsz;
    for (int i = threadIdx.x; i < nstates; i += blockDim.x) st[i] = states[i];
    if (threadIdx.x < 18) soff[threadIdx.x] = po.off[threadIdx.x];
    __syncthreads();
    for (int64_t b = (int64_t)blockIdx.x * W + wid; b < B; b += (int64_t)gridDim.x * W) {
        const double* src = w + b * k * k;
        for (int i = lane; i < k * k; i += kWarp) E[(i / k) * kHS + (i % k)] = src[i];
        __syncwarp();
        double t = warp_held_karp(k, E, h, st, soff, lane);
        if (lane == 0) {
            total[b] = t;
            if (order) held_karp_order(k, E, h, t, order + b * k);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// launchers

static WarpLayout warp_layout(int k, int m) {
    WarpLayout wl;
    int km = k * m;
    int hsz = std::max((1 << k) * kHS, km);
    int o = 0;
    wl.h_off = o;
    o += hsz * 8;
    wl.e_off = o;
    o += kHS * kHS * 8;
    wl.pg_off = o;
    o += kHS * 8;
    wl.mem_off = o;
    o += (km * 2 + 15) & ~15;
    wl.seen_off = o;
    o += 32 * 4;
    wl.bytes = (o + 15) & ~15;
    return wl;
}

int launch_build_tables(int n, const double* lat, const double* bw, int d_dp, double dp_num, double pp_num,
                        double sw_num, double* dp, double* pp, double* sw, cudaStream_t s) {
    int64_t nn = (int64_t)n * n;
    int blocks = (int)std::min<int64_t>((nn + 255) / 256, 4096);
    build_tables_kernel<<<blocks, 256, 0, s>>>(n, lat, bw, (double)d_dp, dp_num, pp_num, sw_num, dp, pp, sw);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_rank(int64_t nn, const double* pp, const double* vals, int nvals, uint32_t* rank, cudaStream_t s) {
    int blocks = (int)std::min<int64_t>((nn + 255) / 256, 4096);
    rank_kernel<<<blocks, 256, 0, s>>>(nn, pp, vals, nvals, rank);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int eval_plan(const EvalArgs& a, int sm_count, size_t smem_optin, EvalPlan* plan) {
    WarpLayout wl = warp_layout(a.k, a.m);
    size_t fixed = (size_t)((a.nstates * 2 + 15) & ~15) + 96;
    size_t tables = (size_t)a.n * a.n * 8 + (((size_t)a.n * a.n * 4 + 15) & ~(size_t)15);
    bool smem_tables = fixed + tables + 4 * (size_t)wl.bytes <= smem_optin;
    size_t base = fixed + (smem_tables ? tables : 0);
    if (base + wl.bytes > smem_optin) return -2;
    int W = (int)std::min<size_t>(16, (smem_optin - base) / wl.bytes);
    plan->smem_tables = smem_tables;
    plan->warps = W;
    plan->smem = base + (size_t)W * wl.bytes;
    plan->blocks = sm_count;
    return 0;
}

int launch_eval(const EvalArgs& a, const EvalPlan& plan, cudaStream_t s) {
    if (a.P == 0) return 0;
    WarpLayout wl = warp_layout(a.k, a.m);
    int64_t warps_needed = a.P;
    int blocks = (int)std::min<int64_t>(plan.blocks, (warps_needed + plan.warps - 1) / plan.warps);
    if (plan.smem_tables) {
        cudaFuncSetAttribute(eval_warp_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
        eval_warp_kernel<true><<<blocks, plan.warps * 32, plan.smem, s>>>(a, wl);
    } else {
        cudaFuncSetAttribute(eval_warp_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
        eval_warp_kernel<false><<<blocks, plan.warps * 32, plan.smem, s>>>(a, wl);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_bottleneck_batch(const double* w, int m, int64_t B, double* out, cudaStream_t s) {
    if (B == 0) return 0;
    int blocks = (int)std::min<int64_t>((B + 127) / 128, 65535);
    bottleneck_batch_kernel<<<blocks, 128, 0, s>>>(w, m, B, out);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_path_batch(const double* w, int k, int64_t B, const uint16_t* states, int nstates, const PathOff& po,
                      double* total, int8_t* order, int sm_count, cudaStream_t s) {
    if (B == 0) return 0;
    int W = 4;
    size_t smem = (size_t)((nstates * 2 + 15) & ~15) + 96 + (size_t)W * ((1 << k) * kHS + kHS * kHS) * 8;
    cudaFuncSetAttribute(path_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = (int)std::min<int64_t>((B + W - 1) / W, (int64_t)sm_count * 8);
    path_batch_kernel<<<blocks, W * 32, smem, s>>>(w, k, B, states, nstates, po, total, order);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace hs
