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
#include "hs_warp_eval.cuh"

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

// warps per CTA of the batch evaluator (one CTA per SM; bounded by smem and
// registers): with the compact Held-Karp table (stage order wanted) and with
// the two-layer one (no order: 4.4 KB less scratch per warp)
constexpr int kEvalWarps = 20;
#ifndef HS_EVAL_WARPS_ROLL
#define HS_EVAL_WARPS_ROLL 24
#endif
constexpr int kEvalWarpsRoll = HS_EVAL_WARPS_ROLL;

template <bool kSmemTables, typename KeyT, bool kM8, bool kRoll>
__global__ void __launch_bounds__(32 * (kRoll ? kEvalWarpsRoll : kEvalWarps))
    eval_warp_kernel(EvalArgs a, ScratchLayout wl) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int k = a.k, m = kM8 ? 8 : a.m, km = k * m;
    const HKTables& hkt = kRoll ? a.hk_roll : a.hk;
    HKSmem hk = hk_stage(hkt, smem);
    size_t off = hk_smem_bytes(hkt);
    EvalView<KeyT> v = stage_tables<kSmemTables, KeyT>(a.n, k, m, a.dp, a.rank, a.vals, hk, smem, off);
    unsigned char* wbase = smem + off + (size_t)wid * wl.bytes;
    WarpScratch ws = scratch_at(wbase, wl);
    int16_t* mem = reinterpret_cast<int16_t*>(wbase + wl.mem_off);
    __syncthreads();

    for (int64_t p = (int64_t)blockIdx.x * W + wid; p < a.P; p += (int64_t)gridDim.x * W) {
        const int16_t* gsrc = a.groups + p * km;
        for (int i = lane; i < km; i += kWarp) mem[i] = gsrc[i];
        __syncwarp();
        if (!warp_valid(a.n, k, m, mem, ws.seen, lane)) {
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
        double datap, pipe;
        warp_price<KeyT, kM8>(v, ws, mem, lane, datap, pipe);
        if (lane == 0) {
            a.total[p] = datap + pipe;
            if (a.datap) a.datap[p] = datap;
            if (a.pipe) a.pipe[p] = pipe;
            if (!kRoll && a.order) held_karp_order(k, ws.E, ws.h, hk.hoff, pipe, a.order + p * k);
        }
        if (a.per_group && lane < k) a.per_group[p * k + lane] = ws.pg[lane];
        __syncwarp();
    }
}


__global__ void bottleneck_batch_kernel(const double* __restrict__ w, int m, int64_t B, double* __restrict__ out) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
        const double* W = w + b * m * m;
        out[b] = bottleneck_threshold<double>(m, [&](int r, int c) { return W[r * m + c]; }, kInf);
    }
}

__global__ void path_batch_kernel(const double* __restrict__ w, int k, int64_t B, HKTables t,
                                  double* __restrict__ total, int8_t* __restrict__ order) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    HKSmem hk = hk_stage(t, smem);
    size_t off = hk_smem_bytes(t);
    const int hsz = (k << (k - 1)) + 8 * kES;
    double* h = reinterpret_cast<double*>(smem + off) + (size_t)wid * hsz;
    double* E = h + (k << (k - 1));
    __syncthreads();
    for (int64_t b = (int64_t)blockIdx.x * W + wid; b < B; b += (int64_t)gridDim.x * W) {
        const double* src = w + b * k * k;
        for (int i = lane; i < k * k; i += kWarp) E[(i / k) * kES + (i % k)] = src[i];
        __syncwarp();
        double tt = warp_held_karp(k, E, h, hk.states, hk.lay, lane, hk.final_off);
        if (lane == 0) {
            total[b] = tt;
            if (order) held_karp_order(k, E, h, hk.hoff, tt, order + b * k);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// launchers

static size_t hk_bytes_host(const HKTables& t) { return hk_smem_bytes(t); }

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

__global__ void narrow_kernel(int64_t nn, const uint32_t* __restrict__ src, uint16_t* __restrict__ dst) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nn; x += (int64_t)gridDim.x * blockDim.x)
        dst[x] = (uint16_t)src[x];
}

int launch_narrow(int64_t nn, const uint32_t* src, uint16_t* dst, cudaStream_t s) {
    int blocks = (int)std::min<int64_t>((nn + 255) / 256, 4096);
    narrow_kernel<<<blocks, 256, 0, s>>>(nn, src, dst);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

static int plan_for(const EvalArgs& a, const HKTables& t, int wmax, size_t smem_optin, bool* smem_tables, int* warps,
                    size_t* smem) {
    ScratchLayout wl = scratch_layout(a.k, a.m, t.hsize);
    size_t fixed = hk_bytes_host(t);
    size_t keyb = a.key16 ? 2 : 4;
    size_t tables = staged_table_bytes(a.n, keyb);
    *smem_tables = fixed + tables + 4 * (size_t)wl.bytes <= smem_optin;
    size_t base = fixed + (*smem_tables ? tables : 0);
    if (base + wl.bytes > smem_optin) return -2;
    *warps = (int)std::min<size_t>(wmax, (smem_optin - base) / wl.bytes);
    *smem = base + (size_t)*warps * wl.bytes;
    return 0;
}

int eval_plan(const EvalArgs& a, int sm_count, size_t smem_optin, EvalPlan* plan) {
    if (plan_for(a, a.hk, kEvalWarps, smem_optin, &plan->smem_tables, &plan->warps, &plan->smem)) return -2;
    if (plan_for(a, a.hk_roll, kEvalWarpsRoll, smem_optin, &plan->roll_smem_tables, &plan->roll_warps,
                 &plan->roll_smem))
        return -2;
    plan->blocks = sm_count;
    plan->m8 = a.key16 && a.m == 8;
    return 0;
}

template <bool S, typename KT, bool M8, bool R>
static void launch_one(const EvalArgs& a, int warps, size_t smem, int blocks, cudaStream_t s) {
    ScratchLayout wl = scratch_layout(a.k, a.m, R ? a.hk_roll.hsize : a.hk.hsize);
    cudaFuncSetAttribute(eval_warp_kernel<S, KT, M8, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    eval_warp_kernel<S, KT, M8, R><<<blocks, warps * 32, smem, s>>>(a, wl);
}

template <bool R>
static void launch_variant(const EvalArgs& a, const EvalPlan& plan, cudaStream_t s) {
    const int warps = R ? plan.roll_warps : plan.warps;
    const size_t smem = R ? plan.roll_smem : plan.smem;
    const bool st = R ? plan.roll_smem_tables : plan.smem_tables;
    int blocks = (int)std::min<int64_t>(plan.blocks, (a.P + warps - 1) / warps);
    if (plan.m8) {
        if (st)
            launch_one<true, uint16_t, true, R>(a, warps, smem, blocks, s);
        else
            launch_one<false, uint16_t, true, R>(a, warps, smem, blocks, s);
    } else if (a.key16) {
        if (st)
            launch_one<true, uint16_t, false, R>(a, warps, smem, blocks, s);
        else
            launch_one<false, uint16_t, false, R>(a, warps, smem, blocks, s);
    } else {
        if (st)
            launch_one<true, uint32_t, false, R>(a, warps, smem, blocks, s);
        else
            launch_one<false, uint32_t, false, R>(a, warps, smem, blocks, s);
    }
}

int launch_eval(const EvalArgs& a, const EvalPlan& plan, cudaStream_t s) {
    if (a.P == 0) return 0;
    // without an order output the compact table (needed to walk the optimal
    // path back) is not kept: two-layer schedule, more warps per SM
    if (a.order)
        launch_variant<false>(a, plan, s);
    else
        launch_variant<true>(a, plan, s);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_bottleneck_batch(const double* w, int m, int64_t B, double* out, cudaStream_t s) {
    if (B == 0) return 0;
    int blocks = (int)std::min<int64_t>((B + 127) / 128, 65535);
    bottleneck_batch_kernel<<<blocks, 128, 0, s>>>(w, m, B, out);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_path_batch(const double* w, int k, int64_t B, const HKTables& t, double* total, int8_t* order,
                      int sm_count, cudaStream_t s) {
    if (B == 0) return 0;
    int W = 4;
    size_t smem = hk_bytes_host(t) + (size_t)W * ((k << (k - 1)) + 8 * kES) * 8;
    cudaFuncSetAttribute(path_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = (int)std::min<int64_t>((B + W - 1) / W, (int64_t)sm_count * 8);
    path_batch_kernel<<<blocks, W * 32, smem, s>>>(w, k, B, t, total, order);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace hs
