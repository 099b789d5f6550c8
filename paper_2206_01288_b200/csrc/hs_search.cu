// hs_search.cu -- K2 (surrogate swap gains / local search) and K3 (the GA
// generation loop) on sm_100a, bit-for-bit with hetsched/scheduler.py.
//
// One CTA runs one GA instance (an island).  Warp 0 is the driver: it owns
// the numpy PCG64 stream (lane 0) and executes crossover (scheduler.py:139-174)
// and the refinement passes (_pass_ours :394-428 with _best_candidate :260-276
// and _chain_round :299-391; _pass_kl :431-449) with its 32 lanes sharing the
// data-parallel parts (fast edge, pairwise sums, group means, home costs, KL
// gain matrices).  The passes never read true costs (H4), so a
// generation is: driver produces the offspring plus <= max_passes snapshots ->
// every warp prices snapshots with the K1 warp evaluator -> driver applies
// _refine's first-strict-minimum rule and evolve's replacement / trace rules
// (:548-569).  Population, costs, best and RNG live in global memory between
// launches, so a run can be cut into epochs (island migration).


#include "hs_search_impl.cuh"

namespace hs {

extern template int launch_ga_c<false>(const GAArgs&, const SearchPlan&, int, bool, cudaStream_t);
extern template int launch_ga_c<true>(const GAArgs&, const SearchPlan&, int, bool, cudaStream_t);
extern template int launch_refine_c<false>(const RefineArgs&, const SearchPlan&, int, bool, cudaStream_t);
extern template int launch_refine_c<true>(const RefineArgs&, const SearchPlan&, int, bool, cudaStream_t);

// crossover(p1, p2, rng) on a batch (one warp each)
__global__ void crossover_kernel(int n, int k, int m, const int16_t* p1, const int16_t* p2, hs_pcg64* rngs,
                                 int16_t* out, int B) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x;
    if (b >= B) return;
    const int km = k * m, cap = m + 1;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        unsigned char* p = smem + off;
        off += (bytes + 15) & ~(size_t)15;
        return p;
    };
    LS s;
    s.n = n;
    s.k = k;
    s.m = m;
    s.cap = cap;
    s.W = nullptr;
    s.w_sh = 0;
    s.lat = false;
    s.G = reinterpret_cast<int16_t*>(take((size_t)k * cap * 2));
    s.sz = reinterpret_cast<int*>(take((size_t)k * 4));
    s.perm = reinterpret_cast<int16_t*>(take((size_t)(k * k + cap) * 2));
    s.i32 = reinterpret_cast<int*>(take((size_t)(3 * k + 8) * 4));
    s.grp_of = reinterpret_cast<int8_t*>(take((size_t)n));
    int16_t* a1 = reinterpret_cast<int16_t*>(take((size_t)km * 2));
    int16_t* a2 = reinterpret_cast<int16_t*>(take((size_t)km * 2));
    int16_t* o = reinterpret_cast<int16_t*>(take((size_t)km * 2));
    copy16(a1, p1 + (size_t)b * km, km, lane);
    copy16(a2, p2 + (size_t)b * km, km, lane);
    __syncwarp();
    Pcg64 rng;
    rng.load(rngs[b]);
    crossover(s, a1, a2, rng, o, lane);
    copy16(out + (size_t)b * km, o, km, lane);
    if (lane == 0) rng.store(rngs[b]);
}

// gain_ours / gain_kl (scheduler.py:181-230) for a batch of queries, one
// thread each; q = (j, j2, d1, d2, d1p, d2p) or (d, d2, jd, jd2).
__global__ void gains_kernel(int n, int k, int m, const double* __restrict__ sw, const int16_t* __restrict__ groups,
                             const int32_t* __restrict__ q, int kind, int B, double* __restrict__ out) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int16_t* G = groups + (size_t)b * k * m;
    const int32_t* Q = q + (size_t)b * 6;
    auto psum = [&](int u, const int16_t* grp, int cnt, int skip) {
        // numpy pairwise sum of w[u, grp] (optionally without member `skip`)
        double buf[64];
        int c = 0;
        for (int i = 0; i < cnt; i++)
            if (grp[i] != skip) buf[c++] = sw[(size_t)u * n + grp[i]];
        return pairwise_sum(c, [&](int i) { return buf[i]; });
    };
    if (kind == 0) {
        int j = Q[0], j2 = Q[1], d1 = Q[2], d2 = Q[3], d1p = Q[4], d2p = Q[5];
        const int16_t* gj = G + j * m;
        const int16_t* gj2 = G + j2 * m;
        double t1 = psum(d1, gj2, m, -1) / (double)m - sw[(size_t)d1 * n + d2];
        double t2 = psum(d1p, gj, m, -1) / (double)m - sw[(size_t)d1p * n + d2p];
        out[b] = t1 + t2;
    } else {
        int d = Q[0], d2 = Q[1], jd = Q[2], jd2 = Q[3];
        const int16_t* gj = G + jd * m;
        const int16_t* gj2 = G + jd2 * m;
        double t1 = psum(d, gj2, m, -1);
        double t2 = psum(d, gj, m, d);
        double t3 = psum(d2, gj, m, -1);
        double t4 = psum(d2, gj2, m, d2);
        out[b] = t1 - t2 + t3 - t4 - 2.0 * sw[(size_t)d * n + d2];
    }
}

// ---------------------------------------------------------------------------
// one refinement pass without pricing (gains-only stress, BASELINE config 5:
// 1024 devices in 32 x 32 groups, where exact pricing is out of range).  One
// warp per partition; the n x k mean cache lives in global memory.
__global__ void __launch_bounds__(32) pass_kernel(PassArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x, b = blockIdx.x;
    const int n = a.n, k = a.k, m = a.m, km = k * m, cap = m + 1;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        unsigned char* p = smem + off;
        off += (bytes + 15) & ~(size_t)15;
        return p;
    };
    LS s;
    s.n = n;
    s.k = k;
    s.m = m;
    s.cap = cap;
    s.W = a.sw;
    s.w_sh = 0;
    s.lat = false;
    s.G = reinterpret_cast<int16_t*>(take((size_t)k * cap * 2));
    s.sz = reinterpret_cast<int*>(take((size_t)k * 4));
    s.mean = a.mean + (size_t)b * n * k;
    s.mver = a.mver + (size_t)b * n * k;
    s.cver = reinterpret_cast<uint32_t*>(take((size_t)k * 4));
    s.home = reinterpret_cast<double*>(take((size_t)n * 8));
    s.valid = reinterpret_cast<int*>(take(16));
    s.fe = reinterpret_cast<int16_t*>(take((size_t)k * 4));
    s.bpv = reinterpret_cast<double*>(take((size_t)n * 8));
    s.bpp = reinterpret_cast<int16_t*>(take((size_t)n * 2));
    s.locked = reinterpret_cast<uint32_t*>(take((size_t)((n + 31) >> 5) * 4));
    s.nlocked = reinterpret_cast<int*>(take(4));
    s.perm = reinterpret_cast<int16_t*>(take((size_t)(k * k + cap) * 2));
    s.f64 = reinterpret_cast<double*>(take((size_t)(4 * cap + 2 * k + 2) * 8));
    s.i32 = reinterpret_cast<int*>(take((size_t)(3 * k + 8) * 4));
    s.grp_of = reinterpret_cast<int8_t*>(take((size_t)n));
    for (int t = lane; t < n * k; t += kWarp) s.mver[t] = 0;
    for (int t = lane; t < k; t += kWarp) s.cver[t] = 1;
    __syncwarp();
    Pcg64 rng;
    rng.load(a.rng[b]);
    load_groups(s, a.groups + (size_t)b * km, lane);
    bool ch = a.kind == 0 ? ((s.sz[0] < 2) ? false : (a.phase % 2 == 0 ? pass_sweep(s, rng, lane) : pass_chains(s, lane)))
                          : pass_kl(s, lane);
    store_groups(s, a.out_groups + (size_t)b * km, lane);
    if (lane == 0) {
        a.changed[b] = ch;
        rng.store(a.rng[b]);
    }
}

// _refine's selection (scheduler.py:483-487) over batch-priced snapshots:
// first strict minimum; one warp per partition
__global__ void refine_commit_kernel(RefineArgs a, const double* __restrict__ cost, int B) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= B) return;
    const int km = a.k * a.m, n = a.snap_cnt[b];
    const double* c = cost + (size_t)b * a.snap_stride;
    int bsi = 0;
    for (int q = 1; q < n; q++)
        if (c[q] < c[bsi]) bsi = q;
    const int16_t* src = a.snap_buf + ((size_t)b * a.snap_stride + bsi) * km;
    for (int t = lane; t < km; t += 32) a.out_groups[(size_t)b * km + t] = src[t];
    if (lane == 0) {
        a.out_cost[b] = c[bsi];
        a.evaluations[b] = n;
    }
}

int launch_refine_commit(const RefineArgs& a, const double* snap_cost, int B, cudaStream_t st) {
    if (B == 0) return 0;
    refine_commit_kernel<<<(B + 7) / 8, 256, 0, st>>>(a, snap_cost, B);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

size_t pass_smem_bytes(int n, int k, int m) {
    auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
    int cap = m + 1;
    return al((size_t)k * cap * 2) + al((size_t)k * 4) + al((size_t)k * 4) + al((size_t)n * 8) + al(16) +
           al((size_t)k * 4) + al((size_t)n * 8) + al((size_t)n * 2) + al((size_t)((n + 31) >> 5) * 4) + al(4) +
           al((size_t)(k * k + cap) * 2) + al((size_t)(4 * cap + 2 * k + 2) * 8) + al((size_t)(3 * k + 8) * 4) +
           al((size_t)n);
}

int launch_pass(const PassArgs& a, int B, cudaStream_t st) {
    if (B == 0) return 0;
    size_t smem = pass_smem_bytes(a.n, a.k, a.m);
    cudaFuncSetAttribute(pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    pass_kernel<<<B, 32, smem, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---------------------------------------------------------------------------
// launchers

static size_t ls_bytes(int n, int k, int m) {
    int cap = m + 1;
    auto al = [](size_t b) { return (b + 15) & ~(size_t)15; };
    return al((size_t)k * cap * 2) + al((size_t)k * 4) + al((size_t)n * k * 8) + al((size_t)n * k * 4) +
           al((size_t)k * 4) + al((size_t)n * 8) + al(16) +
           al((size_t)k * 4) + al((size_t)n * 8) + al((size_t)n * 2) +
           al((size_t)((n + 31) >> 5) * 4) + al(4) + al((size_t)(k * k + cap) * 2) +
           al((size_t)(4 * cap + 2 * k + 2) * 8) + al((size_t)(3 * k + 8) * 4) + al((size_t)n);
}

static size_t ga_bytes(const SearchShape& sh, int W, bool smem_tables, int P, bool warp_islands = false) {
    auto al = [](size_t b) { return (b + 15) & ~(size_t)15; };
    ScratchLayout wl = scratch_layout(sh.k <= 8 ? sh.k : 8, sh.m);
    int km = sh.k * sh.m, ms = 1 + sh.max_passes;
    size_t b = sh.k <= 8 ? kHKGlobalBytes + (size_t)W * wl.bytes : al(cta_scratch_bytes(sh.k, sh.m));
    if (smem_tables)
        b += staged_table_bytes(sh.n, sh.key16 ? 2 : 4) + (size_t)sh.n * sh.n * 8;
    size_t isl = al((size_t)ms * km * 2) + al((size_t)ms * 8) + al((size_t)P * 8) + al((size_t)km * 2) +
                 al((size_t)2 * km * 2) + al(64) + ls_bytes(sh.n, sh.k, sh.m) + al(sizeof(GAState));
    b += (warp_islands ? (size_t)W : 1) * isl;
    return b;
}

int search_plan(const SearchShape& sh, int P, size_t smem_optin, SearchPlan* plan, bool warp_islands) {
    plan->warp_islands = warp_islands && sh.k <= 8;
    for (int W : {8, 6, 4, 2, 1}) {
        for (int st = 1; st >= 0; st--) {
            size_t b = ga_bytes(sh, W, st, P, plan->warp_islands);
            if (b <= smem_optin) {
                plan->warps = W;
                plan->smem_tables = st;
                plan->smem = b;
                plan->m8 = sh.key16 && sh.m == 8;
                plan->cta = sh.k > 8;
                return 0;
            }
        }
    }
    return -2;
}

int launch_ga(const GAArgs& a, const SearchPlan& plan, int islands, bool key16, cudaStream_t st) {
    return plan.cta ? launch_ga_c<true>(a, plan, islands, key16, st) : launch_ga_c<false>(a, plan, islands, key16, st);
}

int launch_refine(const RefineArgs& a, const SearchPlan& plan, int B, bool key16, cudaStream_t st) {
    if (B == 0) return 0;
    return plan.cta ? launch_refine_c<true>(a, plan, B, key16, st) : launch_refine_c<false>(a, plan, B, key16, st);
}

int launch_crossover(int n, int k, int m, const int16_t* p1, const int16_t* p2, hs_pcg64* rngs, int16_t* out, int B,
                     cudaStream_t st) {
    if (B == 0) return 0;
    size_t smem = ls_bytes(n, k, m) + 3 * (((size_t)k * m * 2 + 15) & ~(size_t)15) + 256;
    cudaFuncSetAttribute(crossover_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    crossover_kernel<<<B, 32, smem, st>>>(n, k, m, p1, p2, rngs, out, B);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_gains(int n, int k, int m, const double* sw, const int16_t* groups, const int32_t* q, int kind, int B,
                 double* out, cudaStream_t st) {
    if (B == 0) return 0;
    gains_kernel<<<(B + 127) / 128, 128, 0, st>>>(n, k, m, sw, groups, q, kind, B, out);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---------------------------------------------------------------------------
// island migration (new capability)

// export: each island's E best members by (cost, index), one warp per island
__global__ void export_kernel(int P, int km, int E, const int16_t* __restrict__ pop, const double* __restrict__ cost,
                              int16_t* __restrict__ out, double* __restrict__ out_cost) {
    const int isl = blockIdx.x, lane = threadIdx.x;
    const int16_t* ip = pop + (size_t)isl * P * km;
    const double* ic = cost + (size_t)isl * P;
    uint64_t taken[4] = {0, 0, 0, 0};  // P <= 256
    for (int e = 0; e < E; e++) {
        double bv = kInf;
        int bi = INT_MAX;
        for (int i = lane; i < P; i += kWarp)
            if (!(taken[i >> 6] >> (i & 63) & 1) && (ic[i] < bv || (ic[i] == bv && i < bi))) {
                bv = ic[i];
                bi = i;
            }
        warp_argmin(bv, bi);
        taken[bi >> 6] |= 1ull << (bi & 63);
        copy16(out + ((size_t)isl * E + e) * km, ip + (size_t)bi * km, km, lane);
        if (lane == 0) out_cost[(size_t)isl * E + e] = bv;
    }
}

// import: island i receives migrants[src[i]]; each replaces the current
// worst member (first maximum) when strictly cheaper, and may become best.
__global__ void import_kernel(int P, int km, int E, int16_t* __restrict__ pop, double* __restrict__ cost,
                              int16_t* __restrict__ best, GAState* __restrict__ state, const int16_t* __restrict__ mig,
                              const double* __restrict__ mig_cost, const int32_t* __restrict__ src) {
    const int isl = blockIdx.x, lane = threadIdx.x;
    int16_t* ip = pop + (size_t)isl * P * km;
    double* ic = cost + (size_t)isl * P;
    const int s = src[isl];
    for (int e = 0; e < E; e++) {
        const int16_t* g = mig + ((size_t)s * E + e) * km;
        double c = mig_cost[(size_t)s * E + e];
        double wv = -kInf;
        int wi = INT_MAX;
        for (int i = lane; i < P; i += kWarp)
            if (ic[i] > wv || (ic[i] == wv && i < wi)) {
                wv = ic[i];
                wi = i;
            }
        warp_argmax(wv, wi);
        if (c < wv) {
            copy16(ip + (size_t)wi * km, g, km, lane);
            __syncwarp();
            if (lane == 0) ic[wi] = c;
        }
        if (c < state[isl].best_total) {
            copy16(best + (size_t)isl * km, g, km, lane);
            __syncwarp();
            if (lane == 0) {
                state[isl].best_total = c;
                state[isl].since = 0;
            }
        }
        __syncwarp();
    }
}

// init_population draws from one stream (lane 0), then lanes sort groups
__global__ void random_partitions_kernel(int n, int k, int m, int B, hs_pcg64* rng_io, int16_t* out) {
    const int lane = threadIdx.x;
    Pcg64 rng;
    if (lane == 0) rng.load(*rng_io);
    for (int b = 0; b < B; b++) {
        int16_t* d = out + (size_t)b * n;
        if (lane == 0) {
            for (int t = 0; t < n; t++) d[t] = (int16_t)t;
            for (int t = n - 1; t >= 1; t--) {
                int jx = (int)rng.interval((uint64_t)t);
                int16_t x = d[t];
                d[t] = d[jx];
                d[jx] = x;
            }
        }
        __syncwarp();
        for (int j = lane; j < k; j += kWarp) {
            int16_t* gp = d + j * m;
            for (int a = 1; a < m; a++) {
                int16_t x = gp[a];
                int q = a - 1;
                while (q >= 0 && gp[q] > x) {
                    gp[q + 1] = gp[q];
                    q--;
                }
                gp[q + 1] = x;
            }
        }
        __syncwarp();
    }
    if (lane == 0) rng.store(*rng_io);
}

int launch_export(int islands, int P, int km, int E, const int16_t* pop, const double* cost, int16_t* out,
                  double* out_cost, cudaStream_t st) {
    export_kernel<<<islands, 32, 0, st>>>(P, km, E, pop, cost, out, out_cost);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_import(int islands, int P, int km, int E, int16_t* pop, double* cost, int16_t* best, GAState* state,
                  const int16_t* mig, const double* mig_cost, const int32_t* src, cudaStream_t st) {
    import_kernel<<<islands, 32, 0, st>>>(P, km, E, pop, cost, best, state, mig, mig_cost, src);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_random_partitions(int n, int k, int m, int B, hs_pcg64* rng, int16_t* out, cudaStream_t st) {
    random_partitions_kernel<<<1, 32, 0, st>>>(n, k, m, B, rng, out);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace hs
