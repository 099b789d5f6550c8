// hs_assign.cu -- fixed-layout pricing and layout materialization on sm_100a
// (hetsched/evaluation.py:162-243, combinatorics.py:134-189).
//
//   materialize_kernel : one warp per partition: bottleneck edges + Held-Karp
//                        order (the K1 warp evaluator), then the
//                        lexicographically smallest optimal pairing of each
//                        consecutive stage pair (one lane each) and the grid.
//   evaluate_kernel    : one warp per assignment grid (m rows x k columns):
//                        per-column datap, per-boundary worst row edge,
//                        right-to-left pipeline sum.
//   random_assign_kernel : one thread per trial stream (random_partition then
//                        permutation(k)), so SeedSequence children stay
//                        independent of execution order.
#include <algorithm>
#include <climits>

#include "hs_assign.h"
#include "hs_rng.cuh"
#include "hs_warp_eval.cuh"

namespace hs {

// Is there a perfect matching of `rows` into `cols` within adj (<= 64 x 64)?
__device__ inline bool has_matching(const uint64_t* adj, uint64_t rows, uint64_t cols) {
    int8_t match_col[64];
    for (int i = 0; i < 64; i++) match_col[i] = -1;
    uint64_t rr = rows;
    while (rr) {
        int u = __ffsll((long long)rr) - 1;
        rr &= rr - 1;
        // BFS for an augmenting path from u
        uint64_t rows_in = 1ull << u, cols_in = 0, frontier = rows_in;
        int8_t parent[64];
        int found = -1;
        while (frontier && found < 0) {
            int r = __ffsll((long long)frontier) - 1;
            frontier &= frontier - 1;
            uint64_t cand = adj[r] & cols & ~cols_in;
            while (cand) {
                int c = __ffsll((long long)cand) - 1;
                cand &= cand - 1;
                parent[c] = (int8_t)r;
                cols_in |= 1ull << c;
                if (match_col[c] < 0) {
                    found = c;
                    break;
                }
                rows_in |= 1ull << match_col[c];
                frontier |= 1ull << match_col[c];
            }
        }
        if (found < 0) return false;
        // augment: walk back along parents, flipping matched edges
        int c = found;
        for (;;) {
            int r = parent[c];
            int prev = -1;
            for (int x = 0; x < 64; x++)
                if (match_col[x] == r) prev = x;
            match_col[c] = (int8_t)r;
            if (r == u) break;
            c = prev;
        }
    }
    return true;
}

// _lex_smallest_pairing (combinatorics.py:147-189): rows in order take the
// smallest column that still leaves a perfect matching for the rest.
__device__ inline void lex_pairing(int m, const uint64_t* adj, int8_t* pairs) {
    uint64_t all = m == 64 ? ~0ull : ((1ull << m) - 1);
    uint64_t used = 0;
    for (int r = 0; r < m; r++) {
        uint64_t rest_rows = all & ~((2ull << r) - 1);
        if (r == 63) rest_rows = 0;
        uint64_t cand = adj[r] & ~used;
        while (cand) {
            int c = __ffsll((long long)cand) - 1;
            cand &= cand - 1;
            if (has_matching(adj, rest_rows, all & ~used & ~(1ull << c))) {
                pairs[r] = (int8_t)c;
                used |= 1ull << c;
                break;
            }
        }
    }
}

template <typename KeyT>
__global__ void __launch_bounds__(256) materialize_kernel(MaterializeArgs a, ScratchLayout wl) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int n = a.n, k = a.k, m = a.m, km = k * m;
    HKSmem hk = hk_stage(a.hk, smem);
    size_t off = hk_smem_bytes(a.hk);
    EvalView<KeyT> v = stage_tables<false, KeyT>(n, k, m, a.dp, a.rank, a.vals, hk, smem, off);
    unsigned char* wbase = smem + off + (size_t)wid * (wl.bytes + 64 * 16 + 64 * 8);
    WarpScratch ws = scratch_at(wbase, wl);
    int16_t* mem = reinterpret_cast<int16_t*>(wbase + wl.mem_off);
    int8_t* order = reinterpret_cast<int8_t*>(wbase + wl.bytes);            // 16
    int8_t* pairs = order + 16;                                              // (k-1) x m  (<= 15 x 64)
    int16_t* cols = reinterpret_cast<int16_t*>(wbase + wl.bytes + 64 * 16);  // 64
    __syncthreads();
    for (int64_t p = (int64_t)blockIdx.x * W + wid; p < a.B; p += (int64_t)gridDim.x * W) {
        for (int i = lane; i < km; i += kWarp) mem[i] = a.groups[p * km + i];
        __syncwarp();
        double dp, pp;
        if (m == 8 && sizeof(KeyT) == 2)
            warp_price<KeyT, true>(v, ws, mem, lane, dp, pp);
        else
            warp_price<KeyT, false>(v, ws, mem, lane, dp, pp);
        if (lane == 0) held_karp_order(k, ws.E, ws.h, hk.hoff, pp, order);
        __syncwarp();
        // pairing of consecutive stages b-1, b (rows: lower group index)
        for (int b = 1 + lane; b < k; b += kWarp) {
            int g1 = order[b - 1], g2 = order[b];
            int lo = g1 < g2 ? g1 : g2, hi = g1 < g2 ? g2 : g1;
            const int16_t* A = mem + lo * m;
            const int16_t* Bg = mem + hi * m;
            double bv = ws.E[lo * kES + hi];
            uint64_t adj[64];
            for (int r = 0; r < m; r++) {
                uint64_t row = 0;
                for (int c = 0; c < m; c++)
                    if (v.vals[v.RK[(size_t)A[r] * n + Bg[c]]] <= bv) row |= 1ull << c;
                adj[r] = row;
            }
            lex_pairing(m, adj, pairs + (b - 1) * m);
        }
        __syncwarp();
        if (lane == 0) {
            // cols[0] = sorted(groups[pi[0]]); then follow the stored matchings
            const int16_t* g0 = mem + order[0] * m;
            for (int i = 0; i < m; i++) cols[i] = g0[i];
            int16_t* grid = a.grid + p * km;  // [m][k]
            for (int i = 0; i < m; i++) grid[i * k] = cols[i];
            for (int b = 1; b < k; b++) {
                int prev = order[b - 1], cur = order[b];
                int lo = prev < cur ? prev : cur, hi = prev < cur ? cur : prev;
                const int16_t* lo_d = mem + lo * m;
                const int16_t* hi_d = mem + hi * m;
                const int8_t* pr = pairs + (b - 1) * m;
                for (int i = 0; i < m; i++) {
                    int d = cols[i], nx = -1;
                    if (prev == lo) {
                        for (int r = 0; r < m; r++)
                            if (lo_d[r] == d) nx = hi_d[pr[r]];
                    } else {
                        for (int r = 0; r < m; r++)
                            if (hi_d[pr[r]] == d) nx = lo_d[r];
                    }
                    cols[i] = (int16_t)nx;
                    grid[i * k + b] = (int16_t)nx;
                }
            }
            for (int b = 0; b < k; b++) a.order[p * k + b] = order[b];
        }
        __syncwarp();
    }
}

// evaluate_assignment (evaluation.py:195-229) on grids [B][m][k]
__global__ void __launch_bounds__(256) evaluate_kernel(int n, int k, int m, const double* __restrict__ dp,
                                                       const double* __restrict__ pp, const int16_t* __restrict__ grids,
                                                       int64_t B, double* __restrict__ out3,
                                                       double* __restrict__ per_col) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    int16_t* col = reinterpret_cast<int16_t*>(smem) + (size_t)wid * (k * m + 64);
    double* pc = reinterpret_cast<double*>(smem + (size_t)W * (k * m + 64) * 2) + (size_t)wid * 32;
    for (int64_t p = (int64_t)blockIdx.x * W + wid; p < B; p += (int64_t)gridDim.x * W) {
        const int16_t* gr = grids + p * k * m;
        // columns, sorted ascending (datap_cost_group sorts, costmodel.py:156)
        for (int b = lane; b < k; b += kWarp) {
            int16_t* cb = col + b * m;
            for (int i = 0; i < m; i++) cb[i] = gr[i * k + b];
            for (int x = 1; x < m; x++) {
                int16_t y = cb[x];
                int q = x - 1;
                while (q >= 0 && cb[q] > y) {
                    cb[q + 1] = cb[q];
                    q--;
                }
                cb[q + 1] = y;
            }
            double worst = 0.0;
            if (m > 1) {
                for (int r = 0; r < m; r++) {
                    const double* row = dp + (size_t)cb[r] * n;
                    double s = pairwise_sum(m, [&](int c) { return row[cb[c]]; });
                    worst = r == 0 ? s : dmax(worst, s);
                }
            }
            pc[b] = worst;
        }
        __syncwarp();
        if (lane == 0) {
            double datap = pc[0];
            for (int b = 1; b < k; b++) datap = dmax(datap, pc[b]);
            double bnd[16];
            for (int b = 0; b + 1 < k; b++) {
                double worst = 0.0;
                for (int i = 0; i < m; i++) {
                    double c = pp[(size_t)gr[i * k + b] * n + gr[i * k + b + 1]];
                    if (c > worst) worst = c;
                }
                bnd[b] = worst;
            }
            double pipe = 0.0;
            for (int b = k - 2; b >= 0; b--) pipe = bnd[b] + pipe;
            out3[p * 3 + 0] = datap + pipe;
            out3[p * 3 + 1] = datap;
            out3[p * 3 + 2] = pipe;
            if (per_col)
                for (int b = 0; b < k; b++) per_col[p * k + b] = pc[b];
        }
        __syncwarp();
    }
}

// random_assignment (evaluation.py:232-243), one stream per trial
__global__ void random_assign_kernel(int n, int k, int m, int B, hs_pcg64* rngs, int16_t* perm_scratch, int16_t* grids,
                                     int8_t* orders) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    Pcg64 rng;
    rng.load(rngs[b]);
    int16_t* d = perm_scratch + (size_t)b * n;
    for (int t = 0; t < n; t++) d[t] = (int16_t)t;
    for (int t = n - 1; t >= 1; t--) {
        int jx = (int)rng.interval((uint64_t)t);
        int16_t x = d[t];
        d[t] = d[jx];
        d[jx] = x;
    }
    for (int j = 0; j < k; j++) {  // Partition sorts members
        int16_t* gp = d + j * m;
        for (int x = 1; x < m; x++) {
            int16_t y = gp[x];
            int q = x - 1;
            while (q >= 0 && gp[q] > y) {
                gp[q + 1] = gp[q];
                q--;
            }
            gp[q + 1] = y;
        }
    }
    int8_t pi[64];
    for (int t = 0; t < k; t++) pi[t] = (int8_t)t;
    for (int t = k - 1; t >= 1; t--) {
        int jx = (int)rng.interval((uint64_t)t);
        int8_t x = pi[t];
        pi[t] = pi[jx];
        pi[jx] = x;
    }
    int16_t* grid = grids + (size_t)b * n;
    for (int c = 0; c < k; c++)
        for (int i = 0; i < m; i++) grid[i * k + c] = d[pi[c] * m + i];
    for (int c = 0; c < k; c++) orders[(size_t)b * k + c] = pi[c];
    rng.store(rngs[b]);
}

int launch_materialize(const MaterializeArgs& a, int sm_count, cudaStream_t s) {
    if (a.B == 0) return 0;
    ScratchLayout wl = scratch_layout(a.k, a.m);
    const int W = 4;
    size_t smem = hk_smem_bytes(a.hk) + (size_t)W * (wl.bytes + 64 * 16 + 64 * 8);
    if (a.key16) {
        cudaFuncSetAttribute(materialize_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        materialize_kernel<uint16_t><<<sm_count, W * 32, smem, s>>>(a, wl);
    } else {
        cudaFuncSetAttribute(materialize_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        materialize_kernel<uint32_t><<<sm_count, W * 32, smem, s>>>(a, wl);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_evaluate(int n, int k, int m, const double* dp, const double* pp, const int16_t* grids, int64_t B,
                    double* out3, double* per_col, int sm_count, cudaStream_t s) {
    if (B == 0) return 0;
    const int W = 8;
    size_t smem = (size_t)W * (k * m + 64) * 2 + (size_t)W * 32 * 8 + 16;
    cudaFuncSetAttribute(evaluate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = (int)std::min<int64_t>((B + W - 1) / W, (int64_t)sm_count * 4);
    evaluate_kernel<<<blocks, W * 32, smem, s>>>(n, k, m, dp, pp, grids, B, out3, per_col);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_random_assign(int n, int k, int m, int B, hs_pcg64* rngs, int16_t* scratch, int16_t* grids, int8_t* orders,
                         cudaStream_t s) {
    if (B == 0) return 0;
    random_assign_kernel<<<(B + 63) / 64, 64, 0, s>>>(n, k, m, B, rngs, scratch, grids, orders);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// bottleneck_perfect_matching (combinatorics.py:134-144) of B matrices
// [B][m][m]: optimal threshold, then the lexicographically smallest pairing
// among the perfect matchings that stay within it.  One thread per matrix.
__global__ void bottleneck_match_kernel(const double* __restrict__ w, int m, int64_t B, double* __restrict__ value,
                                        int8_t* __restrict__ pairs) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
        const double* W = w + b * m * m;
        double L = bottleneck_threshold<double>(m, [&](int r, int c) { return W[r * m + c]; }, kInf);
        uint64_t adj[kMaxM];
        for (int r = 0; r < m; r++) {
            uint64_t row = 0;
            for (int c = 0; c < m; c++)
                if (W[r * m + c] <= L) row |= 1ull << c;
            adj[r] = row;
        }
        value[b] = L;
        if (pairs) lex_pairing(m, adj, pairs + b * m);
    }
}

// datap_cost_group (costmodel.py:154-168) of G gathered m x m blocks of raw
// lat / bw: dp_pair_seconds with a zero diagonal, numpy-pairwise row sums,
// largest row.  One warp per group, one lane per row.
__global__ void datap_group_kernel(const double* __restrict__ lat, const double* __restrict__ bw, int m, int64_t G,
                                   double ddp, double dp_num, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t W = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); g < G; g += W) {
        const double* L = lat + g * m * m;
        const double* Bw = bw + g * m * m;
        double best = -kInf;
        for (int r = lane; r < m; r += kWarp) {
            double s = pairwise_sum(m, [&](int c) {
                return c == r ? 0.0 : 2.0 * (L[r * m + c] + dp_num / (ddp * Bw[r * m + c]));
            });
            best = dmax(best, s);
        }
        for (int o = 16; o; o >>= 1) best = dmax(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) out[g] = m == 1 ? 0.0 : best;
    }
}

int launch_bottleneck_match(const double* w, int m, int64_t B, double* value, int8_t* pairs, cudaStream_t s) {
    if (B == 0) return 0;
    int blocks = (int)std::min<int64_t>((B + 63) / 64, 148 * 16);
    bottleneck_match_kernel<<<blocks, 64, 0, s>>>(w, m, B, value, pairs);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_datap_group(const double* lat, const double* bw, int m, int64_t G, double ddp, double dp_num, double* out,
                       cudaStream_t s) {
    if (G == 0) return 0;
    int blocks = (int)std::min<int64_t>((G + 7) / 8, 148 * 8);
    datap_group_kernel<<<blocks, 256, 0, s>>>(lat, bw, m, G, ddp, dp_num, out);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace hs
