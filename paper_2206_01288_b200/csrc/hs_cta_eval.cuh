// hs_cta_eval.cuh -- one CTA prices one candidate with 9 <= d_pp <= 16
// (BASELINE config 4: 512 devices, 16 x 32; Held-Karp over 2^16 subsets).
//
// The compact Held-Karp table k*2^(k-1) - k f64 (4.2 MB at k = 16) does not
// fit shared memory, so it lives in a per-CTA global scratch
// slice that stays L2-resident while the CTA sweeps the popcount layers;
// __syncthreads separates layers.  Same state words as the warp version
// (hs_eval.cuh), widened to 64 bits: off[r] (20) | dst (20) | u (4) | r (16).
#pragma once
#include "hs_warp_eval.cuh"

namespace hs {

constexpr int kCtaK = 16;
constexpr int kES16 = 17;  // padded E row stride

template <int NV>
__device__ __forceinline__ double hk_relax_g(const double* __restrict__ Eu, const double* __restrict__ hr, uint32_t r) {
    double best = kInf;
#pragma unroll
    for (int i = 0; i < NV; i++) {
        int v = __ffs(r) - 1;
        r &= r - 1;
        double c = Eu[v] + hr[i];
        best = c < best ? c : best;
    }
    return best;
}

__device__ inline double cta_held_karp(int k, const double* E, double* h, const HKBig& t, double* red) {
    if (k == 1) return 0.0;
    for (int p = 2; p <= k; p++) {
        const int end = t.lay[p + 1];
        for (int idx = t.lay[p] + threadIdx.x; idx < end; idx += blockDim.x) {
            uint64_t w = t.states[idx];
            uint32_t offr = (uint32_t)(w & 0xFFFFF);
            uint32_t dst = (uint32_t)((w >> 20) & 0xFFFFF);
            int u = (int)((w >> 40) & 0xF);
            uint32_t r = (uint32_t)(w >> 44);
            const double* Eu = E + u * kES16;
            const double* hr = h + offr;
            double best;
            switch (p) {
                case 2: best = Eu[__ffs(r) - 1]; break;  // w[u][v] + 0.0
                case 3: best = hk_relax_g<2>(Eu, hr, r); break;
                case 4: best = hk_relax_g<3>(Eu, hr, r); break;
                case 5: best = hk_relax_g<4>(Eu, hr, r); break;
                case 6: best = hk_relax_g<5>(Eu, hr, r); break;
                case 7: best = hk_relax_g<6>(Eu, hr, r); break;
                case 8: best = hk_relax_g<7>(Eu, hr, r); break;
                case 9: best = hk_relax_g<8>(Eu, hr, r); break;
                case 10: best = hk_relax_g<9>(Eu, hr, r); break;
                case 11: best = hk_relax_g<10>(Eu, hr, r); break;
                case 12: best = hk_relax_g<11>(Eu, hr, r); break;
                case 13: best = hk_relax_g<12>(Eu, hr, r); break;
                case 14: best = hk_relax_g<13>(Eu, hr, r); break;
                case 15: best = hk_relax_g<14>(Eu, hr, r); break;
                default: best = hk_relax_g<15>(Eu, hr, r); break;
            }
            h[dst] = best;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double* hf = h + t.off[(1 << k) - 1];
        double tot = hf[0];
        for (int u = 1; u < k; u++) tot = dmin(tot, hf[u]);
        red[0] = tot;
    }
    __syncthreads();
    return red[0];
}

__device__ __forceinline__ double hk_at_big(const double* h, const uint32_t* off, int s, int u) {
    if ((s & (s - 1)) == 0) return 0.0;
    return h[off[s] + __popc(s & ((1 << u) - 1))];
}

// lexicographically smallest optimal walk (combinatorics.py:277-296); one thread
__device__ inline void held_karp_order_big(int k, const double* E, const double* h, const uint32_t* off, double total,
                                           int8_t* order) {
    if (k == 1) {
        order[0] = 0;
        return;
    }
    int full = (1 << k) - 1;
    int start = 0;
    while (start < k - 1 && hk_at_big(h, off, full, start) != total) start++;
    order[0] = (int8_t)start;
    int s = full ^ (1 << start), cur = start, n = 1;
    double target = total;
    while (s) {
        int rem = s, took = 0;
        while (rem) {
            int u = __ffs(rem) - 1;
            rem &= rem - 1;
            double hv = hk_at_big(h, off, s, u);
            if (E[cur * kES16 + u] + hv == target) {
                order[n++] = (int8_t)u;
                target = hv;
                cur = u;
                s ^= 1 << u;
                took = 1;
                break;
            }
        }
        if (!took) {
            for (; n < k; n++) order[n] = -1;
            return;
        }
    }
}

// CTA-wide scratch in shared memory (besides the global Held-Karp slice)
struct CtaScratch {
    double* rows;  // k*m row sums
    double* E;     // 16 x 17
    double* pg;    // 16
    double* red;   // 2
    uint32_t* wk;  // kMatchWarps key blocks of m x (m | 1) (warp_bottleneck; unused by the 8 x 8 u16 path)
};

constexpr int kMatchWarps = 4;  // warps of a CTA that solve the m != 8 bottleneck matchings

__host__ __device__ inline size_t cta_wkeys_bytes(int m, int warps) { return (size_t)warps * m * (m | 1) * 4; }

__host__ __device__ inline size_t cta_scratch_bytes(int k, int m) {
    return ((size_t)k * m * 8 + 15) / 16 * 16 + 16 * kES16 * 8 + 16 * 8 + 16 +
           (cta_wkeys_bytes(m, kMatchWarps) + 15) / 16 * 16;
}

__device__ inline CtaScratch cta_scratch_at(unsigned char* base, int k, int m) {
    CtaScratch c;
    c.rows = reinterpret_cast<double*>(base);
    base += ((size_t)k * m * 8 + 15) / 16 * 16;
    c.E = reinterpret_cast<double*>(base);
    base += 16 * kES16 * 8;
    c.pg = reinterpret_cast<double*>(base);
    base += 16 * 8;
    c.red = reinterpret_cast<double*>(base);
    base += 16;
    c.wk = reinterpret_cast<uint32_t*>(base);
    return c;
}

// All threads of the CTA stage the partition in mem[k*m] (smem): cs.pg gets
// per_group_datap (costmodel.py:154-175), cs.E the coarsened stage graph
// (bottleneck edges, costmodel.py:200-208, zero diagonal).  Returns datap.
template <typename KeyT, bool kM8>
__device__ inline double cta_stage(int n, int k, int m_rt, const double* DP, const KeyT* RK, const double* vals,
                                   const CtaScratch& cs, const int16_t* mem, int ds = 0, int rs = 0) {
    if (!ds) ds = n;  // row strides (padded when the tables sit in shared memory)
    if (!rs) rs = n;
    const int m = kM8 ? 8 : m_rt, km = k * m;
    for (int r = threadIdx.x; r < km; r += blockDim.x) {
        int g = r / m;
        const int16_t* gm = mem + g * m;
        const double* row = DP + (size_t)gm[r - g * m] * ds;
        cs.rows[r] = pairwise_sum(m, [&](int c) { return row[gm[c]]; });
    }
    __syncthreads();
    if (threadIdx.x < k) {
        double mx = cs.rows[threadIdx.x * m];
        for (int i = 1; i < m; i++) mx = dmax(mx, cs.rows[threadIdx.x * m + i]);
        cs.pg[threadIdx.x] = mx;
    }
    const int npairs = k * (k - 1) / 2;
    if (kM8) {  // one thread per pair: the branch-free 8 x 8 subset DP
        for (int tt = threadIdx.x; tt < npairs; tt += blockDim.x) {
            int j, j2;
            decode_pair(tt, k, j, j2);
            const int16_t* A = mem + j * m;
            const int16_t* B = mem + j2 * m;
            const uint32_t L = match8_dp([&](int r, uint32_t(&kn)[4]) {
                const KeyT* row = RK + (size_t)A[r] * rs;
#pragma unroll
                for (int q = 0; q < 4; q++) kn[q] = (uint32_t)row[B[q]] | ((uint32_t)row[B[q + 4]] << 16);
            });
            double v = vals[L];
            cs.E[j * kES16 + j2] = v;
            cs.E[j2 * kES16 + j] = v;
        }
    } else {  // one warp per pair (warp_bottleneck on a staged key block)
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        const int MW = min(kMatchWarps, (int)(blockDim.x >> 5)), ks = m | 1;
        if (wid < MW) {
            uint32_t* wk = cs.wk + (size_t)wid * m * ks;
            for (int tt = wid; tt < npairs; tt += MW) {
                int j, j2;
                decode_pair(tt, k, j, j2);
                const int16_t* A = mem + j * m;
                const int16_t* B = mem + j2 * m;
                for (int c = lane; c < m; c += kWarp) {
                    const int bc = B[c];
                    for (int r = 0; r < m; r++) wk[r * ks + c] = (uint32_t)RK[(size_t)A[r] * rs + bc];
                }
                __syncwarp();
                const uint32_t L = warp_bottleneck<uint32_t>(m, wk, ks, lane);
                if (lane == 0) {
                    const double v = vals[L];
                    cs.E[j * kES16 + j2] = v;
                    cs.E[j2 * kES16 + j] = v;
                }
                __syncwarp();
            }
        }
    }
    if (threadIdx.x < k) cs.E[threadIdx.x * kES16 + threadIdx.x] = 0.0;
    __syncthreads();
    double dp = cs.pg[0];
    for (int g = 1; g < k; g++) dp = dmax(dp, cs.pg[g]);
    return dp;
}

// All threads of the CTA price the partition in mem[k*m] (smem).  Returns
// (datap, pipe) in every thread; cs.pg holds per_group_datap and h the
// Held-Karp table (for order reconstruction).
template <typename KeyT, bool kM8>
__device__ inline void cta_price(int n, int k, int m_rt, const double* DP, const KeyT* RK, const double* vals,
                                 const HKBig& t, const CtaScratch& cs, double* h, const int16_t* mem, double& datap,
                                 double& pipe, int ds = 0, int rs = 0) {
    datap = cta_stage<KeyT, kM8>(n, k, m_rt, DP, RK, vals, cs, mem, ds, rs);
    pipe = cta_held_karp(k, cs.E, h, t, cs.red);
}


// ---------------------------------------------------------------------------
// open_loop_tsp(heuristic=True) for k > 16 (combinatorics.py:299-342): nearest
// neighbour from every start (ties to the smaller vertex), first-improvement
// 2-opt with free path ends, cheapest float total wins, orientation
// canonicalised.  One thread; O(k^4) like the reference.
__device__ inline double path_cost_k(const double* E, int es, const int8_t* o, int k) {
    double t = 0.0;
    for (int i = k - 2; i >= 0; i--) t = E[o[i] * es + o[i + 1]] + t;
    return t;
}

__device__ inline void two_opt_k(const double* E, int es, int8_t* o, int k) {
    bool improved = true;
    while (improved) {
        improved = false;
        for (int i = 0; i < k - 1; i++) {
            for (int j = i + 1; j < k; j++) {
                double before = 0.0, after = 0.0;
                if (i > 0) {
                    before += E[o[i - 1] * es + o[i]];
                    after += E[o[i - 1] * es + o[j]];
                }
                if (j < k - 1) {
                    before += E[o[j] * es + o[j + 1]];
                    after += E[o[i] * es + o[j + 1]];
                }
                if (after < before) {
                    for (int x = i, y = j; x < y; x++, y--) {
                        int8_t t = o[x];
                        o[x] = o[y];
                        o[y] = t;
                    }
                    improved = true;
                }
            }
        }
    }
}

__device__ inline double nn_two_opt(const double* E, int es, int k, int8_t* best, int8_t* o) {
    double best_total = kInf;
    for (int start = 0; start < k; start++) {
        uint64_t left = (k == 64 ? ~0ull : ((1ull << k) - 1)) & ~(1ull << start);
        o[0] = (int8_t)start;
        for (int t = 1; t < k; t++) {
            int cur = o[t - 1], nxt = -1;
            double bv = 0.0;
            uint64_t l = left;
            while (l) {
                int v = __ffsll((long long)l) - 1;
                l &= l - 1;
                double x = E[cur * es + v];
                if (nxt < 0 || x < bv) {  // min by (w, v)
                    bv = x;
                    nxt = v;
                }
            }
            o[t] = (int8_t)nxt;
            left &= ~(1ull << nxt);
        }
        two_opt_k(E, es, o, k);
        double tot = path_cost_k(E, es, o, k);
        if (tot < best_total) {
            best_total = tot;
            for (int i = 0; i < k; i++) best[i] = o[i];
        }
    }
    if (best[0] > best[k - 1])
        for (int x = 0, y = k - 1; x < y; x++, y--) {
            int8_t t = best[x];
            best[x] = best[y];
            best[y] = t;
        }
    return path_cost_k(E, es, best, k);
}

}  // namespace hs
