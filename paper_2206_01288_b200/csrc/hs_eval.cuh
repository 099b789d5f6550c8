// hs_eval.cuh -- device building blocks of the fitness evaluation (K0/K1).
//
//   bottleneck_threshold : smallest entry v of an m x m matrix such that the
//                          entries <= v admit a perfect matching.  Same value
//                          as combinatorics.py:106-131 (binary search over
//                          np.unique + Kuhn), computed here by a bottleneck
//                          Hungarian search with uint64 row masks: start at
//                          the row/column-minimum lower bound, grow alternating
//                          trees, and raise the threshold only to the cheapest
//                          edge leaving a Hall-violating tree.
//   warp_held_karp       : Held-Karp over the coarsened k x k stage graph,
//                          one warp, layer by layer (popcount), table in smem.
//                          h[s][u] = min_v (w[u][v] + h[s\u][v]) -- the suffix
//                          association of combinatorics.py:267-276, so totals
//                          are bit-identical (fp add is monotone, hence min
//                          over suffixes commutes with the outer add).
#pragma once
#include "hs_common.cuh"

namespace hs {

constexpr int kMaxM = 64;     // uint64 masks
constexpr int kWarpK = 8;     // warp kernel handles d_pp <= 8
constexpr int kHS = 8;        // HK row stride (u index)

// R(r, c) returns an ordered key (rank or value) of entry (r, c).
template <typename Key, typename At>
__device__ Key bottleneck_threshold(int m, const At& R, Key key_max) {
    Key L = 0;
    for (int r = 0; r < m; r++) {
        Key mn = key_max;
        for (int c = 0; c < m; c++) {
            Key x = R(r, c);
            mn = x < mn ? x : mn;
        }
        L = mn > L ? mn : L;
    }
    for (int c = 0; c < m; c++) {
        Key mn = key_max;
        for (int r = 0; r < m; r++) {
            Key x = R(r, c);
            mn = x < mn ? x : mn;
        }
        L = mn > L ? mn : L;
    }
    int8_t match_col[kMaxM], match_row[kMaxM], parent[kMaxM];
    for (int i = 0; i < m; i++) match_col[i] = match_row[i] = -1;
    for (int u = 0; u < m; u++) {
        uint64_t rows_in = 1ull << u, cols_in = 0, frontier = rows_in;
        int found = -1;
        for (;;) {
            while (frontier && found < 0) {
                int r = __ffsll((long long)frontier) - 1;
                frontier &= frontier - 1;
                uint64_t cand = 0;
                for (int c = 0; c < m; c++)
                    if (R(r, c) <= L) cand |= 1ull << c;
                cand &= ~cols_in;
                while (cand) {
                    int c = __ffsll((long long)cand) - 1;
                    cand &= cand - 1;
                    parent[c] = (int8_t)r;
                    cols_in |= 1ull << c;
                    if (match_col[c] < 0) {
                        found = c;
                        break;
                    }
                    int rr = match_col[c];
                    rows_in |= 1ull << rr;
                    frontier |= 1ull << rr;
                }
            }
            if (found >= 0) break;
            // Hall violator: raise to the cheapest edge leaving the tree.
            Key nl = key_max;
            uint64_t rs = rows_in;
            while (rs) {
                int r = __ffsll((long long)rs) - 1;
                rs &= rs - 1;
                for (int c = 0; c < m; c++) {
                    if (cols_in >> c & 1) continue;
                    Key x = R(r, c);
                    nl = x < nl ? x : nl;
                }
            }
            L = nl;
            frontier = rows_in;
        }
        int c = found;
        for (;;) {
            int r = parent[c];
            int pc = match_row[r];
            match_row[r] = (int8_t)c;
            match_col[c] = (int8_t)r;
            if (r == u) break;
            c = pc;
        }
    }
    return L;
}

// Held-Karp over E (k x k, row stride kHS) by one warp.  h: 2^k * kHS
// doubles (layers >= 2 written; layer 1 is implicit 0.0).  states:
// (s | u << 8) grouped by |s|, layer p in [off[p], off[p+1]).
__device__ __forceinline__ double hk_value(const double* h, int s, int u) {
    return (s & (s - 1)) == 0 ? 0.0 : h[s * kHS + u];
}

__device__ inline double warp_held_karp(int k, const double* E, double* h, const uint16_t* states,
                                        const int* off, int lane) {
    if (k == 1) return 0.0;
    for (int p = 2; p <= k; p++) {
        for (int idx = off[p] + lane; idx < off[p + 1]; idx += kWarp) {
            uint32_t st = states[idx];
            int s = st & 0xff, u = st >> 8;
            int r = s ^ (1 << u);
            const double* Eu = E + u * kHS;
            double best;
            if (p == 2) {
                best = Eu[__ffs(r) - 1];  // w[u][v] + 0.0 == w[u][v]
            } else {
                best = kInf;
                const double* hr = h + r * kHS;
                int rr = r;
                while (rr) {
                    int v = __ffs(rr) - 1;
                    rr &= rr - 1;
                    double c = Eu[v] + hr[v];
                    best = c < best ? c : best;
                }
            }
            h[s * kHS + u] = best;
        }
        __syncwarp();
    }
    int full = (1 << k) - 1;
    double tot = h[full * kHS];
    for (int u = 1; u < k; u++) tot = dmin(tot, h[full * kHS + u]);
    return tot;
}

// Lexicographically smallest optimal walk (combinatorics.py:277-296).
__device__ inline void held_karp_order(int k, const double* E, const double* h, double total,
                                       int8_t* order) {
    if (k == 1) {
        order[0] = 0;
        return;
    }
    int full = (1 << k) - 1;
    int start = 0;
    while (h[full * kHS + start] != total) start++;
    order[0] = (int8_t)start;
    int s = full ^ (1 << start), cur = start, n = 1;
    double target = total;
    while (s) {
        int rem = s, took = 0;
        while (rem) {
            int u = __ffs(rem) - 1;
            rem &= rem - 1;
            double hv = hk_value(h, s, u);
            if (E[cur * kHS + u] + hv == target) {
                order[n++] = (int8_t)u;
                target = hv;
                cur = u;
                s ^= 1 << u;
                took = 1;
                break;
            }
        }
        if (!took) {  // table inconsistent with its recurrence (cannot happen)
            for (; n < k; n++) order[n] = -1;
            return;
        }
    }
}

}  // namespace hs
