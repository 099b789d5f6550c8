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

// Warp-cooperative version of the same value for an m x m key block staged
// in shared memory (m <= 64, row stride ks odd so row-wise and column-wise
// lane reads are both conflict-free).  Lane l owns columns l and l + 32:
// their adjacency over rows at the current threshold (u64), the row they
// are matched to and their BFS parent.  Per inserted row, a BFS level is
// two ballots (columns newly reached, free ones among them) and two OR
// reductions (their matched rows join the tree); a Hall violator raises the
// threshold to the warp-wide minimum key leaving the tree, exactly as
// bottleneck_threshold does, so the returned key is the same (the
// bottleneck of a matrix does not depend on which matching attains it).
template <typename Key>
__device__ Key warp_bottleneck(int m, const Key* K, int ks, int lane) {
    constexpr unsigned kF = 0xffffffffu;
    const int c0 = lane, c1 = lane + 32;
    const bool h0 = c0 < m, h1 = c1 < m;
    // lower bound: max of the row minima and the column minima
    unsigned lb = 0;
    {
        Key cm0 = (Key)~(Key)0, cm1 = cm0, rm0 = cm0, rm1 = cm0;
        for (int i = 0; i < m; i++) {
            if (h0) {
                const Key a = K[i * ks + c0], b = K[c0 * ks + i];
                cm0 = a < cm0 ? a : cm0;
                rm0 = b < rm0 ? b : rm0;
            }
            if (h1) {
                const Key a = K[i * ks + c1], b = K[c1 * ks + i];
                cm1 = a < cm1 ? a : cm1;
                rm1 = b < rm1 ? b : rm1;
            }
        }
        if (h0) lb = max(lb, (unsigned)max(cm0, rm0));
        if (h1) lb = max(lb, (unsigned)max(cm1, rm1));
    }
    Key L = (Key)__reduce_max_sync(kF, lb);
    uint64_t at0 = 0, at1 = 0;  // rows r with K[r][c] <= L
    auto build = [&]() {
        at0 = at1 = 0;
        for (int r = 0; r < m; r++) {
            if (h0 && K[r * ks + c0] <= L) at0 |= 1ull << r;
            if (h1 && K[r * ks + c1] <= L) at1 |= 1ull << r;
        }
    };
    build();
    int mc0 = -1, mc1 = -1;  // row matched to column c0 / c1
    int mr0 = -1, mr1 = -1;  // column matched to row lane / lane + 32
    for (int u = 0; u < m; u++) {
        uint64_t rows_in = 1ull << u, cols_in = 0, F = rows_in;
        int p0 = -1, p1 = -1, found = -1;
        for (;;) {
            const bool n0 = h0 && !(cols_in >> c0 & 1ull) && (at0 & F);
            const bool n1 = h1 && !(cols_in >> c1 & 1ull) && (at1 & F);
            if (n0) p0 = __ffsll((long long)(at0 & F)) - 1;
            if (n1) p1 = __ffsll((long long)(at1 & F)) - 1;
            const uint64_t nc = (uint64_t)__ballot_sync(kF, n0) | ((uint64_t)__ballot_sync(kF, n1) << 32);
            if (nc) {
                cols_in |= nc;
                const uint64_t fr = (uint64_t)__ballot_sync(kF, n0 && mc0 < 0) |
                                    ((uint64_t)__ballot_sync(kF, n1 && mc1 < 0) << 32);
                if (fr) {
                    found = __ffsll((long long)fr) - 1;
                    break;
                }
                // every new column is matched: its row joins the tree
                unsigned lo = 0, hi = 0;
                if (n0) (mc0 < 32 ? lo : hi) |= 1u << (mc0 & 31);
                if (n1) (mc1 < 32 ? lo : hi) |= 1u << (mc1 & 31);
                lo = __reduce_or_sync(kF, lo);
                hi = __reduce_or_sync(kF, hi);
                F = ((uint64_t)hi << 32) | lo;
                rows_in |= F;
                continue;
            }
            // Hall violator: raise to the cheapest edge leaving the tree
            unsigned x = 0xffffffffu;
            for (uint64_t rs = rows_in; rs; rs &= rs - 1) {
                const int r = __ffsll((long long)rs) - 1;
                if (h0 && !(cols_in >> c0 & 1ull)) x = min(x, (unsigned)K[r * ks + c0]);
                if (h1 && !(cols_in >> c1 & 1ull)) x = min(x, (unsigned)K[r * ks + c1]);
            }
            L = (Key)__reduce_min_sync(kF, x);
            build();
            F = rows_in;
        }
        // flip the alternating path found -> ... -> u
        int c = found;
        for (;;) {
            const int r = __shfl_sync(kF, c < 32 ? p0 : p1, c & 31);
            const int pc = __shfl_sync(kF, r < 32 ? mr0 : mr1, r & 31);
            if (lane == (c & 31)) {
                if (c < 32)
                    mc0 = r;
                else
                    mc1 = r;
            }
            if (lane == (r & 31)) {
                if (r < 32)
                    mr0 = c;
                else
                    mr1 = c;
            }
            if (r == u) break;
            c = pc;
        }
    }
    return L;
}

// ---------------------------------------------------------------------------
// 8 x 8 bottleneck matching, register resident.
//
// K[r][q] packs the uint16 keys of columns q (low half) and q+4 (high half)
// of row r; keys must be < 0x8000.  Adjacency at threshold L is one uint64
// (bit 8r+c), built branch-free: per half, (0x8000|L) - key has bit 15 set
// iff key <= L, and never borrows across halves.  Matching state lives in
// packed fields (row -> column nibbles, column -> row bit bytes), so a BFS
// step takes all of a row's new columns at once without a per-column loop.
// bit i of x (i < 8) -> nibble i = 0xF
__device__ __forceinline__ uint32_t nibble_mask(uint32_t x) {
    uint32_t t = (x & 0xFu) | ((x & 0xF0u) << 12);
    t = (t | (t << 6)) & 0x03030303u;
    t = (t | (t << 3)) & 0x11111111u;
    return t * 0xFu;
}

// bit i of x (i < 4) -> byte i = 0xFF
__device__ __forceinline__ uint32_t byte_mask4(uint32_t x) { return ((x * 0x00204081u) & 0x01010101u) * 0xFFu; }

struct Match8 {
    __device__ __forceinline__ static uint32_t get4(uint32_t x, int i) { return (x >> (4 * i)) & 0xFu; }
    __device__ __forceinline__ static uint32_t set4(uint32_t x, int i, uint32_t v) {
        return (x & ~(0xFu << (4 * i))) | (v << (4 * i));
    }

    __device__ __forceinline__ static uint64_t adjacency(const uint32_t (&K)[8][4], uint32_t L) {
        const uint32_t Lp = (L | (L << 16)) | 0x80008000u;
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int r = 0; r < 8; r++) {
            uint32_t t = ((Lp - K[r][0]) >> 15) & 0x00010001u;
            t |= ((Lp - K[r][1]) >> 14) & 0x00020002u;
            t |= ((Lp - K[r][2]) >> 13) & 0x00040004u;
            t |= ((Lp - K[r][3]) >> 12) & 0x00080008u;
            uint32_t row = (t | (t >> 12)) & 0xFFu;
            if (r < 4)
                lo |= row << (8 * r);
            else
                hi |= row << (8 * (r - 4));
        }
        return ((uint64_t)hi << 32) | lo;
    }

    __device__ static uint32_t solve(const uint32_t (&K)[8][4]) {
        // lower bound: every row and every column needs one selected entry
        uint32_t cm0 = 0xFFFFFFFFu, cm1 = 0xFFFFFFFFu, cm2 = 0xFFFFFFFFu, cm3 = 0xFFFFFFFFu;
        uint32_t L = 0;
#pragma unroll
        for (int r = 0; r < 8; r++) {
            uint32_t t = __vminu2(__vminu2(K[r][0], K[r][1]), __vminu2(K[r][2], K[r][3]));
            L = max(L, min(t & 0xFFFFu, t >> 16));
            cm0 = __vminu2(cm0, K[r][0]);
            cm1 = __vminu2(cm1, K[r][1]);
            cm2 = __vminu2(cm2, K[r][2]);
            cm3 = __vminu2(cm3, K[r][3]);
        }
        uint32_t c2 = __vmaxu2(__vmaxu2(cm0, cm1), __vmaxu2(cm2, cm3));
        L = max(L, max(c2 & 0xFFFFu, c2 >> 16));
        uint64_t adj = adjacency(K, L);
        // matching: mrow row -> column nibble (0xF free); mc byte c = bit of
        // the row holding column c (0 if free); mcols = held columns
        uint32_t mrow = 0xFFFFFFFFu, mc_lo = 0, mc_hi = 0, mcols = 0, unmatched = 0;
#pragma unroll
        for (int r = 0; r < 8; r++) {
            uint32_t av = (uint32_t)(adj >> (8 * r)) & 0xFFu & ~mcols;
            if (av) {
                uint32_t c = __ffs(av) - 1;
                mcols |= 1u << c;
                mrow = set4(mrow, r, c);
                if (c < 4)
                    mc_lo |= (1u << r) << (8 * c);
                else
                    mc_hi |= (1u << r) << (8 * (c - 4));
            } else {
                unmatched |= 1u << r;
            }
        }
        while (unmatched) {
            int u = __ffs(unmatched) - 1;
            unmatched &= unmatched - 1;
            uint32_t rows_in = 1u << u, cols_in = 0, frontier = rows_in, parent = 0;
            int found = -1;
            for (;;) {
                // alternating BFS; a popped row takes all its new columns at
                // once (bit-parallel), stopping at the lowest free one
                while (frontier) {
                    uint32_t r = __ffs(frontier) - 1;
                    frontier &= frontier - 1;
                    uint32_t cand = (uint32_t)(adj >> (8 * r)) & 0xFFu & ~cols_in;
                    uint32_t nib = nibble_mask(cand);
                    parent = (parent & ~nib) | (nib & (r * 0x11111111u));
                    cols_in |= cand;
                    uint32_t fr = cand & ~mcols;
                    if (fr) {
                        found = __ffs(fr) - 1;
                        break;
                    }
                    uint32_t nr = (mc_lo & byte_mask4(cand & 0xFu)) | (mc_hi & byte_mask4(cand >> 4));
                    nr |= nr >> 16;
                    nr = (nr | (nr >> 8)) & 0xFFu;
                    rows_in |= nr;
                    frontier |= nr;
                }
                if (found >= 0) break;
                // Hall violator: the optimum needs an edge leaving the tree;
                // raise L to the cheapest such edge.
                uint32_t M[4];
#pragma unroll
                for (int q = 0; q < 4; q++)
                    M[q] = ((cols_in >> q) & 1u ? 0x0000FFFFu : 0u) | ((cols_in >> (q + 4)) & 1u ? 0xFFFF0000u : 0u);
                uint32_t acc = 0xFFFFFFFFu;
#pragma unroll
                for (int r = 0; r < 8; r++) {
                    uint32_t t = __vminu2(__vminu2(K[r][0] | M[0], K[r][1] | M[1]),
                                          __vminu2(K[r][2] | M[2], K[r][3] | M[3]));
                    acc = __vminu2(acc, (rows_in >> r) & 1u ? t : 0xFFFFFFFFu);
                }
                L = min(acc & 0xFFFFu, acc >> 16);
                adj = adjacency(K, L);
                frontier = rows_in;
            }
            // flip the path back to the root
            mcols |= 1u << found;
            uint32_t c = (uint32_t)found;
            for (;;) {
                uint32_t r = get4(parent, c);
                uint32_t pc = get4(mrow, r);
                mrow = set4(mrow, r, c);
                uint32_t sh = 8 * (c & 3), rb = (1u << r) << sh, keep = ~(0xFFu << sh);
                if (c < 4)
                    mc_lo = (mc_lo & keep) | rb;
                else
                    mc_hi = (mc_hi & keep) | rb;
                if (r == (uint32_t)u) break;
                c = pc;
            }
        }
        return L;
    }
};

// ---------------------------------------------------------------------------
// Held-Karp over E (k x k, row stride kES) by one warp, k <= 8.
//
// Compact table: h[off[s] + rank(u in s)] for u in s, |s| >= 2 (layer 1 is
// implicit 0.0).  Iterating v over the bits of r = s\u in ascending order
// visits h[off[r] + i] at consecutive i, so that address is base + const.
// Each state is pre-decoded on the host into 16 bytes (hk_schedule):
//   x = off[r]*8 | dst*8 << 16          (byte offsets into h)
//   y = v0*8 | v1*8 << 8 | v2*8 << 16 | v3*8 << 24
//   z = v4*8 | v5*8 << 8 | v6*8 << 16 | (u*kES) << 24
//   w = r | u << 8                      (for debugging / tools)
// so one relaxation is PRMT + IADD + 2 LDS + DADD + DSETP + 2 FSEL.
// Layers p = |s| live in [lay[p], lay[p+1]).
constexpr int kES = 9;  // padded E row stride (bank spread)

template <int I>
__device__ __forceinline__ uint32_t hk_vbyte(uint32_t y, uint32_t z) {
    return I < 4 ? __byte_perm(y, 0u, 0x4440u + I) : __byte_perm(z, 0u, 0x4440u + (I - 4));
}

template <int NV>
__device__ __forceinline__ double hk_relax(const char* Eu, const char* hr, uint32_t y, uint32_t z) {
    double best = *reinterpret_cast<const double*>(Eu + hk_vbyte<0>(y, z)) + *reinterpret_cast<const double*>(hr);
#pragma unroll
    for (int i = 1; i < NV; i++) {
        uint32_t vb = i < 4 ? __byte_perm(y, 0u, 0x4440u + i) : __byte_perm(z, 0u, 0x4440u + (i - 4));
        double c = *reinterpret_cast<const double*>(Eu + vb) + *reinterpret_cast<const double*>(hr + 8 * i);
        best = c < best ? c : best;
    }
    return best;
}

template <int NV>
__device__ __forceinline__ void hk_layer(const char* Eb, char* hb, const uint4* states, int beg, int end, int lane) {
    for (int idx = beg + lane; idx < end; idx += kWarp) {
        const uint4 st = states[idx];
        const char* Eu = Eb + (st.z >> 24) * 8;
        double best;
        if (NV == 1)  // w[u][v] + 0.0 == w[u][v]
            best = *reinterpret_cast<const double*>(Eu + (st.y & 0xFFu));
        else
            best = hk_relax<NV>(Eu, hb + (st.x & 0xFFFFu), st.y, st.z);
        *reinterpret_cast<double*>(hb + (st.x >> 16)) = best;
    }
}

__device__ inline double warp_held_karp(int k, const double* E, double* h, const uint4* states, const int* lay,
                                        int lane, int final_off) {
    if (k == 1) return 0.0;
    const char* Eb = reinterpret_cast<const char*>(E);
    char* hb = reinterpret_cast<char*>(h);
    for (int p = 2; p <= k; p++) {
        const int beg = lay[p], end = lay[p + 1];
        switch (p) {
            case 2: hk_layer<1>(Eb, hb, states, beg, end, lane); break;
            case 3: hk_layer<2>(Eb, hb, states, beg, end, lane); break;
            case 4: hk_layer<3>(Eb, hb, states, beg, end, lane); break;
            case 5: hk_layer<4>(Eb, hb, states, beg, end, lane); break;
            case 6: hk_layer<5>(Eb, hb, states, beg, end, lane); break;
            case 7: hk_layer<6>(Eb, hb, states, beg, end, lane); break;
            default: hk_layer<7>(Eb, hb, states, beg, end, lane); break;
        }
        __syncwarp();
    }
    // the full set's k entries (compact table: the last k of k*2^(k-1) - k)
    const double* hf = h + final_off;
    double tot = hf[0];
    for (int u = 1; u < k; u++) tot = dmin(tot, hf[u]);
    return tot;
}

// compact index of (s, u), u in s, |s| >= 2
__device__ __forceinline__ double hk_at(const double* h, const uint16_t* hoff, int s, int u) {
    if ((s & (s - 1)) == 0) return 0.0;
    return h[hoff[s] + __popc(s & ((1 << u) - 1))];
}

// Lexicographically smallest optimal walk (combinatorics.py:277-296).
__device__ inline void held_karp_order(int k, const double* E, const double* h, const uint16_t* hoff, double total,
                                       int8_t* order) {
    if (k == 1) {
        order[0] = 0;
        return;
    }
    int full = (1 << k) - 1;
    int start = 0;
    while (start < k - 1 && hk_at(h, hoff, full, start) != total) start++;
    order[0] = (int8_t)start;
    int s = full ^ (1 << start), cur = start, n = 1;
    double target = total;
    while (s) {
        int rem = s, took = 0;
        while (rem) {
            int u = __ffs(rem) - 1;
            rem &= rem - 1;
            double hv = hk_at(h, hoff, s, u);
            if (E[cur * kES + u] + hv == target) {
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
