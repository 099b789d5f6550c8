// hs_search_impl.cuh -- device code of K2/K3 (included by the hs_search*.cu
// translation units; the GA / refine kernel variants are instantiated in
// hs_search_ga_{warp,cta}.cu and hs_search_refine.cu so they compile in
// parallel).
#pragma once
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
#include <cfloat>
#include <climits>

#include "hs_rng.cuh"
#include "hs_search.h"
#include "hs_cta_eval.cuh"
#include "hs_warp_eval.cuh"

namespace hs {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void warp_argmin(double& v, int& i) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        double v2 = __shfl_xor_sync(kFull, v, o);
        int i2 = __shfl_xor_sync(kFull, i, o);
        if (v2 < v || (v2 == v && i2 < i)) {
            v = v2;
            i = i2;
        }
    }
}

__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        double v2 = __shfl_xor_sync(kFull, v, o);
        int i2 = __shfl_xor_sync(kFull, i, o);
        if (v2 > v || (v2 == v && i2 < i)) {
            v = v2;
            i = i2;
        }
    }
}

// numpy pairwise sum of an array (any n; recursion only beyond 128)
__device__ inline double pw_array(const double* a, int n) {
    if (n <= 128) return pairwise_sum(n, [&](int i) { return a[i]; });
    int n2 = n / 2;
    n2 -= n2 % 8;
    return pw_array(a, n2) + pw_array(a + n2, n - n2);
}

// ---------------------------------------------------------------------------
// driver-warp working state (shared memory)

struct LS {
    int n, k, m, cap;
    const double* W;  // surrogate weights n x n (scheduler.py:84-88)
    uint32_t w_sh;    // shared-window address of W when it was staged in shared memory, else 0
    bool lat;         // latency regime: one working warp per SM (CTA islands, refine, spec workers)
    int16_t* G;       // k x cap members, ascending
    int* sz;          // k sizes
    double* mean;     // n x k: mean[u*k+i] = seq_sum(W[u, G_i]) / sz_i, computed lazily
    uint32_t* mver;   // n x k: version of the group a mean entry was computed for
    uint32_t* cver;   // k: group content versions (bumped on every change)
    double* home;     // n: cheapest intra-group link of each device
    int* valid;       // [0]: mean columns valid, [1]: home groups valid, [2]: fast edges valid, [3]: best partners valid (bitmasks)
    int16_t* fe;      // k x 2 cached _fast_edge pairs
    double* bpv;      // n: each device's cheapest intra-group link (value) ...
    int16_t* bpp;     // n: ... and its partner (valid[3]: per group, groups of != 8 members)
    uint32_t* locked;  // n-bit set
    int* nlocked;
    int16_t* perm;    // C(k,2)
    double* f64;      // scratch: 4*cap (KL sums) and chain steps/closers
    int* i32;         // scratch: chain moves (3*k), misc
    int8_t* grp_of;   // n
};

__device__ __forceinline__ void g_remove(LS& s, int j, int d) {
    int16_t* g = s.G + j * s.cap;
    int c = s.sz[j], i = 0;
    while (i < c && g[i] != d) i++;
    for (; i + 1 < c; i++) g[i] = g[i + 1];
    s.sz[j] = c - 1;
}

__device__ __forceinline__ void g_insort(LS& s, int j, int d) {  // bisect.insort
    int16_t* g = s.G + j * s.cap;
    int i = s.sz[j];
    while (i > 0 && g[i - 1] > d) {
        g[i] = g[i - 1];
        i--;
    }
    g[i] = (int16_t)d;
    s.sz[j]++;
}

// _move (:294-296) by the whole warp: remove v from src, insort into dst.
// Members are distinct and ascending, so each element's new slot is its old
// index shifted by one past the removal / insertion point (ballots).
__device__ __forceinline__ void g_move_w(LS& s, int v, int src, int dst, int lane) {
    int16_t* gs = s.G + src * s.cap;
    int16_t* gd = s.G + dst * s.cap;
    const int cs = s.sz[src], cd = s.sz[dst];
    int16_t a[3], b[3];
    int below = 0, pos = INT_MAX;
#pragma unroll
    for (int q = 0; q < 3; q++) {
        int i = lane + 32 * q;
        a[q] = i < cs ? gs[i] : (int16_t)0x7fff;
        b[q] = i < cd ? gd[i] : (int16_t)0x7fff;
        unsigned hit = __ballot_sync(kFull, i < cs && a[q] == v);
        if (hit && pos == INT_MAX) pos = 32 * q + __ffs(hit) - 1;
        below += __popc(__ballot_sync(kFull, i < cd && b[q] < v));
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 3; q++) {
        int i = lane + 32 * q;
        if (i < cs && i != pos) gs[i < pos ? i : i - 1] = a[q];
        if (i < cd) gd[i < below ? i : i + 1] = b[q];
    }
    if (lane == 0) {
        gd[below] = (int16_t)v;
        s.sz[src] = cs - 1;
        s.sz[dst] = cd + 1;
    }
    __syncwarp();
}

// x / cnt, IEEE-exact: for a power-of-two count the reciprocal is exact, so
// the product is the same correctly rounded quotient.
__device__ __forceinline__ double div_count(double x, int cnt) {
    return (cnt & (cnt - 1)) == 0 ? x * (1.0 / (double)cnt) : x / (double)cnt;
}

// _swap (:252-257) by the whole warp, both groups in one pass: group j loses
// a and gains b, group j2 loses b and gains a.  New slot of a surviving
// member x: idx - (out < x) + (in < x); the incomer lands after every
// survivor below it.
__device__ __forceinline__ void swap_one(int16_t* g, int c, int out, int in, int lane) {
    int16_t x[3];
    int below = 0;
#pragma unroll
    for (int q = 0; q < 3; q++) {
        int i = lane + 32 * q;
        x[q] = i < c ? g[i] : (int16_t)0x7fff;
        if (32 * q < c) below += __popc(__ballot_sync(kFull, i < c && x[q] != out && x[q] < in));
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 3; q++) {
        int i = lane + 32 * q;
        if (i < c && x[q] != out) g[i - (out < x[q]) + (in < x[q])] = x[q];
    }
    if (lane == 0) g[below] = (int16_t)in;
    __syncwarp();
}

__device__ __forceinline__ void g_swap_w(LS& s, int a, int j, int b, int j2, int lane) {
    swap_one(s.G + j * s.cap, s.sz[j], a, b, lane);
    swap_one(s.G + j2 * s.cap, s.sz[j2], b, a, lane);
}

// numpy pairwise sum of exactly 8 lane-held values (lanes 8q..8q+7): the
// xor-1/2/4 butterfly is the ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree.
__device__ __forceinline__ double butterfly8(double x) {
    x += __shfl_xor_sync(kFull, x, 1);
    x += __shfl_xor_sync(kFull, x, 2);
    x += __shfl_xor_sync(kFull, x, 4);
    return x;
}

__device__ __forceinline__ double row_pw(const LS& s, int u, const int16_t* grp, int cnt) {
    const double* wr = s.W + (size_t)u * s.n;
    if (cnt < 8) {
        double r = 0.0;
        for (int i = 0; i < cnt; i++) r += wr[grp[i]];
        return r;
    }
    return pairwise_sum(cnt, [&](int i) { return wr[grp[i]]; });
}

__device__ __forceinline__ double row_seq_mean(const LS& s, int u, const int16_t* grp, int cnt) {
    const double* wr = s.W + (size_t)u * s.n;
    double r = 0.0;  // sequential: w[:, grp].mean(axis=1) reduces an F-contiguous array
    int i = 0;
    for (; i + 8 <= cnt; i += 8) {  // eight loads in flight, added in order
        double w[8];
#pragma unroll
        for (int t = 0; t < 8; t++) w[t] = wr[grp[i + t]];
#pragma unroll
        for (int t = 0; t < 8; t++) r += w[t];
    }
    for (; i < cnt; i++) r += wr[grp[i]];
    return div_count(r, cnt);
}

// mean[u][i] (_group_means, scheduler.py:279-284) on demand
__device__ __forceinline__ double mean_at(LS& s, int u, int i) {
    const int x = u * s.k + i;
    const uint32_t ver = s.cver[i];
    if (s.mver[x] != ver) {
        s.mean[x] = row_seq_mean(s, u, s.G + i * s.cap, s.sz[i]);
        s.mver[x] = ver;
    }
    return s.mean[x];
}

static __device__ long long* g_prof = nullptr;

// pair key: (smaller id, larger id) -- members ascend, so the reference's
// "first minimum in scan order" is the minimum by (value, key)
__device__ __forceinline__ int pair_key(int x, int y) { return x < y ? x * 1024 + y : y * 1024 + x; }

__device__ __forceinline__ void argmin_vk(double& v, int& key, int& who) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double v2 = __shfl_xor_sync(kFull, v, o);
        const int k2 = __shfl_xor_sync(kFull, key, o), w2 = __shfl_xor_sync(kFull, who, o);
        if (v2 < v || (v2 == v && k2 < key)) {
            v = v2;
            key = k2;
            who = w2;
        }
    }
}

// best partner of x in group g (c members), minimum by (W[x][y], key); the
// warp cooperates, every lane returns it (W is symmetric: scheduler.py:76)
__device__ inline void best_partner_row(const LS& s, const int16_t* g, int c, int x, int lane, double& bv, int& bp) {
    const double* wx = s.W + (size_t)x * s.n;
    double v = kInf;
    int key = INT_MAX, who = -1;
    for (int t = lane; t < c; t += kWarp) {
        const int y = g[t];
        if (y == x) continue;
        const double w = wx[y];
        const int ky = pair_key(x, y);
        if (w < v || (w == v && ky < key)) {
            v = w;
            key = ky;
            who = y;
        }
    }
    argmin_vk(v, key, who);
    bv = v;
    bp = who;
}

// _fast_edge (:237-249): lexicographically first minimum intra-group pair,
// cached per group until the group changes.  Groups of 8 (the common
// paper shape): lanes over the 28 position pairs.  Other sizes: the group's
// minimum over its members' best partners (bpv / bpp, built eight rows at a
// time when missing, then kept up to date swap by swap in pass_sweep).
__device__ inline void fast_edge(LS& s, int j, int lane, int& a, int& b) {
    if ((unsigned)s.valid[2] >> j & 1u) {
        a = s.fe[2 * j];
        b = s.fe[2 * j + 1];
        return;
    }
    long long f0 = clock64();
    const int16_t* g = s.G + j * s.cap;
    const int c = s.sz[j];
    if (c == 8) {
        double bv = kInf;
        int code = INT_MAX;
        if (lane < 28) {  // lane -> (i, l), i < l, lexicographic
            int i = 0, t = lane;
            while (t >= 7 - i) {
                t -= 7 - i;
                i++;
            }
            int l = i + 1 + t;
            bv = s.W[(size_t)g[i] * s.n + g[l]];
            code = i * 256 + l;
        }
        warp_argmin(bv, code);
        if (code == INT_MAX) code = 1;  // (grp[0], grp[1]) default
        a = g[code >> 8];
        b = g[code & 255];
    } else {
        if (!((unsigned)s.valid[3] >> j & 1u)) {
            // every member's best partner: eight rows at a time, lanes over
            // the partners (independent loads in flight), one argmin per row
            for (int i0 = 0; i0 < c; i0 += 8) {
                for (int l0 = 0; l0 < c; l0 += kWarp) {
                    double v[8];
                    const int l = l0 + lane;
                    const int y = l < c ? g[l] : -1;
#pragma unroll
                    for (int r = 0; r < 8; r++) {
                        const int i = i0 + r;
                        v[r] = (i < c && y >= 0 && l != i) ? s.W[(size_t)g[i] * s.n + y] : kInf;
                    }
#pragma unroll
                    for (int r = 0; r < 8; r++) {
                        const int i = i0 + r;
                        if (i >= c) break;
                        const int x = g[i];
                        double bv = v[r];
                        int key = (y >= 0 && l != i) ? pair_key(x, y) : INT_MAX, who = (y >= 0 && l != i) ? y : -1;
                        argmin_vk(bv, key, who);
                        if (l0 > 0) {  // merge with the earlier column chunk
                            const double ov = s.bpv[x];
                            const int op = s.bpp[x], ok = op >= 0 ? pair_key(x, op) : INT_MAX;
                            if (!(bv < ov || (bv == ov && key < ok))) {
                                bv = ov;
                                who = op;
                            }
                        }
                        __syncwarp();
                        if (lane == 0) {
                            s.bpv[x] = bv;
                            s.bpp[x] = (int16_t)who;
                        }
                        __syncwarp();
                    }
                }
            }
            if (lane == 0) s.valid[3] |= (int)(1u << j);
            __syncwarp();
        }
        // the group's fast edge: minimum over its members' best partners
        double bv = kInf;
        int key = INT_MAX, who = -1;
        for (int t = lane; t < c; t += kWarp) {
            const int x = g[t], y = s.bpp[x];
            if (y < 0) continue;
            const double v = s.bpv[x];
            const int ky = pair_key(x, y);
            if (v < bv || (v == bv && ky < key)) {
                bv = v;
                key = ky;
                who = x;
            }
        }
        argmin_vk(bv, key, who);
        if (key == INT_MAX) {
            a = g[0];  // fewer than two members: (grp[0], grp[1])
            b = g[1];
        } else {
            a = key >> 10;
            b = key & 1023;
        }
    }
    __syncwarp();
    if (lane == 0) {
        s.fe[2 * j] = (int16_t)a;
        s.fe[2 * j + 1] = (int16_t)b;
        s.valid[2] |= (int)(1u << j);
        if (g_prof) {
            g_prof[9] += clock64() - f0;
            g_prof[10] += 1;
        }
    }
    __syncwarp();
}

// group j lost `out` and gained `in` (a _swap); its members' best partners
// were valid before: the joiner scans its row, everyone else compares the
// joiner and re-scans only if its best partner was the one who left
__device__ inline void best_partners_swap(LS& s, int j, int out, int in, int lane) {
    const int16_t* g = s.G + j * s.cap;
    const int c = s.sz[j];
    const double* win = s.W + (size_t)in * s.n;
    // joiner's row (also each member's link to the joiner: W symmetric)
    double jv = kInf;
    int jkey = INT_MAX, jwho = -1;
    for (int t = lane; t < c; t += kWarp) {
        const int x = g[t];
        if (x == in) continue;
        const double w = win[x];
        const int kx = pair_key(in, x);
        if (w < jv || (w == jv && kx < jkey)) {
            jv = w;
            jkey = kx;
            jwho = x;
        }
        if (s.bpp[x] != out) {
            const double ov = s.bpv[x];
            const int ok = s.bpp[x] >= 0 ? pair_key(x, s.bpp[x]) : INT_MAX;
            if (w < ov || (w == ov && kx < ok)) {
                s.bpv[x] = w;
                s.bpp[x] = (int16_t)in;
            }
        }
    }
    argmin_vk(jv, jkey, jwho);
    __syncwarp();
    // members whose best partner left: a full row each
    for (int t0 = 0; t0 < c; t0 += kWarp) {
        const int t = t0 + lane;
        unsigned redo = __ballot_sync(kFull, t < c && g[t] != in && s.bpp[g[t]] == out);
        while (redo) {
            const int u = __ffs(redo) - 1;
            redo &= redo - 1;
            const int x = g[t0 + u];
            double bv;
            int bp;
            best_partner_row(s, g, c, x, lane, bv, bp);
            __syncwarp();
            if (lane == 0) {
                s.bpv[x] = bv;
                s.bpp[x] = (int16_t)bp;
            }
            __syncwarp();
        }
    }
    if (lane == 0) {
        s.bpv[in] = jv;
        s.bpp[in] = (int16_t)jwho;
        s.valid[3] |= (int)(1u << j);
    }
    __syncwarp();
}

// _best_candidate (:260-276) with _gain_ours (:206-209): the four candidates
// need only four row sums, computed by lanes 0..3.
__device__ inline double best_candidate(LS& s, int j, int j2, int lane, int& oa, int& ob) {
    int d1, d2, d1p, d2p;
    fast_edge(s, j, lane, d1, d2);
    fast_edge(s, j2, lane, d1p, d2p);
    const int16_t* gj = s.G + j * s.cap;
    const int16_t* gj2 = s.G + j2 * s.cap;
    int cj = s.sz[j], cj2 = s.sz[j2];
    double S0, S1, S2, S3;
    if (cj == 8 && cj2 == 8) {
        // four 8-term pairwise sums at once: lanes 8q..8q+7 hold one row each
        const int q = lane >> 3, e = lane & 7;
        const int u = q == 0 ? d1 : q == 1 ? d2 : q == 2 ? d1p : d2p;
        const int16_t* gg = q < 2 ? gj2 : gj;
        double x = butterfly8(s.W[(size_t)u * s.n + gg[e]]);
        S0 = __shfl_sync(kFull, x, 0);
        S1 = __shfl_sync(kFull, x, 8);
        S2 = __shfl_sync(kFull, x, 16);
        S3 = __shfl_sync(kFull, x, 24);
    } else if (cj >= 8 && cj2 >= 8 && cj <= 128 && cj2 <= 128) {
        // numpy pairwise sums of the four rows, lanes 8q..8q+7: lane e keeps
        // accumulator r_e (terms e, e + 8, ... in order), the xor butterfly
        // is numpy's tree, the tail is added in order by every lane
        const int q = lane >> 3, e = lane & 7;
        const int u = q == 0 ? d1 : q == 1 ? d2 : q == 2 ? d1p : d2p;
        const int16_t* gg = q < 2 ? gj2 : gj;
        const int c = q < 2 ? cj2 : cj, full = c - c % 8;
        const double* wr = s.W + (size_t)u * s.n;
        double r = wr[gg[e]];
        for (int i = 8 + e; i < full; i += 8) r += wr[gg[i]];
        double x = butterfly8(r);
        for (int i = full; i < c; i++) x += wr[gg[i]];
        S0 = __shfl_sync(kFull, x, 0);
        S1 = __shfl_sync(kFull, x, 8);
        S2 = __shfl_sync(kFull, x, 16);
        S3 = __shfl_sync(kFull, x, 24);
    } else {
        double sum = 0.0;
        if (lane < 4) {
            int u = lane == 0 ? d1 : lane == 1 ? d2 : lane == 2 ? d1p : d2p;
            sum = lane < 2 ? row_pw(s, u, gj2, cj2) : row_pw(s, u, gj, cj);
        }
        S0 = __shfl_sync(kFull, sum, 0);
        S1 = __shfl_sync(kFull, sum, 1);
        S2 = __shfl_sync(kFull, sum, 2);
        S3 = __shfl_sync(kFull, sum, 3);
    }
    const int n = s.n;
    double t1a = div_count(S0, cj2) - s.W[(size_t)d1 * n + d2];   // a = d1, pa = d2
    double t1b = div_count(S1, cj2) - s.W[(size_t)d2 * n + d1];   // a = d2, pa = d1
    double t2a = div_count(S2, cj) - s.W[(size_t)d1p * n + d2p];  // b = d1p, pb = d2p
    double t2b = div_count(S3, cj) - s.W[(size_t)d2p * n + d1p];  // b = d2p, pb = d1p
    double g[4] = {t1a + t2a, t1a + t2b, t1b + t2a, t1b + t2b};
    int A[4] = {d1, d1, d2, d2}, Bv[4] = {d1p, d2p, d1p, d2p};
    double best = -kInf;
    oa = d1;
    ob = d1p;
#pragma unroll
    for (int c = 0; c < 4; c++)
        if (g[c] > best) {
            best = g[c];
            oa = A[c];
            ob = Bv[c];
        }
    return best;
}

__device__ __forceinline__ void invalidate(LS& s, int j) {
    s.valid[1] &= (int)~(1u << j);
    s.valid[2] &= (int)~(1u << j);
    s.valid[3] &= (int)~(1u << j);
    s.cver[j]++;
}

// same, safe when several warps finish pairs at once (sweep waves)
__device__ __forceinline__ void invalidate_atomic(LS& s, int j) {
    atomicAnd(&s.valid[1], (int)~(1u << j));
    atomicAnd(&s.valid[2], (int)~(1u << j));
    atomicAnd(&s.valid[3], (int)~(1u << j));
    atomicAdd(&s.cver[j], 1u);
}

// ---------------------------------------------------------------------------
// Register-resident sweep of one group pair at d_dp = 8, n <= 128.
//
// Both groups live in every lane as 8 packed bytes (member i = byte i,
// ascending).  One _best_candidate round is: each lane prices one intra pair
// (i, l) of each group, the two lexicographic first minima come out of three
// REDUX.MIN stages on the order-preserving 64-bit image of the weight (high
// word, low word, pair code), lanes 4q.. form the four 8-term pairwise row
// sums of _gain_ours, and the swap is two byte-shifts of the packed words.
// No shared-memory state changes until the pair settles.

// W on the register driver paths: explicit ld.shared when the table was
// staged in shared memory (through LS the compiler only sees a generic
// pointer and would emit generic loads).  row(u) is a row handle (byte
// address or element offset), at(row, v) reads w[u][v].
template <bool kSh>
struct WTab {
    const double* g;
    uint32_t sh, rowlen;
    __device__ __forceinline__ uint32_t row(uint32_t u) const { return kSh ? sh + u * rowlen * 8u : u * rowlen; }
    __device__ __forceinline__ double at(uint32_t r, uint32_t v) const {
        if constexpr (kSh) {
            double x;
            asm("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(r + v * 8u));
            return x;
        } else {
            return g[r + v];
        }
    }
};

template <bool kSh>
__device__ __forceinline__ WTab<kSh> wtab(const LS& s) {
    return WTab<kSh>{s.W, s.w_sh, (uint32_t)s.n};
}

__device__ __forceinline__ uint32_t byte_of(uint64_t x, uint32_t i) {
    return __byte_perm((uint32_t)x, (uint32_t)(x >> 32), i) & 0xFFu;
}

__device__ __forceinline__ uint64_t bytes_below(uint32_t c) {  // c in 0..8
    return c >= 8 ? ~0ull : ((1ull << (8 * c)) - 1ull);
}

// group x (8 sorted ids) without its member at position p, then with v
// inserted in order (ids < 128)
__device__ __forceinline__ uint64_t replace_member(uint64_t x, uint32_t p, uint32_t v) {
    const uint64_t lowp = bytes_below(p);
    const uint64_t z = (x & lowp) | ((x >> 8) & ~lowp);  // 7 survivors, byte 7 = 0
    uint32_t c = 0;
    if (v) {  // survivors below v: bit 7 of (0x80 + v - 1 - z) per byte
        const uint64_t t = ((uint64_t)(0x80u + v - 1u) * 0x0101010101010101ull - z) & 0x0080808080808080ull;
        c = __popcll(t);
    }
    const uint64_t lowc = bytes_below(c);
    return (z & lowc) | ((z << 8) & ~bytes_below(c + 1)) | ((uint64_t)v << (8 * c));
}

// order-preserving image of a double (no NaN); -0.0 folds onto +0.0 so
// equal values tie like the reference's `<`
__device__ __forceinline__ uint64_t ord_bits(double v) {
    const uint64_t b = (uint64_t)__double_as_longlong(v + 0.0);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// _fast_edge of two packed groups at once; returns codes i*8+l (i < l)
template <bool kSh>
__device__ __forceinline__ void fast_edges8(const WTab<kSh>& W, uint64_t X, uint64_t Y, int lane, uint32_t pi,
                                            uint32_t pl, uint32_t& cx, uint32_t& cy) {
    uint64_t kx = ~0ull, ky = ~0ull;
    if (lane < 28) {
        kx = ord_bits(W.at(W.row(byte_of(X, pi)), byte_of(X, pl)));
        ky = ord_bits(W.at(W.row(byte_of(Y, pi)), byte_of(Y, pl)));
    }
    const uint32_t hx = (uint32_t)(kx >> 32), hy = (uint32_t)(ky >> 32);
    const uint32_t mhx = __reduce_min_sync(kFull, hx), mhy = __reduce_min_sync(kFull, hy);
    const uint32_t lx = hx == mhx ? (uint32_t)kx : 0xFFFFFFFFu, ly = hy == mhy ? (uint32_t)ky : 0xFFFFFFFFu;
    const uint32_t mlx = __reduce_min_sync(kFull, lx), mly = __reduce_min_sync(kFull, ly);
    const uint32_t code = pi * 8 + pl;
    cx = __reduce_min_sync(kFull, (hx == mhx && lx == mlx && lane < 28) ? code : 0xFFu);
    cy = __reduce_min_sync(kFull, (hy == mhy && ly == mly && lane < 28) ? code : 0xFFu);
}

// the `for _ in range(d_dp)` loop of _pass_ours for pair (j, j2); true if a
// swap was applied
template <bool kSh, bool kAtomic = false>
static __device__ bool sweep_pair8(LS& s, int j, int j2, int lane, uint32_t pi, uint32_t pl) {
    const WTab<kSh> W = wtab<kSh>(s);
    const int16_t* gj = s.G + j * s.cap;
    const int16_t* gj2 = s.G + j2 * s.cap;
    uint64_t X = 0, Y = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        X |= (uint64_t)(uint8_t)gj[i] << (8 * i);
        Y |= (uint64_t)(uint8_t)gj2[i] << (8 * i);
    }
    const int q = lane & 3;
    bool changed = false;
    for (int it = 0; it < 8; it++) {
        uint32_t cx, cy;
        fast_edges8<kSh>(W, X, Y, lane, pi, pl, cx, cy);
        const uint32_t d1 = byte_of(X, cx >> 3), d2 = byte_of(X, cx & 7);
        const uint32_t d1p = byte_of(Y, cy >> 3), d2p = byte_of(Y, cy & 7);
        // lane q: t_q = psum(w[u, other]) / 8 - w[u, partner]  (_gain_ours)
        const uint32_t u = q == 0 ? d1 : q == 1 ? d2 : q == 2 ? d1p : d2p;
        const uint32_t pu = q == 0 ? d2 : q == 1 ? d1 : q == 2 ? d2p : d1p;
        const uint64_t O = q < 2 ? Y : X;
        const uint32_t wr = W.row(u);
        double r[8];
#pragma unroll
        for (int e = 0; e < 8; e++) r[e] = W.at(wr, byte_of(O, e));
        const double sum = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        const double t = div_count(sum, 8) - W.at(wr, pu);
        const double t1a = __shfl_sync(kFull, t, 0), t1b = __shfl_sync(kFull, t, 1);
        const double t2a = __shfl_sync(kFull, t, 2), t2b = __shfl_sync(kFull, t, 3);
        // _best_candidate: (d1,d1p), (d1,d2p), (d2,d1p), (d2,d2p), first best
        // (gains are finite, so a two-level tree that keeps the left operand
        // on ties is the sequential "first strictly greater" scan)
        const double g0 = t1a + t2a, g1 = t1a + t2b, g2 = t1b + t2a, g3 = t1b + t2b;
        const bool s01 = g1 > g0, s23 = g3 > g2;
        const double b01 = s01 ? g1 : g0, b23 = s23 ? g3 : g2;
        const bool right = b23 > b01;
        const double best = right ? b23 : b01;
        const int bc = right ? (s23 ? 3 : 2) : (s01 ? 1 : 0);
        if (!(best > 0.0)) break;
        const uint32_t pa = (bc < 2) ? (cx >> 3) : (cx & 7);      // a = d1 or d2 in group j
        const uint32_t pb = (bc & 1) ? (cy & 7) : (cy >> 3);      // b = d1p or d2p in group j2
        const uint32_t a = byte_of(X, pa), b = byte_of(Y, pb);
        X = replace_member(X, pa, b);  // _swap (:252-257)
        Y = replace_member(Y, pb, a);
        changed = true;
    }
    if (changed) {
        __syncwarp();
        int16_t* wj = s.G + j * s.cap;
        int16_t* wj2 = s.G + j2 * s.cap;
        if (lane < 8) wj[lane] = (int16_t)byte_of(X, lane);
        else if (lane < 16) wj2[lane - 8] = (int16_t)byte_of(Y, lane - 8);
        if (lane == 0) {
            if (kAtomic) {  // sweep waves: other warps finish their pairs at the same time
                invalidate_atomic(s, j);
                invalidate_atomic(s, j2);
            } else {
                invalidate(s, j);
                invalidate(s, j2);
            }
        }
        __syncwarp();
    }
    return changed;
}

// even phase of _pass_ours: swap sweep over rng.permutation(C(k,2)) pairs
static __device__ __noinline__ bool pass_sweep(LS& s, Pcg64& rng, int lane) {
    const int k = s.k, np = k * (k - 1) / 2, d_dp = s.sz[0];
    if (lane == 0) {
        for (int i = 0; i < np; i++) s.perm[i] = (int16_t)i;
        for (int i = np - 1; i >= 1; i--) {
            int jx = (int)rng.interval((uint64_t)i);
            int16_t t = s.perm[i];
            s.perm[i] = s.perm[jx];
            s.perm[jx] = t;
        }
    }
    __syncwarp();
    bool changed = false;
    // this lane's intra pair (i, l), lexicographic, for the d_dp = 8 path
    uint32_t pi = 0, pl = 1;
    if (lane < 28) {
        int i = 0, t = lane;
        while (t >= 7 - i) {
            t -= 7 - i;
            i++;
        }
        pi = (uint32_t)i;
        pl = (uint32_t)(i + 1 + t);
    }
    const bool fast8 = d_dp == 8 && s.n <= 128;
    for (int q = 0; q < np; q++) {
        int j, j2;
        decode_pair(s.perm[q], k, j, j2);
        if (fast8 && s.sz[j] == 8 && s.sz[j2] == 8) {
            if (s.w_sh ? sweep_pair8<true>(s, j, j2, lane, pi, pl) : sweep_pair8<false>(s, j, j2, lane, pi, pl))
                changed = true;
            continue;
        }
        for (int it = 0; it < d_dp; it++) {
            int a, b;
            long long b0 = clock64();
            double gain = best_candidate(s, j, j2, lane, a, b);
            if (g_prof && lane == 0) {
                g_prof[8] += 1;
                g_prof[12] += clock64() - b0;
                g_prof[11] += gain > 0.0;
            }
            if (gain <= 0.0) break;
            g_swap_w(s, a, j, b, j2, lane);  // _swap (:252-257)
            const unsigned bpv = (unsigned)s.valid[3];
            __syncwarp();
            if (lane == 0) {
                invalidate(s, j);
                invalidate(s, j2);
            }
            __syncwarp();
            if (bpv >> j & 1u) best_partners_swap(s, j, a, b, lane);
            if (bpv >> j2 & 1u) best_partners_swap(s, j2, b, a, lane);
            changed = true;
        }
    }
    return changed;
}

// Even phase of _pass_ours on every warp of the CTA (one island per CTA).
// _best_candidate / _swap for pair (j, j2) read and write only groups j and
// j2, so pairs that share no group commute: the permutation is cut into
// waves (a pair's wave = 1 + the latest wave of an earlier pair sharing one
// of its groups; pairs of one wave are disjoint) and each wave's pairs run
// on different warps, with the reference's per-pair results.  Requires every
// group at d_dp = 8 members and n <= 128 (register sweep path); called by all
// threads, returns the same value in all of them.  Scratch: s.perm (pair
// order by wave), s.i32 (wave starts, C(k,2) + 1 <= 3k + 8 entries), flag.
template <bool kSh>
static __device__ bool pass_sweep_waves(LS& s, Pcg64& rng, int wid, int lane, int W, int* flag) {
    const int k = s.k, np = k * (k - 1) / 2;
    int16_t* order = s.perm + np;  // s.perm holds k*k + cap entries
    int* wstart = s.i32;
    if (wid == 0 && lane == 0) {
        int ok = 1;
        for (int j = 0; j < k; j++) ok &= s.sz[j] == 8;
        flag[1] = ok;
    }
    __syncthreads();
    if (!flag[1]) {  // unbalanced groups: the sequential sweep on the driver warp
        if (wid == 0) {
            const bool ch = pass_sweep(s, rng, lane);
            if (lane == 0) flag[0] = ch;
        }
        __syncthreads();
        return flag[0] != 0;
    }
    if (wid == 0 && lane == 0) {
        int16_t* perm = s.perm;
        for (int i = 0; i < np; i++) perm[i] = (int16_t)i;
        for (int i = np - 1; i >= 1; i--) {
            int jx = (int)rng.interval((uint64_t)i);
            int16_t t = perm[i];
            perm[i] = perm[jx];
            perm[jx] = t;
        }
        int ready[16], wave[120], cnt[121];
        for (int j = 0; j < k; j++) ready[j] = 0;
        int nw = 0;
        for (int q = 0; q < np; q++) {
            int j, j2;
            decode_pair(perm[q], k, j, j2);
            const int w = max(ready[j], ready[j2]);
            wave[q] = w;
            ready[j] = ready[j2] = w + 1;
            nw = max(nw, w + 1);
        }
        for (int w = 0; w <= nw; w++) cnt[w] = 0;
        for (int q = 0; q < np; q++) cnt[wave[q] + 1]++;
        for (int w = 0; w < nw; w++) cnt[w + 1] += cnt[w];
        for (int w = 0; w <= nw; w++) wstart[w] = cnt[w];
        for (int q = 0; q < np; q++) order[cnt[wave[q]]++] = perm[q];  // stable: permutation order inside a wave
        wstart[np + 1] = nw;
        *flag = 0;
    }
    __syncthreads();
    uint32_t pi = 0, pl = 1;
    if (lane < 28) {
        int i = 0, t = lane;
        while (t >= 7 - i) {
            t -= 7 - i;
            i++;
        }
        pi = (uint32_t)i;
        pl = (uint32_t)(i + 1 + t);
    }
    const int nw = wstart[np + 1];
    for (int w = 0; w < nw; w++) {
        for (int x = wstart[w] + wid; x < wstart[w + 1]; x += W) {
            int j, j2;
            decode_pair(order[x], k, j, j2);
            HS_JITTER();
            if (sweep_pair8<kSh, true>(s, j, j2, lane, pi, pl) && lane == 0) atomicOr(flag, 1);
        }
        HS_JITTER();
        __syncthreads();
    }
    return *flag != 0;
}

// _home_costs (:287-291) for every group whose members changed
__device__ inline void ensure_caches(LS& s, int lane) {
    const int k = s.k, n = s.n;
    const unsigned all = k >= 32 ? 0xffffffffu : (1u << k) - 1u;
    const unsigned hv = (unsigned)s.valid[1];
    if (hv == all) return;
    for (int i = 0; i < k; i++) {
        if (hv >> i & 1u) continue;
        const int16_t* g = s.G + i * s.cap;
        const int c = s.sz[i];
        for (int a = lane; a < c; a += kWarp) {
            const double* wr = s.W + (size_t)g[a] * n;
            double h = kInf;
            if (s.lat) {  // one driver warp per SM: eight loads in flight (min is order-free)
                for (int b0 = 0; b0 < c; b0 += 8) {
                    double x[8];
#pragma unroll
                    for (int t = 0; t < 8; t++) x[t] = (b0 + t < c && b0 + t != a) ? wr[g[b0 + t]] : kInf;
#pragma unroll
                    for (int t = 0; t < 8; t++) h = dmin(h, x[t]);
                }
            } else {  // many warps per SM hide the latency; fewer instructions win
                for (int b = 0; b < c; b++)
                    if (b != a) h = dmin(h, wr[g[b]]);
            }
            s.home[g[a]] = h;
        }
    }
    __syncwarp();
    if (lane == 0) s.valid[1] = (int)all;
    __syncwarp();
}

// fastest_free (:318-328): min by (home, id) over unlocked members; -1 if none
__device__ __forceinline__ int fastest_free(const LS& s, int i, double& home) {
    const int16_t* g = s.G + i * s.cap;
    int c = s.sz[i];
    if (c < 2) return -1;
    int best = -1;
    double bh = 0.0;
    for (int a = 0; a < c; a++) {
        int d = g[a];
        if (s.locked[d >> 5] >> (d & 31) & 1) continue;
        double h = s.home[d];
        if (best < 0 || h < bh) {
            best = d;
            bh = h;
        }
    }
    home = bh;
    return best;
}

// fastest_free over the warp: lanes over members, min by (home, id)
__device__ __forceinline__ int fastest_free_w(const LS& s, int i, int lane, double& home) {
    const int16_t* g = s.G + i * s.cap;
    const int c = s.sz[i];
    if (c < 2) return -1;
    double bh = kInf;
    int bd = INT_MAX;
    for (int a = lane; a < c; a += kWarp) {
        int d = g[a];
        if (s.locked[d >> 5] >> (d & 31) & 1) continue;
        double h = s.home[d];
        if (h < bh || (h == bh && d < bd)) {
            bh = h;
            bd = d;
        }
    }
    warp_argmin(bh, bd);
    home = bh;
    return bd == INT_MAX ? -1 : bd;
}

// _chain_round (:299-391).  All lanes run the control flow uniformly; the
// member scans, target argmax and group moves are lane-parallel.
static __device__ __noinline__ bool chain_round(LS& s, int lane) {
    const int k = s.k;
    long long c0 = clock64();
    ensure_caches(s, lane);
    if (g_prof && lane == 0) {
        g_prof[4] += clock64() - c0;
        g_prof[5] += 1;
    }
    // start group: largest relocation gain, first on ties
    double gain = -kInf;
    int idx = INT_MAX;
    if (lane < k) {
        double home;
        int v = fastest_free(s, lane, home);
        if (v >= 0) {
            double mx = -kInf;
            bool first = true;
            for (int j = 0; j < k; j++) {
                if (j == lane) continue;
                double x = mean_at(s, v, j);
                if (first || x > mx) mx = x;
                first = false;
            }
            gain = mx - home;
            idx = lane;
        }
    }
    warp_argmax(gain, idx);
    if (idx == INT_MAX) return false;
    const int start = idx;
    int* mv_v = s.i32;
    int* mv_src = s.i32 + k;
    int* mv_dst = s.i32 + 2 * k;
    double* steps = s.f64;
    double* closers = s.f64 + k + 1;
    int cur = start, nm = 0;
    bool natural = false;
    for (int it = 0; it < k; it++) {
        double home;
        const int v = fastest_free_w(s, cur, lane, home);
        if (v < 0) break;
        double sc = -kInf;
        int dst = INT_MAX;
        if (lane < k && lane != cur) {
            sc = mean_at(s, v, lane);
            dst = lane;
        }
        warp_argmax(sc, dst);  // first maximum over targets
        __syncwarp();
        if (lane == 0) {
            closers[nm] = cur != start ? mean_at(s, v, start) - home : -kInf;
            steps[nm] = sc - home;
            mv_v[nm] = v;
            mv_src[nm] = cur;
            mv_dst[nm] = dst;
            s.locked[v >> 5] |= 1u << (v & 31);
            s.nlocked[0]++;
            invalidate(s, cur);
            invalidate(s, dst);
        }
        g_move_w(s, v, cur, dst, lane);
        nm++;
        // refresh the touched mean columns and home costs (scheduler.py:362-363)
        long long c1 = clock64();
        ensure_caches(s, lane);
        if (g_prof && lane == 0) {
            g_prof[6] += clock64() - c1;
            g_prof[7] += 1;
        }
        cur = dst;
        if (cur == start) {
            natural = true;
            break;
        }
    }
    if (nm == 0) return false;
    double prefix = 0.0, best_v = -kInf;
    int best_l = -1;
    // prefix[l] = cumsum of steps[0..l-1] (np.cumsum, sequential)
    for (int l = 0; l < nm; l++) {
        double value = prefix + closers[l];
        if (value > best_v) {
            best_v = value;
            best_l = l;
        }
        prefix = prefix + steps[l];
    }
    if (natural && prefix > best_v) {
        best_v = prefix;
        best_l = nm;
    }
    const bool applied = best_v > 0.0;
    const int keep = applied ? best_l : 0;
    for (int t = nm - 1; t >= keep; t--) g_move_w(s, mv_v[t], mv_dst[t], mv_src[t], lane);
    if (applied && best_l < nm) g_move_w(s, mv_v[best_l], mv_src[best_l], start, lane);
    if (lane == 0) {
        for (int t = 0; t < nm; t++) {
            invalidate(s, mv_src[t]);
            invalidate(s, mv_dst[t]);
        }
        invalidate(s, start);
    }
    __syncwarp();
    return applied;
}

// ---------------------------------------------------------------------------
// Odd phase of _pass_ours for n <= 64, k <= 8, register resident.
//
// Groups are 64-bit membership masks (ascending member order is the bit
// order), lane j holding group j's; lane l owns devices l and l + 32 (their
// group and home cost).  The locked set is one uniform mask.  Every mean the
// chain reads is recomputed from the current masks (a sequential sum over
// the members, as w[:, grp].mean(axis=1) reduces it), so no mean cache is
// kept; home costs are refreshed for the groups a move touched.  Minima and
// maxima with first-index ties are three REDUX stages on the order-preserving
// image of the double (high word, low word, index).

__device__ __forceinline__ double from_ord(uint64_t k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}

// min value over valid lanes, smallest idx among equal minima (INT_MAX if none)
__device__ __forceinline__ int redux_argmin(double v, bool valid, int idx, double& best) {
    const uint64_t k = valid ? ord_bits(v) : ~0ull;
    const uint32_t hi = (uint32_t)(k >> 32), lo = (uint32_t)k;
    const uint32_t mh = __reduce_min_sync(kFull, hi);
    const uint32_t ml = __reduce_min_sync(kFull, hi == mh ? lo : 0xFFFFFFFFu);
    const int wi = (int)__reduce_min_sync(kFull, (valid && hi == mh && lo == ml) ? (unsigned)idx : 0x7FFFFFFFu);
    best = from_ord(((uint64_t)mh << 32) | ml);
    return wi;
}

// max value over valid lanes, smallest idx among equal maxima (INT_MAX if none)
__device__ __forceinline__ int redux_argmax(double v, bool valid, int idx, double& best) {
    const uint64_t k = valid ? ord_bits(v) : 0ull;
    const uint32_t hi = (uint32_t)(k >> 32), lo = (uint32_t)k;
    const uint32_t mh = __reduce_max_sync(kFull, hi);
    const uint32_t ml = __reduce_max_sync(kFull, hi == mh ? lo : 0u);
    const int wi = (int)__reduce_min_sync(kFull, (valid && hi == mh && lo == ml) ? (unsigned)idx : 0x7FFFFFFFu);
    best = from_ord(((uint64_t)mh << 32) | ml);
    return wi;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t x, int src) {
    const uint32_t lo = __shfl_sync(kFull, (uint32_t)x, src), hi = __shfl_sync(kFull, (uint32_t)(x >> 32), src);
    return ((uint64_t)hi << 32) | lo;
}

// A group's members as 16 packed bytes (ascending, 0xFF past the end), held
// by the group's lane as two 64-bit halves: iteration is byte extraction, a
// move is a byte shift at the member's rank.
struct Members {
    uint64_t lo, hi;
};

__device__ __forceinline__ uint32_t mbyte(const Members& L, int t) {  // t static after unrolling
    return (uint32_t)((t < 8 ? L.lo >> (8 * t) : L.hi >> (8 * (t - 8))) & 0xFFu);
}

__device__ __forceinline__ Members shfl_members(const Members& L, int src) {
    return Members{shfl64(L.lo, src), shfl64(L.hi, src)};
}

__device__ __forceinline__ void byte_masks(int p, uint64_t& ml, uint64_t& mh) {  // bytes [0, p), p <= 16
    ml = p >= 8 ? ~0ull : ((1ull << (8 * p)) - 1ull);
    mh = p <= 8 ? 0ull : (p >= 16 ? ~0ull : ((1ull << (8 * (p - 8))) - 1ull));
}

__device__ __forceinline__ void members_remove(Members& L, int p) {
    uint64_t ml, mh;
    byte_masks(p, ml, mh);
    const uint64_t lo_s = (L.lo >> 8) | (L.hi << 56), hi_s = (L.hi >> 8) | (0xFFull << 56);
    L.lo = (L.lo & ml) | (lo_s & ~ml);
    L.hi = (L.hi & mh) | (hi_s & ~mh);
}

__device__ __forceinline__ void members_insert(Members& L, int c, uint32_t v) {
    uint64_t ml, mh, ml1, mh1;
    byte_masks(c, ml, mh);
    byte_masks(c + 1, ml1, mh1);
    const uint64_t lo_s = L.lo << 8, hi_s = (L.hi << 8) | (L.lo >> 56);
    L.lo = (L.lo & ml) | (lo_s & ~ml1) | (c < 8 ? (uint64_t)v << (8 * c) : 0ull);
    L.hi = (L.hi & mh) | (hi_s & ~mh1) | (c >= 8 ? (uint64_t)v << (8 * (c - 8)) : 0ull);
}

// w[u, grp].mean() over cnt packed members: sequential sum (as numpy reduces
// the F-contiguous gather), then / count; all loads issued up front
template <int MAXC, bool kSh>
__device__ __forceinline__ double members_mean(const WTab<kSh>& W, uint32_t wr, const Members& L, int cnt) {
    double w[MAXC];
#pragma unroll
    for (int t = 0; t < MAXC; t++) w[t] = t < cnt ? W.at(wr, mbyte(L, t)) : 0.0;
    double r = 0.0;
#pragma unroll
    for (int t = 0; t < MAXC; t++)
        if (t < cnt) r += w[t];
    return div_count(r, cnt);
}

// min of wr over the members other than `self` (order-free), +inf if none
template <int MAXC, bool kSh>
__device__ __forceinline__ double members_min(const WTab<kSh>& W, uint32_t wr, const Members& L, int cnt,
                                              uint32_t self) {
    double h = kInf;
#pragma unroll
    for (int t = 0; t < MAXC; t++) {
        const uint32_t x = mbyte(L, t);
        if (t < cnt && x != self) h = dmin(h, W.at(wr, x));
    }
    return h;
}

struct ChainRegs {
    uint64_t GM;        // lane j < k: members of group j (mask)
    Members L;          // lane j < k: the same members, packed ascending
    uint64_t locked;    // uniform
    int g0, g1;         // groups of this lane's devices (lane, lane + 32); -1 if absent
    double h0, h1;      // their home costs (kept for unlocked devices)
    bool st0, st1;      // home cost must be recomputed
};

// _move (:294-296): v leaves src for dst (bisect.insort keeps the order).
// Home costs follow exactly (min is order-free): a member of dst takes
// min(home, w[d, v]); a member of src keeps its home unless v was at it.
template <bool kSh>
__device__ __forceinline__ void cmove(const WTab<kSh>& W, ChainRegs& c, int v, int src, int dst, int lane) {
    const uint64_t bit = 1ull << v;
    if (lane == src) {
        members_remove(c.L, __popcll(c.GM & (bit - 1ull)));
        c.GM &= ~bit;
    }
    if (lane == dst) {
        members_insert(c.L, __popcll(c.GM & (bit - 1ull)), (uint32_t)v);
        c.GM |= bit;
    }
    const int d0 = lane, d1 = lane + 32;
    if (d0 == v) {
        c.g0 = dst;
        c.st0 = true;
    } else if ((c.g0 == src || c.g0 == dst) && !(c.locked >> d0 & 1ull) && !c.st0) {
        const double w = W.at(W.row((uint32_t)d0), (uint32_t)v);
        if (c.g0 == dst)
            c.h0 = dmin(c.h0, w);
        else if (!(w > c.h0))
            c.st0 = true;
    }
    if (d1 == v) {
        c.g1 = dst;
        c.st1 = true;
    } else if ((c.g1 == src || c.g1 == dst) && !(c.locked >> d1 & 1ull) && !c.st1) {
        const double w = W.at(W.row((uint32_t)d1), (uint32_t)v);
        if (c.g1 == dst)
            c.h1 = dmin(c.h1, w);
        else if (!(w > c.h1))
            c.st1 = true;
    }
}

// _home_costs (:287-291) for this lane's unlocked devices with a stale home
template <int MAXC, bool kSh>
__device__ __forceinline__ void refresh_homes(const WTab<kSh>& W, ChainRegs& c, int lane) {
    const bool r0 = c.st0 && c.g0 >= 0 && !(c.locked >> lane & 1ull);
    const bool r1 = c.st1 && c.g1 >= 0 && !(c.locked >> (lane + 32) & 1ull);
    if (!__any_sync(kFull, r0 || r1)) return;
    const int s0 = c.g0 < 0 ? 0 : c.g0, s1 = c.g1 < 0 ? 0 : c.g1;
    const Members m0 = shfl_members(c.L, s0), m1 = shfl_members(c.L, s1);
    const int n0 = __popcll(shfl64(c.GM, s0)), n1 = __popcll(shfl64(c.GM, s1));
    if (r0) {
        c.h0 = members_min<MAXC, kSh>(W, W.row((uint32_t)lane), m0, n0, (uint32_t)lane);
        c.st0 = false;
    }
    if (r1) {
        c.h1 = members_min<MAXC, kSh>(W, W.row((uint32_t)(lane + 32)), m1, n1, (uint32_t)(lane + 32));
        c.st1 = false;
    }
}

// this lane's best unlocked device of group i by (home, id); false if none
__device__ __forceinline__ bool lane_free(const ChainRegs& c, int i, int lane, double& h, int& d) {
    const bool ok0 = c.g0 == i && !(c.locked >> lane & 1ull);
    const bool ok1 = c.g1 == i && !(c.locked >> (lane + 32) & 1ull);
    h = (ok0 && !(ok1 && c.h1 < c.h0)) ? c.h0 : c.h1;
    d = (ok0 && !(ok1 && c.h1 < c.h0)) ? lane : lane + 32;
    return ok0 || ok1;
}

// fastest_free (:318-328) of group i: -1 if none
__device__ __forceinline__ int chain_fastest_free(const ChainRegs& c, int i, int lane, double& home) {
    const int cnt = __popcll(shfl64(c.GM, i));
    double h;
    int d;
    const bool ok = lane_free(c, i, lane, h, d);
    const int v = redux_argmin(h, ok, d, home);
    return (cnt < 2 || v == 0x7FFFFFFF) ? -1 : v;
}

// Start-selection state carried from one chain round to the next.  A round
// whose only effect is locking the start group's device (no move survives)
// leaves every other group's fastest free device, its means and the home
// costs unchanged, so the next round recomputes only that group's row.
struct RoundCache {
    int row;  // -1: recompute every row; else only this group's row
    int myv;
    double myh, mrow[2];
};

template <int MAXC, bool kSh>
static __device__ bool chain_round8(LS& s, ChainRegs& c, RoundCache& rc, int lane) {
    const int k = s.k;
    const WTab<kSh> W = wtab<kSh>(s);
    const int row = rc.row;
    rc.row = -1;
    refresh_homes<MAXC, kSh>(W, c, lane);
    // fastest_free (:318-328) of every group: lane i scans group i's packed
    // members (ascending, so a strict '<' keeps the smallest id on ties)
    // against the home costs published in shared memory
    double* hs = s.home;  // n doubles, otherwise unused on this path
    if (row < 0) {
        if (lane < s.n) hs[lane] = c.h0;
        if (lane + 32 < s.n) hs[lane + 32] = c.h1;
        __syncwarp();
    }
    int myv = rc.myv;
    double myh = rc.myh;
    if (lane < k && (row < 0 || lane == row)) {
        myv = -1;
        myh = 0.0;
        const int cnt = __popcll(c.GM);
        if (cnt >= 2) {
#pragma unroll
            for (int t = 0; t < MAXC; t++) {
                const uint32_t d = mbyte(c.L, t);
                if (t < cnt && !(c.locked >> d & 1ull)) {
                    const double h = hs[d];
                    if (myv < 0 || h < myh) {
                        myv = (int)d;
                        myh = h;
                    }
                }
            }
        }
    }
    // gain_i = max_{j != i} mean[v_i, j] - home_i for (i, j) = (e >> 3, e & 7),
    // e = lane + 32 sl: row maxima inside 8-lane segments
    const Members Lj = shfl_members(c.L, lane & 7);
    const int cj = __popcll(shfl64(c.GM, lane & 7));
    double gsl[2], mrow[2];
    int isl[2];
#pragma unroll
    for (int sl = 0; sl < 2; sl++) {
        const int i = (lane >> 3) + 4 * sl, j = lane & 7;
        const int vi = __shfl_sync(kFull, myv, i);
        const double hi = __shfl_sync(kFull, myh, i);
        double x = rc.mrow[sl];
        if (row < 0 || i == row) {
            x = -kInf;
            if (j < k && j != i && vi >= 0) x = members_mean<MAXC, kSh>(W, W.row((uint32_t)vi), Lj, cj);
        }
        mrow[sl] = x;  // mean[v_i, j], reused by the chain's first step when i = start
        x = dmax(x, __shfl_xor_sync(kFull, x, 1));
        x = dmax(x, __shfl_xor_sync(kFull, x, 2));
        x = dmax(x, __shfl_xor_sync(kFull, x, 4));
        gsl[sl] = x - hi;
        isl[sl] = (vi >= 0 && j == 0) ? i : -1;
    }
    // first strict maximum over i from best_start = -inf
    const bool u0 = isl[0] >= 0 && gsl[0] > -kInf, u1 = isl[1] >= 0 && gsl[1] > -kInf;
    const bool take1 = u1 && (!u0 || gsl[1] > gsl[0]);
    double best;
    const int start0 = redux_argmax(take1 ? gsl[1] : gsl[0], u0 || u1, take1 ? isl[1] : isl[0], best);
    if (start0 == 0x7FFFFFFF) return false;
    const int start = start0;
    int* mv_v = s.i32;
    int* mv_src = s.i32 + k;
    int* mv_dst = s.i32 + 2 * k;
    double* steps = s.f64;
    double* closers = s.f64 + k + 1;
    const ChainRegs snap = c;  // pre-chain state: restoring it undoes every move at once
    int cur = start, nm = 0;
    bool natural = false;
    for (int it = 0; it < k; it++) {
        double home, mj = 0.0;
        int v;
        if (it == 0) {
            // nothing moved since the start selection: its fastest free device
            // of the start group and that device's means are the step's own
            v = __shfl_sync(kFull, myv, start);
            home = __shfl_sync(kFull, myh, start);
            mj = __shfl_sync(kFull, start < 4 ? mrow[0] : mrow[1], 8 * (start & 3) + (lane & 7));
        } else {
            const uint64_t gm = shfl64(c.GM, cur);
            if (__popcll(gm) < 2 || !(gm & ~c.locked)) break;  // fastest_free(cur) is None
            refresh_homes<MAXC, kSh>(W, c, lane);
            v = chain_fastest_free(c, cur, lane, home);
            if (v < 0) break;
            // scores = mean[v, targets]; dst = first maximum
            if (lane < k) mj = members_mean<MAXC, kSh>(W, W.row((uint32_t)v), c.L, __popcll(c.GM));
        }
        double sc;
        const int dst = redux_argmax(mj, lane < k && lane != cur, lane, sc);
        if (it == 0 && !(shfl64(c.GM, dst) & ~c.locked)) {
            // dst has no free device even before v arrives (v will be locked), so
            // the chain ends after this move, and a single move is always rejected
            // (see below): the round's only effect is locking v
            c.locked |= 1ull << v;
            rc = RoundCache{start, myv, myh, {mrow[0], mrow[1]}};
            return false;
        }
        const double mstart = __shfl_sync(kFull, mj, start);
        if (lane == 0) {
            closers[nm] = cur != start ? mstart - home : -kInf;
            steps[nm] = sc - home;
            mv_v[nm] = v;
            mv_src[nm] = cur;
            mv_dst[nm] = dst;
        }
        c.locked |= 1ull << v;
        cmove<kSh>(W, c, v, cur, dst, lane);
        nm++;
        cur = dst;
        if (cur == start) {
            natural = true;
            break;
        }
    }
    __syncwarp();
    if (nm == 1) {  // closers[0] is -inf and a single move cannot close the cycle: rejected
        const uint64_t locked = c.locked;
        c = snap;
        c.locked = locked;
        rc = RoundCache{start, myv, myh, {mrow[0], mrow[1]}};  // as a lock-only round
        return false;
    }
    double prefix = 0.0, best_v = -kInf;
    int best_l = -1;
    for (int l = 0; l < nm; l++) {  // prefix[l] = cumsum of steps[0..l-1]
        const double value = prefix + closers[l];
        if (value > best_v) {
            best_v = value;
            best_l = l;
        }
        prefix = prefix + steps[l];
    }
    if (natural && prefix > best_v) {
        best_v = prefix;
        best_l = nm;
    }
    const bool applied = best_v > 0.0;
    // Outcome: moves[0 .. best_l) kept and moves[best_l]'s device sent back to
    // start (if best_l < nm), or nothing kept.  Reach it from whichever end
    // needs fewer moves: undo the tail, or restore the snapshot and replay the
    // kept prefix (home costs are exact minima either way; locks stay).
    const int keep = applied ? best_l : 0;
    if (keep < nm - keep) {
        const uint64_t locked = c.locked;
        c = snap;
        c.locked = locked;
        for (int t = 0; t < keep; t++) cmove<kSh>(W, c, mv_v[t], mv_src[t], mv_dst[t], lane);
    } else {
        for (int t = nm - 1; t >= keep; t--) cmove<kSh>(W, c, mv_v[t], mv_dst[t], mv_src[t], lane);
    }
    if (applied && best_l < nm) cmove<kSh>(W, c, mv_v[best_l], mv_src[best_l], start, lane);
    __syncwarp();
    return applied;
}

template <int MAXC, bool kSh>
static __device__ bool pass_chains8(LS& s, int lane) {
    const int k = s.k, n = s.n;
    ChainRegs c;
    c.GM = 0;
    c.L = Members{~0ull, ~0ull};
    if (lane < k) {
        const int16_t* g = s.G + lane * s.cap;
        for (int t = 0; t < s.sz[lane]; t++) {
            c.GM |= 1ull << g[t];
            if (t < 8)
                c.L.lo = (c.L.lo & ~(0xFFull << (8 * t))) | ((uint64_t)g[t] << (8 * t));
            else
                c.L.hi = (c.L.hi & ~(0xFFull << (8 * (t - 8)))) | ((uint64_t)g[t] << (8 * (t - 8)));
        }
    }
    c.g0 = c.g1 = -1;
    for (int j = 0; j < k; j++) {
        const uint64_t m = shfl64(c.GM, j);
        if (m >> lane & 1ull) c.g0 = j;
        if (lane + 32 < n && (m >> (lane + 32) & 1ull)) c.g1 = j;
    }
    c.h0 = c.h1 = kInf;
    c.st0 = c.st1 = true;
    c.locked = 0;
    RoundCache rc{-1, -1, 0.0, {0.0, 0.0}};
    const uint64_t all = n >= 64 ? ~0ull : ((1ull << n) - 1ull);
    bool changed = false;
    while (c.locked != all) {
        const uint64_t before = c.locked;
        if (chain_round8<MAXC, kSh>(s, c, rc, lane)) changed = true;
        if (c.locked == before) break;
    }
    // back to sorted member lists; every cache of the touched groups is stale
    __syncwarp();
    if (lane < k) {
        const int cnt = __popcll(c.GM);
        int16_t* g = s.G + lane * s.cap;
#pragma unroll
        for (int t = 0; t < MAXC; t++)
            if (t < cnt) g[t] = (int16_t)mbyte(c.L, t);
        s.sz[lane] = cnt;
        s.cver[lane]++;
    }
    if (lane == 0) {
        s.valid[1] = 0;
        s.valid[2] = 0;
        s.valid[3] = 0;
    }
    __syncwarp();
    return changed;
}

// odd phase of _pass_ours: chains until every device is locked
static __device__ __noinline__ bool pass_chains(LS& s, int lane) {
    if (s.n <= 64 && s.k <= 8 && s.m <= 8) return s.w_sh ? pass_chains8<9, true>(s, lane) : pass_chains8<9, false>(s, lane);
    if (s.n <= 64 && s.k <= 8 && s.m <= 15)
        return s.w_sh ? pass_chains8<16, true>(s, lane) : pass_chains8<16, false>(s, lane);
    const int n = s.n;
    for (int i = lane; i < ((n + 31) >> 5); i += kWarp) s.locked[i] = 0;
    if (lane == 0) s.nlocked[0] = 0;
    __syncwarp();
    bool changed = false;
    while (s.nlocked[0] < n) {
        int before = s.nlocked[0];
        if (chain_round(s, lane)) changed = true;
        __syncwarp();
        if (s.nlocked[0] == before) break;
    }
    return changed;
}

// _pass_kl (:431-449)
static __device__ __noinline__ bool pass_kl(LS& s, int lane) {
    const int k = s.k, n = s.n;
    bool changed = false;
    double* s11 = s.f64;
    double* s12 = s11 + s.cap;
    double* s22 = s12 + s.cap;
    double* s21 = s22 + s.cap;
    for (int j = 0; j < k; j++) {
        for (int j2 = j + 1; j2 < k; j2++) {
            const int16_t* a1 = s.G + j * s.cap;
            const int16_t* a2 = s.G + j2 * s.cap;
            const int c1 = s.sz[j], c2 = s.sz[j2];
            for (int t = lane; t < 2 * (c1 + c2); t += kWarp) {
                if (t < c1)
                    s11[t] = row_pw(s, a1[t], a1, c1);
                else if (t < 2 * c1)
                    s12[t - c1] = row_pw(s, a1[t - c1], a2, c2);
                else if (t < 2 * c1 + c2)
                    s22[t - 2 * c1] = row_pw(s, a2[t - 2 * c1], a2, c2);
                else
                    s21[t - 2 * c1 - c2] = row_pw(s, a2[t - 2 * c1 - c2], a1, c1);
            }
            __syncwarp();
            double bg = -kInf;
            int bt = INT_MAX;
            for (int t = lane; t < c1 * c2; t += kWarp) {
                int i = t / c2, l = t - (t / c2) * c2;
                double gn = ((s12[i] - s11[i]) + (s21[l] - s22[l])) - 2.0 * s.W[(size_t)a1[i] * n + a2[l]];
                if (bt == INT_MAX || gn > bg) {
                    bg = gn;
                    bt = t;
                }
            }
            warp_argmax(bg, bt);
            if (bg > 0.0) {
                const int a = a1[bt / c2], b = a2[bt % c2];
                __syncwarp();
                g_swap_w(s, a, j, b, j2, lane);  // _swap (:252-257)
                if (lane == 0) {
                    invalidate(s, j);
                    invalidate(s, j2);
                }
                changed = true;
            }
            __syncwarp();
        }
    }
    return changed;
}

__device__ __forceinline__ void load_groups(LS& s, const int16_t* p, int lane) {
    for (int t = lane; t < s.k * s.m; t += kWarp) s.G[(t / s.m) * s.cap + t % s.m] = p[t];
    if (lane < s.k) s.sz[lane] = s.m;
    if (lane < s.k) s.cver[lane]++;
    if (lane == 0) {
        s.valid[0] = 0;
        s.valid[1] = 0;
        s.valid[2] = 0;
        s.valid[3] = 0;
    }
    __syncwarp();
}

__device__ __forceinline__ void store_groups(const LS& s, int16_t* p, int lane) {
    for (int t = lane; t < s.k * s.m; t += kWarp) p[t] = s.G[(t / s.m) * s.cap + t % s.m];
    __syncwarp();
}

// crossover (:139-174), lane 0 after a lane-parallel group-of map
static __device__ __noinline__ void crossover(LS& s, const int16_t* p1, const int16_t* p2, Pcg64& rng, int16_t* out, int lane) {
    const int k = s.k, m = s.m;
    for (int t = lane; t < k * m; t += kWarp) s.grp_of[p1[t]] = (int8_t)(t / m);
    __syncwarp();
    if (lane == 0) {
        int* slots = s.i32;       // k
        int* cnt = s.i32 + k;     // k
        int16_t* diff = s.perm;   // m (reused)
        int ns = 0;
        for (int j = 0; j < k; j++) {
            int c = 0;
            for (int i = 0; i < m; i++)
                if (s.grp_of[p2[j * m + i]] != j) c++;
            cnt[j] = c;
            if (c) slots[ns++] = j;
        }
        if (ns == 0) {
            for (int t = 0; t < k * m; t++) out[t] = p1[t];
        } else {
            int j = slots[rng.integers(0, ns)];
            int nd = 0;
            for (int i = 0; i < m; i++) {
                int d = p2[j * m + i];
                if (s.grp_of[d] != j) diff[nd++] = (int16_t)d;
            }
            int mi = (int)rng.integers(1, nd + 1);
            // choice(nd, mi, replace=False): Floyd, then the shuffle's draws
            int picked[64];
            int np = 0;
            for (int jj = nd - mi; jj < nd; jj++) {
                int v = (int)rng.bounded((uint64_t)jj);
                bool dup = false;
                for (int t = 0; t < np; t++) dup |= picked[t] == v;
                picked[np++] = dup ? jj : v;
            }
            for (int i = mi - 1; i >= 1; i--) (void)rng.bounded((uint64_t)i);
            for (int a = 1; a < np; a++) {  // sorted(picked)
                int x = picked[a], b = a - 1;
                while (b >= 0 && picked[b] > x) {
                    picked[b + 1] = picked[b];
                    b--;
                }
                picked[b + 1] = x;
            }
            for (int t = 0; t < k * m; t++) s.G[(t / m) * s.cap + t % m] = p1[t];
            for (int t = 0; t < k; t++) s.sz[t] = m;
            int16_t pool[64];
            int npool = m;
            for (int i = 0; i < m; i++) pool[i] = p1[j * m + i];
            for (int t = 0; t < mi; t++) {
                int d = diff[picked[t]];
                int src = s.grp_of[d];
                g_remove(s, src, d);
                g_insort(s, j, d);
                s.grp_of[d] = (int8_t)j;
                int vi = (int)rng.integers(0, npool);
                int victim = pool[vi];
                for (int q = vi; q + 1 < npool; q++) pool[q] = pool[q + 1];
                npool--;
                g_remove(s, j, victim);
                g_insort(s, src, victim);
                s.grp_of[victim] = (int8_t)src;
            }
            for (int t = 0; t < k * m; t++) out[t] = s.G[(t / m) * s.cap + t % m];
        }
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// the GA kernel

struct GASmem {
    LS ls;
    int16_t* snaps;     // max_snaps x km
    double* snapcost;   // max_snaps
    double* popcost;    // P
    int16_t* best;      // km
    int16_t* par;       // 2 x km (parents)
    int* ctl;           // [0] nsnap [1] stop [2] gen
};

__device__ __forceinline__ void copy16(int16_t* d, const int16_t* s, int n, int lane) {
    for (int t = lane; t < n; t += kWarp) d[t] = s[t];
}

// Prices candidates cand[0..cnt) (smem, km each): round-robin over the CTA's
// warps (d_pp <= 8, K1 warp evaluator) or one after another with the whole
// CTA (d_pp 9..16, hs_cta_eval.cuh); cost[i] = datap + pipelinep.  Called by
// every thread of the CTA.
template <typename KeyT, bool kM8, bool kCta>
struct Pricer {
    EvalView<KeyT> v;
    WarpScratch ws;
    CtaScratch cs;
    HKBig hkb;
    double* h;

    __device__ __noinline__ void all(const int16_t* cand, int cnt, int km, double* cost, int wid, int W,
                                     int lane) const {
        if constexpr (kCta) {
            for (int i = 0; i < cnt; i++) {
                double dp, pp;
                cta_price<KeyT, kM8>(v.n, v.k, v.m, v.DP, v.RK, v.vals, hkb, cs, h, cand + (size_t)i * km, dp, pp,
                                     v.ds, v.rs);
                if (threadIdx.x == 0) cost[i] = dp + pp;
                __syncthreads();
            }
        } else {
            for (int i = wid; i < cnt; i += W) {
                double dp, pp;
                warp_price<KeyT, kM8>(v, ws, cand + (size_t)i * km, lane, dp, pp);
                if (lane == 0) cost[i] = dp + pp;
                __syncwarp();
            }
        }
    }

    // warp-island mode: the calling warp prices one candidate with full outputs
    __device__ void one_warp(const int16_t* cand, int lane, double* out3, double* out_pg, int8_t* out_order) const {
        const int k = v.k;
        double dp, pp;
        warp_price<KeyT, kM8>(v, ws, cand, lane, dp, pp);
        if (lane == 0) {
            out3[0] = dp + pp;
            out3[1] = dp;
            out3[2] = pp;
            if (out_order) held_karp_order(k, ws.E, ws.h, v.hk.hoff, pp, out_order);
        }
        if (out_pg && lane < k) out_pg[lane] = ws.pg[lane];
        __syncwarp();
    }

    // price one candidate with full outputs; every thread calls it
    __device__ void one(const int16_t* cand, int wid, int lane, double* out3, double* out_pg, int8_t* out_order) const {
        const int k = v.k;
        if constexpr (kCta) {
            double dp, pp;
            cta_price<KeyT, kM8>(v.n, k, v.m, v.DP, v.RK, v.vals, hkb, cs, h, cand, dp, pp, v.ds, v.rs);
            if (threadIdx.x == 0) {
                out3[0] = dp + pp;
                out3[1] = dp;
                out3[2] = pp;
                if (out_order) held_karp_order_big(k, cs.E, h, hkb.off, pp, out_order);
            }
            if (out_pg && threadIdx.x < k) out_pg[threadIdx.x] = cs.pg[threadIdx.x];
            __syncthreads();
        } else {
            if (wid == 0) {
                double dp, pp;
                warp_price<KeyT, kM8>(v, ws, cand, lane, dp, pp);
                if (lane == 0) {
                    out3[0] = dp + pp;
                    out3[1] = dp;
                    out3[2] = pp;
                    if (out_order) held_karp_order(k, ws.E, ws.h, v.hk.hoff, pp, out_order);
                }
                if (out_pg && lane < k) out_pg[lane] = ws.pg[lane];
            }
            __syncthreads();
        }
    }
};

// Sets up the pricer's shared-memory pieces; advances `off`.
template <bool kSmemTables, typename KeyT, bool kM8, bool kCta>
__device__ inline Pricer<KeyT, kM8, kCta> make_pricer(int n, int k, int m, const double* dp, const void* rank,
                                                      const double* vals, const HKTables& hkt, const HKBig& hkb,
                                                      double* hk_scratch, size_t hk_size, const ScratchLayout& wl,
                                                      unsigned char* smem, size_t& off, int wid, int W) {
    Pricer<KeyT, kM8, kCta> pr;
    HKSmem hk{};
    if constexpr (!kCta) {
        hk = hk_global(hkt, smem);
        off = kHKGlobalBytes;
    }
    pr.v = stage_tables<kSmemTables, KeyT>(n, k, m, dp, rank, vals, hk, smem, off);
    if constexpr (kCta) {
        pr.cs = cta_scratch_at(smem + off, k, m);
        off += (cta_scratch_bytes(k, m) + 15) & ~(size_t)15;
        pr.hkb = hkb;
        pr.h = hk_scratch + (size_t)blockIdx.x * hk_size;
    } else {
        pr.ws = scratch_at(smem + off + (size_t)wid * wl.bytes, wl);
        off += (size_t)W * wl.bytes;
    }
    return pr;
}

// kWI (warp islands): every warp of the CTA runs its own island (its own
// working set, pricing its snapshots itself); the CTA only shares the staged
// tables.  Otherwise one island per CTA, warp 0 drives and all warps price.
template <bool kSmemTables, typename KeyT, bool kM8, bool kCta, bool kWI>
__global__ void __launch_bounds__(256) ga_kernel(GAArgs a, ScratchLayout wl) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int isl = kWI ? blockIdx.x * W + wid : blockIdx.x;
    auto island_sync = [&]() {
        HS_JITTER();
        if constexpr (kWI)
            __syncwarp();
        else
            __syncthreads();
    };
    const int pw = kWI ? 0 : wid, pW = kWI ? 1 : W;  // pricing lanes of this island
    const int n = a.n, k = a.k, m = kM8 ? 8 : a.m, km = k * m, P = a.pop, cap = m + 1;
    const int max_snaps = 1 + a.max_passes;
    size_t off = 0;
    const Pricer<KeyT, kM8, kCta> pr = make_pricer<kSmemTables, KeyT, kM8, kCta>(
        n, k, m, a.dp, a.rank, a.vals, a.hk, a.hkb, a.hk_scratch, a.hk_size, wl, smem, off, wid, W);
    const double* SW;
    if (kSmemTables) {
        double* ssw = reinterpret_cast<double*>(smem + off);
        off += (size_t)n * n * 8;
        for (int i = threadIdx.x; i < n * n; i += blockDim.x) ssw[i] = a.sw[i];
        SW = ssw;
    } else {
        SW = a.sw;
    }
    auto take = [&](size_t bytes) {
        unsigned char* p = smem + off;
        off += (bytes + 15) & ~(size_t)15;
        return p;
    };
    GASmem g;
    GAState* stp = nullptr;
    auto carve = [&]() {
        g.snaps = reinterpret_cast<int16_t*>(take((size_t)max_snaps * km * 2));
        g.snapcost = reinterpret_cast<double*>(take((size_t)max_snaps * 8));
        g.popcost = reinterpret_cast<double*>(take((size_t)P * 8));
        g.best = reinterpret_cast<int16_t*>(take((size_t)km * 2));
        g.par = reinterpret_cast<int16_t*>(take((size_t)2 * km * 2));
        g.ctl = reinterpret_cast<int*>(take(16 * 4));
        LS& s = g.ls;
        s.n = n;
        s.k = k;
        s.m = m;
        s.cap = cap;
        s.W = SW;
        s.w_sh = kSmemTables ? (uint32_t)__cvta_generic_to_shared(SW) : 0u;
        s.lat = !kWI;
        s.G = reinterpret_cast<int16_t*>(take((size_t)k * cap * 2));
        s.sz = reinterpret_cast<int*>(take((size_t)k * 4));
        s.mean = reinterpret_cast<double*>(take((size_t)n * k * 8));
        s.mver = reinterpret_cast<uint32_t*>(take((size_t)n * k * 4));
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
        stp = reinterpret_cast<GAState*>(take(sizeof(GAState)));
    };
    if constexpr (kWI) {
        for (int w = 0; w <= wid; w++) carve();
    } else {
        carve();
    }
    LS& s = g.ls;
    {
        const int t0 = kWI ? lane : threadIdx.x, dt = kWI ? kWarp : blockDim.x;
        for (int t = t0; t < n * k; t += dt) s.mver[t] = 0;
        for (int t = t0; t < k; t += dt) s.cver[t] = 1;
    }
    __syncthreads();
    if (kWI && isl >= a.islands) return;  // no block-wide syncs below in warp-island mode

    GAState& st = *stp;
    if ((kWI ? lane : threadIdx.x) == 0) st = a.state[isl];
    island_sync();

    int16_t* pop = a.pop_buf + (size_t)isl * P * km;
    double* gcost = a.cost_buf + (size_t)isl * P;
    int16_t* gbest = a.best_buf + (size_t)isl * km;
    Pcg64 rng;
    const bool driver = kWI || wid == 0;
    if (driver) rng.load(st.rng);
    if (a.prof && isl == 0 && threadIdx.x == 0) g_prof = a.prof;

    const bool st_was_init = st.initialized;
    int16_t* isnap = a.snap_buf ? a.snap_buf + (size_t)isl * a.snap_stride * km : nullptr;
    // phase 1: hand slots [cnt, snap_stride) over as invalid layouts (the
    // batch pricer skips them)
    auto emit_pad = [&](int cnt) {
        if (driver) {
            for (int q = cnt + lane; q < a.snap_stride; q += kWarp) isnap[(size_t)q * km] = -1;
            if (lane == 0) a.snap_cnt[isl] = cnt;
        }
    };
    bool emitted = false;
    if (!st.initialized) {
        // init_population (scheduler.py:124-136): sequential random_partition
        // draws, then price every member (:537-542)
        if (driver && a.phase != 2) {
            for (int i = 0; i < P; i++) {
                int16_t* dst = g.snaps;  // scratch
                if (lane == 0) {
                    for (int t = 0; t < n; t++) dst[t] = (int16_t)t;
                    for (int t = n - 1; t >= 1; t--) {
                        int jx = (int)rng.interval((uint64_t)t);
                        int16_t x = dst[t];
                        dst[t] = dst[jx];
                        dst[jx] = x;
                    }
                }
                __syncwarp();
                if (lane < k) {  // Partition sorts members
                    int16_t* gp = dst + lane * m;
                    for (int aa = 1; aa < m; aa++) {
                        int16_t x = gp[aa];
                        int b = aa - 1;
                        while (b >= 0 && gp[b] > x) {
                            gp[b + 1] = gp[b];
                            b--;
                        }
                        gp[b + 1] = x;
                    }
                }
                __syncwarp();
                copy16(pop + (size_t)i * km, dst, km, lane);
                __syncwarp();
            }
        }
        __threadfence_block();
        island_sync();
        if (a.phase == 1) {  // the population goes out for batch pricing
            if (driver) copy16(isnap, pop, P * km, lane);
            emit_pad(P);
            emitted = true;
        } else if (a.phase == 2) {
            const int t0 = kWI ? lane : threadIdx.x, dt = kWI ? kWarp : blockDim.x;
            for (int t = t0; t < P; t += dt) g.popcost[t] = a.snap_cost[(size_t)isl * a.snap_stride + t];
            island_sync();
        } else {
            // price the population in chunks of max_snaps through smem
            for (int c0 = 0; c0 < P; c0 += max_snaps) {
                int cnt = min(max_snaps, P - c0);
                const int t0 = kWI ? lane : threadIdx.x, dt = kWI ? kWarp : blockDim.x;
                for (int t = t0; t < cnt * km; t += dt) g.snaps[t] = pop[(size_t)c0 * km + t];
                island_sync();
                pr.all(g.snaps, cnt, km, g.popcost + c0, pw, pW, lane);
                island_sync();
            }
        }
        if (driver && !emitted) {
            if (lane == 0) {
                int bi = 0;
                for (int i = 1; i < P; i++)
                    if (g.popcost[i] < g.popcost[bi]) bi = i;  // min by (total, index)
                st.best_total = g.popcost[bi];
                st.best_idx = bi;
                st.since = 0;
                st.evaluations = P;
                st.gen = 0;
                st.stopped = 0;
                st.initialized = 1;
            }
            __syncwarp();
            copy16(gbest, pop + (size_t)st.best_idx * km, km, lane);
        }
    } else {
        const int t0 = kWI ? lane : threadIdx.x, dt = kWI ? kWarp : blockDim.x;
        for (int t = t0; t < P; t += dt) g.popcost[t] = gcost[t];
    }
    if (driver && lane == 0) {
        g.ctl[1] = st.stopped;
        g.ctl[2] = st.gen;
    }
    __threadfence_block();
    island_sync();

    // an emitted initial population, or its commit, runs no generation
    const bool init_call = emitted || (a.phase == 2 && !st_was_init);
    const int gen_end = init_call ? 0 : min(a.gen_end, a.generations);
    const int stop_after = a.kind == 0 ? 2 : 1;
    // CTA-mode islands with the register sweep path run the even passes as
    // waves over all warps (balanced groups are checked per pass below)
    const bool waves = !kWI && !kCta && a.kind == 0 && m == 8 && n <= 128 && W > 1;
    while (!g.ctl[1] && g.ctl[2] < gen_end) {
        const int gen = g.ctl[2];
        if (driver && a.phase != 2) {
            int i = 0, i2 = 0;
            if (lane == 0) {
                i = (int)rng.integers(0, P);
                i2 = (int)rng.integers(0, P - 1);
                if (i2 >= i) i2++;
            }
            i = __shfl_sync(kFull, i, 0);
            i2 = __shfl_sync(kFull, i2, 0);
            copy16(g.par, pop + (size_t)i * km, km, lane);
            copy16(g.par + km, pop + (size_t)i2 * km, km, lane);
            __syncwarp();
            long long t0 = clock64();
            crossover(s, g.par, g.par + km, rng, g.snaps, lane);
            long long t1 = clock64();
            if (a.prof && isl == 0 && lane == 0) a.prof[0] += t1 - t0;
            int nsnap = 1;
            if (a.kind != 2 && !waves) {  // _refine (:455-487)
                load_groups(s, g.snaps, lane);
                int stale = 0;
                for (int t = 0; t < a.max_passes; t++) {
                    bool changed;
                    long long p0 = clock64();
                    if (a.kind == 0)
                        changed = (s.sz[0] < 2) ? false : (t % 2 == 0 ? pass_sweep(s, rng, lane) : pass_chains(s, lane));
                    else
                        changed = pass_kl(s, lane);
                    long long p1 = clock64();
                    if (a.prof && isl == 0 && lane == 0) a.prof[1 + (t & 1)] += p1 - p0;
                    if (!changed) {
                        stale++;
                        if (stale >= stop_after) break;
                        continue;
                    }
                    stale = 0;
                    store_groups(s, g.snaps + (size_t)nsnap * km, lane);
                    nsnap++;
                }
            }
            if (waves) load_groups(s, g.snaps, lane);
            if (lane == 0) g.ctl[0] = nsnap;
        }
        if (waves && a.phase != 2) {
            // _refine with the even passes spread over the CTA's warps; the
            // odd passes (chains) stay on the driver warp
            island_sync();
            int nsnap = 1, stale = 0;
            for (int t = 0; t < a.max_passes; t++) {
                long long p0 = clock64();
                bool changed;
                if (t % 2 == 0) {
                    changed = s.w_sh ? pass_sweep_waves<true>(s, rng, wid, lane, W, g.ctl + 3)
                                     : pass_sweep_waves<false>(s, rng, wid, lane, W, g.ctl + 3);
                } else {
                    if (driver) {
                        const bool ch = pass_chains(s, lane);
                        if (lane == 0) g.ctl[3] = ch;
                    }
                    __syncthreads();
                    changed = g.ctl[3] != 0;
                }
                long long p1 = clock64();
                if (a.prof && isl == 0 && threadIdx.x == 0) a.prof[1 + (t & 1)] += p1 - p0;
                __syncthreads();  // every thread has read the flag before it is reused
                if (!changed) {
                    stale++;
                    if (stale >= stop_after) break;
                    continue;
                }
                stale = 0;
                if (driver) store_groups(s, g.snaps + (size_t)nsnap * km, lane);
                nsnap++;
            }
            if (threadIdx.x == 0) g.ctl[0] = nsnap;
        }
        long long q0 = clock64();
        island_sync();
        if (a.phase == 1) {  // this generation's snapshots go out for batch pricing
            const int ns = g.ctl[0];
            if (driver) copy16(isnap, g.snaps, ns * km, lane);
            emit_pad(ns);
            emitted = true;
            break;
        }
        if (a.phase == 2 && driver && lane == 0) g.ctl[0] = a.snap_cnt[isl];
        island_sync();
        const int nsnap = g.ctl[0];
        if (a.phase == 2) {
            const int t0 = kWI ? lane : threadIdx.x, dt = kWI ? kWarp : blockDim.x;
            for (int t = t0; t < nsnap; t += dt) g.snapcost[t] = a.snap_cost[(size_t)isl * a.snap_stride + t];
        } else {
            pr.all(g.snaps, nsnap, km, g.snapcost, pw, pW, lane);
        }
        island_sync();
        if (a.prof && isl == 0 && lane == 0 && driver) a.prof[3] += clock64() - q0;
        if (driver) {
            int bsi = 0, worst = 0, replace = 0, improve = 0;
            double cb = 0.0;
            if (lane == 0) {
                for (int q = 1; q < nsnap; q++)
                    if (g.snapcost[q] < g.snapcost[bsi]) bsi = q;  // first strict minimum
                cb = g.snapcost[bsi];
                st.evaluations += nsnap;
                for (int t = 1; t < P; t++)
                    if (g.popcost[t] > g.popcost[worst]) worst = t;  // first maximum
                replace = cb < g.popcost[worst];
                improve = cb < st.best_total;
                if (replace) g.popcost[worst] = cb;
                if (improve) {
                    st.best_total = cb;
                    st.since = 0;
                } else {
                    st.since++;
                }
            }
            bsi = __shfl_sync(kFull, bsi, 0);
            worst = __shfl_sync(kFull, worst, 0);
            replace = __shfl_sync(kFull, replace, 0);
            improve = __shfl_sync(kFull, improve, 0);
            const int16_t* refined = (a.phase == 2 ? isnap : g.snaps) + (size_t)bsi * km;
            if (replace) copy16(pop + (size_t)worst * km, refined, km, lane);
            if (improve) copy16(gbest, refined, km, lane);
            __syncwarp();
            if (lane == 0) {
                if (a.trace_best) a.trace_best[(size_t)isl * a.generations + gen] = st.best_total;
                if (a.trace_mean) a.trace_mean[(size_t)isl * a.generations + gen] = pw_array(g.popcost, P) / (double)P;
                st.gen = gen + 1;
                g.ctl[2] = gen + 1;
                if (a.patience > 0 && st.since >= a.patience) {
                    st.stopped = 1;
                    g.ctl[1] = 1;
                }
            }
        }
        __threadfence_block();
        island_sync();
        if (a.phase == 2) break;  // one generation per commit
    }
    if (a.phase == 1 && !emitted) emit_pad(0);  // stopped or done: nothing to price

    // persist population costs; finalize when the run is over
    {
        const int t0 = kWI ? lane : threadIdx.x, dt = kWI ? kWarp : blockDim.x;
        for (int t = t0; t < P; t += dt) gcost[t] = g.popcost[t];
    }
    bool finished = g.ctl[1] || g.ctl[2] >= a.generations;
    if (finished && a.finalize && !st.finalized && a.phase == 0) {
        // canonical() (costmodel.py:86-88) then a last priced evaluation (:572-574)
        if (driver && lane == 0) {
            int ord[16];
            for (int j = 0; j < k; j++) ord[j] = j;
            for (int x = 1; x < k; x++) {
                int y = ord[x], b = x - 1;
                while (b >= 0 && gbest[ord[b] * m] > gbest[y * m]) {
                    ord[b + 1] = ord[b];
                    b--;
                }
                ord[b + 1] = y;
            }
            for (int j = 0; j < k; j++)
                for (int i = 0; i < m; i++) g.snaps[j * m + i] = gbest[ord[j] * m + i];
        }
        island_sync();
        if constexpr (kWI)
            pr.one_warp(g.snaps, lane, a.out3 + isl * 3, a.out_pg ? a.out_pg + (size_t)isl * k : nullptr,
                        a.out_order ? a.out_order + (size_t)isl * k : nullptr);
        else
            pr.one(g.snaps, wid, lane, a.out3 + isl * 3, a.out_pg ? a.out_pg + (size_t)isl * k : nullptr,
                   a.out_order ? a.out_order + (size_t)isl * k : nullptr);
        if (driver) {
            copy16(a.out_groups + (size_t)isl * km, g.snaps, km, lane);
            if (lane == 0) {
                st.evaluations += 1;
                st.finalized = 1;
            }
        }
    }
    island_sync();
    if (driver && lane == 0) {
        rng.store(st.rng);
        a.state[isl] = st;
    }
}

// ---------------------------------------------------------------------------
// local_search (scheduler.py:490-512): _refine on a batch of partitions, one
// CTA each with its own PCG64 stream; returns the best truly-priced layout.

template <bool kSmemTables, typename KeyT, bool kM8, bool kCta>
__global__ void __launch_bounds__(256) refine_kernel(RefineArgs a, ScratchLayout wl) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int b = blockIdx.x;
    const int n = a.n, k = a.k, m = kM8 ? 8 : a.m, km = k * m, cap = m + 1;
    const int max_snaps = 1 + a.max_passes;
    size_t off = 0;
    const Pricer<KeyT, kM8, kCta> pr = make_pricer<kSmemTables, KeyT, kM8, kCta>(
        n, k, m, a.dp, a.rank, a.vals, a.hk, a.hkb, a.hk_scratch, a.hk_size, wl, smem, off, wid, W);
    const double* SW;
    if (kSmemTables) {
        double* ssw = reinterpret_cast<double*>(smem + off);
        off += (size_t)n * n * 8;
        for (int i = threadIdx.x; i < n * n; i += blockDim.x) ssw[i] = a.sw[i];
        SW = ssw;
    } else {
        SW = a.sw;
    }
    auto take = [&](size_t bytes) {
        unsigned char* p = smem + off;
        off += (bytes + 15) & ~(size_t)15;
        return p;
    };
    int16_t* snaps = reinterpret_cast<int16_t*>(take((size_t)max_snaps * km * 2));
    double* snapcost = reinterpret_cast<double*>(take((size_t)max_snaps * 8));
    int* ctl = reinterpret_cast<int*>(take(16 * 4));
    LS s;
    s.n = n;
    s.k = k;
    s.m = m;
    s.cap = cap;
    s.W = SW;
    s.w_sh = kSmemTables ? (uint32_t)__cvta_generic_to_shared(SW) : 0u;
    s.lat = true;
    s.G = reinterpret_cast<int16_t*>(take((size_t)k * cap * 2));
    s.sz = reinterpret_cast<int*>(take((size_t)k * 4));
    s.mean = reinterpret_cast<double*>(take((size_t)n * k * 8));
    s.mver = reinterpret_cast<uint32_t*>(take((size_t)n * k * 4));
    s.cver = reinterpret_cast<uint32_t*>(take((size_t)k * 4));
    for (int t = threadIdx.x; t < n * k; t += blockDim.x) s.mver[t] = 0;
    for (int t = threadIdx.x; t < k; t += blockDim.x) s.cver[t] = 1;
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
    for (int t = threadIdx.x; t < km; t += blockDim.x) snaps[t] = a.groups[(size_t)b * km + t];
    __syncthreads();
    Pcg64 rng;
    if (wid == 0) {
        rng.load(a.rng[b]);
        int nsnap = 1;
        if (a.single_pass) {
            load_groups(s, snaps, lane);
            bool ch = a.kind == 0 ? ((s.sz[0] < 2) ? false : (a.phase % 2 == 0 ? pass_sweep(s, rng, lane) : pass_chains(s, lane)))
                                  : pass_kl(s, lane);
            store_groups(s, a.out_groups + (size_t)b * km, lane);
            if (lane == 0) a.changed[b] = ch;
        } else {
            load_groups(s, snaps, lane);
            int stale = 0, stop_after = a.kind == 0 ? 2 : 1;
            for (int t = 0; t < a.max_passes; t++) {
                bool changed = a.kind == 0 ? ((s.sz[0] < 2) ? false : (t % 2 == 0 ? pass_sweep(s, rng, lane) : pass_chains(s, lane)))
                                           : pass_kl(s, lane);
                if (!changed) {
                    stale++;
                    if (stale >= stop_after) break;
                    continue;
                }
                stale = 0;
                store_groups(s, snaps + (size_t)nsnap * km, lane);
                nsnap++;
            }
        }
        if (lane == 0) {
            ctl[0] = nsnap;
            rng.store(a.rng[b]);
        }
        if (a.snap_buf && !a.single_pass) {  // snapshots out for batch pricing
            int16_t* dst = a.snap_buf + (size_t)b * a.snap_stride * km;
            copy16(dst, snaps, nsnap * km, lane);
            for (int q = nsnap + lane; q < a.snap_stride; q += kWarp) dst[(size_t)q * km] = -1;
            if (lane == 0) a.snap_cnt[b] = nsnap;
        }
    }
    __syncthreads();
    if (a.single_pass || a.snap_buf) return;
    const int nsnap = ctl[0];
    pr.all(snaps, nsnap, km, snapcost, wid, W, lane);
    __syncthreads();
    if (wid == 0) {
        int bsi = 0;
        if (lane == 0)
            for (int q = 1; q < nsnap; q++)
                if (snapcost[q] < snapcost[bsi]) bsi = q;
        bsi = __shfl_sync(kFull, bsi, 0);
        copy16(a.out_groups + (size_t)b * km, snaps + (size_t)bsi * km, km, lane);
        if (lane == 0) {
            a.out_cost[b] = snapcost[bsi];
            a.evaluations[b] = nsnap;
        }
    }
}

// ---------------------------------------------------------------------------
// kernel-variant launchers (explicitly instantiated per translation unit)

template <bool S, typename KT, bool M8, bool CT>
int launch_ga_t(const GAArgs& a, const SearchPlan& plan, int islands, cudaStream_t st) {
    ScratchLayout wl = scratch_layout(a.k <= 8 ? a.k : 8, a.m);
    if constexpr (!CT) {
        if (plan.warp_islands) {
            cudaFuncSetAttribute(ga_kernel<S, KT, M8, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)plan.smem);
            int blocks = (islands + plan.warps - 1) / plan.warps;
            ga_kernel<S, KT, M8, false, true><<<blocks, plan.warps * 32, plan.smem, st>>>(a, wl);
            return cudaGetLastError() == cudaSuccess ? 0 : -1;
        }
    }
    cudaFuncSetAttribute(ga_kernel<S, KT, M8, CT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
    ga_kernel<S, KT, M8, CT, false><<<islands, plan.warps * 32, plan.smem, st>>>(a, wl);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <bool CT>
int launch_ga_c(const GAArgs& a, const SearchPlan& plan, int islands, bool key16, cudaStream_t st) {
    if (plan.m8) return plan.smem_tables ? launch_ga_t<true, uint16_t, true, CT>(a, plan, islands, st)
                                         : launch_ga_t<false, uint16_t, true, CT>(a, plan, islands, st);
    if (key16) return plan.smem_tables ? launch_ga_t<true, uint16_t, false, CT>(a, plan, islands, st)
                                       : launch_ga_t<false, uint16_t, false, CT>(a, plan, islands, st);
    return plan.smem_tables ? launch_ga_t<true, uint32_t, false, CT>(a, plan, islands, st)
                            : launch_ga_t<false, uint32_t, false, CT>(a, plan, islands, st);
}


template <bool S, typename KT, bool M8, bool CT>
int launch_refine_t(const RefineArgs& a, const SearchPlan& plan, int B, cudaStream_t st) {
    ScratchLayout wl = scratch_layout(a.k <= 8 ? a.k : 8, a.m);
    cudaFuncSetAttribute(refine_kernel<S, KT, M8, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem);
    refine_kernel<S, KT, M8, CT><<<B, plan.warps * 32, plan.smem, st>>>(a, wl);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <bool CT>
int launch_refine_c(const RefineArgs& a, const SearchPlan& plan, int B, bool key16, cudaStream_t st) {
    if (plan.m8) return plan.smem_tables ? launch_refine_t<true, uint16_t, true, CT>(a, plan, B, st)
                                         : launch_refine_t<false, uint16_t, true, CT>(a, plan, B, st);
    if (key16) return plan.smem_tables ? launch_refine_t<true, uint16_t, false, CT>(a, plan, B, st)
                                       : launch_refine_t<false, uint16_t, false, CT>(a, plan, B, st);
    return plan.smem_tables ? launch_refine_t<true, uint32_t, false, CT>(a, plan, B, st)
                            : launch_refine_t<false, uint32_t, false, CT>(a, plan, B, st);
}

}  // namespace hs
