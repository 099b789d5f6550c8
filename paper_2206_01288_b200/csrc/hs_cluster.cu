// hs_cluster.cu -- exact pricing for 9 <= d_pp <= 16 without a stage order
// (BASELINE configs 4 and 5: Held-Karp over up to 2^16 subsets).
//
// Two kernels per chunk of candidates:
//   stage_kernel      one CTA per candidate (many per SM, latency hidden by
//                     occupancy): validation, datap (numpy pairwise row
//                     sums, group maxima) and the C(k,2) bottleneck edges of
//                     the coarsened stage graph -> E in global memory.
//   hk_cluster_kernel one thread-block cluster per candidate: Held-Karp
//                     (combinatorics.py:258-276) keeping only popcount layers
//                     p-1 and p, each layer split by whole sets over the
//                     cluster's CTAs' shared memory.  Work is "pushed": the
//                     CTA owning r reads h[r][.] from its own shared memory
//                     and sends every h[r | u][u] to the owner of r | u as an
//                     asynchronous DSMEM store completing on that CTA's
//                     mbarrier for the layer (st.async ... complete_tx); a
//                     relaxed cluster barrier only guards buffer reuse.  At
//                     k = 16 the two live layers are 2 x 102,960 doubles
//                     (1.65 MB): 16 CTAs x 105 KB, two CTAs per SM, so the
//                     table never leaves the SMs.
// Values are the reference's: h[s][u] = min_v (w[u][v] + h[s\u][v]) with
// strict '<' (the min of a set of doubles does not depend on visit order),
// total = first minimum over the full set.  Stage orders still use the
// full-table CTA path (hs_big.cu).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <vector>

#include "hs_cluster.h"
#include "hs_cta_eval.cuh"
#include "hs_tma.cuh"

namespace cg = cooperative_groups;

namespace hs {

constexpr int kClusterThreads = 512;
static_assert(kStageES == kES16, "stage graph stride");

template <typename KeyT, bool kM8>
__global__ void __launch_bounds__(128) stage_kernel(EvalArgs a, double* __restrict__ Eout, double* __restrict__ dpout,
                                                    uint8_t* __restrict__ bad_out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int k = a.k, m = kM8 ? 8 : a.m, km = k * m;
    CtaScratch cs = cta_scratch_at(smem, k, m);
    size_t off = cta_scratch_bytes(k, m);
    int16_t* mem = reinterpret_cast<int16_t*>(smem + off);
    off += ((size_t)km * 2 + 15) & ~(size_t)15;
    uint32_t* seen = reinterpret_cast<uint32_t*>(smem + off);
    __shared__ int bad;
    const KeyT* RK = reinterpret_cast<const KeyT*>(a.rank);
    const int nwords = (a.n + 31) >> 5;
    for (int64_t p = blockIdx.x; p < a.P; p += gridDim.x) {
        const int16_t* gsrc = a.groups + p * km;
        for (int i = threadIdx.x; i < km; i += blockDim.x) mem[i] = gsrc[i];
        for (int i = threadIdx.x; i < nwords; i += blockDim.x) seen[i] = 0;
        if (threadIdx.x == 0) bad = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < km; i += blockDim.x) {  // costmodel.py:58-72
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
                if (a.datap) a.datap[p] = nan;
                bad_out[p] = 1;
                atomicAdd(a.invalid, 1);
            }
            __syncthreads();
            continue;
        }
        const double datap = cta_stage<KeyT, kM8>(a.n, k, m, a.dp, RK, a.vals, cs, mem);
        double* E = Eout + p * kStageStride;
        for (int i = threadIdx.x; i < k * kES16; i += blockDim.x) E[i] = cs.E[i];
        if (threadIdx.x == 0) {
            dpout[p] = datap;
            bad_out[p] = 0;
            if (a.datap) a.datap[p] = datap;
        }
        if (a.per_group && threadIdx.x < k) a.per_group[p * k + threadIdx.x] = cs.pg[threadIdx.x];
        __syncthreads();
    }
}

// min over NV values as a balanced tree (the value of a min of doubles does
// not depend on the order; a short dependency chain instead of NV - 1)
template <int NV>
__device__ __forceinline__ double tree_min(const double (&c)[NV]) {
    double x[NV];
#pragma unroll
    for (int i = 0; i < NV; i++) x[i] = c[i];
#pragma unroll
    for (int w = 1; w < NV; w *= 2)
#pragma unroll
        for (int i = 0; i + w < NV; i += 2 * w) x[i] = x[i + w] < x[i] ? x[i + w] : x[i];
    return x[0];
}

// ---------------------------------------------------------------------------
// cluster plumbing: asynchronous DSMEM pushes completing on the owner's
// mbarrier (st.async ... complete_tx) and a relaxed cluster barrier that only
// orders layers (no release fence: data visibility comes from the mbarrier)

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t a, uint32_t q) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(q));
    return r;
}
__device__ __forceinline__ void cl_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
__device__ __forceinline__ void push_f64(uint32_t addr, double v, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr), "d"(v),
                 "r"(mbar)
                 : "memory");
}
// announce a phase's bytes (the one arrival of the phase); pushes may land
// before it (the tx-count goes transiently negative: scripts/probes/stas_probe)
__device__ __forceinline__ void expect_bytes(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
// phase wait; traps instead of hanging if a phase never completes (a
// schedule bug must fail the launch, not wedge the GPU)
__device__ __forceinline__ void layer_wait(uint32_t mbar, uint32_t parity) {
    uint32_t done;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(mbar), "r"(parity) : "memory");
    if (done) return;
    const long long t0 = clock64();
    for (;;) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(mbar), "r"(parity) : "memory");
        if (done) return;
#ifdef HS_HK_DEBUG
        if (clock64() - t0 > 4000000000LL) {
            uint64_t raw;
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(raw) : "r"(mbar));
            if ((threadIdx.x & 31) == 0)
                printf("hk timeout: rank %u tid %d mbar %u parity %u raw %016llx\n", cluster_rank(), threadIdx.x, mbar,
                       parity, (unsigned long long)raw);
            return;
        }
#else
        if (clock64() - t0 > 20000000000LL) __trap();
#endif
    }
}

// Where layer p's results go: buffer (p & 1) of the destination CTA, counted
// on that CTA's mbarrier (p & 1).  delta[q] maps a local shared address to
// CTA q's copy (offsets within a CTA's window are preserved).
struct PushTo {
    uint32_t buf;   // local shared address of the destination buffer
    uint32_t mbar;  // local shared address of the destination mbarrier
    const uint32_t* delta;
    __device__ __forceinline__ void put(uint32_t d, double v) const {
        const uint32_t dq = delta[d >> 17];
        push_f64(buf + (d & 0x1FFFFu) * 8u + dq, v, mbar + dq);
    }
};

// Work item (rwords[i]): source set r, local slot of h[r][first member],
// first destination word, and the item's share of the u not in r (skip the
// j0 lowest, take cnt).  Layers with few sources split each source's u over
// several items (one L2 round trip per thread instead of a chain of them).
struct Item {
    uint32_t r, rest;
    int lr, cnt;
    const uint32_t* dw;
    __device__ __forceinline__ Item(uint64_t w, uint32_t full, const uint32_t* __restrict__ dwords) {
        r = (uint32_t)(w & 0xFFFF);
        lr = (int)(w >> 16) & 0x7FFF;
        dw = dwords + ((w >> 31) & 0x1FFFFF);
        const int j0 = (int)(w >> 52) & 0xF;
        cnt = (int)(w >> 56) & 0x1F;
        rest = full & ~r;
        for (int j = 0; j < j0; j++) rest &= rest - 1;
    }
};

// One item of source block r (NV = p - 1 members): h[r][.] (own shared
// memory) and the byte offsets of w[.][v] for v in r stay in registers while
// the item's u are relaxed, two at a time (independent loads / adds / min
// trees).  (Loading the destination words one pair ahead costs registers at
// the 64-register cap: config 4 151k -> 145k, measured.)
template <int NV>
__device__ __forceinline__ void two_source(const double* Es, const double* own, uint64_t w, uint32_t full,
                                           const uint32_t* __restrict__ dwords, const PushTo& to) {
    Item it(w, full, dwords);
    uint32_t r = it.r, rest = it.rest;
    const int cnt = it.cnt;
    const uint32_t* dw = it.dw;
    double hv[NV];
    const char* ev[NV];  // &w[0][v]
#pragma unroll
    for (int i = 0; i < NV; i++) {
        const int v = __ffs(r) - 1;
        r &= r - 1;
        ev[i] = reinterpret_cast<const char*>(Es) + v * 8;
        hv[i] = own[it.lr + i];
    }
    for (int j = 0; j < cnt; j += 2) {
        const uint32_t d0 = __ldg(dw + j), d1 = j + 1 < cnt ? __ldg(dw + j + 1) : 0u;
        const int u0 = __ffs(rest) - 1;
        rest &= rest - 1;
        const bool two = j + 1 < cnt;
        const int u1 = two ? __ffs(rest) - 1 : u0;
        rest &= rest - 1;
        const int o0 = u0 * kES16 * 8, o1 = u1 * kES16 * 8;
        double c0[NV], c1[NV];
#pragma unroll
        for (int i = 0; i < NV; i++) {
            c0[i] = *reinterpret_cast<const double*>(ev[i] + o0) + hv[i];
            c1[i] = *reinterpret_cast<const double*>(ev[i] + o1) + hv[i];
        }
        to.put(d0, tree_min<NV>(c0));
        if (two) to.put(d1, tree_min<NV>(c1));
    }
}

// layer 2: r = {v}, h[r][v] = 0 (implicit): h[{u, v}][u] = w[u][v]
__device__ __forceinline__ void two_source_first(const double* Es, uint64_t w, uint32_t full,
                                                 const uint32_t* __restrict__ dwords, const PushTo& to) {
    Item it(w, full, dwords);
    const int v = __ffs(it.r) - 1;
    uint32_t rest = it.rest;
    for (int j = 0; j < it.cnt; j++) {
        const int u = __ffs(rest) - 1;
        rest &= rest - 1;
        to.put(__ldg(it.dw + j), Es[u * kES16 + v]);  // w[u][v] + 0.0
    }
}

// Layer sequencing per candidate (k - 1 layers, p = 2..k):
//   wait    cluster barrier: every CTA finished layer p - 1's tasks, so no
//           CTA still reads buffer (p & 1) (it held layer p - 2), and every
//           thread here has seen mbarrier (p & 1)'s previous phase complete;
//           thread 0 announces layer p's bytes on it (announcing earlier
//           could complete a 0-byte phase while a slow thread still waits on
//           the previous one with the same parity: measured, a hang)
//   wait    own mbarrier (p - 1) & 1: all of layer p - 1 has landed here
//   tasks   push layer p
//   arrive  (relaxed)
// After layer k, the full set's entries are read on CTA 0 before the last
// arrive.  Two 512-thread CTAs per SM (64
// registers): 16-CTA clusters cover 8 SMs, 18 co-resident clusters.
// Measured and rejected (round 2): the serial min chain at 64 registers, a
// per-CTA mbarrier layer barrier with plain DSMEM stores and release fences,
// three rotating buffers with the cluster barrier a layer off the critical
// path (needs one 1,024-thread CTA per SM: config 4 153k -> 127k, the second
// co-resident cluster per SM is worth more than the barrier slack).
#ifndef HS_HK_MINB
#define HS_HK_MINB 2
#endif
__global__ void __launch_bounds__(kClusterThreads, HS_HK_MINB) hk_cluster_kernel(const double* __restrict__ E, int es,
                                                                     int64_t estride, int k, int64_t B, HKTwo t,
                                                                     const double* __restrict__ add,
                                                                     const uint8_t* __restrict__ bad,
                                                                     double* __restrict__ out_total,
                                                                     double* __restrict__ out_pipe) {
    extern __shared__ __align__(16) double sm2[];
    __shared__ __align__(8) uint64_t mb[2];
    __shared__ uint32_t delta[16];
    const int rank = (int)cluster_rank(), cs = t.cs;
    double* Es = sm2 + 2 * t.Cmax;
    const uint32_t lbuf0 = smem_addr(sm2), lbstride = (uint32_t)t.Cmax * 8u;
    const uint32_t lmb0 = smem_addr(&mb[0]);  // mb[1] is 8 bytes further
    const int64_t ncl = gridDim.x / cs;
    if (threadIdx.x < cs) delta[threadIdx.x] = mapa_rank(lbuf0, threadIdx.x) - lbuf0;
    if (threadIdx.x == 0) {
        mbar_init(&mb[0], 1);
        mbar_init(&mb[1], 1);
    }
    __syncthreads();
    cg::this_cluster().sync();  // mbarrier inits visible cluster-wide
    cl_arrive_relaxed();
    uint32_t phase = 0;  // bit b: parity of the next phase of mb[b]
    const uint32_t full = (1u << k) - 1u;
    for (int64_t b = blockIdx.x / cs; b < B; b += ncl) {
        if (bad && bad[b]) {  // the same for every CTA of the cluster: no layer, no barrier
            if (rank == 0 && threadIdx.x == 0) {
                const double nan = __longlong_as_double(0x7ff8000000000000LL);
                out_total[b] = nan;
                if (out_pipe) out_pipe[b] = nan;
            }
            continue;
        }
        __syncthreads();  // every task of the previous candidate read Es
        const double* src = E + b * estride;
        for (int i = threadIdx.x; i < k * k; i += blockDim.x) {
            const int rr = i / k, cc = i - rr * k;
            Es[rr * kES16 + cc] = src[(size_t)rr * es + cc];
        }
        __syncthreads();
        for (int p = 2; p <= k; p++) {
            HS_JITTER();
            cl_wait();
            if (threadIdx.x == 0)
                expect_bytes(lmb0 + 8 * (p & 1), (uint32_t)((t.sbeg[p][rank + 1] - t.sbeg[p][rank]) * p * 8));
            if (p >= 3) {
                const int pb = (p - 1) & 1;
                layer_wait(lmb0 + 8 * pb, (phase >> pb) & 1u);
                phase ^= 1u << pb;
            }
            const PushTo to{lbuf0 + (p & 1) * lbstride, lmb0 + 8 * (p & 1), delta};
            const double* own = sm2 + ((p - 1) & 1) * t.Cmax;
            const int end = t.rbeg[p][rank + 1];
            for (int x = t.rbeg[p][rank] + (int)threadIdx.x; x < end; x += blockDim.x) {
                const uint64_t rw = __ldg(t.rwords + x);
                switch (p) {
                    case 2: two_source_first(Es, rw, full, t.dwords, to); break;
                    case 3: two_source<2>(Es, own, rw, full, t.dwords, to); break;
                    case 4: two_source<3>(Es, own, rw, full, t.dwords, to); break;
                    case 5: two_source<4>(Es, own, rw, full, t.dwords, to); break;
                    case 6: two_source<5>(Es, own, rw, full, t.dwords, to); break;
                    case 7: two_source<6>(Es, own, rw, full, t.dwords, to); break;
                    case 8: two_source<7>(Es, own, rw, full, t.dwords, to); break;
                    case 9: two_source<8>(Es, own, rw, full, t.dwords, to); break;
                    case 10: two_source<9>(Es, own, rw, full, t.dwords, to); break;
                    case 11: two_source<10>(Es, own, rw, full, t.dwords, to); break;
                    case 12: two_source<11>(Es, own, rw, full, t.dwords, to); break;
                    case 13: two_source<12>(Es, own, rw, full, t.dwords, to); break;
                    case 14: two_source<13>(Es, own, rw, full, t.dwords, to); break;
                    case 15: two_source<14>(Es, own, rw, full, t.dwords, to); break;
                    default: two_source<15>(Es, own, rw, full, t.dwords, to); break;
                }
            }
            HS_JITTER();
            if (p < k) cl_arrive_relaxed();
        }
        {  // layer k: the full set's k entries, slots 0..k-1 of CTA 0
            const int kb = k & 1;
            layer_wait(lmb0 + 8 * kb, (phase >> kb) & 1u);
            phase ^= 1u << kb;
            if (rank == 0 && threadIdx.x == 0) {
                const double* fin = sm2 + kb * t.Cmax;
                double tot = fin[0];
                for (int u = 1; u < k; u++) tot = dmin(tot, fin[u]);
                if (add) {
                    out_total[b] = add[b] + tot;
                    if (out_pipe) out_pipe[b] = tot;
                } else {
                    out_total[b] = tot;
                }
            }
        }
        cl_arrive_relaxed();
    }
    cl_wait();  // no CTA leaves while a peer may still push into its shared memory
}

// ---------------------------------------------------------------------------
// host side

namespace {
struct DeviceHKTwo {
    uint64_t* rw = nullptr;
    uint32_t* dw = nullptr;
    HKTwo t{};
};
std::mutex g_two_mu;
std::map<std::pair<int, int>, DeviceHKTwo> g_two;

uint64_t binom(int n, int r) {
    if (r < 0 || r > n) return 0;
    uint64_t v = 1;
    for (int i = 1; i <= r; i++) v = v * (uint64_t)(n - r + i) / (uint64_t)i;
    return v;
}
}  // namespace

size_t cluster_smem_bytes(const HKTwo& t) { return (size_t)(2 * t.Cmax + 16 * kES16) * 8; }

int get_hk_two(int device, int k, HKTwo* out) {
    if (k < 2 || k > 16) return -3;
    std::lock_guard<std::mutex> lk(g_two_mu);
    auto key = std::make_pair(device, k);
    auto it = g_two.find(key);
    if (it == g_two.end()) {
        int optin = 0;
        if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) return -1;
        auto slice = [&](int cs) {  // longest per-CTA slice, whole sets
            uint64_t m = 0;
            for (int p = 2; p <= k; p++) m = std::max<uint64_t>(m, (binom(k, p) + cs - 1) / cs * (uint64_t)p);
            return m;
        };
        DeviceHKTwo d;
        d.t.cs = 0;
        // smallest cluster whose CTAs fit two per SM (32 resident warps);
        // failing that, the smallest that fits one per SM
        for (int pass = 0; pass < 2 && !d.t.cs; pass++) {
            const uint64_t budget = pass == 0 ? (uint64_t)optin / 2 - 2048 : (uint64_t)optin - 1024;
            for (int cs = 1; cs <= 16; cs *= 2) {
                if ((2 * slice(cs) + 16 * kES16) * 8 <= budget) {
                    d.t.cs = cs;
                    break;
                }
            }
        }
        const int cs = d.t.cs;
        // whole sets per CTA, ceil split (layer k's single set lives on CTA 0)
        std::vector<std::vector<int>> owner(k + 1);
        d.t.Cmax = 0;
        for (int p = 0; p < 18; p++) {
            for (int q = 0; q < 17; q++) d.t.sbeg[p][q] = 0;
            d.t.C[p] = 1;
            if (p < 1 || p > k) continue;
            const uint64_t n = binom(k, p);
            for (int q = 0; q <= cs; q++) d.t.sbeg[p][q] = (int)((n * (uint64_t)q + cs - 1) / (uint64_t)cs);
            for (int q = cs + 1; q < 17; q++) d.t.sbeg[p][q] = (int)n;
            int most = 0;
            owner[p].resize(n);
            for (int q = 0; q < cs; q++) {
                most = std::max(most, d.t.sbeg[p][q + 1] - d.t.sbeg[p][q]);
                for (int i = d.t.sbeg[p][q]; i < d.t.sbeg[p][q + 1]; i++) owner[p][i] = q;
            }
            d.t.C[p] = most * p;
            if (p >= 2) d.t.Cmax = std::max(d.t.Cmax, d.t.C[p]);
        }
        std::vector<int> rank_of((size_t)1 << k, 0), cnt(k + 2, 0);
        for (int s = 0; s < (1 << k); s++) rank_of[s] = cnt[__builtin_popcount(s)]++;
        std::vector<uint64_t> rws;
        std::vector<uint32_t> dws;
        dws.reserve(((size_t)k << (k - 1)));
        std::vector<std::vector<uint64_t>> per(cs);
        std::vector<std::vector<uint32_t>> perd(cs);
        for (int p = 0; p < 18; p++) {
            for (int q = 0; q < 17; q++) d.t.rbeg[p][q] = (int)rws.size();
            if (p < 2 || p > k) continue;
            for (int q = 0; q < cs; q++) {
                per[q].clear();
                perd[q].clear();
            }
            // u per source, and how many items each source is split into so
            // that a CTA's items about fill its threads
            const int U = k - (p - 1);
            const int tmax = (int)((binom(k, p - 1) + cs - 1) / cs);
            const int parts = std::max(1, std::min(U, kClusterThreads / std::max(1, tmax)));
            int spread = 0;
            for (int r = 1; r < (1 << k); r++) {  // sources in rank order of layer p-1
                if (__builtin_popcount(r) != p - 1) continue;
                uint64_t lr = 0;
                int o;
                if (p >= 3) {
                    o = owner[p - 1][rank_of[r]];
                    lr = (uint64_t)(rank_of[r] - d.t.sbeg[p - 1][o]) * (uint64_t)(p - 1);
                } else {
                    o = spread++ % cs;  // layer 1 is implicit zeros: deal sources round-robin
                }
                const uint64_t dw0 = perd[o].size();  // relative; rebased below
                for (int u = 0; u < k; u++) {
                    if (r >> u & 1) continue;
                    const int s = r | (1 << u);
                    const int q = owner[p][rank_of[s]];
                    const uint64_t ls = (uint64_t)(rank_of[s] - d.t.sbeg[p][q]) * (uint64_t)p +
                                        __builtin_popcount(s & ((1 << u) - 1));
                    perd[o].push_back((uint32_t)(((uint64_t)q << 17) | ls));
                }
                for (int c = 0, j0 = 0; c < parts; c++) {
                    const int cnt = U / parts + (c < U % parts ? 1 : 0);
                    per[o].push_back((uint64_t)r | lr << 16 | (dw0 + j0) << 31 | (uint64_t)j0 << 52 |
                                     (uint64_t)cnt << 56);
                    j0 += cnt;
                }
            }
            for (int q = 0; q < cs; q++) {
                d.t.rbeg[p][q] = (int)rws.size();
                const uint64_t base = dws.size();
                for (uint64_t w : per[q]) rws.push_back(w + (base << 31));
                dws.insert(dws.end(), perd[q].begin(), perd[q].end());
            }
            for (int q = cs; q < 17; q++) d.t.rbeg[p][q] = (int)rws.size();
        }
        if (d.t.Cmax >= (1 << 15) || dws.size() >= ((size_t)1 << 21)) return -3;  // item word fields
        if (cudaMalloc(&d.rw, rws.size() * 8) != cudaSuccess) return -1;
        if (cudaMalloc(&d.dw, dws.size() * 4) != cudaSuccess) return -1;
        if (cudaMemcpy(d.rw, rws.data(), rws.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) return -1;
        if (cudaMemcpy(d.dw, dws.data(), dws.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) return -1;
        d.t.rwords = d.rw;
        d.t.dwords = d.dw;
        it = g_two.emplace(key, d).first;
    }
    *out = it->second.t;
    return 0;
}

static cudaLaunchConfig_t cluster_cfg(const HKTwo& t, unsigned grid, cudaStream_t s, cudaLaunchAttribute* at) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kClusterThreads, 1, 1);
    cfg.dynamicSmemBytes = cluster_smem_bytes(t);
    cfg.stream = s;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)t.cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cfg;
}

static int set_cluster_attrs(const HKTwo& t) {
    if (cudaFuncSetAttribute(hk_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)cluster_smem_bytes(t)) != cudaSuccess)
        return -1;
    if (t.cs > 8 && cudaFuncSetAttribute(hk_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                        cudaSuccess)
        return -1;
    return 0;
}

int cluster_grid(const HKTwo& t, int sm_count) {
    if (set_cluster_attrs(t)) return t.cs;
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = cluster_cfg(t, (unsigned)(sm_count * 4 / t.cs * t.cs), 0, at);
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, hk_cluster_kernel, &cfg) != cudaSuccess || clusters < 1) {
        cudaGetLastError();
        clusters = std::max(1, sm_count / t.cs);
    }
    return clusters * t.cs;
}

template <typename KT, bool M8>
static void launch_stage_t(const EvalArgs& a, double* E, double* dp, uint8_t* bad, int blocks, cudaStream_t s) {
    size_t smem = cta_scratch_bytes(a.k, M8 ? 8 : a.m) + (((size_t)a.k * a.m * 2 + 15) & ~(size_t)15) + 32 * 4 * 4;
    cudaFuncSetAttribute(stage_kernel<KT, M8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    stage_kernel<KT, M8><<<blocks, 128, smem, s>>>(a, E, dp, bad);
}

int launch_stage(const EvalArgs& a, double* E, double* datap, uint8_t* bad, int blocks, bool m8, cudaStream_t s) {
    if (a.P == 0) return 0;
    blocks = (int)std::min<int64_t>(blocks, a.P);
    if (m8)
        launch_stage_t<uint16_t, true>(a, E, datap, bad, blocks, s);
    else if (a.key16)
        launch_stage_t<uint16_t, false>(a, E, datap, bad, blocks, s);
    else
        launch_stage_t<uint32_t, false>(a, E, datap, bad, blocks, s);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_hk_cluster(const double* E, int es, int64_t estride, int k, int64_t B, const HKTwo& t, int grid,
                      const double* add, const uint8_t* bad, double* out_total, double* out_pipe, cudaStream_t s) {
    if (B == 0) return 0;
    const int clusters = (int)std::min<int64_t>(grid / t.cs, B);
    if (set_cluster_attrs(t)) return -1;
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = cluster_cfg(t, (unsigned)(clusters * t.cs), s, at);
    if (cudaLaunchKernelEx(&cfg, hk_cluster_kernel, E, es, estride, k, B, t, add, bad, out_total, out_pipe) !=
        cudaSuccess)
        return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace hs
