// hs_eval8.cu -- K1 for the paper shape (d_pp = 8, d_dp = 8, N = 64, u16 keys):
// one warp prices four candidate layouts at a time (comm_cost,
// costmodel.py:217-229), lane = (candidate c = lane / 8, slot g = lane % 8).
//
//   load      : lane (c, g) reads group g of candidate c -- one 16-byte
//               vector (the quad's 512 bytes are one coalesced request);
//               validation (costmodel.py:58-72) by shuffles in the 8 lanes.
//   datap     : lane (c, g) forms the 8 numpy pairwise row sums of group g
//               and their max (datap_cost_group, costmodel.py:154-168); the
//               candidate's datap is the max over its 8 lanes.
//   matchings : the quad's 112 group pairs over the 32 lanes (3.5 rounds),
//               each the branch-free u16x2 subset DP (hs_match8_dp.cuh) ->
//               bottleneck rank -> exact double (costmodel.py:200-208).
//   Held-Karp : lane (c, u) computes every state ending at u from registers
//               holding E[u][.] (hs_hk8_gen.cuh); pipe = min over the lanes.
//
// Tables staged once per persistent CTA: the Held-Karp offset rows, the u16
// rank table and the DP table (odd row strides).  Outputs are bit-identical
// to the schedule-driven warp kernel (hs_kernels.cu) and to the reference.
//
// Occupancy: a Held-Karp block set (4 candidate blocks, 19.2 KB) is needed
// only during the Held-Karp phase (about a third of a quad's instructions),
// so the CTA's 20 warps share 9 sets from a free mask in shared memory: a
// warp computes its matchings with the edge values in registers, takes a
// free set, writes the edges, runs Held-Karp and hands the set back.  That
// more than doubles the resident warps that the 227 KB of shared memory
// allowed with one private set per warp.  20 warps at 96 registers:
// 3.08e8 evals/s against 2.98e8 at 16 warps / 128 registers and 3.05e8 at 24
// (measured; the host path's end-to-end rate is copy-pipeline-bound, within
// 1% either way).
#include <cstdlib>

#include "hs_hk8_gen.cuh"
#include "hs_match8_dp.cuh"
#include "hs_tma.cuh"
#include "hs_warp_eval.cuh"

namespace hs {

#ifndef HS_E8_WARPS
#define HS_E8_WARPS 20
#endif
constexpr int kE8Warps = HS_E8_WARPS;
#ifndef HS_E8_TMA
#define HS_E8_TMA 1
#endif
#if HS_E8_TMA
// rows staged by bulk copies (16-byte aligned destinations): strides of
// 132 and 36 words, 4 banks apart row to row
constexpr int kE8DS = 66;  // DP row stride (doubles)
constexpr int kE8RS = 72;  // rank row stride (u16)
#else
constexpr int kE8DS = 65;  // DP row stride (doubles): odd word count
constexpr int kE8RS = 66;  // rank row stride (u16): 33 words, odd
#endif
constexpr size_t kE8OffBytes = (size_t)8 * kHK8Words * 4 + 64;  // + layer-2 edge slots
constexpr size_t kE8RkBytes = ((size_t)64 * kE8RS * 2 + 15) & ~(size_t)15;
constexpr size_t kE8DpBytes = (size_t)64 * kE8DS * 8;
constexpr size_t kE8SetBytes = (size_t)4 * kHK8Block * 8;      // one Held-Karp block set
constexpr size_t kE8SmemCap = 232448;                          // sm_100 opt-in maximum per CTA

// Shared-memory layout: tables, per warp the quad's groups, the free mask,
// then as many Held-Karp block sets as fit (<= one per warp).
struct E8Layout {
    static constexpr size_t mem = (size_t)4 * 64 * 2;  // per warp: the quad's groups
    static constexpr size_t fixed = kE8OffBytes + kE8RkBytes + kE8DpBytes + kE8Warps * mem + 16;
    static constexpr int fit = (int)((kE8SmemCap - fixed) / kE8SetBytes);
    static constexpr int sets = fit < kE8Warps ? fit : kE8Warps;
    static constexpr size_t smem = fixed + (size_t)sets * kE8SetBytes;
    static_assert(sets >= 1, "no Held-Karp block set fits");
};

__device__ __forceinline__ double shfl_xor_d(double x, int m) {
    return __longlong_as_double(__shfl_xor_sync(0xffffffffu, __double_as_longlong(x), m));
}

__device__ __forceinline__ int i16(uint32_t w, int hi) { return hi ? (int)(int16_t)(w >> 16) : (int)(int16_t)(w & 0xFFFFu); }

// Tables staged once per persistent CTA: the Held-Karp offset rows and
// edge slots, the u16 rank table and the DP table (odd row strides / bulk
// copies), the free mask of the Held-Karp sets.
template <int kSets>
__device__ __forceinline__ void e8_stage(const EvalArgs& a, uint32_t* offs, uint16_t* rk, double* dp,
                                         unsigned* freemask, uint16_t* eslot) {
    const uint16_t* grk = reinterpret_cast<const uint16_t*>(a.rank);
#if HS_E8_TMA
    // tables by the bulk-copy (TMA) engine: warp 0 arms one mbarrier with the
    // byte count and issues 129 row copies (Held-Karp offsets, 64 rank rows,
    // 64 DP rows); the other threads set up the rest meanwhile
    __shared__ __align__(8) uint64_t tbar;
    if (threadIdx.x == 0) mbar_init(&tbar, 1);
    __syncthreads();
    if (threadIdx.x < 32) {
        constexpr uint32_t kOffs = 8 * kHK8Words * 4;
        if (threadIdx.x == 0) mbar_arrive_expect_tx(&tbar, kOffs + 64 * 128 + 64 * 512);
        __syncwarp();
        for (int i = threadIdx.x; i < 129; i += 32) {
            if (i < 64)
                bulk_g2s(rk + i * kE8RS, grk + i * 64, 128, &tbar);
            else if (i < 128)
                bulk_g2s(dp + (i - 64) * kE8DS, a.dp + (i - 64) * 64, 512, &tbar);
            else
                bulk_g2s(offs, kHK8Offs, kOffs, &tbar);
        }
    }
    if (threadIdx.x >= 32 && threadIdx.x < 60) eslot[threadIdx.x - 32] = kHK8Edge[threadIdx.x - 32];
    if (threadIdx.x == 64) *freemask = kSets == 32 ? 0xffffffffu : (1u << kSets) - 1u;
    mbar_wait(&tbar, 0);
    __syncthreads();
#else
    for (int i = threadIdx.x; i < 8 * kHK8Words; i += blockDim.x) offs[i] = kHK8Offs[i];
    if (threadIdx.x < 28) eslot[threadIdx.x] = kHK8Edge[threadIdx.x];
    if (threadIdx.x == 0) *freemask = kSets == 32 ? 0xffffffffu : (1u << kSets) - 1u;
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
        const int r = i >> 6, c = i & 63;
        rk[r * kE8RS + c] = grk[i];
        dp[r * kE8DS + c] = a.dp[i];
    }
    __syncthreads();
#endif
}

// Lane (c, g) of a candidate's 8 lanes: group g loaded as one 16-byte
// vector, validated (costmodel.py:58-72: in range, ascending, the 8 groups
// cover 0..63) by shuffles within the 8 lanes, and its data-parallel value
// (datap_cost_group, costmodel.py:154-168: numpy pairwise row sums, the 0.0
// diagonal in its slot, max over the rows); datap = max over the 8 lanes.
// A malformed candidate is priced as a valid stand-in (bad = true -> NaN).
struct E8Cand {
    uint4 gm;
    bool bad;
    double pg, datap;
};

__device__ __forceinline__ E8Cand e8_load(const uint4* gsrc, int64_t p, bool live, int g, const double* dp) {
    const uint4 ident = make_uint4((uint32_t)(8 * g) | (uint32_t)(8 * g + 1) << 16,
                                   (uint32_t)(8 * g + 2) | (uint32_t)(8 * g + 3) << 16,
                                   (uint32_t)(8 * g + 4) | (uint32_t)(8 * g + 5) << 16,
                                   (uint32_t)(8 * g + 6) | (uint32_t)(8 * g + 7) << 16);
    E8Cand r;
    r.gm = live ? __ldcg(gsrc + p * 8 + g) : ident;  // L2 path: a streamed batch lands while the kernel runs
    int mem[8];
    mem[0] = i16(r.gm.x, 0), mem[1] = i16(r.gm.x, 1), mem[2] = i16(r.gm.y, 0), mem[3] = i16(r.gm.y, 1);
    mem[4] = i16(r.gm.z, 0), mem[5] = i16(r.gm.z, 1), mem[6] = i16(r.gm.w, 0), mem[7] = i16(r.gm.w, 1);
    bool ok = true;
    uint64_t cover = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        ok = ok && mem[i] >= 0 && mem[i] < 64 && (i == 0 || mem[i - 1] < mem[i]);
        cover |= 1ull << (mem[i] & 63);
    }
    uint32_t cl = (uint32_t)cover, ch = (uint32_t)(cover >> 32), okb = ok;
#pragma unroll
    for (int m = 1; m < 8; m <<= 1) {
        cl |= __shfl_xor_sync(0xffffffffu, cl, m);
        ch |= __shfl_xor_sync(0xffffffffu, ch, m);
        okb &= __shfl_xor_sync(0xffffffffu, okb, m);
    }
    r.bad = live && !(okb && cl == 0xffffffffu && ch == 0xffffffffu);
    if (r.bad) {  // price a valid stand-in, report NaN
        r.gm = ident;
#pragma unroll
        for (int i = 0; i < 8; i++) mem[i] = 8 * g + i;
    }
    double pg = 0.0;
#pragma unroll
    for (int rr = 0; rr < 8; rr++) {
        const double* row = dp + mem[rr] * kE8DS;
        const double s = ((row[mem[0]] + row[mem[1]]) + (row[mem[2]] + row[mem[3]])) +
                         ((row[mem[4]] + row[mem[5]]) + (row[mem[6]] + row[mem[7]]));
        pg = rr == 0 ? s : dmax(pg, s);
    }
    r.pg = pg;
    double datap = pg;
#pragma unroll
    for (int m = 1; m < 8; m <<= 1) datap = dmax(datap, shfl_xor_d(datap, m));
    r.datap = datap;
    return r;
}

// bottleneck rank of one group pair (job: A-group row | B-group row << 8 in
// the warp's group buffer, 16-byte rows): the branch-free u16x2 subset DP
// (hs_match8_dp.cuh, combinatorics.py:86-131 / costmodel.py:200-208)
__device__ __forceinline__ uint32_t e8_match(const int16_t* memw, const uint16_t* rk, uint32_t jb) {
    const uint4 A4 = reinterpret_cast<const uint4*>(memw)[jb & 0xFFu];
    const uint4 B4 = reinterpret_cast<const uint4*>(memw)[(jb >> 8) & 0xFFu];
    const uint32_t Aw[4] = {A4.x, A4.y, A4.z, A4.w};
    const uint32_t Bw[4] = {B4.x, B4.y, B4.z, B4.w};
    int b[8];
#pragma unroll
    for (int k = 0; k < 8; k++) b[k] = i16(Bw[k >> 1], k & 1);
    // both half orders packed on the FMA pipe (IMAD): the DP is ALU-bound.
    // (Moving 3/8 of the maxima to the FMA pipe as HFMA2.RELU + HADD2 on fp16
    // patterns of the ranks balanced the pipes but issued 191 more
    // instructions per matching: 2.92e8 vs 2.98e8 evals/s, measured, removed.)
    return match8_dp_m<1>([&](int r, uint32_t(&kn)[4], uint32_t(&ks)[4]) {
        const uint16_t* row = rk + i16(Aw[r >> 1], r & 1) * kE8RS;
#pragma unroll
        for (int qq = 0; qq < 4; qq++) {
            const uint32_t lo = row[b[qq]], hi = row[b[qq + 4]];
            uint32_t w, x;
            asm("mad.lo.u32 %0, %1, 65536, %2;" : "=r"(w) : "r"(hi), "r"(lo));
            asm("mad.lo.u32 %0, %1, 65536, %2;" : "=r"(x) : "r"(lo), "r"(hi));
            kn[qq] = w;
            ks[qq] = x;
        }
    });
}

// a free Held-Karp block set (lane 0 claims it from the CTA's mask)
template <int kSets>
__device__ __forceinline__ int e8_take(unsigned* freemask, int lane) {
    HS_JITTER();
    int set = 0;
    if (lane == 0) {
        unsigned old = *reinterpret_cast<volatile unsigned*>(freemask);
        for (;;) {
            if (old) {
                set = __ffs(old) - 1;
                const unsigned prev = atomicAnd(freemask, ~(1u << set));
                if (prev & (1u << set)) break;
                old = prev & ~(1u << set);
            } else {
                __nanosleep(32);
                old = *reinterpret_cast<volatile unsigned*>(freemask);
            }
        }
        __threadfence_block();
    }
    return __shfl_sync(0xffffffffu, set, 0);
}

__device__ __forceinline__ void e8_release(unsigned* freemask, int set, int lane) {
    HS_JITTER();
    __syncwarp();  // every lane is done with the set
    if (lane == 0) {
        __threadfence_block();
        atomicOr(freemask, 1u << set);
    }
}

__device__ __forceinline__ void e8_out(const EvalArgs& a, int64_t p, bool live, int g, bool bad, double datap,
                                       double pipe, double pg, bool per_group) {
    if (!live) return;
    if (g == 0) {
        if (bad) {
            const double nan = __longlong_as_double(0x7ff8000000000000LL);
            a.total[p] = nan;
            if (a.datap) a.datap[p] = nan;
            if (a.pipe) a.pipe[p] = nan;
            atomicAdd(a.invalid, 1);
        } else {
            a.total[p] = datap + pipe;
            if (a.datap) a.datap[p] = datap;
            if (a.pipe) a.pipe[p] = pipe;
        }
    }
    if (per_group && !bad) a.per_group[p * 8 + g] = pg;
}

// kC = candidates per warp: 4 (lane (c, g)) or 1 (latency mode for small
// batches: every 8-lane group mirrors candidate 0's groups, its 28
// matchings take one round, only lanes 0..7's Held-Karp result is used).
template <bool kPerGroup, int kC>
__global__ void __launch_bounds__(32 * kE8Warps, 1) eval8_kernel(EvalArgs a) {
    using L = E8Layout;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* offs = reinterpret_cast<uint32_t*>(smem);
    uint16_t* rk = reinterpret_cast<uint16_t*>(smem + kE8OffBytes);
    double* dp = reinterpret_cast<double*>(smem + kE8OffBytes + kE8RkBytes);
    unsigned char* memsm = smem + kE8OffBytes + kE8RkBytes + kE8DpBytes;
    unsigned* freemask = reinterpret_cast<unsigned*>(memsm + kE8Warps * L::mem);
    char* sets = reinterpret_cast<char*>(memsm + kE8Warps * L::mem + 16);
    uint16_t* eslot = reinterpret_cast<uint16_t*>(offs + 8 * kHK8Words);
    e8_stage<L::sets>(a, offs, rk, dp, freemask, eslot);

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int c = lane >> 3, g = lane & 7;
    int16_t* memw = reinterpret_cast<int16_t*>(memsm + (size_t)wid * L::mem);
    const uint4* t4 = reinterpret_cast<const uint4*>(offs + g * kHK8Words);
    const uint4* gsrc = reinterpret_cast<const uint4*>(a.groups);

    // this lane's share of the quad's 112 group pairs, t = lane + 32 i (loop
    // invariant): A-group row | B-group row << 8 | edge slot << 16 (0 = none)
    uint32_t job[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int t = lane + 32 * i;
        job[i] = 0;
        if (t < 28 * kC) {
            const int cc = t / 28, pi = t - cc * 28;
            int j, j2;
            decode_pair(pi, 8, j, j2);
            job[i] = (uint32_t)(cc * 8 + j) | (uint32_t)(cc * 8 + j2) << 8 |
                     (uint32_t)(cc * kHK8Block + eslot[pi]) << 16;
        }
    }

    // latency mode: consecutive candidates on different CTAs (SMs) first
    const int64_t q0 = kC == 4 ? (int64_t)blockIdx.x * W + wid : (int64_t)wid * gridDim.x + blockIdx.x;
    int64_t chunk = -1, done = 0;  // streamed batch: current chunk, quads finished in it
    auto chunk_of = [&](int64_t q) { return q * kC < a.c0 ? 0 : 1 + (q * kC - a.c0) / a.c; };
    auto report = [&]() {  // this warp is past `chunk`
        HS_JITTER();
        if (chunk >= 0 && lane == 0) {
            __threadfence();  // the chunk's outputs before its count
            atomicAdd(a.finished + chunk, (uint32_t)done);
        }
    };
    for (int64_t q = q0; q * kC < a.P; q += (int64_t)gridDim.x * W) {
        if (a.arrived) {
            const int64_t ci = chunk_of(q);
            if (ci != chunk) {
                report();
                chunk = ci;
                done = 0;
                if (lane == 0) {
                    uint32_t v;
                    const long long t0 = clock64();
                    for (;;) {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.arrived + ci) : "memory");
                        if ((int32_t)(v - a.epoch) >= 0) break;
                        if (clock64() - t0 > 40000000000LL) __trap();  // ~20 s: a chunk that never arrives fails the launch
                        __nanosleep(256);
                    }
                }
                __syncwarp();
                HS_JITTER();
            }
            done++;
        }
        const int64_t p = q * kC + (kC == 4 ? c : 0);
        const bool live = (kC == 4 || c == 0) && p < a.P;
        const E8Cand cd = e8_load(gsrc, p, live, g, dp);
        reinterpret_cast<uint4*>(memw)[lane] = cd.gm;
        __syncwarp();
        // pipeline edges: 4 x 28 group pairs over 32 lanes (t = lane + 32 i),
        // kept in registers until the warp holds a Held-Karp set
        double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll 1
        for (int i = 0; i < 4; i++) {
            const uint32_t jb = i == 0 ? job[0] : i == 1 ? job[1] : i == 2 ? job[2] : job[3];
            if (jb) {
                const double v = __ldg(a.vals + e8_match(memw, rk, jb));
                e0 = i == 0 ? v : e0;
                e1 = i == 1 ? v : e1;
                e2 = i == 2 ? v : e2;
                e3 = i == 3 ? v : e3;
            }
        }
        const double e[4] = {e0, e1, e2, e3};
        const int set = e8_take<L::sets>(freemask, lane);
        char* blocks = sets + (size_t)set * kE8SetBytes;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            if (job[i]) {
                double* dst = reinterpret_cast<double*>(blocks) + (job[i] >> 16);
                dst[0] = e[i];  // h[{j, j2}][j] and h[{j, j2}][j2]
                dst[kHK8EdgeStride] = e[i];
            }
        }
        HS_JITTER();
        __syncwarp();
        double pipe = hk8_lane(blocks + (size_t)c * kHK8Block * 8, t4);
        e8_release(freemask, set, lane);
#pragma unroll
        for (int m = 1; m < 8; m <<= 1) pipe = dmin(pipe, shfl_xor_d(pipe, m));
        e8_out(a, p, live, g, cd.bad, cd.datap, pipe, cd.pg, kPerGroup);
        __syncwarp();
    }
    if (a.arrived) report();
}

bool eval8_applicable(const EvalArgs& a, size_t smem_optin) {
    // 16-byte group loads: the layout array must be 16-byte aligned (views at
    // odd offsets take the schedule-driven kernel)
    return a.k == 8 && a.m == 8 && a.n == 64 && a.key16 && !a.order && E8Layout::smem <= smem_optin &&
           ((uintptr_t)a.groups & 15) == 0;
}

template <int kC>
static void launch_eval8_c(const EvalArgs& a, int blocks, cudaStream_t s) {
    constexpr int sm = (int)E8Layout::smem;
    if (a.per_group) {
        cudaFuncSetAttribute(eval8_kernel<true, kC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        eval8_kernel<true, kC><<<blocks, 32 * kE8Warps, sm, s>>>(a);
    } else {
        cudaFuncSetAttribute(eval8_kernel<false, kC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        eval8_kernel<false, kC><<<blocks, 32 * kE8Warps, sm, s>>>(a);
    }
}

// candidates one full wave of the throughput kernel prices (four per warp)
int64_t eval8_wave(int sm_count) { return (int64_t)sm_count * kE8Warps * 4; }

int launch_eval8(const EvalArgs& a, int sm_count, cudaStream_t s) {
    if (a.P == 0) return 0;
    if (a.arrived) {  // streamed batch: the throughput kernel, whatever P
        launch_eval8_c<4>(a, (int)std::min<int64_t>(sm_count, (a.P + 3) / 4), s);
        return cudaGetLastError() == cudaSuccess ? 0 : -1;
    }
    // small batches: one candidate per warp when the batch does not fill
    // the GPU's warps (a warp's latency is the floor), else four.  (Eight per
    // warp -- seven full matching rounds instead of 3.5 per quad -- cut the
    // instructions 6% but the larger loop body missed the instruction cache
    // more: 2.69e8 vs 2.98e8 evals/s, measured and removed.)
    static const int64_t kLatencyMax = getenv("HS_E8_LATENCY_MAX") ? atoll(getenv("HS_E8_LATENCY_MAX")) : -1;
    const int64_t lat_max = kLatencyMax >= 0 ? kLatencyMax : (int64_t)sm_count * kE8Warps;
    if (a.P <= lat_max) {
        launch_eval8_c<1>(a, (int)std::min<int64_t>(sm_count, a.P), s);
    } else {
        const int64_t quads = (a.P + 3) / 4;
        launch_eval8_c<4>(a, (int)std::min<int64_t>(sm_count, quads), s);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace hs
