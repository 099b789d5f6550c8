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
// so the CTA's 16 warps share kE8Sets < 16 sets from a free mask in shared
// memory: a warp computes its matchings with the edge values in registers,
// takes a free set, writes the edges, runs Held-Karp and hands the set back.
// That doubles the resident warps (16 per SM at <= 128 registers) that the
// 227 KB of shared memory allowed with one private set per warp.
#include <cstdlib>

#include "hs_hk8_gen.cuh"
#include "hs_match8_dp.cuh"
#include "hs_tma.cuh"
#include "hs_warp_eval.cuh"

namespace hs {

#ifndef HS_E8_WARPS
#define HS_E8_WARPS 16
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
constexpr size_t kE8MemBytes = (size_t)4 * 64 * 2;             // per warp: the quad's groups
constexpr size_t kE8SetBytes = (size_t)4 * kHK8Block * 8;      // one Held-Karp block set
constexpr size_t kE8Fixed = kE8OffBytes + kE8RkBytes + kE8DpBytes + kE8Warps * kE8MemBytes + 16;
constexpr size_t kE8SmemCap = 232448;                          // sm_100 opt-in maximum per CTA
constexpr int kE8Sets = (int)((kE8SmemCap - kE8Fixed) / kE8SetBytes) < kE8Warps
                            ? (int)((kE8SmemCap - kE8Fixed) / kE8SetBytes) : kE8Warps;
constexpr size_t kE8Smem = kE8Fixed + (size_t)kE8Sets * kE8SetBytes;
static_assert(kE8Sets >= 1, "no Held-Karp block set fits");

__device__ __forceinline__ double shfl_xor_d(double x, int m) {
    return __longlong_as_double(__shfl_xor_sync(0xffffffffu, __double_as_longlong(x), m));
}

__device__ __forceinline__ int i16(uint32_t w, int hi) { return hi ? (int)(int16_t)(w >> 16) : (int)(int16_t)(w & 0xFFFFu); }

// kC = candidates per warp: 4 (throughput: lane (c, g)) or 1 (latency mode
// for small batches: every 8-lane group mirrors candidate 0's groups, its
// 28 matchings take one round, only lanes 0..7's Held-Karp result is used).
template <bool kPerGroup, int kC>
__global__ void __launch_bounds__(32 * kE8Warps, 1) eval8_kernel(EvalArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* offs = reinterpret_cast<uint32_t*>(smem);
    uint16_t* rk = reinterpret_cast<uint16_t*>(smem + kE8OffBytes);
    double* dp = reinterpret_cast<double*>(smem + kE8OffBytes + kE8RkBytes);
    unsigned char* memsm = smem + kE8OffBytes + kE8RkBytes + kE8DpBytes;
    unsigned* freemask = reinterpret_cast<unsigned*>(memsm + kE8Warps * kE8MemBytes);
    char* sets = reinterpret_cast<char*>(memsm + kE8Warps * kE8MemBytes + 16);
    const uint16_t* grk = reinterpret_cast<const uint16_t*>(a.rank);
    uint16_t* eslot = reinterpret_cast<uint16_t*>(offs + 8 * kHK8Words);
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
    if (threadIdx.x == 64) *freemask = kE8Sets == 32 ? 0xffffffffu : (1u << kE8Sets) - 1u;
    mbar_wait(&tbar, 0);
    __syncthreads();
#else
    for (int i = threadIdx.x; i < 8 * kHK8Words; i += blockDim.x) offs[i] = kHK8Offs[i];
    if (threadIdx.x < 28) eslot[threadIdx.x] = kHK8Edge[threadIdx.x];
    if (threadIdx.x == 0) *freemask = kE8Sets == 32 ? 0xffffffffu : (1u << kE8Sets) - 1u;
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
        const int r = i >> 6, c = i & 63;
        rk[r * kE8RS + c] = grk[i];
        dp[r * kE8DS + c] = a.dp[i];
    }
    __syncthreads();
#endif

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
    const int c = lane >> 3, g = lane & 7;
    int16_t* memw = reinterpret_cast<int16_t*>(memsm + (size_t)wid * kE8MemBytes);
    const uint4* t4 = reinterpret_cast<const uint4*>(offs + g * kHK8Words);
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    const uint4* gsrc = reinterpret_cast<const uint4*>(a.groups);
    const uint4 ident = make_uint4((uint32_t)(8 * g) | (uint32_t)(8 * g + 1) << 16,
                                   (uint32_t)(8 * g + 2) | (uint32_t)(8 * g + 3) << 16,
                                   (uint32_t)(8 * g + 4) | (uint32_t)(8 * g + 5) << 16,
                                   (uint32_t)(8 * g + 6) | (uint32_t)(8 * g + 7) << 16);

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
    for (int64_t q = q0; q * kC < a.P; q += (int64_t)gridDim.x * W) {
        const int64_t p = q * kC + (kC == 4 ? c : 0);
        const bool live = (kC == 4 || c == 0) && p < a.P;
        uint4 gm = live ? __ldg(gsrc + p * 8 + g) : ident;
        // validation: in range, ascending, the candidate's 8 groups cover 0..63
        int mem[8];
        mem[0] = i16(gm.x, 0), mem[1] = i16(gm.x, 1), mem[2] = i16(gm.y, 0), mem[3] = i16(gm.y, 1);
        mem[4] = i16(gm.z, 0), mem[5] = i16(gm.z, 1), mem[6] = i16(gm.w, 0), mem[7] = i16(gm.w, 1);
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
        const bool bad = live && !(okb && cl == 0xffffffffu && ch == 0xffffffffu);
        if (bad) {  // price a valid stand-in, report NaN
            gm = ident;
#pragma unroll
            for (int i = 0; i < 8; i++) mem[i] = 8 * g + i;
        }
        reinterpret_cast<uint4*>(memw)[lane] = gm;
        // data-parallel level: numpy pairwise row sums (the 0.0 diagonal in
        // its slot), max over the group's rows
        double pg = 0.0;
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const double* row = dp + mem[r] * kE8DS;
            const double s = ((row[mem[0]] + row[mem[1]]) + (row[mem[2]] + row[mem[3]])) +
                             ((row[mem[4]] + row[mem[5]]) + (row[mem[6]] + row[mem[7]]));
            pg = r == 0 ? s : dmax(pg, s);
        }
        double datap = pg;
#pragma unroll
        for (int m = 1; m < 8; m <<= 1) datap = dmax(datap, shfl_xor_d(datap, m));
        __syncwarp();
        // pipeline edges: 4 x 28 group pairs over 32 lanes (t = lane + 32 i),
        // kept in registers until the warp holds a Held-Karp set
        double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
#pragma unroll 1
        for (int i = 0; i < 4; i++) {
            const uint32_t jb = i == 0 ? job[0] : i == 1 ? job[1] : i == 2 ? job[2] : job[3];
            if (jb) {
                const uint4 A4 = reinterpret_cast<const uint4*>(memw)[jb & 0xFFu];
                const uint4 B4 = reinterpret_cast<const uint4*>(memw)[(jb >> 8) & 0xFFu];
                const uint32_t Aw[4] = {A4.x, A4.y, A4.z, A4.w};
                const uint32_t Bw[4] = {B4.x, B4.y, B4.z, B4.w};
                int b[8];
#pragma unroll
                for (int k = 0; k < 8; k++) b[k] = i16(Bw[k >> 1], k & 1);
                const uint32_t L = match8_dp([&](int r, uint32_t(&kn)[4]) {
                    const uint16_t* row = rk + i16(Aw[r >> 1], r & 1) * kE8RS;
#pragma unroll
                    for (int qq = 0; qq < 4; qq++) {  // lo + hi * 65536 on the FMA pipe (IMAD), not PRMT
                        uint32_t w;
                        asm("mad.lo.u32 %0, %1, 65536, %2;" : "=r"(w) : "r"((uint32_t)row[b[qq + 4]]),
                            "r"((uint32_t)row[b[qq]]));
                        kn[qq] = w;
                    }
                });
                const double v = __ldg(a.vals + L);
                e0 = i == 0 ? v : e0;
                e1 = i == 1 ? v : e1;
                e2 = i == 2 ? v : e2;
                e3 = i == 3 ? v : e3;
            }
        }
        const double e[4] = {e0, e1, e2, e3};
        // take a free Held-Karp set
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
        set = __shfl_sync(0xffffffffu, set, 0);
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
        HS_JITTER();
        __syncwarp();  // every lane is done with the set
        if (lane == 0) {
            __threadfence_block();
            atomicOr(freemask, 1u << set);
        }
#pragma unroll
        for (int m = 1; m < 8; m <<= 1) pipe = dmin(pipe, shfl_xor_d(pipe, m));
        if (live) {
            if (g == 0) {
                if (bad) {
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
            if (kPerGroup && !bad) a.per_group[p * 8 + g] = pg;
        }
        __syncwarp();
    }
}

bool eval8_applicable(const EvalArgs& a, size_t smem_optin) {
    // 16-byte group loads: the layout array must be 16-byte aligned (views at
    // odd offsets take the schedule-driven kernel)
    return a.k == 8 && a.m == 8 && a.n == 64 && a.key16 && !a.order && kE8Smem <= smem_optin &&
           ((uintptr_t)a.groups & 15) == 0;
}

template <int kC>
static void launch_eval8_c(const EvalArgs& a, int blocks, cudaStream_t s) {
    if (a.per_group) {
        cudaFuncSetAttribute(eval8_kernel<true, kC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kE8Smem);
        eval8_kernel<true, kC><<<blocks, 32 * kE8Warps, kE8Smem, s>>>(a);
    } else {
        cudaFuncSetAttribute(eval8_kernel<false, kC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kE8Smem);
        eval8_kernel<false, kC><<<blocks, 32 * kE8Warps, kE8Smem, s>>>(a);
    }
}

int launch_eval8(const EvalArgs& a, int sm_count, cudaStream_t s) {
    if (a.P == 0) return 0;
    // small batches: one candidate per warp when the batch does not fill
    // the GPU's warps (a warp's latency is the floor), else four
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
