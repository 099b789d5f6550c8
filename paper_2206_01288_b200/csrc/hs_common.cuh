// hs_common.cuh -- shared device helpers for the sm_100a hetsched kernels.
//
// Float-order rules (restated from the reference):
//   * numpy pairwise summation for contiguous reductions
//     (costmodel.py:168, scheduler.py:207-208,438-443,567);
//   * sequential summation for w[:, grp].mean(axis=1) (scheduler.py:283,363),
//     whose fancy-index result is F-contiguous;
//   * no FMA contraction anywhere (the library is built with -fmad=false).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hs {

constexpr int kWarp = 32;
constexpr double kInf = __builtin_huge_val();

// Race stress (compute-sanitizer is unavailable on the GPU pool): a build
// with -DHS_RACE_JITTER sleeps a pseudo-random 0..2 us per thread at the
// cross-warp / cross-CTA hand-off points (HS_JITTER()), so a missing
// barrier or fence shows up as a parity failure against the oracle
// (scripts/race_stress.sh).  Compiles to nothing otherwise.
#ifdef HS_RACE_JITTER
__device__ __forceinline__ void hs_jitter() {
    unsigned x = (unsigned)clock() ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu);
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    __nanosleep(x & 2047u);
}
#define HS_JITTER() ::hs::hs_jitter()
#else
#define HS_JITTER() \
    do {            \
    } while (0)
#endif

__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }

// numpy pairwise_sum for n <= 128 over values produced by get(i), i < n.
// (n < 8: sequential from 0.0; else 8 strided accumulators, fixed tree,
// then the tail sequentially.)  Larger n recurses like numpy.
template <typename Get>
__device__ __forceinline__ double pairwise_sum(int n, Get get) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; i++) r += get(i);
        return r;
    }
    double r0 = get(0), r1 = get(1), r2 = get(2), r3 = get(3);
    double r4 = get(4), r5 = get(5), r6 = get(6), r7 = get(7);
    int i = 8;
    int full = n - (n % 8);
    for (; i < full; i += 8) {
        r0 += get(i + 0);
        r1 += get(i + 1);
        r2 += get(i + 2);
        r3 += get(i + 3);
        r4 += get(i + 4);
        r5 += get(i + 5);
        r6 += get(i + 6);
        r7 += get(i + 7);
    }
    double res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    for (; i < n; i++) res += get(i);
    return res;
}

}  // namespace hs
