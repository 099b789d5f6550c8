// hs_brute.cu -- exhaustive k! oracles of combinatorics.py on sm_100a.
//
//   brute_force_bottleneck_matching (combinatorics.py:192-207): the first
//     permutation (itertools order = lexicographic) whose largest selected
//     entry w[r][perm[r]] is strictly smallest.
//   brute_force_open_loop_tsp (combinatorics.py:345-361): the first
//     permutation whose right-to-left path_cost (:68-79) is strictly
//     smallest.
//
// Every thread unranks permutations (Lehmer code, lexicographic rank) over a
// grid-stride range.  Pass 1 takes the minimum value with a u64 atomicMin on
// the IEEE bits (all values are finite and >= 0, so the bit order is the
// numeric order); pass 2 takes the smallest rank attaining it, i.e. the
// permutation the reference's strict `<` scan keeps.
#include <cstdint>

#include "../../include/hetsched_b200.h"
#include "hs_instance.h"

namespace hs {

constexpr int kMaxBrute = 10;

__device__ __forceinline__ void unrank_perm(int k, uint64_t rank, int8_t* perm) {
    // factorial digits, most significant first
    uint64_t fact[kMaxBrute + 1];
    fact[0] = 1;
    for (int i = 1; i <= k; i++) fact[i] = fact[i - 1] * i;
    uint32_t avail = (1u << k) - 1;
    for (int i = 0; i < k; i++) {
        uint64_t f = fact[k - 1 - i];
        int d = (int)(rank / f);
        rank -= (uint64_t)d * f;
        // d-th smallest still available value
        uint32_t a = avail;
        for (int j = 0; j < d; j++) a &= a - 1;
        int v = __ffs(a) - 1;
        perm[i] = (int8_t)v;
        avail &= ~(1u << v);
    }
}

__device__ __forceinline__ double perm_value(const double* w, int k, int kind, const int8_t* perm) {
    if (kind == 0) {
        double mx = w[perm[0]];
        for (int r = 1; r < k; r++) {
            double x = w[r * k + perm[r]];
            mx = x > mx ? x : mx;
        }
        return mx;
    }
    double total = 0.0;
    for (int i = k - 2; i >= 0; i--) total = w[perm[i] * k + perm[i + 1]] + total;
    return total;
}

__global__ void brute_min_kernel(const double* __restrict__ w, int k, int kind, uint64_t count,
                                 unsigned long long* __restrict__ best_bits) {
    int8_t perm[kMaxBrute];
    unsigned long long mine = ~0ull;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < count; r += (uint64_t)gridDim.x * blockDim.x) {
        unrank_perm(k, r, perm);
        unsigned long long b = (unsigned long long)__double_as_longlong(perm_value(w, k, kind, perm));
        mine = b < mine ? b : mine;
    }
    for (int o = 16; o; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, mine, o);
        mine = t < mine ? t : mine;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(best_bits, mine);
}

__global__ void brute_rank_kernel(const double* __restrict__ w, int k, int kind, uint64_t count,
                                  const unsigned long long* __restrict__ best_bits,
                                  unsigned long long* __restrict__ best_rank) {
    int8_t perm[kMaxBrute];
    const unsigned long long target = *best_bits;
    unsigned long long mine = ~0ull;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < count; r += (uint64_t)gridDim.x * blockDim.x) {
        if (r >= mine) break;
        unrank_perm(k, r, perm);
        if ((unsigned long long)__double_as_longlong(perm_value(w, k, kind, perm)) == target) mine = r;
    }
    for (int o = 16; o; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, mine, o);
        mine = t < mine ? t : mine;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(best_rank, mine);
}

__global__ void brute_out_kernel(int k, const unsigned long long* __restrict__ best_bits,
                                 const unsigned long long* __restrict__ best_rank, double* __restrict__ value,
                                 int8_t* __restrict__ perm) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        *value = __longlong_as_double((long long)*best_bits);
        unrank_perm(k, *best_rank, perm);
    }
}

}  // namespace hs

extern "C" {

int hs_brute_force(const double* w, int k, int kind, double* value, int8_t* perm, int device, void* stream) {
    if (k < 1 || k > hs::kMaxBrute) return hsx::fail(-3, "brute force: k must be in 1..10");
    if (kind != 0 && kind != 1) return hsx::fail(-2, "brute force: kind must be 0 (matching) or 1 (path)");
    if (!w || !value || !perm) return hsx::fail(-2, "null argument");
    hsx::DeviceGuard dg(device);
    cudaStream_t s = (cudaStream_t)stream;
    uint64_t count = 1;
    for (int i = 2; i <= k; i++) count *= i;
    unsigned long long* d = nullptr;
    CK(cudaMallocAsync((void**)&d, 16, s), "cudaMallocAsync");
    CK(cudaMemsetAsync(d, 0xff, 16, s), "cudaMemsetAsync");
    int threads = 256;
    int blocks = (int)((count + threads - 1) / threads);
    if (blocks > 148 * 16) blocks = 148 * 16;
    hs::brute_min_kernel<<<blocks, threads, 0, s>>>(w, k, kind, count, d);
    hs::brute_rank_kernel<<<blocks, threads, 0, s>>>(w, k, kind, count, d, d + 1);
    hs::brute_out_kernel<<<1, 32, 0, s>>>(k, d, d + 1, value, perm);
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(d, s);
    if (e != cudaSuccess) return hsx::fail(-1, "brute force launch", e);
    return 0;
}

}  // extern "C"
