// hs_enum.cu -- exhaustive balanced-partition enumeration for brute_force_best
// (costmodel.py:232-266) on the GPU.
//
// _balanced_partitions anchors each group at the smallest unplaced device and
// walks the partner combinations in lexicographic order, so the enumeration
// order is the lexicographic order of canonical keys.  unrank_kernel maps an
// index straight to that partition: with f(s) = #partitions of s devices into
// groups of m, index = q * f(s - m) + rest, q ranking the (m-1)-subset of
// partners among the s-1 remaining devices (combinatorial number system).
#include <algorithm>
#include <cstdint>

#include "../../include/hetsched_b200.h"

namespace hs {

__host__ __device__ inline double binom_d(int n, int r) {
    if (r < 0 || r > n) return 0.0;
    double c = 1.0;
    for (int i = 1; i <= r; i++) c = c * (n - r + i) / i;
    return c;
}

__host__ __device__ inline int64_t binom(int n, int r) { return (int64_t)(binom_d(n, r) + 0.5); }

// partitions of s devices into groups of m
__host__ __device__ inline int64_t count_parts(int s, int m) {
    int64_t c = 1;
    while (s > 0) {
        c *= binom(s - 1, m - 1);
        s -= m;
    }
    return c;
}

__global__ void unrank_kernel(int n, int k, int m, int64_t start, int64_t count, int16_t* __restrict__ out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= count) return;
    int64_t idx = start + t;
    int16_t rem[64];
    for (int i = 0; i < n; i++) rem[i] = (int16_t)i;
    int s = n;
    int16_t* o = out + t * n;
    for (int g = 0; g < k; g++) {
        int64_t tail = count_parts(s - m, m);
        int64_t q = idx / tail;
        idx -= q * tail;
        o[g * m] = rem[0];
        // q-th (m-1)-combination of rem[1..s-1] in lexicographic order
        int pos = 1, chosen = 0;
        int16_t pick[64];
        int npick = 0;
        while (chosen < m - 1) {
            int64_t with = binom(s - pos - 1, m - 2 - chosen);  // combos that take rem[pos]
            if (q < with) {
                pick[npick++] = (int16_t)pos;
                chosen++;
            } else {
                q -= with;
            }
            pos++;
        }
        for (int i = 0; i < m - 1; i++) o[g * m + 1 + i] = rem[pick[i]];
        // drop rem[0] and the picked positions
        int w = 0, pi = 0;
        for (int i = 1; i < s; i++) {
            if (pi < npick && pick[pi] == i) {
                pi++;
                continue;
            }
            rem[w++] = rem[i];
        }
        s -= m;
    }
}

}  // namespace hs

extern "C" {

int64_t hs_count_partitions(int n, int d_dp) {
    if (d_dp < 1 || n % d_dp) return -1;
    return hs::count_parts(n, d_dp);
}

int hs_unrank_partitions(int n, int d_pp, int d_dp, int64_t start, int64_t count, int16_t* out, void* stream) {
    if (n != d_pp * d_dp || n > 64 || count < 0) return -2;
    if (count == 0) return 0;
    hs::unrank_kernel<<<(unsigned)((count + 127) / 128), 128, 0, (cudaStream_t)stream>>>(n, d_pp, d_dp, start, count,
                                                                                      out);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // extern "C"
