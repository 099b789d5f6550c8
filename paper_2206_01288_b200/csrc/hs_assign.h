// hs_assign.h -- host interface of the fixed-layout kernels (hs_assign.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hetsched_b200.h"
#include "hs_internal.h"

namespace hs {

struct MaterializeArgs {
    int n, k, m, nvals;
    bool key16;
    const double* dp;
    const void* rank;
    const double* vals;
    HKTables hk;
    const int16_t* groups;  // [B][k][m]
    int64_t B;
    int16_t* grid;   // [B][m][k]
    int8_t* order;   // [B][k]
};

int launch_materialize(const MaterializeArgs& a, int sm_count, cudaStream_t s);
int launch_evaluate(int n, int k, int m, const double* dp, const double* pp, const int16_t* grids, int64_t B,
                    double* out3, double* per_col, int sm_count, cudaStream_t s);
int launch_random_assign(int n, int k, int m, int B, hs_pcg64* rngs, int16_t* scratch, int16_t* grids, int8_t* orders,
                         cudaStream_t s);
int launch_bottleneck_match(const double* w, int m, int64_t B, double* value, int8_t* pairs, cudaStream_t s);
int launch_datap_group(const double* lat, const double* bw, int m, int64_t G, double ddp, double dp_num, double* out,
                       cudaStream_t s);

}  // namespace hs
