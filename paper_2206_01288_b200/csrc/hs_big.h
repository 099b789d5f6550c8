// hs_big.h -- host interface of the 9 <= d_pp <= 16 (CTA per candidate) path.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hs_internal.h"

namespace hs {

size_t hk_big_size(int k);
int big_blocks(int sm_count, int k);
int launch_eval_cta(const EvalArgs& a, const HKBig& t, double* scratch, int blocks, bool m8, cudaStream_t s);
int launch_path_cta(const double* w, int k, int64_t B, const HKBig& t, double* scratch, int blocks, double* total,
                    int8_t* order, cudaStream_t s);

int launch_path_heuristic(const double* w, int k, int64_t B, double* total, int8_t* order, int8_t* scratch,
                          cudaStream_t s);
int launch_eval_heur(const EvalArgs& a, double* Ebuf, int blocks, cudaStream_t s);

}  // namespace hs
