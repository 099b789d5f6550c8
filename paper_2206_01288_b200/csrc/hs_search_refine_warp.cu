// hs_search_refine_warp.cu -- instantiates one family of K2/K3 kernel variants (see
// hs_search_impl.cuh); split out so nvcc compiles the variants in parallel.
#include "hs_search_impl.cuh"

namespace hs {
template int launch_refine_c<false>(const RefineArgs&, const SearchPlan&, int, bool, cudaStream_t);
}  // namespace hs
