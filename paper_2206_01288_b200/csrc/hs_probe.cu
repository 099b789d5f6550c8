// hs_probe.cu -- measured shared-memory bandwidth of this GPU: the
// denominator of bench.py's on-chip roofline (MEASURED_PEAKS.json has no
// shared-memory figure).  Every warp streams conflict-free 16-byte LDS
// (4 wavefronts of 128 B per warp instruction) over a 32 KB buffer; the
// result is bytes delivered per second over the whole GPU.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/hetsched_b200.h"
#include "hs_instance.h"

namespace {

constexpr int kProbeThreads = 1024;
constexpr int kProbeVec = 2048;     // uint4 elements = 32 KB (static shared memory)
constexpr int kProbeIters = 4096;

__global__ void __launch_bounds__(kProbeThreads, 1) smem_probe_kernel(uint32_t* sink, int stride) {
    __shared__ uint4 buf[kProbeVec];
    for (int i = threadIdx.x; i < kProbeVec; i += blockDim.x) buf[i] = make_uint4(i, i * 3u, i * 5u, i * 7u);
    __syncthreads();
    uint32_t acc = 0;
    int idx = threadIdx.x;
#pragma unroll 8
    for (int it = 0; it < kProbeIters; it++) {
        const uint4 v = buf[idx];  // a warp reads 512 contiguous bytes: 4 conflict-free wavefronts
        acc += v.x ^ v.y ^ v.z ^ v.w;
        idx = (idx + stride) & (kProbeVec - 1);  // stride is a runtime argument: no load is provably redundant
    }
    if (acc == 0x12345678u) sink[threadIdx.x] = acc;  // keeps the loads alive
}

}  // namespace

extern "C" int hs_probe_smem_bandwidth(int device, double* bytes_per_s, double* ms) {
    if (!bytes_per_s) return hsx::fail(-2, "null argument");
    hsx::DeviceGuard dg(device);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    uint32_t* sink = nullptr;
    CK(cudaMalloc(&sink, kProbeThreads * sizeof(uint32_t)), "cudaMalloc");
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = prop.multiProcessorCount;
    smem_probe_kernel<<<grid, kProbeThreads>>>(sink, kProbeThreads + 16);  // warm-up (clocks up)
    smem_probe_kernel<<<grid, kProbeThreads>>>(sink, kProbeThreads + 16);
    cudaEventRecord(a);
    const int reps = 10;
    for (int r = 0; r < reps; r++) smem_probe_kernel<<<grid, kProbeThreads>>>(sink, kProbeThreads + 16);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (e != cudaSuccess) return hsx::fail(-1, "smem probe", e);
    const double bytes = (double)reps * grid * kProbeThreads * (double)kProbeIters * 16.0;
    *bytes_per_s = bytes / (t * 1e-3);
    if (ms) *ms = t / reps;
    return 0;
}
