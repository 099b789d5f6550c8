// Probe: st.async DSMEM pushes completing on the destination's mbarrier
// (the hk_cluster_kernel layer protocol), in isolation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o stas_probe stas_probe.cu
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_rank(uint32_t a, uint32_t q) {
    uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(q)); return r; }

template <int MODE>  // 0: delta = mapa(base) - base; 1: mapa per address; 2: expect posted late
__global__ void probe(int cs, int per, int self, unsigned long long* out) {
    extern __shared__ __align__(16) double buf[];
    __shared__ __align__(8) uint64_t mb;
    __shared__ uint32_t delta[16];
    uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t base = sa(buf);
    if (threadIdx.x < cs) delta[threadIdx.x] = mapa_rank(base, threadIdx.x) - base;
    for (int i = threadIdx.x; i < per; i += blockDim.x) buf[i] = -1.0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&mb)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (MODE != 2)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&mb)), "r"(per * 8) : "memory");
    }
    __syncthreads();
    cg::this_cluster().sync();
    // every CTA sends `per` values in total to every... CTA q receives slot i from CTA (i % cs) (or i%(cs-1) remote-only)
    for (int q = 0; q < cs; q++) {
        for (int i = threadIdx.x; i < per; i += blockDim.x) {
            int src = self ? (int)(i % cs) : (int)((q + 1 + i % (cs - 1)) % cs);
            if (cs == 1) src = 0;
            if (src != (int)rank) continue;
            double v = q * 1e6 + i;
            uint32_t a, m;
            if (MODE != 1) { a = base + i * 8 + delta[q]; m = sa(&mb) + delta[q]; }
            else { a = mapa_rank(base + i * 8, q); m = mapa_rank(sa(&mb), q); }
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" :: "r"(a), "d"(v), "r"(m) : "memory");
        }
    }
    if (MODE == 2 && threadIdx.x == 0) {  // complete_tx from peers lands before the expect
        long long w = clock64();
        while (clock64() - w < 2000000) {}
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&mb)), "r"(per * 8) : "memory");
    }
    uint32_t done = 0; long long t0 = clock64(); bool to = false;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(sa(&mb)) : "memory");
        if (clock64() - t0 > 4000000000LL) { to = true; break; }
    }
    int bad = 0;
    for (int i = threadIdx.x; i < per; i += blockDim.x) bad += buf[i] != rank * 1e6 + i;
    atomicAdd(out, (unsigned long long)bad);
    if (to) atomicAdd(out + 1, 1ull);
    cg::this_cluster().sync();
}

int main() {
    unsigned long long* d; cudaMalloc(&d, 16); 
    for (int cs : {2, 8, 16}) for (int self : {0, 1}) for (int mode : {0, 1, 2}) {
        cudaMemset(d, 0, 16);
        int per = 6000;
        cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
        cfg.gridDim = dim3(cs * 4); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = per * 8;
        at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        auto f = mode == 2 ? probe<2> : mode ? probe<1> : probe<0>;
        cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, per * 8);
        cudaError_t e = cudaLaunchKernelEx(&cfg, f, cs, per, self, d);
        cudaError_t e2 = cudaDeviceSynchronize();
        unsigned long long h[2] = {0, 0}; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("cs=%2d self=%d mode=%d launch=%s sync=%s mismatches=%llu timeouts=%llu\n", cs, self, mode,
               cudaGetErrorString(e), cudaGetErrorString(e2), h[0], h[1]);
        if (e2 != cudaSuccess) return 1;
    }
    return 0;
}
