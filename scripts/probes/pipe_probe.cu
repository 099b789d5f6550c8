// Probe: issue throughput of the min/max flavours the 8x8 bottleneck DP can
// use (VIMNMX.U16x2 / VIMNMX3.U16x2 on the ALU pipe; HMNMX2 on ?), alone and
// mixed.  One CTA per SM, 16 warps, 8 independent chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

template <int MODE>
__global__ void k(uint32_t* out, int iters, uint32_t seed) {
    uint32_t a[8];
    for (int i = 0; i < 8; i++) a[i] = seed * (threadIdx.x + i + 1);
    const uint32_t b = seed ^ 0x1234u, c = seed ^ 0x0777u;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (MODE == 0 || (MODE == 2 && (i & 1)) || (MODE == 5 && (i & 1)))
                asm volatile("max.u16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            if (MODE == 1 || (MODE == 2 && !(i & 1)))
                asm volatile("max.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b));
            if (MODE == 3) asm volatile("min.u16x2 %0, %0, %1;\n\tmin.u16x2 %0, %0, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
            if (MODE == 4 || (MODE == 5 && !(i & 1))) asm volatile("mad.lo.u32 %0, %0, 3, %1;" : "+r"(a[i]) : "r"(b));
        }
    }
    uint32_t s = 0;
    for (int i = 0; i < 8; i++) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* d; cudaMalloc(&d, sms * 1024 * 4);
    const char* names[] = {"VIMNMX.U16x2", "HMNMX2", "VIMNMX+HMNMX2 mix", "VIMNMX3.U16x2", "IMAD", "VIMNMX+IMAD mix"};
    const int iters = 20000;
    for (int m = 0; m < 6; m++) {
        for (int warps : {16, 32}) {
            auto f = m == 0 ? k<0> : m == 1 ? k<1> : m == 2 ? k<2> : m == 3 ? k<3> : m == 4 ? k<4> : k<5>;
            f<<<sms, 32 * warps>>>(d, 10, 1);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            f<<<sms, 32 * warps>>>(d, iters, 1);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double inst = (double)sms * warps * iters * 8;  // warp-instructions of the op
            printf("%-20s warps/SM %2d: %.3f ms, %.2f warp-inst/clk/SM at 1.965 GHz\n", names[m], warps, ms,
                   inst / sms / (ms * 1e-3 * 1.965e9));
        }
    }
    return 0;
}
