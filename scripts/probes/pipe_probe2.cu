// Probe: per-instruction issue rates (warp-instr / clk / SM) of the ALU ops
// in the 8x8 bottleneck DP: VIMNMX (2-input, alternating max/min so ptxas
// cannot fuse), VIMNMX3, PRMT, LOP3, IADD3, IMAD; and mixes.
#include <cstdio>
#include <cstdint>
template <int M>
__global__ void k(uint32_t* out, int iters, uint32_t seed) {
    uint32_t a[8], b[8];
    for (int i = 0; i < 8; i++) { a[i] = seed * (threadIdx.x + i + 1); b[i] = seed ^ (i * 0x9E3779B9u); }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (M == 0) { asm volatile("max.u16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i])); asm volatile("min.u16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b[(i + 1) & 7])); }
            if (M == 1) { asm volatile("prmt.b32 %0, %0, %1, 0x1032;" : "+r"(a[i]) : "r"(b[i])); asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(a[i]) : "r"(b[(i+1)&7])); }
            if (M == 2) { asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(b[i]), "r"(b[(i+3)&7])); asm volatile("lop3.b32 %0, %0, %1, %2, 0xE8;" : "+r"(a[i]) : "r"(b[(i+1)&7]), "r"(b[(i+2)&7])); }
            if (M == 3) { asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i])); asm volatile("xor.b32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[(i+1)&7])); }
            if (M == 4) { asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(b[(i+1)&7])); asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[(i+2)&7]), "r"(b[(i+3)&7])); }
            if (M == 5) { asm volatile("max.u16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i])); asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[(i+2)&7]), "r"(b[(i+3)&7])); }
            if (M == 7) { asm volatile("fma.rn.relu.f16x2 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(b[(i+1)&7])); asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b[(i+2)&7])); }
            if (M == 8) { asm volatile("max.u16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i])); asm volatile("fma.rn.relu.f16x2 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[(i+1)&7]), "r"(b[(i+2)&7])); }
            if (M == 9) { asm volatile("max.u16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i])); asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b[(i+2)&7])); }
            if (M == 6) { asm volatile("max.u16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i])); asm volatile("prmt.b32 %0, %0, %1, 0x1032;" : "+r"(a[i]) : "r"(b[(i+1)&7])); }
        }
    }
    uint32_t s = 0;
    for (int i = 0; i < 8; i++) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* d; cudaMalloc(&d, sms * 1024 * 4);
    const char* names[] = {"VIMNMX max/min", "PRMT", "LOP3", "IADD/XOR", "IMAD", "VIMNMX+IMAD", "VIMNMX+PRMT", "HFMA2.RELU+HADD2", "VIMNMX+HFMA2.RELU", "VIMNMX+HADD2"};
    void (*fs[])(uint32_t*, int, uint32_t) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>};
    for (int m = 0; m < 10; m++) {
        const int warps = 32, iters = 20000;
        fs[m]<<<sms, 32 * warps>>>(d, 10, 1);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        fs[m]<<<sms, 32 * warps>>>(d, iters, 1);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double inst = (double)sms * warps * iters * 16;
        printf("%-16s %.3f ms  %.2f warp-inst/clk/SM (1.965 GHz)\n", names[m], ms, inst / sms / (ms * 1e-3 * 1.965e9));
    }
}
