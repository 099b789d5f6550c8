// Probe: raw mbarrier words after init / expect_tx / complete_tx / phase flip
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ uint64_t raw(uint64_t* m) { uint64_t r; asm volatile("ld.shared.b64 %0, [%1];" : "=l"(r) : "r"(sa(m)) : "memory"); return r; }
__global__ void k() {
    __shared__ __align__(8) uint64_t mb;
    __shared__ __align__(8) double buf[4];
    if (threadIdx.x) return;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&mb)));
    printf("init(1)            %016llx  addr %08x\n", (unsigned long long)raw(&mb), sa(&mb));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 24;" :: "r"(sa(&mb)) : "memory");
    printf("arrive.expect(24)  %016llx\n", (unsigned long long)raw(&mb));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" :: "r"(sa(buf)), "d"(1.0), "r"(sa(&mb)) : "memory");
    for (int i = 0; i < 1000; i++) __nanosleep(100);
    printf("1 push             %016llx\n", (unsigned long long)raw(&mb));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" :: "r"(sa(buf+1)), "d"(1.0), "r"(sa(&mb)) : "memory");
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" :: "r"(sa(buf+2)), "d"(1.0), "r"(sa(&mb)) : "memory");
    for (int i = 0; i < 1000; i++) __nanosleep(100);
    printf("3 pushes (done)    %016llx\n", (unsigned long long)raw(&mb));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" :: "r"(sa(buf+3)), "d"(1.0), "r"(sa(&mb)) : "memory");
    for (int i = 0; i < 1000; i++) __nanosleep(100);
    printf("push before expect %016llx\n", (unsigned long long)raw(&mb));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8;" :: "r"(sa(&mb)) : "memory");
    printf("then expect(8)     %016llx\n", (unsigned long long)raw(&mb));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 0;" :: "r"(sa(&mb)) : "memory");
    printf("expect(0)          %016llx\n", (unsigned long long)raw(&mb));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" :: "r"(sa(&mb)) : "memory");
    printf("expect(16)         %016llx\n", (unsigned long long)raw(&mb));
}
int main() { k<<<1, 32>>>(); printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize())); }
