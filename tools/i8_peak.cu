// int8 tensor-pipe peak for the M2L roofline denominator: tcgen05.mma.cta_group::1.kind::i8
// (M128 N256 K32, the instruction shape of csrc/m2l_i8.cu) issued back to back by one
// thread per SM from shared-memory operands that never change (no loads), accumulating
// into TMEM; one CTA per SM, all 148 SMs. Prints one JSON line (int8 TOP/s, 2 ops / MAC).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_peak tools/i8_peak.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                                                       \
    do {                                                                                                            \
        cudaError_t e = (x);                                                                                        \
        if (e != cudaSuccess) {                                                                                     \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);                         \
            exit(1);                                                                                                \
        }                                                                                                           \
    } while (0)

constexpr int M = 128, N = 256, KB = 128; // one 128-byte K chunk per operand tile
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}

__global__ void __launch_bounds__(128, 1) i8_loop(int iters, int *out) {
    extern __shared__ unsigned char raw[];
    unsigned char *s = (unsigned char *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tm;
    for (int i = threadIdx.x; i < (M + N) * KB / 4; i += blockDim.x) ((int *)s)[i] = 0x01010101 * (i & 3);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(su32(&tm)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (threadIdx.x == 0) {
        const uint64_t ad = desc(su32(s)), bd = desc(su32(s + M * KB));
        for (int i = 0; i < iters; i++) {
#pragma unroll
            for (int k = 0; k < KB / 32; k++)
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                             "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(IDESC), "r"((i | k) ? 1u : 0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar))
                     : "memory");
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
                         su32(&bar))
                     : "memory");
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tm + ((threadIdx.x & 96) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (v == 0x7fffffff) out[0] = v;
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tm));
}

int main() {
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    int *out;
    CK(cudaMalloc(&out, 4));
    const int smem = (M + N) * KB + 1024;
    CK(cudaFuncSetAttribute(i8_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int iters = 20000;
    i8_loop<<<sms, 128, smem>>>(100, out);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        CK(cudaEventRecord(a));
        i8_loop<<<sms, 128, smem>>>(iters, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    const double ops = 2.0 * M * N * KB * (double)iters * sms;
    printf("{\"probe\": \"tcgen05.mma kind::i8 M128 N256 K32 loop, smem operands, 1 CTA/SM\", \"sms\": %d, "
           "\"int8_tops\": %.1f, \"ms\": %.3f, \"clock_khz_attr\": %d}\n",
           sms, ops / (best * 1e-3) / 1e12, best, clk);
    return 0;
}
