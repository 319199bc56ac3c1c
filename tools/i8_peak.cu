// int8 tensor-pipe peak for the M2L roofline denominator: tcgen05.mma.cta_group::1.kind::i8
// issued back to back by one thread per SM from shared-memory operands that never change
// (no loads), accumulating into TMEM; one CTA per SM, all SMs. Prints JSON lines (int8
// TOP/s, 2 ops / MAC):
//   mode "loop":  M128 x N x K32 MMAs back to back (N = 256: the roofline peak; N = 224: the
//                 M2L kernel's tile)
//   mode "stage": the M2L kernel's per-stage protocol without loads -- every 4 MMAs the
//                 issuing thread commits to an mbarrier and waits on a ready one, with the
//                 fence.proxy.async + tcgen05.fence of the real mainloop
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

constexpr int M = 128, NMAX = 256, KB = 128; // one 128-byte K chunk per operand tile

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
__device__ __forceinline__ void wait_bar(uint64_t *b, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                     su32(b)),
                 "r"(par)
                 : "memory");
}

__global__ void __launch_bounds__(128, 1)
    i8_loop(int iters, int n, int staged, int fill, const int4 *gsrc, unsigned long long *filled, int *out) {
    extern __shared__ unsigned char raw[];
    unsigned char *s = (unsigned char *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t bar, done;
    __shared__ uint32_t tm;
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    for (int i = threadIdx.x; i < (M + NMAX) * KB / 4; i += blockDim.x) ((int *)s)[i] = 0x01010101 * (i & 3);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&done)));
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
    if (fill && threadIdx.x >= 32 && (fill == 2 || threadIdx.x < 96)) {
        // fill warps: cp.async 16 B chunks from an L2-resident buffer into a separate 32 KB
        // smem region, two 16 KB groups in flight, until the MMA thread is done
        unsigned char *f = s + (M + NMAX) * KB;
        const int t = threadIdx.x - 32;
        unsigned long long bytes = 0;
        int it = 0;
        while (!stop) {
            const int grp = it & 1;
#pragma unroll
            for (int i = 0; i < 16; i++) {
                const int chunk = (t + 64 * i) & 1023; // 1024 chunks = 16 KB
                const int4 *g = gsrc + ((size_t)(blockIdx.x * 4096 + it * 1024 + chunk) & ((1 << 18) - 1));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(f + grp * 16384 + chunk * 16)),
                             "l"(g));
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
            if (fill == 2) asm volatile("cp.async.wait_group 3;\n" ::: "memory");
            else asm volatile("cp.async.wait_group 1;\n" ::: "memory");
            bytes += 16 * 16;
            it++;
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        atomicAdd(filled, bytes);
    }
    if (threadIdx.x == 0) {
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint64_t ad = desc(su32(s)), bd = desc(su32(s + M * KB));
        for (int i = 0; i < iters; i++) {
            if (staged) {
                // a "full" barrier that is already complete (phase 0 of a fresh barrier: parity 1)
                wait_bar(&done, 1);
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            }
#pragma unroll
            for (int k = 0; k < KB / 32; k++)
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                             "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(idesc), "r"((i | k) ? 1u : 0u));
            if (staged)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                                 su32(&bar))
                             : "memory");
        }
        if (!staged)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             su32(&bar))
                         : "memory");
        // wait for the last commit: parity of the iters-th (staged) or first completion
        const int completions = staged ? iters : 1;
        wait_bar(&bar, (completions - 1) & 1);
        stop = 1;
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
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int *out;
    CK(cudaMalloc(&out, 4));
    const int smem = (M + NMAX) * KB + 32768 + 1024;
    int4 *gsrc;
    unsigned long long *filled;
    CK(cudaMalloc(&gsrc, (1 << 18) * sizeof(int4)));
    CK(cudaMemset(gsrc, 1, (1 << 18) * sizeof(int4)));
    CK(cudaMalloc(&filled, 8));
    CK(cudaFuncSetAttribute(i8_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int iters = 20000;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int cases[][3] = {{256, 0, 0}, {224, 0, 0}, {192, 0, 0}, {128, 0, 0}, {224, 1, 0}, {256, 1, 0}, {224, 0, 1}, {224, 0, 2}};
    for (auto &c : cases) {
        const int n = c[0], staged = c[1], fill = c[2];
        i8_loop<<<sms, 128, smem>>>(100, n, staged, fill, gsrc, filled, out);
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 5; r++) {
            CK(cudaEventRecord(a));
            CK(cudaMemset(filled, 0, 8));
            i8_loop<<<sms, 128, smem>>>(iters, n, staged, fill, gsrc, filled, out);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (ms < best) best = ms;
        }
        const double ops = 2.0 * M * n * KB * (double)iters * sms;
        unsigned long long fb = 0;
        CK(cudaMemcpy(&fb, filled, 8, cudaMemcpyDeviceToHost));
        printf("{\"probe\": \"tcgen05.mma kind::i8 M128 N%d K32, %s%s, smem operands, 1 CTA/SM\", \"sms\": %d, "
               "\"int8_tops\": %.1f, \"ms\": %.3f, \"fill_GBps_total\": %.1f}\n",
               n, staged ? "per-4-MMA commit + barrier wait + fences (M2L stage protocol)" : "back to back",
               fill == 2 ? " + concurrent cp.async smem fills (3 warps, 4 groups in flight)" : fill ? " + concurrent cp.async smem fills (2 warps)" : "", sms, ops / (best * 1e-3) / 1e12, best,
               fb / (best * 1e-3) / 1e9);
    }
    return 0;
}
