// Pipeline-handshake probe for the M2L int8 kernel: the full/empty mbarrier ring of
// m2l_i8_kernel with NO data movement. One producer warp waits "empty[s]" and arrives on
// "full[s]"; one MMA thread waits "full[s]", issues `mma` M128 x N x K32 kind::i8 MMAs
// from fixed shared-memory operands and tcgen05.commit's "empty[s]". Prints int8 TOP/s per
// (stages, MMAs per stage, N), so the ring's round-trip cost can be read against the
// back-to-back peak (tools/i8_peak.cu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_pipe_probe tools/i8_pipe_probe.cu
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

constexpr int M = 128, NMAX = 256, KB = 128;
#ifndef TIMING
#define TIMING 0
#endif
#define CLK() (TIMING ? clock64() : 0LL)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
    return (uint64_t)((a & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
__device__ __forceinline__ bool try_bar(uint64_t *b, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok)
                 : "r"(su32(b)), "r"(par)
                 : "memory");
    return ok;
}
__device__ __forceinline__ void wait_bar(uint64_t *b, uint32_t par) {
    while (!try_bar(b, par)) {
    }
}
// spin styles: 0 plain try_wait loop, 1 try_wait with a suspend-time hint, 2 test_wait + nanosleep
__device__ __forceinline__ void wait_style(uint64_t *b, uint32_t par, int style) {
    if (style == 1) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok)
                         : "r"(su32(b)), "r"(par), "r"(1000000)
                         : "memory");
    } else if (style == 2) {
        uint32_t ok = 0;
        while (true) {
            asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok)
                         : "r"(su32(b)), "r"(par)
                         : "memory");
            if (ok) break;
            __nanosleep(64);
        }
    } else {
        wait_bar(b, par);
    }
}

__global__ void __launch_bounds__(128, 1) pipe(int iters, int ns, int mmas, int n, int all_lanes, int style, int lane0, int *out) {
    extern __shared__ unsigned char raw[];
    unsigned char *s = (unsigned char *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full[8], empty[8], done;
    __shared__ uint32_t tm;
    for (int i = threadIdx.x; i < (M + NMAX) * KB / 4; i += blockDim.x) ((int *)s)[i] = 0x01010101 * (i & 3);
    if (threadIdx.x == 0) {
        for (int i = 0; i < ns; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&full[i])), "r"(all_lanes ? 32 : 1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&empty[i])));
        }
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
    const int warp = __shfl_sync(0xffffffffu, (int)threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
    if (warp == 1 && !(style & 96)) {
        long long pw = 0, pa = 0;
        for (int i = 0; i < iters; i++) {
            const int st = i % ns;
            const long long c0 = CLK();
            if (!lane0 || lane == 0) wait_style(&empty[st], ((i / ns) & 1) ^ 1, style & 3);
            __syncwarp();
            const long long c1 = CLK();
            if (all_lanes || lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&full[st])) : "memory");
            const long long c2 = CLK();
            pw += c1 - c0, pa += c2 - c1;
        }
        if (lane == 0 && blockIdx.x == 0) out[4] = (int)(pw / iters), out[5] = (int)(pa / iters);
    } else if (warp == 0 && (style & 16)) {
        // whole warp runs the loop; one elected lane issues the MMAs / commit (warp-uniform operands)
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint64_t ad = desc(su32(s)), bd = desc(su32(s + M * KB));
        long long tw = 0, tf = 0, tc = 0;
        for (int i = 0; i < iters; i++) {
            const int st = i % ns;
            const long long c0 = CLK();
            if (style & 64) {
            } else if (style & 32) wait_bar(&empty[st], ((i / ns) & 1) ^ 1);
            else wait_bar(&full[st], (i / ns) & 1);
            const long long c1 = CLK();
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const long long c2 = CLK();
            for (int k = 0; k < mmas; k++)
                asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
                             "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                             "l"(ad + 2 * (k & 3)), "l"(bd + 2 * (k & 3)), "r"(idesc), "r"((i | k) ? 1u : 0u));
            asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                             su32(&empty[(style & 128) ? 0 : st]))
                         : "memory");
            const long long c4 = CLK();
            tw += c1 - c0, tf += c2 - c1, tc += c4 - c2;
        }
        if (lane == 0) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&done))
                         : "memory");
            wait_bar(&done, 0);
            if (blockIdx.x == 0) out[1] = (int)(tw / iters), out[2] = (int)(tf / iters), out[3] = (int)(tc / iters);
        }
        __syncwarp();
    } else if (warp == 0 && lane == 0) {
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint64_t ad = desc(su32(s)), bd = desc(su32(s + M * KB));
        long long tw = 0, tf = 0, tc = 0;
        for (int i = 0; i < iters; i++) {
            const int st = i % ns;
            const long long c0 = CLK();
            if (!(style & 64)) wait_style(&full[st], (i / ns) & 1, (style >> 2) & 3);
            const long long c1 = CLK();
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const long long c2 = CLK();
            for (int k = 0; k < mmas; k++)
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tm),
                             "l"(ad + 2 * (k & 3)), "l"(bd + 2 * (k & 3)), "r"(idesc), "r"((i | k) ? 1u : 0u));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             su32(&empty[st]))
                         : "memory");
            const long long c4 = CLK();
            tw += c1 - c0, tf += c2 - c1, tc += c4 - c2;
        }
        if (blockIdx.x == 0) out[1] = (int)(tw / iters), out[2] = (int)(tf / iters), out[3] = (int)(tc / iters);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&done))
                     : "memory");
        wait_bar(&done, 0);
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
    CK(cudaMalloc(&out, 32));
    const int smem = (M + NMAX) * KB + 1024;
    CK(cudaFuncSetAttribute(pipe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    // stages, MMAs per stage, N, 32 arrivals, spin style (producer | MMA thread << 2), lane-0 spin
    const int cases[][6] = {{4, 4, 224, 0, 64, 0}, {4, 4, 224, 0, 0, 0}, {4, 4, 224, 0, 16+64, 0}, {4, 4, 224, 0, 16, 0}, {8, 4, 224, 0, 16, 0}};
    for (auto &c : cases) {
        const int ns = c[0], mmas = c[1], n = c[2], all = c[3], style = c[4], l0 = c[5];
        const int iters = 80000 / mmas;
        pipe<<<sms, 128, smem>>>(100, ns, mmas, n, all, style, l0, out);
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 3; r++) {
            CK(cudaEventRecord(a));
            pipe<<<sms, 128, smem>>>(iters, ns, mmas, n, all, style, l0, out);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (ms < best) best = ms;
        }
        const double ops = 2.0 * M * n * 32 * (double)iters * mmas * sms;
        int h[8];
        CK(cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost));
        printf("clk/iter: wait %d fences %d mma+commit %d | producer wait %d arrive %d\n", h[1], h[2], h[3], h[4], h[5]);
        printf("{\"stages\": %d, \"mmas_per_stage\": %d, \"N\": %d, \"arrivals\": %d, \"spin\": %d, \"lane0\": %d, "
               "\"int8_tops\": %.1f, \"ms\": %.3f}\n",
               ns, mmas, n, all ? 32 : 1, style, l0, ops / (best * 1e-3) / 1e12, best);
    }
    return 0;
}
