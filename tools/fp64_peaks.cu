// FP64 peak microbenchmarks for the roofline denominators (MEASURED_PEAKS.json
// carries only HBM copy and bf16 GEMM). Measures: DFMA vector pipe, DMMA
// (mma.sync m8n8k4 f64) tensor pipe, cuBLAS DGEMM, and an HBM copy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lcublas fp64_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cublas_v2.h>
#include <cuda_runtime.h>

#define CK(x)                                                                                                       \
    do {                                                                                                            \
        cudaError_t e = (x);                                                                                        \
        if (e != cudaSuccess) {                                                                                     \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);                         \
            exit(1);                                                                                                \
        }                                                                                                           \
    } while (0)

__global__ void dfma_loop(double *out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
           x7 = x0 + 7;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) {
            x0 = fma(x0, a, b);
            x1 = fma(x1, a, b);
            x2 = fma(x2, a, b);
            x3 = fma(x3, a, b);
            x4 = fma(x4, a, b);
            x5 = fma(x5, a, b);
            x6 = fma(x6, a, b);
            x7 = fma(x7, a, b);
        }
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) out[0] = s;
}

// the same with three per-thread (vector-register) operands, as a real kernel's DFMA has:
// x_i = fma(x_i, y_i, z_i), y and z rotating through registers
__global__ void dfma3_loop(double *out, int iters, double a, double b) {
    double x[8], y[8], z[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        x[k] = threadIdx.x * 1e-9 + k;
        y[k] = a + k * 1e-12 + threadIdx.x * 1e-15;
        z[k] = b + k * 1e-13;
    }
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++)
#pragma unroll
            for (int k = 0; k < 8; k++) x[k] = fma(x[k], y[(k + j) & 7], z[(k + 3 * j) & 7]);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += x[k];
    if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int CHAINS> __global__ void dmma_loop(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
    double c[CHAINS][2];
#pragma unroll
    for (int k = 0; k < CHAINS; k++) c[k][0] = c[k][1] = 0.0;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < CHAINS; k++) dmma(c[k][0], c[k][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < CHAINS; k++) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double4 *__restrict__ a, double4 *__restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
    double *dout;
    CK(cudaMalloc(&dout, 64));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;

    // DFMA
    for (int occ : {4, 8, 16}) {
        const int iters = 4000, threads = 256, blocks = sms * occ;
        dfma_loop<<<blocks, threads>>>(dout, 10, 1.0000001, 1e-9);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 16 * 8 * (double)iters * threads * blocks;
        {
            dfma3_loop<<<blocks, threads>>>(dout, 10, 1.0000001, 1e-9);
            CK(cudaEventRecord(e0));
            dfma3_loop<<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms3 = 0;
            CK(cudaEventElapsedTime(&ms3, e0, e1));
            const double fl3 = 2.0 * 8 * 16 * (double)iters * blocks * threads;
            printf("{\"kind\": \"dfma_3vec\", \"blocks_per_sm\": %d, \"tflops\": %.3f, \"ms\": %.3f}\n", occ,
                   fl3 / (ms3 * 1e-3) / 1e12, ms3);
        }
        printf("{\"kind\": \"dfma\", \"blocks_per_sm\": %d, \"tflops\": %.3f, \"ms\": %.3f}\n", occ,
               flops / (ms * 1e-3) / 1e12, ms);
    }
    // DMMA
    for (int occ : {1, 2, 4, 8}) {
        const int iters = 20000, threads = 128, blocks = sms * occ;
        dmma_loop<8><<<blocks, threads>>>(dout, 10);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        dmma_loop<8><<<blocks, threads>>>(dout, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks;
        printf("{\"kind\": \"dmma_m8n8k4\", \"blocks_per_sm\": %d, \"warps_per_block\": 4, \"tflops\": %.3f, \"ms\": %.3f}\n",
               occ, flops / (ms * 1e-3) / 1e12, ms);
    }
    // cuBLAS DGEMM
    {
        cublasHandle_t h;
        cublasCreate(&h);
        for (int n : {2048, 4096, 8192}) {
            double *A, *B, *C;
            CK(cudaMalloc(&A, sizeof(double) * n * n));
            CK(cudaMalloc(&B, sizeof(double) * n * n));
            CK(cudaMalloc(&C, sizeof(double) * n * n));
            cudaMemset(A, 0, sizeof(double) * n * n);
            cudaMemset(B, 0, sizeof(double) * n * n);
            const double one = 1.0, zero = 0.0;
            for (int w = 0; w < 3; w++) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
            CK(cudaDeviceSynchronize());
            const int reps = n >= 8192 ? 5 : 20;
            cudaEventRecord(e0);
            for (int r = 0; r < reps; r++)
                cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            printf("{\"kind\": \"cublas_dgemm\", \"n\": %d, \"tflops\": %.3f}\n", n,
                   2.0 * n * (double)n * n * reps / (ms * 1e-3) / 1e12);
            cudaFree(A);
            cudaFree(B);
            cudaFree(C);
        }
        cublasDestroy(h);
    }
    // HBM copy
    {
        const size_t n = (size_t)1 << 28; // 256M doubles... as double4 count below
        double4 *a, *b;
        CK(cudaMalloc(&a, n * 8));
        CK(cudaMalloc(&b, n * 8));
        cudaMemset(a, 0, n * 8);
        const size_t n4 = n / 4;
        copy_kernel<<<sms * 8, 512>>>(a, b, n4);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < 10; r++) copy_kernel<<<sms * 8, 512>>>(a, b, n4);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"kind\": \"hbm_copy\", \"gbs\": %.1f}\n", 2.0 * n * 8 * 10 / (ms * 1e-3) / 1e9);
    }
    return 0;
}
