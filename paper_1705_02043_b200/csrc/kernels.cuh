// Device-side kernel evaluation (Laplace 1/r, Stokeslet (1/8pi)(I/r + r r^T/r^3)),
// surface-point generation and the pair-sum inner loop.
#pragma once

#include <cuda_runtime.h>

namespace pkgpu {

constexpr double kOneOver8Pi = 0.039788735772973836; // 1/(8 pi), src/kernel.cpp:10

// ---------------------------------------------------------------------------
// Bit-exact operator assembly. kernel_block calls the out-of-line
// kernel_eval_nocheck (src/kernel.cpp:29-47), which the reference build (-O3, FMA
// available) compiles to (read off its x86 code):
//   r2     = (rx*rx + ry*ry) + rz*rz            (products reused -> not contracted)
//   entry  = k8 * fma(ra*ra, rinv3, rinv)        (diagonal), k8 * ((ra*rb)*rinv3) (off)
// with rinv = 1/sqrt(r2) and rinv3 = rinv/r2 correctly rounded. Written with explicit
// intrinsics so nvcc cannot re-associate; pinned by tests against refdump kblock vectors.
__device__ __forceinline__ double r2_exact(double rx, double ry, double rz) {
    return __dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), __dmul_rn(rz, rz));
}

template <int KERNEL>
__device__ __forceinline__ void kernel_entry_exact(double xx, double xy, double xz, double yx, double yy, double yz,
                                                   double *blk) {
    const double rx = __dsub_rn(xx, yx), ry = __dsub_rn(xy, yy), rz = __dsub_rn(xz, yz);
    const double r2 = r2_exact(rx, ry, rz);
    const double rinv = __ddiv_rn(1.0, __dsqrt_rn(r2));
    if (KERNEL == 0) {
        blk[0] = rinv;
        return;
    }
    const double rinv3 = __ddiv_rn(rinv, r2);
    const double r[3] = {rx, ry, rz};
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) {
            double v;
            if (a == b)
                v = __fma_rn(__dmul_rn(r[a], r[a]), rinv3, rinv);
            else if (b > a)
                v = __dmul_rn(__dmul_rn(r[a], r[b]), rinv3);
            else
                v = __dmul_rn(__dmul_rn(r[b], r[a]), rinv3); // block[3] = block[1] etc.
            blk[3 * a + b] = __dmul_rn(kOneOver8Pi, v);
        }
}

// surface point i: fma(half_edge, t_i, center) per coordinate (src/geometry.cpp:60-71
// as contracted by the reference build; t is the fma(g, 2/(p-1), -1) template).
__device__ __forceinline__ double surf_coord(double half, double t, double c) { return __fma_rn(half, t, c); }

// ---------------------------------------------------------------------------
// Fast reciprocal square root for the pair sums: MUFU.RSQ64H seed + one
// Halley-type correction (cubic convergence, ~2^-23 -> below 1 ulp before the
// final rounding). Returns 0 for r2 == 0 (the coincident-pair convention of
// src/kernel.cpp:97-98).
__device__ __forceinline__ double rinv_fast(double r2) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
    // r2 == 0 (ftz: anything below the smallest normal) -> 0: an integer select on the seed's high
    // word (MUFU.RSQ64H defines only that word; the low word of the approximation is zero), off the
    // FP64 pipe; the correction maps a zero seed to zero
    y = __hiloint2double(__double2hiint(r2) < 0x00100000 ? 0 : __double2hiint(y), 0);
    const double e = __fma_rn(-r2 * y, y, 1.0);  // 1 - r2 y^2
    const double c = __fma_rn(0.375, e, 0.5);    // 1/2 + 3/8 e
    return __fma_rn(y * e, c, y);
}

// The same pair arithmetic for a tile of M = TT targets x NS sources, written step by step
// across the M pairs: each pair is one dependent chain of ~20 FP64 operations, and issued one
// pair after the other (as pair_laplace / pair_stokes in a loop compile under the register
// cap) every operation waits out its predecessor's latency -- 34% of the leaf pass's warp
// stalls were that wait (ncu source view, profiles/r02_lattice_step_ncu.txt). Interleaved,
// the M chains fill each other's latency. Results are bit-identical to the pair functions
// (same operations, same order of accumulation per target).
template <int KERNEL, int TT, int NS>
__device__ __forceinline__ void pair_tile(const double (&ux)[TT], const double (&uy)[TT], const double (&uz)[TT],
                                          const double2 (&sxy)[NS], const double2 (&szd)[NS], const double2 (&sdd)[NS],
                                          double (&acc)[TT][3]) {
    constexpr int M = TT * NS;
    double rx[M], ry[M], rz[M], r2[M], y[M], t[M], e[M];
#pragma unroll
    for (int i = 0; i < M; i++) {
        rx[i] = ux[i % TT] - sxy[i / TT].x;
        ry[i] = uy[i % TT] - sxy[i / TT].y;
        rz[i] = uz[i % TT] - szd[i / TT].x;
    }
#pragma unroll
    for (int i = 0; i < M; i++) r2[i] = ry[i] * ry[i];
#pragma unroll
    for (int i = 0; i < M; i++) r2[i] = __fma_rn(rx[i], rx[i], r2[i]);
#pragma unroll
    for (int i = 0; i < M; i++) r2[i] = __fma_rn(rz[i], rz[i], r2[i]);
#pragma unroll
    for (int i = 0; i < M; i++) {
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y[i]) : "d"(r2[i]));
        y[i] = __hiloint2double(__double2hiint(r2[i]) < 0x00100000 ? 0 : __double2hiint(y[i]), 0);
    }
#pragma unroll
    for (int i = 0; i < M; i++) t[i] = -r2[i] * y[i];
#pragma unroll
    for (int i = 0; i < M; i++) e[i] = __fma_rn(t[i], y[i], 1.0);
#pragma unroll
    for (int i = 0; i < M; i++) t[i] = y[i] * e[i];
#pragma unroll
    for (int i = 0; i < M; i++) e[i] = __fma_rn(0.375, e[i], 0.5);
#pragma unroll
    for (int i = 0; i < M; i++) y[i] = __fma_rn(t[i], e[i], y[i]);
    if (KERNEL == 0) {
#pragma unroll
        for (int i = 0; i < M; i++) acc[i % TT][0] = __fma_rn(szd[i / TT].y, y[i], acc[i % TT][0]);
    } else {
#pragma unroll
        for (int i = 0; i < M; i++) t[i] = ry[i] * sdd[i / TT].x;
#pragma unroll
        for (int i = 0; i < M; i++) t[i] = __fma_rn(rx[i], szd[i / TT].y, t[i]);
#pragma unroll
        for (int i = 0; i < M; i++) t[i] = __fma_rn(rz[i], sdd[i / TT].y, t[i]);
#pragma unroll
        for (int i = 0; i < M; i++) t[i] = t[i] * y[i];
#pragma unroll
        for (int i = 0; i < M; i++) t[i] = t[i] * y[i];
#pragma unroll
        for (int i = 0; i < M; i++) {
            rx[i] = __fma_rn(rx[i], t[i], szd[i / TT].y);
            ry[i] = __fma_rn(ry[i], t[i], sdd[i / TT].x);
            rz[i] = __fma_rn(rz[i], t[i], sdd[i / TT].y);
        }
#pragma unroll
        for (int i = 0; i < M; i++) {
            acc[i % TT][0] = __fma_rn(rx[i], y[i], acc[i % TT][0]);
            acc[i % TT][1] = __fma_rn(ry[i], y[i], acc[i % TT][1]);
            acc[i % TT][2] = __fma_rn(rz[i], y[i], acc[i % TT][2]);
        }
    }
}

// Laplace pair: acc += rho / r
__device__ __forceinline__ void pair_laplace(double tx, double ty, double tz, double sx, double sy, double sz,
                                             double rho, double &acc) {
    const double rx = tx - sx, ry = ty - sy, rz = tz - sz;
    const double r2 = __fma_rn(rz, rz, __fma_rn(rx, rx, ry * ry));
    acc = __fma_rn(rho, rinv_fast(r2), acc);
}

// Stokeslet pair (src/kernel.cpp:114-122), the 1/(8 pi) applied once by the caller:
//   rdotf = (r.f) rinv^2 ; a_k += (f_k + r_k rdotf) rinv
__device__ __forceinline__ void pair_stokes(double tx, double ty, double tz, double sx, double sy, double sz,
                                            double f0, double f1, double f2, double &a0, double &a1, double &a2) {
    const double rx = tx - sx, ry = ty - sy, rz = tz - sz;
    const double r2 = __fma_rn(rz, rz, __fma_rn(rx, rx, ry * ry));
    const double rinv = rinv_fast(r2);
    const double rdotf = __fma_rn(rz, f2, __fma_rn(rx, f0, ry * f1)) * rinv * rinv;
    a0 = __fma_rn(__fma_rn(rx, rdotf, f0), rinv, a0);
    a1 = __fma_rn(__fma_rn(ry, rdotf, f1), rinv, a1);
    a2 = __fma_rn(__fma_rn(rz, rdotf, f2), rinv, a2);
}

} // namespace pkgpu
