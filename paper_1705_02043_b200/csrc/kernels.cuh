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
