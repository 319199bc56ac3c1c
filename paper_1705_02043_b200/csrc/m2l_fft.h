// FFT-accelerated M2L (the PVFMM scheme) for the V lists of
// src/fmm.cpp:560-574: an alternative to the dense offset operators of src/fmm.cpp:135-175.
//
// The equivalent (source) and check (target) points of an M2L pair are the same surface
// lattice (inner 1.05 surface, spacing 1.05 / (p - 1) at the root) around the two box
// centres, so for a fixed cell offset d the operator is a convolution on the lattice:
//   q_a(g_i) = sum_b sum_j k_{d,ab}(g_i - g_j) phi_b(g_j),  k_{d,ab}(dg) = K_ab(dg D - d)
// (root scale; level l scales by 2^l, degree -1 kernels, as the dense path). On an N^3 grid,
// N = 2p - 1 (every surface difference once), the cyclic convolution equals the linear one at
// every surface point. Per level:
//   phi_b of every source box scattered onto the grid, batched R2C FFTs (cuFFT);
//   Q^_a(w) = sum over V entries sum_b K^_{d,ab}(w) Phi^_{src,b}(w)   (fft_hadamard_kernel);
//   batched C2R FFTs, check potentials gathered at the surface points.
// FP64 throughout (no fixed point); rounding differs from the dense product only at the
// FFT's ~1e-15 relative level. K^ (316 offsets x kt x ks spectra) is built once per (kernel, p).
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <vector>

#include "common.h"

namespace pkgpu {

struct KifmmOps;

// Lattice M2L of one level shape (parent-lattice edges mx, my, mz; see m2l_lattice_level):
// the stencil spectra M_e(kappa, w) for the 14 box-offset classes e >= 0 (the other 13 are
// their conjugates), symmetric (a, b) components only.
struct LatticeShape {
    int m[3] = {0, 0, 0};
    int64_t M3 = 0;
    double *M = nullptr;            // [M3][14][ncomp][nw] complex, ncomp = ks (ks + 1) / 2
    int64_t *pairs = nullptr;       // [npairs] (kappa, -kappa) packed low | high << 32
    int64_t npairs = 0;
};

struct FftOps {
    int N = 0, nw = 0;               // grid edge 2p - 1; half spectrum N * N * (N / 2 + 1)
    double *khat = nullptr;          // [316][kt][ks][nw] complex (interleaved re, im)
    int *gidx = nullptr;             // [n] grid index of surface point i
    bool ready = false;
    std::map<int, long long> plans_r2c, plans_c2r; // cufftHandle per batch size
    std::map<std::array<int, 3>, LatticeShape> lattice; // per parent-lattice shape
    ~FftOps();
};

struct FftLevelArgs {
    int ncols = 0;               // multiple of 8
    const int *out_box = nullptr; // [ncols] output box, -1 padding
    const int *src = nullptr;     // [316 * ld] source box per (slot, column), -1 none
    int64_t ld = 0;
    int64_t box0 = 0, box1 = 0;   // the level's boxes (every source lies in [box0, box1))
    const double *X = nullptr;    // phi_up [box][Kp]
    double *Y = nullptr;          // q [box][Kp]: Y += alpha * M2L
    double alpha = 1.0;
};

// Lattice M2L of a filled level (SURVEY §8f rank 3 taken one step further): with the
// level's boxes embedded in their lattice (absent boxes = zero densities), the V lists of
// every target of octant o are the same box stencil, so the V-list sum is a convolution on
// the PARENT lattice u (box 2u + c, c the octant):
//   Q_o(u) = sum_c sum_{D in {-1,0,1}^3, |2D + c - o| >= 2} K_{2D+c-o} phi_c(u + D),
// periodic axes wrapping (edge m = 2^(l-1)), free axes zero-padded to 2m. After the surface
// FFT (Phi^) and a 3D FFT over u, it is a pointwise 24 x 24 (Stokes) product per
// (kappa, w) with M_e(kappa, w) = sum_D K^_{2D+e}(w) exp(+2 pi i kappa.D / m), e = c - o.
struct LatticeLevelArgs {
    int level = 0;                 // l >= 1
    int periodic[3] = {0, 0, 0};
    int64_t box0 = 0, box1 = 0;    // the level's boxes (BFS ids)
    const int4 *cell = nullptr;    // box cells (x, y, z, level)
    const int2 *srng = nullptr, *trng = nullptr; // boxes' source / target ranges (the check: the evaluate
                                                 // lists leave out source-less sources and target-less targets)
    const int *mask = nullptr;     // the check, partitioned evaluates: boxes with mask[b] == 0 have empty lists
    const double *X = nullptr;     // phi_up [box][Kp]
    double *Y = nullptr;           // q [box][Kp]: Y += alpha * M2L
    double alpha = 1.0;
    // defer_scatter: m2l_lattice_level stops after the inverse lattice transform (result left in
    // the workspace); m2l_lattice_scatter adds it into Y later, on any stream ordered after it
    bool defer_scatter = false;
    // stage profiler hook (optional): mark(user, stage, 1) before / (.., 0) after the phases
    // "lat_fwd" (gather, lattice FFT, surface DFT), "lat_mul" (pointwise products) and
    // "lat_inv" (surface DFT, lattice FFT, scatter); work(user, stage, units, per_unit)
    // reports lat_mul's algorithmic bytes
    void (*mark)(void *user, const char *stage, int begin) = nullptr;
    void (*work)(void *user, const char *stage, double units, double per_unit) = nullptr;
    void *user = nullptr;
};
// device workspace bytes the level needs (kernel spectra, grids, lattice spectra)
int64_t m2l_lattice_bytes(const KifmmOps &ops, int level, const int periodic[3]);
// counts into bad[0] the (slot, column) V-list entries of the dense layout that differ from
// the lattice stencil (0: the lattice sum equals the V-list sum exactly)
// (with a mask the level's boxes need not all be output columns: a rank's columns are the
// boxes meeting its leaves)
int m2l_lattice_check(KifmmOps &ops, const LatticeLevelArgs &a, const int *table, int64_t ld, const int *out_box,
                      int ncols, int *bad, Workspace &ws, cudaStream_t st);
int m2l_lattice_level(KifmmOps &ops, const LatticeLevelArgs &a, Workspace &ws, cudaStream_t st);
// the deferred last step of m2l_lattice_level (same args and workspace): Y += alpha * M2L
int m2l_lattice_scatter(KifmmOps &ops, const LatticeLevelArgs &a, Workspace &ws, cudaStream_t st);

// builds K^ on first use; returns kernel launches
int m2l_fft_prepare(KifmmOps &ops, Workspace &ws, cudaStream_t st);
int m2l_fft_level(KifmmOps &ops, const FftLevelArgs &a, Workspace &ws, cudaStream_t st);

} // namespace pkgpu
