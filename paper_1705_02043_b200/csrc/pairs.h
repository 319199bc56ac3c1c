// Pair-sum kernels on the FP64 vector pipe: every use of kernel_block_apply
// (src/kernel.cpp:80-129) on the evaluate path.
#pragma once

#include "tree.h"

namespace pkgpu {

struct PairGeom {
    int kernel = 0, p = 0, n = 0, Kp = 0;
    const double *tmpl = nullptr; // n x 3 surface template
};

// Fused leaf pass (src/fmm.cpp:603-633 + far field src/periodize.cpp:173-187):
// out[kt*orig(t)] = L2T(phi_dn[b]) + sum_W M2T(phi_up[c], shift) + sum_U P2P(c, shift)
//                   + far(phi_far on the root 2.95 surface)
void leaf_pass(const PairGeom &g, const DeviceTree &T, const DeviceLists &L, const double *phi_dn,
               const double *phi_up, const double *phi_far, double *out, cudaStream_t st,
               const int *leaves = nullptr, int nleaves = 0);

// S2M at leaves (src/fmm.cpp:539-542): q[b] = K(outer check of b, sources of b) rho
// `leaves`/`nleaves` restrict the pass to a leaf subset (partitioned runs); null: all leaves
void s2m_pass(const PairGeom &g, const DeviceTree &T, double *q, cudaStream_t st, const int *leaves = nullptr,
              int nleaves = 0);

// X list / S2L (src/fmm.cpp:580-588): q[b] += K(inner check of b - shift, sources of c) rho
void x_pass(const PairGeom &g, const DeviceTree &T, const DeviceLists &L, double *q, cudaStream_t st);

// Brute force over image offsets (direct mode, src/fmm.cpp:711-719) and the generic
// kernel_block_apply primitive: out[kt*i] (+)= sum_offsets sum_j K((t_i - d) - s_j) rho_j.
// Coincident pairs at a zero offset are skipped when skip_zero; any other coincident
// pair is counted into *d_coincident (device int).
void direct_pairs(int kernel, const double *d_trg, int64_t nt, const double *d_src, const double *d_den, int64_t ns,
                  const double *d_offsets, int noff, int skip_zero, const PairGeom *far_geom, const double *phi_far,
                  double *d_out, int accumulate, int *d_coincident, Workspace &ws, cudaStream_t st);

// q = K(outer root surface, all sources) rho  (direct_root_upward_density check step,
// src/fmm.cpp:676-686), deterministic split reduction.
void root_check_potential(const PairGeom &g, const double *d_src, const double *d_den, int64_t ns, double *d_q,
                          Workspace &ws, cudaStream_t st);

} // namespace pkgpu
