// Batched dense translations on the FP64 tensor pipe (DMMA via mma.sync m8n8k4 f64):
//
//   Y[:, out(c)] = epi( sum_{slot} A[mat(slot)] * X[:, src(slot, c)] )
//
// A single "gather GEMM" covers every translation of the KIFMM passes:
//   M2L (src/fmm.cpp:560-574, 135-175): slots = the 316 cell offsets, src = V-list box
//   M2M (src/fmm.cpp:544-548):          slots = 8 child octants, src = child box
//   L2L (src/fmm.cpp:589-592):          slots = 8 octants, src = parent box
//   pinv_apply (src/linalg.cpp:78-87):  1 slot, A = U^T then V, identity gather
// Vectors are box-major (each box's K values contiguous, padded to Kp); matrices are
// row-major Kp x Kp, zero-padded.
#pragma once

#include <cstdint>

#include "common.h"

namespace pkgpu {

struct GemmArgs {
    int Kp = 0;                      // padded K (rows of A, length of vectors); multiple of 64
    int ncols = 0;                   // output columns, multiple of kGemmBN
    const int *out_box = nullptr;    // [ncols] output box per column (-1 = padding), or null: box0 + c (< nvalid)
    int box0 = 0, nvalid = 0;
    int nslots = 1;
    const int *src = nullptr;        // [nslots * ld_src] source box per (slot, column); -1 none. null: identity
    int64_t ld_src = 0;
    const int *slot_mat = nullptr;   // [nslots] matrix id per slot, null: slot index
    const int *tile_mat = nullptr;   // [ncols / 64] matrix id per column tile (overrides slot_mat)
    const double *A = nullptr;       // matrices, Kp*Kp each
    int nmat = 1;                    // number of stacked matrices at A (TMA tensor map extent)
    int bn = 64;                     // 128: columns come in homogeneous 128-blocks (wide tiles allowed)
    const double *X = nullptr;       // input vectors [box][Kp]
    double *Y = nullptr;             // output vectors [box][Kp]
    double alpha = 1.0, beta = 0.0;  // y = beta*y + alpha*acc
    const double *rdiv = nullptr;    // pinv stage 1: y = (rdiv[r] > rdiv_eps) ? acc / rdiv[r] : 0
    double rdiv_eps = 0.0;
    int napps = 0;                   // upper bound on the (valid column, sourced slot) pairs when the caller
                                     // knows it (the top levels: 1-64): such launches take the skinny kernel
};

constexpr int kGemmBN = 64;

// Launches on `stream`; may use `ws` for split-reduction partials. Returns launches.
int gather_gemm(const GemmArgs &a, Workspace &ws, cudaStream_t stream, int num_sms);

// y[i] = beta*y[i] + alpha * sum_j A[i, j] x[j] for a single vector (rows x cols row-major).
void gemv(const double *A, int rows, int cols, int lda, const double *x, double *y, double alpha, double beta,
          const double *rdiv, double rdiv_eps, cudaStream_t stream);

} // namespace pkgpu
