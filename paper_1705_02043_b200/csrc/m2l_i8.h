// M2L on the integer tensor pipe: tcgen05.mma kind::i8 with TMEM accumulators.
//
// B200 has no FP64 tcgen05 kind; DMMA (mma.sync f64) tops out at ~37 TF/s while the
// int8 pipe runs at ~4.5 POP/s. The M2L products (src/fmm.cpp:560-574) are therefore
// computed EXACTLY in a residue number system:
//   A_int = rint(M_o[r,k] 2^(beta_a - e_r))      per output row r, e_r from max_o,k |M_o[r,k]|
//   X_int = rint(phi[b,k] 2^(beta_b - E_l))      per level l, E_l from max |phi| over the level
//   S[r,c] = sum_slot sum_k A_int X_int           (|S| < 2^(beta_a + beta_b + 19))
// S mod m_t for pairwise-coprime moduli m_t <= 256 is an int8 x int8 -> int32 GEMM per
// modulus (balanced residues, |x| <= 128); the Chinese remainder theorem (Garner mixed
// radix, Horner in FP64) rebuilds S from the residues and q += 2^l 2^(e_r + E - beta_a -
// beta_b) S. The only approximation is the two fixed-point roundings (2^-beta of the
// row / level maxima). Default: 16 moduli (2^125.4), beta_a = beta_b = 52 -- end-to-end
// results indistinguishable from the FP64 DMMA path (profiles/r01_m2l_arith_study.md).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.h"
#include "tuning.h"

namespace pkgpu {

constexpr int kI8MaxModuli = 20;
constexpr int kI8Tile = 256; // columns per tile: level column counts are padded to this
constexpr int64_t kI8Window = 65536; // columns per M2L gemm/finish window
// columns per window (tuning().i8_window, default kI8Window): the int32 residue sums R stay
// small enough for their atomics to hit L2 (one window of cfg4's 262k-box level: 85.8 ms, four: 82.5 ms)
int64_t i8_window(int nmod, int Ki);

// operator rows per tile: as few tiles as possible, N a multiple of 32 (<= 256), from the
// true K (operator rows past K inside the 128-padded Ki are never computed)
inline int rowtiles_of(int K) { return (K + 255) / 256; }
inline int nt_of(int K) { return ((K + rowtiles_of(K) - 1) / rowtiles_of(K) + 31) / 32 * 32; }

struct I8Operators {          // residues of the stacked M2L operators (built once per KifmmOps)
    int nmod = 0, beta_a = 0, Ki = 0, nmat = 0, K = 0;
    int8_t *res = nullptr;    // [nmod][nmat][rowtiles][Ki / 128][Nt][128] (tile-contiguous), Ki = roundup(K, 128)
    int *rowexp = nullptr;    // [Ki] e_r
};

struct I8Settings {
    bool enabled = false;
    bool trans = false;       // M2M / L2L / pseudo-inverses on the int8 pipe too (i8_translate)
    bool fft = false;         // M2L by FFT on the surface lattice (m2l_fft.h) instead of dense products
    bool lattice = false;     // filled levels by the lattice FFT M2L (m2l_lattice_level), any path but DMMA
    int nmod = 16, beta_a = 52, beta_b = 52; // accuracy study: profiles/r01_m2l_arith_study.md
    int64_t min_boxes = 1;    // levels with fewer boxes stay on the DMMA gather-GEMM
};
// the settings a call with nslots x K products per output actually uses: |S| <=
// nslots K 2^(beta_a + beta_b) must stay below M / 2 (M = product of the moduli), so moduli
// are added (up to kI8MaxModuli) while it does not; if even that is short, int8 is disabled
// for the call (M2L on DMMA). Stokes p <= 16 fits the default 16 moduli.
I8Settings i8_settings_for(const I8Settings &s, int64_t nslots, int K);
// process defaults from tuning() (PKGPU_M2L, PKGPU_M2L_I8, PKGPU_M2L_I8_MIN, PKGPU_TRANS)
const I8Settings &i8_settings();

// `tag` names the operator set's workspace buffers (one I8Operators per matrix stack)
void i8_build_operators(I8Operators &o, Workspace &ws, const double *A, int nmat, int K, int Kp, int nmod,
                        int beta_a, cudaStream_t st, const char *tag = "m2l");

// The other dense translations on the int8 pipe, same residue arithmetic with a fixed-point
// scale PER OUTPUT COLUMN (E_c from the column's own sources): valid when every source box
// of the call feeds columns of one exponent, i.e. each source feeds one column (M2M:
// children -> parent; pinv: identity) or each column has one source (L2L: parent -> child).
//   Y[out(c)][r] = rdiv ? (rdiv[r] > eps ? S / rdiv[r] : 0) : beta Y + alpha S,
//   S = sum_slot A[slot] X[src(slot, c)]
// Replaces gather_gemm for M2M (src/fmm.cpp:544-548), L2L (:589-592) and pinv_apply
// (src/linalg.cpp:78-87, two calls: U^T then V).
struct I8TransArgs {
    int K = 0, Kp = 0;
    int ncols = 0;                   // multiple of kI8Tile
    const int *out_box = nullptr;    // [ncols] output box, -1 padding
    int nslots = 1;                  // = operator stack size (slot s uses matrix s)
    const int *src = nullptr;        // [nslots * ld_src] source box, -1 none
    int64_t ld_src = 0;
    int64_t src_lo = 0, src_hi = 0;  // every source box lies in [src_lo, src_hi)
    const double *X = nullptr;       // [box][Kp]
    double *Y = nullptr;             // [box][Kp]
    double alpha = 1.0, beta = 0.0;
    const double *rdiv = nullptr;
    double rdiv_eps = 0.0;
};
int i8_translate(const I8Operators &o, const I8TransArgs &a, int beta_b, Workspace &ws, cudaStream_t st);

constexpr int kI8MaxLevels = 16;

// One call covers a run of consecutive levels (M2L needs only phi_up, so every level's
// M2L can run in one launch before the downward L2L chain): their boxes are contiguous in
// BFS order and their column ranges contiguous in the layout, each level with its own
// fixed-point scale E_l and factor 2^l.
struct I8Levels {
    int n = 0;
    int64_t box0[kI8MaxLevels + 1] = {}; // first box of each level; box0[n] = end of the run
    int64_t col0[kI8MaxLevels + 1] = {}; // first column (relative to the call's columns); col0[n] = ncols
    double alpha[kI8MaxLevels] = {};     // 2^l
};

struct I8LevelArgs {
    int K = 0, Kp = 0;
    int ncols = 0;               // multiple of kI8Tile (each level's range too)
    const int *out_box = nullptr; // [ncols] output box per column, -1 padding
    int nslots = 0;
    const int *src = nullptr;     // [nslots * ld_src] global source box ids, -1 none
    int64_t ld_src = 0;
    I8Levels lv;                  // sources of a column are boxes of the column's own level
    const double *X = nullptr;    // [box][Kp]
    double *Y = nullptr;          // [box][Kp]: Y += alpha_l * sum_slot M X
    bool big = false;             // one large level: the pair-dual kernel (see select_kernel)
    unsigned long long *mma_rows = nullptr; // profiling: += 128 x active (pair tile, slot, half) triples
};
struct I8LevelWork {
    const int8_t *xres = nullptr;     // [nmod][nbox + 1][Ki] density residues (last row zero)
    int *R = nullptr;                 // [nmod][ncols][Ki] residue sums
    int *R_ext = nullptr;             // caller-provided R (modulus split across ranks), or null
    int t0 = 0, t1 = -1;              // moduli this launch computes (-1: all)
    unsigned long long *mx = nullptr; // per-level max |phi| (bit patterns)
    int64_t rows = 0;
    int *tile_slots = nullptr, *tile_nact = nullptr; // active V slots per column tile
    int *tile_below = nullptr;                       // per tile: active slots below each slot index
    uint8_t *tile_hmask = nullptr;                   // dual kernel: per (pair tile, slot) active halves
    I8Kernel kind = I8Kernel::automatic;             // kernel variant (select_kernel)
    I8Kernel win_kind = I8Kernel::automatic;         // variant of the current column window
};
// The three steps of one level (separately timed by the stage profiler):
//   prepare: level max, density residues
//   window:  R = 0, active-slot scan (column window)
//   gemm:    the kind::i8 gather-GEMM (column window)
//   finish:  CRT rebuild, Y += alpha 2^(...) S (column window)
I8LevelWork m2l_i8_prepare(const I8Operators &o, const I8LevelArgs &a, int beta_b, Workspace &ws, cudaStream_t st,
                           int64_t *launches);
// gemm / finish act on the column window [c0, c1) (multiples of kI8Tile): R holds only the
// window's residue sums, so big levels run in windows of at most kI8Window columns
int m2l_i8_window(const I8Operators &o, const I8LevelArgs &a, I8LevelWork &w, int64_t c0, int64_t c1, Workspace &ws,
                  cudaStream_t st); // R = 0, active-slot scan of the window
int m2l_i8_gemm(const I8Operators &o, const I8LevelArgs &a, I8LevelWork &w, int64_t c0, int64_t c1, Workspace &ws,
                cudaStream_t st);
int m2l_i8_finish(const I8Operators &o, const I8LevelArgs &a, const I8LevelWork &w, int64_t c0, int64_t c1,
                  int beta_b, cudaStream_t st);
// All three; returns kernel launches.
int m2l_i8_level(const I8Operators &o, const I8LevelArgs &a, int beta_b, Workspace &ws, cudaStream_t st);

// The integer gather-GEMM alone (tests): for t < nmod, columns c < ncols, rows r < Ki
//   R[t][c][r] += sum over slots s with a source of sum_k A[t][s][r][k] * B[t][row(s, c)][k]
// reduced mod m_t per work unit (|partial| <= 3 m / 2), where row(s, c) = src - box0 for
// a source, zero_row otherwise; B has rows_per_mod rows per modulus.
int i8_gather_gemm(const int8_t *A, int nmat, const int8_t *B, int rows_per_mod, int zero_row, int Ki, int nmod,
                   const int *src, int64_t ld_src, int64_t box0, int nslots, int ncols, int *R, Workspace &ws,
                   cudaStream_t st);

const int *i8_moduli(); // host copy, kI8MaxModuli entries

} // namespace pkgpu
