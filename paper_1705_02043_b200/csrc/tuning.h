// Process-wide tuning knobs of libpkgpu, all read once from the environment here and
// nowhere else. Every default is the measured best on B200; the knobs exist
// for comparison runs and are documented in INTEGRATION.md ("Tuning knobs").
#pragma once

#include <cstdint>

namespace pkgpu {

enum class I8Kernel : int {
    automatic = -1, // pair-dual for big levels, dual for the packed small-level runs
    single = 0,     // m2l_i8_kernel: one CTA, 128-box tiles
    dual = 1,       // m2l_i8_dual_kernel: one CTA, 256-box pair tiles
    pairdual = 2,   // m2l_i8_pairdual_kernel: CTA pair (cta_group::2), 512-box quads
};

struct Tuning {
    bool m2l_int8 = true;              // PKGPU_M2L = i8 | dmma: default M2L arithmetic of new contexts
    bool trans_int8 = false;           // PKGPU_TRANS = i8 | dmma: M2M / L2L / pinv on the int8 pipe
    int nmod = 16, beta_a = 52, beta_b = 52; // PKGPU_M2L_I8 = "nmod,beta_a,beta_b"
    int64_t i8_min_boxes = 1;          // PKGPU_M2L_I8_MIN: levels with fewer boxes use DMMA
    int64_t i8_small_boxes = 1024;     // PKGPU_I8_SMALL: levels up to this size share packed runs
    int64_t i8_window = 0;             // PKGPU_I8_WINDOW: columns per int8 M2L window (0: 65536, 8192 at p >= 10)
    I8Kernel i8_kernel = I8Kernel::automatic; // PKGPU_I8_KERNEL = single | dual | pairdual
    int i8_by_index = -1;              // PKGPU_I8_BYINDEX = 0 | 1: chunks as slot-index windows (-1: per kernel)
    int i8_tile_fast = -1;             // PKGPU_I8_TILEFAST = 0 | 1: unit order, column tile fastest
    int i8_min_chunks = 0;             // PKGPU_I8_CHUNKS: at least this many slot chunks per tile
    int i8_dynamic = 0;                // PKGPU_I8_DYNAMIC = 0 | 1: dynamic unit schedule (dual-tile kernels)
    int64_t gemm_units_per_cta = 32;   // PKGPU_GEMM_UNITS: DMMA gather-GEMM work units per CTA
    int64_t gemm_min_iters = 16;       // PKGPU_GEMM_MINIT: k-iterations per split-K unit
    int64_t gemm_min_iters_small = 4;  // PKGPU_GEMM_MINIT_SMALL: same, latency-bound one-slot GEMMs
    bool gemm_hybrid = true;           // PKGPU_GEMM_HYBRID = 0 | 1: whole tiles for the full waves + an equal tail chunk per CTA
    int64_t gemm_skinny_apps = 8;      // PKGPU_GEMM_SKINNY: launches of at most this many (column, slot) pairs
                                       // take the skinny row-per-warp kernel (0: never)
    bool overlap_lists = true;         // PKGPU_OVERLAP_LISTS = 0 | 1: lists on the auxiliary stream beside the upward pass
    bool overlap_m2l = true;           // PKGPU_OVERLAP_M2L = 0 | 1: the deepest lattice level's M2L on the auxiliary
                                       // stream beside the coarse levels' downward chain
    int64_t tree_cap = 0;              // PKGPU_TREE_CAP: first box capacity of the tree arrays (0: four boxes per full
                                       // leaf); a small value exercises the grow-and-rebuild path (tests)
    int64_t list_warp_max = 50000;     // PKGPU_LIST_WARP_MAX: trees up to this size list a warp per box
    int leaf_tt = 2;                   // PKGPU_LEAF_TT = 1 | 2 | 4: targets per thread in the leaf pass
    bool m2l_lattice = true;           // PKGPU_M2L_LATTICE = 0 | 1: filled levels by the lattice FFT M2L
    double lattice_fill = 0.5;         // PKGPU_LATTICE_FILL: least fraction of the level's lattice present
    int64_t lattice_budget = 48LL << 30; // PKGPU_LATTICE_GB: device bytes the lattice levels may use
    int lattice_max_ranks = 4;         // PKGPU_LATTICE_RANKS: partitioned evaluates of more ranks keep the dense M2L
};

const Tuning &tuning();

} // namespace pkgpu
