// Device-resident adaptive octree (FmmTree, src/fmm.cpp:301-413) and its interaction
// lists (src/fmm.cpp:422-503), built with Morton keys + radix sort + per-box closed forms.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "common.h"

namespace pkgpu {

constexpr int kMaxLevels = kMaxDepth + 1;

// POD view passed to kernels.
struct TreeView {
    int64_t level_off[kMaxLevels + 1]; // BFS box ranges per level
    int depth;
    int nboxes;
    const unsigned long long *prefix; // Morton prefix of the box cell at its level
    const int4 *cell;                 // (cx, cy, cz, level)
    const int *parent;
    const int *child;   // 8 per box, -1 absent
    const int *isleaf;  // 1 leaf
    const int2 *srng;   // source range [begin, end) in sorted order
    const int2 *trng;   // target range
};

struct DeviceTree {
    int64_t ns = 0, nt = 0;
    int leaf_capacity = 0;
    int depth = 0;
    int64_t nboxes = 0, nleaves = 0;
    std::vector<int64_t> level_off; // size depth + 2
    std::vector<int> oct_hist;      // boxes per (level, octant): [kMaxLevels * 8]
    std::vector<int> m2m_count;     // internal boxes with sources per level: [kMaxLevels + 1]
    Workspace ws;                   // owns all device arrays below
    unsigned long long *prefix = nullptr;
    int4 *cell = nullptr;
    int *parent = nullptr, *child = nullptr, *isleaf = nullptr;
    int2 *srng = nullptr, *trng = nullptr;
    int *src_perm = nullptr, *trg_perm = nullptr; // sorted position -> original index
    int *leaves = nullptr;                        // leaf box ids, BFS order
    int *m2m_list = nullptr;                      // internal boxes with sources, BFS order (sum of m2m_count)
    double4 *src_pos = nullptr;                   // sorted sources (x, y, z, charge-or-0)
    double4 *src_f = nullptr;                     // sorted Stokes forces (f0, f1, f2, 0)
    double4 *trg_pos = nullptr;                   // sorted targets (x, y, z, 0)
    int *h_flags = nullptr;                       // pinned host scratch (4 ints), allocated once
    void *h_header = nullptr;                     // pinned copy of the level loop's header (tree.cu)
    bool full_sort = false;                       // a tree here needed more than 8 levels: sort all 36 key bits
    size_t box_capacity = 0;                      // boxes the arrays above hold (kept between builds)
    ~DeviceTree() {
        if (h_flags) cudaFreeHost(h_flags);
        if (h_header) cudaFreeHost(h_header);
    }

    TreeView view() const;
};

// Builds the tree on `stream`. Points are device pointers (packed xyz). Throws
// InvalidArgument (points outside [0,1)^3, message as src/fmm.cpp:307-323; the host
// copies are used only to format that message) or RuntimeError (leaf over capacity
// at depth 12, src/fmm.cpp:335-337).
void build_tree(DeviceTree &T, const double *d_src, int64_t ns, const double *d_trg, int64_t nt, int leaf_capacity,
                cudaStream_t stream, int64_t *launches);

// Gathers strengths into sorted order (src_pos.w for Laplace, src_f for Stokes).
void gather_strengths(DeviceTree &T, const double *d_str, int ks, cudaStream_t stream, int64_t *launches);

// Host-side export: box table (18 int32 per box), leaf index lists in increasing
// original index, and structure_hash (src/fmm.cpp:397-413).
void export_tree(const DeviceTree &T, std::vector<int32_t> &table, std::vector<int32_t> &srcidx,
                 std::vector<int32_t> &trgidx, uint64_t &hash);

// ---------------------------------------------------------------------------
// interaction lists
struct ListSetup {
    int periodic[3]; // wrap axes (image_offsets(setup, 1, 1) set), all 0 if none
};

struct CsrList {
    int64_t *off = nullptr; // nboxes + 1
    int2 *ent = nullptr;    // (box, code): code = shift code for U/W/X, offset code for V
    int64_t count = 0;
};

struct DeviceLists {
    Workspace ws;
    CsrList u, v, w, x;
    int64_t v_total = 0; // V applications (evaluate path: entries written to the M2L table)
};

// Partitioned runs: need[b] = bit mask of the ranks that read box b's equivalent density
// (V / W sources of target boxes meeting rank r's leaf range [rlo[c], rhi[c]]); all boxes
// enumerated, nothing stored but the masks (ranks < 64).
// (skip_v_levels: bit l set = level l's V sources are not needed -- its M2L runs on the lattice,
// from the gathered level)
void need_masks(const DeviceTree &T, const ListSetup &S, const int *rlo, const int *rhi, unsigned long long *need,
                cudaStream_t st, unsigned skip_v_levels = 0);

// Full CSR lists for all four types (export / tests).
void build_lists_csr(const DeviceTree &T, const ListSetup &S, DeviceLists &L, cudaStream_t stream,
                     int64_t *launches);

// Evaluate-path lists: U/W/X as CSR; V written straight into the M2L gather table
// table[slot * ld + col(b)] = c (slot = M2L offset slot, col from col_of_box).
// `mask` (optional): only boxes with mask[b] != 0 get lists (partitioned runs).
void build_lists_eval(const DeviceTree &T, const ListSetup &S, DeviceLists &L, int *m2l_table, int64_t ld,
                      const int *col_of_box, const int *slot_of_code, cudaStream_t stream, int64_t *launches,
                      const int *mask = nullptr);

} // namespace pkgpu
