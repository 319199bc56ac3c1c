// The one place libpkgpu reads PKGPU_* tuning variables (see tuning.h).
#include "tuning.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace pkgpu {

namespace {
int64_t env_int(const char *name, int64_t def, int64_t lo) {
    const char *e = std::getenv(name);
    return e && *e ? std::max<int64_t>(lo, std::atoll(e)) : def;
}
} // namespace

const Tuning &tuning() {
    static const Tuning t = [] {
        Tuning r;
        if (const char *e = std::getenv("PKGPU_M2L")) r.m2l_int8 = std::strcmp(e, "dmma") != 0;
        if (const char *e = std::getenv("PKGPU_TRANS")) r.trans_int8 = std::strcmp(e, "i8") == 0;
        if (const char *e = std::getenv("PKGPU_M2L_I8")) {
            int a = r.nmod, b = r.beta_a, d = r.beta_b;
            if (std::sscanf(e, "%d,%d,%d", &a, &b, &d) == 3) r.nmod = a, r.beta_a = b, r.beta_b = d;
        }
        r.i8_min_boxes = env_int("PKGPU_M2L_I8_MIN", r.i8_min_boxes, 1);
        r.i8_small_boxes = env_int("PKGPU_I8_SMALL", r.i8_small_boxes, 0);
        r.i8_window = env_int("PKGPU_I8_WINDOW", r.i8_window, 0);
        if (const char *e = std::getenv("PKGPU_I8_KERNEL")) {
            if (!std::strcmp(e, "single")) r.i8_kernel = I8Kernel::single;
            else if (!std::strcmp(e, "dual")) r.i8_kernel = I8Kernel::dual;
            else if (!std::strcmp(e, "pairdual")) r.i8_kernel = I8Kernel::pairdual;
        }
        r.i8_by_index = (int)env_int("PKGPU_I8_BYINDEX", r.i8_by_index, -1);
        r.i8_tile_fast = (int)env_int("PKGPU_I8_TILEFAST", r.i8_tile_fast, -1);
        r.i8_min_chunks = (int)env_int("PKGPU_I8_CHUNKS", r.i8_min_chunks, 0);
        r.i8_dynamic = (int)env_int("PKGPU_I8_DYNAMIC", r.i8_dynamic, 0);
        r.gemm_units_per_cta = env_int("PKGPU_GEMM_UNITS", r.gemm_units_per_cta, 1);
        r.gemm_min_iters = env_int("PKGPU_GEMM_MINIT", r.gemm_min_iters, 1);
        r.gemm_min_iters_small = env_int("PKGPU_GEMM_MINIT_SMALL", r.gemm_min_iters_small, 1);
        r.gemm_hybrid = env_int("PKGPU_GEMM_HYBRID", 1, 0) != 0;
        r.gemm_skinny_apps = env_int("PKGPU_GEMM_SKINNY", r.gemm_skinny_apps, 0);
        r.overlap_lists = env_int("PKGPU_OVERLAP_LISTS", 1, 0) != 0;
        r.overlap_m2l = env_int("PKGPU_OVERLAP_M2L", 1, 0) != 0;
        r.tree_cap = env_int("PKGPU_TREE_CAP", 0, 0);
        r.list_warp_max = env_int("PKGPU_LIST_WARP_MAX", r.list_warp_max, 0);
        r.leaf_tt = (int)env_int("PKGPU_LEAF_TT", r.leaf_tt, 1);
        r.m2l_lattice = env_int("PKGPU_M2L_LATTICE", 1, 0) != 0;
        if (const char *e = std::getenv("PKGPU_LATTICE_FILL")) r.lattice_fill = std::atof(e);
        r.lattice_max_ranks = (int)env_int("PKGPU_LATTICE_RANKS", r.lattice_max_ranks, 0);
        r.lattice_budget = env_int("PKGPU_LATTICE_GB", r.lattice_budget >> 30, 0) << 30;
        return r;
    }();
    return t;
}

} // namespace pkgpu
