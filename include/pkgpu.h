/* pkgpu — B200-native (sm_100a) periodic KIFMM evaluator: the C ABI.
 *
 * This is the drop-in boundary for the reference's evaluate path. Every entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj). Plain pointers and sizes only; no torch / C++ types.
 *
 * Status codes carry the reference's exception classes so a C++ shim can rethrow the
 * same type with the same message (include/pkifmm/fmm.hpp:141):
 *   PKGPU_INVALID_ARGUMENT -> std::invalid_argument
 *   PKGPU_CONFIG_ERROR     -> pkifmm::ConfigError      (include/pkifmm/refsum.hpp:16-18)
 *   PKGPU_RUNTIME_ERROR    -> std::runtime_error
 *   PKGPU_CUDA_ERROR       -> std::runtime_error (device failure; no CPU fallback exists)
 */
#ifndef PKGPU_H
#define PKGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PKGPU_OK = 0,
    PKGPU_INVALID_ARGUMENT = 1,
    PKGPU_CONFIG_ERROR = 2,
    PKGPU_RUNTIME_ERROR = 3,
    PKGPU_CUDA_ERROR = 4
} pkgpu_status;

/* KernelType (include/pkifmm/kernel.hpp:14) */
enum { PKGPU_LAPLACE = 0, PKGPU_STOKESLET = 1 };
/* Periodicity (include/pkifmm/geometry.hpp:20) */
enum { PKGPU_NONE = 0, PKGPU_SP = 1, PKGPU_DP = 2, PKGPU_TP = 3 };
/* EvalMode (include/pkifmm/fmm.hpp:112) */
enum { PKGPU_MODE_FMM = 0, PKGPU_MODE_DIRECT = 1 };
/* PeriodicMethod (include/pkifmm/refsum.hpp:33) — provenance only */
enum { PKGPU_DIRECT_SP = 0, PKGPU_EWALD_LAPLACE_DP = 1, PKGPU_EWALD_LAPLACE_TP = 2, PKGPU_EWALD_STOKES_TP = 3 };

typedef struct pkgpu_context pkgpu_context;
typedef struct pkgpu_operator pkgpu_operator;
typedef struct pkgpu_tree pkgpu_tree;

/* PeriodicSetup (include/pkifmm/geometry.hpp:26-40) */
typedef struct {
    int periodicity;
    int axes[3];
    double box_length;
    int ell;
} pkgpu_setup;

/* EvalRequest (include/pkifmm/fmm.hpp:120-131). Point arrays are packed xyz (the
 * layout of std::vector<Eigen::Vector3d>), strengths interleaved ks per source.
 * device_pointers != 0: sources/strengths/targets/out are CUDA device pointers. */
typedef struct {
    int kernel;
    int64_t n_sources;
    const double *sources;
    int64_t n_strengths;
    const double *strengths;
    int64_t n_targets;
    const double *targets;
    pkgpu_setup setup;
    int p;
    const pkgpu_operator *op; /* required unless periodicity none (non-owning) */
    int mode;
    int leaf_capacity;
    int force;
    int device_pointers;
} pkgpu_request;

/* EvalTimings (include/pkifmm/fmm.hpp:116-118), seconds, device-event timed.
 * `far` is 0: the far-field sweep is fused into the leaf pass. */
typedef struct {
    double tree, near, m2l_apply, far;
} pkgpu_timings;

/* CompatReport (include/pkifmm/refsum.hpp:75-79) */
typedef struct {
    int ok;
    double residual;
    char violated[96];
} pkgpu_compat;

/* ---- context: device, stream, device-resident operator caches ------------------- */
/* Replaces the reference's static registries (src/fmm.cpp:238-283). */
pkgpu_status pkgpu_context_create(int device, pkgpu_context **ctx, char *err, size_t errlen);
void pkgpu_context_destroy(pkgpu_context *ctx);
/* Work stream (cudaStream_t as void*); NULL -> the context's own stream. */
pkgpu_status pkgpu_context_set_stream(pkgpu_context *ctx, void *stream);
void *pkgpu_context_stream(pkgpu_context *ctx);
/* Number of kernel launches issued by this context since creation (launch accounting). */
int64_t pkgpu_context_launch_count(pkgpu_context *ctx);

/* Per-stage profiling: with profiling on, evaluate brackets every stage with CUDA
 * events on the work stream and counts its algorithmic work. Stages: "tree", "lists",
 * "s2m", "m2m", "pinv_up", "x", "m2l", "l2l", "pinv_dn", "periodic", "leaf".
 * seconds = summed device time, units = applications (dense) or pairs (pair sums),
 * flops = algorithmic FLOPs (2K^2 per translation, 4K^2+K per pinv, 11 / 28
 * per Laplace / Stokes pair), launches = kernel launches. Accumulated until reset.
 * M2L levels on the int8 pipe add sub-stages "m2l_prep" (density residues), "m2l_i8"
 * (the kind::i8 gather-GEMM; flops = int8 ops, 2 nmod K^2 per application) and
 * "m2l_crt" (CRT rebuild), all also inside "m2l". */
pkgpu_status pkgpu_context_set_profiling(pkgpu_context *ctx, int on);
/* M2L arithmetic path. path 0: int8 tensor pipe (exact residue GEMMs, CRT rebuild in
 * FP64) on levels with >= min_boxes boxes, DMMA FP64 elsewhere (default; min_boxes <= 0
 * keeps the current threshold, 1 unless PKGPU_M2L_I8_MIN says otherwise); path 1:
 * DMMA FP64 everywhere; path 2: as 0, plus M2M / L2L / pseudo-inverses on the int8 pipe
 * (per-column fixed-point scale; opt-in, slower than DMMA at cfg2). nmod / beta_a / beta_b
 * > 0 override the residue parameters
 * (moduli count 14..20, fixed-point bits of operators / densities, beta_a + beta_b +
 * 20 < sum log2 m_t). */
pkgpu_status pkgpu_context_set_m2l(pkgpu_context *ctx, int path, int64_t min_boxes, int nmod, int beta_a,
                                   int beta_b);
pkgpu_status pkgpu_context_reset_stats(pkgpu_context *ctx);
pkgpu_status pkgpu_context_stage_stats(pkgpu_context *ctx, const char *stage, double *seconds, double *units,
                                       double *flops, int64_t *launches);

/* ---- the hot path ------------------------------------------------------------------ */
/* pkifmm::evaluate (include/pkifmm/fmm.hpp:141, src/fmm.cpp:690-742). `out` receives
 * kt*n_targets doubles in the caller's target order (src/fmm.cpp:630-632). */
pkgpu_status pkgpu_evaluate(pkgpu_context *ctx, const pkgpu_request *req, double *out, pkgpu_timings *timings,
                            pkgpu_compat *compat, char *err, size_t errlen);

/* ---- multi-GPU: Morton-range partition ---------------------------- */
/* Every rank receives the full request (inputs replicated, so the near-field source halo
 * is implicit) and builds the same tree. Rank r owns a contiguous Morton range of leaves
 * (equal leaf counts; its targets). The upward pass runs over the rank's own leaves; a box
 * whose leaves all belong to one rank (its owner) is then complete there, a box spanning
 * several ranks (a "straddler": the ancestors of the range boundaries, root included) holds
 * a partial sum on each -- the upward chain is linear in the sources.
 * Equivalent-density exchange (with `alltoallv`): one allreduce over the straddlers only,
 * then a halo exchange -- every rank receives, from their owners, the densities of the V-
 * and W-list sources of its own target boxes (need masks from the replicated tree). Without
 * `alltoallv` (NULL): one allreduce of all boxes' densities (round 1's scheme).
 * The small-level int8 M2L run (levels streamed as one launch) is split by modulus when
 * `allgather` is given: each rank computes ceil(nmod / R) moduli of the residue sums for all
 * of the run's columns, gathered before the CRT rebuild.
 * The downward and leaf passes run for the boxes meeting the rank's range; the outputs
 * (each target written by one rank, zeros elsewhere) are summed by a final allreduce so
 * every rank returns the full potentials.
 *   alloc     : device memory the collectives can operate on (e.g. a torch tensor)
 *   allreduce : in-place elementwise sum over ranks of count doubles
 *   alltoallv : send[...] holds nranks consecutive blocks (send_counts[q] doubles for rank q,
 *               q = rank included, count 0); recv receives recv_counts[q] doubles from each q
 *   allgather : buf holds nranks blocks of bytes_per_rank; block `rank` is filled, all are
 *               filled on return
 * The work stream is synchronised before each callback, which must complete (or order its
 * work before any later use of the buffers) before returning. */
typedef void *(*pkgpu_alloc_fn)(void *user, size_t bytes);
typedef int (*pkgpu_allreduce_fn)(void *user, double *device_buf, int64_t count, void *stream);
typedef int (*pkgpu_alltoallv_fn)(void *user, const double *send, const int64_t *send_counts, double *recv,
                                  const int64_t *recv_counts, void *stream);
typedef int (*pkgpu_allgather_fn)(void *user, void *device_buf, int64_t bytes_per_rank, void *stream);
typedef struct {
    int rank, nranks;
    pkgpu_alloc_fn alloc;
    pkgpu_allreduce_fn allreduce;
    void *user;
    pkgpu_alltoallv_fn alltoallv; /* optional */
    pkgpu_allgather_fn allgather; /* optional */
} pkgpu_partition;

pkgpu_status pkgpu_evaluate_partitioned(pkgpu_context *ctx, const pkgpu_request *req, const pkgpu_partition *part,
                                        double *out, pkgpu_timings *timings, pkgpu_compat *compat, char *err,
                                        size_t errlen);

/* ---- periodizing operator (include/pkifmm/periodize.hpp:22-33) -------------------- */
/* load_operator (src/periodize.cpp:231-278): PKM2L magic, header, payload CRC-64/XZ. */
pkgpu_status pkgpu_operator_load(const char *path, pkgpu_operator **op, char *err, size_t errlen);
/* In-memory operator (matrix row-major dim x dim, dim = ks*n) with its provenance. */
pkgpu_status pkgpu_operator_create(int kernel, const pkgpu_setup *setup, int p, const double *matrix, int64_t dim,
                                   pkgpu_operator **op, char *err, size_t errlen);
void pkgpu_operator_free(pkgpu_operator *op);
/* Provenance accessors (kernel, setup, p, dim) for the C++ shim / callers. */
pkgpu_status pkgpu_operator_info(const pkgpu_operator *op, int *kernel, pkgpu_setup *setup, int *p, int64_t *dim,
                                 double *residual_max);
/* Overwrite the provenance (SURVEY §8c config adaptations: SP-x permuted operator,
 * DP-Stokes stand-in). */
pkgpu_status pkgpu_operator_relabel(pkgpu_operator *op, int kernel, const pkgpu_setup *setup);
/* Copy of the matrix (dim*dim doubles). */
pkgpu_status pkgpu_operator_matrix(const pkgpu_operator *op, double *out);
/* CRC-64/XZ (src/periodize.cpp:40-55). */
uint64_t pkgpu_crc64(const void *data, size_t len);

/* Ewald / image-sum parameters (EwaldParams, include/pkifmm/refsum.hpp:21-27). */
typedef struct {
    double xi;           /* 8.0 */
    int real_shells;     /* 2 */
    int wave_cutoff;     /* 64 */
    long long n_images;  /* 1000000 (direct singly periodic sums) */
} pkgpu_ewald;
/* solve_m2l (include/pkifmm/periodize.hpp:42; src/periodize.cpp:57-158) on the GPU: K^{P,F}
 * on the inner root surface by per-pair Ewald / image sums, T = pinv(a_dn) K^{P,F} with
 * the context's downward factors, backward residual gate 1e-11 (gated = 0 skips the gate
 * and records residual_max = -1, the ungated operator of SURVEY §8c cfg 4). Singly
 * periodic along x (cfg 1) is built along z and permuted like the reference's SP-x recipe.
 * Errors: ConfigError for unsupported (kernel, periodicity); RuntimeError past the gate. */
pkgpu_status pkgpu_operator_solve(pkgpu_context *ctx, int kernel, const pkgpu_setup *setup, int p,
                                  const pkgpu_ewald *params, int gated, pkgpu_operator **op, char *err,
                                  size_t errlen);
/* save_operator (include/pkifmm/periodize.hpp:61; src/periodize.cpp:189-229): PKM2L file,
 * same header keys and payload CRC as the reference writes. */
pkgpu_status pkgpu_operator_save(const pkgpu_operator *op, const char *path, char *err, size_t errlen);
/* periodic_block / kpf_block (include/pkifmm/refsum.hpp:68-72): out[(kt i + a)(ks ns) + ks j
 * + b] = K^P(t_i, s_j) (far_only: K^{P,F}); host arrays, xyz interleaved. */
pkgpu_status pkgpu_periodic_block(pkgpu_context *ctx, int kernel, const pkgpu_setup *setup, const pkgpu_ewald *params,
                                  int far_only, const double *targets, int64_t nt, const double *sources, int64_t ns,
                                  double *out, char *err, size_t errlen);
/* oracle_system_eval (include/pkifmm/refsum.hpp:88; src/refsum.cpp:757-770): q_t = sum_s
 * K^P(x_t, y_s) phi_s on the GPU, compatibility checked first (ConfigError). */
pkgpu_status pkgpu_oracle_system_eval(pkgpu_context *ctx, int kernel, const pkgpu_setup *setup,
                                      const pkgpu_ewald *params, const double *sources, int64_t ns,
                                      const double *strengths, const double *targets, int64_t nt, double *out,
                                      char *err, size_t errlen);

/* ---- KIFMM operators (src/fmm.cpp:180-236) --------------------------------------- */
/* Parity mode: inject SVD factors in the reference's layout (SvdFactors,
 * include/pkifmm/linalg.hpp:45-53: u m x k row-major, sigma k, vt k x n row-major) for
 * a_up = K(outer, inner) and a_dn = K(inner, outer). Without injection the context
 * computes them on the device (cuSOLVER gesvd). */
pkgpu_status pkgpu_set_kifmm_factors(pkgpu_context *ctx, int kernel, int p, const double *u_up, const double *s_up,
                                     const double *vt_up, const double *u_dn, const double *s_dn,
                                     const double *vt_dn, char *err, size_t errlen);
/* Read back the factors in use (computing them if needed). Arrays of K*K, K, K*K. */
pkgpu_status pkgpu_get_kifmm_factors(pkgpu_context *ctx, int kernel, int p, double *u_up, double *s_up,
                                     double *vt_up, double *u_dn, double *s_dn, double *vt_dn, char *err,
                                     size_t errlen);
/* Dense kernel matrices used by the translations, for parity checks:
 * which = 0 a_up, 1 a_dn, 2 M2M_o, 3 L2L_o, 4 M2L offset d=(i0,i1,i2), 5 image sum M_img
 * (i0 = periodicity axes bitmask, i1 = ell). out: (kt n) x (ks n) row-major. */
pkgpu_status pkgpu_kifmm_matrix(pkgpu_context *ctx, int kernel, int p, int which, int i0, int i1, int i2,
                                double *out, char *err, size_t errlen);

/* ---- primitives ------------------------------------------------------------------ */
/* kernel_block_apply (src/kernel.cpp:80-129) on the device: out += K((t - shift) - s) rho. */
pkgpu_status pkgpu_kernel_block_apply(pkgpu_context *ctx, int kernel, const double *targets, int64_t nt,
                                      const double *sources, int64_t ns, const double *shift,
                                      const double *density, double *out, int skip_coincident, char *err,
                                      size_t errlen);
/* surface_points (src/geometry.cpp:60-71), bit-exact. */
pkgpu_status pkgpu_surface_points(int p, const double *center, double edge, double *out);

/* The integer tensor-pipe gather-GEMM behind the M2L stage (no reference counterpart:
 * the reference applies M2L as dense FP64 GEMMs, src/fmm.cpp:560-574). Device pointers:
 *   R[t][c][r] += sum_s sum_k A[t][s][r][k] * B[t][row(s, c)][k]   (balanced residues mod m_t)
 * A int8 [nmod][nmat][Ki][Ki], B int8 [nmod][rows_per_mod][Ki], src int32 [nslots][ld_src]
 * (row = src - box0, or zero_row when src < 0), R int32 [nmod][ncols][Ki]; Ki % 128 == 0,
 * ncols % 256 == 0. Exact integer results: the test hook for the kind::i8 kernel. */
pkgpu_status pkgpu_i8_gather_gemm(pkgpu_context *ctx, const int8_t *A, int nmat, const int8_t *B, int rows_per_mod,
                                  int zero_row, int Ki, int nmod, const int32_t *src, int64_t ld_src, int64_t box0,
                                  int nslots, int ncols, int32_t *R, char *err, size_t errlen);
/* The moduli m_t (pairwise coprime, <= 256); returns how many exist. */
int pkgpu_i8_moduli(int32_t *out, int n);

/* ---- tree / lists (debug exports for the bit-exact gates) ------------------------ */
/* FmmTree::FmmTree (src/fmm.cpp:301-356) on the device. */
pkgpu_status pkgpu_tree_build(pkgpu_context *ctx, const double *sources, int64_t ns, const double *targets,
                              int64_t nt, int leaf_capacity, pkgpu_tree **tree, char *err, size_t errlen);
void pkgpu_tree_free(pkgpu_tree *tree);
/* FmmTree::structure_hash (src/fmm.cpp:397-413). */
pkgpu_status pkgpu_tree_info(pkgpu_tree *tree, int64_t *nboxes, int64_t *nleaves, int *depth, uint64_t *hash);
/* Box table in BFS order, 18 int32 per box: level cx cy cz parent leaf nsrc ntrg
 * src_subtree trg_subtree child[8]; leaf point lists in increasing original index. */
pkgpu_status pkgpu_tree_boxes(pkgpu_tree *tree, int32_t *table, int32_t *srcidx, int32_t *trgidx);
/* FmmTree::build_lists (src/fmm.cpp:488-503): which = 'u','v','w','x'. off: nboxes+1
 * int64; ent: 4 int32 per entry (box, sx, sy, sz) — V stores the cell offset d. Call
 * with ent == NULL to get the count in off[nboxes]. */
pkgpu_status pkgpu_tree_lists(pkgpu_tree *tree, const pkgpu_setup *setup, int which, int64_t *off, int32_t *ent,
                              char *err, size_t errlen);

/* ---- synthetic workloads (SURVEY §8d protocol, std::mt19937_64) ------------------ */
/* kind: 0 uniform, 1 clusters, 2 mixed (half uniform, half clusters). Writes n*3
 * points and n*ks strengths (mean-subtracted per component). */
pkgpu_status pkgpu_generate(int kind, int64_t n, int nclusters, double sigma, const int periodic_axes[3], int ks,
                            uint64_t seed, double *points, double *strengths);

#ifdef __cplusplus
}
#endif

#endif /* PKGPU_H */
