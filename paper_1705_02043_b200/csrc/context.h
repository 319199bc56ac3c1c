// Context and operator objects behind the C ABI handles.
#pragma once

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/pkgpu.h"
#include "operators.h"
#include "tree.h"

struct pkgpu_operator {
    int kernel = 0;
    pkgpu_setup setup{};
    int p = 0;
    int64_t dim = 0;
    std::vector<double> matrix; // dim x dim row-major (the PKM2L payload)
    int method = 0;
    double residual_max = 0.0;
    uint64_t crc = 0;
    double xi = 8.0;             // EwaldParams of the provenance (save_operator header)
    int real_shells = 2, wave_cutoff = 64;
    long long n_images = 1000000;
    std::string created;
    // device copies, uploaded lazily, one per device
    mutable std::mutex mtx;
    mutable std::map<int, double *> d_matrix;
    ~pkgpu_operator();
    const double *device_matrix(int device, cudaStream_t st) const;
};

struct pkgpu_context {
    int device = 0;
    int num_sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t aux_stream = nullptr;          // list building beside the upward pass (evaluate.cu)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // lattice levels' M2L queued from their pinv_up on (evaluate.cu): the deepest level on
    // aux2_stream (lowest priority), the coarser ones on aux3_stream (between it and the work
    // stream); per level a fork / join event pair and a workspace
    cudaStream_t aux2_stream = nullptr, aux3_stream = nullptr;
    cudaEvent_t ev_lat_fork[pkgpu::kMaxLevels + 1] = {}, ev_lat_join[pkgpu::kMaxLevels + 1] = {};
    pkgpu::Workspace ws_lat[pkgpu::kMaxLevels + 1];
    int *h_layout = nullptr;                    // pinned staging of build_layout's small tables (evaluate.cu)
    cudaEvent_t ev_user = nullptr;              // hand-over between a caller's stream and own_stream (evaluate.cu)
    int64_t launches = 0;
    std::mutex mtx; // calls on one context are serialised (the reference evaluate is reentrant per call)
    pkgpu::OperatorCache ops;
    pkgpu::DeviceTree tree;
    pkgpu::DeviceLists lists;
    pkgpu::Workspace ws;
    cudaEvent_t ev[6]{};
    // per-stage profiling (pkgpu_context_stage_stats)
    struct StageStat {
        double seconds = 0, units = 0, flops = 0;
        int64_t launches = 0;
    };
    bool profiling = false;
    pkgpu::I8Settings i8 = pkgpu::i8_settings(); // M2L arithmetic path (pkgpu_context_set_m2l)
    std::map<std::string, StageStat> stats;
    std::vector<cudaEvent_t> evpool;
};

struct pkgpu_tree {
    pkgpu_context *ctx = nullptr;
    pkgpu::DeviceTree tree;
    std::vector<int32_t> table, srcidx, trgidx;
    uint64_t hash = 0;
    bool exported = false;
};

namespace pkgpu {

void evaluate(pkgpu_context &ctx, const pkgpu_request &req, double *out, pkgpu_timings *timings,
              pkgpu_compat *compat, const pkgpu_partition *part = nullptr);

void kernel_block_apply_device(pkgpu_context &ctx, int kernel, const double *targets, int64_t nt,
                               const double *sources, int64_t ns, const double *shift, const double *density,
                               double *out, int skip);

} // namespace pkgpu
