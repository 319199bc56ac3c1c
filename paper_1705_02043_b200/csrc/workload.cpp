// Synthetic workload generator (pkgpu_generate): the SURVEY.md §8(d) input protocol.
// Compiled with -march=x86-64-v3 like the reference build, because libstdc++'s
// normal_distribution (Marsaglia polar) rounds differently once FMA contraction is on
// and the generated forces must match the oracle's bit for bit.
#include <algorithm>
#include <cmath>
#include <random>
#include <stdexcept>
#include <vector>

#include "../../include/pkgpu.h"

extern "C" {

pkgpu_status pkgpu_generate(int kind, int64_t n, int nclusters, double sigma, const int periodic_axes[3], int ks,
                            uint64_t seed, double *points, double *strengths) {
    // std::mt19937_64(seed); positions first (uniform part, then
    // cluster centres, then clustered points i mod K with sigma * N(0,1) per axis,
    // wrapped on periodic axes, clipped to [0, nextafter(1,0)] otherwise), then
    // strengths (Laplace U(-1,1), Stokes N(0,1)), mean-subtracted per component.
    try {
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> unif(0.0, 1.0);
        std::normal_distribution<double> gauss(0.0, 1.0);
        const int64_t nu = kind == 0 ? n : (kind == 2 ? n / 2 : 0);
        for (int64_t i = 0; i < nu; i++) {
            const double x = unif(rng);
            const double y = unif(rng);
            const double z = unif(rng);
            points[3 * i] = x, points[3 * i + 1] = y, points[3 * i + 2] = z;
        }
        if (n > nu) {
            if (nclusters < 1) throw std::invalid_argument("generate: nclusters must be positive");
            std::vector<double> c(3 * nclusters);
            for (int k = 0; k < nclusters; k++) {
                const double x = unif(rng);
                const double y = unif(rng);
                const double z = unif(rng);
                c[3 * k] = x, c[3 * k + 1] = y, c[3 * k + 2] = z;
            }
            for (int64_t j = 0; j < n - nu; j++) {
                const int k = static_cast<int>(j % nclusters);
                for (int d = 0; d < 3; d++) {
                    const double v = c[3 * k + d] + sigma * gauss(rng);
                    double w;
                    if (periodic_axes[d]) {
                        w = v - std::floor(v);
                        if (w >= 1.0) w = 0.0;
                    } else {
                        w = std::min(std::max(v, 0.0), std::nextafter(1.0, 0.0));
                    }
                    points[3 * (nu + j) + d] = w;
                }
            }
        }
        if (ks == 1) {
            std::uniform_real_distribution<double> cu(-1.0, 1.0);
            for (int64_t i = 0; i < n; i++) strengths[i] = cu(rng);
        } else {
            for (int64_t i = 0; i < ks * n; i++) strengths[i] = gauss(rng);
        }
        for (int a = 0; a < ks; a++) {
            double s = 0.0;
            for (int64_t i = 0; i < n; i++) s += strengths[ks * i + a];
            const double mean = s / static_cast<double>(n);
            for (int64_t i = 0; i < n; i++) strengths[ks * i + a] -= mean;
        }
        return PKGPU_OK;
    } catch (const std::exception &) {
        return PKGPU_INVALID_ARGUMENT;
    }
}


} // extern "C"
