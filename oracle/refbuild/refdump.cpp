// refdump — our own driver around the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp compiled into oracle/_ref/libpkifmm_ref.a).
// TEST INFRASTRUCTURE ONLY: it generates golden vectors (trees, lists,
// potentials, SVD factors, periodizing operators) and times the reference's
// CPU evaluate path for the cpu_baseline. The product (libpkgpu.so) never
// links or calls this.
//
// White-box access goes through the reference's own test hook
// `friend struct FmmTreeTestAccess;` (include/pkifmm/fmm.hpp:67).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "pkifmm/fmm.hpp"
#include "pkifmm/periodize.hpp"
#include "pkifmm/refsum.hpp"

extern "C" void openblas_set_num_threads(int n);

namespace pkifmm {
struct FmmTreeTestAccess {
    static const auto &boxes(const FmmTree &t) { return t.boxes_; }
    static void build_lists(FmmTree &t, const PeriodicSetup *s) { t.build_lists(s); }
    static const auto &lists(const FmmTree &t) { return t.lists_; }
};
} // namespace pkifmm

using namespace pkifmm;
using json = nlohmann::json;

namespace {

std::map<std::string, std::string> parse_args(int argc, char **argv, int start) {
    std::map<std::string, std::string> a;
    for (int i = start; i < argc; i++) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) throw std::invalid_argument("bad arg " + k);
        k = k.substr(2);
        if (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0)
            a[k] = argv[++i];
        else
            a[k] = "1";
    }
    return a;
}

std::string get(const std::map<std::string, std::string> &a, const std::string &k, const std::string &def = "") {
    auto it = a.find(k);
    if (it == a.end()) {
        if (def == "__required__") throw std::invalid_argument("missing --" + k);
        return def;
    }
    return it->second;
}

std::vector<double> read_f64(const std::string &path) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) throw std::runtime_error("cannot open " + path);
    const auto sz = f.tellg();
    f.seekg(0);
    std::vector<double> v(static_cast<size_t>(sz) / 8);
    f.read(reinterpret_cast<char *>(v.data()), static_cast<std::streamsize>(v.size() * 8));
    return v;
}

template <class T> void write_bin(const std::string &path, const std::vector<T> &v) {
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    f.write(reinterpret_cast<const char *>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

std::vector<Vec3> to_vec3(const std::vector<double> &x) {
    std::vector<Vec3> p(x.size() / 3);
    for (size_t i = 0; i < p.size(); i++) p[i] = Vec3(x[3 * i], x[3 * i + 1], x[3 * i + 2]);
    return p;
}

PeriodicSetup make_setup(const std::map<std::string, std::string> &a) {
    const Periodicity per = periodicity_from_name(get(a, "per", "none"));
    PeriodicSetup s = PeriodicSetup::make(per, std::stoi(get(a, "ell", "2")));
    const std::string axes = get(a, "axes", "");
    if (!axes.empty() && per != Periodicity::none)
        s.axes = {axes.find('x') != std::string::npos, axes.find('y') != std::string::npos,
                  axes.find('z') != std::string::npos};
    return s;
}

void set_threads(const std::map<std::string, std::string> &a) {
    const int t = std::stoi(get(a, "threads", "0"));
    if (t > 0) {
#ifdef _OPENMP
        omp_set_num_threads(t);
#endif
        openblas_set_num_threads(t);
    }
}

double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

// ---------------------------------------------------------------------------
// seeded synthetic inputs, SURVEY.md §8(d) protocol (std::mt19937_64)
double wrap01(double x) {
    double y = x - std::floor(x);
    if (y >= 1.0) y = 0.0;
    return y;
}
double clip01(double x) { return std::min(std::max(x, 0.0), std::nextafter(1.0, 0.0)); }

int cmd_gen(const std::map<std::string, std::string> &a) {
    const long n = std::stol(get(a, "n", "__required__"));
    const std::string kind = get(a, "kind", "uniform"); // uniform | clusters | mixed
    const int ncl = std::stoi(get(a, "nclusters", "8"));
    const double sigma = std::stod(get(a, "sigma", "0.04"));
    const std::string axes = get(a, "axes", "xyz"); // periodic axes for wrapping clustered points
    const int ks = std::stoi(get(a, "ks", "1"));
    const uint64_t seed = std::stoull(get(a, "seed", "12345"));
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> unif(0.0, 1.0);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::vector<double> pts(static_cast<size_t>(3 * n));
    long n_uniform = kind == "uniform" ? n : (kind == "mixed" ? n / 2 : 0);
    for (long i = 0; i < n_uniform; i++) {
        const double x = unif(rng);
        const double y = unif(rng);
        const double z = unif(rng);
        pts[3 * i] = x, pts[3 * i + 1] = y, pts[3 * i + 2] = z;
    }
    const long n_cl = n - n_uniform;
    if (n_cl > 0) {
        std::vector<double> c(3 * ncl);
        for (int k = 0; k < ncl; k++) {
            const double x = unif(rng);
            const double y = unif(rng);
            const double z = unif(rng);
            c[3 * k] = x, c[3 * k + 1] = y, c[3 * k + 2] = z;
        }
        for (long j = 0; j < n_cl; j++) {
            const int k = static_cast<int>(j % ncl);
            for (int d = 0; d < 3; d++) {
                const double v = c[3 * k + d] + sigma * gauss(rng);
                const bool per = axes.find("xyz"[d]) != std::string::npos;
                pts[3 * (n_uniform + j) + d] = per ? wrap01(v) : clip01(v);
            }
        }
    }
    std::vector<double> str(static_cast<size_t>(ks * n));
    if (ks == 1) {
        std::uniform_real_distribution<double> cu(-1.0, 1.0);
        for (auto &v : str) v = cu(rng);
    } else {
        for (auto &v : str) v = gauss(rng);
    }
    for (int comp = 0; comp < ks; comp++) {
        double s = 0.0;
        for (long i = 0; i < n; i++) s += str[ks * i + comp];
        const double mean = s / static_cast<double>(n);
        for (long i = 0; i < n; i++) str[ks * i + comp] -= mean;
    }
    write_bin(get(a, "out", "__required__") + ".src.f64", pts);
    write_bin(get(a, "out") + ".str.f64", str);
    std::cout << json{{"n", n}, {"kind", kind}}.dump() << "\n";
    return 0;
}

// ---------------------------------------------------------------------------
// tree + lists dump
int cmd_tree(const std::map<std::string, std::string> &a) {
    const auto src = to_vec3(read_f64(get(a, "src", "__required__")));
    const auto trg = a.count("trg") ? to_vec3(read_f64(get(a, "trg"))) : src;
    const int leaf = std::stoi(get(a, "leaf", "1000"));
    const double t0 = now();
    FmmTree tree(src, trg, leaf);
    const double t_tree = now() - t0;
    const auto &boxes = FmmTreeTestAccess::boxes(tree);
    const std::string out = get(a, "out", "");
    json j{{"hash", tree.structure_hash()}, {"boxes", boxes.size()}, {"leaves", tree.leaf_count()},
           {"depth", tree.depth()}, {"t_tree", t_tree}};
    if (!out.empty()) {
        // box table: level cx cy cz parent leaf nsrc ntrg src_subtree trg_subtree child[8]
        std::vector<int32_t> tab, srcl, trgl;
        for (const auto &b : boxes) {
            tab.insert(tab.end(), {b.level, b.cell[0], b.cell[1], b.cell[2], b.parent, b.leaf ? 1 : 0,
                                   (int)b.src.size(), (int)b.trg.size(), b.src_subtree, b.trg_subtree});
            tab.insert(tab.end(), b.child.begin(), b.child.end());
            srcl.insert(srcl.end(), b.src.begin(), b.src.end());
            trgl.insert(trgl.end(), b.trg.begin(), b.trg.end());
        }
        write_bin(out + ".boxes.i32", tab);
        write_bin(out + ".srcidx.i32", srcl);
        write_bin(out + ".trgidx.i32", trgl);
    }
    if (a.count("lists")) {
        const PeriodicSetup s = make_setup(a);
        const double t1 = now();
        FmmTreeTestAccess::build_lists(tree, &s);
        j["t_lists"] = now() - t1;
        const auto &L = FmmTreeTestAccess::lists(tree);
        // CSR per list: entries (box, sx, sy, sz) as int32, shifts integral
        auto dump = [&](const char *name, const auto &lst) {
            std::vector<int32_t> off{0}, ent;
            size_t total = 0;
            for (const auto &v : lst) {
                for (const auto &[c, s] : v) {
                    ent.push_back(c);
                    for (int d = 0; d < 3; d++) ent.push_back(static_cast<int32_t>(s[d]));
                }
                total += v.size();
                off.push_back(static_cast<int32_t>(total));
            }
            if (!out.empty()) {
                write_bin(out + "." + name + ".off.i32", off);
                write_bin(out + "." + name + ".ent.i32", ent);
            }
            j[std::string("n_") + name] = total;
        };
        dump("u", L.u);
        dump("v", L.v);
        dump("w", L.w);
        dump("x", L.x);
    }
    std::cout << j.dump() << "\n";
    return 0;
}

// ---------------------------------------------------------------------------
std::shared_ptr<PeriodizingOperator> load_or_null(const std::map<std::string, std::string> &a) {
    const std::string path = get(a, "op", "");
    if (path.empty()) return nullptr;
    return std::make_shared<PeriodizingOperator>(load_operator(path));
}

int cmd_eval(const std::map<std::string, std::string> &a) {
    set_threads(a);
    EvalRequest req;
    req.kernel = KernelSpec::from_name(get(a, "kernel", "laplace"));
    req.sources = to_vec3(read_f64(get(a, "src", "__required__")));
    req.strengths = read_f64(get(a, "str", "__required__"));
    req.targets = a.count("trg") ? to_vec3(read_f64(get(a, "trg"))) : req.sources;
    req.setup = make_setup(a);
    req.p = std::stoi(get(a, "p", "8"));
    req.leaf_capacity = std::stoi(get(a, "leaf", "1000"));
    req.mode = get(a, "mode", "fmm") == "direct" ? EvalMode::direct : EvalMode::fmm;
    req.force = a.count("force") > 0;
    auto op = load_or_null(a);
    if (op) {
        // config adaptations: relabel the operator provenance
        // to the request setup (SP-x permuted operator, DP-Stokes stand-in)
        if (a.count("relabel")) {
            op->setup = req.setup;
            op->kernel = req.kernel;
        }
        req.op = op.get();
    }
    const int repeat = std::stoi(get(a, "repeat", "1"));
    const std::string out = get(a, "out", "");
    json runs = json::array();
    EvalResult res;
    if (a.count("near-only")) {
        // near field only (FmmTree::eval_near_field / eval_free_space) + root density
        for (int r = 0; r < repeat; r++) {
            const double t0 = now();
            FmmTree tree(req.sources, req.targets, req.leaf_capacity);
            const double t1 = now();
            res.potentials = req.setup.periodicity != Periodicity::none
                                 ? tree.eval_near_field(req.kernel, req.p, req.strengths, req.setup)
                                 : tree.eval_free_space(req.kernel, req.p, req.strengths);
            const double t2 = now();
            runs.push_back({{"tree", t1 - t0}, {"near", t2 - t1}});
            if (r == repeat - 1 && !out.empty()) {
                const auto up = tree.root_upward_density(req.kernel, req.p, req.strengths);
                write_bin(out + ".phiup0.f64", up.values);
            }
        }
    } else {
        for (int r = 0; r < repeat; r++) {
            const double t0 = now();
            res = evaluate(req);
            const double wall = now() - t0;
            runs.push_back({{"tree", res.timings.tree},
                            {"near", res.timings.near},
                            {"m2l_apply", res.timings.m2l_apply},
                            {"far", res.timings.far},
                            {"wall", wall}});
        }
        if (!out.empty() && req.mode == EvalMode::fmm) {
            FmmTree tree(req.sources, req.targets, req.leaf_capacity);
            const auto up = tree.root_upward_density(req.kernel, req.p, req.strengths);
            write_bin(out + ".phiup0.f64", up.values);
        }
    }
    if (!out.empty()) write_bin(out + ".pot.f64", res.potentials);
    int threads = 1;
#ifdef _OPENMP
    threads = omp_get_max_threads();
#endif
    std::cout << json{{"runs", runs},
                      {"n_targets", req.targets.size()},
                      {"threads", threads},
                      {"compat_ok", res.compat.ok},
                      {"compat_residual", res.compat.residual}}
                     .dump()
              << "\n";
    return 0;
}

// truth: the reference's own ground-truth evaluator (pairwise Ewald / direct sums,
// oracle_system_eval, include/pkifmm/refsum.hpp:88) at a stride sample of `ntrg` source
// points (index i * (N / ntrg)), for the SURVEY §8(c)(iii) accuracy check
int cmd_truth(const std::map<std::string, std::string> &a) {
    set_threads(a);
    const KernelSpec kernel = KernelSpec::from_name(get(a, "kernel", "laplace"));
    const auto src = to_vec3(read_f64(get(a, "src", "__required__")));
    const auto str = read_f64(get(a, "str", "__required__"));
    const PeriodicSetup setup = make_setup(a);
    const int ntrg = std::stoi(get(a, "ntrg", "64"));
    const size_t stride = std::max<size_t>(1, src.size() / ntrg);
    std::vector<Vec3> trg;
    for (int i = 0; i < ntrg && i * stride < src.size(); i++) trg.push_back(src[i * stride]);
    const double t0 = now();
    const auto spec = make_periodic_spec(kernel, setup);
    const auto q = oracle_system_eval(spec, src, str, trg);
    write_bin(get(a, "out", "__required__") + ".truth.f64", q);
    std::cout << json{{"ntrg", trg.size()}, {"stride", stride}, {"seconds", now() - t0}}.dump() << "\n";
    return 0;
}

// ---------------------------------------------------------------------------
// operators: SVD factors and periodizing operator
void dump_factors(const SvdFactors &f, const std::string &out) {
    write_bin(out + ".u.f64", f.u.data);
    write_bin(out + ".s.f64", f.sigma);
    write_bin(out + ".vt.f64", f.vt.data);
}

int cmd_factors(const std::map<std::string, std::string> &a) {
    set_threads(a);
    const KernelSpec k = KernelSpec::from_name(get(a, "kernel", "laplace"));
    const int p = std::stoi(get(a, "p", "8"));
    const auto ops = kifmm_operators(k, p);
    const std::string out = get(a, "out", "__required__");
    dump_factors(upward_factors(*ops), out + ".aup");
    dump_factors(downward_factors(*ops), out + ".adn");
    std::cout << json{{"dim", upward_factors(*ops).sigma.size()},
                      {"eps_up", upward_factors(*ops).eps_svd},
                      {"eps_dn", downward_factors(*ops).eps_svd},
                      {"rank_up", upward_factors(*ops).numerical_rank},
                      {"rank_dn", downward_factors(*ops).numerical_rank}}
                     .dump()
              << "\n";
    return 0;
}

// surface index map of the axis permutation Q(x,y,z) = (y,z,x): pi[i] = index
// of grid point (g_y, g_z, g_x); used to turn an SP-z operator into SP-x
// (cfg 1 adaptation)
std::vector<int> sp_x_perm(int p) {
    const auto grid = surface_grid_indices(p);
    std::map<std::array<int, 3>, int> lookup;
    for (size_t i = 0; i < grid.size(); i++) lookup[{grid[i][0], grid[i][1], grid[i][2]}] = static_cast<int>(i);
    std::vector<int> pi(grid.size());
    for (size_t i = 0; i < grid.size(); i++) pi[i] = lookup.at({grid[i][1], grid[i][2], grid[i][0]});
    return pi;
}

int cmd_precompute(const std::map<std::string, std::string> &a) {
    set_threads(a);
    const KernelSpec k = KernelSpec::from_name(get(a, "kernel", "laplace"));
    const int p = std::stoi(get(a, "p", "8"));
    PeriodicSetup setup = make_setup(a);
    const bool spx = a.count("spx") > 0;
    if (spx) setup = PeriodicSetup::make(Periodicity::sp, setup.ell); // build along z, permute below
    EwaldParams params;
    if (a.count("n-images")) params.n_images = std::stoll(get(a, "n-images"));
    const PeriodicKernelSpec spec = make_periodic_spec(k, setup, params);
    const auto ops = kifmm_operators(k, p);
    const double t0 = now();
    PeriodizingOperator op;
    if (a.count("ungated")) {
        // public API path that bypasses the 1e-11 residual gate (cfg 4)
        const DenseMatrix q = assemble_kpf_matrix(spec, p);
        op.matrix = pinv_apply_block(downward_factors(*ops), q);
        op.kernel = k;
        op.setup = setup;
        op.p = p;
        op.method = spec.method;
        op.params = spec.params;
        op.residual_max = -1.0;
    } else {
        op = solve_m2l(spec, p, downward_factors(*ops));
    }
    if (spx) {
        if (k.ks != 1) throw std::invalid_argument("spx permutation implemented for scalar kernels only");
        const auto pi = sp_x_perm(p);
        DenseMatrix t(op.matrix.rows, op.matrix.cols);
        for (int i = 0; i < t.rows; i++)
            for (int j = 0; j < t.cols; j++) t(i, j) = op.matrix(pi[i], pi[j]);
        op.matrix = std::move(t);
        op.setup.axes = {true, false, false};
    }
    const double dt = now() - t0;
    save_operator(op, get(a, "out", "__required__"));
    std::cout << json{{"seconds", dt}, {"residual", op.residual_max}, {"dim", op.matrix.rows}}.dump() << "\n";
    return 0;
}

// kernel_block_apply golden vectors (pair-sum primitive, src/kernel.cpp:80-129)
int cmd_pairs(const std::map<std::string, std::string> &a) {
    const KernelSpec k = KernelSpec::from_name(get(a, "kernel", "laplace"));
    const auto trg = to_vec3(read_f64(get(a, "trg", "__required__")));
    const auto src = to_vec3(read_f64(get(a, "src", "__required__")));
    const auto den = read_f64(get(a, "den", "__required__"));
    const auto sh = read_f64(get(a, "shift", "__required__"));
    std::vector<double> out(static_cast<size_t>(k.kt) * trg.size(), 0.0);
    std::string err;
    try {
        kernel_block_apply(k, trg, src, Vec3(sh[0], sh[1], sh[2]), den, out, a.count("skip") > 0);
    } catch (const std::exception &e) {
        err = e.what();
    }
    write_bin(get(a, "out", "__required__") + ".pot.f64", out);
    std::cout << json{{"error", err}}.dump() << "\n";
    return 0;
}

// dense kernel matrices (kernel_block) between surfaces, for operator parity
int cmd_kblock(const std::map<std::string, std::string> &a) {
    const KernelSpec k = KernelSpec::from_name(get(a, "kernel", "laplace"));
    const auto trg = to_vec3(read_f64(get(a, "trg", "__required__")));
    const auto src = to_vec3(read_f64(get(a, "src", "__required__")));
    const DenseMatrix m = kernel_block(k, trg, src);
    write_bin(get(a, "out", "__required__") + ".kb.f64", m.data);
    std::cout << json{{"rows", m.rows}, {"cols", m.cols}}.dump() << "\n";
    return 0;
}

int cmd_surface(const std::map<std::string, std::string> &a) {
    const int p = std::stoi(get(a, "p", "8"));
    const double cx = std::stod(get(a, "cx", "0.5")), cy = std::stod(get(a, "cy", "0.5")),
                 cz = std::stod(get(a, "cz", "0.5"));
    const double edge = std::stod(get(a, "edge", "1.05"));
    const auto pts = surface_points(p, Vec3(cx, cy, cz), edge);
    std::vector<double> v;
    for (const auto &x : pts) v.insert(v.end(), {x[0], x[1], x[2]});
    write_bin(get(a, "out", "__required__") + ".surf.f64", v);
    std::cout << json{{"n", pts.size()}}.dump() << "\n";
    return 0;
}

} // namespace

int main(int argc, char **argv) {
    if (argc < 2) {
        std::cerr << "usage: refdump gen|tree|eval|factors|precompute|pairs|kblock|surface --opts\n";
        return 1;
    }
    try {
        const std::string cmd = argv[1];
        const auto a = parse_args(argc, argv, 2);
        if (cmd == "gen") return cmd_gen(a);
        if (cmd == "tree") return cmd_tree(a);
        if (cmd == "eval") return cmd_eval(a);
        if (cmd == "factors") return cmd_factors(a);
        if (cmd == "precompute") return cmd_precompute(a);
        if (cmd == "pairs") return cmd_pairs(a);
        if (cmd == "kblock") return cmd_kblock(a);
        if (cmd == "surface") return cmd_surface(a);
        if (cmd == "truth") return cmd_truth(a);
        std::cerr << "unknown command " << cmd << "\n";
        return 1;
    } catch (const ConfigError &e) {
        std::cout << json{{"exception", "ConfigError"}, {"what", e.what()}}.dump() << "\n";
        return 3;
    } catch (const std::invalid_argument &e) {
        std::cout << json{{"exception", "invalid_argument"}, {"what", e.what()}}.dump() << "\n";
        return 3;
    } catch (const std::runtime_error &e) {
        std::cout << json{{"exception", "runtime_error"}, {"what", e.what()}}.dump() << "\n";
        return 3;
    }
}
