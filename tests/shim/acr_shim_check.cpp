// Compile-and-run check of the reference-side C++ shim of INTEGRATION.md §2.
//
// The shim a maintainer adds to /root/reference/proj/core/src/acr.cpp is written against the
// reference's own types (BlockTridiagonalSystem, AcrConfig, the errors.hpp exception classes,
// Eigen vectors).  Eigen is not available in this image, so those types are restated here as
// minimal stand-ins with the same member names (core/include/acr/block.hpp:38-101,
// acr.hpp:15-23, errors.hpp:10-60); the shim body below is the INTEGRATION.md code with
// Eigen::VectorXd replaced by std::vector<double>.  It is compiled against include/acrgpu.h
// and linked with libacrgpu.so by tests/test_boundary.py (CPU) and run on the B200 by
// tests/test_gpu_shim.py:
//   acr_shim_check            -> factors poisson(n=8), solves, prints "shim ok <residual> <largest rank>"
//   acr_shim_check singular   -> must raise acr::SingularBlockError(level 0, plane 2)
#include <cmath>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "acrgpu.h"

namespace acr {
// ---- stand-ins of the reference types the shim touches
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct DimensionError : Error { int plane; DimensionError(const std::string& m, int p = -1) : Error(m), plane(p) {} };
struct SingularBlockError : Error {
    int level, plane;
    SingularBlockError(const std::string& m, int l, int p) : Error(m), level(l), plane(p) {}
};
struct LeafMemoryError : Error { using Error::Error; };
struct UsageError : Error { using Error::Error; };
struct IndefiniteError : Error { using Error::Error; };
struct DivergenceError : Error { using Error::Error; };
enum class Admissibility { Standard, Weak };
struct AcrConfig {  // acr.hpp:15-23 (H-matrix mode fields)
    double eps = 1e-3, eta = 2.0;
    int leaf_size = 32;
    Admissibility admissibility = Admissibility::Standard;
    int stop_planes = 1;
    long leaf_memory_cap = 2L << 30;
};
struct Entry { int row, col; double value; };
struct Point { double x, y; };
struct PlaneBlock {  // block.hpp:38-60
    std::vector<Entry> e;
    std::vector<Point> pts;
    const std::vector<Entry>& entries() const { return e; }
    const std::vector<Point>& coords() const { return pts; }
};
struct BlockTridiagonalSystem {  // block.hpp:62-101
    int n = 0, d = 0;
    std::vector<PlaneBlock> Dv, Ev, Fv;  // Ev[j-1] = E(j), Fv[j] = F(j)
    int plane_count() const { return n; }
    int plane_dim() const { return d; }
    const PlaneBlock& D(int j) const { return Dv[j]; }
    const PlaneBlock& E(int j) const { return Ev[j - 1]; }
    const PlaneBlock& F(int j) const { return Fv[j]; }
};
struct PlaneVector { std::vector<double> v; int plane; };

// ---- the shim
namespace {
[[noreturn]] void rethrow(const acrgpu_error& e) {
    switch (e.code) {
        case ACRGPU_E_DIMENSION: throw DimensionError(e.msg, e.plane);
        case ACRGPU_E_SINGULAR:  throw SingularBlockError(e.msg, e.level, e.plane);
        case ACRGPU_E_LEAFMEM:   throw LeafMemoryError(e.msg);
        case ACRGPU_E_USAGE:     throw UsageError(e.msg);
        case ACRGPU_E_INDEFINITE: throw IndefiniteError(e.msg);
        case ACRGPU_E_DIVERGENCE: throw DivergenceError(e.msg);
        default:                 throw Error(e.msg);
    }
}
acrgpu_ctx* gpu_ctx() {
    static acrgpu_ctx* ctx = [] { acrgpu_ctx* c; acrgpu_error e;
        if (acrgpu_ctx_create(-1, &c, &e)) rethrow(e); return c; }();
    return ctx;
}
}  // namespace

struct GpuFactorization {
    std::shared_ptr<acrgpu_fact> f;
    int n, d;
    static GpuFactorization make(const BlockTridiagonalSystem& s, const AcrConfig& c) {
        const int n = s.plane_count(), d = s.plane_dim();
        std::vector<double> xy; for (auto& p : s.D(0).coords()) { xy.push_back(p.x); xy.push_back(p.y); }
        std::vector<long> off{0}; std::vector<int> r, cc; std::vector<double> v;
        auto put = [&](const PlaneBlock& b) { for (auto& e : b.entries()) { r.push_back(e.row); cc.push_back(e.col); v.push_back(e.value); }
                                              off.push_back((long)v.size()); };
        for (int j = 0; j < n; ++j) put(s.D(j));
        for (int j = 1; j < n; ++j) put(s.E(j));
        for (int j = 0; j + 1 < n; ++j) put(s.F(j));
        acrgpu_system sys{n, d, xy.data(), off.data(), r.data(), cc.data(), v.data()};
        acrgpu_config cfg{c.eps, c.eta, c.leaf_size, c.admissibility == Admissibility::Weak,
                          c.stop_planes, c.leaf_memory_cap, 0};
        acrgpu_fact* f; acrgpu_error e;
        if (acrgpu_factor(gpu_ctx(), &sys, &cfg, &f, &e)) rethrow(e);
        return {std::shared_ptr<acrgpu_fact>(f, acrgpu_factor_destroy), n, d};
    }
    std::vector<PlaneVector> solve(const std::vector<std::vector<double>>& rhs) const {
        if ((int)rhs.size() != n) throw DimensionError("solve: plane count mismatch");
        std::vector<double> in((size_t)n * d), out(in.size());
        for (int j = 0; j < n; ++j) {
            if ((int)rhs[j].size() != d) throw DimensionError("solve: plane dimension mismatch", j);
            std::copy(rhs[j].begin(), rhs[j].end(), in.begin() + (size_t)j * d);
        }
        acrgpu_error e;
        if (acrgpu_solve(f.get(), 1, in.data(), out.data(), &e)) rethrow(e);
        std::vector<PlaneVector> u(n);
        for (int j = 0; j < n; ++j) u[j] = {std::vector<double>(out.begin() + (size_t)j * d, out.begin() + (size_t)(j + 1) * d), j};
        return u;
    }
    long factor_bytes() const { acrgpu_rankstats s; acrgpu_stats(f.get(), &s); return s.factor_bytes; }
    int largest_rank() const { acrgpu_rankstats s; acrgpu_stats(f.get(), &s); return s.largest_rank; }
};
}  // namespace acr

// assemble_poisson(n) (discretize.cpp:46-71): h^2-scaled 7-point Laplacian, D = 5-point in-plane
// stencil with centre 6, E = F = -I; coordinates of the plane grid.
static acr::BlockTridiagonalSystem poisson(int n) {
    acr::BlockTridiagonalSystem s;
    s.n = n;
    s.d = n * n;
    acr::PlaneBlock D, I;
    for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) {
            const int i = y * n + x;
            D.pts.push_back({(x + 1.0) / (n + 1), (y + 1.0) / (n + 1)});
            if (y > 0) D.e.push_back({i, i - n, -1.0});
            if (x > 0) D.e.push_back({i, i - 1, -1.0});
            D.e.push_back({i, i, 6.0});
            if (x + 1 < n) D.e.push_back({i, i + 1, -1.0});
            if (y + 1 < n) D.e.push_back({i, i + n, -1.0});
            I.e.push_back({i, i, -1.0});
        }
    I.pts = D.pts;
    s.Dv.assign(n, D);
    s.Ev.assign(n - 1, I);
    s.Fv.assign(n - 1, I);
    return s;
}

int main(int argc, char** argv) {
    const bool singular = argc > 1 && std::string(argv[1]) == "singular";
    acr::AcrConfig cfg;
    cfg.eps = 1e-6;
    cfg.leaf_size = 16;
    if (singular) {  // test_acr.cpp:223-241: D(2) = 0 -> SingularBlockError at level 0, plane 2
        acr::BlockTridiagonalSystem s = poisson(4);
        s.Dv[2].e.clear();
        s.Ev.assign(3, {});
        s.Fv.assign(3, {});
        try {
            acr::GpuFactorization::make(s, cfg);
        } catch (const acr::SingularBlockError& e) {
            std::printf("shim singular ok level %d plane %d\n", e.level, e.plane);
            return (e.level == 0 && e.plane == 2) ? 0 : 2;
        }
        std::printf("shim: no SingularBlockError\n");
        return 1;
    }
    const int n = 8;
    acr::BlockTridiagonalSystem s = poisson(n);
    acr::GpuFactorization f = acr::GpuFactorization::make(s, cfg);
    std::vector<std::vector<double>> rhs(n, std::vector<double>(n * n));
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n * n; ++i) rhs[j][i] = std::sin(0.37 * (j * n * n + i) + 1.0);
    const std::vector<acr::PlaneVector> u = f.solve(rhs);
    // relative residual ||f - A u|| / ||f|| (block.cpp:109-123)
    double rn = 0, fn = 0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n * n; ++i) {
            double a = 0;
            for (auto& e : s.D(j).entries()) if (e.row == i) a += e.value * u[j].v[e.col];
            if (j > 0) a -= u[j - 1].v[i];
            if (j + 1 < n) a -= u[j + 1].v[i];
            rn += (rhs[j][i] - a) * (rhs[j][i] - a);
            fn += rhs[j][i] * rhs[j][i];
        }
    const double res = std::sqrt(rn / fn);
    std::printf("shim ok %.3e %d %ld\n", res, f.largest_rank(), f.factor_bytes());
    try {
        f.solve(std::vector<std::vector<double>>(n - 1, std::vector<double>(n * n)));
        return 3;
    } catch (const acr::DimensionError&) {
    }
    return res < 1e-5 ? 0 : 4;
}
