// dropin_tests.cpp -- the reference's hot-path test cases, re-hosted against
// the drop-in headers (include/latsum/*.hpp) that run on the B200. Each case
// cites the reference test it mirrors (proj/tests/*.cpp). Build:
//   g++ -std=c++20 -O2 -Iinclude -Iinclude/eigen_compat tests/cpp/dropin_tests.cpp
//       -Lpaper_1405_2270_b200 -llatsum_cuda -Wl,-rpath,<repo>/paper_1405_2270_b200
#include <unistd.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <functional>
#include <limits>
#include <random>

#include "latsum/latsum.hpp"
#include "minitest.hpp"

using namespace latsum;

namespace {

// Scalar-loop oracle independent of the expansion kernel (test_support.hpp:13-25).
DenseTensor3 scalar_oracle(const CanonicalTensor3& t) {
    DenseTensor3 out(t.dim(0), t.dim(1), t.dim(2));
    for (Index k = 0; k < t.dim(2); ++k)
        for (Index j = 0; j < t.dim(1); ++j)
            for (Index i = 0; i < t.dim(0); ++i) {
                double s = 0.0;
                for (Index q = 0; q < t.rank(); ++q)
                    s += t.weights()[q] * t.factor(0)(i, q) * t.factor(1)(j, q) * t.factor(2)(k, q);
                out(i, j, k) = s;
            }
    return out;
}

double max_abs(const DenseTensor3& d) {
    double m = 0.0;
    for (Index e = 0; e < d.size(); ++e) m = std::max(m, std::abs(d.data()[e]));
    return m;
}

double rel_diff(const DenseTensor3& got, const DenseTensor3& want) {
    return max_norm_diff(got, want) / std::max(max_abs(want), 1e-300);
}

CanonicalTensor3 random_tensor(std::mt19937& gen, const Dims3& dims, Index rank) {
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::array<Matrix, 3> f;
    for (int l = 0; l < 3; ++l) {
        f[l].resize(dims[l], rank);
        for (Index q = 0; q < rank; ++q)
            for (Index i = 0; i < dims[l]; ++i) f[l](i, q) = u(gen);
    }
    Vector w(rank);
    for (Index q = 0; q < rank; ++q) w[q] = u(gen);
    return CanonicalTensor3(std::move(f), std::move(w));
}

Dims3 random_dims(std::mt19937& gen, Index lo = 2, Index hi = 8) {
    std::uniform_int_distribution<Index> d(lo, hi);
    return {d(gen), d(gen), d(gen)};
}

CanonicalTensor3 constant_tensor(const Dims3& dims, double weight) {
    std::array<Matrix, 3> f{Matrix::Ones(dims[0], 1), Matrix::Ones(dims[1], 1), Matrix::Ones(dims[2], 1)};
    Vector w(1);
    w[0] = weight;
    return CanonicalTensor3(std::move(f), std::move(w));
}

LatticeSpec make_spec(std::array<Index, 3> L, Index n, double b, std::vector<Charge> charges) {
    LatticeSpec spec;
    spec.L = L;
    spec.unit = GridSpec{b, n};
    spec.charges = std::move(charges);
    return spec;
}

// Exponential-sum kernel at exact offsets, explicit loops (test_lattice.cpp:16-54).
double physical_potential(const LatticeSpec& spec, const QuadratureRule& rule, const std::array<Index, 3>& idx,
                          bool periodic) {
    const double h = spec.unit.h(), b = spec.unit.b;
    const Dims3 N = spec.target_dims();
    double total = 0.0;
    for (const Charge& c : spec.charges)
        for (Index k1 = 0; k1 < spec.L[0]; ++k1)
            for (Index k2 = 0; k2 < spec.L[1]; ++k2)
                for (Index k3 = 0; k3 < spec.L[2]; ++k3) {
                    const Index cell[3] = {k1, k2, k3};
                    double d2 = 0.0;
                    for (int l = 0; l < 3; ++l) {
                        const Index off = periodic ? (spec.L[l] / 2) * spec.unit.n : 0;
                        const double x = (static_cast<double>(idx[l] + off) + 0.5 - static_cast<double>(N[l]) / 2.0) * h;
                        const double y = -static_cast<double>(spec.L[l]) * b / 2.0 + static_cast<double>(cell[l]) * b +
                                         c.pos[l] + b / 2.0;
                        d2 += (x - y) * (x - y);
                    }
                    double kern = 0.0;
                    for (Index q = 0; q < rule.node_count(); ++q)
                        kern += rule.weights[q] * std::exp(-rule.exponents[q] * rule.exponents[q] * d2);
                    total += c.Z * kern;
                }
    return total;
}

double simpson(const std::function<double(double)>& f, double a, double b) {
    std::function<double(double, double, double, double, double, double, double, int)> rec =
        [&](double lo, double hi, double flo, double fm, double fhi, double whole, double tol, int depth) {
            const double m = 0.5 * (lo + hi), lm = 0.5 * (lo + m), rm = 0.5 * (m + hi);
            const double flm = f(lm), frm = f(rm);
            const double left = (m - lo) / 6.0 * (flo + 4.0 * flm + fm);
            const double right = (hi - m) / 6.0 * (fm + 4.0 * frm + fhi);
            if (depth <= 0 || std::abs(left + right - whole) < 15.0 * tol)
                return left + right + (left + right - whole) / 15.0;
            return rec(lo, m, flo, flm, fm, left, 0.5 * tol, depth - 1) + rec(m, hi, fm, frm, fhi, right, 0.5 * tol, depth - 1);
        };
    const double m = 0.5 * (a + b);
    const double fa = f(a), fm = f(m), fb = f(b);
    return rec(a, b, fa, fm, fb, (b - a) / 6.0 * (fa + 4.0 * fm + fb), 1e-14, 40);
}

}  // namespace

// ------------------------------------------------------------------ grid / quadrature
TEST(Grid, ValidatesAndComputesMidpoints) {  // grid.hpp:21-36
    EXPECT_THROW(GridSpec(2.0, 3), validation_error);
    EXPECT_THROW(GridSpec(-1.0, 4), validation_error);
    GridSpec g(2.0, 8);
    EXPECT_EQ(g.h(), 0.25);
    EXPECT_EQ(g.midpoint(0), -0.875);
    EXPECT_EQ(g.midpoint(7), 0.875);
}

TEST(Tolerance, DefaultBandAndValidation) {  // test_newton.cpp:230-238
    GridSpec grid{4.0, 16};
    KernelTolerance tol = default_tolerance(grid, 1e-5);
    EXPECT_EQ(tol.a_min, grid.h());
    EXPECT_EQ(tol.a_max, std::sqrt(3.0) * grid.b);
    EXPECT_THROW((KernelTolerance{0.1, 2.0, 1.0}.validate()), validation_error);
    EXPECT_THROW((KernelTolerance{2.0, 0.5, 1.0}.validate()), validation_error);
}

TEST(SincQuadrature, NodeLayoutAndPositivity) {  // test_newton.cpp:98-113
    QuadratureRule rule = sinc_quadrature(1e-6, 0.01, 10.0, 20, 1.0);
    ASSERT_EQ(rule.node_count(), 41);
    EXPECT_GT(rule.step, 0.0);
    for (Index j = 0; j < rule.node_count(); ++j) {
        EXPECT_GT(rule.weights[j], 0.0);
        EXPECT_GE(rule.exponents[j], 0.0);
        if (j > 0) {
            EXPECT_GT(rule.nodes[j], rule.nodes[j - 1]);
            EXPECT_GT(rule.exponents[j], rule.exponents[j - 1]);
        }
    }
    EXPECT_THROW(sinc_quadrature(1e-6, 0.01, 10.0, 0, 1.0), validation_error);
    EXPECT_THROW(sinc_quadrature(0.0, 0.01, 10.0, 5, 1.0), validation_error);
    EXPECT_THROW(sinc_quadrature(1e-6, 1.0, 0.5, 5, 1.0), validation_error);
}

TEST(SincQuadrature, ApproximatesInverseRadius) {  // test_newton.cpp:115-123
    const double a_min = 0.05, a_max = 4.0, eps = 1e-6;
    QuadratureRule rule = sinc_quadrature(eps, a_min, a_max, 40, 2.0);
    for (int i = 0; i <= 50; ++i) {
        const double r = a_min * std::pow(a_max / a_min, i / 50.0);
        EXPECT_LT(std::abs(quadrature_value(rule, r) * r - 1.0), eps);
    }
}

// ------------------------------------------------------------------ generator (GPU)
TEST(GaussianMoments, ZeroExponentGivesCellWidths) {  // test_newton.cpp:32-40
    GridSpec grid{4.0, 8};
    Vector v = gaussian_moment_vector(grid, 0.0, false);
    ASSERT_EQ(v.size(), 8);
    for (Index i = 0; i < 8; ++i) EXPECT_EQ(v[i], grid.h());
    Vector d = gaussian_moment_vector(grid, 0.0, true);
    ASSERT_EQ(d.size(), 16);
    for (Index i = 0; i < 16; ++i) EXPECT_EQ(d[i], grid.h());
}

TEST(GaussianMoments, UnitCellMatchesErfIntegral) {  // test_newton.cpp:42-52
    Vector v = gaussian_moment_vector(GridSpec{2.0, 2}, 1.0, false);
    const double want = 0.5 * std::sqrt(M_PI) * std::erf(1.0);
    EXPECT_NEAR(v[0], want, 1e-15);
    EXPECT_NEAR(v[1], want, 1e-15);
    EXPECT_NEAR(v[1], simpson([](double x) { return std::exp(-x * x); }, 0.0, 1.0), 1e-12);
}

TEST(GaussianMoments, MatchesAdaptiveQuadraturePerCell) {  // test_newton.cpp:54-69
    GridSpec grid{3.0, 6};
    const double t = 0.7;
    for (bool doubled : {false, true}) {
        Vector v = gaussian_moment_vector(grid, t, doubled);
        const Index len = doubled ? 12 : 6;
        ASSERT_EQ(v.size(), len);
        for (Index i = 0; i < len; ++i) {
            const double lo = static_cast<double>(i - len / 2) * grid.h();
            EXPECT_NEAR(v[i], simpson([t](double x) { return std::exp(-t * t * x * x); }, lo, lo + grid.h()), 1e-12);
        }
    }
}

TEST(GaussianMoments, EvenSymmetryIsExact) {  // test_newton.cpp:71-77
    for (double t : {0.3, 1.0, 4.5}) {
        Vector v = gaussian_moment_vector(GridSpec{5.0, 10}, t, false);
        for (Index i = 0; i < v.size(); ++i) EXPECT_EQ(v[i], v[v.size() - 1 - i]);
    }
}

TEST(GaussianMoments, RejectsBadArguments) {  // test_newton.cpp:79-84
    EXPECT_THROW(gaussian_moment_vector(GridSpec{2.0, 4}, -1.0, false), validation_error);
    EXPECT_THROW(gaussian_moment_vector(GridSpec{2.0, 3}, 1.0, false), validation_error);
}

TEST(GaussianSamples, MatchesMidpointValues) {  // test_newton.cpp:86-96
    const Index len = 6;
    const double h = 0.5, t = 1.3;
    Vector v = gaussian_sample_vector(len, h, t);
    for (Index i = 0; i < len; ++i) {
        const double x = (static_cast<double>(i) + 0.5 - 3.0) * h;
        EXPECT_NEAR(v[i], std::exp(-t * t * x * x), 4 * std::numeric_limits<double>::epsilon() * v[i]);
        EXPECT_EQ(v[i], v[len - 1 - i]);
    }
    EXPECT_THROW(gaussian_sample_vector(5, h, t), validation_error);
}

TEST(NewtonTensor, SharedAxesAndRank) {  // test_newton.cpp:125-141
    GridSpec grid{2.0, 8};
    QuadratureRule rule = sinc_quadrature(1e-4, grid.h(), 4.0, 10, 1.0);
    CanonicalTensor3 t = build_newton_tensor(grid, rule);
    EXPECT_EQ(t.rank(), rule.node_count());
    EXPECT_TRUE((t.dims() == Dims3{8, 8, 8}));
    EXPECT_TRUE((t.factor(0).array() == t.factor(1).array()).all());
    EXPECT_TRUE((t.factor(0).array() == t.factor(2).array()).all());
    EXPECT_TRUE((t.weights().array() == rule.weights.array()).all());
    EXPECT_TRUE((build_newton_tensor(grid, rule, true).dims() == Dims3{16, 16, 16}));
    CanonicalTensor3 m = build_newton_master({8, 6, 8}, grid.h(), rule);
    EXPECT_EQ(m.dim(1), 6);
    EXPECT_TRUE((m.factor(0).array() == m.factor(2).array()).all());
}

TEST(NewtonTensor, EntryEqualsQuadratureValueAtRadius) {  // test_newton.cpp:143-158
    GridSpec grid{2.0, 16};
    QuadratureRule rule = sinc_quadrature(1e-5, grid.h(), 4.0, 25, 2.0);
    CanonicalTensor3 t = build_newton_tensor(grid, rule);
    for (Index i : {0, 3, 8, 11})
        for (Index j : {1, 8, 14}) {
            const Index k = 5;
            const double x = grid.midpoint(i), y = grid.midpoint(j), z = grid.midpoint(k);
            const double r = std::sqrt(x * x + y * y + z * z);
            EXPECT_NEAR(eval_point(t, i, j, k), quadrature_value(rule, r), 1e-12 * quadrature_value(rule, r));
        }
}

TEST(ProbeSet, CoversBandDeterministically) {  // test_newton.cpp:160-183
    GridSpec grid{2.0, 32};
    KernelTolerance tol = default_tolerance(grid, 1e-4);
    std::vector<ProbePoint> probes = kernel_probe_set(grid, tol);
    ASSERT_TRUE(!probes.empty());
    for (std::size_t e = 0; e < probes.size(); ++e) {
        EXPECT_GE(probes[e].r, tol.a_min);
        EXPECT_LE(probes[e].r, tol.a_max);
        if (e > 0)
            EXPECT_TRUE(probes[e].i != probes[e - 1].i || probes[e].j != probes[e - 1].j || probes[e].k != probes[e - 1].k);
    }
    EXPECT_EQ(kernel_probe_set(grid, tol).size(), probes.size());
}

TEST(Calibration, MeetsRequestedAccuracy) {  // test_newton.cpp:185-196
    GridSpec grid{2.0, 16};
    KernelTolerance tol = default_tolerance(grid, 1e-4);
    CalibrationTrace trace;
    QuadratureRule rule = calibrate_quadrature(grid, tol, &trace);
    EXPECT_FALSE(trace.entries.empty());
    EXPECT_LE(measure_probe_error(build_newton_tensor(grid, rule), kernel_probe_set(grid, tol)), tol.eps);
    EXPECT_EQ(trace.entries.back().M, rule.M);
}

TEST(Calibration, RankGrowsAsToleranceTightens) {  // test_newton.cpp:198-204
    GridSpec grid{2.0, 16};
    EXPECT_LT(calibrate_quadrature(grid, default_tolerance(grid, 1e-3)).M,
              calibrate_quadrature(grid, default_tolerance(grid, 1e-6)).M);
}

TEST(Calibration, CapExhaustionRaisesResourceGuard) {  // test_newton.cpp:206-210
    GridSpec grid{2.0, 16};
    EXPECT_THROW(calibrate_quadrature(grid, default_tolerance(grid, 1e-9), nullptr, 3), resource_guard_error);
}

TEST(Calibration, KernelIsStrictlyPositive) {  // test_newton.cpp:212-219
    GridSpec grid{2.0, 16};
    QuadratureRule rule = calibrate_quadrature(grid, default_tolerance(grid, 1e-4));
    DenseTensor3 dense = densify(build_newton_tensor(grid, rule));
    EXPECT_GT(dense.data().minCoeff(), 0.0);
}

// ------------------------------------------------------------------ canonical (GPU expansion)
TEST(CanonicalTensor, ZeroTensorIsRankZero) {  // test_canonical.cpp:39-46
    CanonicalTensor3 z(Dims3{3, 4, 5});
    EXPECT_EQ(z.rank(), 0);
    EXPECT_EQ(eval_point(z, 1, 2, 3), 0.0);
    EXPECT_EQ(max_abs(densify(z)), 0.0);
}

TEST(CanonicalTensor, ConstructorValidation) {  // test_canonical.cpp:48-61
    std::array<Matrix, 3> bad{Matrix::Ones(2, 2), Matrix::Ones(2, 1), Matrix::Ones(2, 2)};
    EXPECT_THROW(CanonicalTensor3(std::move(bad), Vector::Ones(2)), validation_error);
    std::array<Matrix, 3> nan{Matrix::Ones(2, 1), Matrix::Ones(2, 1), Matrix::Ones(2, 1)};
    nan[1](0, 0) = std::numeric_limits<double>::quiet_NaN();
    EXPECT_THROW(CanonicalTensor3(std::move(nan), Vector::Ones(1)), validation_error);
}

TEST(CanonicalTensor, DensifyMatchesScalarLoops) {  // test_canonical.cpp:63-69
    std::mt19937 gen(7);
    for (int trial = 0; trial < 10; ++trial) {
        CanonicalTensor3 t = random_tensor(gen, random_dims(gen), 3);
        EXPECT_LT(rel_diff(densify(t), scalar_oracle(t)), 1e-13);
    }
}

TEST(CanonicalTensor, DensifyIsIndependentOfThreadCap) {  // test_canonical.cpp:71-81
    std::mt19937 gen(8);
    CanonicalTensor3 t = random_tensor(gen, {6, 5, 7}, 4);
    const int old = max_threads();
    set_max_threads(1);
    DenseTensor3 serial = densify(t);
    set_max_threads(4);
    DenseTensor3 parallel = densify(t);
    set_max_threads(old);
    EXPECT_EQ(max_norm_diff(serial, parallel), 0.0);
}

TEST(CanonicalTensor, DensifyGuardRejectsLargeGrid) {  // test_canonical.cpp:83-86
    EXPECT_THROW(densify(constant_tensor({8, 8, 8}, 1.0), 100), resource_guard_error);
}

TEST(CanonicalTensor, EvalPointMatchesDense) {  // test_canonical.cpp:88-98
    std::mt19937 gen(9);
    CanonicalTensor3 t = random_tensor(gen, {4, 5, 6}, 3);
    DenseTensor3 d = scalar_oracle(t);
    for (Index k = 0; k < 6; ++k)
        for (Index j = 0; j < 5; ++j)
            for (Index i = 0; i < 4; ++i) EXPECT_NEAR(eval_point(t, i, j, k), d(i, j, k), 1e-13);
    EXPECT_THROW(eval_point(t, 4, 0, 0), validation_error);
    EXPECT_THROW(eval_point(t, 0, -1, 0), validation_error);
}

TEST(ScalarProduct, AllOnesCountsEntries) {  // test_canonical.cpp:100-103
    EXPECT_EQ(scalar_product(constant_tensor({2, 2, 2}, 1.0), constant_tensor({2, 2, 2}, 1.0)), 8.0);
}

TEST(ScalarProduct, ZeroTensorGivesZero) {  // test_canonical.cpp:105-110
    CanonicalTensor3 z(Dims3{3, 3, 3});
    EXPECT_EQ(scalar_product(z, constant_tensor({3, 3, 3}, 2.0)), 0.0);
}

TEST(ScalarProduct, MatchesDenseDotProduct) {  // test_canonical.cpp:112-122
    std::mt19937 gen(11);
    for (int trial = 0; trial < 20; ++trial) {
        Dims3 dims = random_dims(gen);
        CanonicalTensor3 a = random_tensor(gen, dims, 3), b = random_tensor(gen, dims, 4);
        DenseTensor3 da = scalar_oracle(a), db = scalar_oracle(b);
        double want = 0.0;
        for (Index e = 0; e < da.size(); ++e) want += da.data()[e] * db.data()[e];
        EXPECT_NEAR(scalar_product(a, b), want, 1e-11 * std::max(1.0, std::abs(want)));
    }
}

TEST(ScalarProduct, DeterministicAcrossRepeats) {  // test_canonical.cpp:133-139
    std::mt19937 gen(13);
    CanonicalTensor3 a = random_tensor(gen, {7, 6, 5}, 5), b = random_tensor(gen, {7, 6, 5}, 4);
    const double first = scalar_product(a, b);
    for (int rep = 0; rep < 5; ++rep) EXPECT_EQ(scalar_product(a, b), first);
}

TEST(ScalarProduct, RejectsDimMismatch) {  // test_canonical.cpp:141-145
    EXPECT_THROW(scalar_product(constant_tensor({2, 2, 2}, 1.0), constant_tensor({2, 2, 3}, 1.0)), validation_error);
}

TEST(Algebra, AddHadamardCoalescingMatchDense) {  // test_canonical.cpp:147-227
    std::mt19937 gen(21);
    Dims3 dims{4, 3, 5};
    CanonicalTensor3 a = random_tensor(gen, dims, 2), b = random_tensor(gen, dims, 3);
    CanonicalTensor3 s = add(a, b);
    EXPECT_EQ(s.rank(), 5);
    DenseTensor3 da = scalar_oracle(a), db = scalar_oracle(b), want(dims[0], dims[1], dims[2]);
    for (Index e = 0; e < want.size(); ++e) want.data()[e] = da.data()[e] + db.data()[e];
    EXPECT_LT(rel_diff(densify(s), want), 1e-12);
    CanonicalTensor3 h = hadamard(a, b);
    EXPECT_EQ(h.rank(), 6);
    for (Index e = 0; e < want.size(); ++e) want.data()[e] = da.data()[e] * db.data()[e];
    EXPECT_LT(rel_diff(densify(h), want), 1e-12);
    std::array<Matrix, 3> cf{a.factor(0), a.factor(1), a.factor(2)};
    cf[1] = random_tensor(gen, dims, 2).factor(1);
    CanonicalTensor3 c(std::move(cf), a.weights());
    CanonicalTensor3 co = add_coalescing(a, c, 1);
    DenseTensor3 dc = scalar_oracle(c);
    for (Index e = 0; e < want.size(); ++e) want.data()[e] = da.data()[e] + dc.data()[e];
    EXPECT_LT(rel_diff(densify(co), want), 1e-12);
    EXPECT_THROW(add_coalescing(a, b, 0), validation_error);
}

TEST(StreamingDiff, MatchesDenseDifference) {  // test_canonical.cpp:276-285
    std::mt19937 gen(61);
    CanonicalTensor3 a = random_tensor(gen, {9, 8, 7}, 3), b = random_tensor(gen, {9, 8, 7}, 4);
    StreamDiff d = max_norm_diff_canonical(a, b);
    DenseTensor3 da = scalar_oracle(a), db = scalar_oracle(b);
    EXPECT_NEAR(d.max_diff, max_norm_diff(da, db), 1e-13);
    EXPECT_NEAR(d.max_abs_b, max_abs(db), 1e-13);
}

TEST(StreamingDiff, ZeroRankSideExpandsToZero) {  // canonical.hpp:282-301 with a rank-0 tensor
    std::mt19937 gen(62);
    CanonicalTensor3 b = random_tensor(gen, {9, 8, 7}, 3), z(Dims3{9, 8, 7});
    DenseTensor3 db = scalar_oracle(b);
    StreamDiff d = max_norm_diff_canonical(z, b);
    EXPECT_NEAR(d.max_diff, max_abs(db), 1e-13);
    EXPECT_NEAR(d.max_abs_b, max_abs(db), 1e-13);
    StreamDiff e = max_norm_diff_canonical(b, z);
    EXPECT_NEAR(e.max_diff, max_abs(db), 1e-13);
    EXPECT_EQ(e.max_abs_b, 0.0);
}

// ------------------------------------------------------------------ lattice (GPU assembly)
TEST(Window, ValidatesBoundsAndExtracts) {  // test_lattice.cpp:62-82
    EXPECT_NO_THROW(WindowOp(4, 8, 4));
    EXPECT_THROW(WindowOp(-1, 8, 4), validation_error);
    EXPECT_THROW(WindowOp(5, 8, 4), validation_error);
    EXPECT_THROW(WindowOp(0, 8, 0), validation_error);
    Vector m(8);
    for (Index i = 0; i < 8; ++i) m[i] = static_cast<double>(i);
    Vector mid = window_apply(m, WindowOp(2, 8, 4));
    for (Index i = 0; i < 4; ++i) EXPECT_EQ(mid[i], static_cast<double>(i + 2));
    EXPECT_THROW(window_apply(m, WindowOp(0, 9, 4)), validation_error);
}

TEST(Window, StartsStayInsideDoubledMaster) {  // test_lattice.cpp:84-101
    const Index n = 8;
    for (Index L : {1, 2, 3, 5})
        for (Index ia = 0; ia <= n; ++ia)
            for (Index k = 0; k < L; ++k) {
                const Index N = L * n;
                EXPECT_GE(window_start_box(N, n, ia, k), 0);
                EXPECT_LE(window_start_box(N, n, ia, k) + N, 2 * N);
                EXPECT_GE(window_start_periodic(N, n, ia, k, L), 0);
                EXPECT_LE(window_start_periodic(N, n, ia, k, L) + n, 2 * N);
            }
}

TEST(LatticeSpec, SnapsOnlyExactGridPoints) {  // test_lattice.cpp:103-123
    EXPECT_THROW(make_spec({0, 2, 2}, 8, 2.0, {Charge{}}).validate(), validation_error);
    EXPECT_THROW(make_spec({2, 2, 2}, 8, 2.0, {}).validate(), validation_error);
    EXPECT_THROW(make_spec({2, 2, 2}, 8, 2.0, {Charge{{0, 0, 0}, -1.0}}).validate(), validation_error);
    LatticeSpec on = make_spec({1, 1, 1}, 8, 2.0, {Charge{{0.25, -1.0, 1.0}, 1.0}});
    EXPECT_EQ(on.charge_grid_index(0, 0), 5);
    EXPECT_EQ(on.charge_grid_index(1, 0), 0);
    EXPECT_EQ(on.charge_grid_index(2, 0), 8);
    EXPECT_THROW(make_spec({1, 1, 1}, 8, 2.0, {Charge{{0.1, 0.0, 0.0}, 1.0}}).validate(), validation_error);
    EXPECT_THROW(make_spec({1, 1, 1}, 8, 2.0, {Charge{{1.25, 0.0, 0.0}, 1.0}}).validate(), validation_error);
}

TEST(DirectSum, SingleCellIsCenteredWindowOfMaster) {  // test_lattice.cpp:125-137
    LatticeSpec spec = make_spec({1, 1, 1}, 16, 2.0, {Charge{}});
    QuadratureRule rule = sinc_quadrature(1e-4, spec.unit.h(), std::sqrt(3.0) * 2.0, 10, 1.0);
    CanonicalTensor3 master = build_lattice_master(spec, rule);
    SumResult sum = direct_sum(spec, master);
    EXPECT_EQ(sum.rank, rule.node_count());
    for (int l = 0; l < 3; ++l)
        EXPECT_TRUE((sum.tensor.factor(l).array() == master.factor(l).middleRows(8, 16).array()).all());
}

TEST(DirectSum, MatchesPhysicalOracle) {  // test_lattice.cpp:139-155
    LatticeSpec spec = make_spec({2, 2, 2}, 8, 2.0, {Charge{{0.0, 0.0, 0.0}, 1.0}, Charge{{-0.5, 0.25, 0.75}, 2.5}});
    QuadratureRule rule = calibrate_for_lattice(spec, 1e-4);
    SumResult sum = direct_sum(spec, build_lattice_master(spec, rule));
    EXPECT_EQ(sum.rank, 2 * 8 * rule.node_count());
    DenseTensor3 dense = densify(sum.tensor);
    double worst = 0.0;
    for (Index k = 0; k < 16; ++k)
        for (Index j = 0; j < 16; ++j)
            for (Index i = 0; i < 16; ++i) {
                const double want = physical_potential(spec, rule, {i, j, k}, false);
                worst = std::max(worst, std::abs(dense(i, j, k) - want) / std::abs(want));
            }
    EXPECT_LT(worst, 1e-12);
}

TEST(DirectSum, LinearInCharges) {  // test_lattice.cpp:157-172
    Charge a{{0.0, 0.0, 0.0}, 1.0}, b{{0.25, -0.25, 0.5}, 3.0};
    LatticeSpec both = make_spec({2, 1, 2}, 8, 2.0, {a, b});
    QuadratureRule rule = calibrate_for_lattice(both, 1e-4);
    CanonicalTensor3 master = build_lattice_master(both, rule);
    LatticeSpec only_a = both, only_b = both;
    only_a.charges = {a};
    only_b.charges = {b};
    StreamDiff d = max_norm_diff_canonical(add(direct_sum(only_a, master).tensor, direct_sum(only_b, master).tensor),
                                           direct_sum(both, master).tensor);
    EXPECT_EQ(d.max_diff, 0.0);
}

TEST(DirectSum, GuardsAndRejects) {  // test_lattice.cpp:189-203
    LatticeSpec spec = make_spec({4, 4, 4}, 8, 2.0, {Charge{}});
    CanonicalTensor3 master = build_lattice_master(spec, sinc_quadrature(1e-4, 0.25, 14.0, 10, 1.0));
    EXPECT_THROW(direct_sum(spec, master, 100), resource_guard_error);
    LatticeSpec s2 = make_spec({2, 1, 1}, 8, 2.0, {Charge{}});
    QuadratureRule r2 = sinc_quadrature(1e-4, 0.25, 7.0, 8, 1.0);
    EXPECT_THROW(direct_sum(s2, build_newton_master({16, 16, 16}, s2.unit.h(), r2)), validation_error);
    EXPECT_THROW(direct_sum(s2, CanonicalTensor3(Dims3{32, 16, 16})), validation_error);
}

TEST(AssembledSum, SingleCellEqualsDirect) {  // test_lattice.cpp:205-216
    LatticeSpec spec = make_spec({1, 1, 1}, 16, 2.0, {Charge{}});
    QuadratureRule rule = calibrate_for_lattice(spec, 1e-4);
    CanonicalTensor3 master = build_lattice_master(spec, rule);
    SumResult as = assembled_box_sum(spec, master), ds = direct_sum(spec, master);
    EXPECT_EQ(as.rank, ds.rank);
    for (int l = 0; l < 3; ++l) EXPECT_TRUE((as.tensor.factor(l).array() == ds.tensor.factor(l).array()).all());
    EXPECT_TRUE((as.tensor.weights().array() == ds.tensor.weights().array()).all());
}

TEST(AssembledSum, MatchesDirectSumAcrossShapes) {  // test_lattice.cpp:218-241
    struct Case {
        std::array<Index, 3> L;
        Index n;
        std::vector<Charge> charges;
    };
    const std::vector<Case> cases = {
        {{2, 2, 2}, 16, {Charge{}}},
        {{4, 2, 1}, 8, {Charge{{0.0, 0.0, 0.0}, 1.0}, Charge{{0.5, -0.25, 0.25}, 2.0}}},
        {{3, 1, 2}, 8, {Charge{{-0.75, 0.5, 0.0}, 0.5}}},
    };
    for (const Case& c : cases) {
        LatticeSpec spec = make_spec(c.L, c.n, 2.0, c.charges);
        QuadratureRule rule = calibrate_for_lattice(spec, 1e-4);
        CanonicalTensor3 master = build_lattice_master(spec, rule);
        SumResult as = assembled_box_sum(spec, master), ds = direct_sum(spec, master);
        EXPECT_EQ(as.rank, spec.charge_count() * rule.node_count());
        EXPECT_EQ(ds.rank, spec.charge_count() * spec.cell_count() * rule.node_count());
        StreamDiff d = max_norm_diff_canonical(as.tensor, ds.tensor);
        EXPECT_LT(d.max_diff / d.max_abs_b, 1e-12);
    }
}

TEST(AssembledSum, RankIsIndependentOfLatticeSize) {  // test_lattice.cpp:243-253
    for (Index L : {1, 2, 4}) {
        LatticeSpec spec = make_spec({L, L, L}, 8, 2.0, {Charge{}});
        QuadratureRule rule = sinc_quadrature(1e-4, spec.unit.h(), std::sqrt(3.0) * 2.0 * L, 12, 1.0);
        SumResult sum = assembled_box_sum(spec, build_lattice_master(spec, rule));
        EXPECT_EQ(sum.rank, rule.node_count());
        EXPECT_TRUE((sum.grid_dims == spec.target_dims()));
    }
}

TEST(PeriodicSum, SingleCellRestrictsToReferenceCell) {  // test_lattice.cpp:255-264
    LatticeSpec spec = make_spec({1, 1, 1}, 16, 2.0, {Charge{}});
    QuadratureRule rule = calibrate_for_lattice(spec, 1e-4);
    CanonicalTensor3 master = build_lattice_master(spec, rule);
    SumResult per = assembled_periodic_sum(spec, master), box = assembled_box_sum(spec, master);
    EXPECT_TRUE((per.grid_dims == Dims3{16, 16, 16}));
    for (int l = 0; l < 3; ++l) EXPECT_TRUE((per.tensor.factor(l).array() == box.tensor.factor(l).array()).all());
}

TEST(PeriodicSum, MatchesPhysicalOracleOnReferenceCell) {  // test_lattice.cpp:266-283
    LatticeSpec spec = make_spec({4, 2, 1}, 8, 2.0, {Charge{{0.0, 0.0, 0.0}, 1.0}, Charge{{0.25, 0.5, -0.25}, 1.5}});
    QuadratureRule rule = calibrate_for_lattice(spec, 1e-4);
    SumResult sum = assembled_periodic_sum(spec, build_lattice_master(spec, rule));
    EXPECT_EQ(sum.rank, 2 * rule.node_count());
    DenseTensor3 dense = densify(sum.tensor);
    double worst = 0.0;
    for (Index k = 0; k < 8; ++k)
        for (Index j = 0; j < 8; ++j)
            for (Index i = 0; i < 8; ++i) {
                const double want = physical_potential(spec, rule, {i, j, k}, true);
                worst = std::max(worst, std::abs(dense(i, j, k) - want) / std::abs(want));
            }
    EXPECT_LT(worst, 1e-12);
}

TEST(Series, CenterValuesGrowWithBoxSize) {  // test_lattice.cpp:285-296
    std::vector<SeriesPoint> pts = center_value_series(SeriesKind::cube, {1, 2, 4}, GridSpec{2.0, 8}, 1e-4);
    ASSERT_EQ(pts.size(), 3u);
    EXPECT_LT(pts[0].p_center, pts[1].p_center);
    EXPECT_LT(pts[1].p_center, pts[2].p_center);
    EXPECT_EQ(pts[0].rank, pts[2].rank);
    EXPECT_EQ(richardson_extrapolate(2.0, 3.0, RichardsonOrder::linear), 1.0);
}

// ------------------------------------------------------------------ projection
TEST(PotentialMatrix, OnesBasisSumsAllEntries) {  // test_project.cpp:100-110
    GridSpec grid{2.0, 4};
    Rank1Basis basis = sample_gaussian_basis(grid, {GaussianBasisSpec{{0.0, 0.0, 0.0}, 1e9}});
    CanonicalTensor3 ones = constant_tensor({4, 4, 4}, 0.5);
    EXPECT_NEAR(potential_matrix(basis, ones, false)(0, 0), 0.5 * 64.0, 1e-10);
    EXPECT_NEAR(potential_matrix(basis, ones, true)(0, 0), 0.5 * 64.0 * std::pow(0.5, 3), 1e-10);
}

TEST(PotentialMatrix, SymmetricBilinearAndValidated) {  // test_project.cpp:90-98, 127-148
    GridSpec grid{2.0, 6};
    std::vector<GaussianBasisSpec> specs = {{{0.0, 0.0, 0.0}, 0.5}, {{0.3, -0.2, 0.1}, 0.7}, {{-0.4, 0.4, 0.0}, 0.4}};
    Rank1Basis basis = sample_gaussian_basis(grid, specs);
    std::mt19937 gen(100);
    CanonicalTensor3 A = random_tensor(gen, {6, 6, 6}, 3), B = random_tensor(gen, {6, 6, 6}, 2);
    Matrix VA = potential_matrix(basis, A, true), VB = potential_matrix(basis, B, true);
    Matrix VAB = potential_matrix(basis, add(A, B), true);
    for (Index k = 0; k < 3; ++k)
        for (Index m = 0; m < 3; ++m) {
            EXPECT_EQ(VA(k, m), VA(m, k));
            EXPECT_NEAR(VAB(k, m), VA(k, m) + VB(k, m), 1e-13 * VAB.cwiseAbs().maxCoeff());
        }
    // dense triple-loop oracle (test_project.cpp:21-57, 112-125)
    DenseTensor3 dA = scalar_oracle(A);
    for (Index k = 0; k < 3; ++k)
        for (Index m = 0; m < 3; ++m) {
            double want = 0.0;
            for (Index z = 0; z < 6; ++z)
                for (Index y = 0; y < 6; ++y)
                    for (Index x = 0; x < 6; ++x)
                        want += basis.funcs[k][0][x] * basis.funcs[m][0][x] * basis.funcs[k][1][y] * basis.funcs[m][1][y] *
                                basis.funcs[k][2][z] * basis.funcs[m][2][z] * dA(x, y, z);
            want *= std::pow(grid.h(), 3);
            EXPECT_NEAR(VA(k, m), want, 1e-11 * VA.cwiseAbs().maxCoeff());
        }
    EXPECT_THROW(sample_gaussian_basis(grid, {}), validation_error);
    EXPECT_THROW(sample_gaussian_basis(grid, {GaussianBasisSpec{{0, 0, 0}, 0.0}}), validation_error);
    EXPECT_THROW(potential_matrix(basis, random_tensor(gen, {6, 6, 4}, 2), true), validation_error);
}

// ------------------------------------------------------------------ acceptance criterion 1 (fig5)
TEST(Acceptance, Fig5AssembledMatchesDirect) {  // acceptance.cpp:112-115 -> repro.hpp:67-99
    const auto t0 = std::chrono::steady_clock::now();
    LatticeSpec spec = make_spec({8, 8, 2}, 64, 2.0, {Charge{}});
    QuadratureRule rule = calibrate_for_lattice(spec, 1e-6);
    CanonicalTensor3 master = build_lattice_master(spec, rule);
    SumResult as = assembled_box_sum(spec, master), ds = direct_sum(spec, master);
    StreamDiff d = max_norm_diff_canonical(as.tensor, ds.tensor);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("    fig5: rank %ld vs direct %ld, rel %.3e, %.2f s\n", static_cast<long>(as.rank),
                static_cast<long>(ds.rank), d.max_diff / d.max_abs_b, secs);
    EXPECT_LE(d.max_diff / d.max_abs_b, 1e-12);
    EXPECT_LT(secs, 60.0);
}

// ------------------------------------------------------------------ device-resident API
TEST(DevicePotential, MatchesHostPipelineAndEnergy) {  // additive API over ls_pipeline_*
    LatticeSpec spec = make_spec({3, 2, 2}, 8, 2.0, {Charge{{0.0, 0.0, 0.0}, 1.0}, Charge{{0.5, -0.25, 0.25}, 2.0}});
    QuadratureRule rule = sinc_quadrature(1e-4, spec.unit.h(), std::sqrt(3.0) * 6.0, 10, 1.0);
    DevicePotential dev(spec, rule, Generator::midpoint);
    const Dims3 d = dev.dims();
    EXPECT_TRUE((d == Dims3{24, 16, 16}));
    EXPECT_EQ(dev.rank(), 2 * rule.node_count());
    DeviceBuffer grid(static_cast<std::size_t>(d[0] * d[1] * d[2]));
    dev.step(0, d[2], grid.data());
    std::vector<double> got(grid.size());
    grid.download(got.data(), got.size());
    // the same lattice through the drop-in host path
    SumResult s = assembled_box_sum(spec, build_lattice_master(spec, rule));
    DenseTensor3 want = densify(s.tensor);
    double md = 0.0;
    for (std::size_t e = 0; e < got.size(); ++e) md = std::max(md, std::abs(got[e] - want.data()[static_cast<Index>(e)]));
    EXPECT_LT(md / max_abs(want), 1e-14);
    CanonicalTensor3 t = dev.tensor();
    for (int l = 0; l < 3; ++l) EXPECT_TRUE((t.factor(l).array() == s.tensor.factor(l).array()).all());
    // energy against the 1D form (scalar_product with a rank-1 density)
    std::array<Vector, 3> r;
    for (int l = 0; l < 3; ++l) {
        r[l].resize(d[l]);
        for (Index i = 0; i < d[l]; ++i) r[l][i] = 1.0 / (1.0 + static_cast<double>(i));
    }
    DeviceBuffer r1(d[0]), r2(d[1]), r3(d[2]), e(1);
    r1.upload(r[0].data(), d[0]);
    r2.upload(r[1].data(), d[1]);
    r3.upload(r[2].data(), d[2]);
    dev.energy(r1.data(), r2.data(), r3.data(), 0, d[2], e.data());
    double energy = 0.0;
    e.download(&energy, 1);
    std::array<Matrix, 3> rf{Matrix(r[0]), Matrix(r[1]), Matrix(r[2])};
    const double want_e = scalar_product(s.tensor, CanonicalTensor3(std::move(rf), Vector::Ones(1)));
    EXPECT_NEAR(energy, want_e, 1e-12 * std::abs(want_e));
    // z-slab shards cover the grid exactly once
    Index covered = 0;
    for (int rk = 0; rk < 3; ++rk) covered += slab_range(d[2], rk, 3).second - slab_range(d[2], rk, 3).first;
    EXPECT_EQ(covered, d[2]);
}

TEST(DevicePotential, GridFunctionalsMatchScalarProduct) {  // full-grid batch vs the 1D form
    LatticeSpec spec = make_spec({2, 3, 2}, 8, 2.0, {Charge{{0.0, 0.0, 0.0}, 1.0}});
    QuadratureRule rule = sinc_quadrature(1e-4, spec.unit.h(), std::sqrt(3.0) * 6.0, 10, 1.0);
    DevicePotential dev(spec, rule, Generator::erf, /*periodic=*/true);
    dev.generate();
    dev.assemble();
    const Dims3 d = dev.dims();
    const int F = 5;
    std::array<Matrix, 3> rho;
    for (int l = 0; l < 3; ++l) {
        rho[l].resize(d[l], F);
        for (Index i = 0; i < d[l]; ++i)
            for (int f = 0; f < F; ++f) rho[l](i, f) = std::exp(-0.1 * (f + 1) * static_cast<double>((i - 3) * (i - 3)));
    }
    DeviceBuffer X(d[0] * F), Y(d[1] * F), Z(d[2] * F), out(F), scratch(static_cast<std::size_t>(d[0] * d[1] * d[2]));
    X.upload(rho[0].data(), X.size());
    Y.upload(rho[1].data(), Y.size());
    Z.upload(rho[2].data(), Z.size());
    // two slab chunks, the second accumulating
    dev.grid_functionals(X.data(), Y.data(), Z.data(), F, 0, 3, scratch.data(), out.data());
    dev.grid_functionals(X.data(), Y.data(), Z.data(), F, 3, d[2], scratch.data(), out.data(), true);
    std::vector<double> got(F);
    out.download(got.data(), F);
    CanonicalTensor3 t = dev.tensor();
    for (int f = 0; f < F; ++f) {
        std::array<Matrix, 3> rf{Matrix(rho[0].col(f)), Matrix(rho[1].col(f)), Matrix(rho[2].col(f))};
        const double want = scalar_product(t, CanonicalTensor3(std::move(rf), Vector::Ones(1)));
        EXPECT_NEAR(got[f], want, 1e-12 * std::abs(want));
    }
    EXPECT_THROW(dev.grid_functionals(X.data(), Y.data(), Z.data(), F, 2, 1, scratch.data(), out.data()),
                 validation_error);
}


// ------------------------------------------------------------------ factor algebra and 1D convolution
TEST(Convolve1d, DeltaAndBoxIdentities) {  // test_canonical.cpp:230-246
    Vector a(7);
    for (Index i = 0; i < 7; ++i) a[i] = 0.5 * static_cast<double>(i) - 1.25;
    Vector delta = Vector::Zero(5);
    delta[5 / 2] = 1.0;  // centred unit impulse: "same" mode must give a back unchanged
    Vector same = convolve1d(a, delta, ConvMode::same);
    EXPECT_TRUE((same.array() == a.array()).all());
    Vector box = Vector::Ones(3);
    Vector tri = convolve1d(box, box, ConvMode::full);  // 1 2 3 2 1
    ASSERT_EQ(tri.size(), 5);
    const double want[5] = {1.0, 2.0, 3.0, 2.0, 1.0};
    for (Index i = 0; i < 5; ++i) EXPECT_EQ(tri[i], want[i]);
}

TEST(Convolve1d, FullLengthAndCommutativity) {  // test_canonical.cpp:248-258
    std::mt19937 gen(2024);
    std::uniform_real_distribution<double> u(-2.0, 2.0);
    Vector a(9), b(5);
    for (Index i = 0; i < 9; ++i) a[i] = u(gen);
    for (Index i = 0; i < 5; ++i) b[i] = u(gen);
    Vector ab = convolve1d(a, b, ConvMode::full), ba = convolve1d(b, a, ConvMode::full);
    ASSERT_EQ(ab.size(), 13);
    ASSERT_EQ(ba.size(), 13);
    EXPECT_LT((ab - ba).cwiseAbs().maxCoeff(), 1e-14);
}

TEST(ConvolveCanonical, MatchesDenseConvolution) {  // test_canonical.cpp:260-274
    std::mt19937 gen(77);
    for (ConvMode mode : {ConvMode::full, ConvMode::same}) {
        for (int trial = 0; trial < 4; ++trial) {
            const Dims3 d = random_dims(gen, 2, 5);
            CanonicalTensor3 a = random_tensor(gen, d, 2), b = random_tensor(gen, d, 3);
            CanonicalTensor3 c = convolve1d_canonical(a, b, mode);
            EXPECT_EQ(c.rank(), 6);
            // dense 3D convolution of the two materialised tensors by scalar loops
            const DenseTensor3 da = scalar_oracle(a), db = scalar_oracle(b);
            Dims3 full{2 * d[0] - 1, 2 * d[1] - 1, 2 * d[2] - 1};
            std::vector<double> conv(static_cast<size_t>(full[0] * full[1] * full[2]), 0.0);
            for (Index k = 0; k < d[2]; ++k)
                for (Index j = 0; j < d[1]; ++j)
                    for (Index i = 0; i < d[0]; ++i)
                        for (Index kk = 0; kk < d[2]; ++kk)
                            for (Index jj = 0; jj < d[1]; ++jj)
                                for (Index ii = 0; ii < d[0]; ++ii)
                                    conv[static_cast<size_t>((i + ii) + full[0] * ((j + jj) + full[1] * (k + kk)))] +=
                                        da(i, j, k) * db(ii, jj, kk);
            const Dims3 out = c.dims();
            const Index off[3] = {mode == ConvMode::same ? d[0] / 2 : 0, mode == ConvMode::same ? d[1] / 2 : 0,
                                  mode == ConvMode::same ? d[2] / 2 : 0};
            const DenseTensor3 dc = scalar_oracle(c);
            double md = 0.0, mx = 0.0;
            for (Index k = 0; k < out[2]; ++k)
                for (Index j = 0; j < out[1]; ++j)
                    for (Index i = 0; i < out[0]; ++i) {
                        const double w = conv[static_cast<size_t>((i + off[0]) +
                                                                  full[0] * ((j + off[1]) + full[1] * (k + off[2])))];
                        md = std::max(md, std::abs(dc(i, j, k) - w));
                        mx = std::max(mx, std::abs(w));
                    }
            EXPECT_LT(md / mx, 1e-12);
        }
    }
}

TEST(Algebra, ZeroOperands) {  // test_canonical.cpp:162-168, 186-193
    std::mt19937 gen(5);
    CanonicalTensor3 a = random_tensor(gen, {4, 3, 5}, 3);
    CanonicalTensor3 zero(Dims3{4, 3, 5});
    CanonicalTensor3 h = hadamard(a, zero);  // anything times the zero tensor is the zero tensor
    EXPECT_EQ(h.rank(), 0);
    EXPECT_TRUE((h.dims() == Dims3{4, 3, 5}));
    CanonicalTensor3 s = add(a, zero);  // and adding it changes nothing, bit for bit
    EXPECT_EQ(s.rank(), a.rank());
    EXPECT_EQ(max_norm_diff(densify(s), densify(a)), 0.0);
}

TEST(AddCoalescing, RejectsMismatchedInputs) {  // test_canonical.cpp:219-228
    std::mt19937 gen(8);
    CanonicalTensor3 a = random_tensor(gen, {3, 4, 3}, 2), b = random_tensor(gen, {3, 4, 3}, 2);
    EXPECT_THROW(add_coalescing(a, b, 1), validation_error);  // the other two axes differ
    EXPECT_THROW(add_coalescing(a, random_tensor(gen, {3, 4, 3}, 4), 1), validation_error);  // ranks differ
    EXPECT_THROW(add_coalescing(a, a, -1), validation_error);
    EXPECT_THROW(add_coalescing(a, a, 3), validation_error);
}

TEST(CanonicalProperty, RandomTrialsAgainstScalarOracles) {  // test_canonical.cpp (100 random trials)
    std::mt19937 gen(100);
    for (int trial = 0; trial < 100; ++trial) {
        const Dims3 d = random_dims(gen, 1, 6);
        std::uniform_int_distribution<Index> rk(0, 5);
        CanonicalTensor3 a = random_tensor(gen, d, rk(gen)), b = random_tensor(gen, d, rk(gen));
        const DenseTensor3 da = scalar_oracle(a), db = scalar_oracle(b);
        const DenseTensor3 ga = densify(a);
        EXPECT_LE(max_norm_diff(ga, da), 1e-13 * std::max(1.0, max_abs(da)));
        double dot = 0.0, na = 0.0, nb = 0.0;
        for (Index e = 0; e < da.size(); ++e) {
            dot += da.data()[e] * db.data()[e];
            na += da.data()[e] * da.data()[e];
            nb += db.data()[e] * db.data()[e];
        }
        EXPECT_LE(std::abs(scalar_product(a, b) - dot), 1e-11 * std::max(1.0, std::sqrt(na * nb)));
        std::uniform_int_distribution<Index> pi(0, d[0] - 1), pj(0, d[1] - 1), pk(0, d[2] - 1);
        const Index i = pi(gen), j = pj(gen), k = pk(gen);
        EXPECT_LE(std::abs(eval_point(a, i, j, k) - da(i, j, k)), 1e-13 * std::max(1.0, max_abs(da)));
    }
}

TEST(ScalarProduct, SelfProductIsNonNegative) {  // test_canonical.cpp:124-131
    std::mt19937 gen(14);
    for (int trial = 0; trial < 20; ++trial) {
        CanonicalTensor3 a = random_tensor(gen, random_dims(gen), 4);
        const DenseTensor3 da = scalar_oracle(a);
        double n2 = 0.0;
        for (Index e = 0; e < da.size(); ++e) n2 += da.data()[e] * da.data()[e];
        EXPECT_GE(scalar_product(a, a), -1e-12 * std::max(1.0, n2));
    }
}

// ------------------------------------------------------------------ lattice specification and windows
TEST(LatticeSpec, ValidatesShapeAndCharges) {  // test_lattice.cpp:103-109
    EXPECT_NO_THROW(make_spec({1, 3, 2}, 8, 2.0, {Charge{{0.0, 0.0, 0.0}, 1.0}}).validate());
    EXPECT_THROW(make_spec({1, 0, 2}, 8, 2.0, {Charge{{0.0, 0.0, 0.0}, 1.0}}).validate(), validation_error);
    EXPECT_THROW(make_spec({1, 1, 1}, 8, 2.0, {}).validate(), validation_error);
    EXPECT_THROW(make_spec({1, 1, 1}, 8, 2.0, {Charge{{0.0, 0.0, 0.0}, 0.0}}).validate(), validation_error);
    EXPECT_THROW(make_spec({1, 1, 1}, 7, 2.0, {Charge{{0.0, 0.0, 0.0}, 1.0}}).validate(), validation_error);
}

TEST(DirectSum, EquivalentChargePlacementsCoincideBitwise) {  // test_lattice.cpp:174-187
    // A charge on the face between cells k and k+1 is vertex n of cell k or vertex 0 of cell k+1:
    // both descriptions must select the same master window.
    const Index n = 8, N = 3 * n;
    EXPECT_EQ(window_start_box(N, n, n, 1), window_start_box(N, n, 0, 2));
    LatticeSpec spec = make_spec({3, 1, 1}, n, 2.0, {Charge{{1.0, 0.0, 0.0}, 1.0}});
    QuadratureRule rule = sinc_quadrature(1e-4, spec.unit.h(), std::sqrt(3.0) * 6.0, 8, 1.0);
    CanonicalTensor3 master = build_lattice_master(spec, rule);
    for (Index q = 0; q < master.rank(); q += 3) {
        Vector lo = window_apply(master.factor(0).col(q), WindowOp(window_start_box(N, n, n, 1), 2 * N, N));
        Vector hi = window_apply(master.factor(0).col(q), WindowOp(window_start_box(N, n, 0, 2), 2 * N, N));
        EXPECT_TRUE((lo.array() == hi.array()).all());
    }
}

// ------------------------------------------------------------------ Gaussian bases, potential matrix
TEST(GaussianBasis, SamplesCenteredWideAndRejects) {  // test_project.cpp:32-88
    GridSpec g{2.0, 8};
    Rank1Basis b = sample_gaussian_basis(g, {GaussianBasisSpec{{0.0, 0.25, -0.5}, 0.3}, GaussianBasisSpec{{0.0, 0.0, 0.0}, 1e300}});
    ASSERT_EQ(b.size(), 2);
    EXPECT_EQ(b.n, 8);
    EXPECT_EQ(b.h, 0.25);
    for (Index i = 0; i < 8; ++i) {
        const double d = g.midpoint(i) - 0.25;
        EXPECT_NEAR(b.funcs[0][1][i], std::exp(-d * d / (2.0 * 0.09)), 1e-15);  // midpoint samples
        EXPECT_EQ(b.funcs[0][0][i], b.funcs[0][0][7 - i]);                     // centred: exactly even
        for (int l = 0; l < 3; ++l) EXPECT_EQ(b.funcs[1][static_cast<size_t>(l)][i], 1.0);  // huge width: ones
    }
    EXPECT_THROW(sample_gaussian_basis(g, {}), validation_error);
    EXPECT_THROW(sample_gaussian_basis(g, {GaussianBasisSpec{{0.0, 0.0, 0.0}, 0.0}}), validation_error);
    EXPECT_THROW(sample_gaussian_basis(g, {GaussianBasisSpec{{0.0, 0.0, 0.0}, -1.0}}), validation_error);
    EXPECT_THROW(sample_gaussian_basis(g, {GaussianBasisSpec{{std::numeric_limits<double>::quiet_NaN(), 0.0, 0.0}, 1.0}}),
                 validation_error);
}

TEST(PotentialMatrix, MatchesDenseTripleLoopOracle) {  // test_project.cpp:112-125
    std::mt19937 gen(61);
    GridSpec g{2.0, 6};
    CanonicalTensor3 P = random_tensor(gen, {6, 6, 6}, 3);
    std::vector<GaussianBasisSpec> specs{GaussianBasisSpec{{0.1, -0.2, 0.3}, 0.4}, GaussianBasisSpec{{-0.3, 0.0, 0.2}, 0.6},
                                         GaussianBasisSpec{{0.0, 0.5, -0.5}, 0.8}};
    Rank1Basis basis = sample_gaussian_basis(g, specs);
    for (bool vol : {false, true}) {
        Matrix V = potential_matrix(basis, P, vol);
        const DenseTensor3 dp = scalar_oracle(P);
        const double scale = vol ? g.h() * g.h() * g.h() : 1.0;
        for (Index a = 0; a < 3; ++a)
            for (Index c = 0; c < 3; ++c) {
                double want = 0.0;
                for (Index k = 0; k < 6; ++k)
                    for (Index j = 0; j < 6; ++j)
                        for (Index i = 0; i < 6; ++i)
                            want += dp(i, j, k) * basis.funcs[static_cast<size_t>(a)][0][i] * basis.funcs[static_cast<size_t>(c)][0][i] *
                                    basis.funcs[static_cast<size_t>(a)][1][j] * basis.funcs[static_cast<size_t>(c)][1][j] *
                                    basis.funcs[static_cast<size_t>(a)][2][k] * basis.funcs[static_cast<size_t>(c)][2][k];
                EXPECT_NEAR(V(a, c), scale * want, 1e-11 * std::max(1.0, std::abs(scale * want)));
            }
    }
    CanonicalTensor3 wrong = random_tensor(gen, {6, 6, 5}, 2);  // basis grid 6^3, potential 6x6x5
    EXPECT_THROW(potential_matrix(basis, wrong, false), validation_error);
}

// ------------------------------------------------------------------ series and extrapolation
TEST(Richardson, EliminatesLeadingGrowthExactly) {  // test_lattice.cpp (Richardson)
    const double a = 1.75, c = 0.5, L = 8.0;
    // p(L) = a + c L (linear growth), p(2L) = a + 2 c L
    EXPECT_EQ(richardson_extrapolate(a + c * L, a + 2.0 * c * L, RichardsonOrder::linear), a);
    // p(L) = a + c L^2 (quadratic growth), p(2L) = a + 4 c L^2
    EXPECT_EQ(richardson_extrapolate(a + c * L * L, a + 4.0 * c * L * L, RichardsonOrder::quadratic), a);
}

TEST(Series, ShapesAndRejectsBadLists) {  // test_lattice.cpp (Series)
    EXPECT_TRUE((series_cells(SeriesKind::line, 5) == std::array<Index, 3>{5, 1, 1}));
    EXPECT_TRUE((series_cells(SeriesKind::plane, 5) == std::array<Index, 3>{5, 5, 1}));
    EXPECT_TRUE((series_cells(SeriesKind::cube, 5) == std::array<Index, 3>{5, 5, 5}));
    GridSpec unit{2.0, 8};
    EXPECT_THROW(center_value_series(SeriesKind::line, {}, unit, 1e-4), validation_error);
    EXPECT_THROW(center_value_series(SeriesKind::line, {2, 2}, unit, 1e-4), validation_error);
    EXPECT_THROW(center_value_series(SeriesKind::line, {4, 2}, unit, 1e-4), validation_error);
}

// ------------------------------------------------------------------ bundle / CSV formats
std::string golden_dir() {
    const char* d = std::getenv("LATSUM_GOLDEN_DIR");
    return d ? d : "tests/golden";
}

std::string tmp_path(const std::string& name) {
    return "/tmp/latsum_dropin_" + std::to_string(static_cast<long>(::getpid())) + "_" + name;
}

TEST(Bundle, RoundTripIsExact) {  // test_bundle.cpp:33-58
    std::mt19937 gen(71);
    TensorBundle b;
    b.tensor = random_tensor(gen, {5, 4, 3}, 3);
    b.h = 0.125;
    b.origin = {-1.0, 0.5, 2.0};
    const std::string path = tmp_path("rt.bin");
    save_bundle(path, b);
    TensorBundle r = load_bundle(path);
    EXPECT_EQ(r.h, b.h);
    EXPECT_TRUE(r.origin == b.origin);
    EXPECT_EQ(r.tensor.rank(), 3);
    for (int l = 0; l < 3; ++l) EXPECT_TRUE((r.tensor.factor(l).array() == b.tensor.factor(l).array()).all());
    EXPECT_TRUE((r.tensor.weights().array() == b.tensor.weights().array()).all());
    std::remove(path.c_str());
}

TEST(Bundle, ReadsAndRewritesReferenceFileBitForBit) {  // bundle.hpp:18-94 (reference-written fixture)
    const std::string ref = golden_dir() + "/ref_bundle_mc_box.bin";
    TensorBundle b = load_bundle(ref);
    EXPECT_TRUE((b.tensor.dims() == Dims3{24, 16, 16}));
    EXPECT_EQ(b.tensor.rank(), 63);
    EXPECT_EQ(b.h, 0.25);
    const std::string path = tmp_path("rewrite.bin");
    save_bundle(path, b);
    std::ifstream x(ref, std::ios::binary), y(path, std::ios::binary);
    std::string bx((std::istreambuf_iterator<char>(x)), std::istreambuf_iterator<char>());
    std::string by((std::istreambuf_iterator<char>(y)), std::istreambuf_iterator<char>());
    EXPECT_TRUE(bx == by);
    // the loaded tensor expands on the GPU like any other
    DenseTensor3 d = densify(b.tensor);
    EXPECT_LT(rel_diff(d, scalar_oracle(b.tensor)), 1e-13);
    std::remove(path.c_str());
}

TEST(Bundle, RejectsBadFiles) {  // test_bundle.cpp:60-86
    const std::string path = tmp_path("bad.bin");
    {
        std::ofstream o(path, std::ios::binary);
        o << "NOTABUNDLE";
    }
    EXPECT_THROW(load_bundle(path), validation_error);
    {
        std::ofstream o(path, std::ios::binary);
        o.write(bundle_magic, 8);
        const std::int64_t hdr[4] = {2, 2, 2, 1};
        o.write(reinterpret_cast<const char*>(hdr), sizeof(hdr));
    }
    EXPECT_THROW(load_bundle(path), validation_error);  // truncated
    EXPECT_THROW(load_bundle(tmp_path("missing.bin")), validation_error);
    std::remove(path.c_str());
}

TEST(Csv, ReadsChargesAndBasis) {  // test_bundle.cpp:88-140
    const std::string c = tmp_path("charges.csv"), bpath = tmp_path("basis.csv"), bad = tmp_path("bad.csv");
    {
        std::ofstream o(c);
        o << "x,y,z,Z\n0,0,0,1\n\n0.25, -0.5, 0.75, 2.5\n";
    }
    std::vector<Charge> ch = read_charges_csv(c);
    ASSERT_EQ(ch.size(), 2u);
    EXPECT_EQ(ch[1].pos[1], -0.5);
    EXPECT_EQ(ch[1].Z, 2.5);
    {
        std::ofstream o(bpath);
        o << "0,0,0,0.5\n0.1,0.2,0.3,0.7\n-0.5,0,0,0.9\n";
    }
    std::vector<GaussianBasisSpec> bs = read_basis_csv(bpath);
    ASSERT_EQ(bs.size(), 3u);
    EXPECT_EQ(bs[2].sigma, 0.9);
    EXPECT_EQ(bs[2].center[0], -0.5);
    {
        std::ofstream o(bad);
        o << "1,2,3\n";
    }
    EXPECT_THROW(read_charges_csv(bad), validation_error);
    {
        std::ofstream o(bad);
        o << "1,2,3,4\nfoo,1,2,3\n";
    }
    EXPECT_THROW(read_charges_csv(bad), validation_error);
    {
        std::ofstream o(bad);
        o << "x,y,z,Z\n";
    }
    EXPECT_THROW(read_charges_csv(bad), validation_error);
    EXPECT_THROW(read_charges_csv(tmp_path("nope.csv")), validation_error);
    EXPECT_EQ(format_double(0.1), std::string("0.10000000000000001"));
    for (const auto& f : {c, bpath, bad}) std::remove(f.c_str());
}


TEST(FormatDouble, RoundTripsExactly) {  // bundle.hpp format_double
    std::mt19937_64 gen(9);
    std::uniform_real_distribution<double> u(-1e6, 1e6);
    const double specials[] = {0.0, -0.0, 1.0 / 3.0, 0.1, 1e-300, 6.02214076e23, std::numeric_limits<double>::max(),
                               std::numeric_limits<double>::denorm_min()};
    for (double x : specials) EXPECT_EQ(std::strtod(format_double(x).c_str(), nullptr), x);
    for (int e = 0; e < 200; ++e) {
        const double x = u(gen) * std::pow(10.0, static_cast<double>(static_cast<int>(gen() % 40) - 20));
        EXPECT_EQ(std::strtod(format_double(x).c_str(), nullptr), x);
    }
}

TEST(Bundle, RankZeroAndLatticeResultsRoundTrip) {  // test_bundle.cpp (rank zero, lattice results)
    const std::string path = tmp_path("r0.bin");
    TensorBundle z;
    z.tensor = CanonicalTensor3(Dims3{3, 2, 4});
    z.h = 0.5;
    save_bundle(path, z);
    TensorBundle zr = load_bundle(path);
    EXPECT_EQ(zr.tensor.rank(), 0);
    EXPECT_TRUE((zr.tensor.dims() == Dims3{3, 2, 4}));
    EXPECT_EQ(zr.h, 0.5);
    // a lattice sum written and read back densifies to the same grid, bit for bit
    LatticeSpec spec = make_spec({2, 1, 2}, 8, 2.0, {Charge{{0.25, 0.0, -0.5}, 1.5}});
    QuadratureRule rule = sinc_quadrature(1e-4, spec.unit.h(), std::sqrt(3.0) * 4.0, 8, 1.0);
    SumResult sum = assembled_box_sum(spec, build_lattice_master(spec, rule));
    TensorBundle b;
    b.tensor = sum.tensor;
    b.h = spec.unit.h();
    b.origin = {-2.0 + 0.125, -1.0 + 0.125, -2.0 + 0.125};
    save_bundle(path, b);
    TensorBundle br = load_bundle(path);
    EXPECT_EQ(br.origin[0], b.origin[0]);
    EXPECT_EQ(max_norm_diff(densify(br.tensor), densify(sum.tensor)), 0.0);
    std::remove(path.c_str());
}

// ------------------------------------------------------------------ QTT (GPU TT-SVD sweep)
Vector qtt_random(std::mt19937& gen, Index n) {
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    Vector v(n);
    for (Index i = 0; i < n; ++i) v[i] = dist(gen);
    return v;
}
double qtt_rel_err(const QTTVector& t, const Vector& v) {
    const Vector r = qtt_reconstruct(t);
    double num = 0.0, den = 0.0;
    for (Index i = 0; i < v.size(); ++i) {
        num += (r[i] - v[i]) * (r[i] - v[i]);
        den += v[i] * v[i];
    }
    return std::sqrt(num / den);
}

TEST(QttBasics, HelpersAndBadInput) {  // test_qtt.cpp:22-39
    EXPECT_TRUE(is_power_of_two(1024));
    EXPECT_FALSE(is_power_of_two(3));
    EXPECT_FALSE(is_power_of_two(-4));
    EXPECT_EQ(log2_exact(4096), 12);
    EXPECT_THROW(qtt_compress(Vector::Ones(6), 1e-8), validation_error);
    EXPECT_THROW(qtt_compress(Vector::Ones(1), 1e-8), validation_error);
    EXPECT_THROW(qtt_compress(Vector::Ones(8), 0.0), validation_error);
    EXPECT_THROW(unfolding_rank_profile(Vector::Ones(6), 1e-8), validation_error);
}

TEST(QttRanks, KnownRanks) {  // test_qtt.cpp:41-89: constant, geometric, impulse, sinusoid, cubic
    QTTVector t = qtt_compress(Vector::Constant(256, 3.25), 1e-12);
    EXPECT_EQ(qtt_rank_profile(t).max_rank, 1);
    EXPECT_LT(qtt_rel_err(t, Vector::Constant(256, 3.25)), 1e-12);
    Vector g(512);
    for (Index i = 0; i < 512; ++i) g[i] = std::pow(0.99, static_cast<double>(i));
    t = qtt_compress(g, 1e-12);
    EXPECT_EQ(qtt_rank_profile(t).max_rank, 1);
    EXPECT_LT(qtt_rel_err(t, g), 1e-12);
    for (Index pos : {Index{0}, Index{7}, Index{100}, Index{255}}) {
        Vector v = Vector::Zero(256);
        v[pos] = 1.0;
        t = qtt_compress(v, 1e-12);
        EXPECT_EQ(qtt_rank_profile(t).max_rank, 1);
        EXPECT_LT(qtt_rel_err(t, v), 1e-13);
    }
    for (double omega : {0.01, 0.37, 2.1}) {
        Vector v(1024);
        for (Index i = 0; i < 1024; ++i) v[i] = std::sin(omega * static_cast<double>(i) + 0.3);
        t = qtt_compress(v, 1e-10);
        EXPECT_LE(qtt_rank_profile(t).max_rank, 2);
        EXPECT_LT(qtt_rel_err(t, v), 1e-10);
    }
    Vector p(2048);
    for (Index i = 0; i < 2048; ++i) {
        const double x = static_cast<double>(i) / 2048.0;
        p[i] = ((x - 0.4) * x + 0.25) * x - 1.0;
    }
    t = qtt_compress(p, 1e-11);
    EXPECT_LE(qtt_rank_profile(t).max_rank, 4);
    EXPECT_LT(qtt_rel_err(t, p), 1e-11);
}

TEST(QttRanks, RandomVectorHasMaximalRanks) {  // test_qtt.cpp:91-102
    std::mt19937 gen(77);
    Vector v = qtt_random(gen, 256);
    QTTVector t = qtt_compress(v, 1e-14);
    const std::vector<Index> ranks = t.ranks();
    ASSERT_EQ(ranks.size(), 7u);
    for (std::size_t k = 0; k < ranks.size(); ++k)
        EXPECT_EQ(ranks[k], std::min(Index{1} << (k + 1), Index{256} >> (k + 1)));
    EXPECT_LT(qtt_rel_err(t, v), 1e-12);
}

TEST(QttCompress, HonorsErrorContractAndCompresses) {  // test_qtt.cpp:104-130
    std::mt19937 gen(78);
    for (double eps : {1e-2, 1e-4, 1e-8}) {
        for (int trial = 0; trial < 7; ++trial) {
            Vector v = qtt_random(gen, 1024);
            for (Index i = 0; i < 1024; ++i)
                v[i] = std::exp(-std::pow((static_cast<double>(i) - 512.0) / 150.0, 2)) + 0.01 * v[i];
            QTTVector t = qtt_compress(v, eps);
            EXPECT_LE(qtt_rel_err(t, v), eps);
        }
    }
    Vector s(4096);
    for (Index i = 0; i < 4096; ++i) {
        const double x = (static_cast<double>(i) + 0.5) / 4096.0 * 10.0 - 5.0;
        s[i] = std::exp(-x * x);
    }
    QTTVector t = qtt_compress(s, 1e-6);
    EXPECT_LE(qtt_rank_profile(t).max_rank, 25);
    EXPECT_LT(qtt_rank_profile(t).avg_rank, 15.0);
}

TEST(UnfoldingRanks, KnownCasesAndSweepDominates) {  // test_qtt.cpp:132-160
    for (Index r : unfolding_rank_profile(Vector::Constant(128, 2.0), 1e-10)) EXPECT_EQ(r, 1);
    std::mt19937 gen(79);
    Vector v = qtt_random(gen, 128);
    std::vector<Index> rr = unfolding_rank_profile(v, 1e-14);
    ASSERT_EQ(rr.size(), 6u);
    for (std::size_t k = 0; k < rr.size(); ++k) EXPECT_EQ(rr[k], std::min(Index{1} << (k + 1), Index{128} >> (k + 1)));
    EXPECT_EQ(max_unfolding_rank(v, 0.999), 1);
    std::mt19937 gen2(80);
    for (int trial = 0; trial < 5; ++trial) {
        Vector w = qtt_random(gen2, 512);
        for (Index i = 0; i < 512; ++i) w[i] += 3.0 * std::cos(0.02 * static_cast<double>(i));
        std::vector<Index> sweep = qtt_compress(w, 1e-4).ranks(), intrinsic = unfolding_rank_profile(w, 1e-4);
        ASSERT_EQ(sweep.size(), intrinsic.size());
        for (std::size_t k = 0; k < sweep.size(); ++k) EXPECT_GE(sweep[k], intrinsic[k]);
    }
}

TEST(Modulation, BoundsHoldAndShapesChecked) {  // test_qtt.cpp:162-201
    const Index block = 64, n_blocks = 8, total = block * n_blocks;
    Vector x0(block);
    for (Index i = 0; i < block; ++i) x0[i] = std::exp(-std::pow((static_cast<double>(i) + 0.5 - 32.0) / 6.0, 2));
    Vector F(total);
    for (Index i = 0; i < total; ++i) {
        const double tpos = (static_cast<double>(i) + 0.5) / static_cast<double>(total);
        F[i] = std::sin(2.0 * M_PI * 3.0 * tpos + 0.4) + 1.2;
    }
    ModulationReport rep = block_modulated_vector(x0, n_blocks, F, 1e-10);
    EXPECT_TRUE(rep.tiling_bound_ok);
    EXPECT_TRUE(rep.product_bound_ok);
    EXPECT_LE(rep.rfx, rep.rF * rep.r0);
    for (Index blk = 0; blk < n_blocks; ++blk)
        for (Index i = 0; i < block; ++i) EXPECT_EQ(rep.x[blk * block + i], x0[i]);
    ModulationReport id = block_modulated_vector(x0, 1, Vector::Ones(64), 1e-10);
    EXPECT_EQ(id.rF, 1);
    EXPECT_EQ(id.rx, id.r0);
    EXPECT_THROW(block_modulated_vector(Vector::Ones(6), 2, Vector::Ones(12), 1e-8), validation_error);
    EXPECT_THROW(block_modulated_vector(Vector::Ones(64), 3, Vector::Ones(192), 1e-8), validation_error);
    EXPECT_THROW(block_modulated_vector(Vector::Ones(64), 2, Vector::Ones(100), 1e-8), validation_error);
}

TEST(AssembledQtt, ReportsPaddingAndRebuild) {  // test_qtt.cpp:203-265
    LatticeSpec spec = make_spec({2, 1, 1}, 8, 2.0, {Charge{}});
    QuadratureRule rule = calibrate_for_lattice(spec, 1e-4);
    CanonicalTensor3 master = build_lattice_master(spec, rule);
    AssembledQttResult res = assembled_qtt_sum(spec, master, 1e-8, &rule);
    const Index R = rule.node_count();
    ASSERT_EQ(res.columns.size(), static_cast<std::size_t>(3 * R));
    EXPECT_TRUE((res.padded_len == Dims3{16, 8, 8}));
    for (const QttColumnReport& rep : res.reports) {
        EXPECT_LE(rep.rec_err, 1e-8);
        EXPECT_TRUE(rep.regime == 0 || rep.regime == 1);
    }
    for (const QttColumnReport& rep : assembled_qtt_sum(spec, master, 1e-8).reports) EXPECT_EQ(rep.regime, -1);
    LatticeSpec s3 = make_spec({3, 1, 1}, 6, 2.0, {Charge{}});
    QuadratureRule r3 = calibrate_for_lattice(s3, 1e-4);
    CanonicalTensor3 m3 = build_lattice_master(s3, r3);
    EXPECT_TRUE((assembled_qtt_sum(s3, m3, 1e-8, &r3).padded_len == Dims3{32, 8, 8}));
    EXPECT_THROW(assembled_qtt_sum(s3, m3, 1e-8, &r3, 16), resource_guard_error);
    // rebuilding the factors from the trains reproduces the assembled tensor (test_qtt.cpp:239-265)
    const double eps = 1e-8;
    LatticeSpec s2 = make_spec({2, 2, 2}, 4, 2.0, {Charge{}});
    QuadratureRule r2 = calibrate_for_lattice(s2, 1e-4);
    CanonicalTensor3 m2 = build_lattice_master(s2, r2);
    SumResult assembled = assembled_box_sum(s2, m2);
    AssembledQttResult q2 = assembled_qtt_sum(s2, m2, eps, &r2);
    const Index R2 = r2.node_count();
    std::array<Matrix, 3> factors;
    for (int axis = 0; axis < 3; ++axis) {
        const Index N = s2.target_cells(axis);
        factors[static_cast<std::size_t>(axis)].resize(N, R2);
        for (Index q = 0; q < R2; ++q) {
            const Vector rec = qtt_reconstruct(q2.columns[static_cast<std::size_t>(axis * R2 + q)]);
            for (Index i = 0; i < N; ++i) factors[static_cast<std::size_t>(axis)](i, q) = rec[i];
        }
    }
    CanonicalTensor3 rebuilt(std::move(factors), Vector(assembled.tensor.weights()));
    StreamDiff d = max_norm_diff_canonical(rebuilt, assembled.tensor);
    EXPECT_LE(d.max_diff, 10.0 * eps * d.max_abs_b);
}

TEST(GaussianRankGrowth, LogarithmicInTolerance) {  // test_qtt.cpp:267-290
    const Index N = Index{1} << 12;
    std::vector<double> lx, mr;
    for (double eps : {1e-3, 1e-5, 1e-7}) {
        const double a = std::sqrt(2.0) * std::sqrt(std::log(1.0 / eps));
        Vector v(N);
        for (Index i = 0; i < N; ++i) {
            const double x = (static_cast<double>(i) + 0.5) / static_cast<double>(N) * 2.0 * a - a;
            v[i] = std::exp(-x * x / 2.0);
        }
        const Index r = max_unfolding_rank(v, eps);
        lx.push_back(std::log(1.0 / eps));
        mr.push_back(static_cast<double>(r));
        EXPECT_LE(r, 25);
    }
    const double slope = (mr[2] - mr[0]) / (lx[2] - lx[0]);
    EXPECT_GE(slope, 0.0);
    EXPECT_LE(slope, 4.0);
}

int main(int argc, char** argv) { return minitest::run_all(argc, argv); }
