// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C entry points over the reference's OWN hot-path headers, compiled
// unmodified from /root/reference/proj/include/latsum/ against the
// self-written Eigen subset in include/eigen_compat (Eigen3 is absent from
// the image). oracle/Makefile builds this into oracle/_ref/libref_latsum.so,
// which (a) pins the C restatement oracle/latsum_oracle.c, (b) generates the
// golden vectors in tests/golden/, and (c) is the CPU baseline
// ("kind": "reference") that bench.py --impl reference times on the host
// cores. Signatures mirror oracle/latsum_oracle.h with the ref_ prefix.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "latsum/bundle.hpp"
#include "latsum/canonical.hpp"
#include "latsum/errors.hpp"
#include "latsum/grid.hpp"
#include "latsum/lattice.hpp"
#include "latsum/newton.hpp"
#include "latsum/parallel.hpp"
#include "latsum/project.hpp"
#include "latsum/quadrature.hpp"

using namespace latsum;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const validation_error& e) {
        g_err = e.what();
        return 2;
    } catch (const resource_guard_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

Matrix to_matrix(const double* p, Index r, Index c) {
    Matrix m(r, c);
    if (r * c) std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(r * c));
    return m;
}
Vector to_vector(const double* p, Index n) {
    Vector v(n);
    if (n) std::memcpy(v.data(), p, sizeof(double) * static_cast<size_t>(n));
    return v;
}
void from_matrix(const Matrix& m, double* out) {
    if (m.size()) std::memcpy(out, m.data(), sizeof(double) * static_cast<size_t>(m.size()));
}
QuadratureRule make_rule(const double* tau, const double* w, int R) {
    QuadratureRule rule;
    rule.M = (R - 1) / 2;
    rule.exponents = to_vector(tau, R);
    rule.weights = to_vector(w, R);
    rule.nodes = Vector::Zero(R);
    return rule;
}
LatticeSpec make_spec(const int64_t L[3], int64_t n, double b, const double* charges, int M0) {
    LatticeSpec spec;
    spec.L = {L[0], L[1], L[2]};
    spec.unit = GridSpec(b, n);
    for (int nu = 0; nu < M0; ++nu)
        spec.charges.push_back(Charge{{charges[4 * nu], charges[4 * nu + 1], charges[4 * nu + 2]},
                                      charges[4 * nu + 3]});
    return spec;
}
CanonicalTensor3 make_tensor(const int64_t d[3], int R, const double* A, const double* B,
                             const double* C, const double* w) {
    std::array<Matrix, 3> f{to_matrix(A, d[0], R), to_matrix(B, d[1], R), to_matrix(C, d[2], R)};
    return CanonicalTensor3(CanonicalTensor3::trusted_components_t{}, std::move(f), to_vector(w, R));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { set_max_threads(n); }
int ref_max_threads() { return max_threads(); }

int ref_sinc_quadrature(double eps, double a_min, double a_max, int M, double C0, double* nodes,
                        double* exponents, double* weights, double* step) {
    return guarded([&] {
        QuadratureRule r = sinc_quadrature(eps, a_min, a_max, M, C0);
        from_matrix(r.exponents, exponents);
        from_matrix(r.weights, weights);
        if (nodes) from_matrix(r.nodes, nodes);
        if (step) *step = r.step;
    });
}

double ref_quadrature_value(const double* tau, const double* w, int R, double r) {
    return quadrature_value(make_rule(tau, w, R), r);
}

int ref_gaussian_sample_vector(int64_t len, double h, double t, double* out) {
    return guarded([&] { from_matrix(gaussian_sample_vector(len, h, t), out); });
}

int ref_gaussian_moment_vector(double b, int64_t n, double t, int doubled, double* out) {
    return guarded([&] { from_matrix(gaussian_moment_vector(GridSpec(b, n), t, doubled != 0), out); });
}

// mode 0: build_lattice_master (midpoint); mode 1: erf master from gaussian_moment_vector
// columns on GridSpec(L_l * b, L_l * n), doubled.
int ref_lattice_master(int mode, const int64_t L[3], int64_t n, double b, const double* tau,
                       const double* w, int R, const double* charges, int M0, double* f0, double* f1,
                       double* f2, double* time_ms) {
    return guarded([&] {
        const LatticeSpec spec = make_spec(L, n, b, charges, M0);
        const QuadratureRule rule = make_rule(tau, w, R);
        const auto t0 = std::chrono::steady_clock::now();
        double* f[3] = {f0, f1, f2};
        if (mode == 0) {
            CanonicalTensor3 m = build_lattice_master(spec, rule);
            for (int l = 0; l < 3; ++l) from_matrix(m.factor(l), f[l]);
        } else {
            spec.validate();
            for (int l = 0; l < 3; ++l) {
                const GridSpec g(static_cast<double>(L[l]) * b, L[l] * n);
                Matrix fl(2 * L[l] * n, R);
                for (int q = 0; q < R; ++q) fl.col(q) = gaussian_moment_vector(g, tau[q], true);
                from_matrix(fl, f[l]);
            }
        }
        if (time_ms)
            *time_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

// assembled_box_sum / assembled_periodic_sum (lattice.hpp:303-312) on a given master.
int ref_assembled_sum(int periodic, const int64_t L[3], int64_t n, double b, const double* charges,
                      int M0, const double* f0, const double* f1, const double* f2, const double* w,
                      int R, double* o0, double* o1, double* o2, double* wout, double* time_ms) {
    return guarded([&] {
        const LatticeSpec spec = make_spec(L, n, b, charges, M0);
        const int64_t d[3] = {2 * L[0] * n, 2 * L[1] * n, 2 * L[2] * n};
        const CanonicalTensor3 master = make_tensor(d, R, f0, f1, f2, w);
        SumResult s = periodic ? assembled_periodic_sum(spec, master) : assembled_box_sum(spec, master);
        from_matrix(s.tensor.factor(0), o0);
        from_matrix(s.tensor.factor(1), o1);
        from_matrix(s.tensor.factor(2), o2);
        from_matrix(s.tensor.weights(), wout);
        if (time_ms) *time_ms = s.time_ms;
    });
}

int ref_direct_sum(const int64_t L[3], int64_t n, double b, const double* charges, int M0,
                   const double* f0, const double* f1, const double* f2, const double* w, int R,
                   double* o0, double* o1, double* o2, double* wout) {
    return guarded([&] {
        const LatticeSpec spec = make_spec(L, n, b, charges, M0);
        const int64_t d[3] = {2 * L[0] * n, 2 * L[1] * n, 2 * L[2] * n};
        SumResult s = direct_sum(spec, make_tensor(d, R, f0, f1, f2, w));
        from_matrix(s.tensor.factor(0), o0);
        from_matrix(s.tensor.factor(1), o1);
        from_matrix(s.tensor.factor(2), o2);
        from_matrix(s.tensor.weights(), wout);
    });
}

// detail::densify_slab (canonical.hpp:241-246) for k in [k0, k1), parallel over k like densify.
int ref_densify_slabs(int64_t n1, int64_t n2, int64_t n3, int R, const double* A, const double* B,
                      const double* C, const double* w, int64_t k0, int64_t k1, double* out) {
    return guarded([&] {
        const int64_t d[3] = {n1, n2, n3};
        const CanonicalTensor3 t = make_tensor(d, R, A, B, C, w);
        parallel_for(k1 - k0, [&](std::int64_t kk) {
            Matrix slab;
            detail::densify_slab(t, static_cast<Index>(k0 + kk), slab);
            std::memcpy(out + kk * n1 * n2, slab.data(), sizeof(double) * static_cast<size_t>(n1 * n2));
        });
    });
}

// densify (canonical.hpp:251-266) with its guard.
int ref_densify(int64_t n1, int64_t n2, int64_t n3, int R, const double* A, const double* B,
                const double* C, const double* w, uint64_t guard, double* out) {
    return guarded([&] {
        const int64_t d[3] = {n1, n2, n3};
        DenseTensor3 dt = densify(make_tensor(d, R, A, B, C, w), guard);
        from_matrix(dt.data(), out);
    });
}

// Streaming timing harness for the CPU baseline: densify_slab over slabs [k0,k1) into a reused
// per-thread slab buffer, fused with the separable rho reduction.
// Returns the functional; *ms receives the wall time.
double ref_stream_functional(int64_t n1, int64_t n2, int64_t n3, int R, const double* A,
                             const double* B, const double* C, const double* w, const double* r1,
                             const double* r2, const double* r3, int64_t k0, int64_t k1, double* ms) {
    const int64_t d[3] = {n1, n2, n3};
    const CanonicalTensor3 t = make_tensor(d, R, A, B, C, w);
    std::vector<double> part(static_cast<size_t>(k1 - k0), 0.0);
    const auto t0 = std::chrono::steady_clock::now();
    parallel_for(k1 - k0, [&](std::int64_t kk) {
        Matrix slab;
        detail::densify_slab(t, static_cast<Index>(k0 + kk), slab);
        double sk = 0.0;
        for (Index j = 0; j < n2; ++j) {
            double sj = 0.0;
            for (Index i = 0; i < n1; ++i) sj += slab(i, j) * r1[i];
            sk += sj * r2[j];
        }
        part[static_cast<size_t>(kk)] = sk * r3[k0 + kk];
    });
    double total = 0.0;
    for (double p : part) total += p;
    if (ms) *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return total;
}

// Streaming expansion harness: densify_slab over [k0,k1), each slab copied into out (host grid
// storage), as densify does (canonical.hpp:260-264) but without the 2^27 guard.
int ref_expand_into(int64_t n1, int64_t n2, int64_t n3, int R, const double* A, const double* B,
                    const double* C, const double* w, int64_t k0, int64_t k1, double* out, double* ms) {
    return guarded([&] {
        const int64_t d[3] = {n1, n2, n3};
        const CanonicalTensor3 t = make_tensor(d, R, A, B, C, w);
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for(k1 - k0, [&](std::int64_t kk) {
            Matrix slab;
            detail::densify_slab(t, static_cast<Index>(k0 + kk), slab);
            Eigen::Map<Matrix>(out + kk * n1 * n2, n1, n2) = slab;
        });
        if (ms) *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

double ref_eval_point(int64_t n1, int64_t n2, int64_t n3, int R, const double* A, const double* B,
                      const double* C, const double* w, int64_t i, int64_t j, int64_t k) {
    const int64_t d[3] = {n1, n2, n3};
    return eval_point(make_tensor(d, R, A, B, C, w), i, j, k);
}

double ref_scalar_product(int64_t n1, int64_t n2, int64_t n3, int Ra, const double* A0,
                          const double* A1, const double* A2, const double* wa, int Rb,
                          const double* B0, const double* B1, const double* B2, const double* wb) {
    const int64_t d[3] = {n1, n2, n3};
    return scalar_product(make_tensor(d, Ra, A0, A1, A2, wa), make_tensor(d, Rb, B0, B1, B2, wb));
}

int ref_max_norm_diff_canonical(int64_t n1, int64_t n2, int64_t n3, int Ra, const double* A0,
                                const double* A1, const double* A2, const double* wa, int Rb,
                                const double* B0, const double* B1, const double* B2,
                                const double* wb, double* max_diff, double* max_abs_b) {
    return guarded([&] {
        const int64_t d[3] = {n1, n2, n3};
        StreamDiff s = max_norm_diff_canonical(make_tensor(d, Ra, A0, A1, A2, wa),
                                               make_tensor(d, Rb, B0, B1, B2, wb));
        *max_diff = s.max_diff;
        *max_abs_b = s.max_abs_b;
    });
}

// sample_gaussian_basis (project.hpp:30-57) for nb functions: centers nb x 3, sigmas nb;
// out nb x 3 x n.
int ref_sample_gaussian_basis(double b, int64_t n, int nb, const double* centers,
                              const double* sigmas, double* out) {
    return guarded([&] {
        std::vector<GaussianBasisSpec> specs(static_cast<size_t>(nb));
        for (int f = 0; f < nb; ++f)
            specs[f] = GaussianBasisSpec{{centers[3 * f], centers[3 * f + 1], centers[3 * f + 2]}, sigmas[f]};
        Rank1Basis basis = sample_gaussian_basis(GridSpec(b, n), specs);
        for (int f = 0; f < nb; ++f)
            for (int l = 0; l < 3; ++l)
                from_matrix(basis.funcs[f][l], out + (static_cast<size_t>(f) * 3 + l) * n);
    });
}

int ref_potential_matrix(double b, int64_t n, int nb, const double* centers, const double* sigmas,
                         int R, const double* P0, const double* P1, const double* P2,
                         const double* wp, int volume_element, double* V) {
    return guarded([&] {
        std::vector<GaussianBasisSpec> specs(static_cast<size_t>(nb));
        for (int f = 0; f < nb; ++f)
            specs[f] = GaussianBasisSpec{{centers[3 * f], centers[3 * f + 1], centers[3 * f + 2]}, sigmas[f]};
        Rank1Basis basis = sample_gaussian_basis(GridSpec(b, n), specs);
        const int64_t d[3] = {n, n, n};
        from_matrix(potential_matrix(basis, make_tensor(d, R, P0, P1, P2, wp), volume_element != 0), V);
    });
}

// save_bundle (bundle.hpp:33-54) of a tensor; used to produce the reference-written fixture.
int ref_save_bundle(const char* path, int64_t n1, int64_t n2, int64_t n3, int R, const double* A, const double* B,
                    const double* C, const double* w, double h, double ox, double oy, double oz) {
    return guarded([&] {
        const int64_t d[3] = {n1, n2, n3};
        TensorBundle b;
        b.tensor = make_tensor(d, R, A, B, C, w);
        b.h = h;
        b.origin = {ox, oy, oz};
        save_bundle(path, b);
    });
}

// calibrate_quadrature (newton.hpp:161-189) on GridSpec(b, n) with KernelTolerance(eps, a_min, a_max):
// returns M (or -1 on failure) and the winning C0; the rule itself follows from sinc_quadrature.
int ref_calibrate_quadrature(double b, int64_t n, double eps, double a_min, double a_max, int m_cap, double* C0,
                             int* trace_len) {
    int M = -1;
    int rc = guarded([&] {
        CalibrationTrace trace;
        QuadratureRule r = calibrate_quadrature(GridSpec(b, n), KernelTolerance(eps, a_min, a_max), &trace, m_cap);
        M = r.M;
        *C0 = r.C0;
        *trace_len = static_cast<int>(trace.entries.size());
    });
    return rc ? -rc : M;
}

// calibrate_for_lattice (lattice.hpp:118-126) for one unit charge at the cell centre.
int ref_calibrate_for_lattice(const int64_t L[3], int64_t n, double b, double eps, double* C0) {
    int M = -1;
    int rc = guarded([&] {
        const double ch[4] = {0.0, 0.0, 0.0, 1.0};
        QuadratureRule r = calibrate_for_lattice(make_spec(L, n, b, ch, 1), eps);
        M = r.M;
        *C0 = r.C0;
    });
    return rc ? -rc : M;
}

}  // extern "C"
