// latsum/quadrature.hpp -- drop-in for the reference's sinc quadrature
// (/root/reference/proj/include/latsum/quadrature.hpp:20-100):
//   1/r ~= sum_q w_q exp(-tau_q^2 r^2),  2M+1 nodes on a sinh-substituted axis.
// The rule (2M+1 scalars) is computed by the engine's host code
// (ls_sinc_quadrature) so the C++ API, the Python mirror and the benchmark
// share one implementation; quadrature_value is a scalar O(R) host loop.
#pragma once

#include <cmath>
#include <string>

#include "latsum/errors.hpp"
#include "latsum/grid.hpp"
#include "latsum_cuda.h"

namespace latsum {

struct QuadratureRule {
    int M = 0;          // half node count; 2M+1 nodes
    double C0 = 1.0;    // window depth (working tolerance eps * 10^-C0)
    double step = 0.0;  // spacing of the substitution nodes
    Vector nodes;       // substitution points, ascending
    Vector exponents;   // tau_q >= 0, ascending
    Vector weights;     // w_q > 0

    Index node_count() const { return static_cast<Index>(2 * M + 1); }
};

inline QuadratureRule sinc_quadrature(double eps, double a_min, double a_max, int M, double C0) {
    QuadratureRule rule;
    rule.M = M;
    rule.C0 = C0;
    const Index count = M >= 1 ? static_cast<Index>(2 * M + 1) : 1;
    rule.nodes.resize(count);
    rule.exponents.resize(count);
    rule.weights.resize(count);
    cuda::check(ls_sinc_quadrature(eps, a_min, a_max, M, C0, rule.nodes.data(), rule.exponents.data(),
                                   rule.weights.data(), &rule.step),
                "quadrature");
    return rule;
}

// Exponential sum at radius r, accumulated in node order.
inline double quadrature_value(const QuadratureRule& rule, double r) {
    double acc = 0.0;
    for (Index q = 0; q < rule.node_count(); ++q) {
        const double x = rule.exponents[q] * r;
        acc += rule.weights[q] * std::exp(-x * x);
    }
    return acc;
}

}  // namespace latsum
