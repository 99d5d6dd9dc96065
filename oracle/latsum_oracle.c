/* latsum_oracle.c -- TEST INFRASTRUCTURE ONLY (see latsum_oracle.h).
 *
 * A plain-C restatement of the reference hot path, written from the
 * reference's behaviour; every function cites the reference lines it follows
 * (paths relative to /root/reference/proj/include/latsum/). Compiled with
 * -ffp-contract=off so each expression rounds exactly as written.
 */
#include "latsum_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* quadrature.hpp:35-46: bisection for the smallest t with f(t) <= target. */
static double solve_decreasing(double (*f)(double), double target, double hi) {
    double lo = 1e-3;
    while (f(hi) > target) hi *= 1.5;
    for (int it = 0; it < 200; ++it) {
        double mid = 0.5 * (lo + hi);
        if (f(mid) <= target)
            hi = mid;
        else
            lo = mid;
    }
    return hi;
}
static double left_tail(double t) { return 2.0 * t * exp(-t); }       /* quadrature.hpp:62-63 */
static double right_tail(double t) { return sqrt(t) * exp(-t); }      /* quadrature.hpp:64-65 */

/* quadrature.hpp:50-89 */
int orc_sinc_quadrature(double eps, double a_min, double a_max, int M, double C0,
                        double* nodes, double* exponents, double* weights, double* step_out) {
    if (M < 1) return 2;
    if (!(eps > 0.0) || !(eps < 1.0)) return 2;
    if (!(a_min > 0.0) || !(a_min < a_max)) return 2;
    const double eps_w = eps * pow(10.0, -C0);
    const double r0 = a_min / a_max;
    const double t1 = solve_decreasing(left_tail, eps_w, 5.0);
    const double t2 = solve_decreasing(right_tail, eps_w * r0, 5.0);
    const double s1 = -log(2.0 * t1);
    const double s2 = 0.5 * log(t2 / (r0 * r0));
    const int count = 2 * M + 1;
    const double step = (s2 - s1) / (double)(count - 1);
    const double c = 4.0 / sqrt(M_PI);
    for (int j = 0; j < count; ++j) {
        const double s = s1 + step * (double)j;
        const double sh = sinh(s);
        const double G = sh > 30.0 ? sh : log1p(exp(sh));
        if (nodes) nodes[j] = s;
        exponents[j] = 2.0 * G / a_max;
        weights[j] = step * c * cosh(s) / (1.0 + exp(-(sh < 700.0 ? sh : 700.0))) / a_max;
    }
    if (step_out) *step_out = step;
    return 0;
}

/* quadrature.hpp:93-100 */
double orc_quadrature_value(const double* exponents, const double* weights, int R, double r) {
    double sum = 0.0;
    for (int j = 0; j < R; ++j) {
        const double tr = exponents[j] * r;
        sum += weights[j] * exp(-tr * tr);
    }
    return sum;
}

/* grid.hpp:32-34 */
static double midpoint(int64_t i, int64_t len, double h) {
    return ((double)i + 0.5 - (double)len / 2.0) * h;
}

/* newton.hpp:43-52 */
int orc_gaussian_sample_vector(int64_t len, double h, double t, double* out) {
    if (len < 2 || len % 2 != 0) return 2;
    for (int64_t i = 0; i < len; ++i) {
        const double x = t * midpoint(i, len, h);
        out[i] = exp(-x * x);
    }
    return 0;
}

/* newton.hpp:21-37 with GridSpec(b, n) (grid.hpp:14-29) */
int orc_gaussian_moment_vector(double b, int64_t n, double t, int doubled, double* out) {
    if (!(b > 0.0) || !isfinite(b) || n < 2 || n % 2 != 0) return 2;
    if (!(t >= 0.0) || !isfinite(t)) return 2;
    const int64_t len = doubled ? 2 * n : n;
    const double h = b / (double)n;
    if (t == 0.0) {
        for (int64_t i = 0; i < len; ++i) out[i] = h;
        return 0;
    }
    const double scale = sqrt(M_PI) / (2.0 * t);
    for (int64_t i = 0; i < len; ++i) {
        const double v1 = (double)(i + 1 - len / 2) * h;
        const double v0 = (double)(i - len / 2) * h;
        out[i] = scale * (erf(t * v1) - erf(t * v0));
    }
    return 0;
}

/* newton.hpp:34 and :50 call std::erf / std::exp: the host libm, element by element. */
int orc_libm_eval(int fn, const double* x, double* y, int64_t n) {
    if (fn != 0 && fn != 1) return 2;
    for (int64_t i = 0; i < n; ++i) y[i] = fn == 0 ? erf(x[i]) : exp(x[i]);
    return 0;
}

/* lattice.hpp:109-113 -> newton.hpp:57-75 (mode 0) or the erf master (mode 1). Axes with
 * equal length share the factor (newton.hpp:60-69), which here just recomputes bit-equal data. */
int orc_lattice_master(int mode, const int64_t L[3], int64_t n, double b, const double* tau, int R,
                       double* f0, double* f1, double* f2) {
    double* f[3] = {f0, f1, f2};
    if (n < 2 || n % 2 != 0 || !(b > 0.0)) return 2;
    const double h = b / (double)n;
    for (int l = 0; l < 3; ++l) {
        if (L[l] < 1) return 2;
        const int64_t len = 2 * L[l] * n;
        for (int q = 0; q < R; ++q) {
            int rc = mode == 0 ? orc_gaussian_sample_vector(len, h, tau[q], f[l] + (int64_t)q * len)
                               : orc_gaussian_moment_vector((double)L[l] * b, L[l] * n, tau[q], 1,
                                                            f[l] + (int64_t)q * len);
            if (rc) return rc;
        }
    }
    return 0;
}

/* lattice.hpp:57-68 */
int64_t orc_charge_grid_index(double b, int64_t n, double p) {
    const double h = b / (double)n;
    const double x = (p + b / 2.0) / h;
    const double r = round(x);
    if (fabs(x - r) > 1e-9 * (double)n || r < 0.0 || r > (double)n) return -1;
    return (int64_t)r;
}

/* lattice.hpp:98 */
int64_t orc_window_start_box(int64_t N, int64_t n, int64_t i_a, int64_t k) { return N - i_a - k * n; }
/* lattice.hpp:104-106 */
int64_t orc_window_start_periodic(int64_t N, int64_t n, int64_t i_a, int64_t k, int64_t L) {
    return N + (L / 2 - k) * n - i_a;
}

/* lattice.hpp:220-274. The reference's eight-stream blocking adds strictly left to right in
 * ascending k, which is the sequential recurrence acc = m[s0+i]; acc += m[s0-k*n+i]. */
int orc_assembled_axis(const double* master, int R, int M0, const int64_t* i_a, int64_t n,
                       int64_t L, int periodic, double* out) {
    const int64_t N = L * n;
    const int64_t mlen = 2 * N;
    const int64_t out_len = periodic ? n : N;
    for (int nu = 0; nu < M0; ++nu) {
        const int64_t s0 = periodic ? orc_window_start_periodic(N, n, i_a[nu], 0, L)
                                    : orc_window_start_box(N, n, i_a[nu], 0);
        for (int q = 0; q < R; ++q) {
            const double* base = master + (int64_t)q * mlen + s0;
            double* o = out + ((int64_t)nu * R + q) * out_len;
            for (int64_t i = 0; i < out_len; ++i) {
                double acc = base[i];
                for (int64_t k = 1; k < L; ++k) acc = acc + base[i - k * n];
                o[i] = acc;
            }
        }
    }
    return 0;
}

/* lattice.hpp:284-287 */
void orc_assembled_weights(const double* Z, int M0, const double* w, int R, double* w_out) {
    for (int nu = 0; nu < M0; ++nu)
        for (int q = 0; q < R; ++q) w_out[nu * R + q] = Z[nu] * w[q];
}

/* lattice.hpp:163-209 (column order: charge-major, then cell (k1,k2,k3) lexicographic, then q) */
int orc_direct_sum(const int64_t L[3], int64_t n, const int64_t* i_a, const double* Z, int M0,
                   const double* f0, const double* f1, const double* f2, const double* w, int R,
                   double* o0, double* o1, double* o2, double* wout) {
    const double* f[3] = {f0, f1, f2};
    double* o[3] = {o0, o1, o2};
    const int64_t cells = L[0] * L[1] * L[2];
    const int64_t groups = (int64_t)M0 * cells;
    for (int64_t g = 0; g < groups; ++g) {
        const int64_t nu = g / cells, kflat = g % cells;
        const int64_t kk[3] = {kflat / (L[1] * L[2]), (kflat / L[2]) % L[1], kflat % L[2]};
        const int64_t base = g * R;
        for (int l = 0; l < 3; ++l) {
            const int64_t Nl = L[l] * n;
            const int64_t s = orc_window_start_box(Nl, n, i_a[nu * 3 + l], kk[l]);
            for (int q = 0; q < R; ++q)
                memcpy(o[l] + (base + q) * Nl, f[l] + (int64_t)q * 2 * Nl + s, sizeof(double) * Nl);
        }
        for (int q = 0; q < R; ++q) wout[base + q] = Z[nu] * w[q];
    }
    return 0;
}

/* canonical.hpp:241-246: slab k = A1 * diag(w .* A3(k,:)) * A2^T, summed in rank order. */
int orc_densify_slabs(int64_t n1, int64_t n2, int64_t n3, int R, const double* A, const double* B,
                      const double* C, const double* w, int64_t k0, int64_t k1, double* out) {
    if (k0 < 0 || k1 > n3 || k0 > k1) return 2;
    double* scale = (double*)malloc(sizeof(double) * (R > 0 ? R : 1));
    for (int64_t k = k0; k < k1; ++k) {
        for (int q = 0; q < R; ++q) scale[q] = w[q] * C[k + n3 * q];
        double* slab = out + (k - k0) * n1 * n2;
        for (int64_t j = 0; j < n2; ++j)
            for (int64_t i = 0; i < n1; ++i) {
                double s = 0.0;
                for (int q = 0; q < R; ++q) s += (A[i + n1 * q] * scale[q]) * B[j + n2 * q];
                slab[i + n1 * j] = s;
            }
    }
    free(scale);
    return 0;
}

/* canonical.hpp:304-314 */
double orc_eval_point(int64_t n1, int64_t n2, int64_t n3, int R, const double* A, const double* B,
                      const double* C, const double* w, int64_t i, int64_t j, int64_t k) {
    double sum = 0.0;
    for (int q = 0; q < R; ++q) sum += w[q] * A[i + n1 * q] * B[j + n2 * q] * C[k + n3 * q];
    return sum;
}

static double dot(const double* x, const double* y, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}

/* canonical.hpp:126-136: Gram matrices per axis, then the rank-major (i outer, j inner)
 * reduction sum += wa_i * wb_j * G0 * G1 * G2. */
double orc_scalar_product(int64_t n1, int64_t n2, int64_t n3,
                          int Ra, const double* A0, const double* A1, const double* A2, const double* wa,
                          int Rb, const double* B0, const double* B1, const double* B2, const double* wb) {
    if (Ra == 0 || Rb == 0) return 0.0;
    const int64_t n[3] = {n1, n2, n3};
    const double* A[3] = {A0, A1, A2};
    const double* B[3] = {B0, B1, B2};
    double* G = (double*)malloc(sizeof(double) * 3 * (size_t)Ra * (size_t)Rb);
    for (int l = 0; l < 3; ++l)
        for (int j = 0; j < Rb; ++j)
            for (int i = 0; i < Ra; ++i)
                G[((size_t)l * Rb + j) * Ra + i] = dot(A[l] + n[l] * i, B[l] + n[l] * j, n[l]);
    double sum = 0.0;
    for (int i = 0; i < Ra; ++i)
        for (int j = 0; j < Rb; ++j)
            sum += wa[i] * wb[j] * G[((size_t)0 * Rb + j) * Ra + i] * G[((size_t)1 * Rb + j) * Ra + i] *
                   G[((size_t)2 * Rb + j) * Ra + i];
    free(G);
    return sum;
}

/* project.hpp:30-57 */
int orc_sample_gaussian(double b, int64_t n, const double center[3], double sigma, double* out) {
    if (!(sigma > 0.0) || !isfinite(sigma)) return 2;
    const double h = b / (double)n;
    for (int l = 0; l < 3; ++l) {
        if (!isfinite(center[l])) return 2;
        for (int64_t i = 0; i < n; ++i) {
            const double d = midpoint(i, n, h) - center[l];
            out[l * n + i] = exp(-d * d / (2.0 * sigma * sigma));
        }
    }
    return 0;
}

/* project.hpp:65-97: V(k,m) = scale * <G_k .* G_m, P>, upper triangle mirrored. */
int orc_potential_matrix(int64_t n, double h, int nb, const double* basis, int R, const double* P0,
                         const double* P1, const double* P2, const double* wp, int volume_element,
                         double* V) {
    if (nb < 1) return 2;
    const double scale = volume_element ? h * h * h : 1.0;
    double* pair = (double*)malloc(sizeof(double) * 3 * (size_t)n);
    const double one = 1.0;
    for (int k = 0; k < nb; ++k)
        for (int m = k; m < nb; ++m) {
            for (int l = 0; l < 3; ++l)
                for (int64_t i = 0; i < n; ++i)
                    pair[l * n + i] = basis[((size_t)k * 3 + l) * n + i] * basis[((size_t)m * 3 + l) * n + i];
            const double v = scale * orc_scalar_product(n, n, n, 1, pair, pair + n, pair + 2 * n, &one,
                                                        R, P0, P1, P2, wp);
            V[k + (int64_t)nb * m] = v;
            V[m + (int64_t)nb * k] = v;
        }
    free(pair);
    return 0;
}

double orc_grid_functional(int64_t n1, int64_t n2, int64_t n3, int R, const double* A,
                           const double* B, const double* C, const double* w, const double* r1,
                           const double* r2, const double* r3, int64_t k0, int64_t k1) {
    double* slab = (double*)malloc(sizeof(double) * (size_t)(n1 * n2));
    double total = 0.0;
    for (int64_t k = k0; k < k1; ++k) {
        orc_densify_slabs(n1, n2, n3, R, A, B, C, w, k, k + 1, slab);
        double sk = 0.0;
        for (int64_t j = 0; j < n2; ++j) {
            double sj = 0.0;
            for (int64_t i = 0; i < n1; ++i) sj += slab[i + n1 * j] * r1[i];
            sk += sj * r2[j];
        }
        total += sk * r3[k];
    }
    free(slab);
    return total;
}
