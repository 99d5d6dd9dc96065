/* latsum_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference latsum hot path (arXiv 1405.2270,
 * /root/reference/proj/include/latsum), used as the parity checker for the
 * CUDA path. Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
 * leg may load it. It is never linked into liblatsum_cuda.so.
 *
 * Parity pinning: every function here is checked against the reference's own
 * headers compiled unmodified (oracle/_ref, built by oracle/Makefile) and
 * against the committed golden vectors in tests/golden/ generated from them.
 *
 * Layout conventions (same as the product C ABI): matrices are column-major,
 * factor l of a canonical tensor is dims[l] x R with leading dimension
 * dims[l]; dense grids are i-fastest, data[i + n1*(j + n2*k)].
 * Return value: 0 ok, 2 validation error (mirrors latsum::validation_error),
 * 4 resource guard (mirrors latsum::resource_guard_error).
 */
#ifndef LATSUM_ORACLE_H
#define LATSUM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* quadrature.hpp:50-89 */
int orc_sinc_quadrature(double eps, double a_min, double a_max, int M, double C0,
                        double* nodes, double* exponents, double* weights, double* step);
/* quadrature.hpp:93-100 */
double orc_quadrature_value(const double* exponents, const double* weights, int R, double r);
/* newton.hpp:43-52 (midpoint samples) */
int orc_gaussian_sample_vector(int64_t len, double h, double t, double* out);
/* newton.hpp:21-37 (erf-difference cell integrals); grid = (b, n) */
int orc_gaussian_moment_vector(double b, int64_t n, double t, int doubled, double* out);
/* y[i] = erf(x[i]) (fn 0) or exp(x[i]) (fn 1) from the host libm: the calls std::erf / std::exp
 * make in gaussian_moment_vector / gaussian_sample_vector (newton.hpp:34, :50). */
int orc_libm_eval(int fn, const double* x, double* y, int64_t n);
/* mode 0: build_lattice_master (lattice.hpp:109-113 -> newton.hpp:57-75, midpoint)
 * mode 1: erf master, column q = gaussian_moment_vector(GridSpec(L_l*b, L_l*n), tau_q, true)
 * f[l] receives 2*L[l]*n x R. */
int orc_lattice_master(int mode, const int64_t L[3], int64_t n, double b, const double* tau, int R,
                       double* f0, double* f1, double* f2);
/* lattice.hpp:57-68: charge grid index of coordinate p on a unit cell (b, n); -1 if off-grid */
int64_t orc_charge_grid_index(double b, int64_t n, double p);
/* lattice.hpp:98 and :104-106 */
int64_t orc_window_start_box(int64_t N, int64_t n, int64_t i_a, int64_t k);
int64_t orc_window_start_periodic(int64_t N, int64_t n, int64_t i_a, int64_t k, int64_t L);
/* lattice.hpp:220-274 for one axis: master (2*L*n x R), i_a[M0] charge indices on this axis,
 * out (out_len x M0*R), out_len = n (periodic) or L*n. Columns ordered (nu, q) nu-major. */
int orc_assembled_axis(const double* master, int R, int M0, const int64_t* i_a, int64_t n,
                       int64_t L, int periodic, double* out);
/* lattice.hpp:276-296 weights: w_out[nu*R+q] = Z_nu * w_q */
void orc_assembled_weights(const double* Z, int M0, const double* w, int R, double* w_out);
/* lattice.hpp:163-209: direct (concatenation) sum factors for axis l and weights.
 * out_l is N_l x (M0*cells*R). */
int orc_direct_sum(const int64_t L[3], int64_t n, const int64_t* i_a /* M0 x 3 */, const double* Z,
                   int M0, const double* f0, const double* f1, const double* f2, const double* w,
                   int R, double* o0, double* o1, double* o2, double* wout);
/* canonical.hpp:241-246 over k in [k0, k1): out receives (k1-k0) slabs n1 x n2. */
int orc_densify_slabs(int64_t n1, int64_t n2, int64_t n3, int R, const double* A, const double* B,
                      const double* C, const double* w, int64_t k0, int64_t k1, double* out);
/* canonical.hpp:304-314 */
double orc_eval_point(int64_t n1, int64_t n2, int64_t n3, int R, const double* A, const double* B,
                      const double* C, const double* w, int64_t i, int64_t j, int64_t k);
/* canonical.hpp:126-136 (both tensors on the same dims) */
double orc_scalar_product(int64_t n1, int64_t n2, int64_t n3,
                          int Ra, const double* A0, const double* A1, const double* A2, const double* wa,
                          int Rb, const double* B0, const double* B1, const double* B2, const double* wb);
/* project.hpp:30-57, one function: out is 3 x n (axis-major) */
int orc_sample_gaussian(double b, int64_t n, const double center[3], double sigma, double* out);
/* project.hpp:65-97: basis (nb x 3 x n), P factors (n x R each), V (nb x nb col-major) */
int orc_potential_matrix(int64_t n, double h, int nb, const double* basis, int R, const double* P0,
                         const double* P1, const double* P2, const double* wp, int volume_element,
                         double* V);
/* streamed sum_{ijk} V(i,j,k) * r1(i) r2(j) r3(k) over slabs [k0,k1), summing each slab's
 * i-then-j partials in order (no reference function: BASELINE a18; oracle for the fused
 * full-grid functional). */
double orc_grid_functional(int64_t n1, int64_t n2, int64_t n3, int R, const double* A,
                           const double* B, const double* C, const double* w, const double* r1,
                           const double* r2, const double* r3, int64_t k0, int64_t k1);

#ifdef __cplusplus
}
#endif
#endif
