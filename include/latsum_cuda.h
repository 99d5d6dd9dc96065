/* latsum_cuda.h -- C ABI of liblatsum_cuda.so, the B200 (sm_100a) engine behind
 * the drop-in latsum C++ API (the headers under include/latsum/).
 *
 * The reference (arXiv 1405.2270, /root/reference/proj) is a header-only C++
 * library with no FFI; its "operator API" is the set of inline functions in
 * proj/include/latsum/. Each entry point below names the reference function
 * whose hot loop it replaces (file:line under proj/include/latsum/).
 *
 * Conventions
 *  - Plain pointers and sizes only. `_d` pointers are device memory on the
 *    current CUDA device, `_h` pointers are host memory. `stream` is a
 *    cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Matrices are column-major with an explicit leading dimension (the
 *    layout of Eigen::MatrixXd, canonical.hpp:17-19). Factor l of a rank-R
 *    canonical tensor is dims[l] x R. Dense grids are i-fastest:
 *    out[i + n1*(j + n2*k)] (DenseTensor3, canonical.hpp:94-99).
 *  - All arithmetic is FP64.
 *  - Return status: LS_OK, LS_EVALIDATION (reference validation_error,
 *    errors.hpp:9-12), LS_EGUARD (resource_guard_error, errors.hpp:17-20),
 *    LS_ECUDA (CUDA runtime failure). ls_last_error() returns a thread-local
 *    message for the last failing call on the calling thread.
 *  - Device-level calls are asynchronous on `stream`; host-level (`ls_h_*`)
 *    calls are synchronous and own their device buffers.
 *  - There is no CPU fallback: without a usable sm_100 device every call
 *    returns LS_ECUDA.
 */
#ifndef LATSUM_CUDA_H
#define LATSUM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LS_OK 0
#define LS_EVALIDATION 2
#define LS_EGUARD 4
#define LS_ECUDA 5

#define LS_GEN_MIDPOINT 0 /* gaussian_sample_vector, newton.hpp:43-52 */
#define LS_GEN_ERF 1      /* gaussian_moment_vector, newton.hpp:21-37 */

/* ---- lifecycle / diagnostics -------------------------------------------- */
int ls_abi_version(void);
const char* ls_last_error(void);
/* Sets the CUDA device used by the host-level calls of this thread. */
int ls_set_device(int device);
/* Kernel watchdog: 1 if a kernel on the current device abandoned an mbarrier wait after
 * 20 s (its results are garbage; the kernel drained and exited, the context is intact), else
 * 0; reset != 0 clears the flag. The host-level ls_h_* calls check it themselves and return
 * LS_ECUDA. */
int ls_fault_status(int reset);
/* 1 if this build reads the development A/B knobs (LS_EXPAND_PLAN, LS_EXPAND_DEBUG, ...) from
 * the environment (-DLS_DEV_KNOBS); the product build returns 0 and ignores them. */
int ls_dev_knobs_enabled(void);
/* Host threads the host-level calls use to move grid data out of their bounded pinned
 * staging ring into a pageable destination (0 = min(8, hardware threads)). One process per
 * GPU on a shared host: give each rank its share of the cores. */
int ls_set_host_threads(int n);
/* Number of kernel launches this library issued since load (all threads). */
int64_t ls_launch_count(void);

/* ---- host-side quadrature rule (no device work) -------------------------
 * sinc_quadrature(eps, a_min, a_max, M, C0) (quadrature.hpp:50-89): writes
 * the 2M+1 substitution nodes (may be NULL), exponents tau_q (ascending) and
 * weights w_q, and the node spacing (*step, may be NULL). */
int ls_sinc_quadrature(double eps, double a_min, double a_max, int M, double C0, double* nodes_h,
                       double* exponents_h, double* weights_h, double* step);

/* ---- host-side validation (no device work) -------------------------------
 * The single implementation of GridSpec::validate (grid.hpp:21-27), LatticeSpec::validate
 * and charge_grid_index (lattice.hpp:33-68), with the reference's messages; the drop-in
 * headers, the host-level calls, the pipeline and the Python mirror all call these.
 * charges_h is M0 x {x, y, z, Z} row-major; ia_out (optional) receives the vertex index of
 * charge nu on axis l at [l * M0 + nu]. */
int ls_validate_grid(double b, int64_t n);
int ls_charge_grid_index(double b, int64_t n, double p, int axis, int nu, int64_t* out);
int ls_validate_lattice(const int64_t L[3], int64_t n, double b, const double* charges_h, int M0,
                        int64_t* ia_out);

/* ---- K1: rank-R Newton-kernel generator --------------------------------
 * Replaces the column loop of build_newton_master (newton.hpp:57-75) with
 * gaussian_sample_vector (mode LS_GEN_MIDPOINT, newton.hpp:43-52) or
 * gaussian_moment_vector(GridSpec, t, doubled) (mode LS_GEN_ERF,
 * newton.hpp:21-37): out_d[i + ld*q], i < len, q < R. One thread per (q, i).
 * len must be even (>= 2); h > 0; tau_d[q] >= 0 finite. */
int ls_gen_master(int mode, const double* tau_d, int R, int64_t len, double h, double* out_d,
                  int64_t ld, void* stream);

/* Device instantiation of the generator's libm routines (csrc/glibc_math.cuh):
 * y_d[i] = erf(x_d[i]) (fn LS_LIBM_ERF) or exp(x_d[i]) (fn LS_LIBM_EXP), bit-identical to
 * glibc 2.39's x86-64 erf and FMA exp, which std::erf / std::exp resolve to in the reference
 * (newton.hpp:34, :50). Exposed so the parity tests can sweep arguments beyond the masters. */
#define LS_LIBM_ERF 0
#define LS_LIBM_EXP 1
int ls_libm_eval(int fn, const double* x_d, double* y_d, int64_t n, void* stream);

/* ---- K2: assembled lattice summation ----------------------------------
 * Replaces detail::assembled_axis_columns (lattice.hpp:220-274) for one
 * axis: column c = nu*R + q of out_d (out_len x M0*R, leading dim ld_out) is
 * sum_{k=0}^{L-1} master[s0(nu) - k*n + i], accumulated in ascending k
 * (bit-identical to the reference's blocked left-to-right adds), with
 * s0 = window_start_box(N, n, i_a, 0) (lattice.hpp:98) or
 * window_start_periodic(N, n, i_a, 0, L) (lattice.hpp:104-106), N = L*n.
 * master_d is (2N x R, leading dim ld_master); ia_d holds the M0 charge grid
 * indices on this axis (LatticeSpec::charge_grid_index, lattice.hpp:57-68).
 * out_len = n when periodic, else N. */
int ls_assemble_axis(const double* master_d, int64_t ld_master, int R, int M0, const int64_t* ia_d,
                     int64_t n, int64_t L, int periodic, double* out_d, int64_t ld_out, void* stream);

/* ---- K3: rank-R expansion onto the full grid -----------------------------
 * Replaces densify / detail::densify_slab (canonical.hpp:241-266) for the
 * z-slab range [k0, k1): V(i,j,k) = sum_q (A(i,q) * (w_q*C(k,q))) * B(j,q),
 * written to out_d[(k-k0)*ldz + j*ldy + i] (ldy >= N1, ldz >= ldy*N2; pass
 * 0 for the dense defaults ldy = N1, ldz = N1*N2). FP64 DMMA tensor-core
 * tiles with the scaled left factor resident in tensor memory for ranks up
 * to 121, in shared memory beyond (ls_expand_plan_name); one z-shard per
 * call, no inter-GPU traffic. Bitwise deterministic run to run.
 * Optional fused epilogue (BASELINE functional): when rho1_d
 * is non-NULL, partial_d receives ls_expand_partial_count() partial sums of
 *     sum_{i,j,k} V(i,j,k) * rho1(i) * rho2(j) * rho3(k)
 * (one per work unit and warp, each in a fixed order); reduce them with
 * ls_sum_partials. out_d may be NULL to skip storing the grid. */
int ls_expand(const double* A_d, int64_t lda, const double* B_d, int64_t ldb, const double* C_d,
              int64_t ldc, const double* w_d, int64_t N1, int64_t N2, int64_t N3, int R, int64_t k0,
              int64_t k1, double* out_d, int64_t ldy, int64_t ldz, const double* rho1_d,
              const double* rho2_d, const double* rho3_d, double* partial_d, void* stream);
int64_t ls_expand_partial_count(int64_t N1, int64_t N2, int R, int64_t k0, int64_t k1);
/* Human-readable description of the expansion plan ls_expand picks for rank R (kernel, CTA
 * shape, where A1k lives, k-steps, DFMA ranks) into out (NUL-terminated, at most len bytes). */
int ls_expand_plan_name(int R, char* out, int len);
/* Deterministic fixed-order sum of count doubles into *out_d (device). */
int ls_sum_partials(const double* partial_d, int64_t count, double* out_d, void* stream);

/* ---- K4: functionals and point evaluation -------------------------------
 * eval_point (canonical.hpp:304-314) for P index triples idx_d[3*p+{0,1,2}]:
 * out_d[p] = sum_q w_q*A(i,q)*B(j,q)*C(k,q), accumulated in rank order. */
int ls_eval_points(const double* A_d, int64_t lda, const double* B_d, int64_t ldb,
                   const double* C_d, int64_t ldc, const double* w_d, int R, const int64_t* idx_d,
                   int64_t P, double* out_d, void* stream);
/* Gram matrix G = X^T Y (Rx x Ry) of two n-row column-major matrices: the
 * per-axis products of scalar_product (canonical.hpp:130). Deterministic
 * fixed-order dot products, one warp per entry. G_d is Rx x Ry, ld = Rx. */
int ls_gram(const double* X_d, int64_t ldx, int Rx, const double* Y_d, int64_t ldy, int Ry, int64_t n,
            double* G_d, void* stream);
/* scalar_product(a, b) (canonical.hpp:126-136) from the three Gram matrices
 * (each Ra x Rb, ld Ra): out_d[0] = sum_i sum_j wa_i*wb_j*G0*G1*G2 in the
 * reference's rank-major order. */
int ls_gram_reduce(const double* G0_d, const double* G1_d, const double* G2_d, const double* wa_d,
                   int Ra, const double* wb_d, int Rb, double* out_d, void* stream);
/* Batched 1D functional: for F rank-1 densities rho_f = x_f (x) y_f (x) z_f
 * (columns of X_d, Y_d, Z_d; n1/n2/n3 rows), out_d[f] = scalar_product(P, rho_f)
 * (canonical.hpp:126-136 with Rb = 1), optionally times `scale`
 * (potential_matrix's h^3 volume element, project.hpp:74). Workspace-free:
 * Gram columns are formed in shared memory per f. */
int ls_functional_batch(const double* A_d, int64_t lda, const double* B_d, int64_t ldb,
                        const double* C_d, int64_t ldc, const double* w_d, int R, int64_t n1,
                        int64_t n2, int64_t n3, const double* X_d, int64_t ldx, const double* Y_d,
                        int64_t ldy, const double* Z_d, int64_t ldz, int F, double scale,
                        double* out_d, void* stream);

/* Full-grid form of a functional batch: for F
 * separable densities rho_f = X(:,f) (x) Y(:,f) (x) Z(:,f) and a dense device
 * grid V (i fastest; element (i,j,k) at V_d[i + ldy*j + ldz*k]),
 *     out_d[f] (+)= scale * sum_{i,j,k} V(i,j,k) X(i,f) Y(j,f) Z(k,f).
 * X, Y, Z are column-major (N1/N2/N3 x F). One fused FP64-DMMA GEMM over
 * rows (j,k) with the Y*Z weighting and the row reduction in its epilogue, then
 * a fixed-order sum over row tiles: bitwise reproducible. accumulate != 0 adds
 * into out_d (slab-chunked grids: pass Z_d offset to the chunk's first slab).
 * The reference has only the 1D form (scalar_product, canonical.hpp:126-136),
 * which it matches to rounding. */
int ls_grid_functional_batch(const double* V_d, int64_t N1, int64_t N2, int64_t N3, int64_t ldy, int64_t ldz,
                             const double* X_d, int64_t ldx, const double* Y_d, int64_t ldyy, const double* Z_d,
                             int64_t ldzz, int F, double scale, int accumulate, double* out_d, void* stream);

/* Probe error of the rank-R Newton-kernel tensor on a length-len midpoint
 * grid (build_newton_tensor, newton.hpp:79-84) straight from the rule:
 * out_d[0] = max_p |T(i_p, j_p, k_p) r_p - 1| (measure_probe_error,
 * newton.hpp:136-144) without materializing the factors; bit-identical to
 * eval_point on the generated master. idx_d holds P (i, j, k) triples. */
int ls_probe_error(const double* tau_d, const double* w_d, int R, int64_t len, double h, const int64_t* idx_d,
                   const double* r_d, int64_t P, double* out_d, void* stream);

/* Streaming compare: for every block b of a launch of nblocks blocks,
 * part_d[2b] = max(part_d[2b], max|a - b|) and part_d[2b+1] = max(.., max|b|)
 * over n entries (max_norm_diff_canonical's per-slab reduction,
 * canonical.hpp:289-293; max is exact, so the order does not matter). */
int ls_maxdiff_accumulate(const double* a_d, const double* b_d, int64_t n, double* part_d, int nblocks,
                          void* stream);

/* ---- device-resident pipeline (native runtime object) -------------------
 * generator -> assembled sum -> expansion -> functional with every stage in
 * HBM on the current device; the handle owns the master, assembled factors
 * and weights (Z_nu * w_q). charges_h holds M0 rows (x, y, z, Z) in
 * unit-cell coordinates [-b/2, b/2] (validated and snapped like
 * LatticeSpec, lattice.hpp:28-69). dims = n^3 (periodic) or (L*n)^3-shaped.
 * The handle remembers its device: every call runs there and restores the
 * caller's current device. Calls on one handle are stream-ordered on the
 * caller's stream; a handle is not meant for concurrent use from several
 * threads or streams (energy reuses one partial buffer) -- use one handle per
 * stream, as ShardedPotential does per rank. */
typedef struct ls_pipeline ls_pipeline;
int ls_pipeline_create(int mode, const int64_t L[3], int64_t n, double b, const double* tau_h, const double* w_h,
                       int R, const double* charges_h, int M0, int periodic, ls_pipeline** out);
int ls_pipeline_destroy(ls_pipeline* p);
/* dims, total rank M0*R and the device factors / weights (any output may be NULL). */
int ls_pipeline_info(const ls_pipeline* p, int64_t dims[3], int* rank_total, const double** A_d,
                     const double** B_d, const double** C_d, const double** w_d);
int ls_pipeline_generate(ls_pipeline* p, void* stream);
int ls_pipeline_assemble(ls_pipeline* p, void* stream);
/* generate + assemble: build_lattice_master (lattice.hpp:109-113) / the erf generator
 * (newton.hpp:21-37) followed by assembled_box_sum / assembled_periodic_sum (lattice.hpp:276-312),
 * as ONE launch when every master column fits shared memory (small lattices, e.g. cfg0 / cfg1;
 * bit-identical to the two calls, which it falls back to otherwise); ls_pipeline_step runs it. */
int ls_pipeline_prepare(ls_pipeline* p, void* stream);
/* slabs [k0, k1) into out_d (dense, i-fastest, (k1-k0)*N1*N2 doubles). */
int ls_pipeline_expand(ls_pipeline* p, int64_t k0, int64_t k1, double* out_d, void* stream);
int ls_pipeline_step(ls_pipeline* p, int64_t k0, int64_t k1, double* out_d, void* stream);
/* out_d[0] = sum over slabs [k0,k1) of V * rho1(i) rho2(j) rho3(k) (fused, V never stored). */
int ls_pipeline_energy(ls_pipeline* p, const double* r1_d, const double* r2_d, const double* r3_d, int64_t k0,
                       int64_t k1, double* out_d, void* stream);

/* ---- multi-GPU: the scalar all-reduce of the sharded path ------
 * One process per GPU; each owns a contiguous z-slab range of the grid (the reference's
 * k-slab parallel_for, canonical.hpp:251-266, spread over GPUs) and recomputes the
 * generator and assembly, so the only collective is the all-reduce of functional partials.
 * Rank 0 creates an id with ls_comm_unique_id and the caller hands its LS_COMM_ID_BYTES
 * bytes to every rank (file, socket, MPI ...); each rank then calls ls_comm_init on its own
 * device. NCCL (libnccl.so.2) is loaded with dlopen on first use. */
#define LS_COMM_ID_BYTES 128
#define LS_REDUCE_SUM 0
#define LS_REDUCE_MAX 1
typedef struct ls_comm ls_comm;
int ls_comm_unique_id(void* id_out, int bytes);
int ls_comm_init(int world, int rank, const void* id, int bytes, ls_comm** out);
int ls_comm_destroy(ls_comm* c);
int ls_comm_info(const ls_comm* c, int* world, int* rank);
/* In-place all-reduce (sum or max) of n doubles in device memory, on `stream`. */
int ls_comm_allreduce_f64(ls_comm* c, double* buf_d, int64_t n, int op, void* stream);
/* ls_pipeline_energy over this rank's slabs [k0, k1), then the sum over all ranks: every
 * rank's out_d[0] receives the whole-grid energy. */
int ls_pipeline_energy_allreduce(ls_pipeline* p, const double* r1_d, const double* r2_d, const double* r3_d,
                                 int64_t k0, int64_t k1, double* out_d, ls_comm* c, void* stream);

/* Small runtime helpers for callers without the CUDA headers: device memory
 * on the current device, a synchronous copy in any direction (cudaMemcpyDefault
 * on `stream`), and a stream wait. */
int ls_device_malloc(size_t bytes, void** out_d);
int ls_device_free(void* p_d);
int ls_memcpy(void* dst, const void* src, size_t bytes, void* stream);
int ls_synchronize(void* stream);

/* ---- host-level entry points (drop-in headers, e2e path) ----------------
 * Synchronous; all pointers host memory; results copied back. */
/* calibrate_quadrature(GridSpec(b, n), KernelTolerance(eps, a_min, a_max),
 * trace, m_cap) (newton.hpp:161-189): smallest M, best C0 in {1,2,3,4}, whose
 * kernel meets eps on the probe set (newton.hpp:97-132); all probes of a
 * candidate evaluated by ls_probe_error. The trace arrays (capacity
 * trace_cap; may be NULL with trace_len NULL) receive every candidate.
 * No rule within m_cap -> LS_EGUARD (resource_guard_error). */
int ls_h_calibrate_quadrature(double b, int64_t n, double eps, double a_min, double a_max, int m_cap, int* M_out,
                              double* C0_out, int* trace_len, int* trace_M, double* trace_C0, double* trace_err,
                              int trace_cap);
/* build_newton_master(lens, h, rule) (newton.hpp:57-75) in either generator
 * mode: f_h[l] is lens[l] x R column-major; equal-length axes share data. */
int ls_h_newton_master(int mode, const int64_t lens[3], double h, const double* tau_h, int R, double* f0_h,
                       double* f1_h, double* f2_h);
/* Batched scale * scalar_product(P, x_f (x) y_f (x) z_f) for F rank-1 tensors
 * (columns of X/Y/Z, dims[l] rows): potential_matrix's pair projections
 * (project.hpp:65-97) and the BASELINE energy functionals. */
int ls_h_functional_batch(const int64_t dims[3], int R, const double* A_h, const double* B_h, const double* C_h,
                          const double* w_h, int F, const double* X_h, const double* Y_h, const double* Z_h,
                          double scale, double* out_h);
/* max_norm_diff_canonical(a, b) (canonical.hpp:282-301): both tensors are
 * expanded slab-chunk by slab-chunk on the device and compared there. */
int ls_h_max_norm_diff(const int64_t dims[3], int Ra, const double* A0_h, const double* A1_h, const double* A2_h,
                       const double* wa_h, int Rb, const double* B0_h, const double* B1_h, const double* B2_h,
                       const double* wb_h, double* max_diff_h, double* max_abs_b_h);
/* build_lattice_master (lattice.hpp:109-113) / erf master: f_h[l] is
 * (2*L[l]*n x R), column-major. */
int ls_h_lattice_master(int mode, const int64_t L[3], int64_t n, double b, const double* tau_h,
                        int R, double* f0_h, double* f1_h, double* f2_h);
/* gaussian_sample_vector / gaussian_moment_vector for one column. */
int ls_h_gen_column(int mode, double t, int64_t len, double h, double* out_h);
/* detail::assembled_axis_columns (lattice.hpp:220-274) on a host master. */
int ls_h_assemble_axis(const double* master_h, int64_t master_len, int R, int M0,
                       const int64_t* ia_h, int64_t n, int64_t L, int periodic, double* out_h);
/* densify_slab over [k0, k1) (canonical.hpp:241-266) into a host grid;
 * device compute overlapped with chunked device->host copies. */
int ls_h_expand(const int64_t dims[3], int R, const double* A_h, const double* B_h,
                const double* C_h, const double* w_h, int64_t k0, int64_t k1, double* out_h);
/* eval_point batch (canonical.hpp:304-314). */
int ls_h_eval_points(const int64_t dims[3], int R, const double* A_h, const double* B_h,
                     const double* C_h, const double* w_h, const int64_t* idx_h, int64_t P,
                     double* out_h);
/* scalar_product (canonical.hpp:126-136). */
int ls_h_scalar_product(const int64_t dims[3], int Ra, const double* A0_h, const double* A1_h,
                        const double* A2_h, const double* wa_h, int Rb, const double* B0_h,
                        const double* B1_h, const double* B2_h, const double* wb_h, double* out_h);
/* Full-grid functional sum V * rho over slabs [k0,k1) without storing V. */
int ls_h_grid_functional(const int64_t dims[3], int R, const double* A_h, const double* B_h,
                         const double* C_h, const double* w_h, const double* r1_h,
                         const double* r2_h, const double* r3_h, int64_t k0, int64_t k1,
                         double* out_h);

/* End-to-end lattice potential (the e2e path of bench.py): generator (mode),
 * assembled box (periodic = 0) or periodic (periodic = 1) sum for the charges
 * (M0 x 4 rows: x, y, z, Z in unit-cell coordinates [-b/2, b/2]), then the
 * expansion of slabs [k0, k1) of the assembled tensor into grid_h (host).
 * Optionally also returns the assembled factors (f*_h may be NULL) and
 * weights. Inputs/outputs are host memory; all copies are inside the call. */
int ls_h_lattice_potential(int mode, const int64_t L[3], int64_t n, double b, const double* tau_h,
                           const double* w_h, int R, const double* charges_h, int M0, int periodic,
                           int64_t k0, int64_t k1, double* grid_h, double* f0_h, double* f1_h,
                           double* f2_h, double* wout_h);

/* ---- QTT (qtt.hpp) ---------------------------------------
 * TT-SVD sweep of every column of V_d (N = 2^L rows, ld ldv), one CTA per column with a
 * one-sided Jacobi SVD: cores of column c packed at cores_d + c * core_stride (core k is
 * (2 r_{k-1}) x r_k column-major), ranks_d + c * (L + 1) = r_0 .. r_L, capped_d[c] = 1 if a rank
 * hit rmax (<= 64). core_stride >= ls_qtt_core_stride(N, rmax). Truncation: qtt.hpp:49-86. */
int64_t ls_qtt_core_stride(int64_t N, int rmax);
int ls_qtt_compress(const double* V_d, int64_t ldv, int64_t N, int ncols, double eps, int rmax, double* cores_d,
                    int64_t core_stride, int* ranks_d, int* capped_d, void* stream);
/* eps-rank of every 2^k x 2^(L-k) unfolding, k = 1 .. L-1 (qtt.hpp:131-152): ranks_d + c * (L - 1). */
int ls_qtt_unfolding_ranks(const double* V_d, int64_t ldv, int64_t N, int ncols, double eps, int* ranks_d,
                           void* stream);
/* Host-level forms (host buffers in and out). */
int ls_h_qtt_compress(const double* V_h, int64_t N, int ncols, double eps, int rmax, double* cores_h,
                      int64_t core_stride, int* ranks_h, int* capped_h);
int ls_h_qtt_unfolding_ranks(const double* V_h, int64_t N, int ncols, double eps, int* ranks_h);

/* End-to-end energy (BASELINE configs[2]'s functional): the same generator and assembled sum,
 * then <V, rho> over slabs [k0, k1) for the separable density rho = r1 (x) r2 (x) r3 (host
 * vectors of the full axis lengths), fused into the expansion so V never leaves the device;
 * energy_h (host) receives the fixed-order sum. Inputs are host memory. */
int ls_h_lattice_energy(int mode, const int64_t L[3], int64_t n, double b, const double* tau_h, const double* w_h,
                        int R, const double* charges_h, int M0, int periodic, int64_t k0, int64_t k1,
                        const double* r1_h, const double* r2_h, const double* r3_h, double* energy_h);

#ifdef __cplusplus
}
#endif
#endif /* LATSUM_CUDA_H */
