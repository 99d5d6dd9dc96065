// functional.cu -- K4: functionals of the canonical tensor and point evaluation.
//
// References: scalar_product (canonical.hpp:126-136) = per-axis Gram matrices
// then a rank-major reduction; potential_matrix (project.hpp:65-97) = batched
// scalar products against rank-1 Gaussian pairs; eval_point
// (canonical.hpp:304-314). Dot products use a fixed lane-strided order and a
// fixed xor tree, so every result is bitwise reproducible run to run.
#include "common.cuh"
#include "glibc_math.cuh"

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

__device__ __forceinline__ double warp_dot(const double* __restrict__ x, const double* __restrict__ y,
                                           int64_t n, int lane) {
    double s = 0.0;
    for (int64_t i = lane; i < n; i += 32) s = fma(x[i], y[i], s);
    return warp_sum(s);
}

// eval_point: sum += w_q * A(i,q) * B(j,q) * C(k,q), left to right, rank order.
__global__ void eval_points_kernel(const double* __restrict__ A, int64_t lda,
                                   const double* __restrict__ B, int64_t ldb,
                                   const double* __restrict__ C, int64_t ldc,
                                   const double* __restrict__ w, int R,
                                   const int64_t* __restrict__ idx, int64_t P,
                                   double* __restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx[3 * p], j = idx[3 * p + 1], k = idx[3 * p + 2];
        double sum = 0.0;
        for (int q = 0; q < R; ++q)
            sum = rn_add(sum, rn_mul(rn_mul(rn_mul(w[q], A[i + lda * q]), B[j + ldb * q]), C[k + ldc * q]));
        out[p] = sum;
    }
}

// G(x, y) = <X[:, x], Y[:, y]>, one warp per entry.
__global__ void gram_kernel(const double* __restrict__ X, int64_t ldx, int Rx,
                            const double* __restrict__ Y, int64_t ldy, int Ry, int64_t n,
                            double* __restrict__ G) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= (int64_t)Rx * Ry) return;
    const int x = static_cast<int>(warp % Rx);
    const int y = static_cast<int>(warp / Rx);
    const double s = warp_dot(X + ldx * x, Y + ldy * y, n, lane);
    if (lane == 0) G[x + (int64_t)Rx * y] = s;
}

// canonical.hpp:131-135: i outer (rank of a), j inner (rank of b).
__global__ void gram_reduce_kernel(const double* __restrict__ G0, const double* __restrict__ G1,
                                   const double* __restrict__ G2, const double* __restrict__ wa,
                                   int Ra, const double* __restrict__ wb, int Rb,
                                   double* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double sum = 0.0;
    for (int i = 0; i < Ra; ++i)
        for (int j = 0; j < Rb; ++j) {
            const int64_t e = i + (int64_t)Ra * j;
            sum = rn_add(sum, rn_mul(rn_mul(rn_mul(rn_mul(wa[i], wb[j]), G0[e]), G1[e]), G2[e]));
        }
    out[0] = sum;
}

// Small batches (F below a few per SM): one block per density f: 3R Gram entries <P_l[:,q], rho_l[:,f]> by warps into
// shared memory, then thread 0 forms scale * sum_q ((w_q * 1) * G0) * G1 * G2.
__global__ void functional_batch_single_kernel(const double* __restrict__ A, int64_t lda,
                                        const double* __restrict__ B, int64_t ldb,
                                        const double* __restrict__ C, int64_t ldc,
                                        const double* __restrict__ w, int R, int64_t n1,
                                        int64_t n2, int64_t n3, const double* __restrict__ X,
                                        int64_t ldx, const double* __restrict__ Y, int64_t ldy,
                                        const double* __restrict__ Z, int64_t ldz, double scale,
                                        double* __restrict__ out) {
    extern __shared__ double gsh[];  // [3][R]
    const int f = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    for (int e = warp; e < 3 * R; e += nwarps) {
        const int l = e / R, q = e % R;
        double s;
        if (l == 0)
            s = warp_dot(A + lda * q, X + ldx * f, n1, lane);
        else if (l == 1)
            s = warp_dot(B + ldb * q, Y + ldy * f, n2, lane);
        else
            s = warp_dot(C + ldc * q, Z + ldz * f, n3, lane);
        if (lane == 0) gsh[e] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sum = 0.0;
        for (int q = 0; q < R; ++q)
            sum = rn_add(sum, rn_mul(rn_mul(rn_mul(rn_mul(w[q], 1.0), gsh[q]), gsh[R + q]), gsh[2 * R + q]));
        out[f] = rn_mul(scale, sum);
    }
}

// One block per kFBatch densities f: the 3R Gram entries <P_l[:,q], rho_l[:,f]> of each f, by
// warps into shared memory, then one thread per f forms scale * sum_q ((w_q * 1) * G0) * G1 * G2.
// A warp computes an entry for the block's densities together, so each factor column is read
// from L2 once per kFBatch densities (cfg4: 252 -> 63 MB of L2 reads; the density columns stay
// in L1 across the R entries of an axis). Kernel 33.5 -> 29.0 us at cfg4 (F = 1024, ncu warm);
// 2 densities per block measured the same, 8 and 16 slower (57.6 / 75.8 us: fewer blocks, the
// per-warp entry loop is latency-bound). LS_FBATCH is a build-time lab knob.
#ifndef LS_FBATCH
#define LS_FBATCH 4
#endif
constexpr int kFBatch = LS_FBATCH;
__global__ void functional_batch_kernel(const double* __restrict__ A, int64_t lda,
                                        const double* __restrict__ B, int64_t ldb,
                                        const double* __restrict__ C, int64_t ldc,
                                        const double* __restrict__ w, int R, int64_t n1,
                                        int64_t n2, int64_t n3, const double* __restrict__ X,
                                        int64_t ldx, const double* __restrict__ Y, int64_t ldy,
                                        const double* __restrict__ Z, int64_t ldz, int F, double scale,
                                        double* __restrict__ out) {
    extern __shared__ double gsh[];  // [kFBatch][3][R]
    const int f0 = blockIdx.x * kFBatch;
    const int nf = F - f0 < kFBatch ? F - f0 : kFBatch;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    for (int e = warp; e < 3 * R; e += nwarps) {
        const int l = e / R, q = e % R;
        const double* x = l == 0 ? A + lda * q : l == 1 ? B + ldb * q : C + ldc * q;
        const double* y = l == 0 ? X : l == 1 ? Y : Z;
        const int64_t ld = l == 0 ? ldx : l == 1 ? ldy : ldz;
        const int64_t n = l == 0 ? n1 : l == 1 ? n2 : n3;
        double s[kFBatch] = {};
        for (int64_t i = lane; i < n; i += 32) {
            const double xv = x[i];
#pragma unroll
            for (int u = 0; u < kFBatch; ++u)
                if (u < nf) s[u] = fma(xv, y[ld * (f0 + u) + i], s[u]);
        }
#pragma unroll
        for (int u = 0; u < kFBatch; ++u) {
            const double t = warp_sum(s[u]);
            if (lane == 0) gsh[u * 3 * R + e] = t;
        }
    }
    __syncthreads();
    if (threadIdx.x < nf) {
        const double* g = gsh + threadIdx.x * 3 * R;
        double sum = 0.0;
        for (int q = 0; q < R; ++q)
            sum = rn_add(sum, rn_mul(rn_mul(rn_mul(rn_mul(w[q], 1.0), g[q]), g[R + q]), g[2 * R + q]));
        out[f0 + threadIdx.x] = rn_mul(scale, sum);
    }
}

// Ranks whose Gram entries do not fit in shared memory: G_l (R x Fc, from gram_kernel, the same
// warp_dot as above) comes from global scratch, and one thread per density forms the same
// rank-ordered sum, so the result is bit-identical to the shared-memory kernels.
__global__ void functional_reduce_kernel(const double* __restrict__ G0, const double* __restrict__ G1,
                                         const double* __restrict__ G2, const double* __restrict__ w, int R,
                                         int Fc, double scale, double* __restrict__ out) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= Fc) return;
    const int64_t c = static_cast<int64_t>(R) * f;
    double sum = 0.0;
    for (int q = 0; q < R; ++q)
        sum = rn_add(sum, rn_mul(rn_mul(rn_mul(rn_mul(w[q], 1.0), G0[c + q]), G1[c + q]), G2[c + q]));
    out[f] = rn_mul(scale, sum);
}

// Block-partial max |a - b| and max |b| over n entries (max is order-independent: exact).
__global__ void maxdiff_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                               double* __restrict__ part) {
    __shared__ double sd[256], sb[256];
    double md = 0.0, mb = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        md = fmax(md, fabs(a[e] - b[e]));
        mb = fmax(mb, fabs(b[e]));
    }
    sd[threadIdx.x] = md;
    sb[threadIdx.x] = mb;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            sd[threadIdx.x] = fmax(sd[threadIdx.x], sd[threadIdx.x + w]);
            sb[threadIdx.x] = fmax(sb[threadIdx.x], sb[threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = fmax(part[2 * blockIdx.x], sd[0]);
        part[2 * blockIdx.x + 1] = fmax(part[2 * blockIdx.x + 1], sb[0]);
    }
}

// Probe error of the rank-R Newton-kernel tensor straight from the rule (newton.hpp:136-144 on
// build_newton_tensor, newton.hpp:79-84): each probe's three factor entries are generated with
// the midpoint formula of gen_midpoint_kernel (bit-identical to the materialized master) and
// combined in eval_point's rank order; max |v r - 1| via an atomic max on the bit pattern
// (non-negative doubles order like their bits, and max is exact).
__global__ void probe_error_kernel(const double* __restrict__ tau, const double* __restrict__ w, int R,
                                   int64_t len, double h, const int64_t* __restrict__ idx,
                                   const double* __restrict__ r, int64_t P,
                                   unsigned long long* __restrict__ out_bits) {
    const double half_len = static_cast<double>(len) / 2.0;
    double worst = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
        const double mi = rn_mul(rn_sub(rn_add(static_cast<double>(idx[3 * p]), 0.5), half_len), h);
        const double mj = rn_mul(rn_sub(rn_add(static_cast<double>(idx[3 * p + 1]), 0.5), half_len), h);
        const double mk = rn_mul(rn_sub(rn_add(static_cast<double>(idx[3 * p + 2]), 0.5), half_len), h);
        double sum = 0.0;
        for (int q = 0; q < R; ++q) {
            const double t = tau[q];
            const double xi = rn_mul(t, mi), xj = rn_mul(t, mj), xk = rn_mul(t, mk);
            const double fi = ls::gm::exp(-rn_mul(xi, xi)), fj = ls::gm::exp(-rn_mul(xj, xj)),
                         fk = ls::gm::exp(-rn_mul(xk, xk));
            sum = rn_add(sum, rn_mul(rn_mul(rn_mul(w[q], fi), fj), fk));
        }
        worst = fmax(worst, fabs(rn_sub(rn_mul(sum, r[p]), 1.0)));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out_bits, static_cast<unsigned long long>(__double_as_longlong(worst)));
}

}  // namespace

extern "C" int ls_probe_error(const double* tau_d, const double* w_d, int R, int64_t len, double h,
                              const int64_t* idx_d, const double* r_d, int64_t P, double* out_d, void* stream) {
    if (R < 0 || P < 0 || len < 2 || len % 2 != 0 || !(h > 0.0))
        return ls::fail(LS_EVALIDATION, "probe_error: bad arguments");
    const cudaStream_t s = ls::as_stream(stream);
    LS_CUDA(cudaMemsetAsync(out_d, 0, sizeof(double), s));
    if (P == 0) return LS_OK;
    const int64_t blocks = std::min<int64_t>(ls::ceil_div(P, 256), 4 * ls::sm_count());
    probe_error_kernel<<<(unsigned)blocks, 256, 0, s>>>(tau_d, w_d, R, len, h, idx_d, r_d, P,
                                                         reinterpret_cast<unsigned long long*>(out_d));
    LS_LAUNCHED("probe_error_kernel");
    return LS_OK;
}

extern "C" int ls_maxdiff_accumulate(const double* a_d, const double* b_d, int64_t n, double* part_d, int nblocks,
                                     void* stream) {
    if (n < 0 || nblocks < 1 || nblocks > 4096) return ls::fail(LS_EVALIDATION, "maxdiff: bad arguments");
    if (n == 0) return LS_OK;
    maxdiff_kernel<<<nblocks, 256, 0, ls::as_stream(stream)>>>(a_d, b_d, n, part_d);
    LS_LAUNCHED("maxdiff_kernel");
    return LS_OK;
}

extern "C" int ls_eval_points(const double* A_d, int64_t lda, const double* B_d, int64_t ldb,
                              const double* C_d, int64_t ldc, const double* w_d, int R,
                              const int64_t* idx_d, int64_t P, double* out_d, void* stream) {
    if (P < 0 || R < 0) return ls::fail(LS_EVALIDATION, "eval_points: negative count");
    if (P == 0) return LS_OK;
    const int64_t blocks = std::min<int64_t>(ls::ceil_div(P, 256), 65535);
    eval_points_kernel<<<(unsigned)blocks, 256, 0, ls::as_stream(stream)>>>(A_d, lda, B_d, ldb, C_d,
                                                                           ldc, w_d, R, idx_d, P, out_d);
    LS_LAUNCHED("eval_points_kernel");
    return LS_OK;
}

extern "C" int ls_gram(const double* X_d, int64_t ldx, int Rx, const double* Y_d, int64_t ldy,
                       int Ry, int64_t n, double* G_d, void* stream) {
    if (Rx < 0 || Ry < 0 || n < 0 || ldx < n || ldy < n)
        return ls::fail(LS_EVALIDATION, "gram: bad shape");
    const int64_t warps = (int64_t)Rx * Ry;
    if (warps == 0) return LS_OK;
    const int64_t blocks = ls::ceil_div(warps * 32, 256);
    gram_kernel<<<(unsigned)blocks, 256, 0, ls::as_stream(stream)>>>(X_d, ldx, Rx, Y_d, ldy, Ry, n, G_d);
    LS_LAUNCHED("gram_kernel");
    return LS_OK;
}

extern "C" int ls_gram_reduce(const double* G0_d, const double* G1_d, const double* G2_d,
                              const double* wa_d, int Ra, const double* wb_d, int Rb,
                              double* out_d, void* stream) {
    if (Ra < 0 || Rb < 0) return ls::fail(LS_EVALIDATION, "gram_reduce: negative rank");
    gram_reduce_kernel<<<1, 32, 0, ls::as_stream(stream)>>>(G0_d, G1_d, G2_d, wa_d, Ra, wb_d, Rb, out_d);
    LS_LAUNCHED("gram_reduce_kernel");
    return LS_OK;
}

extern "C" int ls_functional_batch(const double* A_d, int64_t lda, const double* B_d, int64_t ldb,
                                   const double* C_d, int64_t ldc, const double* w_d, int R,
                                   int64_t n1, int64_t n2, int64_t n3, const double* X_d,
                                   int64_t ldx, const double* Y_d, int64_t ldy, const double* Z_d,
                                   int64_t ldz, int F, double scale, double* out_d, void* stream) {
    if (R < 1 || F < 0 || n1 < 1 || n2 < 1 || n3 < 1 || lda < n1 || ldb < n2 || ldc < n3 ||
        ldx < n1 || ldy < n2 || ldz < n3)
        return ls::fail(LS_EVALIDATION, "functional_batch: bad shape");
    if (F == 0) return LS_OK;
    // Batches too small to fill the GPU with kFBatch densities per block take one per block
    // with the single-density kernel (cfg2's one energy density); either kernel keeps its 3R
    // Gram entries per density in shared memory, and ranks beyond that take the global-scratch
    // path (bit-identical results).
    constexpr size_t kSmemCap = 200 * 1024;
    const size_t per_f = sizeof(double) * 3 * static_cast<size_t>(R);
    const int fb = (F >= kFBatch * ls::sm_count() && per_f * kFBatch <= kSmemCap) ? kFBatch : 1;
    const size_t smem = per_f * fb;
    const cudaStream_t s = ls::as_stream(stream);
    if (smem > kSmemCap) {
        // F chunked so the three R x Fc Gram blocks stay within 256 MiB of scratch.
        const int64_t Fc = std::max<int64_t>(1, std::min<int64_t>(F, (int64_t(32) << 20) / (3 * (int64_t)R)));
        ls::ensure_pool();
        ls::AsyncScratch scratch(s);
        LS_CUDA(scratch.alloc(sizeof(double) * 3 * static_cast<size_t>(R) * Fc));
        double* G = scratch.as<double>();
        for (int64_t f0 = 0; f0 < F; f0 += Fc) {
            const int fc = static_cast<int>(std::min<int64_t>(Fc, F - f0));
            const double* fac[3] = {A_d, B_d, C_d};
            const int64_t ldf[3] = {lda, ldb, ldc};
            const double* rho[3] = {X_d, Y_d, Z_d};
            const int64_t ldr[3] = {ldx, ldy, ldz};
            const int64_t nl[3] = {n1, n2, n3};
            for (int l = 0; l < 3; ++l) {
                const int64_t blocks = ls::ceil_div((int64_t)R * fc * 32, 256);
                gram_kernel<<<(unsigned)blocks, 256, 0, s>>>(fac[l], ldf[l], R, rho[l] + ldr[l] * f0, ldr[l], fc,
                                                             nl[l], G + (int64_t)l * R * Fc);
                LS_LAUNCHED("gram_kernel");
            }
            functional_reduce_kernel<<<(unsigned)ls::ceil_div(fc, 128), 128, 0, s>>>(
                G, G + (int64_t)R * Fc, G + 2 * (int64_t)R * Fc, w_d, R, fc, scale, out_d + f0);
            LS_LAUNCHED("functional_reduce_kernel");
        }
        return LS_OK;
    }
    if (fb == 1) {
        auto kern = functional_batch_single_kernel;
        if (smem > 48 * 1024)
            LS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<F, 256, smem, s>>>(A_d, lda, B_d, ldb, C_d, ldc, w_d, R, n1, n2, n3, X_d, ldx, Y_d, ldy, Z_d, ldz,
                                  scale, out_d);
        LS_LAUNCHED("functional_batch_single_kernel");
        return LS_OK;
    }
    auto kern = functional_batch_kernel;
    if (smem > 48 * 1024)
        LS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(F + fb - 1) / fb, 256, smem, s>>>(A_d, lda, B_d, ldb, C_d, ldc, w_d, R, n1, n2, n3, X_d, ldx, Y_d, ldy,
                                              Z_d, ldz, F, scale, out_d);
    LS_LAUNCHED("functional_batch_kernel");
    return LS_OK;
}
