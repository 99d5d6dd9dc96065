// qtt.cu -- quantized tensor-train (QTT) compression of canonical factor columns, on the GPU.
//
// Reference: proj/include/latsum/qtt.hpp: qtt_compress (:49-86) is a
// left-to-right TT-SVD sweep of a length-2^L vector -- at step k the carry, a (r_{k-1} x rest)
// column-major buffer, is reinterpreted as the (2 r_{k-1}) x (rest / 2) matrix M, M = U S V^T,
// the singular tail with Frobenius norm <= delta = eps ||v|| / sqrt(L - 1) is dropped, U's kept
// columns become core k and S V^T the next carry; unfolding_rank_profile (:131-152) takes the
// eps-rank of every 2^k x 2^(L-k) unfolding. The reference factorises with Eigen's BDCSVD on the
// host; here one CTA per vector runs the whole sweep (or all unfoldings) with a one-sided
// (Hestenes) Jacobi SVD -- relative accuracy for the small singular values the truncation
// looks at -- on a transposed copy of M in global scratch, rotations accumulated in shared
// memory, a fixed round-robin pair order and fixed-order reductions (deterministic).
// Singular vectors are defined up to sign (and rotation within repeated singular values), so
// cores can differ from Eigen's by such factors; ranks, singular values and reconstructions
// agree to rounding.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace {

constexpr int kQttThreads = 256, kQttWarps = kQttThreads / 32;
constexpr int kQttMaxSweeps = 40;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// Round-robin tournament: round rd of n2 - 1 (n2 even), pair pi < n2 / 2 -> columns (i, j).
__device__ __forceinline__ void rr_pair(int n2, int rd, int pi, int& i, int& j) {
    auto pos = [&](int x) { return x == 0 ? 0 : 1 + (x - 1 + rd) % (n2 - 1); };
    i = pos(pi);
    j = pos(n2 - 1 - pi);
    if (i > j) {
        const int t = i;
        i = j;
        j = t;
    }
}

// One-sided Jacobi on the m x n column-major W (global, ld m): W <- W V with orthogonal
// columns; V (n x n, shared, may be null) accumulates the rotations. Returns in sig[i] the
// column norms (the singular values, unsorted). CTA-wide; n <= kQttMaxN.
__device__ void jacobi_svd(double* W, int64_t m, int n, double* V, double* sig, int* flag) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (V)
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) V[e] = (e % n == e / n) ? 1.0 : 0.0;
    const int n2 = n + (n & 1);
    __syncthreads();
    for (int sweep = 0; sweep < kQttMaxSweeps && n > 1; ++sweep) {
        if (threadIdx.x == 0) *flag = 0;
        __syncthreads();
        for (int rd = 0; rd < n2 - 1; ++rd) {
            for (int pi = warp; pi < n2 / 2; pi += kQttWarps) {
                int i, j;
                rr_pair(n2, rd, pi, i, j);
                if (j >= n) continue;
                double* x = W + m * i;
                double* y = W + m * j;
                double a = 0.0, b = 0.0, c = 0.0;
                for (int64_t k = lane; k < m; k += 32) {
                    const double xv = x[k], yv = y[k];
                    a = fma(xv, xv, a);
                    b = fma(yv, yv, b);
                    c = fma(xv, yv, c);
                }
                a = warp_sum(a);
                b = warp_sum(b);
                c = warp_sum(c);
                if (!(fabs(c) > 1e-15 * sqrt(a * b)) || c == 0.0) continue;
                const double zeta = (b - a) / (2.0 * c);
                const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
                for (int64_t k = lane; k < m; k += 32) {
                    const double xv = x[k], yv = y[k];
                    x[k] = cs * xv - sn * yv;
                    y[k] = sn * xv + cs * yv;
                }
                if (V)
                    for (int k = lane; k < n; k += 32) {
                        const double vi = V[k + n * i], vj = V[k + n * j];
                        V[k + n * i] = cs * vi - sn * vj;
                        V[k + n * j] = sn * vi + cs * vj;
                    }
                if (lane == 0) *flag = 1;
            }
            __syncthreads();
        }
        if (*flag == 0) break;
        __syncthreads();
    }
    for (int i = warp; i < n; i += kQttWarps) {
        const double* x = W + m * i;
        double a = 0.0;
        for (int64_t k = lane; k < m; k += 32) a = fma(x[k], x[k], a);
        a = warp_sum(a);
        if (lane == 0) sig[i] = sqrt(a);
    }
    __syncthreads();
}

// Descending order of sig[0..n) into idx (ties by index), and the eps-rank: the smallest r whose
// discarded tail has Frobenius norm <= thresh (qtt.hpp:63-69), at least 1. Thread 0.
__device__ int order_and_rank(const double* sig, int n, int* idx, double thresh) {
    for (int i = 0; i < n; ++i) idx[i] = i;
    for (int i = 1; i < n; ++i) {  // insertion sort, n <= a few hundred
        const int v = idx[i];
        int j = i - 1;
        while (j >= 0 && (sig[idx[j]] < sig[v] || (sig[idx[j]] == sig[v] && idx[j] > v))) {
            idx[j + 1] = idx[j];
            --j;
        }
        idx[j + 1] = v;
    }
    int keep = n;
    double tail = 0.0;
    for (int i = n; i-- > 0;) {
        const double s = sig[idx[i]];
        tail += s * s;
        if (sqrt(tail) > thresh) break;
        keep = i;
    }
    return keep > 1 ? keep : 1;
}

__device__ double cta_norm(const double* v, int64_t N, double* red) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double a = 0.0;
    for (int64_t k = threadIdx.x; k < N; k += blockDim.x) a = fma(v[k], v[k], a);
    a = warp_sum(a);
    if (lane == 0) red[warp] = a;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < kQttWarps; ++w) s += red[w];
    __syncthreads();
    return sqrt(s);
}

// TT-SVD sweep of column c of V (N = 2^L, ld ldv): cores packed at cores + c * core_stride (core
// k is (2 r_{k-1}) x r_k column-major), ranks + c * (L + 1) receives r_0 .. r_L, capped[c] is set
// when a rank hit rmax. scratch: 2 N doubles per column.
__global__ void __launch_bounds__(kQttThreads) qtt_compress_kernel(const double* __restrict__ Vin, int64_t ldv,
                                                                   int64_t N, int L, double eps, int rmax,
                                                                   double* __restrict__ cores, int64_t core_stride,
                                                                   int* __restrict__ ranks, int* __restrict__ capped,
                                                                   double* __restrict__ scratch) {
    extern __shared__ double sm[];
    const int nmax = 2 * rmax;
    double* Vr = sm;                    // [nmax * nmax]
    double* sig = Vr + nmax * nmax;     // [nmax]
    double* red = sig + nmax;           // [kQttWarps]
    int* idx = reinterpret_cast<int*>(red + kQttWarps);  // [nmax]
    int* sh = idx + nmax;               // flag, keep
    const int c = blockIdx.x;
    const double* v = Vin + ldv * c;
    double* carry = scratch + 2 * N * c;
    double* W = carry + N;
    double* core = cores + core_stride * c;
    int* rk = ranks + (L + 1) * c;
    for (int64_t k = threadIdx.x; k < N; k += blockDim.x) carry[k] = v[k];
    __syncthreads();
    const double delta = eps * cta_norm(carry, N, red) / sqrt(static_cast<double>(L - 1 > 1 ? L - 1 : 1));
    int r_prev = 1;
    int64_t rest = N, off = 0;
    if (threadIdx.x == 0) {
        rk[0] = 1;
        capped[c] = 0;
    }
    for (int k = 0; k + 1 < L; ++k) {
        const int n = 2 * r_prev;
        const int64_t m = rest / 2;
        // W = M^T (m x n), M(i, j) = carry[i + n j]
        for (int64_t e = threadIdx.x; e < m * n; e += blockDim.x) {
            const int64_t j = e % m, i = e / m;
            W[e] = carry[i + n * j];
        }
        __syncthreads();
        jacobi_svd(W, m, n, Vr, sig, sh);
        if (threadIdx.x == 0) {
            int keep = order_and_rank(sig, n, idx, delta);
            if (keep > rmax) {
                keep = rmax;
                capped[c] = 1;
            }
            sh[1] = keep;
            rk[k + 1] = keep;
        }
        __syncthreads();
        const int keep = sh[1];
        // core k = U_M[:, idx[0:keep]] = V[:, idx] (n x keep); next carry = S V_M^T = W[:, idx]^T
        for (int e = threadIdx.x; e < n * keep; e += blockDim.x) core[off + e] = Vr[(e % n) + n * idx[e / n]];
        __syncthreads();
        for (int64_t e = threadIdx.x; e < keep * m; e += blockDim.x) {
            const int64_t i = e % keep, j = e / keep;
            carry[e] = W[j + m * idx[i]];
        }
        __syncthreads();
        off += static_cast<int64_t>(n) * keep;
        r_prev = keep;
        rest = m;
    }
    for (int e = threadIdx.x; e < 2 * r_prev; e += blockDim.x) core[off + e] = carry[e];
    if (threadIdx.x == 0) rk[L] = 1;
}

// eps-rank of every unfolding 2^k x 2^(L-k), k = 1 .. L-1, of column c (singular values only):
// out + c * (L - 1). scratch: N doubles per column.
__global__ void __launch_bounds__(kQttThreads) qtt_unfolding_kernel(const double* __restrict__ Vin, int64_t ldv,
                                                                    int64_t N, int L, double eps,
                                                                    int* __restrict__ out,
                                                                    double* __restrict__ scratch) {
    extern __shared__ double sm[];
    const int nmax = 1 << ((L + 1) / 2);
    double* sig = sm;                   // [nmax]
    double* red = sig + nmax;           // [kQttWarps]
    int* idx = reinterpret_cast<int*>(red + kQttWarps);
    int* sh = idx + nmax;
    const int c = blockIdx.x;
    const double* v = Vin + ldv * c;
    double* W = scratch + N * c;
    const double thresh = eps * cta_norm(v, N, red);
    for (int k = 1; k < L; ++k) {
        const int64_t rows = int64_t(1) << k, cols = int64_t(1) << (L - k);
        // columns of the orientation with fewer of them: W is m x n
        const bool tr = rows <= cols;
        const int n = static_cast<int>(tr ? rows : cols);
        const int64_t m = tr ? cols : rows;
        for (int64_t e = threadIdx.x; e < N; e += blockDim.x) {
            const int64_t a = e % m, b = e / m;  // W(a, b)
            W[e] = tr ? v[b + rows * a] : v[a + rows * b];
        }
        __syncthreads();
        jacobi_svd(W, m, n, nullptr, sig, sh);
        if (threadIdx.x == 0) out[(L - 1) * c + (k - 1)] = order_and_rank(sig, n, idx, thresh);
        __syncthreads();
    }
}

int log2_pow2(int64_t N) {
    if (N < 2 || (N & (N - 1)) != 0) return -1;
    int L = 0;
    while ((int64_t(1) << L) < N) ++L;
    return L;
}

}  // namespace

extern "C" {

int64_t ls_qtt_core_stride(int64_t N, int rmax) {
    const int L = log2_pow2(N);
    if (L < 1 || rmax < 1) return -1;
    auto rb = [&](int k) -> int64_t {  // bound on r_k
        if (k <= 0 || k >= L) return 1;
        return std::min<int64_t>({int64_t(1) << std::min(k, 40), int64_t(1) << std::min(L - k, 40), rmax});
    };
    int64_t s = 0;
    for (int k = 0; k + 1 < L; ++k) s += 2 * rb(k) * rb(k + 1);
    return s + 2 * rb(L - 1);
}

int ls_qtt_compress(const double* V_d, int64_t ldv, int64_t N, int ncols, double eps, int rmax, double* cores_d,
                    int64_t core_stride, int* ranks_d, int* capped_d, void* stream) {
    const int L = log2_pow2(N);
    if (L < 1) return ls::fail(LS_EVALIDATION, "qtt_compress: length " + std::to_string(N) + " is not a power of two >= 2");
    if (!(eps > 0.0)) return ls::fail(LS_EVALIDATION, "qtt_compress: eps must be positive");
    if (ncols < 0 || ldv < N || rmax < 1 || rmax > 64) return ls::fail(LS_EVALIDATION, "qtt_compress: bad arguments");
    if (core_stride < ls_qtt_core_stride(N, rmax)) return ls::fail(LS_EVALIDATION, "qtt_compress: core stride too small");
    if (ncols == 0) return LS_OK;
    const cudaStream_t s = ls::as_stream(stream);
    ls::ensure_pool();
    ls::AsyncScratch scratch(s);
    LS_CUDA(scratch.alloc(sizeof(double) * 2 * N * ncols));
    const int nmax = 2 * rmax;
    const size_t smem = sizeof(double) * (nmax * nmax + nmax + kQttWarps) + sizeof(int) * (nmax + 2);
    LS_CUDA(cudaFuncSetAttribute(qtt_compress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    qtt_compress_kernel<<<ncols, kQttThreads, smem, s>>>(V_d, ldv, N, L, eps, rmax, cores_d, core_stride, ranks_d,
                                                         capped_d, scratch.as<double>());
    LS_LAUNCHED("qtt_compress_kernel");
    return LS_OK;
}

int ls_qtt_unfolding_ranks(const double* V_d, int64_t ldv, int64_t N, int ncols, double eps, int* ranks_d,
                           void* stream) {
    const int L = log2_pow2(N);
    if (L < 1) return ls::fail(LS_EVALIDATION, "unfolding_rank_profile: length is not a power of two >= 2");
    if (!(eps > 0.0)) return ls::fail(LS_EVALIDATION, "unfolding_rank_profile: eps must be positive");
    if (ncols < 0 || ldv < N) return ls::fail(LS_EVALIDATION, "unfolding_rank_profile: bad arguments");
    if (L > 26) return ls::fail(LS_EGUARD, "unfolding_rank_profile: length above 2^26");
    if (ncols == 0 || L < 2) return LS_OK;
    const cudaStream_t s = ls::as_stream(stream);
    ls::ensure_pool();
    ls::AsyncScratch scratch(s);
    LS_CUDA(scratch.alloc(sizeof(double) * N * ncols));
    const int nmax = 1 << ((L + 1) / 2);
    const size_t smem = sizeof(double) * (nmax + kQttWarps) + sizeof(int) * (nmax + 2);
    LS_CUDA(cudaFuncSetAttribute(qtt_unfolding_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    qtt_unfolding_kernel<<<ncols, kQttThreads, smem, s>>>(V_d, ldv, N, L, eps, ranks_d, scratch.as<double>());
    LS_LAUNCHED("qtt_unfolding_kernel");
    return LS_OK;
}

}  // extern "C"
