// expand.cu -- K3: rank-R expansion of a canonical tensor onto the N1 x N2 x N3
// grid, FP64 on the tensor cores (DMMA, mma.sync.m8n8k4.f64).
//
// Reference: densify (canonical.hpp:251-266) -> detail::densify_slab
// (canonical.hpp:241-246): slab k = A1 * diag(w .* A3(k,:)) * A2^T, an Eigen
// GEMM with inner dimension R. Here each slab is the same GEMM, tiled for the
// B200 FP64 tensor pipe:
//
//   V(i, j, k) = sum_q A1k(i, q) * A2(j, q),   A1k(i, q) = A1(i, q) * (w_q * A3(k, q))
//
// (the scaled left factor rounds exactly as Eigen's A1 * scale.asDiagonal()).
// Measured on B200 (profiles/r01_fp64_peak_microbench.jsonl): DMMA m8n8k4
// sustains 37.07 TFLOP/s = 64 FMA/clk/SM, DFMA 34.1 TFLOP/s, and the two share
// one pipe; at R = 41 the expansion is 10.25 FLOP per output byte, above the
// HBM ridge (~5.6), so this kernel is FP64-pipe-bound and is built to keep the
// DMMA pipe issuing while the 8-byte-per-point output streams out.
//
// Work decomposition. A work unit is (i-chunk of IC rows, one slab k). A CTA
// of 8 warps scales A1 rows of its chunk by w .* A3(k,:) into shared memory
// (fragment order, conflict-free LDS.64), then sweeps j in chunks of JC
// columns: A2 rows are staged into a double-buffered shared tile with
// cp.async in K-chunks, each warp computes a (8*TN) i x (8*TM) j register
// tile with TM*TN independent DMMA accumulators, and stores it straight from
// the accumulator fragments as 16-byte stores (each lane owns two adjacent
// i). MMA orientation: M = j (A operand = A2 tile), N = i (B operand = A1k
// tile), K = q, so the D fragment (row g, cols 2t, 2t+1) is two consecutive
// i of one (j, k) row -- a 16-byte aligned pair in the i-fastest grid.
// Units are spread over a persistent grid (CTAs per SM x SM count).
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kTM = 4;            // j tiles (of 8) per warp
constexpr int kTN = 4;            // i tiles (of 8) per warp

struct ExpandArgs {
    const double* A;
    const double* B;
    const double* C;
    const double* w;
    int64_t lda, ldb, ldc;
    int64_t N1, N2, N3;
    int R;            // rank
    int KD;           // DMMA k-steps (4 ranks each); ranks >= 4*KD go to the DFMA tail
    int n_tail;       // R - 4*KD in {0, 1, 2}, or 0 when the last k-step is zero-padded
    int64_t k0, k1;
    double* out;
    int64_t ldy, ldz;
    int vec_store;    // 16-byte pair stores legal (aligned base, even strides)
    const double* rho1;
    const double* rho2;
    const double* rho3;
    double* partial;
    int64_t n_ichunks;
    int64_t n_units;
};

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// A2 fragment element for lane (g, t) of j-tile starting at j, k-step ks: A2(j + g, 4 ks + t).
__device__ __forceinline__ double load_b_frag(const ExpandArgs& p, int64_t j, int q) {
    return (j < p.N2 && q < p.R) ? __ldg(p.B + j + p.ldb * q) : 0.0;
}

template <int WI, bool STORE, bool FUNC>
__global__ void __launch_bounds__(kThreads, 2)
expand_dmma_kernel(const ExpandArgs p) {
    constexpr int WJ = kWarps / WI;
    constexpr int IC = 8 * kTN * WI;

    extern __shared__ __align__(16) double smem[];
    const int KD = p.KD;
    double* as = smem;                                       // [IC/8][KD][32] fragment order
    double* tail = as + static_cast<int64_t>(IC) * KD * 4;   // [n_tail][IC]
    double* scale = tail + 2 * IC;                           // [4*KD + n_tail]
    __shared__ double red[kWarps];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2;
    const int t = lane & 3;
    const int wi = warp % WI;
    const int wj = warp / WI;
    const int q_tail0 = 4 * KD;
    const int n_scale = q_tail0 + p.n_tail;

    for (int64_t unit = blockIdx.x; unit < p.n_units; unit += gridDim.x) {
        const int64_t ic = unit % p.n_ichunks;
        const int64_t kk = unit / p.n_ichunks;   // slab offset within [k0, k1)
        const int64_t k = p.k0 + kk;
        const int64_t i_base = ic * IC;

        __syncthreads();  // previous unit finished reading as / tail / scale
        // scale_q = w_q * A3(k, q)   (canonical.hpp:244)
        for (int q = threadIdx.x; q < n_scale; q += kThreads)
            scale[q] = q < p.R ? rn_mul(p.w[q], p.C[k + p.ldc * q]) : 0.0;
        __syncthreads();
        // A1k(i, q) = A1(i, q) * scale_q, Eigen's A1 * scale.asDiagonal(): DMMA part in fragment
        // order (lane (g, t) of i-tile it, k-step ks <-> A1k(8 it + g, 4 ks + t)), tail row-wise.
        for (int e = threadIdx.x; e < IC * KD * 4; e += kThreads) {
            const int ln = e & 31;
            const int ks = (e >> 5) % KD;
            const int it = (e >> 5) / KD;
            const int64_t i = i_base + it * 8 + (ln >> 2);
            const int q = ks * 4 + (ln & 3);
            as[e] = (i < p.N1 && q < p.R) ? rn_mul(p.A[i + p.lda * q], scale[q]) : 0.0;
        }
        for (int e = threadIdx.x; e < p.n_tail * IC; e += kThreads) {
            const int q = q_tail0 + e / IC;
            const int64_t i = i_base + e % IC;
            tail[e] = i < p.N1 ? rn_mul(p.A[i + p.lda * q], scale[q]) : 0.0;
        }
        __syncthreads();

        double fsum = 0.0;  // FUNC: this thread's rho-weighted partial over the unit
        const double* asw = as + (wi * kTN) * (KD * 32) + lane;
        const int64_t ibase = i_base + wi * (8 * kTN);

        // Each warp sweeps its own j-blocks: no block-level synchronisation until the next unit.
        for (int64_t jb = static_cast<int64_t>(wj) * (8 * kTM); jb < p.N2; jb += WJ * (8 * kTM)) {
            double acc[kTM][kTN][2];
#pragma unroll
            for (int m = 0; m < kTM; ++m)
#pragma unroll
                for (int nn = 0; nn < kTN; ++nn) acc[m][nn][0] = acc[m][nn][1] = 0.0;

            // Register double-buffering: fragments of k-step ks+1 load while ks multiplies.
            double a_nx[kTM], b_nx[kTN];
#pragma unroll
            for (int m = 0; m < kTM; ++m) a_nx[m] = load_b_frag(p, jb + 8 * m + g, t);
#pragma unroll
            for (int nn = 0; nn < kTN; ++nn) b_nx[nn] = asw[nn * (KD * 32)];
#pragma unroll 2
            for (int ks = 0; ks < KD; ++ks) {
                double a[kTM], b[kTN];
#pragma unroll
                for (int m = 0; m < kTM; ++m) a[m] = a_nx[m];
#pragma unroll
                for (int nn = 0; nn < kTN; ++nn) b[nn] = b_nx[nn];
                if (ks + 1 < KD) {
#pragma unroll
                    for (int m = 0; m < kTM; ++m) a_nx[m] = load_b_frag(p, jb + 8 * m + g, 4 * (ks + 1) + t);
#pragma unroll
                    for (int nn = 0; nn < kTN; ++nn) b_nx[nn] = asw[nn * (KD * 32) + (ks + 1) * 32];
                }
#pragma unroll
                for (int m = 0; m < kTM; ++m)
#pragma unroll
                    for (int nn = 0; nn < kTN; ++nn) dmma_884(acc[m][nn][0], acc[m][nn][1], a[m], b[nn]);
            }
            // Rank remainder (R mod 4 <= 2) on the DFMA path instead of a zero-padded k-step:
            // lane (g, t) owns V(i = ibase + 8 nn + 2t + {0,1}, j = jb + 8 m + g).
            for (int qt = 0; qt < p.n_tail; ++qt) {
                const int q = q_tail0 + qt;
                double bt[kTM];
#pragma unroll
                for (int m = 0; m < kTM; ++m) bt[m] = load_b_frag(p, jb + 8 * m + g, q);
#pragma unroll
                for (int nn = 0; nn < kTN; ++nn) {
                    const double2 at = *reinterpret_cast<const double2*>(
                        tail + qt * IC + wi * (8 * kTN) + 8 * nn + 2 * t);
#pragma unroll
                    for (int m = 0; m < kTM; ++m) {
                        acc[m][nn][0] = fma(at.x, bt[m], acc[m][nn][0]);
                        acc[m][nn][1] = fma(at.y, bt[m], acc[m][nn][1]);
                    }
                }
            }

            // Epilogue: lane owns (j = jb + 8m + g, i = ibase + 8nn + 2t + {0,1}).
#pragma unroll
            for (int m = 0; m < kTM; ++m) {
                const int64_t j = jb + 8 * m + g;
                if (j >= p.N2) continue;
                double* row = STORE ? p.out + kk * p.ldz + j * p.ldy : nullptr;
                double r2 = 0.0;
                if (FUNC) r2 = p.rho2[j];
#pragma unroll
                for (int nn = 0; nn < kTN; ++nn) {
                    const int64_t i = ibase + 8 * nn + 2 * t;
                    if (i + 1 < p.N1) {
                        if (STORE) {
                            if (p.vec_store) {
                                __stcs(reinterpret_cast<double2*>(row + i),
                                       make_double2(acc[m][nn][0], acc[m][nn][1]));
                            } else {
                                row[i] = acc[m][nn][0];
                                row[i + 1] = acc[m][nn][1];
                            }
                        }
                        if (FUNC)
                            fsum += rn_mul(rn_mul(acc[m][nn][0], p.rho1[i]), r2) +
                                    rn_mul(rn_mul(acc[m][nn][1], p.rho1[i + 1]), r2);
                    } else if (i < p.N1) {
                        if (STORE) row[i] = acc[m][nn][0];
                        if (FUNC) fsum += rn_mul(rn_mul(acc[m][nn][0], p.rho1[i]), r2);
                    }
                }
            }
        }

        if (FUNC) {
            // Fixed-order reduction: lanes by xor-tree, then warps in index order.
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, off);
            if (lane == 0) red[warp] = fsum;
            __syncthreads();
            if (threadIdx.x == 0) {
                double s = 0.0;
                for (int wv = 0; wv < kWarps; ++wv) s += red[wv];
                p.partial[unit] = rn_mul(s, p.rho3[k]);
            }
        }
    }
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int64_t count,
                                    double* __restrict__ out) {
    // One block, fixed order: thread-strided partial sums, then a fixed tree.
    __shared__ double sh[1024];
    double s = 0.0;
    for (int64_t u = threadIdx.x; u < count; u += blockDim.x) s += part[u];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = sh[0];
}

// DMMA k-steps and DFMA tail for rank R: a remainder of 1 or 2 ranks is cheaper on DFMA
// (2 FMA-lanes per output each) than a zero-padded 4-rank DMMA step.
void split_rank(int R, int& KD, int& n_tail) {
    KD = R / 4;
    n_tail = R % 4;
    if (n_tail == 3) {
        KD += 1;
        n_tail = 0;
    }
}

template <int WI>
size_t smem_bytes(int KD) {
    constexpr int IC = 8 * kTN * WI;
    return sizeof(double) * (static_cast<size_t>(IC) * KD * 4 + 2 * static_cast<size_t>(IC) +
                             static_cast<size_t>(KD) * 4 + 4);
}

// Shared-memory budget per CTA (B200: 227 KB opt-in; two CTAs per SM share 228 KB).
constexpr size_t kSmemLimit = 227 * 1024;

int choose_wi(int KD) {
    if (smem_bytes<4>(KD) * 2 <= kSmemLimit - 2048) return 4;  // two CTAs per SM
    if (smem_bytes<1>(KD) * 2 <= kSmemLimit - 2048) return 1;
    if (smem_bytes<1>(KD) <= kSmemLimit) return 1;
    return 0;
}

template <int WI, bool STORE, bool FUNC>
int launch(ExpandArgs& a, cudaStream_t s) {
    constexpr int IC = 8 * kTN * WI;
    a.n_ichunks = ls::ceil_div(a.N1, IC);
    a.n_units = a.n_ichunks * (a.k1 - a.k0);
    const size_t smem = smem_bytes<WI>(a.KD);
    auto kern = expand_dmma_kernel<WI, STORE, FUNC>;
    LS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int per_sm = (2 * smem + 2048 <= kSmemLimit) ? 2 : 1;
    const int64_t grid = std::min<int64_t>(a.n_units, (int64_t)ls::sm_count() * per_sm);
    if (grid <= 0) return LS_OK;
    kern<<<(unsigned)grid, kThreads, smem, s>>>(a);
    LS_LAUNCHED("expand_dmma_kernel");
    return LS_OK;
}

}  // namespace

extern "C" int64_t ls_expand_partial_count(int64_t N1, int64_t N2, int R, int64_t k0, int64_t k1) {
    (void)N2;
    int KD, n_tail;
    split_rank(std::max(R, 1), KD, n_tail);
    const int wi = choose_wi(KD);
    if (wi == 0 || k1 < k0) return -1;
    const int64_t IC = 8 * kTN * wi;
    return ls::ceil_div(N1, IC) * (k1 - k0);
}

extern "C" int ls_expand(const double* A_d, int64_t lda, const double* B_d, int64_t ldb,
                         const double* C_d, int64_t ldc, const double* w_d, int64_t N1, int64_t N2,
                         int64_t N3, int R, int64_t k0, int64_t k1, double* out_d, int64_t ldy,
                         int64_t ldz, const double* rho1_d, const double* rho2_d,
                         const double* rho3_d, double* partial_d, void* stream) {
    if (N1 < 0 || N2 < 0 || N3 < 0 || R < 0)
        return ls::fail(LS_EVALIDATION, "expand: negative dimension or rank");
    if (k0 < 0 || k1 > N3 || k0 > k1) return ls::fail(LS_EVALIDATION, "expand: slab range outside [0, N3]");
    if (lda < N1 || ldb < N2 || ldc < N3) return ls::fail(LS_EVALIDATION, "expand: leading dimension too small");
    if (ldy == 0) ldy = N1;
    if (ldz == 0) ldz = ldy * N2;
    if (ldy < N1 || ldz < ldy * N2) return ls::fail(LS_EVALIDATION, "expand: output strides too small");
    const bool func = rho1_d != nullptr;
    if (func && (!rho2_d || !rho3_d || !partial_d))
        return ls::fail(LS_EVALIDATION, "expand: functional epilogue needs rho1, rho2, rho3 and partial");
    if (!out_d && !func) return ls::fail(LS_EVALIDATION, "expand: nothing to do (no output, no functional)");
    if (N1 == 0 || N2 == 0 || k1 == k0) return LS_OK;
    const cudaStream_t s = ls::as_stream(stream);
    if (R == 0) {
        // Rank-0 tensor is the zero tensor (canonical.hpp:243).
        if (out_d)
            for (int64_t kk = 0; kk < k1 - k0; ++kk)
                LS_CUDA(cudaMemset2DAsync(out_d + kk * ldz, ldy * sizeof(double), 0, N1 * sizeof(double), N2, s));
        if (func) LS_CUDA(cudaMemsetAsync(partial_d, 0, sizeof(double) * ls_expand_partial_count(N1, N2, 4, k0, k1), s));
        return LS_OK;
    }
    ExpandArgs a{};
    a.A = A_d; a.B = B_d; a.C = C_d; a.w = w_d;
    a.lda = lda; a.ldb = ldb; a.ldc = ldc;
    a.N1 = N1; a.N2 = N2; a.N3 = N3;
    a.R = R;
    split_rank(R, a.KD, a.n_tail);
    a.k0 = k0; a.k1 = k1;
    a.out = out_d; a.ldy = ldy; a.ldz = ldz;
    a.vec_store = (ldy % 2 == 0 && ldz % 2 == 0 && (reinterpret_cast<uintptr_t>(out_d) & 15) == 0) ? 1 : 0;
    a.rho1 = rho1_d; a.rho2 = rho2_d; a.rho3 = rho3_d; a.partial = partial_d;
    const int wi = choose_wi(a.KD);
    if (wi == 0) return ls::fail(LS_EGUARD, "expand: rank too large for the shared-memory tile");
    const bool store = out_d != nullptr;
    if (wi == 4) {
        if (store && func) return launch<4, true, true>(a, s);
        if (store) return launch<4, true, false>(a, s);
        return launch<4, false, true>(a, s);
    }
    if (store && func) return launch<1, true, true>(a, s);
    if (store) return launch<1, true, false>(a, s);
    return launch<1, false, true>(a, s);
}

extern "C" int ls_sum_partials(const double* partial_d, int64_t count, double* out_d, void* stream) {
    if (count < 0) return ls::fail(LS_EVALIDATION, "sum_partials: negative count");
    sum_partials_kernel<<<1, 1024, 0, ls::as_stream(stream)>>>(partial_d, count, out_d);
    LS_LAUNCHED("sum_partials_kernel");
    return LS_OK;
}
