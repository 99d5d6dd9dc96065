// grid_batch.cu -- K4b: a batch of F separable functionals of a dense device grid,
//
//   out[f] (+)= scale * sum_{i,j,k} V(i,j,k) * X(i,f) * Y(j,f) * Z(k,f),
//
// the full-grid form of SURVEY a18 for cfg4's batch of 1024 test functions (the 1D rank-term
// form is ls_functional_batch; the reference has only that form, scalar_product at
// canonical.hpp:126-136, which is the parity oracle for this kernel).
//
// It is a GEMM with a fused reduction epilogue. Rows m = j + N2*k of V^T (K = N1 along i)
// times X (K x F):
//   C[m, f] = sum_i V(i, m) X(i, f)            FP64 DMMA m8n8k4, 128 x 64 CTA tiles, K by 16
//   part[m_tile, f] = sum_{m in tile} C[m, f] * Y(j,f) * Z(k,f)      fixed-order epilogue
// then out[f] = scale * sum over m-tiles in a fixed order (grid_batch_reduce_kernel), so the
// result is bitwise reproducible. Operands stream global -> shared through TMA tensor maps
// (grid_batch_tma_kernel), or with cp.async when the slabs are padded (grid_batch_kernel);
// the f-tiles of one m-tile are adjacent in the launch order, so V is read from HBM once and
// re-read from L2. 2 * N1 * N2 * N3 * F FLOP; at cfg4 (256^3, F = 1024) 3.4e10.
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point; no -lcuda)

#include "k3.cuh"

namespace {

// Build-time tile knobs (tools/lab/build_variants.sh with SRC=grid_batch). Measured at cfg4:
// BN 64 x 3 stages 1.48 ms; BN 128 (16 warps, 1 CTA/SM) with 2/3/4 stages 1.59/1.57/1.56 ms.
#ifndef GB_BN
#define GB_BN 64
#endif
#ifndef GB_NS
#define GB_NS 3
#endif
constexpr int BM = 128, BN = GB_BN, BK = 16, PITCH = BK + 4, NSTAGE = GB_NS;  // pitch 20: conflict-free LDS.64
constexpr int kThreads = 32 * 4 * (BN / 32);  // 4 warps along m x BN/32 along f
constexpr int kMinBlocks = kThreads == 256 ? 2 : 1;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
template <int BYTES>
__device__ __forceinline__ void cp_async(double* dst, const double* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(su32(dst)), "l"(src), "n"(BYTES),
                 "r"(valid ? BYTES : 0)
                 : "memory");
}

struct GridBatchArgs {
    const double* V;
    int64_t N1, N2, N3, ldy, ldz;
    const double* X;
    int64_t ldx;
    const double* Y;
    int64_t ldyy;
    const double* Z;
    int64_t ldzz;
    int F;
    int64_t M;  // N2 * N3
    double* part;  // [n_mtiles][F]
    unsigned* fault;  // watchdog word of the device (ls::fault_flag)
};

// Epilogue shared by both feeds: weight by Y(j,f) * Z(k,f), sum this lane's rows (mi ascending),
// then the 8 lanes sharing a column (xor tree over g), then the 4 warps along m (ascending wm).
__device__ __forceinline__ void epilogue(const GridBatchArgs& p, const double (&acc)[4][4][2], double (*red)[BN],
                                         int64_t m0, int f0) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    double s[4][2];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) s[ni][0] = s[ni][1] = 0.0;
    const int64_t mb = m0 + wm * 32 + g;  // this lane's rows: mb + 8 mi
    const int64_t kb = mb / p.N2;
    if (mb + 24 < p.M && (mb + 24) / p.N2 == kb) {
        // All four rows lie in one slab k (the common case): Z(k, f) factors out of the row sum,
        // halving the weight loads and products.
        const int64_t jb = mb - kb * p.N2;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int f = f0 + wn * 32 + 8 * ni + 2 * t + e;
                if (f < p.F) {
                    const double* y = p.Y + jb + p.ldyy * f;
                    double sy = 0.0;
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) sy = fma(acc[mi][ni][e], __ldg(y + 8 * mi), sy);
                    s[ni][e] = rn_mul(sy, __ldg(p.Z + kb + p.ldzz * f));
                }
            }
    } else {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
            const int64_t m = mb + 8 * mi;
            if (m >= p.M) continue;
            const int64_t j = m % p.N2, k = m / p.N2;
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int f = f0 + wn * 32 + 8 * ni + 2 * t + e;
                    if (f < p.F) {
                        const double w = rn_mul(__ldg(p.Y + j + p.ldyy * f), __ldg(p.Z + k + p.ldzz * f));
                        s[ni][e] = fma(acc[mi][ni][e], w, s[ni][e]);
                    }
                }
        }
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double v = s[ni][e];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            if (g == 0) red[wm][wn * 32 + 8 * ni + 2 * t + e] = v;
        }
    __syncthreads();
    if (tid < BN && f0 + tid < p.F) {
        const double v = ((red[0][tid] + red[1][tid]) + red[2][tid]) + red[3][tid];
        p.part[static_cast<int64_t>(blockIdx.y) * p.F + f0 + tid] = v;
    }
}

// VEC: 16-byte copies (V, X 16-byte aligned, even strides); otherwise 8-byte copies.
template <bool VEC>
__global__ void __launch_bounds__(kThreads, kMinBlocks) grid_batch_kernel(const GridBatchArgs p) {
    extern __shared__ __align__(16) double sm[];
    double* As = sm;                           // [NSTAGE][BM][PITCH]
    double* Bs = sm + NSTAGE * BM * PITCH;     // [NSTAGE][BN][PITCH]
    __shared__ double red[4][BN];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const int f0 = blockIdx.x * BN;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
    const int n_kc = static_cast<int>((p.N1 + BK - 1) / BK);

    // Each thread copies fixed rows at a fixed column offset kk of every K chunk, so the row
    // addresses (a 64-bit div/mod for V's (j, k)) are computed once.
    constexpr int E = VEC ? 2 : 1;  // doubles per copy
    constexpr int PER_ROW = BK / E, STEP = kThreads / PER_ROW;
    constexpr int ARPT = BM / STEP, BRPT = BN / STEP;
    const int kk = (tid % PER_ROW) * E, r0 = tid / PER_ROW;
    int64_t abase[ARPT], bbase[BRPT];
#pragma unroll
    for (int n = 0; n < ARPT; ++n) {
        const int64_t m = m0 + r0 + n * STEP;
        abase[n] = m < p.M ? p.ldy * (m % p.N2) + p.ldz * (m / p.N2) : -1;
    }
#pragma unroll
    for (int n = 0; n < BRPT; ++n) {
        const int f = f0 + r0 + n * STEP;
        bbase[n] = f < p.F ? p.ldx * f : -1;
    }
    auto load = [&](int kc, int stage) {
        const int64_t i = static_cast<int64_t>(kc) * BK + kk;  // N1 is even when VEC: pairs never straddle
        double* as = As + stage * BM * PITCH + r0 * PITCH + kk;
        double* bs = Bs + stage * BN * PITCH + r0 * PITCH + kk;
#pragma unroll
        for (int n = 0; n < ARPT; ++n) {
            const bool ok = abase[n] >= 0 && i < p.N1;
            cp_async<8 * E>(as + n * STEP * PITCH, ok ? p.V + abase[n] + i : p.V, ok);
        }
#pragma unroll
        for (int n = 0; n < BRPT; ++n) {
            const bool ok = bbase[n] >= 0 && i < p.N1;
            cp_async<8 * E>(bs + n * STEP * PITCH, ok ? p.X + bbase[n] + i : p.X, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
    for (int s = 0; s < NSTAGE - 1; ++s) {
        if (s < n_kc) load(s, s);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int kc = 0; kc < n_kc; ++kc) {
        asm volatile("cp.async.wait_group %0;" ::"n"(NSTAGE - 2) : "memory");
        __syncthreads();
        const int nxt = kc + NSTAGE - 1;
        if (nxt < n_kc) load(nxt, nxt % NSTAGE);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        const double* as = As + (kc % NSTAGE) * BM * PITCH + (wm * 32 + g) * PITCH + t;
        const double* bs = Bs + (kc % NSTAGE) * BN * PITCH + (wn * 32 + g) * PITCH + t;
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            double a[4], b[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = as[mi * 8 * PITCH + 4 * ks];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = bs[ni * 8 * PITCH + 4 * ks];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");

    epilogue(p, acc, red, m0, f0);
}

// Tensor-map feed (V rows at one stride: slabs contiguous, ldz == ldy * N2). Each K chunk of
// 16 is two TMA boxes, V [128 rows x 128 B] and X [64 rows x 128 B], written with the 128-byte
// swizzle (16-byte chunk index XOR row & 7) into a 4-deep ring on one mbarrier per stage. The
// last warp to finish with a stage refills it, so there is no CTA barrier in the main loop.
// Out-of-range rows and columns arrive as zeros. K-step ks takes columns {2ks, 2ks+1, 2ks+8,
// 2ks+9} (lane t -> 2(ks + 4(t>>1)) + (t&1)), so a half-warp's 16 fragment loads hit 16 distinct
// 8-byte bank slots under the swizzle. A and B use the same column order.
constexpr int kTmaNS = 4;
constexpr int kTmaStageA = BM * BK * 8, kTmaStageB = BN * BK * 8, kTmaStage = kTmaStageA + kTmaStageB;
constexpr size_t kTmaSmem = static_cast<size_t>(kTmaNS) * kTmaStage + 1024;  // + 1024-byte alignment slack

__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(ls_k3::smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(kThreads, kMinBlocks)
    grid_batch_tma_kernel(const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tx,
                          const GridBatchArgs p) {
    extern __shared__ uint8_t raw[];
    __shared__ double red[4][BN];
    __shared__ uint64_t full[kTmaNS];
    __shared__ int released[kTmaNS];
    const uint32_t base = (ls_k3::smem_u32(raw) + 1023u) & ~1023u;
    const uint8_t* gbase = raw + (base - ls_k3::smem_u32(raw));

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const int f0 = blockIdx.x * BN;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
    const int n_kc = static_cast<int>((p.N1 + BK - 1) / BK);

    auto issue = [&](int kc) {  // one thread
        const int st = kc % kTmaNS;
        ls_k3::mbar_arrive_expect_tx(full + st, kTmaStage);
        tma_2d(base + st * kTmaStage, &tv, kc * BK, static_cast<int>(m0), full + st);
        tma_2d(base + st * kTmaStage + kTmaStageA, &tx, kc * BK, f0, full + st);
    };
    if (tid < kTmaNS) {
        ls_k3::mbar_init(full + tid, 1);
        released[tid] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tv)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tx)) : "memory");
        for (int kc = 0; kc < kTmaNS && kc < n_kc; ++kc) issue(kc);
    }

    // this lane's fragment offsets: rows (wm*32 | wn*32) + g + 8*i, swizzled column per k-step
    int col[BK / 4];
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) col[ks] = (((ks + 4 * (t >> 1)) ^ g) << 4) | ((t & 1) << 3);
    const int arow = (wm * 32 + g) * 128, brow = kTmaStageA + (wn * 32 + g) * 128;

    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    for (int kc = 0; kc < n_kc; ++kc) {
        const int st = kc % kTmaNS;
        ls_k3::mbar_wait(full + st, (kc / kTmaNS) & 1, p.fault);
        const uint8_t* sa = gbase + st * kTmaStage + arow;
        const uint8_t* sb = gbase + st * kTmaStage + brow;
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            double a[4], b[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = *reinterpret_cast<const double*>(sa + mi * 1024 + col[ks]);
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = *reinterpret_cast<const double*>(sb + ni * 1024 + col[ks]);
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
        // release the stage; the last warp refills it with chunk kc + kTmaNS
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(released + st, 1) == kThreads / 32 - 1) {
                released[st] = 0;
                __threadfence_block();
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (kc + kTmaNS < n_kc) issue(kc + kTmaNS);
            }
        }
    }
    epilogue(p, acc, red, m0, f0);
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_tiled() {
    static EncodeTiled fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            f = nullptr;
        }
        return reinterpret_cast<EncodeTiled>(f);
    }();
    return fn;
}

// rows x cols (cols contiguous, row stride ld doubles), box BK x box_rows, 128-byte swizzle
bool make_map(CUtensorMap* m, const double* ptr, int64_t cols, int64_t rows, int64_t ld, int box_rows) {
    const EncodeTiled enc = encode_tiled();
    if (enc == nullptr) return false;
    const cuuint64_t dim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t stride[1] = {static_cast<cuuint64_t>(ld) * 8};
    const cuuint32_t box[2] = {BK, static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estride[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dim, stride, box, estride,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// out[f] = scale * sum over m-tiles, in a fixed order: warp w of the block sums m-tiles
// w, w + 8, w + 16, ... (four independent chains interleaved by m mod 32; the tail goes to the first), then the
// block adds the 8 warp sums in ascending w. Lanes take 32 consecutive f, so loads coalesce.
// The order depends only on n_mtiles, so the result is bitwise reproducible.
constexpr int kRedWarps = 8;
__global__ void __launch_bounds__(32 * kRedWarps) grid_batch_reduce_kernel(const double* __restrict__ part,
                                                                          int64_t n_mtiles, int F, double scale,
                                                                          int accumulate, double* __restrict__ out) {
    __shared__ double red[kRedWarps][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int f = blockIdx.x * 32 + lane;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (f < F) {
        int64_t m = w;
        for (; m + 3 * kRedWarps < n_mtiles; m += 4 * kRedWarps)
#pragma unroll
            for (int c = 0; c < 4; ++c) s[c] += part[(m + c * kRedWarps) * F + f];
        for (; m < n_mtiles; m += kRedWarps) s[0] += part[m * F + f];
    }
    red[w][lane] = (s[0] + s[1]) + (s[2] + s[3]);
    __syncthreads();
    if (w == 0 && f < F) {
        double t = red[0][lane];
#pragma unroll
        for (int v = 1; v < kRedWarps; ++v) t += red[v][lane];
        t = rn_mul(t, scale);
        out[f] = accumulate ? out[f] + t : t;
    }
}

}  // namespace

extern "C" int ls_grid_functional_batch(const double* V_d, int64_t N1, int64_t N2, int64_t N3, int64_t ldy,
                                        int64_t ldz, const double* X_d, int64_t ldx, const double* Y_d,
                                        int64_t ldyy, const double* Z_d, int64_t ldzz, int F, double scale,
                                        int accumulate, double* out_d, void* stream) {
    if (N1 < 0 || N2 < 0 || N3 < 0 || F < 0 || ldy < N1 || ldz < ldy * N2 || ldx < N1 || ldyy < N2 || ldzz < N3)
        return ls::fail(LS_EVALIDATION, "grid_functional_batch: bad shape");
    if (F == 0) return LS_OK;
    const cudaStream_t s = ls::as_stream(stream);
    const int64_t M = N2 * N3;
    if (M == 0 || N1 == 0) {
        if (!accumulate) LS_CUDA(cudaMemsetAsync(out_d, 0, sizeof(double) * F, s));
        return LS_OK;
    }
    const int64_t n_mtiles = ls::ceil_div(M, BM);
    if (n_mtiles > 65535) return ls::fail(LS_EGUARD, "grid_functional_batch: more than 65535*128 rows (split k)");
    ls::ensure_pool();
    ls::AsyncScratch scratch(s);  // freed on every exit path
    LS_CUDA(scratch.alloc(sizeof(double) * n_mtiles * F));
    double* part = scratch.as<double>();
    GridBatchArgs a{V_d, N1, N2, N3, ldy, ldz, X_d, ldx, Y_d, ldyy, Z_d, ldzz, F, M, part, ls::fault_flag()};
    const bool vec = (reinterpret_cast<uintptr_t>(V_d) % 16 == 0) && (reinterpret_cast<uintptr_t>(X_d) % 16 == 0) &&
                     N1 % 2 == 0 && ldy % 2 == 0 && ldz % 2 == 0 && ldx % 2 == 0;
    const dim3 grid(static_cast<unsigned>(ls::ceil_div(F, BN)), static_cast<unsigned>(n_mtiles));
    // tensor-map feed when the rows have one stride (and within TMA's limits), else cp.async
    CUtensorMap tv, tx;
    const bool tma = vec && ldz == ldy * N2 && M <= INT32_MAX && ldy < (int64_t(1) << 36) &&
                     ldx < (int64_t(1) << 36) && ls::dev_knob("LS_GRID_BATCH_CPASYNC") == nullptr &&
                     make_map(&tv, V_d, N1, M, ldy, BM) && make_map(&tx, X_d, N1, F, ldx, BN);
    if (tma) {
        LS_CUDA(cudaFuncSetAttribute(grid_batch_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kTmaSmem)));
        grid_batch_tma_kernel<<<grid, kThreads, kTmaSmem, s>>>(tv, tx, a);
        LS_LAUNCHED("grid_batch_tma_kernel");
    } else {
        const size_t smem = sizeof(double) * NSTAGE * (BM + BN) * PITCH;
        void (*kern)(GridBatchArgs) = vec ? grid_batch_kernel<true> : grid_batch_kernel<false>;
        LS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, kThreads, smem, s>>>(a);
        LS_LAUNCHED("grid_batch_kernel");
    }
    grid_batch_reduce_kernel<<<static_cast<unsigned>(ls::ceil_div(F, 32)), 32 * kRedWarps, 0, s>>>(
        part, n_mtiles, F, scale, accumulate, out_d);
    LS_LAUNCHED("grid_batch_reduce_kernel");
    return LS_OK;
}
