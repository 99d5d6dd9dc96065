// generator.cu -- K1: the rank-R sinc-quadrature Newton-kernel master.
//
// Reference: build_newton_master (newton.hpp:57-75) fills column q of each
// axis factor with gaussian_sample_vector(len, h, tau_q) (midpoint samples,
// newton.hpp:43-52), and the BASELINE generator uses the erf-difference cell
// integrals of gaussian_moment_vector (newton.hpp:21-37). Here every (q, i, len-1-i)
// mirrored pair of entries is one thread; the erf mode evaluates each cell vertex once in shared
// memory and differences neighbours, which is bit-identical to evaluating
// erf(t*x_{i+1}) and erf(t*x_i) separately as the reference does, and only the
// lower half of each (exactly even) column is evaluated.
#include "common.cuh"
#include "glibc_math.cuh"

#include <algorithm>

namespace {

constexpr int kGenThreads = 256;

// Both generators produce exactly even columns: cell len-1-i mirrors cell i, bit for bit, in
// the reference as here (test_newton.cpp:71-77, :93). The midpoint of cell len-1-i is the exact
// negation of cell i's ((i + 0.5 - len/2) is exact), and erf is odd, so the vertex erf values
// mirror with a sign flip and (-a) - (-b) rounds exactly like b - a. Each thread therefore
// evaluates one cell of the lower half and writes it and its mirror: half the exp/erf calls.

// newton.hpp:46-50 with GridSpec::midpoint (grid.hpp:32-34):
//   x = t * ((i + 0.5 - len/2) * h);  out = exp(-x*x)
__global__ void gen_midpoint_kernel(const double* __restrict__ tau, int64_t len, double h,
                                    double* __restrict__ out, int64_t ld) {
    pdl_trigger();  // the assembly may start launching (it waits for this grid before reading)
    const int q = blockIdx.y;
    const double t = tau[q];
    const double half_len = static_cast<double>(len) / 2.0;
    double* col = out + ld * q;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len / 2;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double mid = rn_mul(rn_sub(rn_add(static_cast<double>(i), 0.5), half_len), h);
        const double x = rn_mul(t, mid);
        const double v = ls::gm::exp(-rn_mul(x, x));  // glibc exp, bit for bit
        col[i] = v;
        col[len - 1 - i] = v;
    }
}

// newton.hpp:28-36: t == 0 -> h; else sqrt(pi)/(2t) * (erf(t*v(i+1)) - erf(t*v(i))),
// v(i) = (i - len/2) * h. Block b covers the lower-half cells [i0, i0 + blockDim) and the
// blockDim + 1 vertices bounding them; cell len-1-i gets the same value (see above).
__global__ void gen_erf_kernel(const double* __restrict__ tau, int64_t len, double h,
                               double* __restrict__ out, int64_t ld) {
    pdl_trigger();
    __shared__ double ev[kGenThreads + 1];
    const int q = blockIdx.y;
    const double t = tau[q];
    const int64_t half = len / 2;
    const int64_t i0 = blockIdx.x * (int64_t)kGenThreads;
    const int64_t i = i0 + threadIdx.x;
    double* col = out + ld * q;
    if (t == 0.0) {
        if (i < half) col[i] = col[len - 1 - i] = h;
        return;
    }
    for (int v = threadIdx.x; v <= kGenThreads; v += kGenThreads) {
        const int64_t vi = i0 + v;
        if (vi <= half) ev[v] = ls::gm::erf(rn_mul(t, rn_mul(static_cast<double>(vi - half), h)));
    }
    __syncthreads();
    if (i < half) {
        const double scale = __ddiv_rn(sqrt(CUDART_PI), rn_mul(2.0, t));
        const double v = rn_mul(scale, rn_sub(ev[threadIdx.x + 1], ev[threadIdx.x]));
        col[i] = v;
        col[len - 1 - i] = v;
    }
}

// Generator and assembled sum in one launch (small lattices: the step of cfg0 / cfg1 runs two
// latency-bound launches less). Block (q, a) evaluates master column q of axis a into shared
// memory with exactly the expressions of gen_erf_kernel / gen_midpoint_kernel, writes it to HBM
// (ls_pipeline_assemble and the host calls still read it there), then forms every assembled
// output of column q from it, one dependent left-to-right chain per output as in
// assemble_box_kernel / assemble_axis_kernel (lattice.hpp:220-274): bit-identical factors.
constexpr int kGaThreads = 512;
struct GenAsmParams {
    ls::GenAsmAxis ax[3];
    const double* tau;
    int R, M0, mode, periodic;
    int64_t n;
    double h;
};

__global__ void __launch_bounds__(kGaThreads) gen_assemble_kernel(const GenAsmParams p) {
    pdl_wait();  // the previous step's launches may still read the master / factors
    pdl_trigger();
    extern __shared__ double sm[];
    const ls::GenAsmAxis A = p.ax[blockIdx.y];
    const int q = blockIdx.x;
    const int64_t n = p.n, L = A.L, N = L * n, len = 2 * N, half = len / 2;
    double* m = sm;         // [len] master column q
    double* ev = sm + len;  // [half + 1] erf at the cell vertices
    const double t = p.tau[q], h = p.h;
    if (p.mode == LS_GEN_ERF) {
        if (t == 0.0) {
            for (int64_t i = threadIdx.x; i < len; i += blockDim.x) m[i] = h;
        } else {
            for (int64_t v = threadIdx.x; v <= half; v += blockDim.x)
                ev[v] = ls::gm::erf(rn_mul(t, rn_mul(static_cast<double>(v - half), h)));
            __syncthreads();
            const double scale = __ddiv_rn(sqrt(CUDART_PI), rn_mul(2.0, t));
            for (int64_t i = threadIdx.x; i < half; i += blockDim.x) m[i] = m[len - 1 - i] = rn_mul(scale, rn_sub(ev[i + 1], ev[i]));
        }
    } else {
        const double half_len = static_cast<double>(len) / 2.0;
        for (int64_t i = threadIdx.x; i < half; i += blockDim.x) {
            const double x = rn_mul(t, rn_mul(rn_sub(rn_add(static_cast<double>(i), 0.5), half_len), h));
            m[i] = m[len - 1 - i] = ls::gm::exp(-rn_mul(x, x));
        }
    }
    __syncthreads();
    double* mcol = A.master_d + len * q;
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) mcol[i] = m[i];
    const int64_t out_len = p.periodic ? n : N;
    for (int64_t e = threadIdx.x; e < p.M0 * out_len; e += blockDim.x) {
        const int64_t nu = e / out_len, o = e - nu * out_len;
        const double* src = m + ls::window_start(p.periodic, N, L, n, A.ia_d[nu]) + o;
        double acc = src[0];
#pragma unroll 8
        for (int64_t k = 1; k < L; ++k) acc = rn_add(acc, src[-k * n]);
        A.out_d[out_len * (nu * p.R + q) + o] = acc;
    }
}

// Periodic lattices with long chains and one charge (cfg4: L = 64..256, n = 256): the
// generator and the assembled sum fused WITHOUT materializing the master. Every master entry is
// used by exactly one assembled output there, so block (32-residue block, q, axis) evaluates
// the cells its 32 chains need straight from the reference's formula (erf mode: the 33 cell
// vertices of each shift k; every cell directly, as the reference does -- equal, bit for bit,
// to the generator's mirrored half), stages them in shared memory, and one warp runs the 32
// ascending-k chains. The 43 MB master of cfg4 L = 256 is never written or read back.
constexpr int kGpIB = 32;
__global__ void __launch_bounds__(1024) gen_assemble_periodic_kernel(const GenAsmParams p) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double ev[];  // [L][kGpIB + 1]: erf at the vertices (erf) or the cells (midpoint)
    const ls::GenAsmAxis A = p.ax[blockIdx.z];
    const int q = blockIdx.y;
    const int64_t n = p.n, L = A.L, N = L * n, half = N;  // master length 2N, vertex v at (v - N) h
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kGpIB;
    const double t = p.tau[q], h = p.h;
    const int64_t s0 = ls::window_start(1, N, L, n, A.ia_d[0]) + i0;  // cell of chain i0, shift 0
    constexpr int W = kGpIB + 1;
    const bool erf_mode = p.mode == LS_GEN_ERF;
    if (!(erf_mode && t == 0.0)) {
        const double half_len = static_cast<double>(2 * N) / 2.0;
        for (int64_t e = threadIdx.x; e < L * W; e += blockDim.x) {
            const int64_t k = e / W;
            const int c = static_cast<int>(e - k * W);
            const int64_t v = s0 - k * n + c;  // vertex (erf) or cell (midpoint) index
            if (erf_mode) {
                ev[e] = ls::gm::erf(rn_mul(t, rn_mul(static_cast<double>(v - half), h)));
            } else if (c < kGpIB) {
                const double x = rn_mul(t, rn_mul(rn_sub(rn_add(static_cast<double>(v), 0.5), half_len), h));
                ev[e] = ls::gm::exp(-rn_mul(x, x));
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < kGpIB && i0 + threadIdx.x < n) {
        const double* col = ev + threadIdx.x;
        double acc;
        if (erf_mode && t == 0.0) {
            acc = h;
            for (int64_t k = 1; k < L; ++k) acc = rn_add(acc, h);
        } else if (erf_mode) {
            const double scale = __ddiv_rn(sqrt(CUDART_PI), rn_mul(2.0, t));
            acc = rn_mul(scale, rn_sub(col[1], col[0]));
#pragma unroll 8
            for (int64_t k = 1; k < L; ++k) acc = rn_add(acc, rn_mul(scale, rn_sub(col[k * W + 1], col[k * W])));
        } else {
            acc = col[0];
#pragma unroll 8
            for (int64_t k = 1; k < L; ++k) acc = rn_add(acc, col[k * W]);
        }
        A.out_d[n * q + i0 + threadIdx.x] = acc;  // column q (M0 = 1), leading dim n
    }
}

__global__ void libm_eval_kernel(int fn, const double* __restrict__ x, double* __restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = fn == LS_LIBM_ERF ? ls::gm::erf(x[i]) : ls::gm::exp(x[i]);
}

}  // namespace

extern "C" int ls_libm_eval(int fn, const double* x_d, double* y_d, int64_t n, void* stream) {
    if (fn != LS_LIBM_ERF && fn != LS_LIBM_EXP) return ls::fail(LS_EVALIDATION, "libm_eval: unknown function");
    if (n < 0) return ls::fail(LS_EVALIDATION, "libm_eval: negative length");
    if (n == 0) return LS_OK;
    const int blocks = (int)std::min<int64_t>(ls::ceil_div(n, 256), 148 * 16);
    libm_eval_kernel<<<blocks, 256, 0, ls::as_stream(stream)>>>(fn, x_d, y_d, n);
    LS_LAUNCHED("libm_eval_kernel");
    return LS_OK;
}

extern "C" int ls_gen_master(int mode, const double* tau_d, int R, int64_t len, double h,
                             double* out_d, int64_t ld, void* stream) {
    if (len < 2 || len % 2 != 0)
        return ls::fail(LS_EVALIDATION, "gen_master: length must be even and >= 2");
    if (!(h > 0.0)) return ls::fail(LS_EVALIDATION, "gen_master: mesh h must be positive");
    if (R < 0 || ld < len) return ls::fail(LS_EVALIDATION, "gen_master: bad rank or leading dim");
    if (R == 0) return LS_OK;
    if (R > 65535) return ls::fail(LS_EGUARD, "gen_master: rank above 65535");
    const cudaStream_t s = ls::as_stream(stream);
    if (mode == LS_GEN_MIDPOINT) {
        const int64_t blocks = std::min<int64_t>(ls::ceil_div(len / 2, kGenThreads), 4096);
        gen_midpoint_kernel<<<dim3((unsigned)blocks, R), kGenThreads, 0, s>>>(tau_d, len, h, out_d, ld);
        LS_LAUNCHED("gen_midpoint_kernel");
    } else if (mode == LS_GEN_ERF) {
        const int64_t blocks = ls::ceil_div(len / 2, kGenThreads);
        if (blocks > 0x7fffffff) return ls::fail(LS_EGUARD, "gen_master: length too large");
        gen_erf_kernel<<<dim3((unsigned)blocks, R), kGenThreads, 0, s>>>(tau_d, len, h, out_d, ld);
        LS_LAUNCHED("gen_erf_kernel");
    } else {
        return ls::fail(LS_EVALIDATION, "gen_master: unknown mode");
    }
    return LS_OK;
}

namespace ls {

// Shared memory of the fused launch and its bound: master + vertices of the longest axis, and
// at most 8192 assembled outputs per column. Measured (tools/lab/gen_asm.py, back-to-back
// calls): cfg1 7.5 us fused against 7.8 + 7.4 us for the two launches, the cfg0 step 59.9 ->
// 54.9 us; at cfg3 (8 charges x 2048 outputs on 123 blocks) fusing gains nothing (31.5 us
// against 13.3 + 20.0), so the many-block assembly kernels keep such lattices.
constexpr int64_t kGaMaxSmem = 160 * 1024, kGaMaxOutputs = 8192;

int gen_assemble(int mode, const double* tau_d, int R, int M0, int64_t n, double h, int periodic,
                 const GenAsmAxis* ax, int n_ax, cudaStream_t s, bool* master_written) {
    if (master_written) *master_written = true;
    if (n_ax < 1 || n_ax > 3 || R < 1 || M0 < 1) return fail(LS_EVALIDATION, "gen_assemble: bad axis count or rank");
    // Periodic, one charge, long chains: generator and assembly fused, master never written.
    {
        int64_t L_max = 0, L_min = INT64_MAX;
        for (int a = 0; a < n_ax; ++a) {
            L_max = std::max(L_max, ax[a].L);
            L_min = std::min(L_min, ax[a].L);
        }
        const int64_t smem_p = sizeof(double) * L_max * (kGpIB + 1);
        if (periodic && M0 == 1 && L_min >= 32 && smem_p <= kGaMaxSmem && R <= 65535 &&
            (mode == LS_GEN_ERF || mode == LS_GEN_MIDPOINT)) {
            static std::atomic<bool> attr_p[64] = {};
            int dev = 0;
            LS_CUDA(cudaGetDevice(&dev));
            if (dev >= 64 || !attr_p[dev]) {
                LS_CUDA(cudaFuncSetAttribute(gen_assemble_periodic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kGaMaxSmem)));
                if (dev < 64) attr_p[dev] = true;
            }
            // about eight vertex evaluations per thread (tools/lab/gen_asm.py: L = 64 with 256
            // threads, L = 256 with 1024)
            const int64_t gp_threads = std::min<int64_t>(1024, std::max<int64_t>(256, (L_max * (kGpIB + 1) / 8 + 255) / 256 * 256));
            GenAsmParams prm{};
            for (int a = 0; a < n_ax; ++a) prm.ax[a] = ax[a];
            prm.tau = tau_d;
            prm.R = R;
            prm.M0 = M0;
            prm.mode = mode;
            prm.periodic = 1;
            prm.n = n;
            prm.h = h;
            LS_CUDA(launch_pdl(gen_assemble_periodic_kernel,
                               dim3(static_cast<unsigned>(ceil_div(n, kGpIB)), static_cast<unsigned>(R),
                                    static_cast<unsigned>(n_ax)),
                               dim3(static_cast<unsigned>(gp_threads)), static_cast<size_t>(smem_p), s, prm));
            LS_LAUNCHED("gen_assemble_periodic_kernel");
            if (master_written) *master_written = false;
            return LS_OK;
        }
    }
    int64_t len_max = 0;
    bool fused = R <= 65535;
    for (int a = 0; a < n_ax; ++a) {
        const int64_t len = 2 * ax[a].L * n;
        len_max = std::max(len_max, len);
        if (static_cast<int64_t>(M0) * (periodic ? n : ax[a].L * n) > kGaMaxOutputs) fused = false;
    }
    const int64_t smem = sizeof(double) * (len_max + len_max / 2 + 1);
    fused = fused && smem <= kGaMaxSmem && (mode == LS_GEN_ERF || mode == LS_GEN_MIDPOINT);
    if (!fused) {
        for (int a = 0; a < n_ax; ++a) {
            const int64_t len = 2 * ax[a].L * n;
            if (const int rc = ls_gen_master(mode, tau_d, R, len, h, ax[a].master_d, len, s)) return rc;
            if (const int rc = ls_assemble_axis(ax[a].master_d, len, R, M0, ax[a].ia_d, n, ax[a].L, periodic, ax[a].out_d,
                                                periodic ? n : ax[a].L * n, s))
                return rc;
        }
        return LS_OK;
    }
    static std::atomic<bool> attr_set[64] = {};
    int dev = 0;
    LS_CUDA(cudaGetDevice(&dev));
    if (dev >= 64 || !attr_set[dev]) {
        LS_CUDA(cudaFuncSetAttribute(gen_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kGaMaxSmem)));
        if (dev < 64) attr_set[dev] = true;
    }
    GenAsmParams prm{};
    for (int a = 0; a < n_ax; ++a) prm.ax[a] = ax[a];
    prm.tau = tau_d;
    prm.R = R;
    prm.M0 = M0;
    prm.mode = mode;
    prm.periodic = periodic ? 1 : 0;
    prm.n = n;
    prm.h = h;
    LS_CUDA(launch_pdl(gen_assemble_kernel, dim3(static_cast<unsigned>(R), static_cast<unsigned>(n_ax)),
                       dim3(kGaThreads), static_cast<size_t>(smem), s, prm));
    LS_LAUNCHED("gen_assemble_kernel");
    return LS_OK;
}

}  // namespace ls
