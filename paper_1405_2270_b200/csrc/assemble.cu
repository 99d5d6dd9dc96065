// assemble.cu -- K2: the assembled O(N L R) lattice summation.
//
// Reference: detail::assembled_axis_columns (lattice.hpp:220-274). Column
// c = (nu, q) of the per-axis factor is the sum over the L lattice shifts of
// the windowed master column, added strictly left to right in ascending k
// (the reference's eight-stream blocks keep that order, lattice.hpp:240-271).
// One thread per output entry keeps exactly that recurrence, so the result is
// bit-identical to the reference. Consecutive threads own consecutive i, so
// every one of the L loads of a warp is a coalesced 256-byte row of the
// master column; the loads are independent and the adds form one chain.
#include "common.cuh"

namespace {

constexpr int kAsmThreads = 256;

__global__ void assemble_axis_kernel(const double* __restrict__ master, int64_t ld_master, int R,
                                     const int64_t* __restrict__ ia, int64_t n, int64_t L,
                                     int periodic, int64_t out_len, double* __restrict__ out,
                                     int64_t ld_out) {
    pdl_wait();  // the master comes from the preceding generator launch
    pdl_trigger();
    const int c = blockIdx.y;  // column nu*R + q
    const int nu = c / R;
    const int q = c % R;
    const int64_t N = L * n;
    // lattice.hpp:98 / :104-106 at k = 0; the window for shift k starts k*n lower.
    const int64_t s0 = periodic ? N + (L / 2) * n - ia[nu] : N - ia[nu];
    const double* base = master + ld_master * q + s0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < out_len;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double* p = base + i;
        double acc = p[0];
        int64_t k = 1;
        // Loads are hoisted in groups of 8; the adds stay in ascending-k order.
        for (; k + 8 <= L; k += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(p - (k + u) * n);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = rn_add(acc, v[u]);
        }
        for (; k < L; ++k) acc = rn_add(acc, __ldg(p - k * n));
        out[i + ld_out * c] = acc;
    }
}

}  // namespace

extern "C" int ls_assemble_axis(const double* master_d, int64_t ld_master, int R, int M0,
                                const int64_t* ia_d, int64_t n, int64_t L, int periodic,
                                double* out_d, int64_t ld_out, void* stream) {
    if (n < 2 || L < 1 || R < 1 || M0 < 1)
        return ls::fail(LS_EVALIDATION, "assemble_axis: need n >= 2, L >= 1, R >= 1, M0 >= 1");
    const int64_t out_len = periodic ? n : L * n;
    if (ld_master < 2 * L * n || ld_out < out_len)
        return ls::fail(LS_EVALIDATION, "assemble_axis: leading dimension too small");
    const int64_t cols = (int64_t)M0 * R;
    if (cols > 65535) return ls::fail(LS_EGUARD, "assemble_axis: more than 65535 columns");
    const int64_t blocks = std::min<int64_t>(ls::ceil_div(out_len, kAsmThreads), 2048);
    LS_CUDA(ls::launch_pdl(assemble_axis_kernel, dim3((unsigned)blocks, (unsigned)cols), dim3(kAsmThreads), 0,
                           ls::as_stream(stream), master_d, ld_master, R, ia_d, n, L, periodic, out_len, out_d,
                           ld_out));
    LS_LAUNCHED("assemble_axis_kernel");
    return LS_OK;
}
