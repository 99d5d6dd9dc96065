// assemble.cu -- K2: the assembled O(N L R) lattice summation.
//
// Reference: detail::assembled_axis_columns (lattice.hpp:220-274). Column
// c = (nu, q) of the per-axis factor is the sum over the L lattice shifts of
// the windowed master column, added strictly left to right in ascending k
// (the reference's eight-stream blocks keep that order, lattice.hpp:240-271).
// Every output keeps exactly that recurrence in one thread, so the result is
// bit-identical to the reference; the adds of one output form a dependent
// chain that cannot be reassociated.
//
//  * assemble_box_kernel: box sums, out[o] = sum_k m[s0 + o - k n] with
//    o = i + j n. Outputs j and j + 1 of the same residue i read the same
//    master entries one shift apart, so a thread owns eight consecutive j of
//    one i: eight independent chains fed by a sliding register window, one new
//    load per shift instead of eight (cfg3: 8 charges x 41 ranks x 2048
//    outputs x 32 shifts per axis).
//  * assemble_axis_kernel: periodic sums (out_len = n, one chain per residue,
//    no reuse): each element is read once, so the loads stream from L2/HBM
//    with three groups of eight in flight ahead of the adds.
#include "common.cuh"

namespace {

constexpr int kAsmThreads = 256;
constexpr int kJ = 8;  // outputs (consecutive j) per thread in the box kernel
constexpr int kPGroups = 4;  // groups of 8 loads per chain in the periodic kernel's register ring

using ls::window_start;  // lattice.hpp:98 / :104-106 at k = 0 (common.cuh)

__global__ void assemble_box_kernel(const double* __restrict__ master, int64_t ld_master, int R,
                                    const int64_t* __restrict__ ia, int64_t n, int64_t L,
                                    double* __restrict__ out, int64_t ld_out) {
    pdl_wait();  // the master comes from the preceding generator launch
    pdl_trigger();
    const int c = blockIdx.y;  // column nu*R + q
    const int nu = c / R;
    const int q = c % R;
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t n_jb = (L + kJ - 1) / kJ;
    if (x >= n_jb * n) return;
    const int64_t i = x % n;  // consecutive threads: consecutive i, coalesced loads and stores
    const int64_t j0 = (x / n) * kJ;
    // value d (d = j - k) is m[b + d n]; d >= -(L-1) always, d > L-1 only for padded chains
    const double* col = master + ld_master * q + window_start(0, L * n, L, n, ia[nu]) + i;
    double win[kJ], acc[kJ], cur[kJ], nxt[kJ];
    // shift k = 0: the window holds d = j0 .. j0 + 7 (slot d - j0) and starts every chain;
    // d > L - 1 only in the last block's padded chains (zero, never stored)
#pragma unroll
    for (int e = 0; e < kJ; ++e) acc[e] = win[e] = j0 + e <= L - 1 ? __ldg(col + (j0 + e) * n) : 0.0;
    // shift k brings in d = j0 - k (always <= L - 1) into slot (-k) mod 8; chain jj reads slot
    // (jj - k) mod 8. pk points at the entry of shift k0; loads past the last shift are
    // redirected to pk (a valid address) and never used.
    const double* pk = col + (j0 - 1) * n;
#pragma unroll
    for (int s = 0; s < kJ; ++s) cur[s] = __ldg(1 + s < L ? pk - s * n : pk);
    int64_t k0 = 1;  // k0 = 1 mod 8, so every slot index is static
    for (; k0 + kJ <= L; k0 += kJ, pk -= kJ * n) {
#pragma unroll
        for (int s = 0; s < kJ; ++s) nxt[s] = __ldg(k0 + kJ + s < L ? pk - (kJ + s) * n : pk);
#pragma unroll
        for (int s = 0; s < kJ; ++s) {
            win[(kJ - 1 - s) & (kJ - 1)] = cur[s];
#pragma unroll
            for (int jj = 0; jj < kJ; ++jj) acc[jj] = rn_add(acc[jj], win[(jj - 1 - s) & (kJ - 1)]);
        }
#pragma unroll
        for (int s = 0; s < kJ; ++s) cur[s] = nxt[s];
    }
#pragma unroll
    for (int s = 0; s < kJ; ++s) {  // the last, partial block of shifts
        if (k0 + s < L) {
            win[(kJ - 1 - s) & (kJ - 1)] = cur[s];
#pragma unroll
            for (int jj = 0; jj < kJ; ++jj) acc[jj] = rn_add(acc[jj], win[(jj - 1 - s) & (kJ - 1)]);
        }
    }
    double* o = out + ld_out * c + i + j0 * n;
#pragma unroll
    for (int jj = 0; jj < kJ; ++jj)
        if (j0 + jj < L) o[jj * n] = acc[jj];
}

__global__ void assemble_axis_kernel(const double* __restrict__ master, int64_t ld_master, int R,
                                     const int64_t* __restrict__ ia, int64_t n, int64_t L,
                                     int periodic, int64_t out_len, double* __restrict__ out,
                                     int64_t ld_out) {
    pdl_wait();  // the master comes from the preceding generator launch
    pdl_trigger();
    const int c = blockIdx.y;  // column nu*R + q
    const int nu = c / R;
    const int q = c % R;
    const double* base = master + ld_master * q + window_start(periodic, L * n, L, n, ia[nu]);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < out_len;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double* p = base + i;
        double acc = p[0];
        // Groups of 8 shifts; kPGroups - 1 groups of loads stay in flight ahead of the adds,
        // which keep ascending-k order. Loads past the last shift are redirected to p.
        double buf[kPGroups][8];
        const int64_t n_full = (L - 1) / 8;  // full groups of shifts 1 + 8g .. 8 + 8g
#pragma unroll
        for (int g = 0; g < kPGroups - 1; ++g)
#pragma unroll
            for (int u = 0; u < 8; ++u) buf[g][u] = __ldg(g < n_full ? p - (1 + 8 * g + u) * n : p);
        int64_t g0 = 0;
        for (; g0 + kPGroups <= n_full; g0 += kPGroups) {
#pragma unroll
            for (int gg = 0; gg < kPGroups; ++gg) {
                const int64_t gl = g0 + gg + kPGroups - 1;  // group to load into the slot freed last
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    buf[(gg + kPGroups - 1) % kPGroups][u] = __ldg(gl < n_full ? p - (1 + 8 * gl + u) * n : p);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = rn_add(acc, buf[gg][u]);
            }
        }
#pragma unroll
        for (int gg = 0; gg < kPGroups; ++gg) {  // the remaining (< kPGroups) full groups
            if (g0 + gg < n_full) {
                const int64_t gl = g0 + gg + kPGroups - 1;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    buf[(gg + kPGroups - 1) % kPGroups][u] = __ldg(gl < n_full ? p - (1 + 8 * gl + u) * n : p);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = rn_add(acc, buf[gg][u]);
            }
        }
        for (int64_t k = 1 + 8 * n_full; k < L; ++k) acc = rn_add(acc, __ldg(p - k * n));
        out[i + ld_out * c] = acc;
    }
}

// Periodic sums with long chains (cfg4: n = 256 residues x 41 columns, L = 64..256 shifts): the
// per-chain kernel above keeps only 24 loads in flight per chain, and with 10.5K chains on 148
// SMs it waits on L2 latency for every group (8 us at L = 256). Here a block stages the L x 32
// master values of 32 consecutive residues of one column in shared memory with all its threads
// (row k = 32 contiguous doubles, coalesced, all loads in flight at once), then one warp runs
// the 32 chains out of shared memory, still strictly ascending in k: bit-identical sums.
constexpr int kPerIB = 32;
__global__ void __launch_bounds__(256) assemble_periodic_staged_kernel(const double* __restrict__ master,
                                                                      int64_t ld_master, int R,
                                                                      const int64_t* __restrict__ ia, int64_t n,
                                                                      int64_t L, double* __restrict__ out,
                                                                      int64_t ld_out) {
    pdl_wait();  // the master comes from the preceding generator launch
    pdl_trigger();
    extern __shared__ double stage[];  // [L][kPerIB]
    const int c = blockIdx.y;          // column nu*R + q
    const int nu = c / R;
    const int q = c % R;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kPerIB;
    const double* base = master + ld_master * q + window_start(1, L * n, L, n, ia[nu]) + i0;
    const int64_t cnt = L * kPerIB;
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) {
        const int64_t k = e / kPerIB;
        const int ii = static_cast<int>(e - k * kPerIB);
        stage[e] = i0 + ii < n ? __ldg(base + ii - k * n) : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < kPerIB && i0 + threadIdx.x < n) {
        const double* col = stage + threadIdx.x;
        double acc = col[0];
#pragma unroll 8
        for (int64_t k = 1; k < L; ++k) acc = rn_add(acc, col[k * kPerIB]);
        out[i0 + threadIdx.x + ld_out * c] = acc;
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
    const cudaStream_t s = ls::as_stream(stream);
    if (!periodic && L > 1) {
        const int64_t threads = ls::ceil_div(L, kJ) * n;
        const int64_t blocks = ls::ceil_div(threads, kAsmThreads);
        if (blocks > 0x7fffffff) return ls::fail(LS_EGUARD, "assemble_axis: too many output blocks");
        LS_CUDA(ls::launch_pdl(assemble_box_kernel, dim3((unsigned)blocks, (unsigned)cols), dim3(kAsmThreads), 0, s,
                               master_d, ld_master, R, ia_d, n, L, out_d, ld_out));
        LS_LAUNCHED("assemble_box_kernel");
        return LS_OK;
    }
    // periodic, long chains: stage each 32-residue block's L x 32 master values in shared memory
    const size_t staged = sizeof(double) * static_cast<size_t>(L) * kPerIB;
    if (periodic && L >= 32 && staged <= 96 * 1024) {
        static std::atomic<bool> attr_set[64] = {};
        int dev = 0;
        LS_CUDA(cudaGetDevice(&dev));
        if (dev >= 64 || !attr_set[dev]) {
            LS_CUDA(cudaFuncSetAttribute(assemble_periodic_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         96 * 1024));
            if (dev < 64) attr_set[dev] = true;
        }
        LS_CUDA(ls::launch_pdl(assemble_periodic_staged_kernel, dim3((unsigned)ls::ceil_div(out_len, kPerIB), (unsigned)cols),
                               dim3(256), staged, s, master_d, ld_master, R, ia_d, n, L, out_d, ld_out));
        LS_LAUNCHED("assemble_periodic_staged_kernel");
        return LS_OK;
    }
    // periodic: 64-thread blocks spread the few, long chains (n per column) over the SMs
    const int64_t blocks = std::min<int64_t>(ls::ceil_div(out_len, 64), 4096);
    LS_CUDA(ls::launch_pdl(assemble_axis_kernel, dim3((unsigned)blocks, (unsigned)cols), dim3(64), 0, s, master_d,
                           ld_master, R, ia_d, n, L, periodic, out_len, out_d, ld_out));
    LS_LAUNCHED("assemble_axis_kernel");
    return LS_OK;
}
