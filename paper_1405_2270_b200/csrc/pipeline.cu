// pipeline.cu -- the device-resident lattice-potential pipeline as a native object
// (ls_pipeline_*): generator -> assembled sum -> expansion -> functional, every
// intermediate in HBM, launched on a caller stream. This is the runtime both the
// C++ RAII wrapper (include/latsum/device.hpp) and the Python DevicePipeline use.
//
// Reference path it runs (proj/include/latsum/): build_lattice_master
// (lattice.hpp:109-113) or the erf generator (newton.hpp:21-37), assembled_box_sum /
// assembled_periodic_sum (lattice.hpp:276-312), densify_slab over a z range
// (canonical.hpp:241-246), and the <V, rho> functional.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

struct ls_pipeline {
    int device = 0;
    int mode = LS_GEN_ERF;
    int periodic = 0;
    int64_t L[3] = {1, 1, 1};
    int64_t n = 0;
    double h = 0.0;
    int R = 0, M0 = 0, Rt = 0;
    int64_t dims[3] = {0, 0, 0};
    int axis_src[3] = {0, 1, 2};  // axes with equal L and charge indices share buffers
    double* tau = nullptr;        // [R]
    double* w = nullptr;          // [M0 * R]  Z_nu * w_q
    int64_t* ia = nullptr;        // [3][M0]
    double* master[3] = {nullptr, nullptr, nullptr};
    double* fac[3] = {nullptr, nullptr, nullptr};
    double* partial = nullptr;
    int64_t partial_cap = 0;
    bool master_valid = false;  // the fused periodic prepare leaves the master unwritten
};

namespace {

void release(ls_pipeline* p) {
    if (!p) return;
    cudaFree(p->tau);
    cudaFree(p->w);
    cudaFree(p->ia);
    for (int l = 0; l < 3; ++l) {
        if (p->axis_src[l] == l) {
            cudaFree(p->master[l]);
            cudaFree(p->fac[l]);
        }
    }
    cudaFree(p->partial);
    delete p;
}

}  // namespace

extern "C" {

int ls_pipeline_create(int mode, const int64_t L[3], int64_t n, double b, const double* tau_h, const double* w_h,
                       int R, const double* charges_h, int M0, int periodic, ls_pipeline** out) {
    *out = nullptr;
    if (mode != LS_GEN_MIDPOINT && mode != LS_GEN_ERF) return ls::fail(LS_EVALIDATION, "pipeline: unknown mode");
    std::vector<int64_t> ia(static_cast<size_t>(3 * std::max(M0, 0)));
    if (const int rc = ls_validate_lattice(L, n, b, charges_h, M0, ia.data())) return rc;
    if (R < 1) return ls::fail(LS_EVALIDATION, "lattice: master tensor has rank 0");
    for (int q = 0; q < R; ++q)
        if (!(tau_h[q] >= 0.0) || !std::isfinite(tau_h[q]))
            return ls::fail(LS_EVALIDATION, "generator: exponents must be finite and >= 0");
    std::vector<double> wt(static_cast<size_t>(M0) * R);
    for (int nu = 0; nu < M0; ++nu)
        for (int q = 0; q < R; ++q)
            wt[static_cast<size_t>(nu) * R + q] = charges_h[4 * nu + 3] * w_h[q];  // lattice.hpp:284-287
    int device = 0;
    LS_CUDA(cudaGetDevice(&device));
    ls_pipeline* p = new ls_pipeline;
    p->device = device;
    p->mode = mode;
    p->periodic = periodic ? 1 : 0;
    p->n = n;
    p->h = b / static_cast<double>(n);
    p->R = R;
    p->M0 = M0;
    p->Rt = M0 * R;
    for (int l = 0; l < 3; ++l) {
        p->L[l] = L[l];
        p->dims[l] = periodic ? n : L[l] * n;
        p->axis_src[l] = l;
        for (int m = 0; m < l; ++m)
            if (L[m] == L[l] && std::equal(ia.begin() + m * M0, ia.begin() + (m + 1) * M0, ia.begin() + l * M0)) {
                p->axis_src[l] = m;
                break;
            }
    }
    auto fail_cleanup = [&](cudaError_t e, const char* what) {
        release(p);
        return ls::cuda_fail(e, what);
    };
    cudaError_t e;
    if ((e = cudaMalloc(&p->tau, sizeof(double) * R)) != cudaSuccess) return fail_cleanup(e, "cudaMalloc tau");
    if ((e = cudaMalloc(&p->w, sizeof(double) * wt.size())) != cudaSuccess) return fail_cleanup(e, "cudaMalloc w");
    if ((e = cudaMalloc(&p->ia, sizeof(int64_t) * ia.size())) != cudaSuccess) return fail_cleanup(e, "cudaMalloc ia");
    if ((e = cudaMemcpy(p->tau, tau_h, sizeof(double) * R, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(p->w, wt.data(), sizeof(double) * wt.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(p->ia, ia.data(), sizeof(int64_t) * ia.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail_cleanup(e, "cudaMemcpy pipeline inputs");
    for (int l = 0; l < 3; ++l) {
        if (p->axis_src[l] != l) {
            p->master[l] = p->master[p->axis_src[l]];
            p->fac[l] = p->fac[p->axis_src[l]];
            continue;
        }
        if ((e = cudaMalloc(&p->master[l], sizeof(double) * 2 * L[l] * n * R)) != cudaSuccess)
            return fail_cleanup(e, "cudaMalloc master");
        if ((e = cudaMalloc(&p->fac[l], sizeof(double) * p->dims[l] * p->Rt)) != cudaSuccess)
            return fail_cleanup(e, "cudaMalloc factor");
    }
    *out = p;
    return LS_OK;
}

int ls_pipeline_destroy(ls_pipeline* p) {
    if (!p) return LS_OK;
    ls::DeviceGuard dg(p->device);
    release(p);
    return LS_OK;
}

int ls_pipeline_info(const ls_pipeline* p, int64_t dims[3], int* rank_total, const double** A_d, const double** B_d,
                     const double** C_d, const double** w_d) {
    if (!p) return ls::fail(LS_EVALIDATION, "pipeline: null handle");
    for (int l = 0; l < 3; ++l)
        if (dims) dims[l] = p->dims[l];
    if (rank_total) *rank_total = p->Rt;
    if (A_d) *A_d = p->fac[0];
    if (B_d) *B_d = p->fac[1];
    if (C_d) *C_d = p->fac[2];
    if (w_d) *w_d = p->w;
    return LS_OK;
}

#define LS_PIPELINE_ENTRY(p)                                                 \
    if (!(p)) return ls::fail(LS_EVALIDATION, "pipeline: null handle");    \
    ls::DeviceGuard device_guard_((p)->device)

int ls_pipeline_generate(ls_pipeline* p, void* stream) {
    LS_PIPELINE_ENTRY(p);
    for (int l = 0; l < 3; ++l) {
        if (p->axis_src[l] != l) continue;
        const int64_t len = 2 * p->L[l] * p->n;
        const int rc = ls_gen_master(p->mode, p->tau, p->R, len, p->h, p->master[l], len, stream);
        if (rc) return rc;
    }
    p->master_valid = true;
    return LS_OK;
}

int ls_pipeline_assemble(ls_pipeline* p, void* stream) {
    LS_PIPELINE_ENTRY(p);
    if (!p->master_valid) {  // no generate() since creation or a fused prepare: build the master first
        if (const int rc = ls_pipeline_generate(p, stream)) return rc;
    }
    for (int l = 0; l < 3; ++l) {
        if (p->axis_src[l] != l) continue;
        const int rc = ls_assemble_axis(p->master[l], 2 * p->L[l] * p->n, p->R, p->M0, p->ia + l * p->M0, p->n, p->L[l],
                                        p->periodic, p->fac[l], p->dims[l], stream);
        if (rc) return rc;
    }
    return LS_OK;
}

int ls_pipeline_prepare(ls_pipeline* p, void* stream) {
    LS_PIPELINE_ENTRY(p);
    ls::GenAsmAxis ax[3];
    int n_ax = 0;
    for (int l = 0; l < 3; ++l)
        if (p->axis_src[l] == l) ax[n_ax++] = {p->L[l], p->ia + l * p->M0, p->master[l], p->fac[l]};
    bool written = true;
    const int rc =
        ls::gen_assemble(p->mode, p->tau, p->R, p->M0, p->n, p->h, p->periodic, ax, n_ax, ls::as_stream(stream), &written);
    if (rc == LS_OK) p->master_valid = written;
    return rc;
}

int ls_pipeline_expand(ls_pipeline* p, int64_t k0, int64_t k1, double* out_d, void* stream) {
    LS_PIPELINE_ENTRY(p);
    return ls_expand(p->fac[0], p->dims[0], p->fac[1], p->dims[1], p->fac[2], p->dims[2], p->w, p->dims[0], p->dims[1],
                     p->dims[2], p->Rt, k0, k1, out_d, 0, 0, nullptr, nullptr, nullptr, nullptr, stream);
}

int ls_pipeline_step(ls_pipeline* p, int64_t k0, int64_t k1, double* out_d, void* stream) {
    LS_PIPELINE_ENTRY(p);
    int rc = ls_pipeline_prepare(p, stream);
    if (!rc) rc = ls_pipeline_expand(p, k0, k1, out_d, stream);
    return rc;
}

int ls_pipeline_energy(ls_pipeline* p, const double* r1_d, const double* r2_d, const double* r3_d, int64_t k0,
                       int64_t k1, double* out_d, void* stream) {
    LS_PIPELINE_ENTRY(p);
    const int64_t np = ls_expand_partial_count(p->dims[0], p->dims[1], p->Rt, k0, k1);
    if (np < 0) return ls::fail(LS_EGUARD, "energy: no tile plan for this rank");
    if (np > p->partial_cap) {
        LS_SYNC(ls::as_stream(stream));
        cudaFree(p->partial);
        p->partial = nullptr;
        LS_CUDA(cudaMalloc(&p->partial, sizeof(double) * std::max<int64_t>(np, 1)));
        p->partial_cap = np;
    }
    int rc = ls_expand(p->fac[0], p->dims[0], p->fac[1], p->dims[1], p->fac[2], p->dims[2], p->w, p->dims[0],
                       p->dims[1], p->dims[2], p->Rt, k0, k1, nullptr, 0, 0, r1_d, r2_d, r3_d, p->partial, stream);
    if (!rc) rc = ls_sum_partials(p->partial, np, out_d, stream);
    return rc;
}

int ls_device_malloc(size_t bytes, void** out_d) {
    *out_d = nullptr;
    LS_CUDA(cudaMalloc(out_d, bytes ? bytes : 16));
    return LS_OK;
}

int ls_device_free(void* p_d) {
    LS_CUDA(cudaFree(p_d));
    return LS_OK;
}

int ls_memcpy(void* dst, const void* src, size_t bytes, void* stream) {
    LS_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ls::as_stream(stream)));
    LS_SYNC(ls::as_stream(stream));
    return LS_OK;
}

int ls_synchronize(void* stream) {
    LS_SYNC(ls::as_stream(stream));
    return LS_OK;
}

}  // extern "C"
