// latsum/device.hpp -- additive C++ API (no reference counterpart): the lattice
// potential resident in HBM. Wraps the native pipeline object of
// liblatsum_cuda.so (ls_pipeline_*): generator -> assembled sum -> expansion ->
// functional on a caller stream, no host round trips. Use it for grids above
// densify's 2^27-entry guard, for z-slab shards (one process per GPU, see
// slab_range), and to keep the potential on the device for further GPU work.
#pragma once

#include <cstdint>
#include <string>
#include <utility>

#include "latsum/canonical.hpp"
#include "latsum/errors.hpp"
#include "latsum/lattice.hpp"
#include "latsum/quadrature.hpp"
#include "latsum_cuda.h"

namespace latsum {

enum class Generator { midpoint = LS_GEN_MIDPOINT, erf = LS_GEN_ERF };

// Balanced contiguous z-slab range [first, second) of rank `rank` out of `world`.
inline std::pair<Index, Index> slab_range(Index n3, int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) throw validation_error("slab_range: bad rank / world");
    const Index base = n3 / world, extra = n3 % world;
    const Index k0 = rank * base + std::min<Index>(rank, extra);
    return {k0, k0 + base + (rank < extra ? 1 : 0)};
}

class DevicePotential {
public:
    DevicePotential(const LatticeSpec& spec, const QuadratureRule& rule, Generator gen = Generator::erf,
                    bool periodic = false) {
        spec.validate();
        std::vector<double> charges;
        for (const Charge& c : spec.charges) {
            charges.insert(charges.end(), {c.pos[0], c.pos[1], c.pos[2], c.Z});
        }
        const std::int64_t L[3] = {spec.L[0], spec.L[1], spec.L[2]};
        cuda::check(ls_pipeline_create(static_cast<int>(gen), L, spec.unit.n, spec.unit.b, rule.exponents.data(),
                                       rule.weights.data(), static_cast<int>(rule.node_count()), charges.data(),
                                       static_cast<int>(spec.charge_count()), periodic ? 1 : 0, &h_),
                    "DevicePotential");
        std::int64_t d[3];
        int rt = 0;
        cuda::check(ls_pipeline_info(h_, d, &rt, nullptr, nullptr, nullptr, nullptr), "DevicePotential");
        dims_ = {d[0], d[1], d[2]};
        rank_ = rt;
    }
    DevicePotential(const DevicePotential&) = delete;
    DevicePotential& operator=(const DevicePotential&) = delete;
    DevicePotential(DevicePotential&& o) noexcept : h_(o.h_), dims_(o.dims_), rank_(o.rank_) { o.h_ = nullptr; }
    ~DevicePotential() {
        if (h_) ls_pipeline_destroy(h_);
    }

    Dims3 dims() const { return dims_; }
    Index rank() const { return rank_; }
    // The native pipeline object, for C-ABI calls that take it (e.g. ls_pipeline_energy_allreduce).
    ls_pipeline* handle() const { return h_; }

    // Stages on `stream` (a cudaStream_t; nullptr = default stream), asynchronous.
    void generate(void* stream = nullptr) { cuda::check(ls_pipeline_generate(h_, stream), "generate"); }
    void assemble(void* stream = nullptr) { cuda::check(ls_pipeline_assemble(h_, stream), "assemble"); }
    // generate + assemble (one launch on small lattices); what step() runs before the expansion.
    void prepare(void* stream = nullptr) { cuda::check(ls_pipeline_prepare(h_, stream), "prepare"); }
    // Slabs [k0, k1) into device memory out_d ((k1-k0)*N1*N2 doubles, i-fastest).
    void expand(Index k0, Index k1, double* out_d, void* stream = nullptr) {
        cuda::check(ls_pipeline_expand(h_, k0, k1, out_d, stream), "expand");
    }
    void step(Index k0, Index k1, double* out_d, void* stream = nullptr) {
        cuda::check(ls_pipeline_step(h_, k0, k1, out_d, stream), "step");
    }
    // out_d[0] = sum over slabs [k0, k1) of V * r1(i) r2(j) r3(k); all pointers device memory.
    void energy(const double* r1_d, const double* r2_d, const double* r3_d, Index k0, Index k1, double* out_d,
                void* stream = nullptr) {
        cuda::check(ls_pipeline_energy(h_, r1_d, r2_d, r3_d, k0, k1, out_d, stream), "energy");
    }

    // Full-grid functionals of slabs [k0, k1) for F separable densities
    // rho_f = X(:,f) (x) Y(:,f) (x) Z(:,f), X/Y/Z column-major N_l x F in device memory:
    // out_d[f] (+)= sum over the slabs of V * rho_f. The slabs are expanded into scratch_d
    // ((k1-k0)*N1*N2 doubles), then contracted by one fused FP64-DMMA GEMM. Call it per slab
    // chunk with accumulate = true after the first to cover grids larger than the scratch.
    void grid_functionals(const double* X_d, const double* Y_d, const double* Z_d, int F, Index k0, Index k1,
                          double* scratch_d, double* out_d, bool accumulate = false, void* stream = nullptr) {
        if (k0 < 0 || k1 < k0 || k1 > dims_[2]) throw validation_error("grid_functionals: bad slab range");
        expand(k0, k1, scratch_d, stream);
        cuda::check(ls_grid_functional_batch(scratch_d, dims_[0], dims_[1], k1 - k0, dims_[0], dims_[0] * dims_[1],
                                             X_d, dims_[0], Y_d, dims_[1], Z_d + k0, dims_[2], F, 1.0,
                                             accumulate ? 1 : 0, out_d, stream),
                    "grid_functionals");
    }

    // The assembled canonical tensor, copied to the host (after generate + assemble).
    CanonicalTensor3 tensor(void* stream = nullptr) const {
        const double* f[3];
        const double* w = nullptr;
        cuda::check(ls_pipeline_info(h_, nullptr, nullptr, &f[0], &f[1], &f[2], &w), "tensor");
        std::array<Matrix, 3> fac;
        for (int l = 0; l < 3; ++l) {
            fac[l].resize(dims_[l], rank_);
            cuda::check(ls_memcpy(fac[l].data(), f[l], sizeof(double) * static_cast<std::size_t>(fac[l].size()), stream),
                        "tensor");
        }
        Vector wv(rank_);
        cuda::check(ls_memcpy(wv.data(), w, sizeof(double) * static_cast<std::size_t>(rank_), stream), "tensor");
        return CanonicalTensor3(CanonicalTensor3::trusted_components_t{}, std::move(fac), std::move(wv));
    }

private:
    ls_pipeline* h_ = nullptr;
    Dims3 dims_{0, 0, 0};
    Index rank_ = 0;
};

// Which expansion plan the device path uses for a tensor of rank R (kernel, CTA shape, where
// A1k lives, k-steps, DFMA ranks), e.g. for logs next to timings.
inline std::string expansion_plan(Index R) {
    char buf[256];
    cuda::check(ls_expand_plan_name(static_cast<int>(R), buf, static_cast<int>(sizeof(buf))), "expansion_plan");
    return buf;
}

// RAII device buffer for callers without the CUDA headers.
class DeviceBuffer {
public:
    explicit DeviceBuffer(std::size_t count) : n_(count) {
        void* p = nullptr;
        cuda::check(ls_device_malloc(sizeof(double) * count, &p), "DeviceBuffer");
        p_ = static_cast<double*>(p);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    ~DeviceBuffer() { ls_device_free(p_); }
    double* data() { return p_; }
    std::size_t size() const { return n_; }
    void upload(const double* host, std::size_t count) {
        cuda::check(ls_memcpy(p_, host, sizeof(double) * count, nullptr), "upload");
    }
    void download(double* host, std::size_t count) const {
        cuda::check(ls_memcpy(host, p_, sizeof(double) * count, nullptr), "download");
    }

private:
    double* p_ = nullptr;
    std::size_t n_ = 0;
};

}  // namespace latsum
