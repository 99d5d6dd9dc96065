// latsum/sharded.hpp -- additive C++ API (no reference counterpart): the lattice potential
// sharded over GPUs, one process per GPU.
//
// The reference parallelises densify over z-slabs with threads (canonical.hpp:251-266,
// parallel_for over k into disjoint slabs). Here the same split runs across GPUs: rank r of
// `world` owns the contiguous slab range slab_range(N3, r, world), recomputes the generator
// and assembly on its own GPU (microseconds; nothing is sent), and expands only its slabs.
// The one collective is the all-reduce of functional partial sums (NCCL, through the C ABI's
// ls_comm_*), so energies and functional batches come out identical on every rank.
//
//   latsum::Communicator comm = latsum::Communicator::from_id_file(world, rank, "/tmp/job.id");
//   latsum::ShardedPotential pot(spec, rule, comm);          // on this process's device
//   pot.step(out_d, stream);                                 // this rank's slabs into HBM
//   double e = pot.energy(r1_d, r2_d, r3_d, scratch_d, stream);  // whole-grid <V, rho>
#pragma once

#include <array>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>
#include <thread>
#include <utility>

#include "latsum/device.hpp"
#include "latsum/errors.hpp"
#include "latsum_cuda.h"

namespace latsum {

using CommId = std::array<unsigned char, LS_COMM_ID_BYTES>;

class Communicator {
public:
    // A fresh id; rank 0 makes it and the caller hands it to every rank.
    static CommId unique_id() {
        CommId id{};
        cuda::check(ls_comm_unique_id(id.data(), static_cast<int>(id.size())), "Communicator::unique_id");
        return id;
    }

    // Joins the group on the current CUDA device (collective over all ranks).
    Communicator(int world, int rank, const CommId& id) {
        cuda::check(ls_comm_init(world, rank, id.data(), static_cast<int>(id.size()), &c_), "Communicator");
        world_ = world;
        rank_ = rank;
    }

    // Rendezvous through a shared file: rank 0 writes a fresh id to `path` (atomically, via a
    // temporary and a rename), the other ranks wait up to `timeout_s` for it to appear. The
    // path must be new for every job (a stale file from an earlier job would be read).
    static Communicator from_id_file(int world, int rank, const std::string& path, double timeout_s = 120.0) {
        CommId id{};
        if (rank == 0) {
            id = unique_id();
            const std::string tmp = path + ".tmp";
            {
                std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
                f.write(reinterpret_cast<const char*>(id.data()), static_cast<std::streamsize>(id.size()));
                if (!f) throw validation_error("Communicator: cannot write " + tmp);
            }
            if (std::rename(tmp.c_str(), path.c_str()) != 0)
                throw validation_error("Communicator: cannot rename " + tmp + " to " + path);
        } else {
            const auto t0 = std::chrono::steady_clock::now();
            for (;;) {
                std::ifstream f(path, std::ios::binary);
                if (f && f.read(reinterpret_cast<char*>(id.data()), static_cast<std::streamsize>(id.size()))) break;
                if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
                    throw validation_error("Communicator: no id at " + path + " after " + std::to_string(timeout_s) + " s");
                std::this_thread::sleep_for(std::chrono::milliseconds(20));
            }
        }
        return Communicator(world, rank, id);
    }

    Communicator(const Communicator&) = delete;
    Communicator& operator=(const Communicator&) = delete;
    Communicator(Communicator&& o) noexcept : c_(o.c_), world_(o.world_), rank_(o.rank_) { o.c_ = nullptr; }
    ~Communicator() {
        if (c_) ls_comm_destroy(c_);
    }

    int world() const { return world_; }
    int rank() const { return rank_; }
    ls_comm* handle() const { return c_; }

    // In-place all-reduce of n doubles in device memory, stream-ordered.
    void allreduce_sum(double* buf_d, std::int64_t n, void* stream = nullptr) {
        cuda::check(ls_comm_allreduce_f64(c_, buf_d, n, LS_REDUCE_SUM, stream), "allreduce_sum");
    }
    void allreduce_max(double* buf_d, std::int64_t n, void* stream = nullptr) {
        cuda::check(ls_comm_allreduce_f64(c_, buf_d, n, LS_REDUCE_MAX, stream), "allreduce_max");
    }

private:
    ls_comm* c_ = nullptr;
    int world_ = 1;
    int rank_ = 0;
};

class ShardedPotential {
public:
    ShardedPotential(const LatticeSpec& spec, const QuadratureRule& rule, Communicator& comm,
                     Generator gen = Generator::erf, bool periodic = false)
        : pot_(spec, rule, gen, periodic), comm_(comm) {
        const auto r = slab_range(pot_.dims()[2], comm.rank(), comm.world());
        k0_ = r.first;
        k1_ = r.second;
    }

    Dims3 dims() const { return pot_.dims(); }
    Index first_slab() const { return k0_; }
    Index end_slab() const { return k1_; }
    // Doubles this rank's slabs occupy: (k1 - k0) * N1 * N2.
    std::size_t shard_size() const {
        return static_cast<std::size_t>((k1_ - k0_) * pot_.dims()[0] * pot_.dims()[1]);
    }
    DevicePotential& potential() { return pot_; }
    Communicator& communicator() { return comm_; }

    // One pass of the hot path over this rank's slabs: generate, assemble, expand into out_d.
    void step(double* out_d, void* stream = nullptr) { pot_.step(k0_, k1_, out_d, stream); }

    // Whole-grid <V, rho> for rho = r1 (x) r2 (x) r3 (device vectors of the full axis lengths):
    // the fused expansion-reduction over this rank's slabs, then the sum over ranks into
    // out_d[0] on every rank (stream-ordered, no host round trip).
    void energy_async(const double* r1_d, const double* r2_d, const double* r3_d, double* out_d, void* stream = nullptr) {
        cuda::check(ls_pipeline_energy_allreduce(pot_.handle(), r1_d, r2_d, r3_d, k0_, k1_, out_d, comm_.handle(),
                                                 stream),
                    "ShardedPotential::energy");
    }
    // Same, returned to the host (synchronises `stream`); scratch_d holds one double.
    double energy(const double* r1_d, const double* r2_d, const double* r3_d, double* scratch_d,
                  void* stream = nullptr) {
        energy_async(r1_d, r2_d, r3_d, scratch_d, stream);
        double e = 0.0;
        cuda::check(ls_memcpy(&e, scratch_d, sizeof(double), stream), "ShardedPotential::energy");
        return e;
    }

private:
    DevicePotential pot_;
    Communicator& comm_;
    Index k0_ = 0, k1_ = 0;
};

}  // namespace latsum
