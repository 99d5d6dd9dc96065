// latsum_shard_runner -- one rank of the z-slab sharded lattice potential, in C++.
//
// Host code of the multi-GPU path (north_star: host code stays C++, NCCL only for the scalar
// all-reduce). Each process owns one GPU and the slab range slab_range(N3, rank, world) of the
// grid; it builds the rule (sinc_quadrature), the device pipeline (generator -> assembled sum
// -> expansion) and the NCCL communicator through the drop-in headers (include/latsum), runs
// warm-up + timed steps over its slabs, the whole-grid energy <V, rho> (fused per-rank
// functional + one all-reduce) and an end-to-end pass through the host-level API, and prints
// one JSON line (rank 0: with every timing taken as the max over ranks).
//
//   latsum_shard_runner --L 32 --n 64 --b 10 --M 20 [--charges cell.csv] [--periodic]
//                       [--world W --rank R --device D] (default: $WORLD_SIZE $RANK $LOCAL_RANK)
//                       [--id-hex HEX | --id-file PATH]
//                       [--steps K] [--warmup W] [--energy] [--e2e-steps E] [--host-threads T]
//
// bench.py drives it under torchrun for --gpus N > 1: rank 0's runner creates the NCCL id and
// writes it to a fresh --id-file path the launcher's gloo group agreed on (the id's bootstrap
// root lives in the process that created it, so rank 0 must be a runner that stays up). With
// --id-hex the caller moved the id of a living rank 0 itself; world = 1 needs neither.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "latsum/bundle.hpp"
#include "latsum/device.hpp"
#include "latsum/lattice.hpp"
#include "latsum/quadrature.hpp"
#include "latsum/sharded.hpp"

namespace {

struct Args {
    std::int64_t L[3] = {32, 32, 32};
    std::int64_t n = 64;
    double b = 10.0;
    int M = 20;
    double eps = 1e-6, C0 = 1.0;
    std::string charges;
    bool periodic = false;
    int world = -1, rank = -1, device = -1;
    std::string id_hex, id_file;
    int steps = 20, warmup = 3, e2e_steps = 0, host_threads = 0;
    bool energy = false;
    bool midpoint = false;
};

[[noreturn]] void usage(const char* msg) {
    std::fprintf(stderr, "latsum_shard_runner: %s\n", msg);
    std::exit(2);
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

Args parse(int argc, char** argv) {
    Args a;
    for (int i = 1; i < argc; ++i) {
        const std::string k = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) usage(("missing value for " + k).c_str());
            return argv[++i];
        };
        if (k == "--L") {
            const std::string v = val();
            if (std::sscanf(v.c_str(), "%ld,%ld,%ld", &a.L[0], &a.L[1], &a.L[2]) != 3) a.L[0] = a.L[1] = a.L[2] = std::atol(v.c_str());
        } else if (k == "--n") a.n = std::atol(val().c_str());
        else if (k == "--b") a.b = std::atof(val().c_str());
        else if (k == "--M") a.M = std::atoi(val().c_str());
        else if (k == "--eps") a.eps = std::atof(val().c_str());
        else if (k == "--charges") a.charges = val();
        else if (k == "--periodic") a.periodic = true;
        else if (k == "--midpoint") a.midpoint = true;
        else if (k == "--world") a.world = std::atoi(val().c_str());
        else if (k == "--rank") a.rank = std::atoi(val().c_str());
        else if (k == "--device") a.device = std::atoi(val().c_str());
        else if (k == "--id-hex") a.id_hex = val();
        else if (k == "--id-file") a.id_file = val();
        else if (k == "--steps") a.steps = std::atoi(val().c_str());
        else if (k == "--warmup") a.warmup = std::atoi(val().c_str());
        else if (k == "--e2e-steps") a.e2e_steps = std::atoi(val().c_str());
        else if (k == "--host-threads") a.host_threads = std::atoi(val().c_str());
        else if (k == "--energy") a.energy = true;
        else usage(("unknown argument " + k).c_str());
    }
    if (a.world < 0) a.world = env_int("WORLD_SIZE", 1);
    if (a.rank < 0) a.rank = env_int("RANK", 0);
    if (a.device < 0) a.device = env_int("LOCAL_RANK", a.rank);
    if (a.steps < 1 || a.warmup < 0) usage("need --steps >= 1 and --warmup >= 0");
    return a;
}

latsum::CommId from_hex(const std::string& s) {
    latsum::CommId id{};
    if (s.size() != 2 * id.size()) usage("--id-hex needs 2 * LS_COMM_ID_BYTES hex digits");
    for (std::size_t i = 0; i < id.size(); ++i) id[i] = static_cast<unsigned char>(std::stoi(s.substr(2 * i, 2), nullptr, 16));
    return id;
}

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess) {                                                                   \
            std::fprintf(stderr, "latsum_shard_runner: %s: %s\n", #x, cudaGetErrorString(e_));     \
            std::exit(5);                                                                          \
        }                                                                                          \
    } while (0)

struct Timer {
    cudaEvent_t a, b;
    Timer() {
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
    }
    ~Timer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    float ms() const {
        float t = 0;
        CK(cudaEventElapsedTime(&t, a, b));
        return t;
    }
};

std::vector<double> density(std::int64_t N, double h, double sigma) {
    std::vector<double> r(static_cast<std::size_t>(N));
    for (std::int64_t i = 0; i < N; ++i) {
        const double x = (static_cast<double>(i) + 0.5 - static_cast<double>(N) / 2.0) * h;
        r[static_cast<std::size_t>(i)] = std::exp(-x * x / (2.0 * sigma * sigma));
    }
    return r;
}

double wall_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

int main(int argc, char** argv) try {
    const Args a = parse(argc, argv);
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    const int dev = a.device % std::max(ndev, 1);
    CK(cudaSetDevice(dev));
    latsum::cuda::check(ls_set_device(dev), "set_device");
    if (a.host_threads > 0) latsum::cuda::check(ls_set_host_threads(a.host_threads), "set_host_threads");

    // The lattice: a unit charge at each cell centre, or the cell's charges from a CSV
    // (read_charges_csv, the reference's format, bundle.hpp).
    latsum::LatticeSpec spec;
    spec.L = {a.L[0], a.L[1], a.L[2]};
    spec.unit = latsum::GridSpec(a.b, a.n);
    if (a.charges.empty()) spec.charges = {latsum::Charge{{0.0, 0.0, 0.0}, 1.0}};
    else spec.charges = latsum::read_charges_csv(a.charges);
    spec.validate();
    const std::int64_t Lmax = std::max({a.L[0], a.L[1], a.L[2]});
    const latsum::QuadratureRule rule =
        latsum::sinc_quadrature(a.eps, spec.unit.h(), std::sqrt(3.0) * static_cast<double>(Lmax) * a.b, a.M, a.C0);
    const auto gen = a.midpoint ? latsum::Generator::midpoint : latsum::Generator::erf;

    const double t_comm0 = wall_s();
    latsum::CommId id{};
    if (!a.id_hex.empty()) id = from_hex(a.id_hex);
    std::unique_ptr<latsum::Communicator> comm;
    if (!a.id_file.empty()) {
        comm.reset(new latsum::Communicator(latsum::Communicator::from_id_file(a.world, a.rank, a.id_file)));
    } else {
        if (a.id_hex.empty()) {
            if (a.world != 1) usage("world > 1 needs --id-hex or --id-file");
            id = latsum::Communicator::unique_id();
        }
        comm.reset(new latsum::Communicator(a.world, a.rank, id));
    }
    const double comm_init_s = wall_s() - t_comm0;

    latsum::ShardedPotential pot(spec, rule, *comm, gen, a.periodic);
    const latsum::Dims3 N = pot.dims();
    const std::int64_t k0 = pot.first_slab(), k1 = pot.end_slab();
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    double* out = nullptr;
    CK(cudaMalloc(&out, std::max<std::size_t>(pot.shard_size(), 1) * sizeof(double)));
    double* scal = nullptr;
    CK(cudaMalloc(&scal, 4 * sizeof(double)));
    auto barrier = [&] {  // a one-double all-reduce, then the host waits for it
        comm->allreduce_sum(scal + 3, 1, s);
        CK(cudaStreamSynchronize(s));
    };

    // Warm-up, then the timed region: K steps between events, the expansion of each step
    // bracketed by its own events (the roofline kernel).
    for (int i = 0; i < a.warmup; ++i) pot.step(out, s);
    CK(cudaStreamSynchronize(s));
    std::vector<Timer> ev(static_cast<std::size_t>(a.steps));
    Timer total;
    const std::int64_t launches0 = ls_launch_count();
    barrier();
    CK(cudaEventRecord(total.a, s));
    latsum::DevicePotential& dp = pot.potential();
    for (int i = 0; i < a.steps; ++i) {
        dp.prepare(s);
        CK(cudaEventRecord(ev[static_cast<std::size_t>(i)].a, s));
        dp.expand(k0, k1, out, s);
        CK(cudaEventRecord(ev[static_cast<std::size_t>(i)].b, s));
    }
    CK(cudaEventRecord(total.b, s));
    CK(cudaStreamSynchronize(s));
    const std::int64_t launches = ls_launch_count() - launches0;
    double exp_mean = 0.0;
    for (const Timer& t : ev) exp_mean += t.ms();
    exp_mean /= a.steps;
    // max over ranks of {total ms, mean expansion ms}
    double loc[2] = {total.ms(), exp_mean};
    CK(cudaMemcpy(scal, loc, sizeof(loc), cudaMemcpyHostToDevice));
    comm->allreduce_max(scal, 2, s);
    double mx[2];
    CK(cudaMemcpyAsync(mx, scal, sizeof(mx), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double ms_step = mx[0] / a.steps;
    const double pts_total = static_cast<double>(N[0]) * N[1] * N[2];
    const double pts_rank = static_cast<double>(N[0]) * N[1] * static_cast<double>(k1 - k0);

    std::string energy_json = "null";
    if (a.energy) {
        const double sigma = static_cast<double>(Lmax) * a.b / 4.0;  // rho >= e^-2 of its peak on every face
        double* rho[3];
        for (int l = 0; l < 3; ++l) {
            const std::vector<double> r = density(N[l], spec.unit.h(), sigma);
            CK(cudaMalloc(&rho[l], r.size() * sizeof(double)));
            CK(cudaMemcpy(rho[l], r.data(), r.size() * sizeof(double), cudaMemcpyHostToDevice));
        }
        pot.energy(rho[0], rho[1], rho[2], scal, s);  // warm-up
        Timer fused, red;
        barrier();
        CK(cudaEventRecord(fused.a, s));
        dp.energy(rho[0], rho[1], rho[2], k0, k1, scal, s);
        CK(cudaEventRecord(fused.b, s));
        CK(cudaEventRecord(red.a, s));
        comm->allreduce_sum(scal, 1, s);
        CK(cudaEventRecord(red.b, s));
        double e = 0.0;
        CK(cudaMemcpyAsync(&e, scal, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const double t0 = wall_s();
        const double e_api = pot.energy(rho[0], rho[1], rho[2], scal, s);
        const double api_ms = (wall_s() - t0) * 1e3;
        // 1D rank-term form on the device (scalar_product, canonical.hpp:126-136) as the check
        const double* f[3];
        const double* w = nullptr;
        int rt = 0;
        latsum::cuda::check(ls_pipeline_info(dp.handle(), nullptr, &rt, &f[0], &f[1], &f[2], &w), "info");
        latsum::cuda::check(ls_functional_batch(f[0], N[0], f[1], N[1], f[2], N[2], w, rt, N[0], N[1], N[2], rho[0],
                                                N[0], rho[1], N[1], rho[2], N[2], 1, 1.0, scal + 1, s),
                            "functional_batch");
        double e1d = 0.0;
        CK(cudaMemcpyAsync(&e1d, scal + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double tl[3] = {fused.ms(), red.ms(), api_ms};
        CK(cudaMemcpy(scal, tl, sizeof(tl), cudaMemcpyHostToDevice));
        comm->allreduce_max(scal, 3, s);
        double tm[3];
        CK(cudaMemcpyAsync(tm, scal, sizeof(tm), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (double* r : rho) cudaFree(r);
        char buf[1024];
        std::snprintf(buf, sizeof(buf),
                      "{\"value\": %.17g, \"api_value\": %.17g, \"one_d_value\": %.17g, \"rel_diff_vs_1d\": %.3e, "
                      "\"fused_ms_max\": %.4f, \"allreduce_ms_max\": %.4f, \"api_wall_ms_max\": %.3f, "
                      "\"sigma_bohr\": %.6g, \"path\": \"fused expansion-reduction over own z-slabs + ncclAllReduce "
                      "(ls_pipeline_energy_allreduce)\"}",
                      e, e_api, e1d, std::abs(e - e1d) / std::abs(e1d), tm[0], tm[1], tm[2], sigma);
        energy_json = buf;
    }
    CK(cudaFree(out));

    std::string e2e_json = "null";
    if (a.e2e_steps > 0) {
        // End to end through the host-level API: host rule + charges in, this rank's slabs out
        // into ordinary (pageable) host memory through the library's bounded pinned ring, in
        // blocks of <= 1 GiB of slabs (bounded host memory at any shard size).
        const std::int64_t slab = N[0] * N[1];
        const std::int64_t blk = std::max<std::int64_t>(1, std::min<std::int64_t>(k1 - k0, (1ll << 27) / slab));
        std::vector<double> host(static_cast<std::size_t>(blk * slab));
        std::vector<double> ch;
        for (const latsum::Charge& c : spec.charges) ch.insert(ch.end(), {c.pos[0], c.pos[1], c.pos[2], c.Z});
        auto pass = [&] {
            for (std::int64_t ks = k0; ks < k1; ks += blk) {
                const std::int64_t ke = std::min(k1, ks + blk);
                latsum::cuda::check(ls_h_lattice_potential(static_cast<int>(gen), a.L, a.n, a.b, rule.exponents.data(),
                                                           rule.weights.data(), static_cast<int>(rule.node_count()),
                                                           ch.data(), static_cast<int>(spec.charges.size()),
                                                           a.periodic ? 1 : 0, ks, ke, host.data(), nullptr, nullptr,
                                                           nullptr, nullptr),
                                    "lattice_potential");
            }
        };
        pass();  // warm-up
        barrier();
        const double t0 = wall_s();
        for (int i = 0; i < a.e2e_steps; ++i) pass();
        double el = wall_s() - t0;
        CK(cudaMemcpy(scal, &el, sizeof(double), cudaMemcpyHostToDevice));
        comm->allreduce_max(scal, 1, s);
        CK(cudaMemcpyAsync(&el, scal, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const double per = el / a.e2e_steps;
        const std::int64_t h2d = 8 * (2 * rule.node_count() + 4 * static_cast<std::int64_t>(spec.charges.size()));
        char buf[1024];
        std::snprintf(buf, sizeof(buf),
                      "{\"value\": %.4f, \"unit\": \"Gpts/s\", \"h2d_bytes_per_step\": %ld, \"d2h_bytes_per_step\": %ld, "
                      "\"steps\": %d, \"d2h_gbs_per_rank\": %.1f, \"host_block_slabs\": %ld, "
                      "\"api\": \"ls_h_lattice_potential per <=1 GiB slab block into pageable host memory "
                      "(bounded pinned ring inside the library)\"}",
                      pts_total / per / 1e9, static_cast<long>(h2d), static_cast<long>(8 * pts_rank), a.e2e_steps,
                      8 * pts_rank / per / 1e9, static_cast<long>(blk));
        e2e_json = buf;
    }

    if (a.rank == 0) {
        char plan[256] = {0};
        ls_expand_plan_name(static_cast<int>(dp.rank()), plan, sizeof(plan));
        std::printf(
            "{\"runner\": \"latsum_shard_runner\", \"world\": %d, \"grid\": [%ld, %ld, %ld], \"rank_R\": %ld, "
            "\"slabs_rank0\": [%ld, %ld], \"steps\": %d, \"warmup\": %d, \"ms_per_step_max\": %.5f, "
            "\"expand_ms_mean_max\": %.5f, \"value_gpts\": %.4f, \"flops_per_launch_rank0\": %.6e, "
            "\"launches_rank0\": %ld, \"plan\": \"%s\", \"comm_init_s\": %.3f, \"energy\": %s, \"e2e\": %s}\n",
            a.world, static_cast<long>(N[0]), static_cast<long>(N[1]), static_cast<long>(N[2]),
            static_cast<long>(dp.rank()), static_cast<long>(k0), static_cast<long>(k1), a.steps, a.warmup, ms_step,
            mx[1], pts_total / (ms_step * 1e-3) / 1e9, 2.0 * static_cast<double>(dp.rank()) * pts_rank,
            static_cast<long>(launches), plan, comm_init_s, energy_json.c_str(), e2e_json.c_str());
        std::fflush(stdout);
    }
    cudaFree(scal);
    cudaStreamDestroy(s);
    return 0;
} catch (const std::exception& e) {
    std::fprintf(stderr, "latsum_shard_runner: %s\n", e.what());
    return 4;
}
