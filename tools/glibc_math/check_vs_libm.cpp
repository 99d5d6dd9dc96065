// check_vs_libm.cpp -- compares the host instantiation of csrc/glibc_math.cuh with the
// installed libm, bit for bit.
//
//   g++ -std=c++17 -O2 -ffp-contract=off -mfma -pthread -o check_vs_libm check_vs_libm.cpp
//   ./check_vs_libm random <n_per_class> <seed>   seeded sweeps over every branch of erf and exp
//   ./check_vs_libm file <args.f64>               erf(x) and exp(-x*x) for each double in a file
//
// Prints one line per argument class: class, count, erf mismatches, exp mismatches, and the
// first mismatching argument if any. Exit status 1 on any mismatch. Test infrastructure:
// tests/test_glibc_math.py runs a bounded sweep; profiles/r02_glibc_math_sweep.txt holds the
// long one.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>
#include <atomic>

#include "../../paper_1405_2270_b200/csrc/glibc_math.cuh"

namespace {

uint64_t bits_of(double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
}
double from_bits(uint64_t u) {
    double x;
    std::memcpy(&x, &u, 8);
    return x;
}
// NaNs compare equal to NaNs (payloads are not part of the contract); everything else bitwise.
bool same(double a, double b) { return (std::isnan(a) && std::isnan(b)) || bits_of(a) == bits_of(b); }

struct Tally {
    std::atomic<uint64_t> n{0}, erf_bad{0}, exp_bad{0};
    std::atomic<uint64_t> first_bad{0};
    std::atomic<bool> have_first{false};
    void bad(double x) {
        bool f = false;
        if (have_first.compare_exchange_strong(f, true)) first_bad = bits_of(x);
    }
};

void check_one(double x, Tally& t) {
    t.n.fetch_add(1, std::memory_order_relaxed);
    if (!same(ls::gm::erf(x), std::erf(x))) {
        t.erf_bad.fetch_add(1, std::memory_order_relaxed);
        t.bad(x);
    }
    if (!same(ls::gm::exp(x), std::exp(x))) {
        t.exp_bad.fetch_add(1, std::memory_order_relaxed);
        t.bad(x);
    }
    const double y = -x * x;  // the midpoint generator's argument
    if (!same(ls::gm::exp(y), std::exp(y))) {
        t.exp_bad.fetch_add(1, std::memory_order_relaxed);
        t.bad(x);
    }
}

struct Class {
    const char* name;
    // draws one argument
    double (*draw)(std::mt19937_64&);
};

double uni(std::mt19937_64& g, double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(g() >> 11) * 0x1p-53);
}
double sgn(std::mt19937_64& g, double v) { return (g() & 1) ? -v : v; }

const Class kClasses[] = {
    {"any_bit_pattern", [](std::mt19937_64& g) { return from_bits(g()); }},
    {"erf_tiny_lt_2^-28", [](std::mt19937_64& g) { return sgn(g, std::ldexp(uni(g, 1.0, 2.0), -29 - int(g() % 1000))); }},
    {"erf_lt_0.84375", [](std::mt19937_64& g) { return sgn(g, uni(g, 0x1p-28, 0.84375)); }},
    {"erf_0.84375_1.25", [](std::mt19937_64& g) { return sgn(g, uni(g, 0.84375, 1.25)); }},
    {"erf_1.25_2.857", [](std::mt19937_64& g) { return sgn(g, uni(g, 1.25, 1.0 / 0.35)); }},
    {"erf_2.857_6", [](std::mt19937_64& g) { return sgn(g, uni(g, 1.0 / 0.35, 6.0)); }},
    {"erf_6_8", [](std::mt19937_64& g) { return sgn(g, uni(g, 6.0, 8.0)); }},
    {"log_uniform_1e-300_1e3", [](std::mt19937_64& g) { return sgn(g, std::exp(uni(g, -690.0, 6.9))); }},
    {"exp_-745_-708_subnormal", [](std::mt19937_64& g) { return uni(g, -746.0, -707.0); }},
    {"exp_-1100_710", [](std::mt19937_64& g) { return uni(g, -1100.0, 710.0); }},
    {"exp_-40_0", [](std::mt19937_64& g) { return uni(g, -40.0, 0.0); }},
};

int run_random(uint64_t n_per_class, uint64_t seed) {
    const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    int rc = 0;
    for (const Class& c : kClasses) {
        Tally t;
        std::vector<std::thread> th;
        for (unsigned w = 0; w < nt; ++w)
            th.emplace_back([&, w] {
                std::mt19937_64 g(seed * 1000003u + w * 7919u + std::hash<std::string>{}(c.name));
                for (uint64_t i = w; i < n_per_class; i += nt) check_one(c.draw(g), t);
            });
        for (auto& x : th) x.join();
        std::printf("%-26s n=%llu erf_mismatch=%llu exp_mismatch=%llu", c.name, (unsigned long long)t.n.load(),
                    (unsigned long long)t.erf_bad.load(), (unsigned long long)t.exp_bad.load());
        if (t.have_first) std::printf(" first=0x%016llx", (unsigned long long)t.first_bad.load());
        std::printf("\n");
        if (t.erf_bad || t.exp_bad) rc = 1;
    }
    return rc;
}

int run_file(const char* path) {
    FILE* f = std::fopen(path, "rb");
    if (!f) {
        std::perror(path);
        return 2;
    }
    std::vector<double> xs;
    double buf[4096];
    size_t got;
    while ((got = std::fread(buf, 8, 4096, f)) > 0) xs.insert(xs.end(), buf, buf + got);
    std::fclose(f);
    Tally t;
    const unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nt; ++w)
        th.emplace_back([&, w] {
            for (size_t i = w; i < xs.size(); i += nt) check_one(xs[i], t);
        });
    for (auto& x : th) x.join();
    std::printf("%-26s n=%llu erf_mismatch=%llu exp_mismatch=%llu", "file", (unsigned long long)t.n.load(),
                (unsigned long long)t.erf_bad.load(), (unsigned long long)t.exp_bad.load());
    if (t.have_first) std::printf(" first=0x%016llx", (unsigned long long)t.first_bad.load());
    std::printf("\n");
    return (t.erf_bad || t.exp_bad) ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc >= 2 && std::string(argv[1]) == "random")
        return run_random(argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1000000,
                          argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 1);
    if (argc >= 3 && std::string(argv[1]) == "file") return run_file(argv[2]);
    std::fprintf(stderr, "usage: %s random [n_per_class] [seed] | file <args.f64>\n", argv[0]);
    return 2;
}
