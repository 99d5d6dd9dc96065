// expand_host.cpp -- host-side time per ls_expand call on a small grid (development tool).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "latsum_cuda.h"
int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 128;
    const int R = 41;
    double *f, *w, *out;
    cudaMalloc(&f, sizeof(double) * 3 * n * R);
    cudaMalloc(&w, sizeof(double) * R);
    cudaMalloc(&out, sizeof(double) * n * n * n);
    cudaMemset(f, 0, sizeof(double) * 3 * n * R);
    cudaMemset(w, 0, sizeof(double) * R);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    auto call = [&] {
        return ls_expand(f, n, f + n * R, n, f + 2 * n * R, n, w, n, n, n, R, 0, n, out, 0, 0, nullptr, nullptr,
                         nullptr, nullptr, s);
    };
    for (int i = 0; i < 20; ++i) call();
    cudaStreamSynchronize(s);
    const int N = 500;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) call();
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    auto t2 = std::chrono::steady_clock::now();
    printf("n=%lld: host issue %.2f us/call, wall %.2f us/call\n", (long long)n,
           std::chrono::duration<double, std::micro>(t1 - t0).count() / N,
           std::chrono::duration<double, std::micro>(t2 - t0).count() / N);
}
