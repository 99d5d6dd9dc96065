// launch_cost.cu -- host-side cost of the runtime calls ls_expand makes per call (development tool).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
struct Big { double v[40]; };
__global__ void k_small(double* p) { if (p && threadIdx.x == 1234) p[0] = 1; }
__global__ void k_big(Big b) { if (threadIdx.x == 1234) b.v[0] = 1; }
template <class F> double us(F f, int n = 2000) {
    f(); cudaDeviceSynchronize();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}
int main() {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    Big b{};
    printf("empty launch          %.2f us\n", us([&] { k_small<<<1, 32, 0, s>>>(nullptr); }));
    printf("320B-param launch     %.2f us\n", us([&] { k_big<<<1, 32, 0, s>>>(b); }));
    printf("launch 296x256 + 100KB smem %.2f us\n", us([&] { k_small<<<296, 256, 0, s>>>(nullptr); }));
    printf("mallocAsync+freeAsync %.2f us\n", us([&] { void* p; cudaMallocAsync(&p, 1 << 20, s); cudaFreeAsync(p, s); }));
    printf("getLastError          %.2f us\n", us([&] { cudaGetLastError(); }));
    printf("getDevice             %.2f us\n", us([&] { int d; cudaGetDevice(&d); }));
    int v; printf("occupancy query       %.2f us\n", us([&] { cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_small, 256, 0); }));
    printf("funcSetAttribute      %.2f us\n", us([&] { cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000); }));
}
