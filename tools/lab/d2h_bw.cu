// d2h_bw.cu -- device-to-host copy bandwidth with 1, 2 and 4 concurrent streams (development tool).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t total = size_t(4) << 30;
    void *d, *h;
    cudaMalloc(&d, total);
    cudaHostAlloc(&h, total, cudaHostAllocDefault);
    cudaMemset(d, 1, total);
    cudaStream_t s[4];
    for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int ns : {1, 2, 4}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, 0);
            for (int i = 0; i < ns; ++i) cudaStreamWaitEvent(s[i], a, 0);
            const size_t part = total / ns;
            for (int i = 0; i < ns; ++i)
                cudaMemcpyAsync((char*)h + i * part, (char*)d + i * part, part, cudaMemcpyDeviceToHost, s[i]);
            for (int i = 0; i < ns; ++i) { cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, s[i]); cudaStreamWaitEvent(0, e, 0); }
            cudaEventRecord(b, 0);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("%d stream(s): %.1f GB/s\n", ns, total / ms / 1e6);
        }
    }
    // H2D for reference
    cudaEventRecord(a, 0);
    cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, 0);
    cudaEventRecord(b, 0);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("H2D 1 stream: %.1f GB/s\n", total / ms / 1e6);
}
