// issue_cost.cu -- what do non-DMMA instructions cost next to a saturated DMMA pipe? (lab tool)
// The expansion's bare loop (4x4 tiles of 8x8 DMMA accumulators, 10 k-steps per tile, operands
// from shared memory, 2 CTAs x 8 warps per SM) plus EXTRA integer instructions per tile, either
// all at the tile end (WHERE 0, like an epilogue) or spread over the k-steps (WHERE 1).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int N>
__device__ __forceinline__ void extra(int (&x)[4], int lane) {
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("add.s32 %0, %0, %1;" : "+r"(x[i & 3]) : "r"(lane));
}

template <int EXTRA, int WHERE, int KIND>
__global__ void __launch_bounds__(256, 2) k(double* out, int NJ) {
    __shared__ double sm[4 * 11 * 32 * 4 + 64];
    for (int e = threadIdx.x; e < 4 * 11 * 32 * 4; e += 256) sm[e] = 1.0 + e * 1e-9;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const double* asw = sm + lane;
    double acc[4][4][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
    int x[4] = {lane, 1, 2, 3};
    double fx = 1.0 + lane;
    for (int jb = 0; jb < NJ; ++jb) {
#pragma unroll
        for (int ks = 0; ks < 10; ++ks) {
            double a[4], b[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) a[m] = asw[(m * 11 + ks) * 32];
#pragma unroll
            for (int n = 0; n < 4; ++n) b[n] = asw[(n * 11 + ks) * 32 + 64];
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int n = 0; n < 4; ++n) dmma(acc[m][n][0], acc[m][n][1], a[m], b[n]);
            if (WHERE == 1) {
                if (KIND == 0) extra<EXTRA / 10>(x, lane);
                if (KIND == 1) {
#pragma unroll
                    for (int i = 0; i < EXTRA / 10; ++i) asm volatile("fma.rn.f64 %0, %0, %0, %0;" : "+d"(fx));
                }
            }
        }
        if (WHERE == 0) {
            if (KIND == 0) extra<EXTRA>(x, lane);
            if (KIND == 1) {
#pragma unroll
                for (int i = 0; i < EXTRA; ++i) asm volatile("fma.rn.f64 %0, %0, %0, %0;" : "+d"(fx));
            }
        }
    }
    double s = fx;
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n) s += acc[m][n][0] + acc[m][n][1];
    if (s == 1.2345 || x[0] + x[1] + x[2] + x[3] == 123456789) out[0] = s;
}

template <int EXTRA, int WHERE, int KIND>
void run(double* out, int per_sm = 2) {
    const int NJ = 400, grid = 148 * per_sm;
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    k<EXTRA, WHERE, KIND><<<grid, 256>>>(out, NJ); CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0)); k<EXTRA, WHERE, KIND><<<grid, 256>>>(out, NJ); CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    const double flops = 2.0 * 256 * 16 * 10.0 * NJ * grid * 8;
    // per-SMSP clocks per tile-round (4 warps' tiles): best_ms * 1.965e6 / NJ
    printf("{\"ctas_per_sm\":%d,\"extra\":%d,\"where\":\"%s\",\"kind\":\"%s\",\"ms\":%.4f,\"tflops\":%.3f,\"clk_per_warp_tile\":%.1f}\n", per_sm, EXTRA,
           WHERE ? "spread over k-steps" : "tile end", KIND ? "dfma (dependent)" : "iadd", best, flops / best / 1e9,
           best * 1.965e6 / NJ / (2 * per_sm));
}

int main() {
    double* out; CK(cudaMalloc(&out, 1024));
    run<0, 0, 0>(out);
    run<40, 0, 0>(out); run<80, 0, 0>(out); run<160, 0, 0>(out); run<320, 0, 0>(out); run<640, 0, 0>(out);
    run<40, 1, 0>(out); run<80, 1, 0>(out); run<160, 1, 0>(out); run<320, 1, 0>(out); run<640, 1, 0>(out);
    run<40, 0, 1>(out); run<40, 1, 1>(out);
    // one CTA of 8 warps per SM (two warps per sub-partition, the A2-in-TMEM plan's shape)
    run<0, 0, 0>(out, 1); run<40, 0, 0>(out, 1); run<160, 0, 0>(out, 1); run<320, 0, 0>(out, 1); run<640, 0, 0>(out, 1);
    run<160, 1, 0>(out, 1); run<640, 1, 0>(out, 1);
    return 0;
}
