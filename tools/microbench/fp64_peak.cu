// FP64 pipe microbenchmarks for B200 (sm_100a): DFMA, DMMA (mma.sync f64) and
// a write-only HBM stream. Used to pin the FP64 roofline denominator that
// MEASURED_PEAKS.json lacks. Prints one JSON object per measurement.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 1.2345) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// m8n8k4: per warp 8*8*4 = 256 FMA
template <int ACC>
__global__ void dmma884_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  double c[ACC][2];
#pragma unroll
  for (int k = 0; k < ACC; ++k) { c[k][0] = k; c[k][1] = k + 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ACC; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ACC; ++k) s += c[k][0] + c[k][1];
  if (s == 1.2345) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// m16n8k4 f64: per warp 16*8*4 = 512 FMA; A 2 regs, B 1 reg, C 4 regs
template <int ACC>
__global__ void dmma1684_kernel(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-12, a1 = 0.5, b = 0.999999;
  double c[ACC][4];
#pragma unroll
  for (int k = 0; k < ACC; ++k) { c[k][0] = k; c[k][1] = k + 1; c[k][2] = k; c[k][3] = 2; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ACC; ++k)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ACC; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 1.2345) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// m16n8k16 f64: per warp 16*8*16 = 2048 FMA; A 8 regs, B 4 regs, C 4 regs
template <int ACC>
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + i * 1e-3 + threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.999 - i * 1e-4;
  double c[ACC][4];
#pragma unroll
  for (int k = 0; k < ACC; ++k) { c[k][0] = k; c[k][1] = k + 1; c[k][2] = k; c[k][3] = 2; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ACC; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ACC; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 1.2345) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Mixed: even warps DFMA, odd warps DMMA m8n8k4 -- do the two pipes overlap?
__global__ void mixed_kernel(double* out, int iters_fma, int iters_mma) {
  const int warp = threadIdx.x / 32;
  double s = 0;
  if (warp & 1) {
    double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) { c[k][0] = k; c[k][1] = k + 1; }
    for (int it = 0; it < iters_mma; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  } else {
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-9 + c;
    for (int it = 0; it < iters_fma; ++it) {
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], 0.999999, 1e-7);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c];
  }
  if (s == 1.2345) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void write_kernel(double2* out, size_t n2, double v) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride)
    out[i] = make_double2(v, v + 1);
}

template <class F>
float time_ms(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, (size_t)sms * 64 * 1024 * sizeof(double)));
  const int iters = 20000;
  if (argc > 1 && std::string(argv[1]) == "sweep") {
    // DMMA latency and occupancy: one CTA per SM, 1 or 2 warps per sub-partition, 1..16
    // independent accumulators per warp. cycles_per_dmma = per-warp issue interval.
    auto run = [&](auto kern, int acc, int threads) {
      int grid = sms, it = iters / 4;
      float ms = time_ms([&] { kern<<<grid, threads>>>(out, it); }, 5);
      double flops = 2.0 * 256 * acc * it * (double)grid * (threads / 32);
      double cyc = ms * 1e-3 * 1.965e9 / (double(it) * acc);
      printf("{\"bench\":\"dmma_sweep\",\"acc\":%d,\"warps_per_sp\":%d,\"ms\":%.4f,\"tflops\":%.3f,"
             "\"cycles_per_dmma_per_warp\":%.1f}\n", acc, threads / 128, ms, flops / ms / 1e9, cyc);
    };
    for (int threads : {128, 256, 384, 512}) {
      run(dmma884_kernel<1>, 1, threads);
      run(dmma884_kernel<2>, 2, threads);
      run(dmma884_kernel<4>, 4, threads);
      run(dmma884_kernel<8>, 8, threads);
      run(dmma884_kernel<16>, 16, threads);
    }
    return 0;
  }
  // DFMA sweeps
  for (int blocks_per_sm : {2, 4, 8}) {
    int threads = 256;
    int grid = sms * blocks_per_sm;
    float ms = time_ms([&] { dfma_kernel<8><<<grid, threads>>>(out, iters, 0.999999, 1e-7); }, 5);
    double flops = 2.0 * 8 * iters * (double)grid * threads;
    printf("{\"bench\":\"dfma\",\"chains\":8,\"grid\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", grid, threads, ms, flops / ms / 1e9);
  }
  {
    int grid = sms * 4, threads = 256;
    float ms = time_ms([&] { dfma_kernel<16><<<grid, threads>>>(out, iters, 0.999999, 1e-7); }, 5);
    double flops = 2.0 * 16 * iters * (double)grid * threads;
    printf("{\"bench\":\"dfma\",\"chains\":16,\"grid\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", grid, threads, ms, flops / ms / 1e9);
  }
  for (int blocks_per_sm : {2, 4, 8}) {
    int grid = sms * blocks_per_sm, threads = 256;
    int it = iters / 4;
    float ms = time_ms([&] { dmma884_kernel<8><<<grid, threads>>>(out, it); }, 5);
    double flops = 2.0 * 256 * 8 * it * (double)grid * (threads / 32);
    printf("{\"bench\":\"dmma_m8n8k4\",\"acc\":8,\"grid\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", grid, threads, ms, flops / ms / 1e9);
  }
  // 1 CTA of 8 warps per SM (2 warps per sub-partition), 8 and 16 accumulators per warp
  {
    int grid = sms, threads = 256, it = iters / 4;
    float ms = time_ms([&] { dmma884_kernel<8><<<grid, threads>>>(out, it); }, 5);
    double flops = 2.0 * 256 * 8 * it * (double)grid * (threads / 32);
    printf("{\"bench\":\"dmma_m8n8k4\",\"acc\":8,\"grid\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", grid, threads, ms, flops / ms / 1e9);
    ms = time_ms([&] { dmma884_kernel<16><<<grid, threads>>>(out, it); }, 5);
    flops = 2.0 * 256 * 16 * it * (double)grid * (threads / 32);
    printf("{\"bench\":\"dmma_m8n8k4\",\"acc\":16,\"grid\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", grid, threads, ms, flops / ms / 1e9);
  }
  for (int blocks_per_sm : {2, 4}) {
    int grid = sms * blocks_per_sm, threads = 256;
    int it = iters / 8;
    float ms = time_ms([&] { dmma1684_kernel<8><<<grid, threads>>>(out, it); }, 5);
    double flops = 2.0 * 512 * 8 * it * (double)grid * (threads / 32);
    printf("{\"bench\":\"dmma_m16n8k4\",\"acc\":8,\"grid\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", grid, threads, ms, flops / ms / 1e9);
  }
  for (int blocks_per_sm : {2, 4}) {
    int grid = sms * blocks_per_sm, threads = 256;
    int it = iters / 32;
    float ms = time_ms([&] { dmma16816_kernel<4><<<grid, threads>>>(out, it); }, 5);
    double flops = 2.0 * 2048 * 4 * it * (double)grid * (threads / 32);
    printf("{\"bench\":\"dmma_m16n8k16\",\"acc\":4,\"grid\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", grid, threads, ms, flops / ms / 1e9);
  }
  // mixed: choose iteration counts so each half alone would take similar time
  {
    int grid = sms * 4, threads = 256;
    int itf = iters, itm = iters / 4;
    float ms = time_ms([&] { mixed_kernel<<<grid, threads>>>(out, itf, itm); }, 5);
    double ff = 2.0 * 8 * itf * (double)grid * threads / 2;
    double fm = 2.0 * 256 * 8 * itm * (double)grid * (threads / 32) / 2;
    printf("{\"bench\":\"mixed_dfma_dmma\",\"grid\":%d,\"ms\":%.4f,\"tflops\":%.3f,\"dfma_part\":%.3e,\"dmma_part\":%.3e}\n", grid, ms, (ff + fm) / ms / 1e9, ff, fm);
  }
  // write-only HBM stream, 8 GiB
  {
    size_t bytes = (size_t)8 << 30;
    double2* buf; CK(cudaMalloc(&buf, bytes));
    size_t n2 = bytes / 16;
    for (int bps : {4, 8}) {
      int grid = sms * bps, threads = 512;
      float ms = time_ms([&] { write_kernel<<<grid, threads>>>(buf, n2, 1.0); }, 5);
      printf("{\"bench\":\"write_stream\",\"bytes\":%zu,\"grid\":%d,\"ms\":%.4f,\"gbs\":%.1f}\n", bytes, grid, ms, bytes / ms / 1e6);
    }
    CK(cudaFree(buf));
  }
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("{\"sms\":%d,\"clock_khz_attr\":%d}\n", sms, clk);
  return 0;
}
