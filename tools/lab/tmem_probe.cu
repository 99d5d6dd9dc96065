#include <cstdint>
#include <cstdio>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__global__ void k(double* out, const double* in) {
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&taddr_s)), "r"(256) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = taddr_s;
    const uint32_t ta = base + ((uint32_t)((warp & 3) * 32) << 16);
    // store 4 doubles (8 columns) per thread, read back
    double v[4];
    for (int c = 0; c < 4; ++c) v[c] = in[threadIdx.x * 4 + c];
    uint32_t r[8];
    for (int c = 0; c < 4; ++c) { r[2*c] = __double2loint(v[c]); r[2*c+1] = __double2hiint(v[c]); }
    const uint32_t col = (warp >> 2) * 8;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "r"(ta + col), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t o[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]), "=r"(o[7]) : "r"(ta + col) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int c = 0; c < 4; ++c) out[threadIdx.x * 4 + c] = __hiloint2double(o[2*c+1], o[2*c]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(base), "r"(256) : "memory");
}
int main() {
    double *in, *out; cudaMalloc(&in, 256*4*8); cudaMalloc(&out, 256*4*8);
    double h[1024]; for (int i = 0; i < 1024; ++i) h[i] = i * 1.5 + 0.25;
    cudaMemcpy(in, h, 8192, cudaMemcpyHostToDevice);
    k<<<2, 256>>>(out, in);
    cudaError_t e = cudaDeviceSynchronize();
    double g[1024]; cudaMemcpy(g, out, 8192, cudaMemcpyDeviceToHost);
    int bad = 0; for (int i = 0; i < 1024; ++i) bad += g[i] != h[i];
    printf("err=%s bad=%d\n", cudaGetErrorString(e), bad);
}
