// common.cuh -- shared plumbing for liblatsum_cuda.so: status codes, the
// thread-local error message, launch accounting and FP64 helpers.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>

#include <atomic>
#include <cstdlib>
#include <cstdint>
#include <string>
#include <utility>

#include "latsum_cuda.h"

namespace ls {

std::string& last_error();
std::atomic<int64_t>& launch_counter();

inline int fail(int code, const std::string& msg) {
    last_error() = msg;
    return code;
}
inline int cuda_fail(cudaError_t e, const char* where) {
    cudaGetLastError();  // clear a non-sticky error so the next launch check does not report it again
    return fail(LS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define LS_CUDA(expr)                                                   \
    do {                                                                \
        cudaError_t _e = (expr);                                        \
        if (_e != cudaSuccess) return ::ls::cuda_fail(_e, #expr);       \
    } while (0)

// After a kernel launch: count it and surface launch-configuration errors.
#define LS_LAUNCHED(name)                                               \
    do {                                                                \
        ::ls::launch_counter().fetch_add(1, std::memory_order_relaxed); \
        cudaError_t _e = cudaGetLastError();                            \
        if (_e != cudaSuccess) return ::ls::cuda_fail(_e, name);        \
    } while (0)

// Kernel watchdog: a device word per device that a timed-out mbarrier wait sets (k3.cuh
// mbar_wait); every other wait then returns at once, so the kernel drains and exits normally
// (TMEM released, context intact) and the host reports LS_ECUDA instead of hanging or
// trapping. fault_flag() is the current device's word; take_fault() reads and clears it.
unsigned* fault_flag();
bool take_fault();

#define LS_SYNC(stream)                                                                   \
    do {                                                                                  \
        LS_CUDA(cudaStreamSynchronize(stream));                                           \
        if (::ls::take_fault())                                                           \
            return ::ls::fail(LS_ECUDA, "kernel watchdog: an mbarrier wait timed out (results discarded)"); \
    } while (0)

// Development A/B knobs (forced plans, debug modes, verbose plan print) are read from the
// environment only in a build with -DLS_DEV_KNOBS (python -m paper_1405_2270_b200.build --dev);
// the product library never changes its work based on the environment.
inline const char* dev_knob(const char* name) {
#ifdef LS_DEV_KNOBS
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Makes `device` current for the scope and restores the caller's device afterwards
// (pipeline objects remember the device they were created on).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int device) {
        if (cudaGetDevice(&prev) != cudaSuccess || prev == device || cudaSetDevice(device) != cudaSuccess) prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Stream-ordered scratch from the device pool, released on every exit path (early error
// returns included) with cudaFreeAsync on the stream it was allocated on.
struct AsyncScratch {
    void* p = nullptr;
    cudaStream_t s;
    explicit AsyncScratch(cudaStream_t st) : s(st) {}
    cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes, s); }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    ~AsyncScratch() {
        if (p) cudaFreeAsync(p, s);
    }
    AsyncScratch(const AsyncScratch&) = delete;
    AsyncScratch& operator=(const AsyncScratch&) = delete;
};

// Number of SMs of the current device (cached per device).
int sm_count();

// Start of the master window of a charge at grid index ia for lattice shift 0 (the window of
// shift k starts k*n lower): window_start_box (lattice.hpp:98) or window_start_periodic
// (lattice.hpp:104-106), N = L*n.
__host__ __device__ inline int64_t window_start(int periodic, int64_t N, int64_t L, int64_t n, int64_t ia) {
    return periodic ? N + (L / 2) * n - ia : N - ia;
}

// Generator + assembled sum of up to three distinct axes (generator.cu). Axis a: master
// (2 L n x R, leading dim 2 L n) and assembled factor (out_len x M0 R, leading dim out_len =
// periodic ? n : L n) from the M0 charge grid indices ia_d. One launch when every master column
// fits shared memory, else ls_gen_master + ls_assemble_axis per axis; bit-identical either way.
struct GenAsmAxis {
    int64_t L;
    const int64_t* ia_d;
    double* master_d;
    double* out_d;
};
// Periodic lattices with one charge and L >= 32 take a fused launch that never writes the
// master (*master_written = false then); every other lattice gets its master written.
int gen_assemble(int mode, const double* tau_d, int R, int M0, int64_t n, double h, int periodic,
                 const GenAsmAxis* ax, int n_ax, cudaStream_t s, bool* master_written = nullptr);

// Keeps freed stream-ordered allocations cached in the current device's default
// pool (no OS round trip per call). Idempotent per device.
void ensure_pool();

}  // namespace ls

// Programmatic dependent launch (PDL) along the step's kernel chain (generator -> assembly ->
// prep -> expansion): a kernel launched with launch_pdl may start while its predecessor in the
// stream still runs; it must call pdl_wait() before touching anything the predecessor writes.
// pdl_trigger() lets the next kernel in the chain start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

namespace ls {
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace ls

// Rounded FP64 primitives that the compiler can never contract into FMA:
// used wherever the reference's operation order must be reproduced.
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }
