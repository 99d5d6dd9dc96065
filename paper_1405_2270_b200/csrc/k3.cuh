// k3.cuh -- definitions shared by the K3 translation units: the expansion launch arguments,
// the DMMA / mbarrier / TMA helpers, the TMEM kernel constants and the entry points that hand
// the host launcher a TMEM kernel instantiation (expand_tmem8.cu, expand_tmem16.cu, compiled in
// parallel with expand.cu).
#pragma once

#include "common.cuh"

namespace ls_k3 {

struct ExpandArgs {
    const double* A;
    const double* B;
    const double* Bp;   // A2 packed per stage (see pack_b_kernel)
    const double* C;
    const double* w;
    int64_t lda, ldb, ldc;
    int64_t N1, N2, N3;
    int R;            // rank
    int KD;           // DMMA k-steps (4 ranks each); ranks >= 4*KD go to the DFMA tail
    int n_tail;       // R - 4*KD in {0, 1, 2}
    int KC;           // k-steps per stage
    int n_kc;         // k-chunks: ceil(KD / KC)
    int64_t n_jt;     // packed j-tiles (multiple of JT)
    int64_t n_jc;     // j-chunks per unit
    int64_t k0, k1;
    double* out;
    int64_t ldy, ldz;
    int vec_store;    // 16-byte pair stores legal (aligned base, even strides)
    const double* rho1;
    const double* rho2;
    const double* rho3;
    double* partial;
    int64_t n_ichunks;
    int64_t n_units;
    int debug;        // development knobs (LS_EXPAND_DEBUG): 1 no stores (sink), 2 fill once, 4 no tail,
                      // 8 scale once, 16 no epilogue at all
    int accumulate;   // add into out / partial instead of overwriting (rank-chunked expansions)
    const double* S;  // per-slab scales S(k, q) = w_q * A3(k, q), [k][q] (TMEM variant)
    int split_tail;   // TMEM store-only: split the last round of units at stage granularity
    unsigned* fault;  // watchdog word of the device (ls::fault_flag)
    unsigned long long* timeline;  // lab builds with -DLS_TIMELINE only: per-warp event log (else null)
};

// Lab instrumentation (-DLS_TIMELINE builds only; compiled out of the product): lane 0 of each
// warp logs (clock64 << 8 | event) into 128 slots per warp, slot 0 holding the count and the
// SM id, so tools/lab/timeline.py can attribute a CTA's time to waits, DMMA issue, fills and
// epilogues.
#ifdef LS_TIMELINE
__device__ __forceinline__ unsigned long long tl_globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define LS_TL_INIT()                                                                         \
    int tl_n_ = 1;                                                                           \
    unsigned long long* tl_ = p.timeline ? p.timeline + (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 128 : nullptr; \
    if (tl_ && (threadIdx.x & 31) == 0) tl_[126] = ls_k3::tl_globaltimer()
#define LS_TL(ev)                                                                            \
    do {                                                                                     \
        if (tl_ && (threadIdx.x & 31) == 0 && tl_n_ < 126) {                                 \
            tl_[tl_n_++] = (static_cast<unsigned long long>(clock64()) << 8) | (ev);         \
        }                                                                                    \
    } while (0)
#define LS_TL_END()                                                                          \
    do {                                                                                     \
        if (tl_ && (threadIdx.x & 31) == 0) {                                                \
            unsigned smid;                                                                   \
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));                                \
            tl_[0] = (static_cast<unsigned long long>(smid) << 32) | static_cast<unsigned>(tl_n_); \
            tl_[127] = ls_k3::tl_globaltimer();  /* slots 126/127: %globaltimer at warp start/end */ \
        }                                                                                    \
    } while (0)
#else
#define LS_TL_INIT() (void)0
#define LS_TL(ev) (void)0
#define LS_TL_END() (void)0
#endif

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Waits for the phase with the given parity. A wait that has not completed after 20 s (no stage
// of any plan takes more than milliseconds) sets the device's fault word (ls::fault_flag) and
// returns; once the word is set every other wait returns at once too, so the kernel drains,
// releases its TMEM and exits, and the host-level call reports LS_ECUDA (ls_fault_status for
// device-level callers) instead of hanging the GPU or trapping the context.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity, unsigned* fault) {
    if (mbar_try_wait(bar, parity)) return;
    const uint64_t t0 = global_ns();
    while (!mbar_try_wait(bar, parity)) {
        if (*reinterpret_cast<volatile unsigned*>(fault) != 0) return;
        if (global_ns() - t0 > 20000000000ull) {
            atomicExch(fault, 1u);
            return;
        }
    }
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// TMEM columns per CTA: 8-warp CTAs run two per SM (256 columns each), 16-warp CTAs one (512).
__host__ __device__ constexpr int tmem_cols(int warps) { return warps == 8 ? 256 : 512; }
// Fill staging per lane: two tasks in flight (cp.async two tasks ahead), each 4 A1 values + the
// slab scale.
constexpr int kTaskSlots = 5;
constexpr int kFillSlots = 2 * kTaskSlots;
__host__ __device__ constexpr int tmem_stg_elems(int warps) { return warps * kFillSlots * 32; }  // per CTA
// Shared-memory header of the TMEM kernels (doubles): ring mbarriers, per-lane-quarter A1k
// hand-over mbarriers, ring release counters and the TMEM base address.
constexpr int kTmemHdr = 48;

using KernelFn = void (*)(ExpandArgs);

// 8-warp TMEM kernel for ring shape `code` (10 * depth + j-chunks per stage), KD k-steps and
// nt DFMA ranks; nullptr if the shape is not built. Compile-time KD for KD 1..14 with nt = 1.
KernelFn tmem8_kernel(bool store, bool func, int code, int kd, int nt);
// 16-warp TMEM kernel (2-deep ring, one DFMA rank); compile-time KD for KD 15..23 with whole-
// rank stages (kc == kd) and for KD 24..30 with two stages of kc = ceil(kd / 2) k-steps.
KernelFn tmem16_kernel(bool store, bool func, int kd, int kc);

// Single-buffer 16-warp TMEM kernel for KD 31..62 (expand_tmem16s_{a,b}.cu); nullptr outside.
// k-chunks per tile: the fewest whose 2-deep ring of 16-j-tile stages fits next to the fill
// staging in one CTA's shared memory (KD <= 46: two, else three).
__host__ __device__ constexpr int tmem16s_nkc(int kd) { return kd <= 46 ? 2 : 3; }
__host__ __device__ constexpr int tmem16s_kc(int kd) { return (kd + tmem16s_nkc(kd) - 1) / tmem16s_nkc(kd); }
KernelFn tmem16s_kernel_a(bool store, bool func, int kd);
KernelFn tmem16s_kernel_b(bool store, bool func, int kd);
inline KernelFn tmem16s_kernel(bool store, bool func, int kd) {
    return kd <= 45 ? tmem16s_kernel_a(store, func, kd) : tmem16s_kernel_b(store, func, kd);
}

// Small-N2 plan (expand_a2t.cu): A2 resident in TMEM, A1k of 64-row units streamed by TMA from
// a pre-pass; for N2 <= 256 at ranks <= 57.
bool fits_a2t(int64_t N2, int KD, int NT);
int64_t a2t_units(int64_t N1, int64_t k0, int64_t k1);
int launch_a2t(ExpandArgs& a, bool store, bool func, cudaStream_t s, int sm_count,
               int (*setup)(const void*, int, size_t, int&));

// Split-K TMEM plan for ranks beyond the double-buffered TMEM plans (expand_splitk.cu).
bool fits_splitk(int KD, int n_tail);
int launch_splitk(ExpandArgs& a, bool store, bool func, cudaStream_t s, int sm_count,
                  int (*setup)(const void*, int, size_t, int&));

}  // namespace ls_k3
