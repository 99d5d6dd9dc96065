// expand_tmem.cuh -- K3 variant with the scaled left factor A1k resident in tensor
// memory (TMEM), double-buffered across work units. Included by expand.cu.
//
// The shared-memory variant (expand_dmma_kernel) must stop every warp of the CTA at each
// unit boundary: one barrier before A1k of the next slab overwrites the current one, one
// after the fill. Here A1k lives in TMEM (256 of 512 columns per 8-warp CTA, all 512 for the
// 16-warp shape; otherwise unused by an FP64 kernel): two buffers, so the warps fill unit u+1's A1k piece by piece while they
// multiply unit u, and units hand over through mbarriers (as_full / as_empty) instead of
// CTA barriers. Shared memory then holds the TMA ring of A2 stages and a small per-warp
// staging area through which the next fill task's A1/S operands arrive by cp.async.
//
// TMEM layout (per CTA, lanes = warp quarter wi = warp & 3, i.e. the warps sharing i-tiles):
//   buffer b, column b*CB + ks*8 + it*2 + {0,1}: A1k(8*(4*wi + it) + g, 4*ks + t) (lo, hi words)
//   buffer b, column b*CB + 8*KD + qt*16 + n*4 + {0..3}: the two tail-rank values lane (g, t)
//   needs for i-tile n: A1k(32*wi + 8n + 2t + {0,1}, 4*KD + qt)
// CB = 8*KD + 16*n_tail columns: KD <= 14 fits two buffers in 256 columns, KD <= 30 in 512.
// n_tail is always 1 here (a zero rank when R mod 4 is 0 or 3; see tmem_tail in expand.cu).
#pragma once

#include "k3.cuh"

namespace ls_k3 {

namespace tmem {

// Issue a 32-lane x 8-column load (4 doubles per thread); the registers are valid after wait_ld().
// No memory clobbers: ordinary shared-memory loads may be scheduled around these, while the
// volatile asm statements (ld, wait, DMMA) keep their program order.
__device__ __forceinline__ void ld_x8_issue(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void wait_ld(uint32_t (&r)[8]) {
    // The register operands tie the wait to the loaded values, so no use is hoisted above it.
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]));
}
__device__ __forceinline__ void unpack(const uint32_t (&r)[8], double (&v)[4]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = __hiloint2double(static_cast<int>(r[2 * c + 1]), static_cast<int>(r[2 * c]));
}
__device__ __forceinline__ void ld_x8(uint32_t taddr, double (&v)[4]) {
    uint32_t r[8];
    ld_x8_issue(taddr, r);
    wait_ld(r);
    unpack(r, v);
}

__device__ __forceinline__ void st_x8(uint32_t taddr, const double (&v)[4]) {
    uint32_t r[8];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        r[2 * c] = static_cast<uint32_t>(__double2loint(v[c]));
        r[2 * c + 1] = static_cast<uint32_t>(__double2hiint(v[c]));
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

}  // namespace tmem

// 8-byte global->shared copy (LDGSTS); src_size 0 writes zeros without reading.
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Requires: 32x32 warp tiles (TM = TN = 4), WI = 4 warps along i (one per TMEM lane quarter),
// whole rank in one stage (n_kc == 1), n_tail == 1.
// NS: ring depth; JPS: j-chunks per ring stage (each warp computes JPS tiles per stage).
// WARPS = 8 (WJ = 2 warps along j, 2 CTAs/SM, KD <= 14) or 16 (WJ = 4, 1 CTA/SM, all 512 TMEM
// columns; the shared-memory ring limits it to KD <= 23, i.e. ranks up to 93).
// KD_ > 0 fixes the k-step count at compile time (the 8-warp shape is instantiated for every
// KD it covers): the k-step loop is then fully unrolled with immediate shared-memory and TMEM
// offsets, 2.2% faster at cfg1 than the runtime-KD loop. KD_ = 0 reads p.KD.
// KC_ > 0 (16-warp shape, compile-time KD_ only): stages of KC_ k-steps, two per j-chunk, for
// ranks whose whole-rank stage no longer fits the shared-memory ring (KD 24..30); the
// accumulators persist across the two stages of a tile.
// NKC_ (with KC_ > 0): k-chunk stages per tile (the last one may be shorter).
// SINGLE_ (16-warp shape, ranks beyond two A1k buffers: KD 31..62): ONE A1k buffer of up to 512
// columns. The next unit's A1k is written at the unit boundary, each lane quarter as soon as its
// own WJ warps are done with the unit, with all of the quarter's fill loads in flight at once;
// the A2 ring keeps streaming the next unit's stages meanwhile.
template <bool STORE, bool FUNC, int NS, int JPS, int WARPS_ = 8, int KD_ = 0, int NT_ = 1, int KC_ = 0,
          int NKC_ = 2, bool SINGLE_ = false>
__global__ void __launch_bounds__(WARPS_ * 32, WARPS_ == 8 ? 2 : 1) expand_tmem_kernel(const ExpandArgs p) {
    constexpr int WARPS = WARPS_, WI = 4, WJ = WARPS / WI, kTM = 4, kTN = 4, IC = 128, JT = kTM * WJ * JPS,
                  JC = 8 * kTM * WJ, kNS = NS;
    constexpr int kTmemCols = tmem_cols(WARPS);
    constexpr int kThreads = WARPS * 32;
    const int KD = KD_ > 0 ? KD_ : p.KD;
    constexpr int n_tail = NT_;  // 1 or 2 DFMA ranks (launch() makes a zero rank when R mod 4 is 0 or 3)
    const int CB = 8 * KD + 16 * n_tail;
    constexpr bool kChunked = KC_ > 0;
    constexpr bool SINGLE = SINGLE_;
    static_assert(!kChunked || (KD_ > (NKC_ - 1) * KC_ && KD_ <= NKC_ * KC_ && JPS == 1),
                  "k-chunked stages: NKC_ per tile");
    static_assert(!SINGLE || (WARPS_ == 16 && kChunked), "single A1k buffer: 16-warp chunked shape");
    const int KCs = kChunked ? KC_ : KD;          // k-steps per stage
    constexpr int n_kc = kChunked ? NKC_ : 1;     // stages per tile
    const int frag_elems = JT * KCs * 32;
    const int stage_elems = frag_elems + JT * 8 * n_tail;
    const int n_ichunks = static_cast<int>(p.n_ichunks);
    const int n_units = static_cast<int>(p.n_units);
    const int per_unit = static_cast<int>(p.n_jc) * n_kc;
    const unsigned stage_bytes = static_cast<unsigned>(stage_elems * sizeof(double));

    // Shared-memory header (kTmemHdr doubles): ring mbarriers, then the A1k hand-over
    // mbarriers per buffer and TMEM lane quarter, the ring release counters and the TMEM base
    // address; the fill staging and the A2 ring follow.
    static_assert(kNS <= 12, "header holds up to 12 ring slots");
    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);       // [kNS] A2 stage landed
    // A1k buffer b, lane quarter q is written and read only by the WJ warps of that quarter
    // (warp & 3 == q), so the hand-over is per quarter: a quarter's warps never wait for the
    // other quarters' skew at unit boundaries.
    uint64_t* as_full = full + 12;                             // [2][4] quarter's A1k written by its WJ warps
    uint64_t* as_empty = full + 20;                            // [2][4] quarter's A1k released by its WJ warps
    int* released = reinterpret_cast<int*>(smem + 28);         // [kNS] warps done with a ring slot
    uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(smem + 34);
    double* ring = smem + kTmemHdr + tmem_stg_elems(WARPS);    // [kNS][stage_elems]

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2;
    const int t = lane & 3;
    const int wi = warp & 3;  // i-tiles, and the TMEM lane quarter this warp may access
    const int wj = warp >> 2;

    // Work of this CTA: whole units b + n*G over the full rounds. For store-only launches the
    // partial last round is split at stage granularity instead (balanced contiguous ranges of its
    // stages), so every CTA finishes within one stage of the others: at cfg1 (8192 units on 296
    // CTAs) the whole-unit tail left 1.2% of the GPU idle. Functional launches keep whole units
    // (one writer per per-warp partial).
    const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
    const bool kSplitTail = STORE && !FUNC && !kChunked && p.split_tail;
    const int n_full = kSplitTail ? n_units / G : 0;
    int t0 = 0, t1 = 0, tu0 = 0, n_tu = 0;  // this CTA's stages [t0, t1) of the tail round
    if (kSplitTail) {
        const int tail_stages = (n_units - n_full * G) * per_unit;
        t0 = static_cast<int>(static_cast<int64_t>(tail_stages) * b / G);
        t1 = static_cast<int>(static_cast<int64_t>(tail_stages) * (b + 1) / G);
        if (t1 > t0) {
            tu0 = t0 / per_unit;
            n_tu = (t1 - 1) / per_unit - tu0 + 1;
        }
    }
    const int my_units = kSplitTail ? n_full + n_tu : (n_units > b ? (n_units - 1 - b) / G + 1 : 0);
    const int full_stages = n_full * per_unit;
    const int n_stages = kSplitTail ? full_stages + (t1 - t0) : my_units * per_unit;
    auto unit_of = [&](int n) { return n < n_full || !kSplitTail ? b + n * G : n_full * G + tu0 + (n - n_full); };

    auto issue = [&](int st) {
        const int w = (kSplitTail && st >= full_stages) ? (t0 + st - full_stages) % per_unit : st % per_unit;
        // packed stage (k-chunk kcs, j-chunk jc) sits at (kcs * n_jc + jc) (pack_b_kernel)
        const int c = kChunked ? (w % n_kc) * static_cast<int>(p.n_jc) + w / n_kc : w;
        const double* src = p.Bp + static_cast<int64_t>(c) * stage_elems;
        uint64_t* bar = full + (st % kNS);
        mbar_arrive_expect_tx(bar, stage_bytes);
        tma_bulk_g2s(ring + (st % kNS) * stage_elems, src, stage_bytes, bar);
    };

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_s)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        for (int b = 0; b < kNS; ++b) {
            mbar_init(full + b, 1);
            released[b] = 0;
        }
        for (int b = 0; b < 8; ++b) {
            mbar_init(as_full + b, WJ);
            mbar_init(as_empty + b, WJ);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    // TMEM allocation and barrier set-up overlap the tail of the preceding (prep) launch; the
    // packed A2, the scale table and the factors are read only after it completes.
    pdl_wait();
    LS_TL_INIT();
    LS_TL(1);  // set-up done
    const uint32_t tq = *tmem_base_s + (static_cast<uint32_t>(32 * wi) << 16);  // this warp's lane quarter
    double* stg = smem + kTmemHdr + warp * (kFillSlots * 32) + lane;  // this lane's fill staging (stride 32)

    // Fill tasks of one unit for this warp: fragment k-steps ks = wj, wj+WJ, ... (4 values each),
    // then (warp wj == 0 only) the tail ranks, each as two half tasks of 4 values (so every
    // task stages 4 A1 values + 1 scale).
    const int n_frag_tasks = (KD - wj + WJ - 1) / WJ;
    const int n_tasks = n_frag_tasks + (wj == 0 ? 2 * n_tail : 0);
#ifdef LS_DEV_KNOBS
    const bool lab_nofill = (p.debug & 2) != 0;   // lab A/B: later units reuse the first A1k
    const bool lab_nostore = (p.debug & 1) != 0;  // lab A/B: epilogue without stores
#else
    constexpr bool lab_nofill = false, lab_nostore = false;
#endif
    // A fill task's operands are copied global->shared asynchronously TWO tasks ahead, through two
    // staging slots: the copy for task e + 2 is issued right after task e is consumed, so even
    // when a stage consumes two tasks back to back (short units: 4 stages per unit at 256^3)
    // the L2 latency of the A1/S reads stays off the warp's critical path. Tasks form one
    // sequence per warp over the units after the first: e = (nu - 1) * n_tasks + task.
    auto task_issue = [&](int u, int task, double* sg) {
        const int ib = (u % n_ichunks) * IC;
        const int64_t k = p.k0 + u / n_ichunks;
        if (task < n_frag_tasks) {
            const int ks = wj + WJ * task;
            const int q = 4 * ks + t;
            cp_async8(sg + 4 * 32, p.S + k * p.R + (q < p.R ? q : 0), q < p.R);
#pragma unroll
            for (int it = 0; it < 4; ++it) {
                const int i = ib + 8 * (4 * wi + it) + g;
                const bool ok = i < p.N1 && q < p.R;
                cp_async8(sg + it * 32, ok ? p.A + i + p.lda * q : p.A, ok);
            }
        } else {
            const int ht = task - n_frag_tasks;           // half task: tail rank ht / 2, half ht % 2
            const int q = 4 * KD + (ht >> 1);              // q >= R: the zero rank (see below)
            cp_async8(sg + 4 * 32, q < p.R ? p.S + k * p.R + q : p.S, q < p.R);
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) {
                const int e = 4 * (ht & 1) + e4;
                const int i = ib + 32 * wi + 8 * (e >> 1) + 2 * t + (e & 1);
                const bool ok = i < p.N1 && q < p.R;
                cp_async8(sg + e4 * 32, ok ? p.A + i + p.lda * q : p.A, ok);
            }
        }
        cp_async_commit();
    };
    const int n_seq = SINGLE ? 0 : (my_units - 1) * n_tasks;  // fill tasks after the prologue's unit
    int n_issued = 0;                             // cp.async groups committed (one per task)
    auto seq_issue = [&](int e) {
        if (e >= n_seq) return;
#ifdef LS_DEV_KNOBS
        if (p.debug & 32) return;  // lab A/B: no fill loads (stale staging)
#endif
        task_issue(unit_of(1 + e / n_tasks), e % n_tasks, stg + (e & 1) * (kTaskSlots * 32));
        ++n_issued;
    };
    auto task_consume = [&](int buf, int task, int e) {
        // the group of task e is complete once at most n_issued - e - 1 (0 or 1) groups are pending
        if (n_issued - e - 1 >= 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else cp_async_wait_all();
        const double* sg = stg + (e & 1) * (kTaskSlots * 32);
        const double sv = sg[4 * 32];
        const uint32_t col = static_cast<uint32_t>(buf * CB);
        double v[4];
#pragma unroll
        for (int it = 0; it < 4; ++it) v[it] = rn_mul(sg[it * 32], sv);  // Eigen's A1 * scale.asDiagonal()
#ifdef LS_DEV_KNOBS
        if (p.debug & 64)
#pragma unroll
            for (int it = 0; it < 4; ++it) v[it] = sg[it * 32];  // lab A/B: no DMUL
        if (p.debug & 16) return;                               // lab A/B: no TMEM store
#endif
        if (task < n_frag_tasks) {
            tmem::st_x8(tq + col + 8 * (wj + WJ * task), v);
        } else {
            const int ht = task - n_frag_tasks;
            tmem::st_x8(tq + col + 8 * KD + 16 * (ht >> 1) + 8 * (ht & 1), v);
        }
    };
    // Consume task `task` of this CTA's unit number nu into buffer buf, then start the copy two
    // tasks further down the sequence.
    auto run_task = [&](int nu, int task, int buf) {
        const int e = (nu - 1) * n_tasks + task;
        task_consume(buf, task, e);
        seq_issue(e + 2);
    };
    auto publish = [&](int buf) {
        tmem::wait_st();
        tmem::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(as_full + 4 * buf + wi);
    };

    // The first ring stages load while the warps build the first unit's A1k.
    if (threadIdx.x == 0)
        for (int st = 0; st < kNS && st < n_stages; ++st) issue(st);
    // Fill of a whole unit's A1k into buffer buf by this warp, with the global loads of
    // kBatch tasks in flight at once (no accumulators are live here, so the registers are
    // free): the prologue's first unit, and every unit boundary of the single-buffer shape.
    constexpr int kBatch = 4;
    auto fill_all = [&](int u, int buf) {
        const int ib = (u % n_ichunks) * IC;
        const int64_t k = p.k0 + u / n_ichunks;
        const uint32_t col = static_cast<uint32_t>(buf * CB);
        for (int t0 = 0; t0 < n_tasks; t0 += kBatch) {
            double av[kBatch][4], sv[kBatch];
#pragma unroll
            for (int b = 0; b < kBatch; ++b) {
                const int task = t0 + b;
                if (task >= n_tasks) break;
                if (task < n_frag_tasks) {
                    const int q = 4 * (wj + WJ * task) + t;
                    sv[b] = q < p.R ? __ldg(p.S + k * p.R + q) : 0.0;
#pragma unroll
                    for (int it = 0; it < 4; ++it) {
                        const int i = ib + 8 * (4 * wi + it) + g;
                        av[b][it] = (i < p.N1 && q < p.R) ? __ldg(p.A + i + p.lda * q) : 0.0;
                    }
                } else {
                    const int ht = task - n_frag_tasks;
                    const int q = 4 * KD + (ht >> 1);
                    sv[b] = q < p.R ? __ldg(p.S + k * p.R + q) : 0.0;
#pragma unroll
                    for (int e4 = 0; e4 < 4; ++e4) {
                        const int e = 4 * (ht & 1) + e4;
                        const int i = ib + 32 * wi + 8 * (e >> 1) + 2 * t + (e & 1);
                        av[b][e4] = (i < p.N1 && q < p.R) ? __ldg(p.A + i + p.lda * q) : 0.0;
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < kBatch; ++b) {
                const int task = t0 + b;
                if (task >= n_tasks) break;
                double v[4];
#pragma unroll
                for (int it = 0; it < 4; ++it) v[it] = rn_mul(av[b][it], sv[b]);
                if (task < n_frag_tasks) {
                    tmem::st_x8(tq + col + 8 * (wj + WJ * task), v);
                } else {
                    const int ht = task - n_frag_tasks;
                    tmem::st_x8(tq + col + 8 * KD + 16 * (ht >> 1) + 8 * (ht & 1), v);
                }
            }
        }
    };
    // Prologue: the first unit's A1k (buffer 0), all tasks now; then the copies for the next
    // unit's first two tasks start the two-ahead chain.
    if (my_units > 0) {
        fill_all(unit_of(0), 0);
        seq_issue(0);
        seq_issue(1);
        publish(0);
    }
    LS_TL(2);  // prologue fill published

    double fsum = 0.0;
    int st = 0;
    for (int n = 0; n < my_units; ++n) {
        const int unit = unit_of(n);
        // A tile's accumulators live within the unit's stages only (dead at the unit boundary,
        // where the single-buffer shape refills A1k with its loads in flight).
        double acc[kTM][kTN][2];
        // j-chunk range of this unit (partial only for the first and last unit of a split tail)
        const int jc_lo = (kSplitTail && n == n_full) ? t0 % per_unit : 0;
        const int jc_hi = (kSplitTail && n >= n_full && n == my_units - 1) ? (t1 - 1) % per_unit + 1 : per_unit;
        // Fill schedule for the next unit. 8-warp shape: the whole fill right after the first
        // stage's DMMAs, so the rest of the unit is pure DMMA issue and the next unit's A1k is
        // ready long before any warp of the quarter reaches it (with the per-quarter hand-over
        // and two-ahead copies: 676 -> 660 us at 1024^2 x 256 slabs, 55.8 -> 54.1 us at 256^3,
        // against tasks spread evenly over the unit's stages). 16-warp shape: spread over the
        // stages from the third on, offset by warp (starting at the first measured -0.5 to
        // -1.5% at ranks 73-113, +1.8% at 121).
        const int n_here = jc_hi - jc_lo;
        const int first_fill = (WARPS == 16 && n_here > 2) ? 2 : 0;
        auto fill_stage = [&](int task) {
            if (WARPS == 8 || SINGLE) return jc_lo;
            return jc_lo + first_fill + ((task * WARPS + warp) * (n_here - first_fill)) / (WARPS * n_tasks);
        };
        const int buf = SINGLE ? 0 : (n & 1);
        const bool has_next = n + 1 < my_units;
        const int ib = (unit % n_ichunks) * IC;
        const int64_t kk = unit / n_ichunks;
        mbar_wait(as_full + 4 * buf + wi, static_cast<unsigned>((SINGLE ? n : n >> 1) & 1), p.fault);
        tmem::fence_after();
        LS_TL(3);  // unit's A1k ready
        const uint32_t tb = tq + static_cast<uint32_t>(buf * CB);
        // rho1 of this lane's eight i columns, held for the whole unit (zero beyond N1, where the
        // accumulators are zero too).
        double r1[kTN][2];
        if (FUNC) {
            fsum = 0.0;
#pragma unroll
            for (int nn = 0; nn < kTN; ++nn)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = ib + wi * (8 * kTN) + 8 * nn + 2 * t + e;
                    r1[nn][e] = i < p.N1 ? __ldg(p.rho1 + i) : 0.0;
                }
        }
        int next_task = 0;
        // Epilogue addressing, strength-reduced: the unit's tiles are visited in ascending j, so
        // the lane's first output row advances by JC rows per tile (ptxas otherwise rebuilds the
        // whole 64-bit address, the lane ids included, in every tile).
        // Measured at 1024^2 (profiles/r02_rowrun_ab.txt): cfg1 2.657 -> 2.634 ms, ranks 21 / 41 at
        // 256 slabs +1.5%, 93 / 113 +0.5%; two DFMA ranks (KD 9: -1.7%, more spills) and the
        // single-buffer shape (rank 164: -1.7%) keep the per-tile address.
        constexpr bool kRowRun = STORE && !SINGLE && n_tail == 1;
        const int ibase = ib + wi * (8 * kTN);
        const bool fast_u = ibase + 8 * kTN <= p.N1 && (!STORE || (p.vec_store && !p.accumulate));
        double* row_run = nullptr;
        if (kRowRun) {
            const int jb0 = ((kChunked ? jc_lo / n_kc : jc_lo) * JPS) * JC + wj * (8 * kTM);
            row_run = p.out + kk * p.ldz + static_cast<int64_t>(jb0 + g) * p.ldy + ibase + 2 * t;
        }

        for (int w = jc_lo; w < jc_hi; ++w, ++st) {
            LS_TL(7);  // stage loop top (previous epilogue done)
            const int jc = kChunked ? w / n_kc : w;  // j-chunk of this stage
            const int kc = kChunked ? w % n_kc : 0;  // k-chunk of this stage
            // Fill task(s) for the next unit: loads now, product + TMEM store after the DMMAs.
            int target = next_task;
            if (has_next && !lab_nofill && !SINGLE)
                while (target < n_tasks && fill_stage(target) <= w) ++target;
            const bool fill_now = target > next_task;
            if (fill_now && next_task == 0 && n >= 1)  // this quarter of buffer buf^1 was read by unit n-1
                mbar_wait(as_empty + 4 * (buf ^ 1) + wi, static_cast<unsigned>(((n - 1) >> 1) & 1), p.fault);

            // The first tail rank's A1k (TMEM, fixed for the unit) does not depend on the ring
            // stage: its loads go out before the stage wait, so their latency overlaps the wait
            // and the loop bookkeeping instead of sitting in front of the tile's first DFMA
            // (bit-identical; cfg1 step 2.6155 -> 2.6067 ms, ranks 9-53 at 1024^2 x 256 slabs +0.3 to
            // +1.6%, profiles/r02_pretail_ab.txt).
            constexpr bool kPreTail = !kChunked;
            uint32_t pre0[8], pre1[8];
            if constexpr (kPreTail) {
                tmem::ld_x8_issue(tb + 8 * KD, pre0);
                tmem::ld_x8_issue(tb + 8 * KD + 8, pre1);
            }
            const int slot = st % kNS;
            mbar_wait(full + slot, static_cast<unsigned>((st / kNS) & 1), p.fault);
            LS_TL(4);  // stage landed
            const double* stage = ring + slot * stage_elems;
#pragma unroll 1
            for (int h = 0; h < JPS; ++h) {
                const int jt0 = h * (kTM * WJ) + wj * kTM;  // first j-tile of this warp's tile in the stage
                if (kc == 0) {
#pragma unroll
                for (int m = 0; m < kTM; ++m)
#pragma unroll
                    for (int nn = 0; nn < kTN; ++nn) acc[m][nn][0] = acc[m][nn][1] = 0.0;
#pragma unroll
                for (int qt = 0; qt < n_tail; ++qt) {
                    // Rank remainder (R mod 4) on DFMA before the DMMAs. (Placing it after the
                    // DMMA loop, where it would overlap the accumulator drain, measured 12% slower:
                    // it then lengthens the exposed drain before the epilogue.)
                    const double* tbp = stage + frag_elems + jt0 * 8 * n_tail + qt * 8 + g;
                    double bt[kTM];
#pragma unroll
                    for (int m = 0; m < kTM; ++m) bt[m] = tbp[m * 8 * n_tail];
                    double at0[4], at1[4];
                    if (kPreTail && h == 0 && qt == 0) {
                        tmem::wait_ld(pre0);
                        tmem::wait_ld(pre1);
                        tmem::unpack(pre0, at0);
                        tmem::unpack(pre1, at1);
                    } else {
                        tmem::ld_x8(tb + 8 * KD + 16 * qt, at0);
                        tmem::ld_x8(tb + 8 * KD + 16 * qt + 8, at1);
                    }
                    const double atx[8] = {at0[0], at0[1], at0[2], at0[3], at1[0], at1[1], at1[2], at1[3]};
#pragma unroll
                    for (int nn = 0; nn < kTN; ++nn)
#pragma unroll
                        for (int m = 0; m < kTM; ++m) {
                            acc[m][nn][0] = fma(atx[2 * nn], bt[m], acc[m][nn][0]);
                            acc[m][nn][1] = fma(atx[2 * nn + 1], bt[m], acc[m][nn][1]);
                        }
                }
                }  // kc == 0
                {
                    const double* bsw = stage + jt0 * (KCs * 32) + lane;
                    const int ks0 = kc * KCs;  // first k-step of this stage
                    auto kstep = [&](int ks) {
                        double a[kTM], b[kTN];
                        uint32_t rb[8];
                        tmem::ld_x8_issue(tb + 8 * ks, rb);
#pragma unroll
                        for (int m = 0; m < kTM; ++m) a[m] = bsw[m * (KCs * 32) + (ks - ks0) * 32];
                        tmem::wait_ld(rb);
                        tmem::unpack(rb, b);
#pragma unroll
                        for (int m = 0; m < kTM; ++m)
#pragma unroll
                            for (int nn = 0; nn < kTN; ++nn) dmma_884(acc[m][nn][0], acc[m][nn][1], a[m], b[nn]);
                    };
                    if constexpr (kChunked) {
#pragma unroll
                        for (int c = 0; c < NKC_; ++c) {
                            if (kc == c) {
#pragma unroll
                                for (int ks = c * KC_; ks < ((c + 1) * KC_ < KD_ ? (c + 1) * KC_ : KD_); ++ks) kstep(ks);
                            }
                        }
                    } else if constexpr (KD_ > 0) {
                        // compile-time k-step count: fully unrolled (2.2% faster at cfg1 than the
                        // rolled loop with the same constant bounds)
#pragma unroll
                        for (int ks = 0; ks < (KD_ > 0 ? KD_ : 1); ++ks) kstep(ks);
                    } else {
#pragma unroll 1
                        for (int ks = 0; ks < KD; ++ks) kstep(ks);
                    }
                }
                LS_TL(5);  // DMMAs issued
                if (h == JPS - 1) {
                    // Release the ring slot; the last warp refills it with stage st + kNS.
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence_block();
                        if (atomicAdd(released + slot, 1) == WARPS - 1) {
                            released[slot] = 0;
                            __threadfence_block();
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            if (st + kNS < n_stages) issue(st + kNS);
                        }
                    }
                    // This stage's fill task(s) for the next unit, after the DMMAs were issued (no fill
                    // state stays live across the DMMA loop, which keeps its operand registers free).
                    if (fill_now) {
                        for (; next_task < target; ++next_task) run_task(n + 1, next_task, buf ^ 1);
                        if (next_task == n_tasks) publish(buf ^ 1);
                    }
                }

                LS_TL(6);  // slot released, fill tasks done
                if (kChunked && kc != n_kc - 1) continue;  // the tile continues in the next stage
                // Epilogue: lane owns (j = jb + 8m + g, i = ibase + 8nn + 2t + {0,1}).
                const int jb = (jc * JPS + h) * JC + wj * (8 * kTM);
                double* row;  // = out + kk ldz + (jb + g) ldy + ibase + 2 t
                if constexpr (kRowRun) {
                    row = row_run;
                    row_run += static_cast<int64_t>(JC) * p.ldy;
                }
                if (fast_u && jb + 8 * kTM <= p.N2) {
                    if constexpr (STORE && !kRowRun)
                        row = p.out + kk * p.ldz + static_cast<int64_t>(jb + g) * p.ldy + ibase + 2 * t;
                    // Interior tile (the common case): no per-element bounds or mode checks. Measured
                    // 2.4% of the whole kernel at cfg1 (2.826 -> 2.760 ms).
#pragma unroll
                    for (int m = 0; m < kTM; ++m) {
                        if (lab_nostore) break;
                        if (FUNC) {
                            double sm = 0.0;
#pragma unroll
                            for (int nn = 0; nn < kTN; ++nn) {
                                sm = fma(acc[m][nn][0], r1[nn][0], sm);
                                sm = fma(acc[m][nn][1], r1[nn][1], sm);
                            }
                            fsum = fma(sm, __ldg(p.rho2 + jb + 8 * m + g), fsum);
                        }
                        if (STORE)
#pragma unroll
                            for (int nn = 0; nn < kTN; ++nn)
                                __stcs(reinterpret_cast<double2*>(row + 8 * m * p.ldy + 8 * nn),
                                       make_double2(acc[m][nn][0], acc[m][nn][1]));
                    }
                    continue;
                }
#pragma unroll
                for (int m = 0; m < kTM; ++m) {
                    const int j = jb + 8 * m + g;
                    if (j >= p.N2) continue;
                    if (FUNC) {
                        double sm = 0.0;
#pragma unroll
                        for (int nn = 0; nn < kTN; ++nn) {
                            sm = fma(acc[m][nn][0], r1[nn][0], sm);
                            sm = fma(acc[m][nn][1], r1[nn][1], sm);
                        }
                        fsum = fma(sm, __ldg(p.rho2 + j), fsum);
                    }
                    if (!STORE) continue;
                    double* row = p.out + kk * p.ldz + static_cast<int64_t>(j) * p.ldy;
#pragma unroll
                    for (int nn = 0; nn < kTN; ++nn) {
                        const int i = ibase + 8 * nn + 2 * t;
                        if (i + 1 < p.N1) {
                            if (p.accumulate) {
                                row[i] += acc[m][nn][0];
                                row[i + 1] += acc[m][nn][1];
                            } else if (p.vec_store) {
                                __stcs(reinterpret_cast<double2*>(row + i), make_double2(acc[m][nn][0], acc[m][nn][1]));
                            } else {
                                row[i] = acc[m][nn][0];
                                row[i + 1] = acc[m][nn][1];
                            }
                        } else if (i < p.N1) {
                            row[i] = p.accumulate ? row[i] + acc[m][nn][0] : acc[m][nn][0];
                        }
                    }
                }
            }
        }
        // This warp is done reading A1k buffer buf.
        tmem::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(as_empty + 4 * buf + wi);
        if (SINGLE) {
            if (has_next) {  // the quarter's WJ warps are done with the one buffer: refill it
                mbar_wait(as_empty + wi, static_cast<unsigned>(n & 1), p.fault);
                tmem::fence_after();
                fill_all(unit_of(n + 1), 0);
                publish(0);
            }
        } else if (has_next && (n_tasks == 0 || lab_nofill)) publish(buf ^ 1);  // no fill share (KD = 1, wj = 1): still arrive
        else if (has_next && next_task < n_tasks) {  // tiny units: finish the fill now
            if (next_task == 0 && n >= 1)
                mbar_wait(as_empty + 4 * (buf ^ 1) + wi, static_cast<unsigned>(((n - 1) >> 1) & 1), p.fault);
            for (; next_task < n_tasks; ++next_task) run_task(n + 1, next_task, buf ^ 1);
            publish(buf ^ 1);
        }
        if (FUNC) {
            // Per-warp partials (no CTA barrier): partial[unit * WARPS + warp], fixed-order xor tree.
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, off);
            if (lane == 0) {
                const double part = rn_mul(fsum, p.rho3[p.k0 + kk]);
                double& slot = p.partial[static_cast<int64_t>(unit) * WARPS + warp];
                slot = p.accumulate ? slot + part : part;
            }
        }
    }
    LS_TL(8);  // all units done
    LS_TL_END();
    tmem::fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base_s), "r"(kTmemCols)
                     : "memory");
}

}  // namespace ls_k3
