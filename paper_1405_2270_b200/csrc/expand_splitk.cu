// expand_splitk.cu -- K3 for ranks whose scaled left factor no longer fits tensor memory twice
// (KD 31..120 k-steps, cfg3's rank 328 among them). Included plans: kPlanSplitK in expand.cu.
//
// A 128-row unit of A1k needs 8 columns per k-step in every lane: 656 columns at rank 328,
// more than the 512 an SM has. Here a unit is 64 rows, and its k-steps are split in two halves
// held by different TMEM lane quarters: quarter q = warp & 3 holds rows 32*(q & 1) .. +32 for
// the k-steps of half q >> 1 (8 columns per k-step, single-buffered: 8*KH + 16*n_tail <= 512).
// Each warp therefore computes a partial 32x32 tile over half the rank; the two warps of a pair
// (same rows and j-tiles, different halves) add their partials through shared memory (an
// mbarrier hand-over, the reducing warp alternating per tile so both halves share the
// epilogue) and the reducer stores. The sum is always half 0 + half 1, so results are
// deterministic. A2 streams through a 2-deep TMA ring of stages holding KC k-steps of both
// halves for 16 j-tiles; a tile takes ceil(KH / KC) stages, its accumulators carried across
// them. The next unit's A1k is written after a CTA barrier (single buffer): about 1% of a unit
// at cfg3. The DFMA rank remainder runs on half 1 when KD is odd (its half is a k-step shorter)
// and otherwise on the tile's writer (the reducer has the add and the epilogue); with R mod 4 = 0
// a zero rank still runs there: without it ranks 251 / 256 ran 7% / 6% slower, the effect the
// TMEM kernel's zero rank shows too (r02 A/B at 1024^2 x 64: ranks 250-350 +0.7-7.8%, cfg3 +0.3%).
#include <utility>

#include "expand_tmem.cuh"

namespace ls_k3 {
namespace {

#ifndef LS_SK_KC
#define LS_SK_KC 6
#endif
#ifndef LS_SK_NS
#define LS_SK_NS 2
#endif
constexpr int kSkWarps = 16, kSkIC = 64, kSkJT = 16, kSkNS = LS_SK_NS, kSkKC = LS_SK_KC;
constexpr int kSkRedElems = 8 * 32 * 32;  // 8 warp pairs x 32 lanes x 32 accumulators

// A2 of stage (k-chunk kc, j-chunk jc) at Bp + (kc * n_jc + jc) * stage_elems:
//   [h][jt][kk][lane] = A2(8 (jc JT + jt) + g, 4 (h KH + kc KC + kk) + t)  (zero past the half)
//   then [jt][qt][g]  = A2(8 (jc JT + jt) + g, 4 KD + qt)                  (DFMA tail ranks)
// With S != nullptr the launch also writes the slab-scale table S[k][q] = w_q * C(k, q).
__global__ void pack_splitk_kernel(const double* __restrict__ B, int64_t ldb, int64_t N2, int R, int KD, int KH,
                                   int n_tail, int n_kc, int64_t n_jc, double* __restrict__ Bp,
                                   const double* __restrict__ w, const double* __restrict__ C, int64_t ldc, int64_t k1,
                                   double* __restrict__ S) {
    pdl_wait();
    pdl_trigger();
    const int64_t half = static_cast<int64_t>(kSkJT) * kSkKC * 32;
    const int64_t stage_elems = 2 * half + static_cast<int64_t>(kSkJT) * 8 * n_tail;
    const int64_t total = static_cast<int64_t>(n_kc) * n_jc * stage_elems;
    const int64_t n_scale = k1 * R;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total + n_scale;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (e >= total) {
            const int64_t x = e - total;
            const int64_t k = x / R;
            const int q = static_cast<int>(x - k * R);
            S[x] = rn_mul(w[q], C[k + ldc * q]);
            continue;
        }
        const int64_t st = e / stage_elems;
        const int64_t o = e - st * stage_elems;
        const int kc = static_cast<int>(st / n_jc);
        const int64_t jc = st % n_jc;
        double v = 0.0;
        if (o < 2 * half) {
            const int h = static_cast<int>(o / half);
            const int64_t r = o - h * half;
            const int lane = static_cast<int>(r & 31);
            const int kk = static_cast<int>((r >> 5) % kSkKC);
            const int jt = static_cast<int>((r >> 5) / kSkKC);
            const int kl = kc * kSkKC + kk;
            const int nks = h == 0 ? KH : KD - KH;
            const int64_t j = (jc * kSkJT + jt) * 8 + (lane >> 2);
            const int q = 4 * (h * KH + kl) + (lane & 3);
            if (kl < nks && j < N2 && q < R) v = B[j + ldb * q];
        } else {
            const int64_t r = o - 2 * half;
            const int g = static_cast<int>(r % 8);
            const int qt = static_cast<int>((r / 8) % n_tail);
            const int jt = static_cast<int>(r / (8 * n_tail));
            const int64_t j = (jc * kSkJT + jt) * 8 + g;
            if (j < N2 && 4 * KD + qt < R) v = B[j + ldb * (4 * KD + qt)];
        }
        Bp[e] = v;
    }
}

template <bool STORE, bool FUNC>
__global__ void __launch_bounds__(kSkWarps * 32, 1) expand_splitk_kernel(const ExpandArgs p) {
    constexpr int WARPS = kSkWarps, kTM = 4, kTN = 4, KC = kSkKC;
    const int KD = p.KD, n_tail = p.n_tail;
    const int KH = (KD + 1) / 2;
    const int n_kc = (KH + KC - 1) / KC;
    const int per_unit = static_cast<int>(p.n_jc) * n_kc;
    const int half_elems = kSkJT * KC * 32;
    const int frag_elems = 2 * half_elems;
    const int stage_elems = frag_elems + kSkJT * 8 * n_tail;
    const unsigned stage_bytes = static_cast<unsigned>(stage_elems * sizeof(double));
    const int n_ichunks = static_cast<int>(p.n_ichunks);
    const int n_units = static_cast<int>(p.n_units);

    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);          // [2] A2 stage landed
    uint64_t* ready = full + kSkNS;                               // [8] pair partial written
    int* released = reinterpret_cast<int*>(smem + 16);            // [kSkNS <= 8] warps done with a slot
    uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(smem + 20);
    static_assert(kSkNS + 8 <= 16 && kSkNS <= 8, "header: ring + pair barriers, counters, TMEM base");
    double* red = smem + 32;                                      // [8][32 accumulators][32 lanes]
    double* ring = red + kSkRedElems;                             // [2][stage_elems]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int q = warp & 3, rg = q & 1, kh = q >> 1, wj = warp >> 2;
    const int pair = rg + 2 * wj;
    const int nks = kh == 0 ? KH : KD - KH;  // k-steps of this warp's half

    const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
    const int my_units = n_units > b ? (n_units - 1 - b) / G + 1 : 0;
    const int n_stages = my_units * per_unit;

    auto issue = [&](int st) {
        const int w = st % per_unit;
        const int jc = w / n_kc, kc = w % n_kc;
        const double* src = p.Bp + (static_cast<int64_t>(kc) * p.n_jc + jc) * stage_elems;
        uint64_t* bar = full + (st % kSkNS);
        mbar_arrive_expect_tx(bar, stage_bytes);
        tma_bulk_g2s(ring + (st % kSkNS) * stage_elems, src, stage_bytes, bar);
    };

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_s)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSkNS; ++s) {
            mbar_init(full + s, 1);
            released[s] = 0;
        }
        for (int s = 0; s < 8; ++s) mbar_init(ready + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    pdl_wait();
    const uint32_t tq = *tmem_base_s + (static_cast<uint32_t>(32 * q) << 16);  // this warp's lane quarter
    if (threadIdx.x == 0)
        for (int st = 0; st < kSkNS && st < n_stages; ++st) issue(st);

    // A1k buffers: double-buffered when two fit in 512 columns (KD <= 60), else one. With two,
    // the warps write the next unit's A1k into the idle buffer piece by piece between the
    // current unit's stages; with one, after the unit barrier (exposed, ~1% of a cfg3 unit).
    const int CB = 8 * KH + 16 * n_tail;
    const bool dbuf = 2 * CB <= 512;
    // This warp's fill tasks of a unit: frag task f writes k-step kl = wj + 4 f of its half (the
    // four i-tiles of its rows); then (wj == 0, in the halves that run the tail) one task per
    // tail rank.
    const int n_frag_tasks = nks > wj ? (nks - wj + 3) / 4 : 0;
    // The DFMA rank remainder goes where it balances the pair: with KD odd half 1 (one k-step
    // fewer) always takes it; with KD even the tile's writer does (the reducer has the add and
    // the epilogue). Both halves' quarters then hold the tail columns.
    const bool tail_fixed = (KD & 1) != 0;
    auto tail_here = [&](int tl) { return tail_fixed ? kh == 1 : kh != (tl & 1); };
    const bool holds_tail = tail_fixed ? kh == 1 : true;
    const int n_tasks = n_frag_tasks + ((holds_tail && wj == 0) ? n_tail : 0);
    // Tasks [t0, t1) of unit u into buffer buf. Rounds like Eigen's A1 * scale.asDiagonal().
    auto fill = [&](int u, int buf, int t0, int t1) {
        const int ib = (u % n_ichunks) * kSkIC + 32 * rg;
        const double* S = p.S + (p.k0 + u / n_ichunks) * p.R;
        const uint32_t col = static_cast<uint32_t>(buf * CB);
#pragma unroll 1
        for (int task = t0; task < t1 && task < n_frag_tasks; ++task) {
            const int kl = wj + 4 * task;
            const int qq = 4 * (kh * KH + kl) + t;
            const double sv = qq < p.R ? __ldg(S + qq) : 0.0;
            double v[4];
#pragma unroll
            for (int it = 0; it < 4; ++it) {
                const int i = ib + 8 * it + g;
                v[it] = (i < p.N1 && qq < p.R) ? rn_mul(__ldg(p.A + i + p.lda * qq), sv) : 0.0;
            }
            tmem::st_x8(tq + col + 8 * kl, v);
        }
        for (int task = t0 > n_frag_tasks ? t0 : n_frag_tasks; task < t1 && task < n_tasks; ++task) {
            const int qt = task - n_frag_tasks;
            const int qq = 4 * KD + qt;
            const double sv = qq < p.R ? __ldg(S + qq) : 0.0;
            double v0[4], v1[4];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int i = ib + 8 * (e >> 1) + 2 * t + (e & 1);
                const double x = (i < p.N1 && qq < p.R) ? rn_mul(__ldg(p.A + i + p.lda * qq), sv) : 0.0;
                if (e < 4) v0[e] = x;
                else v1[e - 4] = x;
            }
            tmem::st_x8(tq + col + 8 * KH + 16 * qt, v0);
            tmem::st_x8(tq + col + 8 * KH + 16 * qt + 8, v1);
        }
    };
    if (dbuf && my_units > 0) fill(b, 0, 0, n_tasks);  // prologue: the first unit, all tasks

    double acc[kTM][kTN][2];
    double fsum = 0.0;
    int st = 0, tile = 0;
    for (int n = 0; n < my_units; ++n) {
        const int unit = b + n * G;
        const int ib = (unit % n_ichunks) * kSkIC;
        const int64_t kk = unit / n_ichunks;
        const int buf = dbuf ? (n & 1) : 0;
        // Unit barrier: every warp is past the previous unit (its buffer may be overwritten) and
        // has written its share of this unit's A1k (double-buffered: during the previous unit).
        tmem::wait_st();
        tmem::fence_before();
        __syncthreads();
        tmem::fence_after();
        if (!dbuf) {
            fill(unit, 0, 0, n_tasks);
            tmem::wait_st();
            tmem::fence_before();
            __syncthreads();
            tmem::fence_after();
        }
        const uint32_t tb = tq + static_cast<uint32_t>(buf * CB);
        const bool fill_next = dbuf && n + 1 < my_units;
        double r1[kTN][2];
        if (FUNC) {
            fsum = 0.0;
#pragma unroll
            for (int nn = 0; nn < kTN; ++nn)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = ib + 32 * rg + 8 * nn + 2 * t + e;
                    r1[nn][e] = i < p.N1 ? __ldg(p.rho1 + i) : 0.0;
                }
        }

        for (int w = 0; w < per_unit; ++w, ++st) {
            const int jc = w / n_kc, kc = w % n_kc;
            const int slot = st % kSkNS;
            mbar_wait(full + slot, static_cast<unsigned>((st / kSkNS) & 1), p.fault);
            const double* stage = ring + slot * stage_elems;
            const int jt0 = wj * kTM;
            if (kc == 0) {
#pragma unroll
                for (int m = 0; m < kTM; ++m)
#pragma unroll
                    for (int nn = 0; nn < kTN; ++nn) acc[m][nn][0] = acc[m][nn][1] = 0.0;
                if (tail_here(tile)) {
                    // the rank remainder on DFMA (one half per tile)
                    for (int qt = 0; qt < n_tail; ++qt) {
                        const double* tbp = stage + frag_elems + jt0 * 8 * n_tail + qt * 8 + g;
                        double bt[kTM];
#pragma unroll
                        for (int m = 0; m < kTM; ++m) bt[m] = tbp[m * 8 * n_tail];
                        double at0[4], at1[4];
                        tmem::ld_x8(tb + 8 * KH + 16 * qt, at0);
                        tmem::ld_x8(tb + 8 * KH + 16 * qt + 8, at1);
                        const double atx[8] = {at0[0], at0[1], at0[2], at0[3], at1[0], at1[1], at1[2], at1[3]};
#pragma unroll
                        for (int nn = 0; nn < kTN; ++nn)
#pragma unroll
                            for (int m = 0; m < kTM; ++m) {
                                acc[m][nn][0] = fma(atx[2 * nn], bt[m], acc[m][nn][0]);
                                acc[m][nn][1] = fma(atx[2 * nn + 1], bt[m], acc[m][nn][1]);
                            }
                    }
                }
            }
            {
                const double* bsw = stage + kh * half_elems + jt0 * (KC * 32) + lane;
                const int kl0 = kc * KC;
#pragma unroll
                for (int kk2 = 0; kk2 < KC; ++kk2) {
                    if (kl0 + kk2 >= nks) break;
                    double a[kTM], bb[kTN];
                    uint32_t rb[8];
                    tmem::ld_x8_issue(tb + 8 * (kl0 + kk2), rb);
#pragma unroll
                    for (int m = 0; m < kTM; ++m) a[m] = bsw[m * (KC * 32) + kk2 * 32];
                    tmem::wait_ld(rb);
                    tmem::unpack(rb, bb);
#pragma unroll
                    for (int m = 0; m < kTM; ++m)
#pragma unroll
                        for (int nn = 0; nn < kTN; ++nn) dmma_884(acc[m][nn][0], acc[m][nn][1], a[m], bb[nn]);
                }
            }
            // release the ring slot; the last warp refills it
            __syncwarp();
            // No CTA memory barrier here: it would wait for the warp's outstanding grid stores.
            // The slot's operands were all read into registers (the DMMAs above consumed them),
            // so the counter only has to order those reads before the refill.
            if (lane == 0) {
                if (atomicAdd(released + slot, 1) == WARPS - 1) {
                    released[slot] = 0;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if (st + kSkNS < n_stages) issue(st + kSkNS);
                }
            }
            // double-buffered: this stage's share of the next unit's fill tasks, after the DMMAs
            if (fill_next) {
                const int f0 = (w * n_tasks) / per_unit, f1 = ((w + 1) * n_tasks) / per_unit;
                if (f1 > f0) fill(b + (n + 1) * G, buf ^ 1, f0, f1);
            }
            if (kc != n_kc - 1) continue;

            // Pair reduction: the writer hands its partial over through shared memory; the
            // reducer (alternating with the tile parity) adds it and runs the epilogue.
            double* rb = red + pair * 1024 + lane;
            const bool reducer = (tile & 1) == kh;
            const unsigned phase = static_cast<unsigned>((tile >> 0) & 1);
            ++tile;
            if (!reducer) {
#pragma unroll
                for (int m = 0; m < kTM; ++m)
#pragma unroll
                    for (int nn = 0; nn < kTN; ++nn) {
                        rb[((m * kTN + nn) * 2) * 32] = acc[m][nn][0];
                        rb[((m * kTN + nn) * 2 + 1) * 32] = acc[m][nn][1];
                    }
                __syncwarp();
                if (lane == 0) mbar_arrive(ready + pair);
                continue;
            }
            mbar_wait(ready + pair, phase, p.fault);
            // half 0 + half 1, in that order whichever warp reduces
#pragma unroll
            for (int m = 0; m < kTM; ++m)
#pragma unroll
                for (int nn = 0; nn < kTN; ++nn)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const double other = rb[((m * kTN + nn) * 2 + e) * 32];
                        acc[m][nn][e] = kh == 0 ? acc[m][nn][e] + other : other + acc[m][nn][e];
                    }

            // Epilogue: lane owns (j = jb + 8m + g, i = ibase + 8nn + 2t + {0,1}).
            const int jb = jc * (8 * kSkJT) + wj * (8 * kTM);
            const int ibase = ib + 32 * rg;
            if (ibase + 8 * kTN <= p.N1 && jb + 8 * kTM <= p.N2 && (!STORE || (p.vec_store && !p.accumulate))) {
                double* row = STORE ? p.out + kk * p.ldz + static_cast<int64_t>(jb + g) * p.ldy + ibase + 2 * t : nullptr;
#pragma unroll
                for (int m = 0; m < kTM; ++m) {
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
        if (FUNC) {
            // Per-warp partials: partial[unit * WARPS + warp] (writers of a tile contribute to
            // the reducer's sum only), fixed-order xor tree.
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, off);
            if (lane == 0) {
                const double part = rn_mul(fsum, p.rho3[p.k0 + kk]);
                double& slot = p.partial[static_cast<int64_t>(unit) * WARPS + warp];
                slot = p.accumulate ? slot + part : part;
            }
        }
    }
    tmem::fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base_s), "r"(512) : "memory");
}

}  // namespace

int splitk_smem_bytes(int KD, int n_tail) {
    const int stage = 2 * kSkJT * kSkKC * 32 + kSkJT * 8 * n_tail;
    return static_cast<int>(sizeof(double)) * (32 + kSkRedElems + kSkNS * stage);
}

bool fits_splitk(int KD, int n_tail) {
    const int KH = (KD + 1) / 2;
    return n_tail >= 0 && n_tail <= 2 && KD >= 2 && 8 * KH + 16 * n_tail <= 512 &&
           splitk_smem_bytes(KD, n_tail) + 1024 <= 227 * 1024;
}

int launch_splitk(ExpandArgs& a, bool store, bool func, cudaStream_t s, int sm_count,
                  int (*setup)(const void*, int, size_t, int&)) {
    const int KH = (a.KD + 1) / 2;
    const int n_kc = (KH + kSkKC - 1) / kSkKC;
    a.KC = kSkKC;
    a.n_kc = n_kc;
    a.n_ichunks = ls::ceil_div(a.N1, kSkIC);
    a.n_units = a.n_ichunks * (a.k1 - a.k0);
    a.n_jc = ls::ceil_div(a.N2, 8 * kSkJT);
    a.n_jt = a.n_jc * kSkJT;
    a.split_tail = 0;
    // A zero DFMA rank on the tile's writer (see the kernel) where its TMEM columns fit: at KD 128
    // (rank 512) the halves already fill all 512 columns.
    if (a.n_tail == 0 && fits_splitk(a.KD, 1)) a.n_tail = 1;
    if (a.n_units * a.n_jc * n_kc >= (int64_t(1) << 31) || a.N1 + kSkIC >= (int64_t(1) << 31))
        return ls::fail(LS_EGUARD, "expand: grid too large for one launch (split the slab range)");
    const size_t stage_elems = static_cast<size_t>(2 * kSkJT * kSkKC * 32 + kSkJT * 8 * a.n_tail);
    const size_t bp_elems = static_cast<size_t>(n_kc) * a.n_jc * stage_elems;
    const size_t s_elems = static_cast<size_t>(a.k1) * a.R;
    ls::ensure_pool();
    ls::AsyncScratch scratch(s);  // freed on every exit path
    LS_CUDA(scratch.alloc((bp_elems + s_elems) * sizeof(double)));
    double* bp = scratch.as<double>();
    a.S = bp + bp_elems;
    const int64_t pb = std::min<int64_t>(ls::ceil_div(static_cast<int64_t>(bp_elems + s_elems), 256), 4096);
    LS_CUDA(ls::launch_pdl(pack_splitk_kernel, dim3((unsigned)pb), dim3(256), 0, s, a.B, a.ldb, a.N2, a.R, a.KD, KH,
                           a.n_tail, n_kc, a.n_jc, bp, a.w, a.C, a.ldc, a.k1, const_cast<double*>(a.S)));
    LS_LAUNCHED("pack_splitk_kernel");
    a.Bp = bp;
    KernelFn kern = store && func ? expand_splitk_kernel<true, true>
                    : store       ? expand_splitk_kernel<true, false>
                                  : expand_splitk_kernel<false, true>;
    const size_t smem = static_cast<size_t>(splitk_smem_bytes(a.KD, a.n_tail));
    int per_sm = 0;
    if (const int rc = setup(reinterpret_cast<const void*>(kern), kSkWarps * 32, smem, per_sm)) return rc;
    const int64_t grid = std::min<int64_t>(a.n_units, sm_count);
    if (grid > 0) {
        LS_CUDA(ls::launch_pdl(kern, dim3((unsigned)grid), dim3(kSkWarps * 32), smem, s, a));
        LS_LAUNCHED("expand_splitk_kernel");
    }
    return LS_OK;
}

}  // namespace ls_k3
