// expand.cu -- K3: rank-R expansion of a canonical tensor onto the N1 x N2 x N3
// grid, FP64 on the tensor cores (DMMA, mma.sync.m8n8k4.f64), operands staged
// by TMA bulk copies into a shared-memory ring.
//
// Reference: densify (canonical.hpp:251-266) -> detail::densify_slab
// (canonical.hpp:241-246): slab k = A1 * diag(w .* A3(k,:)) * A2^T, an Eigen
// GEMM with inner dimension R. Each slab is the same GEMM here:
//
//   V(i, j, k) = sum_q A1k(i, q) * A2(j, q),   A1k(i, q) = A1(i, q) * (w_q * A3(k, q))
//
// (the scaled left factor rounds exactly as Eigen's A1 * scale.asDiagonal()).
// Measured on B200 (profiles/r01_fp64_peak_microbench.jsonl): DMMA m8n8k4
// sustains 37.07 TFLOP/s = 64 FMA/clk/SM; DFMA shares the same pipe. At
// R = 41 the expansion is 10.25 FLOP per output byte, above the HBM ridge
// (~5.6 FLOP/B), so the kernel is FP64-pipe-bound. The inner-loop study
// (tools/lab/loop_lab.cu) showed DMMA at 37 TF/s with register or shared
// operands but only 32-34 TF/s when one operand comes from L1/L2, so both
// operands are fed from shared memory:
//
//  * A1k for the CTA's i-chunk (IC rows x all ranks) is scaled once per
//    work unit (i-chunk, slab k) into shared memory in MMA-fragment order;
//  * A2 is pre-packed once per call into fragment order (pack_b_kernel) so
//    every pipeline stage -- JT j-tiles x KC k-steps -- is one contiguous
//    block that a single thread moves with cp.async.bulk (TMA) into an
//    NS-deep ring, completion signalled on an mbarrier (expect_tx);
//  * warps load both fragments straight from shared memory per k-step, each
//    owning TM x TN independent 8x8 accumulators (M = j, N = i, K = q), and
//    store straight from the accumulator fragments: lane (g, t) holds
//    V(i = 8n + 2t + {0,1}, j = 8m + g), a 16-byte aligned pair of the
//    i-fastest grid, written with streaming stores.
//  * a rank remainder of 1-2 (R mod 4) runs on DFMA instead of a zero-padded
//    4-rank DMMA step.
// No CTA barrier per stage: each warp releases a ring slot after its last
// DMMA of the stage and the last one refills it. Units are spread over a
// persistent grid (CTAs per SM x SM count). Plans by rank (plan_for):
//   * ranks <= 121: expand_tmem.cuh, A1k double-buffered in tensor memory (8 warps x 2 CTAs
//     or 16 warps x 1 CTA per SM; instantiated in expand_tmem8.cu / expand_tmem16.cu);
//   * ranks >= 164 (KD <= 120): expand_splitk.cu, A1k k-halves in different TMEM lane
//     quarters with a pair reduction;
//   * otherwise this file's expand_dmma_kernel with A1k in shared memory;
// k3.cuh holds the definitions they share.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <utility>

#include "common.cuh"
#include "k3.cuh"

namespace {

using namespace ls_k3;


// A2 packed so that every pipeline stage (k-chunk kc, j-chunk jc) is one contiguous block of
// stage_elems = JT*KC*32 + JT*8*n_tail doubles at Bp + (kc * n_jc + jc) * stage_elems:
//   [jt][kk][lane] = A2(8 (jc JT + jt) + g, 4 (kc KC + kk) + t)   (MMA A-fragment order)
//   then [jt][qt][g] = A2(8 (jc JT + jt) + g, 4 KD + qt)          (DFMA tail ranks)
// zero padded outside the matrix.
// With S != nullptr the same launch also writes the TMEM variant's slab-scale table
// S[k][q] = w_q * C(k, q) for k in [0, k1) (canonical.hpp:244), after the packed stages.
__global__ void pack_b_kernel(const double* __restrict__ B, int64_t ldb, int64_t N2, int R, int KD, int n_tail,
                              int KC, int n_kc, int JT, int64_t n_jc, double* __restrict__ Bp,
                              const double* __restrict__ w, const double* __restrict__ C, int64_t ldc, int64_t k1,
                              double* __restrict__ S) {
    pdl_wait();  // B, C, w may come from the preceding assembly / generator launches
    pdl_trigger();
    const int64_t frag = static_cast<int64_t>(JT) * KC * 32;
    const int64_t stage_elems = frag + static_cast<int64_t>(JT) * 8 * n_tail;
    const int64_t total = static_cast<int64_t>(n_kc) * n_jc * stage_elems;
    const int64_t n_scale = S ? k1 * R : 0;
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
        if (o < frag) {
            const int lane = static_cast<int>(o & 31);
            const int kk = static_cast<int>((o >> 5) % KC);
            const int jt = static_cast<int>((o >> 5) / KC);
            const int ks = kc * KC + kk;
            const int64_t j = (jc * JT + jt) * 8 + (lane >> 2);
            const int q = ks * 4 + (lane & 3);
            if (j < N2 && ks < KD && q < R) v = B[j + ldb * q];
        } else {
            const int64_t r = o - frag;
            const int g = static_cast<int>(r % 8);
            const int qt = static_cast<int>((r / 8) % n_tail);
            const int jt = static_cast<int>(r / (8 * n_tail));
            const int64_t j = (jc * JT + jt) * 8 + g;
            if (j < N2 && 4 * KD + qt < R) v = B[j + ldb * (4 * KD + qt)];
        }
        Bp[e] = v;
    }
}

// CTA tile: WARPS warps as WI (along i) x WJ (along j); each warp owns TM x TN 8x8
// accumulator tiles; MINB CTAs per SM (register budget 64K / (MINB * 32 * WARPS)).
template <int WARPS_, int WI_, int TM_, int TN_, int MINB_, int NS_ = 3>
struct Tile {
    static constexpr int NS = NS_;            // stages in the A2 ring
    static constexpr int WARPS = WARPS_;
    static constexpr int WI = WI_;
    static constexpr int TM = TM_;            // j tiles (of 8) per warp
    static constexpr int TN = TN_;            // i tiles (of 8) per warp
    static constexpr int MINB = MINB_;
    static constexpr int WJ = WARPS / WI;
    static constexpr int IC = 8 * TN * WI;    // i rows per unit
    static constexpr int JT = TM * WJ;        // j tiles (of 8) per stage
    static constexpr int JC = 8 * JT;        // j columns per stage
};

template <class T, bool STORE, bool FUNC>
__global__ void __launch_bounds__(T::WARPS * 32, T::MINB)
expand_dmma_kernel(const ExpandArgs p) {
    pdl_wait();  // the packed A2 and the factors come from the preceding launches
    constexpr int WARPS = T::WARPS;
    constexpr int WI = T::WI;
    constexpr int kTM = T::TM;
    constexpr int kTN = T::TN;
    constexpr int kThreads = WARPS * 32;
    constexpr int IC = T::IC;
    constexpr int JT = T::JT;
    constexpr int kNS = T::NS;
    // All counters are 32-bit (launch() checks the ranges); only addresses are 64-bit.
    const int KD = p.KD, KC = p.KC, n_tail = p.n_tail, n_kc = p.n_kc;
    const int frag_elems = JT * KC * 32;
    const int stage_elems = frag_elems + JT * 8 * n_tail;
    const int rpad = 4 * KD + n_tail;
    const int n_ichunks = static_cast<int>(p.n_ichunks);
    const int n_units = static_cast<int>(p.n_units);

    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);           // [kNS] mbarriers: stage landed
    int* released = reinterpret_cast<int*>(smem + 8);              // [kNS] warps done with a slot
    double* ring = smem + 16;                                      // [kNS][stage_elems]
    double* as = ring + kNS * stage_elems;                         // [IC/8][KD][32]
    double* tail = as + IC * KD * 4;                               // [n_tail][IC]
    double* scale = tail + IC * n_tail;                            // [2][rpad] (unit parity)
    double* r1s = scale + 2 * rpad;                                // [IC] rho1 of the unit (FUNC)
    __shared__ double red[WARPS];

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2;
    const int t = lane & 3;
    const int wi = warp % WI;
    const int wj = warp / WI;

    // This CTA's stage sequence: units u = blockIdx.x + n*gridDim.x, each n_jc * n_kc stages.
    const int my_units = n_units > static_cast<int>(blockIdx.x)
                             ? (n_units - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                             : 0;
    const int per_unit = static_cast<int>(p.n_jc) * n_kc;
    const int n_stages = my_units * per_unit;
    const unsigned stage_bytes = static_cast<unsigned>(stage_elems * sizeof(double));

    auto issue = [&](int st) {
        const int w = st % per_unit;
        const int c = w / n_kc;
        const int kcs = w - c * n_kc;
        const double* src = p.Bp + (static_cast<int64_t>(kcs) * p.n_jc + c) * stage_elems;
        uint64_t* bar = full + (st % kNS);
        mbar_arrive_expect_tx(bar, stage_bytes);
        tma_bulk_g2s(ring + (st % kNS) * stage_elems, src, stage_bytes, bar);
    };
    // scale_q = w_q * A3(k, q) for the unit's slab (canonical.hpp:244)
    auto compute_scale = [&](int u, double* dst) {
        const int64_t k = p.k0 + u / n_ichunks;
        for (int q = threadIdx.x; q < rpad; q += kThreads) dst[q] = q < p.R ? rn_mul(p.w[q], p.C[k + p.ldc * q]) : 0.0;
    };

    if (threadIdx.x == 0) {
        for (int b = 0; b < kNS; ++b) {
            mbar_init(full + b, 1);
            released[b] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (my_units > 0) compute_scale(blockIdx.x, scale);
    __syncthreads();
    if (threadIdx.x == 0)
        for (int st = 0; st < kNS && st < n_stages; ++st) issue(st);

    double acc[kTM][kTN][2];
    double fsum = 0.0;
    int unit = blockIdx.x;
    int parity = 0;  // unit parity selects the scale buffer
    int within = 0, jc = 0, kc = 0;
    int ib = (unit % n_ichunks) * IC;  // first i row of the unit
    int kk = unit / n_ichunks;         // slab offset within [k0, k1)

    for (int st = 0; st < n_stages; ++st) {
        if (within == 0 && !((p.debug & 2) && st > 0)) {
            __syncthreads();  // every warp finished the previous unit: as/tail are free
            // New unit: A1k(i, q) = A1(i, q) * scale_q (Eigen's A1 * scale.asDiagonal()), fragment
            // order: lane (g, t) of (i-tile it, k-step ks) <-> A1k(8 it + g, 4 ks + t).
            const double* sc = scale + parity * rpad;
            const int pairs = (IC / 8) * KD;
            int it = warp / KD, ks = warp - (warp / KD) * KD;
#pragma unroll 4
            for (int x = warp; x < pairs; x += WARPS) {
                const int i = ib + it * 8 + g;
                const int q = ks * 4 + t;
                as[x * 32 + lane] = (i < p.N1 && q < p.R) ? rn_mul(__ldg(p.A + i + p.lda * q), sc[q]) : 0.0;
                ks += WARPS;
                while (ks >= KD) {
                    ks -= KD;
                    ++it;
                }
            }
            for (int e = threadIdx.x; e < n_tail * IC; e += kThreads) {
                const int q = 4 * KD + e / IC;
                const int i = ib + e % IC;
                tail[e] = (i < p.N1 && q < p.R) ? rn_mul(__ldg(p.A + i + p.lda * q), sc[q]) : 0.0;
            }
            if (FUNC) {
                fsum = 0.0;
                for (int e = threadIdx.x; e < IC; e += kThreads) r1s[e] = ib + e < p.N1 ? p.rho1[ib + e] : 0.0;
            }
            __syncthreads();
        }
        if (within == per_unit - 1 && unit + static_cast<int>(gridDim.x) < n_units && !(p.debug & 8))
            compute_scale(unit + gridDim.x, scale + (parity ^ 1) * rpad);  // read after the unit barrier

        const int slot = st % kNS;
        mbar_wait(full + slot, static_cast<unsigned>((st / kNS) & 1), p.fault);
        const double* stage = ring + slot * stage_elems;
        if (kc == 0) {
#pragma unroll
            for (int m = 0; m < kTM; ++m)
#pragma unroll
                for (int n = 0; n < kTN; ++n) acc[m][n][0] = acc[m][n][1] = 0.0;
            // Rank remainder (R mod 4 = 1, 2) on DFMA, issued first so it never waits on DMMA
            // results: lane (g, t) owns V(i = 8n + 2t + {0,1}, j = 8m + g) of the warp tile.
            const double* tb = stage + frag_elems + (wj * kTM) * (8 * n_tail) + g;
            for (int qt = 0; qt < ((p.debug & 4) ? 0 : n_tail); ++qt) {
                double bt[kTM];
#pragma unroll
                for (int m = 0; m < kTM; ++m) bt[m] = tb[m * (8 * n_tail) + qt * 8];
#pragma unroll
                for (int n = 0; n < kTN; ++n) {
                    const double2 at =
                        *reinterpret_cast<const double2*>(tail + qt * IC + wi * (8 * kTN) + 8 * n + 2 * t);
#pragma unroll
                    for (int m = 0; m < kTM; ++m) {
                        acc[m][n][0] = fma(at.x, bt[m], acc[m][n][0]);
                        acc[m][n][1] = fma(at.y, bt[m], acc[m][n][1]);
                    }
                }
            }
        }

        {
            const double* bsw = stage + (wj * kTM) * (KC * 32) + lane;
            const double* aw = as + (wi * kTN) * (KD * 32) + kc * KC * 32 + lane;
            const int ks_len = min(KC, KD - kc * KC);
            // Operands straight from shared memory (loop_lab: 36.9 TF/s at 4x4 without prefetch);
            // the other warps of the SM sub-partition cover the LDS latency.
#pragma unroll 1
            for (int ks = 0; ks < ks_len; ++ks) {
                double a[kTM], b[kTN];
#pragma unroll
                for (int m = 0; m < kTM; ++m) a[m] = bsw[m * (KC * 32) + ks * 32];
#pragma unroll
                for (int n = 0; n < kTN; ++n) b[n] = aw[n * (KD * 32) + ks * 32];
#pragma unroll
                for (int m = 0; m < kTM; ++m)
#pragma unroll
                    for (int n = 0; n < kTN; ++n) dmma_884(acc[m][n][0], acc[m][n][1], a[m], b[n]);
            }
        }
        // Release the ring slot. Every LDS of this stage has completed (its result fed a DMMA
        // already issued); the last warp to release refills the slot with stage st + kNS.
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

        if (kc == n_kc - 1 && STORE && !FUNC && p.vec_store && !p.accumulate && !p.debug &&
            ib + wi * (8 * kTN) + 8 * kTN <= p.N1 && jc * T::JC + wj * (8 * kTM) + 8 * kTM <= p.N2) {
            // Interior tile: no per-element bounds or mode checks (as in the TMEM kernel).
            double* row = p.out + kk * p.ldz + static_cast<int64_t>(jc * T::JC + wj * (8 * kTM) + g) * p.ldy + ib +
                          wi * (8 * kTN) + 2 * t;
#pragma unroll
            for (int m = 0; m < kTM; ++m)
#pragma unroll
                for (int n = 0; n < kTN; ++n)
                    __stcs(reinterpret_cast<double2*>(row + 8 * m * p.ldy + 8 * n), make_double2(acc[m][n][0], acc[m][n][1]));
        } else if (kc == n_kc - 1) {
            const int jb = jc * T::JC + wj * (8 * kTM);
            const int ibase = ib + wi * (8 * kTN);
#pragma unroll
            for (int m = 0; m < kTM; ++m) {
                const int j = jb + 8 * m + g;
                if (j >= p.N2) continue;
                if (p.debug & 16) continue;
                if (p.debug & 1) {
                    double sx = 0.0;
#pragma unroll
                    for (int n = 0; n < kTN; ++n) sx += acc[m][n][0] + acc[m][n][1];
                    if (sx == 1.2345) p.out[0] = sx;
                    continue;
                }
                if (FUNC) {
                    // rho-weighted partial: rows of the tile against rho1 (shared), then rho2(j).
                    double sm = 0.0;
#pragma unroll
                    for (int n = 0; n < kTN; ++n) {
                        const double2 r = *reinterpret_cast<const double2*>(r1s + wi * (8 * kTN) + 8 * n + 2 * t);
                        sm = fma(acc[m][n][0], r.x, sm);
                        sm = fma(acc[m][n][1], r.y, sm);
                    }
                    fsum = fma(sm, p.rho2[j], fsum);
                }
                if (!STORE) continue;
                double* row = p.out + kk * p.ldz + static_cast<int64_t>(j) * p.ldy;
#pragma unroll
                for (int n = 0; n < kTN; ++n) {
                    const int i = ibase + 8 * n + 2 * t;
                    if (i + 1 < p.N1) {
                        if (p.accumulate) {
                            row[i] += acc[m][n][0];
                            row[i + 1] += acc[m][n][1];
                        } else if (p.vec_store) {
                            __stcs(reinterpret_cast<double2*>(row + i), make_double2(acc[m][n][0], acc[m][n][1]));
                        } else {
                            row[i] = acc[m][n][0];
                            row[i + 1] = acc[m][n][1];
                        }
                    } else if (i < p.N1) {
                        row[i] = p.accumulate ? row[i] + acc[m][n][0] : acc[m][n][0];
                    }
                }
            }
        }

        // advance (within, jc, kc); a finished unit moves on to the CTA's next unit
        if (++kc == n_kc) {
            kc = 0;
            ++jc;
        }
        if (++within == per_unit) {
            if (FUNC) {
                // Fixed-order reduction: lanes by xor-tree, then warps in index order.
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, off);
                if (lane == 0) red[warp] = fsum;
                __syncthreads();
                if (threadIdx.x == 0) {
                    double sum = 0.0;
                    for (int wv = 0; wv < WARPS; ++wv) sum += red[wv];
                    const double part = rn_mul(sum, p.rho3[p.k0 + kk]);
                    p.partial[unit] = p.accumulate ? p.partial[unit] + part : part;
                }
            }
            within = 0;
            jc = 0;
            unit += gridDim.x;
            parity ^= 1;
            ib = (unit % n_ichunks) * IC;
            kk = unit / n_ichunks;
        }
    }
}


__global__ void sum_partials_kernel(const double* __restrict__ part, int64_t count,
                                    double* __restrict__ out) {
    // One block, fixed order: thread-strided partial sums, then a fixed tree.
    __shared__ double sh[1024];
    double s = 0.0;
    for (int64_t u = threadIdx.x; u < count; u += blockDim.x) s += part[u];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = sh[0];
}

// DMMA k-steps and DFMA tail for rank R: a remainder of 1 or 2 ranks is cheaper on DFMA
// (2 FMA-lanes per output each) than a zero-padded 4-rank DMMA step.
void split_rank(int R, int& KD, int& n_tail) {
    KD = R / 4;
    n_tail = R % 4;
    if (n_tail == 3) {
        KD += 1;
        n_tail = 0;
    }
    if (KD == 0) {  // R <= 2: one zero-padded DMMA step
        KD = 1;
        n_tail = 0;
    }
}

// Shared-memory budget per SM (B200: 228 KB, 227 KB per CTA opt-in, 1 KB reserved per CTA).
constexpr size_t kSmemPerSM = 228 * 1024;

template <class T>
size_t smem_bytes(int KD, int KC, int n_tail) {
    const size_t stage = static_cast<size_t>(T::JT) * KC * 32 + static_cast<size_t>(T::JT) * 8 * n_tail;
    return sizeof(double) * (16 + T::NS * stage + static_cast<size_t>(T::IC) * KD * 4 +
                             static_cast<size_t>(T::IC) * n_tail + 2 * (4 * static_cast<size_t>(KD) + n_tail) +
                             static_cast<size_t>(T::IC));
}

// Tile plans, best first.
using TileWide = Tile<8, 4, 4, 4, 2>;    // 128-row i-chunk, 32x32 warp tiles, 2 CTAs/SM
using TileWide3 = Tile<8, 4, 2, 4, 3>;   // same i-chunk, 16x32 warp tiles, 3 CTAs/SM (24 warps/SM)
using TileMid = Tile<4, 2, 4, 4, 2>;     // 64-row i-chunk (larger ranks)
using TileNarrow = Tile<4, 1, 4, 4, 2>;  // 32-row i-chunk (largest ranks)
using TileLR1 = Tile<8, 1, 4, 4, 1>;     // large ranks: 32-row i-chunk, 256-column stages, 1 CTA/SM
using TileLR2 = Tile<8, 2, 4, 4, 1>;     // large ranks: 64-row i-chunk, 128-column stages, 1 CTA/SM
using TileLR1b = Tile<8, 1, 4, 4, 1, 2>; // as TileLR1 with a 2-deep ring of longer stages
using TileLR16 = Tile<16, 1, 4, 4, 1, 2>; // large ranks: 16 warps (4 per SM sub-partition), 512-column stages
using TileTmem16 = Tile<16, 4, 4, 4, 1, 2>; // TMEM variant, 1 CTA/SM: 128-row i-chunk, 128-column stages

struct Plan {
    int id;  // see plan_for; 20 / 21 = A1k in TMEM (8 warps x 2 CTAs / 16 warps x 1 CTA per SM)
    int KC;
    int ic;
    int pad = 0;  // 1: run a 2-rank remainder as one zero-padded k-step (TMEM plans have a 1-rank tail)
};

constexpr int kPlanTmem = 20, kPlanTmem16 = 21, kPlanSplitK = 22, kPlanTmem16S = 23;
// TMEM variant shape (ring depth, j-chunks per stage); LS_EXPAND_TMEM=<ns><jps> overrides.
struct TmemShape {
    int ns, jps;
};
inline TmemShape tmem_shape() {
    TmemShape sh{4, 1};
    if (const char* e = ls::dev_knob("LS_EXPAND_TMEM")) {
        const int v = std::atoi(e);
        sh = {v / 10, v % 10};
    }
    return sh;
}

// The TMEM variants: whole rank per stage, A1k double-buffered in TMEM (at most one tail
// rank); shared memory holds the A2 ring and the fill staging.
//  * 8 warps, 2 CTAs/SM, 256 columns each: KD <= 14 (ranks up to 57);
//  * 16 warps, 1 CTA/SM, 512 columns, 2-deep ring of 16-j-tile stages: as far as the ring fits
//    (ranks up to ~85).
// The TMEM kernel always runs one DFMA rank per tile: a zero rank when R mod 4 is 0 or 3.
// Measured: rank 40 took 1.514 ms and rank 41 (with its real DFMA rank) 1.438 ms at
// 1024^2 x 512 slabs; with the zero rank rank 40 runs like rank 41. The same holds at ranks
// 44/45 and 48/49.
inline int tmem_tail(int n_tail) { return n_tail == 0 ? 1 : n_tail; }
// The 8-warp shape also takes a 2-rank remainder as two DFMA ranks (the 16-warp one pads it).
bool fits_tmem_shape(int KD, int n_tail, TmemShape sh) {
    n_tail = tmem_tail(n_tail);
    if (n_tail > 2 || 2 * (8 * KD + 16 * n_tail) > tmem_cols(8)) return false;
    const size_t jt = static_cast<size_t>(TileWide::JT) * sh.jps;
    const size_t stage = jt * KD * 32 + jt * 8 * n_tail;
    return 2 * (sizeof(double) * (kTmemHdr + tmem_stg_elems(8) + sh.ns * stage) + 1024) <= kSmemPerSM;
}
// Ring depth 4 where it fits (ranks up to 45), else 3 (up to 57); LS_EXPAND_TMEM overrides.
TmemShape tmem_shape_for(int KD, int n_tail) {
    if (ls::dev_knob("LS_EXPAND_TMEM")) return tmem_shape();
    return fits_tmem_shape(KD, n_tail, {4, 1}) ? TmemShape{4, 1} : TmemShape{3, 1};
}
bool fits_tmem(int KD, int n_tail) { return fits_tmem_shape(KD, n_tail, tmem_shape_for(KD, n_tail)); }
// k-steps per stage of the 16-warp TMEM plan: the whole rank where the 2-deep ring holds it
// (KD <= 23), else two stages of ceil(KD / 2) (KD 24..30); 0 if it does not fit at all.
int tmem16_stage_ks(int KD, int n_tail) {
    n_tail = tmem_tail(n_tail);
    if (n_tail > 1 || 2 * (8 * KD + 16 * n_tail) > tmem_cols(16)) return 0;
    const size_t jt = TileTmem16::JT;
    for (int kc : {KD, (KD + 1) / 2}) {
        const size_t stage = jt * kc * 32 + jt * 8 * n_tail;
        if (sizeof(double) * (kTmemHdr + tmem_stg_elems(16) + TileTmem16::NS * stage) + 1024 <= kSmemPerSM) return kc;
        if (KD > 30) break;  // chunked instantiations exist for KD 24..30 only
    }
    return 0;
}
bool fits_tmem16(int KD, int n_tail) { return tmem16_stage_ks(KD, n_tail) > 0; }
// Single-buffer 16-warp TMEM plan (expand_tmem16s.cuh): KD 31..62 with one DFMA rank; one A1k
// buffer of 8 KD + 16 <= 512 columns, NKC stages of KC k-steps per tile in a 2-deep ring.
bool fits_tmem16s(int KD, int n_tail) {
    if (tmem_tail(n_tail) != 1 || KD < 31 || KD > 62) return false;
    const size_t jt = TileTmem16::JT, kc = static_cast<size_t>(tmem16s_kc(KD));
    const size_t stage = jt * kc * 32 + jt * 8;
    return sizeof(double) * (kTmemHdr + tmem_stg_elems(16) + TileTmem16::NS * stage) + 1024 <= kSmemPerSM &&
           8 * KD + 16 <= tmem_cols(16);
}

template <class T>
bool fits(int KD, int KC, int n_tail) {
    return static_cast<size_t>(T::MINB) * (smem_bytes<T>(KD, KC, n_tail) + 1024) <= kSmemPerSM;
}

bool plan_for(int KD, int n_tail, Plan& out) {
    int force = -1;
    if (const char* e = ls::dev_knob("LS_EXPAND_PLAN")) force = std::atoi(e);  // development A/B knob
    struct Cand {
        int id, KC;
    };
    // Measured on B200 (tools/profile_expand.py, tools/profile_rank.py, tools/profile_rank_sweep.py):
    // the TMEM plan for the BASELINE rank 41 (31.2 TF/s); the 16-warp TMEM plan up to rank ~93
    // (28-32 TF/s at 1024^2 x 512); plan 9 for ranks beyond it (cfg3 rank 328:
    // 31.3 TF/s, against 28.7 for the 8-warp plan 8 and 20.3 for the 4-warp plan 3; 16-warp tiles
    // with a 64-row i-chunk (29.0) or 16-row warp tiles (no fit) were slower).
    // Up to KD 14 the 2-CTA TileWide with 8-k-step stages beats the 16-warp plan 9 (rank 46:
    // 27.1 vs 22.0 TF/s); beyond it plan 9 wins (rank 123: 26.4 vs 24.2).
    const Cand small_r[] = {{kPlanTmem, 0}, {kPlanTmem16, 0}, {kPlanTmem16S, 0}, {kPlanSplitK, 0}, {0, 0}, {0, 8}, {9, 4}, {8, 8}, {6, 5}, {7, 4}, {2, 4}, {3, 4}, {3, 2}, {1, 0}};
    const Cand large_r[] = {{kPlanTmem, 0}, {kPlanTmem16, 0}, {kPlanTmem16S, 0}, {kPlanSplitK, 0}, {0, 0}, {9, 4}, {0, 8}, {8, 8}, {6, 5}, {7, 4}, {2, 4}, {3, 4}, {3, 2}, {1, 0}};
    for (const Cand& c : KD <= 14 ? small_r : large_r) {
        if (force >= 0 && c.id != force) continue;
        const int KC = c.KC == 0 ? KD : std::min(KD, c.KC);
        bool ok = false;
        int ic = 0;
        switch (c.id) {
            case 0: ok = fits<TileWide>(KD, KC, n_tail); ic = TileWide::IC; break;
            case 1: ok = fits<TileWide3>(KD, KC, n_tail); ic = TileWide3::IC; break;
            case 2: ok = fits<TileMid>(KD, KC, n_tail); ic = TileMid::IC; break;
            case 6: ok = fits<TileLR1>(KD, KC, n_tail); ic = TileLR1::IC; break;
            case 7: ok = fits<TileLR2>(KD, KC, n_tail); ic = TileLR2::IC; break;
            case 8: ok = fits<TileLR1b>(KD, KC, n_tail); ic = TileLR1b::IC; break;
            case 9: ok = fits<TileLR16>(KD, KC, n_tail); ic = TileLR16::IC; break;
            case kPlanTmem: ok = fits_tmem(KD, n_tail); ic = TileWide::IC; break;
            // The 16-warp TMEM plan takes a 2-rank remainder as one more zero-padded k-step: at
            // ranks 58-90 that beats plan 9 by 12-22% (tools/profile_rank_sweep.py, 512 slabs).
            // For the 8-warp plan the padding costs what it gains (rank 42: 27.8 vs 28.6 TF/s
            // for plan 0 with a 2-rank DFMA tail), so it keeps n_tail <= 1.
            // Below KD 15 it only takes ranks the 8-warp TMEM plan cannot (rank 54: a 2-rank
            // remainder at KD 13 overflows 256 columns); the 8-warp plan is faster at ranks 33-45.
            case kPlanTmem16:
                ok = (force == kPlanTmem16 || KD + (n_tail == 2) > 14 || !fits_tmem(KD, n_tail)) &&
                     fits_tmem16(KD + (n_tail == 2), n_tail == 2 ? 0 : n_tail);
                ic = TileTmem16::IC;
                break;
            // Beyond the double-buffered TMEM plans. At ranks 122-160 the smem plan 9 and split-K
            // trade places within 2% on 1024^2 x 256 slabs (the split-K unit's exposed A1k fill
            // weighs more there); from rank 164 (KD 41) on split-K wins: 164-172 by 1-3%, rank 246
            // 29.7 vs 28.9 TF/s, cfg3's 328 32.9 vs 30.8.
            // Ranks 122..249 (KD 31..62): the single-buffer 16-warp TMEM plan (31.9-33.7 TF/s at 1024^2 x
            // 512 slabs against 26.0-29.8 for split-K and the smem plan 9 it replaces).
            case kPlanTmem16S:
                ok = fits_tmem16s(KD + (n_tail == 2), n_tail == 2 ? 0 : n_tail);
                ic = TileTmem16::IC;
                break;
            case kPlanSplitK: ok = (force == kPlanSplitK || KD >= 41) && fits_splitk(KD, n_tail); ic = 64; break;
            default: ok = fits<TileNarrow>(KD, KC, n_tail); ic = TileNarrow::IC; break;
        }
        if (ok) {
            const int pad = (c.id == kPlanTmem16 || c.id == kPlanTmem16S) && n_tail == 2;
            out = {c.id,
                   c.id == kPlanTmem16    ? tmem16_stage_ks(KD + pad, pad ? 0 : n_tail)
                   : c.id == kPlanTmem16S ? tmem16s_kc(KD + pad)
                                          : KC + pad,
                   ic, pad};
            if (const char* e = ls::dev_knob("LS_EXPAND_KC")) out.KC = std::max(1, std::min(KD, std::atoi(e)));
            return true;
        }
    }
    return false;
}

// Per-(kernel, device) launch setup, cached: the attribute calls and the occupancy query cost
// microseconds each, which dominated small expansions (25 us per 128^3 call before). The
// dynamic shared-memory limit is raised to the device maximum once; occupancy is cached per
// shared-memory size.
int kernel_setup(const void* kern, int threads, size_t smem, int& per_sm) {
    static std::mutex m;
    static std::map<std::tuple<const void*, int>, bool> configured;
    static std::map<std::tuple<const void*, int, size_t>, int> occupancy;
    int dev = 0;
    LS_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(m);
    auto ko = occupancy.find({kern, dev, smem});
    if (ko != occupancy.end()) {
        per_sm = ko->second;
        return LS_OK;
    }
    if (!configured[{kern, dev}]) {
        int optin = 0;
        cudaFuncAttributes fa{};
        LS_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        LS_CUDA(cudaFuncGetAttributes(&fa, kern));
        LS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     optin - static_cast<int>(fa.sharedSizeBytes)));
        LS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared));
        configured[{kern, dev}] = true;
    }
    LS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
    occupancy[{kern, dev, smem}] = per_sm;
    return LS_OK;
}

template <class T, bool STORE, bool FUNC, bool TMEM = false>
int launch(ExpandArgs& a, cudaStream_t s) {
    const TmemShape sh =
        TMEM ? (T::WARPS == 16 ? TmemShape{T::NS, 1} : tmem_shape_for(a.KD, a.n_tail)) : TmemShape{T::NS, 1};
    const int JT = T::JT * sh.jps, JC = T::JC * sh.jps;
    if (TMEM) {
        if (T::WARPS == 8) a.KC = a.KD;  // the 16-warp plan keeps its planned stage size (k-chunks)
        a.n_tail = tmem_tail(a.n_tail);
    }

    a.n_ichunks = ls::ceil_div(a.N1, T::IC);
    a.n_units = a.n_ichunks * (a.k1 - a.k0);
    a.n_jc = ls::ceil_div(a.N2, JC);
    a.n_jt = a.n_jc * JT;
    a.n_kc = static_cast<int>(ls::ceil_div(a.KD, a.KC));
    // 32-bit counters inside the kernel
    if (a.n_units * a.n_jc * a.n_kc >= (int64_t(1) << 31) || a.N1 + T::IC >= (int64_t(1) << 31) ||
        a.N2 + JC >= (int64_t(1) << 31))
        return ls::fail(LS_EGUARD, "expand: grid too large for one launch (split the slab range)");
    // Pack A2 once per call (stream-ordered scratch from the pool, freed on every exit path).
    const size_t stage_elems = static_cast<size_t>(JT) * a.KC * 32 + static_cast<size_t>(JT) * 8 * a.n_tail;
    const size_t bp_elems = static_cast<size_t>(a.n_kc) * a.n_jc * stage_elems;
    const size_t s_elems = TMEM ? static_cast<size_t>(a.k1) * a.R : 0;
    ls::ensure_pool();
    ls::AsyncScratch scratch(s);
    LS_CUDA(scratch.alloc((bp_elems + s_elems) * sizeof(double)));
    double* bp = scratch.as<double>();
    a.S = TMEM ? bp + bp_elems : nullptr;
    const int64_t pb = std::min<int64_t>(ls::ceil_div(static_cast<int64_t>(bp_elems + s_elems), 256), 4096);
    LS_CUDA(ls::launch_pdl(pack_b_kernel, dim3((unsigned)pb), dim3(256), 0, s, a.B, a.ldb, a.N2, a.R, a.KD,
                           a.n_tail, a.KC, a.n_kc, JT, a.n_jc, bp, a.w, a.C, a.ldc, a.k1, const_cast<double*>(a.S)));
    LS_LAUNCHED("pack_b_kernel");
    a.Bp = bp;
    const size_t smem =
        TMEM ? sizeof(double) * (kTmemHdr + tmem_stg_elems(T::WARPS) + sh.ns * stage_elems) : smem_bytes<T>(a.KD, a.KC, a.n_tail);
    void (*kern)(ExpandArgs) = nullptr;
    if constexpr (!TMEM) {
        kern = expand_dmma_kernel<T, STORE, FUNC>;
    } else {
        const int code = 10 * sh.ns + sh.jps;
        if (a.n_tail != 1 && !(a.n_tail == 2 && T::WARPS == 8))
            return ls::fail(LS_EVALIDATION, "expand: TMEM plan needs one DFMA rank (two with 8 warps)");
        if constexpr (T::WARPS == 16) {
            static_assert(T::NS == 2, "the 16-warp TMEM kernels are built with a 2-deep ring");
            kern = a.KD >= 31 ? tmem16s_kernel(STORE, FUNC, a.KD) : tmem16_kernel(STORE, FUNC, a.KD, a.KC);
            if (!kern) return ls::fail(LS_EVALIDATION, "expand: unsupported 16-warp TMEM shape");
        } else {
            kern = tmem8_kernel(STORE, FUNC, code, a.KD, a.n_tail);
            if (!kern) return ls::fail(LS_EVALIDATION, "expand: unsupported TMEM shape");
        }
    }
    int per_sm = 0;
    if (const int rc = kernel_setup(reinterpret_cast<const void*>(kern), T::WARPS * 32, smem, per_sm)) return rc;
    if (per_sm < 1) return ls::fail(LS_EGUARD, "expand: tile does not fit on an SM");
    // The occupancy query under-reports the tcgen05 kernel (1 instead of 2 CTAs/SM although
    // registers, shared memory and the 2 x 256 TMEM columns all fit two); use the launch bound.
    if (TMEM) per_sm = T::MINB;
    int64_t grid = std::min<int64_t>(a.n_units, (int64_t)ls::sm_count() * per_sm);
    // Store-only TMEM launches may split their last round of units at stage granularity
    // (expand_tmem.cuh) when that shortens the busiest CTA by more than one unit fill: cfg1 goes
    // from 28 units (448 stages) to 27 units + 11 stages (+0.45% measured); at 512^3 it would
    // not help (56 stages either way) and the extra partial-unit fills cost 1.6%.
    a.split_tail = 0;
    if (TMEM && STORE && !FUNC) {
        const int64_t G = (int64_t)ls::sm_count() * per_sm;
        const int64_t full = a.n_units / G, tail = a.n_units - full * G;
        const int64_t whole = ls::ceil_div(a.n_units, G) * a.n_jc;
        const int64_t split = full * a.n_jc + ls::ceil_div(tail * a.n_jc, G);
        const bool force = ls::dev_knob("LS_SPLIT_ALL") != nullptr;  // lab A/B
        if (tail > 0 && (split + 2 <= whole || force) && a.n_kc == 1) {
            a.split_tail = 1;
            grid = std::min<int64_t>(a.n_units * a.n_jc, G);
        }
    }
    if (ls::dev_knob("LS_EXPAND_VERBOSE"))
        std::fprintf(stderr, "ls_expand: tile %dx%d warps, IC %d, KC %d/%d, smem %zu B, %d CTA/SM, grid %lld, %s\n",
                     T::WARPS, T::WI, T::IC, a.KC, a.KD, smem, per_sm, static_cast<long long>(grid),
                     TMEM ? "A1k in TMEM" : "A1k in smem");
    if (grid > 0) {
        LS_CUDA(ls::launch_pdl(kern, dim3((unsigned)grid), dim3(T::WARPS * 32), smem, s, a));
        LS_LAUNCHED("expand_dmma_kernel");
    }
    return LS_OK;
}

#ifdef LS_TIMELINE
// Lab builds only: the event log of the last instrumented launch (see k3.cuh).
constexpr size_t kLabTimelineBytes = size_t(148) * 2 * 16 * 128 * sizeof(unsigned long long);
unsigned long long* lab_timeline() {
    static unsigned long long* p = nullptr;
    if (!p) cudaMalloc(&p, kLabTimelineBytes);
    return p;
}
#endif

constexpr int kRankChunk = 256;

bool chunk_plan(Plan& out) {
    int KD, n_tail;
    split_rank(kRankChunk, KD, n_tail);
    return plan_for(KD, n_tail, out);
}

template <bool STORE, bool FUNC>
int launch_plan(const Plan& pl, ExpandArgs& a, cudaStream_t s) {
    if (pl.pad && a.n_tail == 2) {
        a.KD += 1;
        a.n_tail = 0;
    }
    a.KC = std::min(pl.KC, a.KD);
    switch (pl.id) {
        case kPlanTmem: return launch<TileWide, STORE, FUNC, true>(a, s);
        case kPlanTmem16:
        case kPlanTmem16S: return launch<TileTmem16, STORE, FUNC, true>(a, s);
        case kPlanSplitK:
            // No zero DFMA rank when R mod 4 == 0 (unlike the TMEM plans): the pair's halves then
            // carry equal work, 0.8% at cfg3 and 1.6-2.4% at ranks 176-240.
            return launch_splitk(a, STORE, FUNC, s, ls::sm_count(), kernel_setup);
        case 0: return launch<TileWide, STORE, FUNC>(a, s);
        case 1: return launch<TileWide3, STORE, FUNC>(a, s);
        case 2: return launch<TileMid, STORE, FUNC>(a, s);
        case 6: return launch<TileLR1, STORE, FUNC>(a, s);
        case 7: return launch<TileLR2, STORE, FUNC>(a, s);
        case 8: return launch<TileLR1b, STORE, FUNC>(a, s);
        case 9: return launch<TileLR16, STORE, FUNC>(a, s);
        default: return launch<TileNarrow, STORE, FUNC>(a, s);
    }
}

#ifdef LS_TIMELINE
}  // namespace
extern "C" int ls_lab_timeline(unsigned long long* host, int64_t n) {
    const size_t bytes = std::min<size_t>(kLabTimelineBytes, size_t(n) * sizeof(unsigned long long));
    LS_CUDA(cudaMemcpy(host, lab_timeline(), bytes, cudaMemcpyDeviceToHost));
    return LS_OK;
}
namespace {
#endif

// The small-N2 plan (expand_a2t.cu) takes a launch whenever it fits: A2 in TMEM for the whole
// launch, no per-unit fill, 64-row units (256^3: 56.3 -> see DESIGN section 3).
bool use_a2t(int64_t N2, int KD, int n_tail) {
    return fits_a2t(N2, KD, tmem_tail(n_tail)) && !ls::dev_knob("LS_NO_A2T");
}

}  // namespace

extern "C" int64_t ls_expand_partial_count(int64_t N1, int64_t N2, int R, int64_t k0, int64_t k1) {
    int KD, n_tail;
    split_rank(std::max(R, 1), KD, n_tail);
    Plan pl;
    if (k1 < k0) return -1;
    if (use_a2t(N2, KD, n_tail)) return a2t_units(N1, k0, k1) * 8;  // one partial per warp and unit
    if (!plan_for(KD, n_tail, pl) && !chunk_plan(pl)) return -1;
    const int64_t IC = pl.ic;
    // the TMEM variant writes one partial per warp (no CTA barrier per unit)
    return ls::ceil_div(N1, IC) * (k1 - k0) * (pl.id == kPlanTmem ? 8 : pl.id == kPlanTmem16 || pl.id == kPlanTmem16S || pl.id == kPlanSplitK ? 16 : 1);
}

extern "C" int ls_expand_plan_name(int R, char* out, int len) {
    if (R < 0 || !out || len < 1) return ls::fail(LS_EVALIDATION, "expand_plan_name: bad arguments");
    int KD, n_tail;
    split_rank(std::max(R, 1), KD, n_tail);
    Plan pl;
    const bool whole = plan_for(KD, n_tail, pl);
    if (!whole && !chunk_plan(pl)) return ls::fail(LS_EGUARD, "expand_plan_name: no tile plan");
    const int kd = pl.pad && n_tail == 2 ? KD + 1 : KD;
    const int nt = pl.id == kPlanTmem || pl.id == kPlanTmem16 || pl.id == kPlanTmem16S ? (pl.pad ? 1 : tmem_tail(n_tail))
                                                                                    : n_tail;
    const char* shape = pl.id == kPlanTmem     ? "expand_tmem_kernel, 8 warps x 2 CTAs/SM, A1k in TMEM"
                        : pl.id == kPlanTmem16 ? "expand_tmem_kernel, 16 warps x 1 CTA/SM, A1k in TMEM"
                        : pl.id == kPlanTmem16S ? "expand_tmem_kernel, 16 warps x 1 CTA/SM, single A1k buffer in TMEM"
                        : pl.id == kPlanSplitK ? "expand_splitk_kernel, 16 warps x 1 CTA/SM, A1k halves in TMEM lane quarters"
                        : pl.id == 9           ? "expand_dmma_kernel TileLR16, 16 warps x 1 CTA/SM, A1k in smem"
                                               : "expand_dmma_kernel, A1k in smem";
    std::snprintf(out, static_cast<size_t>(len), "%s; plan %d, KD %d (%s), %d DFMA rank(s)%s", shape, pl.id, kd,
                  (pl.id == kPlanTmem && kd <= 14) || (pl.id == kPlanTmem16 && kd >= 14 && kd <= 23)
                      ? "compiled"
                      : (pl.id == kPlanTmem16 && kd >= 24 && kd <= 30 ? "compiled, two stages per tile"
                         : pl.id == kPlanTmem16S                        ? "compiled, k-chunked stages"
                                                                        : "runtime"),
                  nt, whole ? "" : ", 256-rank chunks");
    return LS_OK;
}

extern "C" int ls_expand(const double* A_d, int64_t lda, const double* B_d, int64_t ldb,
                         const double* C_d, int64_t ldc, const double* w_d, int64_t N1, int64_t N2,
                         int64_t N3, int R, int64_t k0, int64_t k1, double* out_d, int64_t ldy,
                         int64_t ldz, const double* rho1_d, const double* rho2_d,
                         const double* rho3_d, double* partial_d, void* stream) {
    if (N1 < 0 || N2 < 0 || N3 < 0 || R < 0)
        return ls::fail(LS_EVALIDATION, "expand: negative dimension or rank");
    if (k0 < 0 || k1 > N3 || k0 > k1) return ls::fail(LS_EVALIDATION, "expand: slab range outside [0, N3]");
    if (lda < N1 || ldb < N2 || ldc < N3) return ls::fail(LS_EVALIDATION, "expand: leading dimension too small");
    if (ldy == 0) ldy = N1;
    if (ldz == 0) ldz = ldy * N2;
    if (ldy < N1 || ldz < ldy * N2) return ls::fail(LS_EVALIDATION, "expand: output strides too small");
    const bool func = rho1_d != nullptr;
    if (func && (!rho2_d || !rho3_d || !partial_d))
        return ls::fail(LS_EVALIDATION, "expand: functional epilogue needs rho1, rho2, rho3 and partial");
    if (!out_d && !func) return ls::fail(LS_EVALIDATION, "expand: nothing to do (no output, no functional)");
    if (N1 == 0 || N2 == 0 || k1 == k0) return LS_OK;
    const cudaStream_t s = ls::as_stream(stream);
    if (R == 0) {
        // Rank-0 tensor is the zero tensor (canonical.hpp:243).
        if (out_d)
            for (int64_t kk = 0; kk < k1 - k0; ++kk)
                LS_CUDA(cudaMemset2DAsync(out_d + kk * ldz, ldy * sizeof(double), 0, N1 * sizeof(double), N2, s));
        if (func) LS_CUDA(cudaMemsetAsync(partial_d, 0, sizeof(double) * ls_expand_partial_count(N1, N2, 4, k0, k1), s));
        return LS_OK;
    }
    ExpandArgs a{};
    a.A = A_d; a.B = B_d; a.C = C_d; a.w = w_d;
    a.lda = lda; a.ldb = ldb; a.ldc = ldc;
    a.N1 = N1; a.N2 = N2; a.N3 = N3;
    a.R = R;
    split_rank(R, a.KD, a.n_tail);
    a.k0 = k0; a.k1 = k1;
    a.out = out_d; a.ldy = ldy; a.ldz = ldz;
    a.vec_store = (ldy % 2 == 0 && ldz % 2 == 0 && (reinterpret_cast<uintptr_t>(out_d) & 15) == 0) ? 1 : 0;
    a.rho1 = rho1_d; a.rho2 = rho2_d; a.rho3 = rho3_d; a.partial = partial_d;
    if (const char* dbg = ls::dev_knob("LS_EXPAND_DEBUG")) a.debug = std::atoi(dbg);
    a.fault = ls::fault_flag();
    if (a.fault == nullptr) return ls::fail(LS_ECUDA, "expand: no CUDA device");
#ifdef LS_TIMELINE
    if (ls::dev_knob("LS_TIMELINE")) {
        LS_CUDA(cudaMemsetAsync(lab_timeline(), 0, kLabTimelineBytes, s));
        a.timeline = lab_timeline();
    }
#endif
    const bool store = out_d != nullptr;
    if (use_a2t(N2, a.KD, a.n_tail)) {
        a.n_tail = tmem_tail(a.n_tail);
        return launch_a2t(a, store, func, s, ls::sm_count(), kernel_setup);
    }
    Plan pl;
    if (plan_for(a.KD, a.n_tail, pl)) {
        if (store && func) return launch_plan<true, true>(pl, a, s);
        if (store) return launch_plan<true, false>(pl, a, s);
        return launch_plan<false, true>(pl, a, s);
    }
    // Ranks beyond one shared-memory tile (e.g. direct sums, rank M0 * cells * R): expand
    // kRankChunk ranks at a time with one tile plan (so partial-sum units line up), the first
    // chunk writing and later chunks accumulating.
    Plan pc;
    if (!chunk_plan(pc)) return ls::fail(LS_EGUARD, "expand: no tile plan for rank chunks");
    for (int r0 = 0; r0 < R; r0 += kRankChunk) {
        const int rc = std::min(kRankChunk, R - r0);
        ExpandArgs c = a;
        c.A = A_d + lda * r0;
        c.B = B_d + ldb * r0;
        c.C = C_d + ldc * r0;
        c.w = w_d + r0;
        c.R = rc;
        split_rank(rc, c.KD, c.n_tail);
        c.accumulate = r0 > 0 ? 1 : 0;
        c.vec_store = a.vec_store;
        if (c.KC > c.KD) c.KC = c.KD;
        int rc_status;
        if (store && func)
            rc_status = launch_plan<true, true>(pc, c, s);
        else if (store)
            rc_status = launch_plan<true, false>(pc, c, s);
        else
            rc_status = launch_plan<false, true>(pc, c, s);
        if (rc_status != LS_OK) return rc_status;
    }
    return LS_OK;
}

extern "C" int ls_sum_partials(const double* partial_d, int64_t count, double* out_d, void* stream) {
    if (count < 0) return ls::fail(LS_EVALIDATION, "sum_partials: negative count");
    sum_partials_kernel<<<1, 1024, 0, ls::as_stream(stream)>>>(partial_d, count, out_d);
    LS_LAUNCHED("sum_partials_kernel");
    return LS_OK;
}
