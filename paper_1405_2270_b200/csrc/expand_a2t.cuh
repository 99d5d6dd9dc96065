// expand_a2t.cuh -- K3 for small N2: the right factor A2 resident in TMEM for the whole launch,
// the scaled left factor A1k streamed through the shared-memory ring.
//
// The TMEM kernels (expand_tmem.cuh) keep A1k(i, q) = A1(i, q) * S(k, q) of one (i-chunk, slab)
// unit in TMEM and stream A2 through the ring; each unit's A1k is rebuilt by the warps (loads,
// products, TMEM stores). With N2 = 256 a unit is only 4 ring stages, so that fill is ~10% of the
// time, and the 512 units of a 256^3 grid on 296 CTAs leave the SMs with 4 units setting the
// pace. Here the roles swap: all of A2 (N2 <= 256 at ranks <= 57) sits in TMEM, loaded once per
// CTA, and a unit is a 64-row i-chunk of ONE slab. Its operand stage is the i-chunk's A1 in
// MMA-fragment order (a pre-pass packs the few distinct i-chunks once, pack_a1_kernel) plus the
// slab's scale row S(k, q) = w_q * A3(k, q): two TMA bulk copies per unit, both L2-resident.
// The landed A1 is scaled in place once (A1k = A1 * S, the rounding of the TMEM kernel's fill),
// each warp of a 64-row half scaling one quarter of it (its nn = wj rows), handed over by a
// per-(slot, half) mbarrier. So there is no per-unit TMEM fill, the units are half as large (1024
// at 256^3: 6.9 per SM, at most 7), and the DMMAs see exactly the operands of the TMEM kernel in
// the same order: the grid is bit-identical to it.
//
// Schedule: one CTA of 8 warps per SM (two warps per sub-partition keep the DMMA pipe as busy as
// four: tools/microbench/fp64_peak.cu, 36.9 TF/s), which leaves each thread the registers for
// TWO accumulator sets. A warp's work is a sequence of items (unit, j-chunk); item x's DMMAs go
// into one set while item x-1's stores are spread over x's k-steps, the next unit's share of the
// scaling is spread over chunk 0's k-steps, and the TMEM loads run one k-step ahead. (Against
// 2 CTAs x 8 warps with one set and those steps between the chunks: 51.8 -> 50.3 us at 256^3,
// and R = 57 at 256^3: 76.9 -> 69.3 us.)
//
// TMEM layout (per CTA, 256 or 512 columns, lanes = quarter wj = warp & 3 = the warp's j block):
//   chunk c (128 j), column c*CBJ + 8 ks + 2 m + {0,1}: A2(j = 128 c + 32 wj + 8 m + g, q = 4 ks + t)
//   column c*CBJ + 8 KD + 8 qt + 2 m + {0,1}: A2(j = ..., q = 4 KD + qt) (DFMA tail ranks)
//   CBJ = 8 KD + 8 NT; n_jc chunks need n_jc * CBJ <= 512.
// Ring slot (per unit (ic, k), shared memory): the i-chunk's packed A1
//   [wi][ks][nn][lane] = A1(i = 64 ic + 32 wi + 8 nn + g, q = 4 ks + t), then
//   [wi][qt][e][lane]  = A1(i = 64 ic + 32 wi + 8 (e >> 1) + 2 t + (e & 1), q = 4 KD + qt),
// then the scale row S(k, 0 .. SR) (zero beyond R).
//
// Compiled as two translation units so the kernel table builds in parallel: expand_a2t.cu
// (LS_A2T_PART 0: one DFMA rank, the pre-pass and the host side) and expand_a2t_b.cu
// (LS_A2T_PART 1: the two-DFMA-rank kernels, reached through a2t_kernel_nt2).
#include <type_traits>
#include <utility>

#include "common.cuh"
#include "expand_tmem.cuh"

#ifndef LS_A2T_PART
#error "include from expand_a2t.cu / expand_a2t_b.cu with LS_A2T_PART defined"
#endif

namespace ls_k3 {
namespace {

constexpr int kA2tWarps = 8, kA2tIC = 64, kA2tJC = 128, kA2tNS = 4, kA2tHdr = 48;
// At most 2 j-chunks (N2 <= 256; tools/lab/a2t_vs_tmem.py, profiles/r02_a2t_vs_tmem.txt): at
// N2 = 256 this plan takes 26.1 / 33.7 / 51.5 / 69.3 us at R = 9 / 21 / 41 / 57 against the TMEM
// plan's 30.7 / 35.4 / 58.0 / 77.1 us (256^3); at N2 = 512 the two are within 1.5% either way, and
// beyond, the TMEM plan wins.
constexpr int kA2tMaxJC = 2;

__host__ __device__ constexpr int a2t_stage_elems(int KD, int NT) { return 2 * KD * 128 + 2 * NT * 256; }
// scale-row length, padded to whole 16-byte TMA chunks
__host__ __device__ constexpr int a2t_srow(int KD, int NT) { return (4 * KD + NT + 1) / 2 * 2; }

// Pre-pass: the packed A1 of every 64-row i-chunk (n_ichunks stages, MMA-fragment order), and
// the scale rows S[kk][q] = w_q * A3(k0 + kk, q) of slabs [k0, k1) (pack_b_kernel's rounding),
// zero beyond R. Small: at 256^3 four stages of 24 KB and 256 rows of 42 doubles.
__global__ void pack_a1_kernel(const double* __restrict__ A, int64_t lda, int64_t N1, const double* __restrict__ w,
                               const double* __restrict__ C, int64_t ldc, int R, int KD, int NT, int64_t k0,
                               int64_t n_slabs, int64_t n_ichunks, double* __restrict__ a1p, double* __restrict__ srows) {
    pdl_wait();  // A, C, w may come from the preceding assembly / generator launches
    pdl_trigger();
    const int se = a2t_stage_elems(KD, NT), frag = 2 * KD * 128, sr = a2t_srow(KD, NT);
    const int64_t n_a = n_ichunks * se, n_s = n_slabs * sr;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n_a + n_s; x += (int64_t)gridDim.x * blockDim.x) {
        if (x >= n_a) {
            const int64_t y = x - n_a, kk = y / sr;
            const int q = static_cast<int>(y - kk * sr);
            srows[y] = q < R ? rn_mul(w[q], C[k0 + kk + ldc * q]) : 0.0;
            continue;
        }
        const int64_t ic = x / se;
        const int o = static_cast<int>(x - ic * se), r = o >> 5, lane = o & 31, g = lane >> 2, t = lane & 3;
        int64_t i;
        int q;
        if (o < frag) {  // r = (wi * KD + ks) * 4 + nn
            const int nn = r & 3, wk = r >> 2, wi = wk / KD, ks = wk - wi * KD;
            i = kA2tIC * ic + 32 * wi + 8 * nn + g;
            q = 4 * ks + t;
        } else {  // r - frag / 32 = (wi * NT + qt) * 8 + e
            const int rr = r - (frag >> 5), e = rr & 7, wq = rr >> 3, wi = wq / NT, qt = wq - wi * NT;
            i = kA2tIC * ic + 32 * wi + 8 * (e >> 1) + 2 * t + (e & 1);
            q = 4 * KD + qt;
        }
        a1p[x] = (i < N1 && q < R) ? A[i + lda * q] : 0.0;
    }
}

template <bool STORE, bool FUNC, int KD, int NT>
__global__ void __launch_bounds__(kA2tWarps * 32, 1) expand_a2t_kernel(const ExpandArgs p) {
    constexpr int kThreads = kA2tWarps * 32, kNS = kA2tNS, kTM = 4, kTN = 4;
    constexpr int CBJ = 8 * KD + 8 * NT;
    constexpr int kA1 = a2t_stage_elems(KD, NT), kSR = a2t_srow(KD, NT);
    constexpr int kStage = kA1 + kSR;  // ring slot: packed A1 of the unit's i-chunk, then its slab's scale row
    constexpr int kFrag = 2 * KD * 128;
    constexpr unsigned kA1Bytes = kA1 * sizeof(double), kSRBytes = kSR * sizeof(double);
    extern __shared__ __align__(128) double smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);        // [kNS]
    int* released = reinterpret_cast<int*>(smem + 8);           // [kNS]
    uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(smem + 16);
    uint64_t* scaled = reinterpret_cast<uint64_t*>(smem + 20);  // [kNS][2]: slot's half scaled by its 4 warps
    uint64_t* a2r = reinterpret_cast<uint64_t*>(smem + 32);     // [kA2tMaxJC][4]: A2 chunk c of quarter q in TMEM
    double* ring = smem + kA2tHdr;                              // [kNS][kStage]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int wj = warp & 3;   // j block within a 128-j chunk, and the TMEM lane quarter
    const int wi = warp >> 2;  // i half of the 64-row unit
    const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
    const int n_units = static_cast<int>(p.n_units), n_ichunks = static_cast<int>(p.n_ichunks);
    const int n_jc = static_cast<int>(p.n_jc);
    const uint32_t tmem_cols = n_jc * CBJ <= 256 ? 256u : 512u;  // one CTA per SM: all 512 if needed
    const int my_units = n_units > b ? (n_units - 1 - b) / G + 1 : 0;
    LS_TL_INIT();
#ifdef LS_DEV_KNOBS
    const bool lab_noscale = (p.debug & 2) != 0;  // lab A/B: operands used unscaled (no DMULs)
    const bool lab_nostore = (p.debug & 1) != 0;  // lab A/B: epilogue without stores
#else
    constexpr bool lab_noscale = false, lab_nostore = false;
#endif

    auto issue = [&](int n) {  // this CTA's n-th unit into slot n % kNS
        const int u = b + n * G;
        uint64_t* bar = full + (n % kNS);
        double* dst = ring + (n % kNS) * kStage;
        mbar_arrive_expect_tx(bar, kA1Bytes + kSRBytes);
        tma_bulk_g2s(dst, p.Bp + static_cast<int64_t>(u % n_ichunks) * kA1, kA1Bytes, bar);
        tma_bulk_g2s(dst + kA1, p.S + static_cast<int64_t>(u / n_ichunks) * kSR, kSRBytes, bar);
    };
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_s)),
                     "r"(tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(scaled + 2 * s, 4);
            mbar_init(scaled + 2 * s + 1, 4);
            released[s] = 0;
        }
        for (int x = 0; x < 4 * kA2tMaxJC; ++x) mbar_init(a2r + x, 2);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const uint32_t tq = *tmem_base_s + (static_cast<uint32_t>(32 * wj) << 16);
    LS_TL(1);
    // The pre-pass (the preceding launch) writes the packed A1 and the scale rows, which only the
    // ring's TMA copies read; A2 was written before it (the pre-pass waits for that writer before
    // it lets this launch start). So one thread waits for the pre-pass and issues the first ring
    // stages while the warps load A2 (warp 7 loads the chunk needed last).
    if (threadIdx.x == kThreads - 1) {
        pdl_wait();
        for (int n = 0; n < kNS && n < my_units; ++n) issue(n);
    }

    // A2 into TMEM, once, chunk by chunk: the two warps of quarter wj split each chunk's k-steps
    // (ks = wi, wi + 2, ...), all of a warp's loads of both chunks in flight at once (256^3:
    // 50.9 -> 50.4 us against chunk by chunk); chunk c of quarter wj is handed over by a2r[c][wj]
    // (2 arrivals), so the first tiles wait for chunk 0 only.
    {
        constexpr int kHalf = (KD + NT + 1) / 2;
        double v[kA2tMaxJC][kHalf][4];  // every chunk's loads in flight before the first TMEM store
#pragma unroll
        for (int c = 0; c < kA2tMaxJC; ++c) {
            const int64_t jb = static_cast<int64_t>(kA2tJC) * c + 32 * wj + g;
#pragma unroll
            for (int x = 0; x < kHalf; ++x) {
                const int ks = 2 * x + wi;
                const int q = ks < KD ? 4 * ks + t : 4 * KD + (ks - KD);  // tail ranks: every t the same q
#pragma unroll
                for (int m = 0; m < kTM; ++m) {
                    const int64_t j = jb + 8 * m;
                    v[c][x][m] = (c < n_jc && ks < KD + NT && j < p.N2 && q < p.R) ? __ldg(p.B + j + p.ldb * q) : 0.0;
                }
            }
        }
#pragma unroll
        for (int c = 0; c < kA2tMaxJC; ++c) {
            if (c >= n_jc) break;
#pragma unroll
            for (int x = 0; x < kHalf; ++x) {
                const int ks = 2 * x + wi;
                if (ks < KD + NT) tmem::st_x8(tq + static_cast<uint32_t>(c * CBJ + 8 * ks), v[c][x]);
            }
            tmem::wait_st();
            tmem::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(a2r + 4 * c + wj);
        }
    }
    unsigned a2_ready = 0;  // chunks of A2 this warp has waited for
    LS_TL(2);

    // This warp's quarter of half wi of unit n's operands: A1k = A1 * S in place (rows nn = wj
    // of every k-step, tail rows e = wj, wj + 4), then the hand-over to the half's 4 warps.
    auto scale_share = [&](int n) {
        const int sl = n % kNS;
        mbar_wait(full + sl, static_cast<unsigned>((n / kNS) & 1), p.fault);
        double* st = ring + sl * kStage;
        if (lab_noscale) {
            __syncwarp();
            if (lane == 0) mbar_arrive(scaled + 2 * sl + wi);
            return;
        }
        const double* sr = st + kA1;
        double* fr = st + (wi * KD) * 128 + wj * 32 + lane;
#pragma unroll
        for (int ks = 0; ks < KD; ++ks) fr[ks * 128] = rn_mul(fr[ks * 128], sr[4 * ks + t]);
        double* tl = st + kFrag + (wi * NT) * 256 + wj * 32 + lane;
#pragma unroll
        for (int qt = 0; qt < NT; ++qt) {
            const double sq = sr[4 * KD + qt];
            tl[qt * 256] = rn_mul(tl[qt * 256], sq);
            tl[qt * 256 + 128] = rn_mul(tl[qt * 256 + 128], sq);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(scaled + 2 * sl + wi);
    };
    if (my_units > 0) scale_share(0);

    // Items x = (unit n = x / n_jc, j-chunk c = x % n_jc), in order. The accumulators ping-pong
    // between two register sets: item x's DMMAs go into one while the previous item's stores are
    // spread over x's k-steps (fast path), so the store data leaves the registers while the pipe
    // holds queued DMMAs instead of stalling the warp between chunks.
    const int n_items = my_units * n_jc;
    double fsum = 0.0;
    // An item's place in the grid, advanced from item to item without divisions (the item loop
    // used to divide by n_jc and n_ichunks twice per item: about 150 instructions with MUFU
    // latencies at the head of every item, with only two warps per sub-partition to hide them).
    struct Tile {
        int64_t kk;
        int n, c, unit, ic, ibase, jb;
        bool fast;
    };
    const int g_div = G / n_ichunks, g_mod = G - g_div * n_ichunks;
    auto place = [&](Tile& T) {
        T.ibase = kA2tIC * T.ic + 32 * wi;
        T.jb = kA2tJC * T.c + 32 * wj;
        T.fast = STORE && !FUNC && T.ibase + 8 * kTN <= p.N1 && T.jb + 8 * kTM <= p.N2 && p.vec_store && !p.accumulate;
    };
    auto first_tile = [&]() {
        Tile T;
        T.n = 0;
        T.c = 0;
        T.unit = b;
        T.kk = b / n_ichunks;
        T.ic = b - static_cast<int>(T.kk) * n_ichunks;
        place(T);
        return T;
    };
    auto next_tile = [&](const Tile& P) {
        Tile T = P;
        if (++T.c == n_jc) {
            T.c = 0;
            ++T.n;
            T.unit += G;
            T.kk += g_div;
            T.ic += g_mod;
            if (T.ic >= n_ichunks) {
                T.ic -= n_ichunks;
                ++T.kk;
            }
        }
        place(T);
        return T;
    };
    // Whole epilogue of an item (every path; the fast path is also spread into the next item).
    // Lane owns (j = jb + 8m + g, i = ibase + 8nn + 2t + {0,1}).
    auto epilogue = [&](const Tile& T, double (&acc)[kTM][kTN][2]) {
        double r1[kTN][2];
        if (FUNC) {
#pragma unroll
            for (int nn = 0; nn < kTN; ++nn)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = T.ibase + 8 * nn + 2 * t + e;
                    r1[nn][e] = i < p.N1 ? __ldg(p.rho1 + i) : 0.0;
                }
        }
#pragma unroll
        for (int m = 0; m < kTM; ++m) {
            const int j = T.jb + 8 * m + g;
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
            if (!STORE || lab_nostore) continue;
            double* row = p.out + T.kk * p.ldz + static_cast<int64_t>(j) * p.ldy;
#pragma unroll
            for (int nn = 0; nn < kTN; ++nn) {
                const int i = T.ibase + 8 * nn + 2 * t;
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
        if (FUNC && T.c == n_jc - 1) {
            // Per-warp partials: partial[unit * 8 + warp], fixed-order xor tree (as the TMEM kernel).
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, off);
            if (lane == 0) {
                const double part = rn_mul(fsum, p.rho3[p.k0 + T.kk]);
                double& sl = p.partial[static_cast<int64_t>(T.unit) * kA2tWarps + warp];
                sl = p.accumulate ? sl + part : part;
            }
            fsum = 0.0;
        }
    };
    // Item T into `cur`; P is the previous item (its accumulators in `prev`), if any.
    // maysc (a std::bool_constant): whether this call site can carry the next unit's scaling share
    // at all. With two j-chunks the items alternate chunk 0 / chunk 1 with the accumulator sets,
    // so the chunk-1 call site drops the (predicated-off, but issued) scaling instructions of
    // every k-step at compile time.
    auto item = [&](auto maysc, const Tile& T, const Tile& P, bool have_prev, double (&cur)[kTM][kTN][2],
                    double (&prev)[kTM][kTN][2]) {
        constexpr bool kMaySc = decltype(maysc)::value;
        const int n = T.n, c = T.c;
        const int slot = n % kNS;
        if (c == 0) {
            mbar_wait(scaled + 2 * slot + wi, static_cast<unsigned>((n / kNS) & 1), p.fault);
            LS_TL(3);
        }
        if (!((a2_ready >> c) & 1u)) {  // first use of chunk c: its TMEM columns of this quarter are written
            mbar_wait(a2r + 4 * c + wj, 0u, p.fault);
            tmem::fence_after();
            a2_ready |= 1u << c;
        }
        const double* stage = ring + slot * kStage;
        const double* bfr = stage + (wi * KD) * 128 + lane;          // A1k of k-step ks at [ks * 128 + nn * 32]
        const double* btl = stage + kFrag + (wi * NT) * 256 + lane;  // tail A1k: [qt * 256 + e * 32]
        const uint32_t ta = tq + static_cast<uint32_t>(c * CBJ);
        // The next unit's share of operand scaling (scale_share's work) is spread over chunk 0's
        // k-steps too: one product per k-step, the tail ranks with the last.
        const bool sc = kMaySc && c == 0 && n + 1 < my_units && !lab_noscale;
        double* fr1 = nullptr;
        const double* sr1 = nullptr;
        if (kMaySc && c == 0 && n + 1 < my_units) {
            const int sl1 = (n + 1) % kNS;
            mbar_wait(full + sl1, static_cast<unsigned>(((n + 1) / kNS) & 1), p.fault);
            double* st1 = ring + sl1 * kStage;
            sr1 = st1 + kA1;
            fr1 = st1 + (wi * KD) * 128 + wj * 32 + lane;
        }
        bool spread = false;
        double* prow = nullptr;
        if (have_prev) {
            spread = P.fast && !lab_nostore;
            prow = p.out + P.kk * p.ldz + static_cast<int64_t>(P.jb + g) * p.ldy + P.ibase + 2 * t;
        }
#pragma unroll
        for (int m = 0; m < kTM; ++m)
#pragma unroll
            for (int nn = 0; nn < kTN; ++nn) cur[m][nn][0] = cur[m][nn][1] = 0.0;
        // TMEM loads run one k-step ahead of the DMMAs (two register sets), so the load latency
        // hides behind the previous k-step's DMMA issue; the item's first load travels with the
        // tail operands.
        uint32_t ra[2][8], rt[NT][8];
#pragma unroll
        for (int qt = 0; qt < NT; ++qt) tmem::ld_x8_issue(ta + 8 * KD + 8 * qt, rt[qt]);  // A2 tail, j = 8 m + g
        tmem::ld_x8_issue(ta, ra[0]);
        // Rank remainder on DFMA before the DMMAs (as in the TMEM kernel).
#pragma unroll
        for (int qt = 0; qt < NT; ++qt) {
            double bt[8], at[4];
#pragma unroll
            for (int e = 0; e < 8; ++e) bt[e] = btl[qt * 256 + e * 32];  // A1k tail, i = 8 (e >> 1) + 2 t + (e & 1)
            tmem::wait_ld(rt[qt]);
            tmem::unpack(rt[qt], at);
#pragma unroll
            for (int nn = 0; nn < kTN; ++nn)
#pragma unroll
                for (int m = 0; m < kTM; ++m) {
                    cur[m][nn][0] = fma(bt[2 * nn], at[m], cur[m][nn][0]);
                    cur[m][nn][1] = fma(bt[2 * nn + 1], at[m], cur[m][nn][1]);
                }
        }
        tmem::wait_ld(ra[0]);
#pragma unroll
        for (int ks = 0; ks < KD; ++ks) {
            double a[kTM], bb[kTN], sv, ss;  // sv, ss: set and used under `sc` only (no zeroing per k-step)
            tmem::unpack(ra[ks & 1], a);
            if (ks + 1 < KD) tmem::ld_x8_issue(ta + 8 * (ks + 1), ra[(ks + 1) & 1]);
#pragma unroll
            for (int nn = 0; nn < kTN; ++nn) bb[nn] = bfr[ks * 128 + nn * 32];
            if (sc) {
                sv = fr1[ks * 128];
                ss = sr1[4 * ks + t];
            }
#pragma unroll
            for (int m = 0; m < kTM; ++m)
#pragma unroll
                for (int nn = 0; nn < kTN; ++nn) dmma_884(cur[m][nn][0], cur[m][nn][1], a[m], bb[nn]);
            if (ks + 1 < KD) tmem::wait_ld(ra[(ks + 1) & 1]);
            if (sc) {
                fr1[ks * 128] = rn_mul(sv, ss);
                if (ks == KD - 1) {
                    double* tl = fr1 - (wi * KD) * 128 + kFrag + (wi * NT) * 256;
#pragma unroll
                    for (int qt = 0; qt < NT; ++qt) {
                        const double sq = sr1[4 * KD + qt];
                        tl[qt * 256] = rn_mul(tl[qt * 256], sq);
                        tl[qt * 256 + 128] = rn_mul(tl[qt * 256 + 128], sq);
                    }
                }
            }
            if (spread) {  // pairs [16 ks / KD, 16 (ks + 1) / KD) of the previous item
#pragma unroll
                for (int q = kTM * kTN * ks / KD; q < kTM * kTN * (ks + 1) / KD; ++q)
                    __stcs(reinterpret_cast<double2*>(prow + 8 * (q / kTN) * p.ldy + 8 * (q % kTN)),
                           make_double2(prev[q / kTN][q % kTN][0], prev[q / kTN][q % kTN][1]));
            }
        }
        LS_TL(5);
        if (have_prev && !spread) epilogue(P, prev);  // the other paths, after this item's DMMAs are queued
        if (kMaySc && c == 0 && n + 1 < my_units) {  // unit n + 1's share is scaled: hand it over
            __syncwarp();
            if (lane == 0) mbar_arrive(scaled + 2 * ((n + 1) % kNS) + wi);
            LS_TL(6);
        }
        if (c == n_jc - 1) {
            // Release the ring slot (every operand of this unit has been read into registers);
            // the last warp refills it with this CTA's unit n + kNS.
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(released + slot, 1) == kA2tWarps - 1) {
                    released[slot] = 0;
                    __threadfence_block();
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    if (n + kNS < my_units) issue(n + kNS);
                }
            }
            LS_TL(9);
        }
    };
    double accA[kTM][kTN][2], accB[kTM][kTN][2];
    int x = 0;
    Tile Ta = first_tile(), Tb = Ta;  // Ta: the item going into accA; Tb: the one in accB
    constexpr std::true_type kSc{};
    constexpr std::false_type kNoSc{};
    if (n_jc == 2) {  // even items are chunk 0 (accA), odd items chunk 1 (accB)
        for (; x + 1 < n_items; x += 2) {
            item(kSc, Ta, Tb, x > 0, accA, accB);
            Tb = next_tile(Ta);
            item(kNoSc, Tb, Ta, true, accB, accA);
            Ta = next_tile(Tb);
        }
    } else {
        for (; x + 1 < n_items; x += 2) {
            item(kSc, Ta, Tb, x > 0, accA, accB);
            Tb = next_tile(Ta);
            item(kSc, Tb, Ta, true, accB, accA);
            Ta = next_tile(Tb);
        }
    }
    if (x < n_items) {
        item(kSc, Ta, Tb, x > 0, accA, accB);
        epilogue(Ta, accA);
    } else if (n_items > 0) {
        epilogue(Tb, accB);
    }
    LS_TL(7);
    LS_TL(8);
    LS_TL_END();
    tmem::fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base_s), "r"(tmem_cols) : "memory");
}

template <bool STORE, bool FUNC, int NT, int... KD>
KernelFn pick(int kd, std::integer_sequence<int, KD...>) {
    KernelFn k = nullptr;
    ((kd == KD + 1 ? (k = expand_a2t_kernel<STORE, FUNC, KD + 1, NT>, 0) : 0), ...);
    return k;
}

}  // namespace

// Two-DFMA-rank kernels (expand_a2t_b.cu).
KernelFn a2t_kernel_nt2(bool store, bool func, int kd);

#if LS_A2T_PART == 1
KernelFn a2t_kernel_nt2(bool store, bool func, int kd) {
    using S = std::make_integer_sequence<int, 14>;
    return store && func ? pick<true, true, 2>(kd, S{})
           : store       ? pick<true, false, 2>(kd, S{})
                         : pick<false, true, 2>(kd, S{});
}
#else
namespace {
template <bool STORE, bool FUNC>
KernelFn a2t_kernel(int kd, int nt) {
    using S = std::make_integer_sequence<int, 14>;
    return nt == 1 ? pick<STORE, FUNC, 1>(kd, S{}) : nt == 2 ? a2t_kernel_nt2(STORE, FUNC, kd) : nullptr;
}
}  // namespace

int a2t_smem_bytes(int KD, int NT) {
    return static_cast<int>(sizeof(double)) * (kA2tHdr + kA2tNS * (a2t_stage_elems(KD, NT) + a2t_srow(KD, NT)));
}

bool fits_a2t(int64_t N2, int KD, int NT) {
    if (KD < 1 || KD > 14 || NT < 1 || NT > 2) return false;
    const int64_t n_jc = (N2 + kA2tJC - 1) / kA2tJC;
    return n_jc <= kA2tMaxJC && n_jc * (8 * KD + 8 * NT) <= 512 && a2t_smem_bytes(KD, NT) + 1024 <= 228 * 1024;
}

int64_t a2t_units(int64_t N1, int64_t k0, int64_t k1) { return (N1 + kA2tIC - 1) / kA2tIC * (k1 - k0); }

// Launch for slabs [a.k0, a.k1): the pre-pass (packed A1 + scale rows), then the expansion.
// a.KD / a.n_tail are the plan's (n_tail in {1, 2}; q >= R is a zero rank).
int launch_a2t(ExpandArgs& a, bool store, bool func, cudaStream_t s, int sm_count,
               int (*setup)(const void*, int, size_t, int&)) {
    const int KD = a.KD, NT = a.n_tail;
    KernelFn kern = store && func ? a2t_kernel<true, true>(KD, NT)
                    : store       ? a2t_kernel<true, false>(KD, NT)
                                  : a2t_kernel<false, true>(KD, NT);
    if (!kern) return ls::fail(LS_EVALIDATION, "expand: unsupported A2-in-TMEM shape");
    const size_t smem = static_cast<size_t>(a2t_smem_bytes(KD, NT));
    int per_sm = 0;
    if (const int rc = setup(reinterpret_cast<const void*>(kern), kA2tWarps * 32, smem, per_sm)) return rc;
    const int64_t se = a2t_stage_elems(KD, NT), sr = a2t_srow(KD, NT);
    a.n_ichunks = (a.N1 + kA2tIC - 1) / kA2tIC;
    a.n_units = a.n_ichunks * (a.k1 - a.k0);
    a.n_jc = (a.N2 + kA2tJC - 1) / kA2tJC;
    if (a.n_units >= (int64_t(1) << 31)) return ls::fail(LS_EGUARD, "expand: grid too large for one launch");
    ls::ensure_pool();
    ls::AsyncScratch scratch(s);
    const int64_t n_a = a.n_ichunks * se, n_s = (a.k1 - a.k0) * sr;
    LS_CUDA(scratch.alloc(sizeof(double) * (n_a + n_s)));
    double* a1p = scratch.as<double>();
    double* srows = a1p + n_a;
    const int64_t pb = std::min<int64_t>((n_a + n_s + 255) / 256, 4096);
    LS_CUDA(ls::launch_pdl(pack_a1_kernel, dim3((unsigned)pb), dim3(256), 0, s, a.A, a.lda, a.N1, a.w, a.C, a.ldc,
                           a.R, KD, NT, a.k0, a.k1 - a.k0, a.n_ichunks, a1p, srows));
    LS_LAUNCHED("pack_a1_kernel");
    a.Bp = a1p;
    a.S = srows;
    int64_t grid = std::min<int64_t>(a.n_units, static_cast<int64_t>(sm_count) * per_sm);
    if (const char* g = ls::dev_knob("LS_A2T_GRID")) grid = std::min<int64_t>(a.n_units, std::atoll(g));
    if (grid > 0) {
        LS_CUDA(ls::launch_pdl(kern, dim3((unsigned)grid), dim3(kA2tWarps * 32), smem, s, a));
        LS_LAUNCHED("expand_a2t_kernel");
    }
    return LS_OK;
}

#endif  // LS_A2T_PART

}  // namespace ls_k3
