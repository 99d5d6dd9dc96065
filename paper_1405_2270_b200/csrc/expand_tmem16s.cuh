// expand_tmem16s.cuh -- instantiations of the single-buffer 16-warp TMEM expansion kernel
// (SINGLE_ in expand_tmem.cuh) for KD 31..62 (ranks 122..249): one A1k buffer of up to 512
// TMEM columns, NKC stages of KC k-steps per tile through the 2-deep ring. Split over two
// translation units (expand_tmem16s_a.cu, _b.cu) so they compile in parallel.
#pragma once

#include <utility>

#include "expand_tmem.cuh"

namespace ls_k3 {

template <bool STORE, bool FUNC, int LO, int... KD>
KernelFn pick_tmem16s(int kd, std::integer_sequence<int, KD...>) {
    KernelFn k = nullptr;
    ((kd == KD + LO ? (k = expand_tmem_kernel<STORE, FUNC, 2, 1, 16, KD + LO, 1, tmem16s_kc(KD + LO),
                                              tmem16s_nkc(KD + LO), true>,
                       0)
                    : 0),
     ...);
    return k;
}

}  // namespace ls_k3
