// expand_tmem8.cu -- instantiations of the 8-warp TMEM expansion kernel (expand_tmem.cuh),
// in their own translation unit so they compile in parallel with expand.cu.
#include <utility>

#include "expand_tmem.cuh"

namespace ls_k3 {
namespace {

// Compile-time k-step count for every KD the 8-warp plan covers (one DFMA rank: KD 1..14; two:
// KD 1..12), with the ring depth tmem_shape_for in expand.cu picks for it; other shapes
// (LS_EXPAND_TMEM) take the runtime-KD kernel.
template <bool STORE, bool FUNC, int NS, int NT, int LO, int... KD>
KernelFn pick(int kd, std::integer_sequence<int, KD...>) {
    KernelFn k = nullptr;
    ((kd == KD + LO ? (k = expand_tmem_kernel<STORE, FUNC, NS, 1, 8, KD + LO, NT>, 0) : 0), ...);
    return k;
}

template <bool STORE, bool FUNC>
KernelFn kernel(int code, int kd, int nt) {
    if (nt == 2) {  // two DFMA ranks: depth 4 up to KD 10, depth 3 for KD 11-12
        if (code == 41 && kd <= 10) return pick<STORE, FUNC, 4, 2, 1>(kd, std::make_integer_sequence<int, 10>{});
        if (code == 31 && kd >= 11 && kd <= 12) return pick<STORE, FUNC, 3, 2, 11>(kd, std::make_integer_sequence<int, 2>{});
        if (code == 41) return expand_tmem_kernel<STORE, FUNC, 4, 1, 8, 0, 2>;
        if (code == 31) return expand_tmem_kernel<STORE, FUNC, 3, 1, 8, 0, 2>;
        return nullptr;
    }
    if (nt != 1) return nullptr;
    if (code == 41 && kd <= 11) return pick<STORE, FUNC, 4, 1, 1>(kd, std::make_integer_sequence<int, 11>{});
    if (code == 31 && kd >= 12 && kd <= 14) return pick<STORE, FUNC, 3, 1, 12>(kd, std::make_integer_sequence<int, 3>{});
    if (code == 41) return expand_tmem_kernel<STORE, FUNC, 4, 1>;
    if (code == 31) return expand_tmem_kernel<STORE, FUNC, 3, 1>;
    if (code == 22) return expand_tmem_kernel<STORE, FUNC, 2, 2>;
    return nullptr;
}

}  // namespace

KernelFn tmem8_kernel(bool store, bool func, int code, int kd, int nt) {
    if (store && func) return kernel<true, true>(code, kd, nt);
    if (store) return kernel<true, false>(code, kd, nt);
    if (func) return kernel<false, true>(code, kd, nt);
    return nullptr;
}

}  // namespace ls_k3
