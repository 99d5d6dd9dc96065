// expand_tmem16.cu -- instantiations of the 16-warp TMEM expansion kernel (expand_tmem.cuh),
// in their own translation unit so they compile in parallel with expand.cu.
#include <utility>

#include "expand_tmem.cuh"

namespace ls_k3 {
namespace {

// Compile-time k-step count over the range the 16-warp plan covers (KD 15..23), 2-deep ring.
template <bool STORE, bool FUNC, int... KD>
KernelFn pick(int kd, std::integer_sequence<int, KD...>) {
    KernelFn k = nullptr;
    ((kd == KD + 15 ? (k = expand_tmem_kernel<STORE, FUNC, 2, 1, 16, KD + 15>, 0) : 0), ...);
    return k;
}

template <bool STORE, bool FUNC>
KernelFn kernel(int kd) {
    if (KernelFn k = pick<STORE, FUNC>(kd, std::make_integer_sequence<int, 9>{})) return k;
    return expand_tmem_kernel<STORE, FUNC, 2, 1, 16>;
}

}  // namespace

KernelFn tmem16_kernel(bool store, bool func, int kd) {
    if (store && func) return kernel<true, true>(kd);
    if (store) return kernel<true, false>(kd);
    if (func) return kernel<false, true>(kd);
    return nullptr;
}

}  // namespace ls_k3
