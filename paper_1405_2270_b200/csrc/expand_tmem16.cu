// expand_tmem16.cu -- instantiations of the 16-warp TMEM expansion kernel (expand_tmem.cuh),
// in their own translation unit so they compile in parallel with expand.cu.
#include <utility>

#include "expand_tmem.cuh"

namespace ls_k3 {
namespace {

// Compile-time k-step count over the range the 16-warp plan covers with whole-rank stages
// (KD 14..23; 14 for rank 54, whose 2-rank remainder the 8-warp plan cannot hold), 2-deep ring.
template <bool STORE, bool FUNC, int... KD>
KernelFn pick(int kd, std::integer_sequence<int, KD...>) {
    KernelFn k = nullptr;
    ((kd == KD + 14 ? (k = expand_tmem_kernel<STORE, FUNC, 2, 1, 16, KD + 14>, 0) : 0), ...);
    return k;
}

// KD 24..30: two stages of ceil(KD / 2) k-steps per tile.
template <bool STORE, bool FUNC, int... KD>
KernelFn pick_chunked(int kd, std::integer_sequence<int, KD...>) {
    KernelFn k = nullptr;
    ((kd == KD + 24 ? (k = expand_tmem_kernel<STORE, FUNC, 2, 1, 16, KD + 24, 1, (KD + 25) / 2>, 0) : 0), ...);
    return k;
}

template <bool STORE, bool FUNC>
KernelFn kernel(int kd, int kc) {
    if (kc < kd) return kc == (kd + 1) / 2 ? pick_chunked<STORE, FUNC>(kd, std::make_integer_sequence<int, 7>{}) : nullptr;
    if (KernelFn k = pick<STORE, FUNC>(kd, std::make_integer_sequence<int, 10>{})) return k;
    return expand_tmem_kernel<STORE, FUNC, 2, 1, 16>;
}

}  // namespace

KernelFn tmem16_kernel(bool store, bool func, int kd, int kc) {
    if (store && func) return kernel<true, true>(kd, kc);
    if (store) return kernel<true, false>(kd, kc);
    if (func) return kernel<false, true>(kd, kc);
    return nullptr;
}

}  // namespace ls_k3
