// expand_tmem16s_a.cu -- single-buffer 16-warp TMEM kernels for KD 31..45 (see expand_tmem16s.cuh).
#include "expand_tmem16s.cuh"

namespace ls_k3 {

KernelFn tmem16s_kernel_a(bool store, bool func, int kd) {
    using S = std::make_integer_sequence<int, 15>;
    if (store && func) return pick_tmem16s<true, true, 31>(kd, S{});
    if (store) return pick_tmem16s<true, false, 31>(kd, S{});
    if (func) return pick_tmem16s<false, true, 31>(kd, S{});
    return nullptr;
}

}  // namespace ls_k3
