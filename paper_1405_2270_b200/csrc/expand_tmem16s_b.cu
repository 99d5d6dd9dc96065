// expand_tmem16s_b.cu -- single-buffer 16-warp TMEM kernels for KD 46..62 (see expand_tmem16s.cuh).
#include "expand_tmem16s.cuh"

namespace ls_k3 {

KernelFn tmem16s_kernel_b(bool store, bool func, int kd) {
    using S = std::make_integer_sequence<int, 17>;
    if (store && func) return pick_tmem16s<true, true, 46>(kd, S{});
    if (store) return pick_tmem16s<true, false, 46>(kd, S{});
    if (func) return pick_tmem16s<false, true, 46>(kd, S{});
    return nullptr;
}

}  // namespace ls_k3
