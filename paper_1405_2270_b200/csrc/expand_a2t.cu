// expand_a2t.cu -- the A2-in-TMEM expansion plan (expand_a2t.cuh): one-DFMA-rank kernels, the
// pre-pass and the host side.
#define LS_A2T_PART 0
#include "expand_a2t.cuh"
