// expand_a2t_b.cu -- the A2-in-TMEM expansion plan (expand_a2t.cuh): the two-DFMA-rank kernels, in
// their own translation unit so they compile in parallel with expand_a2t.cu.
#define LS_A2T_PART 1
#include "expand_a2t.cuh"
