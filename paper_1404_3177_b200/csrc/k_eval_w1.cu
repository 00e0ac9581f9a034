// Part 1 of the team-mapping pass-1 instantiations (see k_eval_w.cu): f / 2 = 3 .. 5.
#define MNL_W_PART 1
#include "k_eval_w.cu"
