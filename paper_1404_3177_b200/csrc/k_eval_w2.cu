// Part 2 of the team-mapping pass-1 instantiations (see k_eval_w.cu): f / 2 = 6 .. 8.
#define MNL_W_PART 2
#include "k_eval_w.cu"
