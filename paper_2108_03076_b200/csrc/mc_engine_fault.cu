// The fault-hook test build of the Philox path kernels (see mc_engine.cu).
#define CLTK_AOT_PART 2
#include "mc_engine.cu"
