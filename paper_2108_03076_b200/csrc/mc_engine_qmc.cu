// The QMC path kernels of the ahead-of-time build (see mc_engine.cu).
#define CLTK_AOT_PART 1
#include "mc_engine.cu"
