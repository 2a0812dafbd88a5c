// Backward half of preprocess.cu (k_pre2d_bwd, k_pre3d_bwd[_exact], k_sh_bwd
// and their launchers), compiled WITH FMA contraction: only the forward's FP64
// must round exactly as written (rects bit-exact with the oracle); the
// backward is compared with a tolerance, and contraction shortens its FP64
// dependency chains. preprocess.cu itself (--fmad=false) holds the forward.
#define WIPES_PRE_BWD_TU 1
#include "preprocess.cu"
