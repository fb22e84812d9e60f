// spmm_inst_min_base.cu -- gSpMM instantiations: reducer min, copy_u / u_mul_e.
#define FG_RED R_MIN
#define FG_OPSET 0
#include "spmm_inst.cuh"
