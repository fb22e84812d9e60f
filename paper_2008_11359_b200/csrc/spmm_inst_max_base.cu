// spmm_inst_max_base.cu -- gSpMM instantiations: reducer max, copy_u / u_mul_e.
#define FG_RED R_MAX
#define FG_OPSET 0
#include "spmm_inst.cuh"
